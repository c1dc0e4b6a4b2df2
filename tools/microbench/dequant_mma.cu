// Throughput of the GEMV inner loop (nibble -> bf16 levels -> mma.sync) with
// operands in shared memory; W warps per SM; variants of the dequant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dequant_mma dequant_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned lop_pair(unsigned w, int r, unsigned magic) {
    unsigned o;
    const unsigned v = w >> (4 * r);
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(o) : "r"(v), "r"(magic));
    return o;
}
__device__ __forceinline__ unsigned sub2(unsigned a, unsigned b) {
    unsigned o;
    asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(b));
    return o;
}
__device__ __forceinline__ unsigned fma2(unsigned a, unsigned b, unsigned c) {
    unsigned o;
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(o) : "r"(a), "r"(b), "r"(c));
    return o;
}
__device__ __forceinline__ void mma(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ unsigned lop_only(unsigned v, unsigned magic) {
    unsigned o;
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(o) : "r"(v), "r"(magic));
    return o;
}
__device__ __forceinline__ unsigned mulhi(unsigned a, unsigned b) {
    unsigned o;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(b));
    return o;
}

// V: 0 = LOP3+SHF+HSUB2 (current), 1 = no dequant (raw word as A), 2 = LOP3+SHF only,
//    3 = LOP3+SHF + HFMA2 (sub via fma), 4 = shifts as IMAD.HI (FMA pipe) + LOP3 + HSUB2
template <int V>
__global__ void k(float* out, int iters, unsigned m28 = 1u << 28, unsigned m24 = 1u << 24, unsigned m20 = 1u << 20) {
    __shared__ uint4 buf[64 * 32];
    __shared__ uint4 xb[64 * 8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) buf[i] = make_uint4(i * 7, i * 13, i * 17, i * 19);
    for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) xb[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
    __syncthreads();
    float acc[4][4] = {};
    const unsigned magic = 0x43004300u, off2 = 0x43074307u, one = 0x3f803f80u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int lb = warp; lb < 64; lb += blockDim.x / 32) {
            const uint4 w = buf[lb * 32 + lane];
            const uint4 x0 = xb[lb * 8 + (lane & 3) * 2], x1 = xb[lb * 8 + (lane & 3) * 2 + 1];
            const unsigned ws[4] = {w.x, w.y, w.z, w.w};
            const unsigned xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                unsigned af[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (V == 0) af[r] = sub2(lop_pair(ws[s], r, magic), off2);
                    else if (V == 1) af[r] = ws[s] + r;
                    else if (V == 2) af[r] = lop_pair(ws[s], r, magic);
                    else if (V == 3) af[r] = fma2(lop_pair(ws[s], r, magic), one, off2);
                    else {
                        const unsigned v = r == 0 ? ws[s] : mulhi(ws[s], r == 1 ? m28 : r == 2 ? m24 : m20);
                        af[r] = sub2(lop_only(v, magic), off2);
                    }
                }
                mma(acc[s], af, xs[2 * s], xs[2 * s + 1]);
            }
        }
    }
    float sum = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) sum += acc[s][0] + acc[s][1] + acc[s][2] + acc[s][3];
    if (sum == 1.2345f) out[0] = sum;
}

template <int V>
void run(int warps, float* out, const char* name) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 2000;
    k<V><<<sms, warps * 32>>>(out, 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<V><<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double qblocks_per_sm = 64.0 * iters;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s warps=%2d: %.1f SM-cycles per 64-row block (%.2f us per 64 blocks), %.0f GB/s-equiv of int4 codes\n", name,
           warps, cyc / qblocks_per_sm, ms * 1e3 / iters, 148.0 * 64 * 512 * iters / (ms * 1e-3) / 1e9);
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    for (int w : {8, 16, 32}) {
        run<0>(w, out, "lop+shf+hsub2 (cur)");
        run<1>(w, out, "no dequant");
        run<2>(w, out, "lop+shf only");
        run<3>(w, out, "lop+shf+hfma2");
        run<4>(w, out, "imad.hi+lop+hsub2");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
