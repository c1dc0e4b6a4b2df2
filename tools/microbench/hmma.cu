// Legacy tensor path throughput on B200: mma.sync.m16n8k16 (bf16/f16 ->
// f32), W warps per SM, C independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma hmma.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C, bool F16>
__global__ void k(float* out, int iters) {
    float d[C][4] = {};
    unsigned a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    unsigned b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (F16)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 1.2345f) out[0] = s;
}

template <int C, bool F16>
void run(int warps, float* out) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096;
    k<C, F16><<<sms, warps * 32>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<C, F16><<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = double(sms) * warps * C * iters;
    const double tflops = mmas * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12;
    const double per_sm_clk = mmas / sms / (ms * 1e-3 * clk * 1e3);
    printf("%s warps/SM=%2d chains=%d: %7.1f TFLOP/s  %.3f HMMA/clk/SM (at %d MHz max)\n", F16 ? "f16 " : "bf16", warps, C,
           tflops, per_sm_clk, clk / 1000);
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    for (int w : {4, 8, 16, 32}) {
        run<1, false>(w, out);
        run<4, false>(w, out);
        run<8, false>(w, out);
    }
    run<4, true>(16, out);
    return 0;
}
