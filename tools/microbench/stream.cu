// How fast can one kernel stream N bytes from HBM on B200? (development aid)
// Variants: (a) LDG.128 grid-stride, U loads in flight per thread;
//           (b) persistent CTAs + cp.async.bulk ring (mbarrier), consumers
//               touch one word per stage.
// Each variant is timed over 8 rotated buffers (> L2) with CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void k_ldg(const uint4* __restrict__ p, int64_t n16, unsigned* out) {
    unsigned acc = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16; i += stride * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (i + u * stride < n16) ? __ldg(p + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_bulk(const unsigned char* __restrict__ src, int64_t bytes, int stage_bytes, int stages, unsigned* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * stage_bytes);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32 - 1;
    const int64_t nchunks = (bytes + stage_bytes - 1) / stage_bytes;
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(nw));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto wait = [](uint64_t* b, unsigned par) {
        uint32_t ok;
        do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
        } while (!ok);
    };
    if (warp == nw) {
        if (lane == 0) {
            int it = 0;
            for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
                const int slot = it % stages;
                if (it >= stages) wait(&empty[slot], ((it / stages) - 1) & 1);
                const unsigned nb = static_cast<unsigned>(min(static_cast<int64_t>(stage_bytes), bytes - c * stage_bytes));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(nb) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(sm + static_cast<size_t>(slot) * stage_bytes)), "l"(src + c * stage_bytes), "r"(nb),
                             "r"(su32(&full[slot])) : "memory");
            }
        }
        return;
    }
    unsigned acc = 0;
    int it = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int slot = it % stages;
        wait(&full[slot], (it / stages) & 1);
        acc ^= reinterpret_cast<const unsigned*>(sm + static_cast<size_t>(slot) * stage_bytes)[threadIdx.x];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t sizes[] = {8 << 20, 22 << 20, 64 << 20, 256 << 20};
    const int copies = 8;
    unsigned* out;
    CK(cudaMalloc(&out, 4));
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int64_t bytes : sizes) {
        std::vector<unsigned char*> bufs(copies);
        for (auto& b : bufs) { CK(cudaMalloc(&b, bytes)); cudaMemset(b, 1, bytes); }
        cudaStream_t cs;
        cudaStreamCreate(&cs);
        auto run = [&](const char* name, auto launch) {
            // one round of `copies` launches captured in a CUDA graph
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeGlobal);
            for (auto b : bufs) launch(b, cs);
            cudaStreamEndCapture(cs, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, cs);
            cudaEventRecord(e0, cs);
            const int reps = 10;
            for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, cs);
            cudaEventRecord(e1, cs);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / (reps * copies);
            printf("%6.1f MB %-28s %8.2f us %7.0f GB/s %s\n", bytes / 1048576.0, name, us, bytes / us / 1e3,
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        };
        const int64_t n16 = bytes / 16;
        run("ldg U=4 1184x256", [&](unsigned char* b, cudaStream_t q) { k_ldg<4><<<sms * 8, 256, 0, q>>>((const uint4*)b, n16, out); });
        run("ldg U=8 1184x256", [&](unsigned char* b, cudaStream_t q) { k_ldg<8><<<sms * 8, 256, 0, q>>>((const uint4*)b, n16, out); });
        run("ldg U=4 296x512", [&](unsigned char* b, cudaStream_t q) { k_ldg<4><<<sms * 2, 512, 0, q>>>((const uint4*)b, n16, out); });
        for (int sb : {8192, 16384, 32768}) {
            for (int st : {4, 6}) {
                for (int cps : {1, 2}) {
                    const size_t smem = static_cast<size_t>(sb) * st + 16 * st;
                    if (smem * cps > 220 * 1024) continue;
                    char name[64];
                    snprintf(name, sizeof name, "bulk %dK x%d, %d CTA/SM", sb / 1024, st, cps);
                    run(name, [&](unsigned char* b, cudaStream_t q) { k_bulk<<<sms * cps, 288, smem, q>>>(b, bytes, sb, st, out); });
                }
            }
        }
        CK(cudaGetLastError());
        for (auto b : bufs) cudaFree(b);
    }
    return 0;
}
