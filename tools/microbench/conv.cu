// Throughput of float->double conversion strategies (per SM per clock).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__global__ void conv(unsigned* out, int iters, float a) {
    float f[8];
    unsigned acc = 0;
    double dacc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { f[k] = threadIdx.x * 0.37f + k; dacc[k] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double d;
            if (V == 0) d = (double)f[k];                                    // F2F.F64.F32
            if (V == 1) d = (double)__float2int_rn(f[k]);                    // F2I + I2F.F64
            if (V == 2) {                                                    // magic (q small int)
                unsigned lo = __float_as_uint(f[k]) + 0x34C00000u;
                d = __hiloint2double(0x43380000, (int)lo);
            }
            if (V == 3) {                                                    // int bit-construct (normals)
                unsigned b = __float_as_uint(f[k]);
                unsigned hi = ((b & 0x7fffffffu) >> 3) + 0x38000000u;
                hi |= b & 0x80000000u;
                d = __hiloint2double((int)hi, (int)(b << 29));
            }
            if (V == 4) d = (double)__float2int_rn(f[k]) ; // placeholder same as 1
            unsigned h = __double2hiint(d) ^ __double2loint(d);
            acc ^= h;
            f[k] = __uint_as_float(__float_as_uint(f[k]) ^ (h & 1));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    unsigned* out;
    cudaMalloc(&out, 148 * 16 * 256 * 4);
    int clk = 0, sms = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"F2F.F64.F32", "F2I+I2F.F64", "magic IADD+pair", "int bit-construct", "dup"};
    auto run = [&](auto k, int v) {
        int blocks = sms * 8, threads = 256, iters = 4000;
        k<<<blocks, threads>>>(out, 10, 1.0f);
        cudaEventRecord(a);
        k<<<blocks, threads>>>(out, iters, 1.0f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = 8.0 * iters * blocks * threads;
        printf("%-20s %.3f ms  %.1f conv/clk/SM (incl. 3 ALU consumer ops)\n", names[v], ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    };
    run(conv<0>, 0); run(conv<1>, 1); run(conv<2>, 2); run(conv<3>, 3);
    return 0;
}
