// Diagnostics: FP64 DFMA peak of the device (the roofline denominator of the
// q_range kernel -- MEASURED_PEAKS.json carries no FP64 figure).
#include "runtime.hpp"

namespace ezq {
namespace {
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += r[k];
    if (s == 1234.5) out[0] = s;
}
}  // namespace
}  // namespace ezq

using namespace ezq;

extern "C" int ezq_measure_fp64_peak(double* tflops) {
    *tflops = 0.0;
    int dev;
    if (int s = bind_device(&dev)) return s;
    const DeviceInfo& di = device_info(dev);
    cudaStream_t st = thread_stream(dev);
    double* out = nullptr;
    EZQ_CK(cudaMallocAsync(&out, 64, st));
    const int threads = 512, blocks = di.sms * 4, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_dfma_peak<<<blocks, threads, 0, st>>>(out, 200, 1.0000001, 1e-9);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, st);
        k_dfma_peak<<<blocks, threads, 0, st>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(b, st);
        EZQ_CK(cudaEventSynchronize(b));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeAsync(out, st);
    EZQ_CK(cudaGetLastError());
    *tflops = 2.0 * 16.0 * iters * static_cast<double>(blocks) * threads / (best * 1e-3) / 1e12;
    return clear_error();
}
