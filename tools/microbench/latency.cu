// Dependent-chain latency of the FP64 / conversion / shuffle ops used by the
// sequential (reference-order) chains. One warp, clock64 around N iterations.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(double* out, long long* cyc, int n, double a, float af) {
    double x = threadIdx.x * 1e-9 + 1.0;
    float f = threadIdx.x + 1.0f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = __dadd_rn(x, a);                 // DADD chain
        if (OP == 1) x = fma(x, a, a);                    // DFMA chain
        if (OP == 2) x = __dmul_rn(x, a);                 // DMUL chain
        if (OP == 3) x = (x < a) ? a : x;                 // max via DSETP+SEL
        if (OP == 4) x = __shfl_xor_sync(0xffffffffu, x, 1) + a;  // SHFL.64 + DADD
        if (OP == 5) { f = __fadd_rn(f, af); }            // FADD chain
        if (OP == 6) { x = (double)(float)x + a; }        // F2F round trip + DADD
        if (OP == 7) { x = __ddiv_rn(a, x); }             // DDIV
        if (OP == 8) { x = __dsqrt_rn(x) + a; }           // DSQRT + DADD
        if (OP == 9) { x = fmax(x, a * 0.5); }            // DMNMX?
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + f;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const char* names[] = {"DADD", "DFMA", "DMUL", "DSETP+SEL max", "SHFL.64+DADD", "FADD",
                           "F2F f64->f32->f64 + DADD", "DDIV", "DSQRT+DADD", "fmax(double)"};
    const int n = 4096;
    long long h;
#define RUN(OP)                                                  \
    lat<OP><<<1, 32>>>(out, cyc, 16, 1.0000001, 1.0001f);        \
    lat<OP><<<1, 32>>>(out, cyc, n, 1.0000001, 1.0001f);         \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);              \
    printf("%-28s %.2f cycles/iter\n", names[OP], (double)h / n);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
    return 0;
}
