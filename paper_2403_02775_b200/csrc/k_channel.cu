// Kc: channel-scale entry points, executed on the device in the reference's
// exact sequential order (one thread walks one channel in ascending index
// order with separate roundings), so results are bit-identical to
//   eval_dense            optimize.cpp:30-51
//   optimize_channel_range optimize.cpp:118-184 (incl. the per-step trace)
//   brute_force grid      optimize.cpp:186-229 (one thread per grid point)
//   column_sq_diff        rtn.cpp:34-52 (one thread per column)
//   quantize_channel      rtn.cpp:88-99
// These are latency-bound single-channel utilities (tests, gradcheck,
// acceptance criteria); the throughput path is K3.
#include "ezq_kernels.cuh"

namespace ezq {

namespace {

__device__ __forceinline__ void eval_seq(const float* x, int64_t n, double s, const CfgDev& cfg,
                                         double& err, double& grad) {
    const double inv = __ddiv_rn(1.0, s);
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const FastLevel fl{__double2float_rn(inv), static_cast<float>(cfg.lmin),
                       static_cast<float>(cfg.lmax)};
    err = 0.0;
    grad = 0.0;
#pragma unroll 4
    for (int64_t i = 0; i < n; ++i) {
        const float xf = x[i];
        float rm = 0.f;
        double q = static_cast<double>(level_fast(xf, fl, rm));
        if (rm >= cfg.guard) q = level_exact(static_cast<double>(xf), inv, dmin, dmax);
        seq_accumulate(static_cast<double>(xf), q, s, err, grad);
    }
    grad = 2.0 * grad;
}

__global__ void k_channel_eval(const float* __restrict__ x, int64_t n,
                               const double* __restrict__ scales, int nscales, CfgDev cfg,
                               double* err, double* grad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nscales) return;
    double e, g;
    eval_seq(x, n, scales[i], cfg, e, g);
    err[i] = e;
    if (grad) grad[i] = g;
}

// out[ch*8 + k]: 0 scale(float as double) 1 initial_error 2 final_error
// 3 best_step 4 best_scale 5 best_error; trace[ch*(steps+1)*2 + 2t + {0,1}].
__global__ void k_optimize_channels(const float* __restrict__ x,
                                    const int64_t* __restrict__ offsets, int nch, CfgDev cfg,
                                    int keep_trace, double* out, double* trace) {
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= nch) return;
    const float* v = x + offsets[ch];
    const int64_t n = offsets[ch + 1] - offsets[ch];
    double* o = out + 8 * static_cast<int64_t>(ch);
    if (n == 0) {  // every entry masked (optimize.cpp:128-133)
        o[0] = 1.0;
        o[1] = o[2] = 0.0;
        o[3] = 0.0;
        o[4] = 1.0;
        o[5] = 0.0;
        return;
    }
    double mx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs(static_cast<double>(v[i]));
        mx = (mx < a) ? a : mx;
    }
    double s = snap(initial_scale_from_max(mx, cfg.lmax));
    double err, grad;
    eval_seq(v, n, s, cfg, err, grad);
    double* tr = trace ? trace + static_cast<int64_t>(ch) * (cfg.steps + 1) * 2 : nullptr;
    if (keep_trace && tr) {
        tr[0] = s;
        tr[1] = err;
    }
    const double s0 = s, e0 = err;
    double best_err = err, best_s = s, fixed_s = s, fixed_err = err;
    int best_step = 0;
    double m = 0.0, vv = 0.0;
    for (int t = 1; t <= cfg.steps; ++t) {
        s = snap(adam_update(m, vv, s, grad, cfg.bc1[t], cfg.bc2[t], cfg.adam));
        eval_seq(v, n, s, cfg, err, grad);
        if (keep_trace && tr) {
            tr[2 * t] = s;
            tr[2 * t + 1] = err;
        }
        if (err < best_err) {
            best_err = err;
            best_s = s;
            best_step = t;
        }
        if (t == cfg.fixed_at) {
            fixed_s = s;
            fixed_err = err;
        }
    }
    double scale, fin;
    if (cfg.select == EZQ_SELECT_FIXED) {
        if (fixed_err <= e0) {
            scale = fixed_s;
            fin = fixed_err;
        } else {
            scale = s0;
            fin = e0;
        }
    } else {
        scale = best_s;
        fin = best_err;
    }
    o[0] = static_cast<double>(__double2float_rn(scale));
    o[1] = e0;
    o[2] = fin;
    o[3] = static_cast<double>(best_step);
    o[4] = best_s;
    o[5] = best_err;
}

__global__ void k_recon_error(const float* __restrict__ a, const float* __restrict__ b,
                              int64_t rows, int64_t cols, const int64_t* __restrict__ skip_off,
                              const uint32_t* __restrict__ skip_rows, double* col_sum) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const uint32_t* sk = nullptr;
    int64_t sk_n = 0, sk_i = 0;
    if (skip_off) {
        sk = skip_rows + skip_off[j];
        sk_n = skip_off[j + 1] - skip_off[j];
    }
    double acc = 0.0;
    for (int64_t i = 0; i < rows; ++i) {
        if (sk && sk_i < sk_n && sk[sk_i] == static_cast<uint32_t>(i)) {
            ++sk_i;
            continue;
        }
        const double d = __dsub_rn(static_cast<double>(a[i * cols + j]),
                                   static_cast<double>(b[i * cols + j]));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    col_sum[j] = acc;
}

__global__ void k_quantize_channel(const float* __restrict__ x, int64_t n, double inv,
                                   CfgDev cfg, int16_t* levels) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    levels[i] = static_cast<int16_t>(
        level_exact(static_cast<double>(x[i]), inv, cfg.lmin, cfg.lmax));
}

}  // namespace

void launch_channel_eval(const float* x, int64_t n, const double* scales, int nscales,
                         CfgDev cfg, double* err, double* grad, cudaStream_t st) {
    k_channel_eval<<<(nscales + 127) / 128, 128, 0, st>>>(x, n, scales, nscales, cfg, err, grad);
    count_launch();
}

void launch_optimize_channels(const float* x, const int64_t* offsets, int nch, CfgDev cfg,
                              int keep_trace, double* out, double* trace, cudaStream_t st) {
    k_optimize_channels<<<(nch + 63) / 64, 64, 0, st>>>(x, offsets, nch, cfg, keep_trace, out,
                                                        trace);
    count_launch();
}

void launch_recon_error(const float* a, const float* b, int64_t rows, int64_t cols,
                        const int64_t* skip_off, const uint32_t* skip_rows, double* col_sum,
                        cudaStream_t st) {
    k_recon_error<<<(unsigned)((cols + 127) / 128), 128, 0, st>>>(a, b, rows, cols, skip_off,
                                                                  skip_rows, col_sum);
    count_launch();
}

void launch_quantize_channel(const float* x, int64_t n, double scale, CfgDev cfg,
                             int16_t* levels, cudaStream_t st) {
    if (n == 0) return;
    const double inv = 1.0 / scale;
    k_quantize_channel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, inv, cfg, levels);
    count_launch();
}

}  // namespace ezq
