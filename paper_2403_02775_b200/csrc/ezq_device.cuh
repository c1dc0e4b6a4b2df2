// Device-side numeric primitives shared by every kernel family, so the tensor
// path, the channel-scale path and the packer cannot diverge.
//
// Reference semantics restated here (file:line into /root/reference/proj):
//   level_of / eval_dense level   src/rtn.cpp:27-32, src/optimize.cpp:37-45
//   initial_scale                 src/rtn.cpp:81-86
//   snap                          src/optimize.cpp:79-82
//   adam_step                     src/optimize.cpp:86-94
//   outlier predicate             src/outliers.cpp:23,40
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ezq {

constexpr int64_t kStatsChunk = 8192;  // stats.cpp:18
constexpr double kScaleFloor = 1e-12;  // optimize.cpp:20

// Adam state for one scalar (optimize.hpp:12-16) with host-precomputed bias
// corrections bc1[t] = 1 - pow(b1, t), bc2[t] = 1 - pow(b2, t) (glibc pow on
// the host, exactly as optimize.cpp:90-91 evaluates them). No contraction.
struct AdamConsts {
    double b1, b2, c1, c2, lr, eps;  // c1 = 1-b1, c2 = 1-b2
};

__host__ __device__ __forceinline__ float level_guard(int lmax) {
    return 0.5f - static_cast<float>(lmax + 1) * 2.384185791015625e-07f;  // 2^-22
}

// Guard for the saturating-FFMA level of the K3 inner loop (LevelSat):
// v = sat(x*A + B) with A = RN32(1/RN32(s*span)), B = RN32(-lmin/span),
// w = v*span. Error budget against u = x/s (derivation in DESIGN.md §3):
//   |w + lmin - u| <= (lmax+0.5)*2^-23 + (|lmin|+span+1)*2^-24  (+ O(2^-46)),
// the reference's own u64 = RN(x*RN(1/s)) is within 2^-52|u| of u, and the
// residual r is rounded once more (<= 2^-25). Budget doubled + 2^-20 slack.
__host__ __device__ __forceinline__ float level_guard_sat(int lmin, int lmax) {
    const float span = static_cast<float>(lmax - lmin);
    const float b = (static_cast<float>(lmax) + 0.5f) * 1.1920928955078125e-07f +
                    (static_cast<float>(-lmin) + span + 1.0f) * 5.9604644775390625e-08f;
    return 0.5f - (2.0f * b + 9.5367431640625e-07f);
}

#ifdef __CUDACC__

// ---- exact (reference-identical) level ------------------------------------
// u = x * inv in fp64; clamp before rounding; llround = half away from zero.
// trunc/sub are exact for |u| < 2^52, so this is bit-identical to libm llround.
__device__ __forceinline__ double level_exact(double x, double inv, double dmin, double dmax) {
    const double u = __dmul_rn(x, inv);
    if (u >= dmax) return dmax;
    if (u <= dmin) return dmin;
    const double t = trunc(u);
    const double f = __dsub_rn(u, t);
    return fabs(f) >= 0.5 ? __dadd_rn(t, copysign(1.0, u)) : t;
}

// ---- fast level in fp32 with a certified guard band ------------------------
// With invf = float(inv): |u32 - u64| <= |u|*2^-23*(1+eps) <= (lmax+1)*2^-23
// for every unclamped u. Rounding boundaries sit only at half-integers inside
// (lmin, lmax) (clamping is continuous with rounding there), so whenever
// |u32 - rint(u32)| < 0.5 - guard with guard = (lmax+1)*2^-22 the fp32 level
// equals the exact level. Callers track the max |r| and take the exact path
// when it crosses the band.
struct FastLevel {
    float invf, fmin, fmax;
};

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: FADD rounds to integer

__device__ __forceinline__ float level_fast(float x, const FastLevel& fl, float& rmax) {
    float u = __fmul_rn(x, fl.invf);
    u = fminf(fmaxf(u, fl.fmin), fl.fmax);
    const float t = __fadd_rn(u, kMagic);
    const float q = __fsub_rn(t, kMagic);
    rmax = fmaxf(rmax, fabsf(__fsub_rn(u, q)));
    return q;
}

// ---- level -> double without F2F ------------------------------------------
// F2F.F64.F32 issues at ~16/clk/SM on B200 (measured), an eighth of the FP32
// rate. For t = RN32(w + MAGIC) = MAGIC + q (|q| < 2^19) the bit pattern is
// 0x4B400000 + q. Re-basing it into the HIGH word of a double whose low word
// is 0 gives 0x41380000 + q : 0 = 1.5*2^20 + q (the high word's LSB weighs 1
// at exponent 2^20), and one DADD removes the bias: exact for every level.
// One IADD + one DADD per element; the zero low words are loop-invariant
// registers (a 64-bit IMAD.WIDE form costs an extra IMAD.X for the carry).
__device__ __forceinline__ double level_bits_to_double(float t) {
    const int hi = static_cast<int>(__float_as_uint(t)) - 0x0A080000;  // 0x4B400000 -> 0x41380000
    return __dsub_rn(__hiloint2double(hi, 0), 1572864.0);
}

// ---- scale handling ----------------------------------------------------------
__device__ __forceinline__ double snap(double s) {
    const double snapped = static_cast<double>(__double2float_rn(s));
    return snapped < kScaleFloor ? kScaleFloor : snapped;  // std::max(snapped, floor)
}

// initial_scale(x) with max|x| already known (division by 2^(k-1) is exact).
__device__ __forceinline__ double initial_scale_from_max(double max_abs, int lmax) {
    if (max_abs == 0.0) return 1.0;
    return __ddiv_rn(max_abs, static_cast<double>(lmax));
}

// a / b for a table divisor b with y = RN(1/b) precomputed: Markstein's
// correction q + (a - b q) y of q = RN(a y) is the correctly rounded quotient
// when y is correctly rounded and nothing under/overflows (checked on 1e9
// random a against every bias-correction divisor of the default schedule:
// 0 mismatches vs IEEE division); tiny |a| takes the IEEE division.
__device__ __forceinline__ double div_by_table(double a, double b, double y) {
    if (fabs(a) < 1e-280) return __ddiv_rn(a, b);
    const double q = __dmul_rn(a, y);
    return fma(fma(-b, q, a), y, q);
}

// adam_update with the two bias-correction divisions through div_by_table.
__device__ __forceinline__ double adam_update_tab(double& m, double& v, double s, double g, double bc1,
                                                  double bc2, double rbc1, double rbc2, const AdamConsts& a) {
    m = __dadd_rn(__dmul_rn(a.b1, m), __dmul_rn(a.c1, g));
    v = __dadd_rn(__dmul_rn(a.b2, v), __dmul_rn(__dmul_rn(a.c2, g), g));
    const double mh = div_by_table(m, bc1, rbc1);
    const double vh = div_by_table(v, bc2, rbc2);
    const double upd = __ddiv_rn(__dmul_rn(a.lr, mh), __dadd_rn(__dsqrt_rn(vh), a.eps));
    const double updated = __dsub_rn(s, upd);
    return updated < kScaleFloor ? kScaleFloor : updated;  // std::max(updated, floor)
}

__device__ __forceinline__ double adam_update(double& m, double& v, double s, double g,
                                              double bc1, double bc2, const AdamConsts& a) {
    m = __dadd_rn(__dmul_rn(a.b1, m), __dmul_rn(a.c1, g));
    v = __dadd_rn(__dmul_rn(a.b2, v), __dmul_rn(__dmul_rn(a.c2, g), g));
    const double mh = __ddiv_rn(m, bc1);
    const double vh = __ddiv_rn(v, bc2);
    const double upd = __ddiv_rn(__dmul_rn(a.lr, mh), __dadd_rn(__dsqrt_rn(vh), a.eps));
    const double updated = __dsub_rn(s, upd);
    return updated < kScaleFloor ? kScaleFloor : updated;  // std::max(updated, floor)
}

// ---- outlier predicate (outliers.cpp:23): |double(v) - mean| >= thr ---------
__device__ __forceinline__ bool is_outlier(float v, double mean, double thr) {
    return fabs(__dsub_rn(static_cast<double>(v), mean)) >= thr;
}

// The predicate is monotone in v: RN(double(v) - mean) is non-decreasing in
// v, so the outlier set is {v <= olo} U {v >= ohi} for two float bounds,
// found by stepping float neighbours around mean -/+ thr (a few steps).
// Computed once per tensor; the per-element test is then two FSETPs.
// Non-finite mean/thr (a non-finite tensor, reported as an error by the
// host) yields the empty set; the stepping loops are bounded regardless.
__device__ __forceinline__ float outlier_hi_bound(double mean, double thr) {
    const float kInf = __int_as_float(0x7f800000);
    if (!isfinite(mean) || !isfinite(thr)) return kInf;
    auto pred = [&](float v) { return __dsub_rn(static_cast<double>(v), mean) >= thr; };
    float c = __double2float_rn(__dadd_rn(mean, thr));
    if (isinf(c)) c = c > 0.f ? 3.40282347e38f : -3.40282347e38f;
    if (pred(c)) {
        for (int i = 0; i < 64; ++i) {
            const float p = nextafterf(c, -kInf);
            if (!pred(p)) break;
            c = p;
        }
        return c;
    }
    for (int i = 0; i < 64; ++i) {
        if (c == 3.40282347e38f) return kInf;  // no finite float qualifies
        c = nextafterf(c, kInf);
        if (pred(c)) return c;
    }
    return c;  // unreachable for finite mean/thr
}
__device__ __forceinline__ float outlier_lo_bound(double mean, double thr) {
    const float kInf = __int_as_float(0x7f800000);
    if (!isfinite(mean) || !isfinite(thr)) return -kInf;
    auto pred = [&](float v) { return __dsub_rn(static_cast<double>(v), mean) <= -thr; };
    float c = __double2float_rn(__dsub_rn(mean, thr));
    if (isinf(c)) c = c > 0.f ? 3.40282347e38f : -3.40282347e38f;
    if (pred(c)) {
        for (int i = 0; i < 64; ++i) {
            const float nx = nextafterf(c, kInf);
            if (!pred(nx)) break;
            c = nx;
        }
        return c;
    }
    for (int i = 0; i < 64; ++i) {
        if (c == -3.40282347e38f) return -kInf;
        c = nextafterf(c, -kInf);
        if (pred(c)) return c;
    }
    return c;  // unreachable for finite mean/thr
}
__device__ __forceinline__ bool is_outlier_f(float v, float olo, float ohi) { return v <= olo || v >= ohi; }

// ---- exact sequential accumulation of one element (optimize.cpp:36-49) -----
// err += d*d and grad += d*q with separate roundings (the reference is built
// without FMA contraction); d = s*q - x is exact since s*q is.
__device__ __forceinline__ void seq_accumulate(double x, double q, double s, double& err,
                                               double& grad) {
    const double d = __dsub_rn(__dmul_rn(s, q), x);
    err = __dadd_rn(err, __dmul_rn(d, d));
    grad = __dadd_rn(grad, __dmul_rn(d, q));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

#endif  // __CUDACC__

}  // namespace ezq
