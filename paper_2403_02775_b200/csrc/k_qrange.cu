// K3: per-column q_range optimisation (optimize.cpp:118-184 applied to every
// column by pipeline.cpp:29-63,88-93), and K3b: reference-order errors.
//
// Data layout. A CTA owns a strip of CB columns x all rows of one tensor,
// staged ONCE from HBM into shared memory column-major (column stride
// rstride = rpad + 4 floats: the 16-byte skew keeps the transposing float4
// stores conflict-free), with isolated outliers and padding rows zeroed.
// A zero element has level 0 and residual 0, so it contributes exactly
// nothing -- masked and padded slots need no compaction (pipeline.cpp:33-35
// gathers the normals; summing zeros instead is bit-neutral).
//
// Each column is owned by a team of P = L*W threads (L lanes in each of W
// warps). Every Adam step streams the strip out of SMEM with conflict-free
// LDS.128, computes each element's level in fp32 under a certified guard band
// (exact fp64 redo when any element of the thread lands in the band), and
// accumulates the residual d = s*q - x, d^2 and d*q in fp64 (DFMA). The two
// sums are reduced with a fixed xor-butterfly (every lane ends with the same
// bits, so every lane runs the scalar Adam update redundantly and no
// broadcast is needed) and, for W > 1, a fixed-order sum of per-warp partials
// behind one named barrier per step. Tree order differs from the reference's
// ascending-row order only in the last bits of err/grad; the K3b epilogue
// recomputes the two reported errors per column from the strip in exact
// reference order (sequential fp64, separate roundings).
//
// Roofline: FP64/issue bound. Algorithmic work per element-step = 1 DMUL
// (u) + 3 DFMA (d, d^2, d*q) = 7 flop.
#include <algorithm>
#include <cstdlib>

#include "ezq_kernels.cuh"

namespace ezq {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Fixed-order team reduction of two doubles (sum) -- identical bits in every
// thread of the team.
template <int L, int W>
__device__ __forceinline__ void team_sum2(double& a, double& b, double* red, int team, int wi,
                                          int lane, int teams, int& parity) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(kFull, a, o);
        b += __shfl_xor_sync(kFull, b, o);
    }
    if constexpr (W > 1) {
        double* slot = red + (static_cast<size_t>(parity * teams + team) * W) * 2;
        if (lane == 0) {
            slot[2 * wi] = a;
            slot[2 * wi + 1] = b;
        }
        named_bar(1 + team, W * 32);
        double sa = slot[0], sb = slot[1];
#pragma unroll
        for (int w = 1; w < W; ++w) {
            sa += slot[2 * w];
            sb += slot[2 * w + 1];
        }
        a = sa;
        b = sb;
        parity ^= 1;
    }
}

template <int L, int W>
__device__ __forceinline__ float team_max(float a, double* red, int team, int wi, int lane,
                                          int teams, int& parity) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(kFull, a, o));
    if constexpr (W > 1) {
        double* slot = red + (static_cast<size_t>(parity * teams + team) * W) * 2;
        if (lane == 0) slot[2 * wi] = static_cast<double>(a);
        named_bar(1 + team, W * 32);
        double m = slot[0];
#pragma unroll
        for (int w = 1; w < W; ++w) m = fmax(m, slot[2 * w]);
        a = static_cast<float>(m);
        parity ^= 1;
    }
    return a;
}

struct Acc {
    double ea, eb, ga, gb;
};

__device__ __forceinline__ void elem_exact(float x, double inv, double dmin, double dmax,
                                           double s, double& e, double& g) {
    const double xd = static_cast<double>(x);
    const double qd = level_exact(xd, inv, dmin, dmax);
    const double d = fma(s, qd, -xd);
    e = fma(d, d, e);
    g = fma(d, qd, g);
}

template <int L, int W, bool GLOBAL>
__global__ void __launch_bounds__(512, 1) k_qrange(const TDesc* __restrict__ td,
                                                const K3Group* __restrict__ groups,
                                                int ngroups, Scratch sc, CfgDev cfg, int rpad,
                                                int rstride, int teams, float* gstrip) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int P = L * W;
    float* strip = GLOBAL ? gstrip + static_cast<size_t>(blockIdx.x) * teams * rstride
                          : reinterpret_cast<float*>(smem_raw);
    double* red = reinterpret_cast<double*>(
        smem_raw + (GLOBAL ? 0 : static_cast<size_t>(teams) * rstride * sizeof(float)));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int team = (W == 1) ? warp * (32 / L) + lane / L : warp / W;
    const int pt = (W == 1) ? lane % L : (warp % W) * 32 + lane;
    const int wi = (W == 1) ? 0 : warp % W;
    const int K = rpad / (4 * P);
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const bool optimize = cfg.mode == EZQ_MODE_EASYQUANT;

    for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        const K3Group g = groups[gi];
        const TDesc& d = td[g.tensor];
        const TStats* st = d.st;
        const float olo = st->olo, ohi = st->ohi;
        const int64_t R = d.rows, C = d.cols;

        __syncthreads();  // previous strip fully consumed
        const int R4 = rpad >> 2;
        for (int idx = tid; idx < teams * R4; idx += blockDim.x) {
            const int cc = idx % teams, rq = idx / teams;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (cc < g.ncols) {
                const int64_t r0 = 4 * static_cast<int64_t>(rq);
                const float* src = d.W + r0 * C + (g.col0 + cc);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (r0 + k < R) {
                        const float x = src[k * C];
                        v[k] = is_outlier_f(x, olo, ohi) ? 0.f : x;
                    }
                }
            }
            *reinterpret_cast<float4*>(strip + static_cast<size_t>(cc) * rstride + 4 * rq) =
                make_float4(v[0], v[1], v[2], v[3]);
        }
        __syncthreads();

        // Idle columns: whole warps (W == 1) or whole teams (W > 1) skip the
        // optimisation but still meet the CTA barriers below.
        const bool active = (W == 1) ? (warp * (32 / L) < g.ncols) : (team < g.ncols);
        const float4* col4 =
            reinterpret_cast<const float4*>(strip + static_cast<size_t>(team) * rstride);
        if (active) {
        int parity = 0;

        // initial_scale over the normals (rtn.cpp:81-86): max is order-free.
        float mx = 0.f;
        for (int k = 0; k < K; ++k) {
            const float4 x = col4[pt + k * P];
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
        }
        mx = team_max<L, W>(mx, red, team, wi, lane, teams, parity);
        const double s0_raw = initial_scale_from_max(static_cast<double>(mx), cfg.lmax);
        const bool writer = (pt == 0) && (team < g.ncols);

        // Rtn / OutliersOnly: float(initial_scale), no optimisation
        // (pipeline.cpp:52-55).
        double s_rtn = static_cast<double>(__double2float_rn(s0_raw));
        double s_fin = s_rtn;
        if (optimize) {
        // ---- Adam loop (optimize.cpp:138-167) ----
        double s = snap(s0_raw);
        const double s0 = s;
        double m = 0.0, v = 0.0;
        double e0 = 0.0, best_err = 0.0, best_s = s, fixed_s = s, fixed_err = 0.0;
        const float spanf = static_cast<float>(cfg.lmax - cfg.lmin);
        const float magic_l = kMagic + static_cast<float>(cfg.lmin);  // exact
        const float gsat = cfg.guard_sat;
        for (int t = 0;; ++t) {
            // Level per element (certified fp32, exact fp64 fix inside the
            // guard band): v = sat(x*A + B) maps [lmin, lmax] onto [0, 1];
            // t = RN(v*span + MAGIC + lmin) = MAGIC + q; r = w + lmin - q.
            const float A = __frcp_rn(__fmul_rn(__double2float_rn(s), spanf));
            double ea = 0.0, eb = 0.0, ga = 0.0, gb = 0.0;
            double ec = 0.0, ed = 0.0, gc2 = 0.0, gd = 0.0;
            int k = 0;
            for (; k + 4 <= K; k += 4) {
                float xv[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 x = col4[pt + (k + j) * P];
                    xv[4 * j] = x.x;
                    xv[4 * j + 1] = x.y;
                    xv[4 * j + 2] = x.z;
                    xv[4 * j + 3] = x.w;
                }
                float rmax = 0.f;
                float tv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float v = __saturatef(__fmaf_rn(xv[j], A, cfg.sat_b));
                    tv[j] = __fmaf_rn(v, spanf, magic_l);  // MAGIC + q
                    const float r = __fmaf_rn(v, spanf, __fsub_rn(magic_l, tv[j]));
                    rmax = fmaxf(rmax, fabsf(r));
                }
                double xd[16], qd[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) qd[j] = level_bits_to_double(tv[j]);
                if (rmax >= gsat) {
                    // An element sits within the fp32 error band of a rounding
                    // boundary: take the reference's fp64 levels for this group.
                    const double inv = __ddiv_rn(1.0, s);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        qd[j] = level_exact(static_cast<double>(xv[j]), inv, dmin, dmax);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    // F2F on the XU beats a 4-op ALU bit construction of the double:
                    // 2.29 vs 2.51 ms on C1 (B200, measured).
                    xd[j] = static_cast<double>(xv[j]);
                }
                // Four accumulator pairs keep the DFMA chains short (8.4-cycle
                // latency); lanes sum them in a fixed order below.
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const double d0 = fma(s, qd[j], -xd[j]);
                    const double d1 = fma(s, qd[j + 1], -xd[j + 1]);
                    const double d2 = fma(s, qd[j + 2], -xd[j + 2]);
                    const double d3 = fma(s, qd[j + 3], -xd[j + 3]);
                    ea = fma(d0, d0, ea);
                    ga = fma(d0, qd[j], ga);
                    eb = fma(d1, d1, eb);
                    gb = fma(d1, qd[j + 1], gb);
                    ec = fma(d2, d2, ec);
                    gc2 = fma(d2, qd[j + 2], gc2);
                    ed = fma(d3, d3, ed);
                    gd = fma(d3, qd[j + 3], gd);
                }
            }
            if (k < K) {
                const double inv = __ddiv_rn(1.0, s);
                for (; k < K; ++k) {
                    const float4 x = col4[pt + k * P];
                    elem_exact(x.x, inv, dmin, dmax, s, ea, ga);
                    elem_exact(x.y, inv, dmin, dmax, s, eb, gb);
                    elem_exact(x.z, inv, dmin, dmax, s, ea, ga);
                    elem_exact(x.w, inv, dmin, dmax, s, eb, gb);
                }
            }
            double err = (ea + ec) + (eb + ed), gr = (ga + gc2) + (gb + gd);
            team_sum2<L, W>(err, gr, red, team, wi, lane, teams, parity);
            const double grad = 2.0 * gr;
            if (t == 0) {
                e0 = err;
                best_err = err;
                fixed_err = err;
            } else {
                if (err < best_err) {  // strict: earliest minimum wins (optimize.cpp:158)
                    best_err = err;
                    best_s = s;
                }
                if (t == cfg.fixed_at) {
                    fixed_s = s;
                    fixed_err = err;
                }
            }
            if (t == cfg.steps) break;
            s = snap(adam_update(m, v, s, grad, cfg.bc1[t + 1], cfg.bc2[t + 1], cfg.adam));
        }
        if (cfg.select == EZQ_SELECT_FIXED)
            s_fin = (fixed_err <= e0) ? fixed_s : s0;  // optimize.cpp:169-178
        else
            s_fin = best_s;
        s_rtn = s0;
        }  // optimize
        if (writer) {
            const int64_t gcol = d.col_base + g.col0 + team;
            sc.s_rtn[gcol] = s_rtn;
            sc.s_fin[gcol] = s_fin;
        }
        }  // active
    }
}

// ---- K3b: reference-order errors (rtn_error / final_error per column) ----
// One warp = 32 adjacent columns of one tensor, lane = column. Each lane
// walks its column in ascending row order with the reference's separate
// roundings (eval_dense, optimize.cpp:36-49), skipping isolated outliers
// exactly like normal_mask_apply, and carries both sums -- at the initial
// scale and at the chosen one -- so the row load, the outlier test and the
// x -> double conversion are shared. Rows are read straight from global
// memory (a warp's 32 loads of a row are one 128-byte segment), kRowsK3b
// rows in flight per lane; no shared memory, so occupancy is set by
// registers. The per-column finalisation (stored float scale, per-column
// invariant, 1/scale for K4) follows in the same lane.
constexpr int kRowsK3b = 8;
constexpr int kPipeK3b = 3;  // row groups in flight per lane (K3b, near-tie resolution)
constexpr int kWarpsK3b = 4;

// Squared residual of one normal element at scale s in reference semantics
// (eval_dense, optimize.cpp:37-47): the level equals level_of's; d = s*q - x
// is exact (s*q is), so d*d carries the reference's single rounding.
__device__ __forceinline__ double seq_sq(float x, double xd, double s, float invf, double inv,
                                         float fmin, float fmax, double dmin, double dmax,
                                         float guard) {
    float u = __fmul_rn(x, invf);
    u = fminf(fmaxf(u, fmin), fmax);
    const float t = __fadd_rn(u, kMagic);
    const float r = __fsub_rn(u, __fsub_rn(t, kMagic));
    double q = level_bits_to_double(t);
    if (fabsf(r) >= guard) q = level_exact(xd, inv, dmin, dmax);
    const double d = fma(s, q, -xd);
    return __dmul_rn(d, d);
}

__global__ void __launch_bounds__(kWarpsK3b * 32) k_seq_errors(const TDesc* __restrict__ td,
                                                              const int2* __restrict__ tiles, int ntiles,
                                                              Scratch sc, CfgDev cfg) {
    const int lane = threadIdx.x & 31;
    const int ti = blockIdx.x * kWarpsK3b + (threadIdx.x >> 5);
    if (ti >= ntiles) return;
    const int2 tile = tiles[ti];
    const TDesc& d = td[tile.x];
    const int64_t c0 = tile.y, R = d.rows, C = d.cols;
    const int64_t c = c0 + lane;
    const bool act = c < C;  // idle lanes stay for the nibble-pair shuffles
    const int64_t gc = d.col_base + (act ? c : c0);
    const TStats* st = d.st;
    const float olo = st->olo, ohi = st->ohi;
    const double s_r = sc.s_rtn[gc], s_f = sc.s_fin[gc];
    // Fused K4: the codes at s_fin (pack_levels, rtn.cpp:123-149, outlier
    // slots at level 0) are written here; a column that ends up storing s_rtn
    // is flagged and re-packed by k_repack.
    const bool fused = d.pack_fused != 0;
    const unsigned lbase = __float_as_uint(kMagic) + static_cast<unsigned>(cfg.lmin);
    const unsigned lzero = static_cast<unsigned>(-cfg.lmin);
    const bool both = s_f != s_r;  // chosen == initial: one sum serves both
    const double inv_r = __ddiv_rn(1.0, s_r), inv_f = __ddiv_rn(1.0, s_f);
    const float invf_r = __double2float_rn(inv_r), invf_f = __double2float_rn(inv_f);
    const float fmin = static_cast<float>(cfg.lmin), fmax = static_cast<float>(cfg.lmax);
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const float guard = cfg.guard;
    const float* col = d.W + (act ? c : c0);
    double er = 0.0, ef = 0.0;
    int64_t r = 0;
    auto put = [&](int64_t row, unsigned tbits, bool out) {  // all lanes call it (shuffle)
        const unsigned off = out ? lzero : tbits - lbase;
        if (cfg.bits == 4) {
            const unsigned hi = __shfl_down_sync(0xffffffffu, off, 1);
            if (act && (c & 1) == 0) d.packed[(row * C + c) >> 1] = static_cast<uint8_t>(off | (hi << 4));
        } else if (act) {
            d.packed[row * C + c] = static_cast<uint8_t>(off);
        }
    };
    // Row groups are software-pipelined kPipeK3b deep: the loads of the next
    // groups are in flight while one is computed (a tall tensor has few
    // columns, i.e. few warps, so each must keep many rows in flight).
    float xb[kPipeK3b][kRowsK3b];
#pragma unroll
    for (int p = 0; p < kPipeK3b; ++p)
#pragma unroll
        for (int j = 0; j < kRowsK3b; ++j) {
            const int64_t rr0 = p * kRowsK3b + j;
            xb[p][j] = rr0 < R ? __ldg(col + rr0 * C) : 0.f;
        }
    for (; r + kRowsK3b <= R; r += kRowsK3b) {
        float x[kRowsK3b];
#pragma unroll
        for (int j = 0; j < kRowsK3b; ++j) x[j] = xb[0][j];
#pragma unroll
        for (int p = 0; p + 1 < kPipeK3b; ++p)
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j) xb[p][j] = xb[p + 1][j];
#pragma unroll
        for (int j = 0; j < kRowsK3b; ++j) {
            const int64_t rn = r + kPipeK3b * kRowsK3b + j;
            xb[kPipeK3b - 1][j] = rn < R ? __ldg(col + rn * C) : 0.f;
        }
        // certified fp32 levels for the group at both scales, one guard test
        // per scale (exact fp64 levels for the group when it trips)
        float tr[kRowsK3b], tf[kRowsK3b];
        float rr = 0.f, rf = 0.f;
#pragma unroll
        for (int j = 0; j < kRowsK3b; ++j) {
            float u = fminf(fmaxf(__fmul_rn(x[j], invf_r), fmin), fmax);
            tr[j] = __fadd_rn(u, kMagic);
            rr = fmaxf(rr, fabsf(__fsub_rn(u, __fsub_rn(tr[j], kMagic))));
            u = fminf(fmaxf(__fmul_rn(x[j], invf_f), fmin), fmax);
            tf[j] = __fadd_rn(u, kMagic);
            rf = fmaxf(rf, fabsf(__fsub_rn(u, __fsub_rn(tf[j], kMagic))));
        }
        if (rr >= guard) {
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j)
                tr[j] = __fadd_rn(static_cast<float>(level_exact(static_cast<double>(x[j]), inv_r, dmin, dmax)), kMagic);
        }
        if (both && rf >= guard) {
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j)
                tf[j] = __fadd_rn(static_cast<float>(level_exact(static_cast<double>(x[j]), inv_f, dmin, dmax)), kMagic);
        }
        if (fused) {  // warp-uniform
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j)
                put(r + j, __float_as_uint(both ? tf[j] : tr[j]), is_outlier_f(x[j], olo, ohi));
        }
#pragma unroll
        for (int j = 0; j < kRowsK3b; ++j) {
            // normal_mask_apply: an isolated outlier adds exactly +0
            const bool out = is_outlier_f(x[j], olo, ohi);
            const double xd = static_cast<double>(x[j]);
            const double dr = fma(s_r, level_bits_to_double(tr[j]), -xd);  // exact: s*q is
            er = __dadd_rn(er, out ? 0.0 : __dmul_rn(dr, dr));
            if (both) {
                const double df = fma(s_f, level_bits_to_double(tf[j]), -xd);
                ef = __dadd_rn(ef, out ? 0.0 : __dmul_rn(df, df));
            }
        }
    }
    for (; r < R; ++r) {
        const float x = __ldg(col + r * C);
        const bool out = is_outlier_f(x, olo, ohi);
        const double xd = static_cast<double>(x);
        er = __dadd_rn(er, out ? 0.0 : seq_sq(x, xd, s_r, invf_r, inv_r, fmin, fmax, dmin, dmax, guard));
        if (both) ef = __dadd_rn(ef, out ? 0.0 : seq_sq(x, xd, s_f, invf_f, inv_f, fmin, fmax, dmin, dmax, guard));
        if (fused) {
            const double q = level_exact(xd, inv_f, dmin, dmax);
            put(r, __float_as_uint(__fadd_rn(static_cast<float>(q), kMagic)), out);
        }
    }
    if (!act) return;
    double s_store = s_f;
    if (!both) {
        ef = er;
    } else if (ef > er) {
        // tree/sequential near-tie: keep the initial scale so the per-column
        // invariant final <= rtn holds (pipeline.cpp:107)
        s_store = s_r;
        ef = er;
    }
    if (fused) sc.repack[gc] = (s_store != s_f) ? 1 : 0;
    const float scale = __double2float_rn(s_store);
    if (!(scale > 0.f)) d.st->scale_zero = 1;  // check_scale (rtn.cpp:19-22)
    d.scales[c] = scale;
    const double inv = scale > 0.f ? __ddiv_rn(1.0, static_cast<double>(scale)) : 1.0;
    sc.inv[gc] = inv;
    sc.invf[gc] = __double2float_rn(inv);
    sc.err_rtn[gc] = er;
    sc.err_fin[gc] = ef;
}

// ---- near-tie resolution ------------------------------------
// The reference's whole q_range loop for one column in its own order
// (optimize_channel_range, optimize.cpp:118-184): the fallback for a column
// whose candidates overflowed the slots. The gradient sum is exact in any
// order, so this reproduces the reference bit for bit.
__device__ double column_ref_optimize(const float* col, int64_t R, int64_t C, double s0, float olo, float ohi,
                                      const CfgDev& cfg) {
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    double s = s0, m = 0.0, v = 0.0, best_e = 0.0, best_s = s0, e0 = 0.0, fixed_s = s0, fixed_e = 0.0;
    for (int t = 0;; ++t) {
        const double inv = __ddiv_rn(1.0, s);
        double e = 0.0, g = 0.0;
        for (int64_t r = 0; r < R; ++r) {
            const float x = __ldg(col + r * C);
            if (is_outlier_f(x, olo, ohi)) continue;
            seq_accumulate(static_cast<double>(x), level_exact(static_cast<double>(x), inv, dmin, dmax), s, e, g);
        }
        if (t == 0) {
            e0 = best_e = fixed_e = e;
        } else {
            if (e < best_e) best_e = e, best_s = s;
            if (t == cfg.fixed_at) fixed_s = s, fixed_e = e;
        }
        if (t == cfg.steps) break;
        s = snap(adam_update_tab(m, v, s, 2.0 * g, cfg.bc1[t + 1], cfg.bc2[t + 1], cfg.rbc1[t + 1], cfg.rbc2[t + 1],
                                 cfg.adam));
    }
    if (cfg.select == EZQ_SELECT_FIXED) return fixed_e <= e0 ? fixed_s : s0;
    return best_s;
}

// Near-tie resolution before K3b. One warp = one K3b tile
// (32 adjacent columns, lane = column); warps whose columns carry no
// candidate list return at once (all of them at 4 bits in practice). A
// column's candidates (sc.tie_*, step order) are filtered against the final
// best and de-duplicated; every kept candidate becomes a "pair" (owner lane,
// scale) handed to a lane of the warp, and the pairs' reference-order errors
// (eval_dense's sequential fp64 sum over the column's normals in row order,
// optimize.cpp:36-49) run over one coalesced stream of the tile's rows, each
// pair lane taking its owner's value by shuffle. The owner then applies the
// reference's rule (strict-< earliest minimum, optimize.cpp:158; fixed step:
// fixed_err <= e0, :169-178) and stores the winner in s_fin. More than 32
// pairs in a warp: further passes over the rows (rare). A column whose slots
// overflowed runs the reference's whole loop itself (column_ref_optimize).
struct TiePairs {
    int src[32];     // owner lane of the pair
    double s[32];    // candidate scale
    double err[32];  // reference-order error at s
};

__global__ void __launch_bounds__(kWarpsK3b * 32) k_resolve_ties(const TDesc* __restrict__ td,
                                                                const int2* __restrict__ tiles, int ntiles,
                                                                Scratch sc, CfgDev cfg) {
    __shared__ TiePairs tp_all[kWarpsK3b];
    const int lane = threadIdx.x & 31;
    const int ti = blockIdx.x * kWarpsK3b + (threadIdx.x >> 5);
    if (ti >= ntiles) return;
    TiePairs& tp = tp_all[threadIdx.x >> 5];
    const int2 tile = tiles[ti];
    const TDesc& d = td[tile.x];
    const int64_t c0 = tile.y, R = d.rows, C = d.cols;
    const int64_t c = c0 + lane;
    const bool act = c < C;
    const int64_t gc = d.col_base + (act ? c : c0);
    const int tn = act ? sc.tie_n[gc] : 0;
    if (!__any_sync(0xffffffffu, tn != 0)) return;
    const float olo = d.st->olo, ohi = d.st->ohi;
    const float* col = d.W + (act ? c : c0);
    const int cnt = tn & (kTieFixed - 1);
    const bool tfixed = (tn & kTieFixed) != 0;
    const bool overflow = cnt > cfg.tie_cap;
    if (overflow) {  // divergent, rare: the reference's loop on this column
        atomicAdd(&d.st->ties, 1);
        atomicAdd(&d.st->tie_fallback, 1);
        sc.s_fin[gc] = column_ref_optimize(col, R, C, sc.s_rtn[gc], olo, ohi, cfg);
    }
    __syncwarp();
    const double* ts = sc.tie_s + gc * kTieMax;
    const double* te = sc.tie_e + gc * kTieMax;
    unsigned keep = 0;  // bit i: candidate i kept (within the bound, first of its scale)
    if (cnt >= 2 && !overflow) {
        double e1 = te[0];
        for (int i = 1; i < cnt; ++i) e1 = te[i] < e1 ? te[i] : e1;
        const double gam = (static_cast<double>(R) + 8.0) * 1.1102230246251565e-16 * 1.02;  // rows >= normals
        for (int i = 0; i < cnt; ++i) {
            const double si = ts[i];
            if (!tfixed && te[i] - e1 > gam * (te[i] + e1)) continue;
            bool dup = false;
            for (int j = 0; j < i; ++j) dup |= ((keep >> j) & 1u) && ts[j] == si;
            if (!dup) keep |= 1u << i;
        }
        if (__popc(keep) < 2) keep = 0;  // one distinct candidate: certified after all
    }
    const int mine_n = __popc(keep);
    int base = mine_n;  // exclusive warp scan of the pair counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, base, o);
        if (lane >= o) base += v;
    }
    const int npairs = __shfl_sync(0xffffffffu, base, 31);
    base -= mine_n;
    const float fmin = static_cast<float>(cfg.lmin), fmax = static_cast<float>(cfg.lmax);
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    double mine[kTieMax];
    for (int pb = 0; pb < npairs; pb += 32) {  // warp-uniform
        __syncwarp();
        for (int i = 0, k = base; i < cnt && keep; ++i) {
            if (!((keep >> i) & 1u)) continue;
            if (k >= pb && k < pb + 32) {
                tp.src[k - pb] = lane;
                tp.s[k - pb] = ts[i];
            }
            ++k;
        }
        __syncwarp();
        const bool pown = lane < npairs - pb;
        const int psrc = pown ? tp.src[lane] : 0;
        const double ps = pown ? tp.s[lane] : 1.0;
        const double pinv = __ddiv_rn(1.0, ps);
        const float pinvf = __double2float_rn(pinv);
        double pe = 0.0;
        int64_t r = 0;
        float xb[kPipeK3b][kRowsK3b];  // software pipeline, as in k_seq_errors
#pragma unroll
        for (int p = 0; p < kPipeK3b; ++p)
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j) {
                const int64_t rr0 = p * kRowsK3b + j;
                xb[p][j] = rr0 < R ? __ldg(col + rr0 * C) : 0.f;
            }
        for (; r + kRowsK3b <= R; r += kRowsK3b) {
            float x[kRowsK3b];
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j) x[j] = xb[0][j];
#pragma unroll
            for (int p = 0; p + 1 < kPipeK3b; ++p)
#pragma unroll
                for (int j = 0; j < kRowsK3b; ++j) xb[p][j] = xb[p + 1][j];
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j) {
                const int64_t rn = r + kPipeK3b * kRowsK3b + j;
                xb[kPipeK3b - 1][j] = rn < R ? __ldg(col + rn * C) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < kRowsK3b; ++j) {
                const float xv = __shfl_sync(0xffffffffu, x[j], psrc);
                if (pown && !is_outlier_f(xv, olo, ohi))
                    pe = __dadd_rn(pe, seq_sq(xv, static_cast<double>(xv), ps, pinvf, pinv, fmin, fmax, dmin, dmax,
                                              cfg.guard));
            }
        }
        for (; r < R; ++r) {
            const float xv = __shfl_sync(0xffffffffu, __ldg(col + r * C), psrc);
            if (pown && !is_outlier_f(xv, olo, ohi))
                pe = __dadd_rn(pe, seq_sq(xv, static_cast<double>(xv), ps, pinvf, pinv, fmin, fmax, dmin, dmax,
                                          cfg.guard));
        }
        tp.err[lane] = pe;
        __syncwarp();
        for (int k = 0; k < mine_n; ++k) {
            const int slot = base + k - pb;
            if (slot >= 0 && slot < 32) mine[k] = tp.err[slot];
        }
    }
    if (!keep) return;
    int k = 0, first = 1;
    double be = 0.0, bs = 0.0, e_s0 = 0.0, s_s0 = 0.0, e_fx = 0.0, s_fx = 0.0;
    for (int i = 0; i < cnt; ++i) {
        if (!((keep >> i) & 1u)) continue;
        const double si = ts[i], ei = mine[k++];
        if (tfixed) {  // [s0, s_fixed]
            if (first) e_s0 = ei, s_s0 = si;
            else e_fx = ei, s_fx = si;
        } else if (first || ei < be) {  // strict: earliest minimum wins
            be = ei;
            bs = si;
        }
        first = 0;
    }
    sc.s_fin[gc] = tfixed ? (e_fx <= e_s0 ? s_fx : s_s0) : bs;
    atomicAdd(&d.st->ties, 1);
}

// Fix-up of the fused pack: columns flagged by K3b (stored scale s_rtn, codes
// written at s_fin) get their codes recomputed at the stored scale with the
// reference's fp64 level; for k = 4 the even lane of a nibble pair rewrites
// the shared byte (both nibbles at their columns' stored scales). Warps whose
// 32 columns carry no flag return at once.
__global__ void __launch_bounds__(kWarpsK3b * 32) k_repack(const TDesc* __restrict__ td,
                                                          const int2* __restrict__ tiles, int ntiles, Scratch sc,
                                                          CfgDev cfg) {
    const int lane = threadIdx.x & 31;
    const int ti = blockIdx.x * kWarpsK3b + (threadIdx.x >> 5);
    if (ti >= ntiles) return;
    const int2 tile = tiles[ti];
    const TDesc& d = td[tile.x];
    if (!d.pack_fused) return;
    const int64_t C = d.cols, R = d.rows, c = tile.y + lane;
    const bool act = c < C;
    const bool flag = act && sc.repack[d.col_base + c];
    const bool nflag = __shfl_down_sync(0xffffffffu, flag, 1) != 0;
    if (!__any_sync(0xffffffffu, flag)) return;
    const bool k4 = cfg.bits == 4;
    const bool mine = k4 ? (act && (c & 1) == 0 && (flag || nflag)) : flag;
    if (!mine) return;
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const float olo = d.st->olo, ohi = d.st->ohi;
    const double inv0 = sc.inv[d.col_base + c];
    const double inv1 = (k4 && c + 1 < C) ? sc.inv[d.col_base + c + 1] : 1.0;
    auto off = [&](float x, double inv) -> unsigned {
        if (is_outlier_f(x, olo, ohi)) return static_cast<unsigned>(-cfg.lmin);
        return static_cast<unsigned>(static_cast<int>(level_exact(static_cast<double>(x), inv, dmin, dmax)) - cfg.lmin);
    };
    for (int64_t r = 0; r < R; ++r) {
        const float x0 = d.W[r * C + c];
        if (k4) {
            const unsigned lo = off(x0, inv0);
            const unsigned hi = c + 1 < C ? off(d.W[r * C + c + 1], inv1) : 0u;
            d.packed[(r * C + c) >> 1] = static_cast<uint8_t>(lo | (hi << 4));
        } else {
            d.packed[r * C + c] = static_cast<uint8_t>(off(x0, inv0));
        }
    }
}

// Column-ordered tensor totals (pipeline.cpp:96-103): one CTA per tensor
// stages the per-column errors through SMEM (coalesced) and one thread adds
// them in column order.
__global__ void __launch_bounds__(256) k_tensor_totals(const TDesc* __restrict__ td, Scratch sc) {
    const TDesc& d = td[blockIdx.x];
    __shared__ double buf[2][2048];
    double rtn = 0.0, fin = 0.0;
    for (int64_t base = 0; base < d.cols; base += 2048) {
        const int cnt = static_cast<int>(min(static_cast<int64_t>(2048), d.cols - base));
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            buf[0][i] = sc.err_rtn[d.col_base + base + i];
            buf[1][i] = sc.err_fin[d.col_base + base + i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int i = 0;
            for (; i + 8 <= cnt; i += 8) {
                double a[8], b[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    a[j] = buf[0][i + j];
                    b[j] = buf[1][i + j];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    rtn = __dadd_rn(rtn, a[j]);
                    fin = __dadd_rn(fin, b[j]);
                }
            }
            for (; i < cnt; ++i) {
                rtn = __dadd_rn(rtn, buf[0][i]);
                fin = __dadd_rn(fin, buf[1][i]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        d.st->rtn_error = rtn;
        d.st->final_error = fin;
    }
}

template <int L, int W>
void launch_k3_lw(const K3Launch& kl, const TDesc* td, const K3Group* groups, int ngroups,
                  Scratch sc, CfgDev cfg, float* gstrip, int grid, cudaStream_t st) {
    if (kl.global_strip) {
        auto k = k_qrange<L, W, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kl.smem);
        k<<<grid, kl.threads, kl.smem, st>>>(td, groups, ngroups, sc, cfg, kl.rpad, kl.rstride,
                                             kl.teams, gstrip);
    } else {
        auto k = k_qrange<L, W, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kl.smem);
        k<<<grid, kl.threads, kl.smem, st>>>(td, groups, ngroups, sc, cfg, kl.rpad, kl.rstride,
                                             kl.teams, gstrip);
    }
}

}  // namespace

// Geometry: ~128 elements per thread per step; columns per CTA (CB) chosen
// by the caller (choose_k3_width) for load balance across the SMs.
K3Launch plan_k3(int64_t rows, int64_t /*total_cols_hint*/, int /*num_sms*/, int max_smem) {
    K3Launch kl{};
    kl.rows = rows;
    if (rows <= 1024) {
        kl.L = 8, kl.W = 1;
    } else if (rows <= 2048) {
        kl.L = 16, kl.W = 1;
    } else if (rows <= 4096) {
        kl.L = 32, kl.W = 1;
    } else if (rows <= 8192) {
        kl.L = 32, kl.W = 2;
    } else if (rows <= 16384) {
        kl.L = 32, kl.W = 4;
    } else if (rows <= 32768) {
        kl.L = 32, kl.W = 8;
    } else {
        kl.L = 32, kl.W = 16;
    }
    // (Measured on B200: doubling warps per column (24 warps/SM) is slower --
    // 6.50e9 vs 7.25e9 weights/s on the OPT-1.3B set -- the extra per-warp
    // Adam/reduction work outweighs the latency hiding.)
    const int P = kl.L * kl.W;
    kl.rpad = static_cast<int>(((rows + 4 * P - 1) / (4 * P)) * (4 * P));
    kl.rstride = kl.rpad + 4;
    const int unit = (kl.W == 1) ? 32 / kl.L : 1;  // columns per warp-granule
    kl.teams = unit;
    kl.global_strip = k3_smem(kl, unit) > static_cast<size_t>(max_smem);
    set_k3_width(kl, unit);
    return kl;
}

size_t k3_smem(const K3Launch& kl, int teams) {
    return static_cast<size_t>(teams) * kl.rstride * sizeof(float) + k3_small_smem(kl, teams);
}

// Reduction slots [2][teams][W][2].
size_t k3_small_smem(const K3Launch& kl, int teams) {
    return static_cast<size_t>(2) * teams * kl.W * 2 * sizeof(double);
}

void set_k3_width(K3Launch& kl, int teams) {
    kl.teams = teams;
    kl.threads = (kl.W == 1) ? ((teams * kl.L + 31) / 32) * 32 : teams * kl.W * 32;
    kl.smem = kl.global_strip ? k3_small_smem(kl, teams) : k3_smem(kl, teams);
}

void launch_k3(const K3Launch& kl, const TDesc* td, const K3Group* groups, int ngroups,
               Scratch sc, CfgDev cfg, float* gstrip, int grid, cudaStream_t st) {
    if (ngroups == 0) return;
    switch (kl.L * 100 + kl.W) {
        case 801: launch_k3_lw<8, 1>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        case 1601: launch_k3_lw<16, 1>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        case 3201: launch_k3_lw<32, 1>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        case 3202: launch_k3_lw<32, 2>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        case 3204: launch_k3_lw<32, 4>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        case 3208: launch_k3_lw<32, 8>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
        default: launch_k3_lw<32, 16>(kl, td, groups, ngroups, sc, cfg, gstrip, grid, st); break;
    }
    count_launch();
}

void launch_seq_errors(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg,
                       cudaStream_t st) {
    if (ntiles == 0) return;
    k_seq_errors<<<(ntiles + kWarpsK3b - 1) / kWarpsK3b, kWarpsK3b * 32, 0, st>>>(td, tiles, ntiles, sc, cfg);
    count_launch();
}

void launch_resolve_ties(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg, cudaStream_t st) {
    if (ntiles == 0 || cfg.mode != EZQ_MODE_EASYQUANT) return;
    k_resolve_ties<<<(ntiles + kWarpsK3b - 1) / kWarpsK3b, kWarpsK3b * 32, 0, st>>>(td, tiles, ntiles, sc, cfg);
    count_launch();
}

void launch_repack(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg, cudaStream_t st) {
    if (ntiles == 0) return;
    k_repack<<<(ntiles + kWarpsK3b - 1) / kWarpsK3b, kWarpsK3b * 32, 0, st>>>(td, tiles, ntiles, sc, cfg);
    count_launch();
}

void launch_tensor_totals(const TDesc* td, int ntens, Scratch sc, cudaStream_t st) {
    k_tensor_totals<<<ntens, 256, 0, st>>>(td, sc);
    count_launch();
}

}  // namespace ezq
