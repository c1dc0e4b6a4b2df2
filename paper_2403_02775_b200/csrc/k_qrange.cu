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
// ascending-row order only in the last bits of err/grad; K3b recomputes the
// two reported errors per column in exact reference order.
//
// Roofline: FP64/issue bound. Algorithmic work per element-step = 1 DMUL
// (u) + 3 DFMA (d, d^2, d*q) = 7 flop.
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

__device__ __forceinline__ void elem_fast(float x, const FastLevel& fl, double s, float& rmax,
                                          double& e, double& g) {
    const float q = level_fast(x, fl, rmax);
    const double qd = static_cast<double>(q);
    const double d = fma(s, qd, -static_cast<double>(x));
    e = fma(d, d, e);
    g = fma(d, qd, g);
}

__device__ __forceinline__ void elem_exact(float x, double inv, double dmin, double dmax,
                                           double s, double& e, double& g) {
    const double xd = static_cast<double>(x);
    const double qd = level_exact(xd, inv, dmin, dmax);
    const double d = fma(s, qd, -xd);
    e = fma(d, d, e);
    g = fma(d, qd, g);
}

template <int L, int W, bool GLOBAL>
__global__ void __launch_bounds__(512) k_qrange(const TDesc* __restrict__ td,
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
        const double mean = st->mean, thr = st->thr;
        const int mask = st->mask;
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
                        v[k] = (mask && is_outlier(x, mean, thr)) ? 0.f : x;
                    }
                }
            }
            *reinterpret_cast<float4*>(strip + static_cast<size_t>(cc) * rstride + 4 * rq) =
                make_float4(v[0], v[1], v[2], v[3]);
        }
        __syncthreads();

        // Idle columns: whole warps (W == 1) or whole teams (W > 1) skip.
        if (W == 1) {
            if (warp * (32 / L) >= g.ncols) continue;
        } else if (team >= g.ncols) {
            continue;
        }
        const float4* col4 =
            reinterpret_cast<const float4*>(strip + static_cast<size_t>(team) * rstride);
        int parity = 0;

        // initial_scale over the normals (rtn.cpp:81-86): max is order-free.
        float mx = 0.f;
        for (int k = 0; k < K; ++k) {
            const float4 x = col4[pt + k * P];
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
        }
        mx = team_max<L, W>(mx, red, team, wi, lane, teams, parity);
        const double s0_raw = initial_scale_from_max(static_cast<double>(mx), cfg.lmax);
        const int64_t gc = d.col_base + g.col0 + team;
        const bool writer = (pt == 0) && (team < g.ncols);

        if (!optimize) {
            if (writer) sc.s0[gc] = s0_raw;
            continue;
        }

        // ---- Adam loop (optimize.cpp:138-167) ----
        double s = snap(s0_raw);
        const double s0 = s;
        double m = 0.0, v = 0.0;
        double e0 = 0.0, best_err = 0.0, best_s = s, fixed_s = s, fixed_err = 0.0;
        const float guard = cfg.guard;
        for (int t = 0;; ++t) {
            const double inv = __ddiv_rn(1.0, s);
            const FastLevel fl{__double2float_rn(inv), static_cast<float>(cfg.lmin),
                               static_cast<float>(cfg.lmax)};
            double ea = 0.0, eb = 0.0, ga = 0.0, gb = 0.0;
            float rmax = 0.f;
#pragma unroll 4
            for (int k = 0; k < K; ++k) {
                const float4 x = col4[pt + k * P];
                elem_fast(x.x, fl, s, rmax, ea, ga);
                elem_fast(x.y, fl, s, rmax, eb, gb);
                elem_fast(x.z, fl, s, rmax, ea, ga);
                elem_fast(x.w, fl, s, rmax, eb, gb);
            }
            if (rmax >= guard) {
                // Some element sits within the fp32 error band of a rounding
                // boundary: redo this thread's slice with exact fp64 levels.
                ea = eb = ga = gb = 0.0;
                for (int k = 0; k < K; ++k) {
                    const float4 x = col4[pt + k * P];
                    elem_exact(x.x, inv, dmin, dmax, s, ea, ga);
                    elem_exact(x.y, inv, dmin, dmax, s, eb, gb);
                    elem_exact(x.z, inv, dmin, dmax, s, ea, ga);
                    elem_exact(x.w, inv, dmin, dmax, s, eb, gb);
                }
            }
            double err = ea + eb, gr = ga + gb;
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
        if (writer) {
            sc.s0[gc] = s0;
            double chosen;
            if (cfg.select == EZQ_SELECT_FIXED)
                chosen = (fixed_err <= e0) ? fixed_s : s0;  // optimize.cpp:169-178
            else
                chosen = best_s;
            sc.s_opt[gc] = chosen;
        }
    }
}

// ---- K3b: reference-order errors -------------------------------------------
// Block = 64 threads = one tile of 32 adjacent columns x {rtn, final}; each
// thread walks its column in ascending row order (coalesced 128-byte rows per
// warp) with the reference's separate-rounding accumulation.
__global__ void __launch_bounds__(64) k_seq_errors(const TDesc* __restrict__ td,
                                                   const int2* __restrict__ tiles, Scratch sc,
                                                   CfgDev cfg) {
    const int2 tile = tiles[blockIdx.x];
    const TDesc& d = td[tile.x];
    const int lane = threadIdx.x & 31, which = threadIdx.x >> 5;
    const int64_t c = tile.y + lane;
    if (c >= d.cols) return;
    const int64_t gc = d.col_base + c;
    const bool eq = cfg.mode == EZQ_MODE_EASYQUANT;
    double s;
    if (which == 0) {
        // Easyquant: error at the snapped initial scale (optimize.cpp:138-141);
        // Rtn / OutliersOnly: at float(initial_scale) (pipeline.cpp:52-55).
        s = eq ? sc.s0[gc] : static_cast<double>(__double2float_rn(sc.s0[gc]));
    } else {
        if (!eq || sc.s_opt[gc] == sc.s0[gc]) {
            sc.err_fin[gc] = __longlong_as_double(0x7ff8000000000000ll);  // "same as rtn"
            return;
        }
        s = sc.s_opt[gc];
    }
    if (!(s > 0.0) || !isfinite(s)) {  // check_scale (rtn.cpp:19-22)
        d.st->scale_zero = 1;
        s = 1.0;
    }
    const TStats* st = d.st;
    const double mean = st->mean, thr = st->thr;
    const int mask = st->mask;
    const double inv = __ddiv_rn(1.0, s);
    const FastLevel fl{__double2float_rn(inv), static_cast<float>(cfg.lmin),
                       static_cast<float>(cfg.lmax)};
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const float guard = cfg.guard;
    double err = 0.0;
    const float* p = d.W + c;
    const int64_t R = d.rows, C = d.cols;
#pragma unroll 8
    for (int64_t r = 0; r < R; ++r) {
        const float x = p[r * C];
        if (mask && is_outlier(x, mean, thr)) continue;
        float rm = 0.f;
        double q = static_cast<double>(level_fast(x, fl, rm));
        if (rm >= guard) q = level_exact(static_cast<double>(x), inv, dmin, dmax);
        const double dd = __dsub_rn(__dmul_rn(s, q), static_cast<double>(x));
        err = __dadd_rn(err, __dmul_rn(dd, dd));
    }
    if (which == 0)
        sc.err_rtn[gc] = err;
    else
        sc.err_fin[gc] = err;
}

// Per column: pick the stored scale, keep final <= rtn per column, and
// publish float scales + 1/scale for the packer.
__global__ void __launch_bounds__(32) k_col_finalize(const TDesc* __restrict__ td,
                                                     const int2* __restrict__ tiles, Scratch sc,
                                                     CfgDev cfg) {
    const int2 tile = tiles[blockIdx.x];
    const TDesc& d = td[tile.x];
    const int64_t c = tile.y + threadIdx.x;
    if (c >= d.cols) return;
    const int64_t gc = d.col_base + c;
    const double rtn = sc.err_rtn[gc];
    double fin = rtn;
    float scale;
    if (cfg.mode == EZQ_MODE_EASYQUANT) {
        double s = sc.s_opt[gc];
        const double f = sc.err_fin[gc];
        if (!isnan(f)) {
            if (f > rtn) {
                s = sc.s0[gc];  // tree/sequential near-tie: keep the initial scale
            } else {
                fin = f;
            }
        }
        scale = __double2float_rn(s);
    } else {
        scale = __double2float_rn(sc.s0[gc]);
    }
    sc.err_fin[gc] = fin;
    d.scales[c] = scale;
    sc.inv[gc] = scale > 0.f ? __ddiv_rn(1.0, static_cast<double>(scale)) : 1.0;
}

// Column-ordered tensor totals (pipeline.cpp:96-103).
__global__ void k_tensor_totals(const TDesc* __restrict__ td, int ntens, Scratch sc) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntens) return;
    const TDesc& d = td[t];
    double rtn = 0.0, fin = 0.0;
    for (int64_t c = 0; c < d.cols; ++c) {
        rtn = __dadd_rn(rtn, sc.err_rtn[d.col_base + c]);
        fin = __dadd_rn(fin, sc.err_fin[d.col_base + c]);
    }
    d.st->rtn_error = rtn;
    d.st->final_error = fin;
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

// Geometry: ~128 elements per thread per step, 12-16 warps per CTA.
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
    const int P = kl.L * kl.W;
    kl.rpad = static_cast<int>(((rows + 4 * P - 1) / (4 * P)) * (4 * P));
    kl.rstride = kl.rpad + 4;
    const int max_warps = 16;
    const int team_unit = (kl.W == 1) ? 32 / kl.L : 1;  // teams per warp-granule
    int teams = (kl.W == 1) ? max_warps * (32 / kl.L) : max_warps / kl.W;
    auto smem_for = [&](int t) {
        return static_cast<size_t>(t) * kl.rstride * sizeof(float) +
               static_cast<size_t>(2) * t * kl.W * 2 * sizeof(double);
    };
    while (teams > team_unit && smem_for(teams) > static_cast<size_t>(max_smem)) teams -= team_unit;
    kl.global_strip = smem_for(teams) > static_cast<size_t>(max_smem);
    if (kl.global_strip) teams = (kl.W == 1) ? team_unit : 1;
    kl.teams = teams;
    kl.threads = (kl.W == 1) ? ((teams * kl.L + 31) / 32) * 32 : teams * kl.W * 32;
    kl.smem = kl.global_strip ? static_cast<size_t>(2) * teams * kl.W * 2 * sizeof(double)
                              : smem_for(teams);
    return kl;
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
    k_seq_errors<<<ntiles, 64, 0, st>>>(td, tiles, sc, cfg);
    count_launch();
}

void launch_col_finalize(const TDesc* td, const int2* tiles, int ntiles, Scratch sc,
                         CfgDev cfg, cudaStream_t st) {
    if (ntiles == 0) return;
    k_col_finalize<<<ntiles, 32, 0, st>>>(td, tiles, sc, cfg);
    count_launch();
}

void launch_tensor_totals(const TDesc* td, int ntens, Scratch sc, cudaStream_t st) {
    k_tensor_totals<<<(ntens + 63) / 64, 64, 0, st>>>(td, ntens, sc);
    count_launch();
}

}  // namespace ezq
