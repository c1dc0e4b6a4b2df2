// K3s: the per-column q_range Adam loop on SORTED normals (SURVEY.md §8
// rows a6-a11; reference optimize.cpp:118-184, eval_dense :30-51).
//
// The reference evaluates err(s) = sum (s*q_i - x_i)^2 and grad(s) =
// 2 sum (s*q_i - x_i) q_i over all normals at every one of the steps+1
// scales, q_i = clamp(llround(x_i * (1/s))). The level is a monotone step
// function of x, so over the column's normals sorted ascending every level
// v owns one contiguous range, and
//
//   err = sum_v [ n_v (s v)^2 - 2 s v S1_v + S2_v ],
//   grad/2 = sum_v [ n_v s v^2 - v S1_v ],
//
// with n_v, S1_v = sum x, S2_v = sum x^2 over the range. Per Adam step the
// kernel therefore only (a) moves the 2^k - 1 range boundaries and (b) moves
// the boundary prefix sums by the elements that crossed:
//  - boundaries: level(x) >= v  <=>  RN(x * RN(1/s)) >= v - 1/2 (> for
//    v <= 0: half away from zero), so each boundary is "x >= X_v" for one
//    float X_v, found with the reference's exact fp64 product at a couple of
//    candidate floats; the search over the sorted column is then float
//    compares, galloping from the previous step's position;
//  - prefix sums: exact 128-bit fixed point (LSB 2^(E-109) for x, 2^(2E-109)
//    for x^2, |x| < 2^E), so crossings are integer adds and every sum is
//    exact and order-independent; per level the sums go to double-double,
//    the level's err/grad terms are formed there (they cancel by ~10 bits),
//    rounded once, and summed over levels in fixed butterfly order. err and
//    grad are thus the exact values to ~1e-16 -- the agreement regime of the
//    reference's own sequential sums and of the streaming K3.
//
// Work per column: one bitonic sort in shared memory plus O(levels) per step
// instead of O(rows). Two columns per warp for k <= 4 (16 levels per group
// of 16 lanes), one for k = 5; k > 5 uses the streaming K3.
#include "ezq_kernels.cuh"

namespace ezq {
namespace {

typedef __int128 i128;
typedef unsigned __int128 u128;

struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    const DD t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, fma(a, b, -p)};
}
__device__ __forceinline__ DD dd_mul_d(DD a, double b) {
    DD p = dd_prod(a.hi, b);
    p.lo = fma(a.lo, b, p.lo);
    return two_sum(p.hi, p.lo);
}

// x * 2^bias as a 128-bit integer, truncated toward zero (exact whenever the
// float's LSB is at or above 2^-bias: everything but negligible tails).
__device__ __forceinline__ i128 fix_f(float x, int bias) {
    const unsigned u = __float_as_uint(x);
    int ex = static_cast<int>((u >> 23) & 255u);
    unsigned m = u & 0x7fffffu;
    if (ex == 0) {
        if (m == 0) return 0;
        ex = 1;
    } else {
        m |= 0x800000u;
    }
    const int sh = ex - 150 + bias;  // |x| = m * 2^(ex - 150)
    i128 v = static_cast<i128>(m);
    if (sh >= 0)
        v <<= sh;
    else
        v = sh <= -24 ? static_cast<i128>(0) : (v >> -sh);
    return (u >> 31) ? -v : v;
}
// y >= 0 (here x^2, exact in fp64) * 2^bias, truncated.
__device__ __forceinline__ i128 fix_d(double y, int bias) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(y));
    int ex = static_cast<int>((u >> 52) & 2047u);
    unsigned long long m = u & 0xfffffffffffffull;
    if (ex == 0) {
        if (m == 0) return 0;
        ex = 1;
    } else {
        m |= 0x10000000000000ull;
    }
    const int sh = ex - 1075 + bias;
    i128 v = static_cast<i128>(m);
    if (sh >= 0)
        v <<= sh;
    else
        v = sh <= -53 ? static_cast<i128>(0) : (v >> -sh);
    return v;
}
// 128-bit integer * 2^-bias -> double-double (top 53 bits exact, the rest
// rounded once: relative error ~2^-106).
__device__ __forceinline__ DD unfix(i128 v, int bias) {
    if (v == 0) return {0.0, 0.0};
    const bool neg = v < 0;
    const u128 a = neg ? static_cast<u128>(-v) : static_cast<u128>(v);
    const unsigned long long hi = static_cast<unsigned long long>(a >> 64);
    const unsigned long long lo = static_cast<unsigned long long>(a);
    const int lz = hi ? __clzll(static_cast<long long>(hi)) : 64 + __clzll(static_cast<long long>(lo));
    const int top = 128 - lz;
    const int drop = top > 53 ? top - 53 : 0;
    const unsigned long long head = static_cast<unsigned long long>(a >> drop);  // <= 53 bits
    const u128 rest = a - (static_cast<u128>(head) << drop);                      // < 2^drop
    const int drop2 = drop > 64 ? drop - 64 : 0;
    const unsigned long long tail = static_cast<unsigned long long>(rest >> drop2);
    double d1 = ldexp(static_cast<double>(head), drop - bias);
    double d2 = ldexp(static_cast<double>(tail), drop2 - bias);
    if (neg) d1 = -d1, d2 = -d2;
    return two_sum(d1, d2);
}

__device__ __forceinline__ i128 join128(long long hi, unsigned long long lo) {
    return (static_cast<i128>(hi) << 64) | static_cast<i128>(lo);
}
__device__ __forceinline__ i128 shfl_up_i128(i128 v, int d, int width) {
    const unsigned long long lo = __shfl_up_sync(0xffffffffu, static_cast<unsigned long long>(v), d, width);
    const long long hi = __shfl_up_sync(0xffffffffu, static_cast<long long>(v >> 64), d, width);
    return join128(hi, lo);
}
__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int o, int width) {
    const unsigned long long lo = __shfl_xor_sync(0xffffffffu, static_cast<unsigned long long>(v), o, width);
    const long long hi = __shfl_xor_sync(0xffffffffu, static_cast<long long>(v >> 64), o, width);
    return join128(hi, lo);
}

// Smallest float x with level(x) >= v at scale s: RN(x*inv) >= t (> t for
// v <= 0), t = v - 1/2. Candidates start at RN32(t*s) (t*s is exact in
// fp64) and step by float neighbours (one or two steps in practice).
__device__ __forceinline__ float level_threshold(int v, double s, double inv) {
    const double t = static_cast<double>(v) - 0.5;
    const bool strict = v <= 0;
    const float kInf = __int_as_float(0x7f800000);
    float c = __double2float_rn(__dmul_rn(t, s));
    auto pred = [&](float x) {
        const double u = __dmul_rn(static_cast<double>(x), inv);
        return strict ? (u > t) : (u >= t);
    };
    if (pred(c)) {
        for (int i = 0; i < 16; ++i) {
            const float p = nextafterf(c, -kInf);
            if (!pred(p)) break;
            c = p;
        }
    } else {
        for (int i = 0; i < 16; ++i) {
            c = nextafterf(c, kInf);
            if (pred(c)) break;
        }
    }
    return c;
}

// First index in [0, n] with a[k] >= X (a ascending; n acts as +inf),
// galloping from `guess`.
__device__ __forceinline__ int search_from(const float* a, int n, int guess, float X) {
    guess = min(max(guess, 0), n);
    int lo, hi;
    if (guess == n || a[guess] >= X) {
        hi = guess;
        int step = 1, p = guess - 1;
        while (p >= 0 && a[p] >= X) {
            hi = p;
            step <<= 1;
            p = hi - step;
        }
        lo = max(p + 1, 0);
    } else {
        lo = guess + 1;
        int step = 1, p = guess + 1;
        while (p < n && a[p] < X) {
            lo = p + 1;
            step <<= 1;
            p = lo + step - 1;
        }
        hi = min(p, n);
    }
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] >= X)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

// Bitonic sort of a power-of-two shared-memory array by the G lanes of a
// group; `live` groups sort, the others only meet the warp barriers.
template <int G>
__device__ void group_bitonic_sort(float* a, int n, int gl, bool live) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (live) {
                for (int p = gl; p < (n >> 1); p += G) {
                    const int i = ((p / j) * 2 * j) + (p % j);
                    const int ij = i + j;
                    const float x = a[i], y = a[ij];
                    if ((x > y) == ((i & k) == 0)) {
                        a[i] = y;
                        a[ij] = x;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Exact fixed-point sums of x and x^2 over a[lo, hi), by the G lanes of a
// group (every lane of the warp must call it: the shuffles are warp-wide).
template <int G>
__device__ __forceinline__ void group_range_fix(const float* a, int lo, int hi, int gl, int b1, int b2, i128& s1,
                                                i128& s2) {
    i128 p1 = 0, p2 = 0;
    for (int k = lo + gl; k < hi; k += G) {
        const float x = a[k];
        const double xd = static_cast<double>(x);
        p1 += fix_f(x, b1);
        p2 += fix_d(__dmul_rn(xd, xd), b2);
    }
#pragma unroll
    for (int o = G / 2; o; o >>= 1) {
        p1 += shfl_xor_i128(p1, o, G);
        p2 += shfl_xor_i128(p2, o, G);
    }
    s1 = p1;
    s2 = p2;
}

// CPW columns per warp (groups of G = 32 / CPW lanes). Lane gl of a group
// owns boundary gl (between levels lmin+gl and lmin+gl+1) and level gl.
template <int CPW>
__global__ void __launch_bounds__(256) k_qrange_sorted(const TDesc* __restrict__ td,
                                                       const K3Group* __restrict__ groups, int ngroups,
                                                       Scratch sc, CfgDev cfg, int npad, int cpb) {
    constexpr int G = 32 / CPW;
    extern __shared__ __align__(16) float strip[];  // [cpb][npad]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int gl = lane % G, grp = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
    const int nb = cfg.lmax - cfg.lmin;  // boundaries (<= G - 1)
    const bool optimize = cfg.mode == EZQ_MODE_EASYQUANT;
    const float kInf = __int_as_float(0x7f800000);

    for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        const K3Group g = groups[gi];
        const TDesc& d = td[g.tensor];
        const float olo = d.st->olo, ohi = d.st->ohi;
        const int64_t R = d.rows, C = d.cols;
        __syncthreads();  // previous group's columns fully consumed
        for (int idx = tid; idx < cpb * npad; idx += blockDim.x) {
            const int cc = idx % cpb, r = idx / cpb;
            float v = kInf;
            if (cc < g.ncols && r < R) {
                const float x = d.W[static_cast<int64_t>(r) * C + g.col0 + cc];
                v = is_outlier_f(x, olo, ohi) ? kInf : x;
            }
            strip[cc * npad + r] = v;
        }
        __syncthreads();

        for (int base = warp * CPW; base < cpb; base += nwarps * CPW) {  // warp-uniform
            const int cc = base + grp;
            const bool live = cc < g.ncols;
            float* a = strip + min(cc, cpb - 1) * npad;
            group_bitonic_sort<G>(a, npad, gl, live);
            int n = 0;
            if (live) {
                int lo = 0, hi = npad;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (a[mid] < kInf)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                n = lo;
            }
            const double mx =
                n ? fmax(fabs(static_cast<double>(a[0])), fabs(static_cast<double>(a[n - 1]))) : 0.0;
            const double s0_raw = initial_scale_from_max(mx, cfg.lmax);
            double s_rtn = static_cast<double>(__double2float_rn(s0_raw));
            double s_fin = s_rtn;
            if (optimize) {  // uniform across the warp
                // fixed-point biases from the column's magnitude: |x| < 2^E
                const int E = mx > 0.0 ? ilogb(mx) + 1 : 0;
                const int b1 = 109 - E, b2 = 109 - 2 * E;
                double s = snap(s0_raw);
                const double s0 = s;
                double m = 0.0, vv = 0.0;
                double e0 = 0.0, best_err = 0.0, best_s = s, fixed_s = s, fixed_err = 0.0;
                double inv = __ddiv_rn(1.0, s);
                const bool own_b = live && gl < nb;
                int ib = n;
                if (own_b) ib = search_from(a, n, n >> 1, level_threshold(cfg.lmin + gl + 1, s, inv));
                // level sums, then prefix sums at the boundaries (all exact)
                i128 P1 = 0, P2 = 0;
                for (int j = 0; j <= nb; ++j) {
                    const int lo = j == 0 ? 0 : __shfl_sync(0xffffffffu, ib, j - 1, G);
                    const int hi = j == nb ? n : __shfl_sync(0xffffffffu, ib, j, G);
                    i128 s1, s2;
                    group_range_fix<G>(a, lo, hi, gl, b1, b2, s1, s2);
                    if (gl == j) P1 = s1, P2 = s2;
                }
#pragma unroll
                for (int o = 1; o < G; o <<= 1) {
                    const i128 u1 = shfl_up_i128(P1, o, G), u2 = shfl_up_i128(P2, o, G);
                    if (gl >= o) P1 += u1, P2 += u2;
                }
                for (int t = 0;; ++t) {
                    // ---- err and grad at s from the level ranges ----
                    double ev = 0.0, gv = 0.0;
                    {
                        const int up_lo = __shfl_up_sync(0xffffffffu, ib, 1, G);
                        const i128 lo1 = shfl_up_i128(P1, 1, G), lo2 = shfl_up_i128(P2, 1, G);
                        const int lo_i = gl == 0 ? 0 : up_lo;
                        const int hi_i = gl == nb ? n : ib;
                        if (gl <= nb && hi_i > lo_i) {
                            const i128 S1 = gl == 0 ? P1 : P1 - lo1;
                            const i128 S2 = gl == 0 ? P2 : P2 - lo2;
                            const double v = static_cast<double>(cfg.lmin + gl);
                            const double cnt = static_cast<double>(hi_i - lo_i);
                            const double sv = __dmul_rn(s, v);  // exact: float * small int
                            const DD s1 = unfix(S1, b1), s2 = unfix(S2, b2);
                            DD e = dd_mul_d(dd_prod(sv, sv), cnt);  // n (s v)^2
                            e = dd_add(e, dd_mul_d(s1, -2.0 * sv));  // - 2 s v S1
                            e = dd_add(e, s2);                       // + S2
                            DD q = dd_mul_d(dd_prod(sv, v), cnt);   // n s v^2
                            q = dd_add(q, dd_mul_d(s1, -v));         // - v S1
                            ev = __dadd_rn(e.hi, e.lo);
                            gv = __dadd_rn(q.hi, q.lo);
                        }
                    }
#pragma unroll
                    for (int o = G / 2; o; o >>= 1) {
                        ev = __dadd_rn(ev, __shfl_xor_sync(0xffffffffu, ev, o, G));
                        gv = __dadd_rn(gv, __shfl_xor_sync(0xffffffffu, gv, o, G));
                    }
                    const double err = ev;
                    const double grad = 2.0 * gv;
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
                    s = snap(adam_update(m, vv, s, grad, cfg.bc1[t + 1], cfg.bc2[t + 1], cfg.adam));
                    inv = __ddiv_rn(1.0, s);
                    // ---- move the boundaries and their exact prefix sums ----
                    int nib = ib;
                    if (own_b) nib = search_from(a, n, ib, level_threshold(cfg.lmin + gl + 1, s, inv));
                    const int lo = min(nib, ib), hi = max(nib, ib);
                    const bool grow = nib > ib;
                    const bool big = (hi - lo) > 8;
                    if (!big) {
                        for (int k = lo; k < hi; ++k) {
                            const float x = a[k];
                            const double xd = static_cast<double>(x);
                            const i128 f1 = fix_f(x, b1), f2 = fix_d(__dmul_rn(xd, xd), b2);
                            if (grow)
                                P1 += f1, P2 += f2;
                            else
                                P1 -= f1, P2 -= f2;
                        }
                    }
                    // large moves: the group sums each range cooperatively; all
                    // groups iterate the warp-wide maximum count (uniform shuffles)
                    const unsigned bigw = __ballot_sync(0xffffffffu, big);
                    unsigned mine = bigw & gmask;
                    int rounds = __popc(mine);
#pragma unroll
                    for (int o = G; o < 32; o <<= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
                    for (int it = 0; it < rounds; ++it) {
                        const bool act = mine != 0;
                        const int src = act ? ((__ffs(mine) - 1) % G) : 0;
                        if (act) mine &= mine - 1;
                        const int blo = __shfl_sync(0xffffffffu, lo, src, G);
                        const int bhi = __shfl_sync(0xffffffffu, hi, src, G);
                        const bool bgrow = __shfl_sync(0xffffffffu, grow, src, G) != 0;
                        i128 s1, s2;
                        group_range_fix<G>(a, act ? blo : 0, act ? bhi : 0, gl, b1, b2, s1, s2);
                        if (act && gl == src) {
                            if (bgrow)
                                P1 += s1, P2 += s2;
                            else
                                P1 -= s1, P2 -= s2;
                        }
                    }
                    ib = nib;
                }
                if (cfg.select == EZQ_SELECT_FIXED)
                    s_fin = (fixed_err <= e0) ? fixed_s : s0;  // optimize.cpp:169-178
                else
                    s_fin = best_s;
                s_rtn = s0;
            }
            if (live && gl == 0) {
                const int64_t gcol = d.col_base + g.col0 + cc;
                sc.s_rtn[gcol] = s_rtn;
                sc.s_fin[gcol] = s_fin;
            }
        }
    }
}

}  // namespace

int k3s_npad(int64_t rows) {
    int n = 32;
    while (n < rows) n <<= 1;
    return n;
}

size_t k3s_smem(int64_t rows, int cpb) { return sizeof(float) * static_cast<size_t>(k3s_npad(rows)) * cpb; }

bool k3s_supported(int bits) { return bits >= 2 && bits <= 5; }

void launch_k3_sorted(int64_t rows, int cpb, const TDesc* td, const K3Group* groups, int ngroups, Scratch sc,
                      CfgDev cfg, int grid, cudaStream_t st) {
    if (ngroups == 0) return;
    const int npad = k3s_npad(rows);
    const size_t smem = k3s_smem(rows, cpb);
    const int cpw = (cfg.lmax - cfg.lmin) <= 15 ? 2 : 1;
    const int threads = 32 * ((cpb + cpw - 1) / cpw);
    if (cpw == 2) {
        auto k = k_qrange_sorted<2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k<<<grid, threads, smem, st>>>(td, groups, ngroups, sc, cfg, npad, cpb);
    } else {
        auto k = k_qrange_sorted<1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k<<<grid, threads, smem, st>>>(td, groups, ngroups, sc, cfg, npad, cpb);
    }
    count_launch();
}

}  // namespace ezq
