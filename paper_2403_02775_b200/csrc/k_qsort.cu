// K3s: the per-column q_range Adam loop on SORTED normals (SURVEY.md §8
// rows a6-a11; reference optimize.cpp:118-184, eval_dense :30-51).
//
// The reference evaluates err(s) = sum (s*q_i - x_i)^2 and grad(s) =
// 2 sum (s*q_i - x_i) q_i over all normals at every one of the steps+1
// scales, q_i = clamp(llround(x_i * RN(1/s))). Regrouped,
//
//   err(s) = A s^2 - 2 Q s + C,   grad(s) = 2 (A s - Q),
//   A = sum q^2,  Q = sum q x,  C = sum x^2 (constant per column).
//
// The level is a monotone step function of x, so on the column's normals
// sorted ascending, "level(x) >= j" holds on a suffix [ib_j, n) for each of
// the 2^k - 1 level thresholds j = lmin+1 .. lmax, and
//
//   A = sum_{j>=1} (2j-1) (n - ib_j)  +  sum_{j<=0} (1-2j) ib_j,
//   Q = sum_{j>=1} S(ib_j)  -  sum_{j<=0} P(ib_j),
//
// with S(k) = sum_{i>=k} x_i, P(k) = sum_{i<k} x_i. So after one sort per
// column a step costs O(levels), not O(rows):
//  - threshold j: level(x) >= j  <=>  RN(x * inv) >= j - 1/2 (> for j <= 0:
//    half away from zero), i.e. "x >= X_j" for one float X_j, found with the
//    reference's own fp64 product at a couple of candidate floats; ib_j is a
//    galloping search from the previous step's position;
//  - S(ib_j) and P(ib_j) are single loads from a per-column table written
//    once after the sort (suffix sums over x >= 0, prefix sums over x < 0).
//    Every sum used spans same-sign elements of magnitude >= s/2, so it is
//    EXACT in fp64 (<= 13 + 24 + log2(max/(s/2)) significant bits, < 53
//    unless s falls below max * 2^-16), and so are A, Q and their
//    cross-lane sums, in any order;
//  - grad = 2 (A s - Q) is rounded once from exact terms; the selection
//    compares err - C = A s^2 - 2 Q s as exact double-doubles (C is constant
//    per column), so both are the exact values (to ~2^-100) -- at least as
//    close to the true sums as the reference's own sequential fp64 sums (the
//    agreement regime of DESIGN.md §4).
//
// Layout: a CTA stages cpb columns, sorts each with a block radix sort in
// registers and replaces it by its (rows + 2)-double table; the x values are
// recovered exactly as differences of neighbouring entries. Then two columns
// per warp (groups of 16 lanes, k <= 4) or one (k = 5) run the loop, lane j
// owning threshold lmin + 1 + j.
#include <algorithm>
#include <cstdlib>

#include <cub/block/block_radix_sort.cuh>

#include "ezq_kernels.cuh"

namespace ezq {
namespace {

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
// Normalized double-doubles (hi = RN(hi + lo)) compare lexicographically.
__device__ __forceinline__ bool dd_lt(DD a, DD b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
__device__ __forceinline__ bool dd_le(DD a, DD b) { return a.hi < b.hi || (a.hi == b.hi && a.lo <= b.lo); }
// err(s) - C = A s^2 - 2 Q s (s a float: s^2 exact), normalized: the
// selection only compares errors of one column, so the column constant
// C = sum x^2 drops out and the comparison is of the exact values.
__device__ __forceinline__ DD err_minus_c(double Ad, double q, double s) {
    const DD p1 = dd_prod(Ad, __dmul_rn(s, s));
    const DD p2 = dd_prod(__dmul_rn(-2.0, q), s);
    const DD h = two_sum(p1.hi, p2.hi);
    return two_sum(h.hi, __dadd_rn(h.lo, __dadd_rn(p1.lo, p2.lo)));
}

// ---- selection near-ties -------------------------------------
// The reference's eval_dense sums the squared residuals sequentially in fp64,
// so its error of a step is within gamma_n * err of the exact one (n
// rounded products and additions of non-negative terms, gamma_n = n u /
// (1 - n u)); its gradient sum is exact (every partial sum of the d*q terms
// is a multiple of one quantum and fits 53 bits), so only the best-error
// selection can differ. A step whose exact error lies within
// gamma * (err_a + err_b) of the running best is a candidate: the column's
// candidates (distinct scales, step order) go to sc.tie_* and
// k_resolve_ties re-evaluates them in reference order. gamma here is
// (n + 8) u with 1% slack, in float (the comparison uses double approximations
// of the exact errors, ~1e-16 relative, far inside the slack).
__device__ __forceinline__ float tie_gamma(int n) {
    return (static_cast<float>(n) + 8.0f) * 1.1102230246251565e-16f * 1.01f;
}
// Pre-filter of the per-step check: the window best -/+ gamma (2 best + 2 C)
// (with slack) around the running best; a step outside it is certified
// (a far new best only empties the list), so the hot loop pays one compare
// per step and tie_step runs only inside it.
__device__ __forceinline__ void tie_window(double best, double cfull, float gam, double& lo, double& hi) {
    const double w = static_cast<double>(gam) * 2.0002 * __dadd_rn(best, cfull);
    lo = __dsub_rn(best, w);  // a new best at or above lo is near the old one
    hi = __dadd_rn(best, w);  // a later step at or below hi is near the best
}
// Candidate bookkeeping of one column, kept by its writer lane (the running
// count in a register; the list in global memory, touched only by near
// steps). best/err are err - C; cfull
// = C (an estimate) converts to full errors. The list (sc.tie_s / tie_e,
// step order) holds the distinct scales whose exact errors lie within the
// bound of the running best: a new best drops the entries now beyond it (the
// filter reads back the writer's own stores), a far new best empties it.
// count > cap: a candidate was lost (the column takes the whole-loop
// fallback). Out of line: the slow path's registers stay out of the loop.
__device__ __forceinline__ void tie_step(int& nc, const Scratch& sc, int64_t gcol, int cap, bool lt, double err_hi,
                                         double err_lo, double best_hi, double best_lo, double s, double best_s,
                                         float gam, double cfull) {
    if (!lt && s == best_s) return;  // same scale: same error in both orders
    double* ts = sc.tie_s + gcol * kTieMax;
    double* te = sc.tie_e + gcol * kTieMax;
    const double gap = fabs(__dadd_rn(__dsub_rn(err_hi, best_hi), __dsub_rn(err_lo, best_lo)));
    const double ef = __dadd_rn(err_hi, cfull), bf = __dadd_rn(best_hi, cfull);
    auto push = [&](double sv, double e) {
        if (nc < cap) ts[nc] = sv, te[nc] = e;
        ++nc;
    };
    if (gap <= static_cast<double>(gam) * __dadd_rn(ef, bf)) {
        if (nc == 0) {
            push(best_s, bf);
        } else if (lt && nc <= cap) {  // keep the entries still within the bound of the new best
            int k = 0;
            for (int j = 0; j < nc; ++j) {
                const double e = te[j];
                if (__dsub_rn(e, ef) <= static_cast<double>(gam) * __dadd_rn(e, ef)) {
                    ts[k] = ts[j];
                    te[k] = e;
                    ++k;
                }
            }
            nc = k;
        }
        push(s, ef);
    } else if (lt) {
        nc = 0;  // every earlier candidate is now beyond the bound
    }
}

// fixed-step selection (optimize.cpp:169-178): fixed_err <= e0 inside the bound
__device__ __forceinline__ void tie_fixed(const Scratch& sc, int64_t gcol, double fe_hi, double fe_lo, double e0_hi,
                                       double e0_lo, double fs, double s0, float gam, double cfull) {
    int nc = 0;
    if (fs != s0) {
        const double gap = fabs(__dadd_rn(__dsub_rn(fe_hi, e0_hi), __dsub_rn(fe_lo, e0_lo)));
        const double ef = __dadd_rn(fe_hi, cfull), bf = __dadd_rn(e0_hi, cfull);
        if (gap <= static_cast<double>(gam) * __dadd_rn(ef, bf)) {
            sc.tie_s[gcol * kTieMax] = s0, sc.tie_e[gcol * kTieMax] = bf;
            sc.tie_s[gcol * kTieMax + 1] = fs, sc.tie_e[gcol * kTieMax + 1] = ef;
            nc = 2 | kTieFixed;
        }
    }
    sc.tie_n[gcol] = nc;
}

// Smallest float x with level(x) >= v at scale s: RN(x*inv) >= t (> t for
// v <= 0), t = v - 1/2. Candidates start at RN32(t*s) (t*s is exact in
// fp64) and step by float neighbours (one or two steps in practice).
__device__ __forceinline__ float level_threshold(int v, double s, double inv) {
    const double t = static_cast<double>(v) - 0.5;
    const bool strict = v <= 0;
    const float kInf = __int_as_float(0x7f800000);
    auto pred = [&](float x) {
        const double u = __dmul_rn(static_cast<double>(x), inv);
        return strict ? (u > t) : (u >= t);
    };
    float c = __double2float_rn(__dmul_rn(t, s));
    if (c != 0.f && fabsf(c) < 3.0e38f) {
        // float neighbours by bit steps (c != 0, finite): down / up
        const int b = __float_as_int(c), dn = c > 0.f ? -1 : 1;
        const float pv = __int_as_float(b + dn), nx = __int_as_float(b - dn);
        const bool pp = pred(pv), pc = pred(c), pn = pred(nx);
        if (!pp && pc) return c;
        if (!pc && pn) return nx;
        c = pp ? pv : nx;  // rare: walk on below
    }
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

// The common case of level_threshold, branch-free: RN32(t s) or one of its
// float neighbours is the threshold (ok = false otherwise: call
// level_threshold). Keeps the hot loop free of divergent early returns.
__device__ __forceinline__ float level_threshold_fast(int v, double s, double inv, bool& ok) {
    const double t = static_cast<double>(v) - 0.5;
    const bool strict = v <= 0;
    auto pred = [&](float x) {
        const double u = __dmul_rn(static_cast<double>(x), inv);
        return strict ? (u > t) : (u >= t);
    };
    const float c = __double2float_rn(__dmul_rn(t, s));
    const int b = __float_as_int(c), dn = c > 0.f ? -1 : 1;
    const float pv = __int_as_float(b + dn), nx = __int_as_float(b - dn);
    const bool pp = pred(pv), pc = pred(c), pn = pred(nx);
    const bool a1 = !pp && pc, a2 = !pc && pn;
    ok = c != 0.f && fabsf(c) < 3.0e38f && (a1 || a2);
    return a1 ? c : nx;
}

// Column table: D[k] = P(k) for k <= kz (kz = count of x < 0), D[k + 1] =
// S(k) for kz <= k <= n. x_k = D[k+1] - D[k] (k < kz), D[k+1] - D[k+2]
// (kz <= k < n): exact wherever a threshold can fall.
struct ColInfo {
    int n, kz;
    float lo, hi;     // smallest / largest normal
    double chi, clo;  // C = sum x^2, double-double
};

// Per-slot table: D (dstride doubles, above), then the sorted normals as
// floats, +inf-padded to n + 16 (xs: the search runs on these).
struct ColTab {
    const double* D;
    const float* xs;
    int n;
};

// First index in [0, n] with xs[k] >= X (xs[k] = +inf for k >= n), galloping
// from `guess`.
__device__ __forceinline__ int search_from(const ColTab& c, int guess, float X) {
    const int n = c.n;
    guess = min(max(guess, 0), n);
    int lo, hi;
    if (guess == n || __ldg(c.xs + guess) >= X) {
        hi = guess;
        int step = 1, p = guess - 1;
        while (p >= 0 && __ldg(c.xs + p) >= X) {
            hi = p;
            step <<= 1;
            p = hi - step;
        }
        lo = max(p + 1, 0);
    } else {
        lo = guess + 1;
        int step = 1, p = guess + 1;
        while (p < n && __ldg(c.xs + p) < X) {
            lo = p + 1;
            step <<= 1;
            p = lo + step - 1;
        }
        hi = min(p, n);
    }
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(c.xs + mid) >= X)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

// Same, starting from a predicted index: an aligned window of sixteen floats
// (four 16-byte loads, one round trip) usually holds the answer; one window
// move, then the galloping search. `span` returns x[k0+15] - x[k0] of the
// final window (the local spacing for the next prediction; +inf/0 when the
// window reached the padding or a run of equal values).
__device__ __forceinline__ int search_near(const ColTab& c, int guess, float X, float& span) {
    int k0 = max(guess - 6, 0) & ~3;  // guess sits at k0 + 6 .. k0 + 9
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
        const float4* w = reinterpret_cast<const float4*>(c.xs + k0);
        const float4 a = __ldg(w), b = __ldg(w + 1), e = __ldg(w + 2), f = __ldg(w + 3);
        const int cnt = (a.x < X) + (a.y < X) + (a.z < X) + (a.w < X) + (b.x < X) + (b.y < X) + (b.z < X) +
                        (b.w < X) + (e.x < X) + (e.y < X) + (e.z < X) + (e.w < X) + (f.x < X) + (f.y < X) +
                        (f.z < X) + (f.w < X);
        if (cnt == 0 && k0 > 0) {
            k0 = max(k0 - 16, 0);
        } else if (cnt == 16) {
            k0 += 16;
        } else {
            span = f.w - a.x;  // 15 gaps: the local spacing for the next prediction
            return k0 + cnt;
        }
    }
    span = 0.f;
    return search_from(c, k0, X);
}

// One aligned 16-float window around the predicted index (the common case
// of search_near, branch-free); ok = false when the answer lies outside it.
__device__ __forceinline__ int search_window(const ColTab& c, int guess, float X, float& span, bool& ok) {
    const int k0 = max(guess - 6, 0) & ~3;
    const float4* w = reinterpret_cast<const float4*>(c.xs + k0);
    const float4 a = __ldg(w), b = __ldg(w + 1), e = __ldg(w + 2), f = __ldg(w + 3);
    const int cnt = (a.x < X) + (a.y < X) + (a.z < X) + (a.w < X) + (b.x < X) + (b.y < X) + (b.z < X) + (b.w < X) +
                    (e.x < X) + (e.y < X) + (e.z < X) + (e.w < X) + (f.x < X) + (f.y < X) + (f.z < X) + (f.w < X);
    ok = cnt < 16 && (cnt > 0 || k0 == 0);
    span = f.w - a.x;
    return k0 + cnt;
}

constexpr int kSortRadixBits = 6;

// Padded shared-memory index of table entry k (two spare doubles per 32: the
// blocked writes below hit at most 2-way bank conflicts, and pairs (k, k+1)
// with k even stay 16-byte aligned for the vector copy out).
__host__ __device__ __forceinline__ int dpad(int k) { return k + 2 * (k >> 5); }  // even for even k

// CTA-wide exclusive scans of one double per thread: prefix (ascending tid)
// and suffix (descending tid). Every partial sum is over a contiguous run of
// threads, in a fixed order. Contains a CTA barrier.
template <int NW>
__device__ __forceinline__ void block_scans(double vp, double vs, double& ep, double& es, double* wp,
                                            double* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double ip = vp, is = vs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double up = __shfl_up_sync(0xffffffffu, ip, o);
        const double dn = __shfl_down_sync(0xffffffffu, is, o);
        if (lane >= o) ip = __dadd_rn(up, ip);
        if (lane + o < 32) is = __dadd_rn(is, dn);
    }
    if (lane == 31) wp[warp] = ip;
    if (lane == 0) ws[warp] = is;
    double xp = __shfl_up_sync(0xffffffffu, ip, 1);
    double xs = __shfl_down_sync(0xffffffffu, is, 1);
    if (lane == 0) xp = 0.0;
    if (lane == 31) xs = 0.0;
    __syncthreads();
    double bp = 0.0, bs = 0.0;
    for (int w = 0; w < warp; ++w) bp = __dadd_rn(bp, wp[w]);
    for (int w = NW - 1; w > warp; --w) bs = __dadd_rn(ws[w], bs);
    ep = __dadd_rn(bp, xp);
    es = __dadd_rn(xs, bs);
}

// Sort of one staged column (THREADS x IPT floats, +inf last) into blocked
// order. Instead of a full 32-bit radix sort (6 passes) the keys are binned
// by value -- bin(x) = min(NB - 2, trunc((x - min) * (NB - 2) / (max - min))),
// +inf -> NB - 1, NB = one bin per key slot -- which is monotone in x (each
// float op is), so a counting sort by bin (shared-memory histogram, warp
// scans, atomic scatter) leaves every key within its bin of the final
// position; odd-even transposition rounds over the blocked array then finish
// the order (one or two rounds at ~1 key per bin), checked block-wide;
// columns still unsorted after 8 rounds (e.g. a few huge values squeezing the
// rest into one bin) take the full float radix sort. Equal keys may land in
// any order, which changes nothing downstream.
template <int THREADS, int IPT>
struct ColumnSorter {
    static constexpr int NPAD = THREADS * IPT;
    static constexpr int NB = NPAD;  // bins
    typedef cub::BlockRadixSort<float, THREADS, IPT, cub::NullType, kSortRadixBits> Full;
    static constexpr size_t kCount = sizeof(int) * (NB + NB / 16) + sizeof(float) * (NPAD + NPAD / 16);
    static constexpr size_t kTemp =
        sizeof(typename Full::TempStorage) > kCount ? sizeof(typename Full::TempStorage) : kCount;

    __device__ __forceinline__ static void cas(float& a, float& b) {
        const float lo = fminf(a, b), hi = fmaxf(a, b);
        a = lo;
        b = hi;
    }

    // temp: kTemp bytes; edge: 2 * THREADS floats; red: 2 * (THREADS / 32) floats
    __device__ static void sort(float (&keys)[IPT], void* temp, float* edge, float* red) {
        constexpr int NW = THREADS / 32;
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        const float kInf = __int_as_float(0x7f800000);
        float mn = kInf, mx = -kInf;
#pragma unroll
        for (int i = 0; i < IPT; ++i)
            if (keys[i] < kInf) mn = fminf(mn, keys[i]), mx = fmaxf(mx, keys[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) red[warp] = mn, red[NW + warp] = mx;
        __syncthreads();
        mn = red[0];
        mx = red[NW];
        for (int w = 1; w < NW; ++w) mn = fminf(mn, red[w]), mx = fmaxf(mx, red[NW + w]);
        if (!(mn <= mx)) return;  // no finite keys: all +inf (block-uniform)
        const float span = mx - mn;
        const float scale = (span > 0.f && span < kInf) ? static_cast<float>(NB - 2) / span : 0.f;
        // bins padded one int per 16 (bin b at b + b / 16): thread t owns bins
        // [t IPT, t IPT + IPT) for the scan, conflict-free
        int* cnt = static_cast<int*>(temp);                    // [NB + NB / 16]
        float* outv = reinterpret_cast<float*>(cnt + NB + NB / 16);  // [NPAD + NPAD/16], one pad per 16
        int* wsum = reinterpret_cast<int*>(red);               // red is free again after the barrier below
        int bk[IPT];
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const float t = (keys[i] - mn) * scale;
            const int b = keys[i] < kInf ? (t < static_cast<float>(NB - 2) ? static_cast<int>(t) : NB - 2) : NB - 1;
            bk[i] = b + (b >> 4);
        }
        for (int k = tid; k < NB + NB / 16; k += THREADS) cnt[k] = 0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) atomicAdd(cnt + bk[i], 1);
        __syncthreads();
        // exclusive scan of the counts: per-thread runs, then the thread totals
        int* cw = cnt + tid * IPT + ((tid * IPT) >> 4);
        int tot = 0;
#pragma unroll
        for (int j = 0; j < IPT; ++j) tot += cw[j + (j >> 4)];
        int inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        int run = inc - tot;
        for (int w = 0; w < warp; ++w) run += wsum[w];
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const int v = cw[j + (j >> 4)];
            cw[j + (j >> 4)] = run;
            run += v;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int pos = atomicAdd(cnt + bk[i], 1);
            outv[pos + (pos >> 4)] = keys[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int k = tid * IPT + i;
            keys[i] = outv[k + (k >> 4)];
        }
        for (int round = 0; round < 8; ++round) {
#pragma unroll
            for (int i = 0; i + 1 < IPT; i += 2) cas(keys[i], keys[i + 1]);
#pragma unroll
            for (int i = 1; i + 1 < IPT; i += 2) cas(keys[i], keys[i + 1]);
            __syncthreads();  // edge reuse
            edge[tid] = keys[0];
            edge[THREADS + tid] = keys[IPT - 1];
            __syncthreads();
            if (tid + 1 < THREADS) keys[IPT - 1] = fminf(keys[IPT - 1], edge[tid + 1]);
            if (tid > 0) keys[0] = fmaxf(keys[0], edge[THREADS + tid - 1]);
            bool ok = true;
#pragma unroll
            for (int i = 0; i + 1 < IPT; ++i) ok &= keys[i] <= keys[i + 1];
            if (!__syncthreads_or(!ok)) return;
        }
        Full(*static_cast<typename Full::TempStorage*>(temp)).Sort(keys);
    }
};

// ---- K3s-a: sort each column and write its table ---------------------------
// One CTA per group of cpb adjacent columns (slot = group * cpb + column):
// the columns are staged (outliers and padding as +inf, sorted last), each is
// sorted in registers with a block radix sort, and its table D (rows + 2
// doubles) and ColInfo go to global memory for the loop kernel.
template <int THREADS, int IPT>
__global__ void __launch_bounds__(THREADS, 3072 / THREADS / 4) k_qsort_tables(const TDesc* __restrict__ td,
                                                          const K3Group* __restrict__ groups, int cpb, int prows,
                                                          int dstride, int xstride, int tstride, int need_c,
                                                          double* __restrict__ tables,
                                                          ColInfo* __restrict__ infos) {
    constexpr int NPAD = THREADS * IPT;
    constexpr int NW = THREADS / 32;
    typedef ColumnSorter<THREADS, IPT> Sorter;
    __shared__ double wp[NW], ws[NW], wc[NW][2];
    __shared__ int wn[NW][2];
    __shared__ float edge[2 * THREADS], red[2 * NW];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* stage = reinterpret_cast<float*>(smem_raw);  // [cpb][NPAD]
    unsigned char* uni = smem_raw + sizeof(float) * static_cast<size_t>(cpb) * NPAD;
    void* sort_tmp = uni;
    double* Ds = reinterpret_cast<double*>(uni);  // aliases sort_tmp: used after each sort
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float kInf = __int_as_float(0x7f800000);

    const K3Group g = groups[blockIdx.x];
    const TDesc& d = td[g.tensor];
    const float olo = d.st->olo, ohi = d.st->ohi;
    const int64_t C = d.cols;
    const int64_t R = min(static_cast<int64_t>(prows), d.rows - g.row0);  // this piece's rows
    const float* W0 = d.W + static_cast<int64_t>(g.row0) * C + g.col0;
    const int lcpb = __ffs(cpb) - 1;  // cpb is a power of two
    const int cc0 = tid & (cpb - 1);   // a thread's column never changes (THREADS % cpb == 0)
    const int rstep = THREADS >> lcpb;  // rows between a thread's consecutive loads
    for (int base = 0; base < cpb * NPAD; base += 8 * THREADS) {  // 8 loads in flight
        float v[8];
        const int r0 = (base + tid) >> lcpb;
        const float* src = W0 + static_cast<int64_t>(r0) * C + cc0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int r = r0 + u * rstep;
            v[u] = (cc0 < g.ncols && r < R) ? __ldg(src) : kInf;
            src += static_cast<int64_t>(rstep) * C;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * THREADS + tid;
            stage[(idx & (cpb - 1)) * NPAD + (idx >> lcpb)] = is_outlier_f(v[u], olo, ohi) ? kInf : v[u];
        }
    }
    __syncthreads();
    for (int c = 0; c < g.ncols; ++c) {
        const int64_t slot = static_cast<int64_t>(blockIdx.x) * cpb + c;
        float keys[IPT];
#pragma unroll
        for (int i = 0; i < IPT; ++i) keys[i] = stage[c * NPAD + i * THREADS + tid];
        Sorter::sort(keys, sort_tmp, edge, red);  // blocked: thread t holds ranks [t*IPT, t*IPT + IPT)
        // counts, sums of x per sign, and C = sum x^2: x^2 is exact in fp64
        // and, walking the negatives up and the non-negatives down, each
        // term is no larger than the running sum, so Fast2Sum keeps C exact
        // to double-double
        int cneg = 0, cfin = 0;
        double tneg = 0.0, tpos = 0.0;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {  // two independent chains: negatives up, the rest down
            const float xn = keys[i], xp = keys[IPT - 1 - i];
            cneg += xn < 0.f;
            cfin += xn < kInf;
            if (xn < 0.f) tneg = __dadd_rn(tneg, static_cast<double>(xn));
            if (xp >= 0.f && xp < kInf) tpos = __dadd_rn(tpos, static_cast<double>(xp));
        }
        DD sq = {0.0, 0.0};
        if (!need_c) {
            // the Adam loop compares err - C and needs C only for the
            // near-tie bound (an estimate: the bound carries the slack)
#pragma unroll
            for (int i = 0; i < IPT; ++i)
                if (keys[i] < kInf) sq.hi = fma(static_cast<double>(keys[i]), static_cast<double>(keys[i]), sq.hi);
#pragma unroll
            for (int o = 16; o; o >>= 1) sq.hi = __dadd_rn(sq.hi, __shfl_xor_sync(0xffffffffu, sq.hi, o));
        } else {  // C = sum x^2 exactly as a double-double (grid oracle)
            DD sp = {0.0, 0.0};
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const float xn = keys[i], xp = keys[IPT - 1 - i];
                if (xn < 0.f) {
                    const double xd = static_cast<double>(xn);
                    const double y = __dmul_rn(xd, xd), t = __dadd_rn(sq.hi, y);
                    sq.lo = __dadd_rn(sq.lo, __dsub_rn(y, __dsub_rn(t, sq.hi)));
                    sq.hi = t;
                }
                if (xp >= 0.f && xp < kInf) {
                    const double xd = static_cast<double>(xp);
                    const double y = __dmul_rn(xd, xd), t = __dadd_rn(sp.hi, y);
                    sp.lo = __dadd_rn(sp.lo, __dsub_rn(y, __dsub_rn(t, sp.hi)));
                    sp.hi = t;
                }
            }
            sq = dd_add(two_sum(sq.hi, sq.lo), two_sum(sp.hi, sp.lo));
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const DD u = {__shfl_xor_sync(0xffffffffu, sq.hi, o), __shfl_xor_sync(0xffffffffu, sq.lo, o)};
                sq = dd_add(sq, u);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            cneg += __shfl_xor_sync(0xffffffffu, cneg, o);
            cfin += __shfl_xor_sync(0xffffffffu, cfin, o);
        }
        if (lane == 0) {
            wn[warp][0] = cneg;
            wn[warp][1] = cfin;
            wc[warp][0] = sq.hi;
            wc[warp][1] = sq.lo;
        }
        double ep, es;
        block_scans<NW>(tneg, tpos, ep, es, wp, ws);  // its barrier also retires sort_tmp
        int kz = 0, n = 0;
        for (int w = 0; w < NW; ++w) kz += wn[w][0], n += wn[w][1];
        double P = ep;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int k = tid * IPT + i;
            if (keys[i] < 0.f) {
                Ds[dpad(k)] = P;
                P = __dadd_rn(P, static_cast<double>(keys[i]));
                if (k + 1 == kz) Ds[dpad(kz)] = P;
            }
        }
        double S = es;
#pragma unroll
        for (int i = IPT - 1; i >= 0; --i) {
            const int k = tid * IPT + i;
            if (keys[i] >= 0.f && keys[i] < kInf) {
                S = __dadd_rn(S, static_cast<double>(keys[i]));
                Ds[dpad(k + 1)] = S;
            }
        }
        if (tid == 0) {
            Ds[dpad(n + 1)] = 0.0;
            if (kz == 0) Ds[0] = 0.0;
            DD cs = {wc[0][0], wc[0][1]};
            for (int w = 1; w < NW; ++w) cs = dd_add(cs, DD{wc[w][0], wc[w][1]});
            infos[slot].n = n;
            infos[slot].kz = kz;
            infos[slot].chi = cs.hi;
            infos[slot].clo = cs.lo;
        }
        if (n > 0) {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const int k = tid * IPT + i;
                if (k == 0) infos[slot].lo = keys[i];
                if (k == n - 1) infos[slot].hi = keys[i];
            }
        }
        __syncthreads();
        double* out = tables + slot * tstride;
        for (int k = 2 * tid; k < n + 2; k += 2 * THREADS)  // 16-byte copies (entry n + 2 is scratch)
            *reinterpret_cast<double2*>(out + k) = *reinterpret_cast<const double2*>(Ds + dpad(k));
        float* xo = reinterpret_cast<float*>(out + dstride);
#pragma unroll
        for (int i = 0; i < IPT; i += 4)  // sorted keys, +inf past n (blocked: 16-byte stores)
            *reinterpret_cast<float4*>(xo + tid * IPT + i) = make_float4(keys[i], keys[i + 1], keys[i + 2], keys[i + 3]);
        for (int k = NPAD + tid; k < xstride; k += THREADS) xo[k] = kInf;
        __syncthreads();  // Ds / sort_tmp / wp / ws / wn / wc reuse
    }
}

// ---- K3s-b: the Adam loop on the tables -------------------------------------
// G lanes per column (32 / G columns per warp), each lane owning TPL level
// thresholds: index u * G + gl -> level lmin + 1 + index. The per-step scalar
// work (err/grad, Adam) is shared by the column's lanes, so packing more
// columns per warp divides it; the TPL searches of a lane are independent
// (ILP). The tables are read through L1 (a step touches a few lines per
// threshold), so occupancy is bounded by registers only.
template <int G, int TPL, bool FIXED>
__global__ void __launch_bounds__(256, 4) k_qrange_tables(const TDesc* __restrict__ td,
                                                       const K3Group* __restrict__ groups, int nslots, int cpb,
                                                       int dstride, int tstride, const double* __restrict__ tables,
                                                       const ColInfo* __restrict__ infos, Scratch sc,
                                                       CfgDev cfg) {
    constexpr int CPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G, grp = lane / G;
    const int nb = cfg.lmax - cfg.lmin;  // thresholds (<= G * TPL)
    const int64_t wslot = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * CPW;
    if (wslot >= nslots) return;  // warp-uniform
    const int slot = static_cast<int>(wslot) + grp;
    const K3Group g = groups[min(slot, nslots - 1) / cpb];
    const int cc = slot % cpb;
    const bool live = slot < nslots && cc < g.ncols;
    ColInfo ci = {0, 0, 0.f, 0.f, 0.0, 0.0};
    if (live) ci = infos[slot];
    ColTab ct;
    ct.D = tables + static_cast<int64_t>(live ? slot : 0) * tstride;
    ct.xs = reinterpret_cast<const float*>(ct.D + dstride);
    ct.n = ci.n;
    const int n = ci.n;
    const double mx = n ? fmax(fabs(static_cast<double>(ci.lo)), fabs(static_cast<double>(ci.hi))) : 0.0;
    const double s0_raw = initial_scale_from_max(mx, cfg.lmax);
    double s_rtn = static_cast<double>(__double2float_rn(s0_raw));
    double s_fin = s_rtn;
    const int64_t gcol = live ? td[g.tensor].col_base + g.col0 + cc : 0;
    if (live && gl == 0) sc.tie_n[gcol] = 0;
    int tie_nc_out = 0;
    if (cfg.mode == EZQ_MODE_EASYQUANT) {  // uniform across the warp
        double s = snap(s0_raw);
        const double s0 = s;
        double m = 0.0, vv = 0.0;
        // BEST: best_err / best_s is the running best (strict <); FIXED:
        // best_err / best_s hold e0 / s0, fixed_err / fixed_s the chosen step
        DD best_err = {0.0, 0.0}, fixed_err = {0.0, 0.0};
        double best_s = s, fixed_s = s;
        const float gam = tie_gamma(n);
        const bool track = !FIXED && cfg.tie_cap > 0;
        const double cfull = ci.chi;
        double tie_thr = 0.0, tie_lo = 0.0;
        int tie_nc = 0;
        static_assert(TPL == 1, "one threshold per lane");
        // lane gl owns threshold level j = lmin + 1 + gl; a lane without one
        // (gl >= nb, or a dead slot) searches a valid threshold with weight 0
        // and contributes nothing -- the step stays free of divergence
        const bool own = live && gl < nb;
        const int j = own ? cfg.lmin + 1 + gl : cfg.lmax;
        const bool pos = j >= 1;
        const int wA = own ? (pos ? 2 * j - 1 : 1 - 2 * j) : 0;
        int ib = n >> 1;
        float Xp = 0.f, span = 0.f;  // previous threshold; x[k0+15] - x[k0] near it
        auto threshold = [&](double inv) {
            bool ok;
            float X = level_threshold_fast(j, s, inv, ok);
            if (!ok) X = level_threshold(j, s, inv);  // rare
            return X;
        };
        // A s^2 - 2 Q s (+ C) and the gradient from this lane's threshold
        auto reduce = [&](DD& err, double& grad) {
            int a = wA * (pos ? n - ib : ib);
            const double dv = __ldg(ct.D + ib + (pos ? 1 : 0));
            double q = own ? (pos ? dv : -dv) : 0.0;
#pragma unroll
            for (int o = G / 2; o; o >>= 1) {  // exact in any order
                a += __shfl_xor_sync(0xffffffffu, a, o, G);
                q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o, G));
            }
            const double Ad = static_cast<double>(a);
            // both products exact as pairs; the leading parts summed exactly,
            // the tails added after
            err = err_minus_c(Ad, q, s);
            grad = 2.0 * __dsub_rn(__dmul_rn(Ad, s), q);  // A s exact
        };
        DD err;
        double grad;
        {  // step 0 (optimize.cpp:138-145): galloping search from the middle
            const float X = threshold(__drcp_rn(s));  // RN(1/s), as the reference's 1.0 / s
            ib = search_from(ct, ib, X);
            if (ib + 8 <= n && ib >= 8) span = __ldg(ct.xs + ib + 7) - __ldg(ct.xs + ib - 8);
            Xp = X;
            reduce(err, grad);
            best_err = err;
            fixed_err = err;
            if (track) tie_window(err.hi, cfull, gam, tie_lo, tie_thr);
        }
        for (int t = 1; t <= cfg.steps; ++t) {
            s = snap(adam_update_tab(m, vv, s, grad, cfg.bc1[t], cfg.bc2[t], cfg.rbc1[t], cfg.rbc2[t], cfg.adam));
            const float X = threshold(__drcp_rn(s));
            // predict the shift from the threshold's move and the spacing seen
            // around the old position; one aligned window usually holds it
            const float dk = (span > 0.f && span < 3.0e38f) ? __fdividef(15.f * (X - Xp), span) : 0.f;
            const int guess = min(max(ib + static_cast<int>(rintf(fminf(fmaxf(dk, -256.f), 256.f))), 0), n);
            bool ok;
            ib = search_window(ct, guess, X, span, ok);
            if (!ok) ib = search_near(ct, guess, X, span);  // rare
            Xp = X;
            reduce(err, grad);
            if (!FIXED) {
                const bool lt = dd_lt(err, best_err);  // strict: earliest minimum wins (optimize.cpp:158)
                // near the running best (from above or, as a new best, from below)?
                if (track && (lt ? err.hi >= tie_lo : err.hi <= tie_thr)) {  // rare
                    if (live && gl == 0)
                        tie_step(tie_nc, sc, gcol, cfg.tie_cap, lt, err.hi, err.lo, best_err.hi, best_err.lo, s, best_s,
                                 gam, infos[slot].chi);
                } else if (lt) {
                    tie_nc = 0;  // a far new best: every earlier candidate is beyond the bound
                }
                if (lt) {
                    best_err = err;
                    best_s = s;
                    if (track) tie_window(err.hi, cfull, gam, tie_lo, tie_thr);
                }
            } else if (t == cfg.fixed_at) {
                fixed_s = s;
                fixed_err = err;
            }
        }
        if (FIXED) {
            s_fin = dd_le(fixed_err, best_err) ? fixed_s : s0;  // optimize.cpp:169-178 (best_err = e0)
            if (cfg.tie_cap > 0 && live && gl == 0)
                tie_fixed(sc, gcol, fixed_err.hi, fixed_err.lo, best_err.hi, best_err.lo, fixed_s, s0, gam, infos[slot].chi);
        } else {
            s_fin = best_s;
            tie_nc_out = tie_nc;
        }
        s_rtn = s0;
    }
    if (live && gl == 0) {
        sc.s_rtn[gcol] = s_rtn;
        sc.s_fin[gcol] = s_fin;
        if (cfg.select != EZQ_SELECT_FIXED) sc.tie_n[gcol] = tie_nc_out >= 2 ? tie_nc_out : 0;  // 1: the best itself
    }
}

template <int G, int TPL>
void launch_loop_t(int64_t nslots64, int cpb, int dstride, int tstride, const TDesc* td, const K3Group* groups,
                   const double* tables, const ColInfo* infos, const Scratch& sc, const CfgDev& cfg,
                   cudaStream_t st) {
    constexpr int CPW = 32 / G;
    const int nslots = static_cast<int>(nslots64);
    const int warps = (nslots + CPW - 1) / CPW;
    const int grid = (warps + 7) / 8;
    if (cfg.select == EZQ_SELECT_FIXED)
        k_qrange_tables<G, TPL, true><<<grid, 256, 0, st>>>(td, groups, nslots, cpb, dstride, tstride, tables, infos,
                                                            sc, cfg);
    else
        k_qrange_tables<G, TPL, false><<<grid, 256, 0, st>>>(td, groups, nslots, cpb, dstride, tstride, tables, infos,
                                                             sc, cfg);
}

// ---- K3s-b for row pieces / k = 5: one column per warp ------------------------
// A column of P pieces has P tables; "level >= j" counts and sums add over
// pieces, so every (threshold, piece) pair is searched independently: lane
// l takes pairs l, l + 32, ... (PPL per lane) and the warp butterfly sums A
// and Q -- exact, as every term is (same argument as above). Slots: column c
// of column group g, piece p is slot (g * P + p) * cpb + c.
template <int PPL, bool FIXED>
__global__ void __launch_bounds__(256) k_qrange_pieces(const TDesc* __restrict__ td,
                                                       const K3Group* __restrict__ groups, int ncolgroups, int P,
                                                       int cpb, int dstride, int tstride,
                                                       const double* __restrict__ tables,
                                                       const ColInfo* __restrict__ infos, Scratch sc, CfgDev cfg) {
    const int lane = threadIdx.x & 31;
    const int cidx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int g = cidx / cpb, cc = cidx % cpb;
    if (g >= ncolgroups) return;  // warp-uniform
    const K3Group G0 = groups[g * P];
    if (cc >= G0.ncols) return;  // warp-uniform
    const int nb = cfg.lmax - cfg.lmin;
    // column totals over the pieces, in piece order
    int nall = 0;
    double mx = 0.0, call = 0.0;
    for (int p = 0; p < P; ++p) {
        const ColInfo ci = infos[(g * P + p) * cpb + cc];
        nall += ci.n;
        call += ci.chi;
        if (ci.n) mx = fmax(mx, fmax(fabs(static_cast<double>(ci.lo)), fabs(static_cast<double>(ci.hi))));
    }
    const double s0_raw = initial_scale_from_max(mx, cfg.lmax);
    double s_rtn = static_cast<double>(__double2float_rn(s0_raw));
    double s_fin = s_rtn;
    const int64_t gcol = td[G0.tensor].col_base + G0.col0 + cc;
    if (lane == 0) sc.tie_n[gcol] = 0;
    int tie_nc_out = 0;
    if (cfg.mode == EZQ_MODE_EASYQUANT) {  // uniform across the warp
        double s = snap(s0_raw);
        const double s0 = s;
        double m = 0.0, vv = 0.0;
        DD best_err = {0.0, 0.0}, fixed_err = {0.0, 0.0};  // FIXED: best_err holds e0
        double best_s = s, fixed_s = s;
        const float gam = tie_gamma(nall);
        const bool track = !FIXED && cfg.tie_cap > 0;
        double tie_thr = 0.0, tie_lo = 0.0;
        int tie_nc = 0;
        bool own[PPL];
        int jl[PPL], np[PPL], ib[PPL];
        ColTab ct[PPL];
        float Xp[PPL], sp[PPL];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
            const int pair = lane + 32 * u;
            own[u] = pair < nb * P;
            const int thr = own[u] ? pair % nb : 0, piece = own[u] ? pair / nb : 0;
            const int slot = (g * P + piece) * cpb + cc;
            jl[u] = cfg.lmin + 1 + thr;
            ct[u].D = tables + static_cast<int64_t>(slot) * tstride;
            ct[u].xs = reinterpret_cast<const float*>(ct[u].D + dstride);
            ct[u].n = np[u] = own[u] ? infos[slot].n : 0;
            ib[u] = np[u] >> 1;
            Xp[u] = 0.f;
            sp[u] = 0.f;
        }
        for (int t = 0;; ++t) {
            int a = 0;
            double q = 0.0;
            const double inv = __drcp_rn(s);  // RN(1/s), as the reference's 1.0 / s
#pragma unroll
            for (int u = 0; u < PPL; ++u) {
                if (!own[u]) continue;
                const int j = jl[u], n = np[u];
                const float X = level_threshold(j, s, inv);
                if (t == 0) {
                    ib[u] = search_from(ct[u], ib[u], X);
                    if (ib[u] + 8 <= n && ib[u] >= 8) sp[u] = __ldg(ct[u].xs + ib[u] + 7) - __ldg(ct[u].xs + ib[u] - 8);
                } else {
                    const float spu = sp[u];
                    const float dk = (spu > 0.f && spu < 3.0e38f) ? __fdividef(15.f * (X - Xp[u]), spu) : 0.f;
                    const int guess = ib[u] + static_cast<int>(rintf(fminf(fmaxf(dk, -256.f), 256.f)));
                    ib[u] = search_near(ct[u], min(max(guess, 0), n), X, sp[u]);
                }
                Xp[u] = X;
                const bool pos = j >= 1;
                a += (pos ? 2 * j - 1 : 1 - 2 * j) * (pos ? n - ib[u] : ib[u]);
                q = __dadd_rn(q, pos ? __ldg(ct[u].D + ib[u] + 1) : -__ldg(ct[u].D + ib[u]));
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {  // exact in any order
                a += __shfl_xor_sync(0xffffffffu, a, o);
                q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
            }
            const double Ad = static_cast<double>(a);
            const DD err = err_minus_c(Ad, q, s);
            const double grad = 2.0 * __dsub_rn(__dmul_rn(Ad, s), q);  // A s exact
            if (t == 0) {
                best_err = err;
                fixed_err = err;
                if (track) tie_window(err.hi, call, gam, tie_lo, tie_thr);
            } else if (!FIXED) {
                const bool lt = dd_lt(err, best_err);  // strict: earliest minimum wins (optimize.cpp:158)
                if (track && (lt ? err.hi >= tie_lo : err.hi <= tie_thr)) {  // rare: near the running best
                    if (lane == 0)
                        tie_step(tie_nc, sc, gcol, cfg.tie_cap, lt, err.hi, err.lo, best_err.hi, best_err.lo, s, best_s,
                                 gam, call);
                } else if (lt) {
                    tie_nc = 0;  // a far new best
                }
                if (lt) {
                    best_err = err;
                    best_s = s;
                    if (track) tie_window(err.hi, call, gam, tie_lo, tie_thr);
                }
            } else if (t == cfg.fixed_at) {
                fixed_s = s;
                fixed_err = err;
            }
            if (t == cfg.steps) break;
            s = snap(adam_update_tab(m, vv, s, grad, cfg.bc1[t + 1], cfg.bc2[t + 1], cfg.rbc1[t + 1],
                                     cfg.rbc2[t + 1], cfg.adam));
        }
        if (FIXED) {
            s_fin = dd_le(fixed_err, best_err) ? fixed_s : s0;  // optimize.cpp:169-178 (best_err = e0)
            if (cfg.tie_cap > 0 && lane == 0)
                tie_fixed(sc, gcol, fixed_err.hi, fixed_err.lo, best_err.hi, best_err.lo, fixed_s, s0, gam, call);
        } else {
            s_fin = best_s;
            tie_nc_out = tie_nc;
        }
        s_rtn = s0;
    }
    if (lane == 0) {
        sc.s_rtn[gcol] = s_rtn;
        sc.s_fin[gcol] = s_fin;
        if (cfg.select != EZQ_SELECT_FIXED) sc.tie_n[gcol] = tie_nc_out >= 2 ? tie_nc_out : 0;  // 1: the best itself
    }
}

template <int PPL>
void launch_pieces_t(int ncolgroups, int P, int cpb, int dstride, int tstride, const TDesc* td,
                     const K3Group* groups, const double* tables, const ColInfo* infos, const Scratch& sc,
                     const CfgDev& cfg, cudaStream_t st) {
    const int64_t cols = static_cast<int64_t>(ncolgroups) * cpb;  // one warp each
    const int grid = static_cast<int>((cols + 7) / 8);
    if (cfg.select == EZQ_SELECT_FIXED)
        k_qrange_pieces<PPL, true><<<grid, 256, 0, st>>>(td, groups, ncolgroups, P, cpb, dstride, tstride, tables,
                                                         infos, sc, cfg);
    else
        k_qrange_pieces<PPL, false><<<grid, 256, 0, st>>>(td, groups, ncolgroups, P, cpb, dstride, tstride, tables,
                                                          infos, sc, cfg);
}

// ---- Grid oracle on the tables (brute_force_optimal_scale, optimize.cpp:186-229)
// One column per warp, (threshold, piece) pairs over the lanes as in
// k_qrange_pieces. The grid is the reference's: `points` scales
// lo + (hi - lo) i / (points - 1), lo = s0 / 8, hi = 1.25 s0, plus s0 itself,
// ascending and de-duplicated; err at each is the exact A s^2 - 2 Q s + C
// (the scales are doubles here, so s^2 is a double-double); the strict-<
// ascending scan keeps the smaller scale on ties. Writes the best grid scale
// and its error to s_fin / err_fin.
template <int PPL>
__global__ void __launch_bounds__(256) k_grid_tables(const TDesc* __restrict__ td,
                                                     const K3Group* __restrict__ groups, int ncolgroups, int P,
                                                     int cpb, int dstride, int tstride,
                                                     const double* __restrict__ tables,
                                                     const ColInfo* __restrict__ infos, Scratch sc, CfgDev cfg,
                                                     int points) {
    const int lane = threadIdx.x & 31;
    const int cidx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int g = cidx / cpb, cc = cidx % cpb;
    if (g >= ncolgroups) return;  // warp-uniform
    const K3Group G0 = groups[g * P];
    if (cc >= G0.ncols) return;  // warp-uniform
    const int nb = cfg.lmax - cfg.lmin;
    int nall = 0;
    double mx = 0.0;
    DD Cd = {0.0, 0.0};
    for (int p = 0; p < P; ++p) {
        const ColInfo ci = infos[(g * P + p) * cpb + cc];
        nall += ci.n;
        if (ci.n) mx = fmax(mx, fmax(fabs(static_cast<double>(ci.lo)), fabs(static_cast<double>(ci.hi))));
        Cd = dd_add(Cd, DD{ci.chi, ci.clo});
    }
    double best_s = 1.0, best_e = 0.0;  // empty column: {1.0, 0.0} (optimize.cpp:198)
    if (nall > 0) {
        const double s0 = initial_scale_from_max(mx, cfg.lmax);
        const double lo = s0 / 8.0, hi = s0 * 1.25;
        bool own[PPL];
        int jl[PPL], np[PPL], ib[PPL];
        ColTab ct[PPL];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
            const int pair = lane + 32 * u;
            own[u] = pair < nb * P;
            const int thr = own[u] ? pair % nb : 0, piece = own[u] ? pair / nb : 0;
            const int slot = (g * P + piece) * cpb + cc;
            jl[u] = cfg.lmin + 1 + thr;
            ct[u].D = tables + static_cast<int64_t>(slot) * tstride;
            ct[u].xs = reinterpret_cast<const float*>(ct[u].D + dstride);
            ct[u].n = np[u] = own[u] ? infos[slot].n : 0;
            ib[u] = np[u] >> 1;
        }
        bool s0_done = false, first = true;
        double prev = 0.0;
        for (int i = 0; i <= points; ++i) {  // warp-uniform
            double s;
            if (i < points) {
                const double gi = lo + (hi - lo) * static_cast<double>(i) / static_cast<double>(points - 1);
                if (!s0_done && s0 <= gi) {  // merge s0 into the ascending grid
                    s = s0;
                    s0_done = true;
                    --i;
                } else {
                    s = gi;
                }
            } else {
                if (s0_done) break;
                s = s0;
                s0_done = true;
            }
            if (!first && s == prev) continue;  // std::unique
            prev = s;
            int a = 0;
            double q = 0.0;
            const double inv = __drcp_rn(s);
#pragma unroll
            for (int u = 0; u < PPL; ++u) {
                if (!own[u]) continue;
                const int j = jl[u];
                ib[u] = search_from(ct[u], ib[u], level_threshold(j, s, inv));
                const bool pos = j >= 1;
                a += (pos ? 2 * j - 1 : 1 - 2 * j) * (pos ? np[u] - ib[u] : ib[u]);
                q = __dadd_rn(q, pos ? __ldg(ct[u].D + ib[u] + 1) : -__ldg(ct[u].D + ib[u]));
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
            }
            const double Ad = static_cast<double>(a);
            const DD ss = dd_prod(s, s);
            DD e = dd_prod(Ad, ss.hi);
            e.lo = fma(Ad, ss.lo, e.lo);
            e = dd_add(e, dd_prod(__dmul_rn(-2.0, q), s));
            e = dd_add(e, Cd);
            const double err = __dadd_rn(e.hi, e.lo);
            if (first || err < best_e) {
                best_e = err;
                best_s = s;
            }
            first = false;
        }
    }
    if (lane == 0) {
        const TDesc& d = td[G0.tensor];
        const int64_t gcol = d.col_base + G0.col0 + cc;
        sc.s_fin[gcol] = best_s;
        sc.err_fin[gcol] = best_e;
    }
}

template <int PPL>
void launch_grid_t(int ncolgroups, int P, int cpb, int dstride, int tstride, const TDesc* td,
                   const K3Group* groups, const double* tables, const ColInfo* infos, const Scratch& sc,
                   const CfgDev& cfg, int points, cudaStream_t st) {
    const int64_t cols = static_cast<int64_t>(ncolgroups) * cpb;
    const int grid = static_cast<int>((cols + 7) / 8);
    k_grid_tables<PPL><<<grid, 256, 0, st>>>(td, groups, ncolgroups, P, cpb, dstride, tstride, tables, infos, sc, cfg,
                                              points);
}

struct SortShape {
    int threads, ipt;
};
SortShape sort_shape(int npad) {
    switch (npad) {
        case 1024: return {128, 8};
        case 2048: return {128, 16};  // 256 x 8 measured slower (fewer keys per thread)
        case 4096: return {256, 16};
        case 6144: return {384, 16};
        default: return {512, 16};
    }
}

template <int THREADS, int IPT>
size_t sort_union_bytes() {
    const size_t d = sizeof(double) * static_cast<size_t>(dpad(THREADS * IPT + 2) + 1);
    return std::max(ColumnSorter<THREADS, IPT>::kTemp, d);
}

template <int THREADS, int IPT>
size_t sort_smem(int cpb) {
    const size_t u = sort_union_bytes<THREADS, IPT>();
    return sizeof(float) * static_cast<size_t>(THREADS * IPT) * cpb + ((u + 15) & ~size_t(15));
}

template <int THREADS, int IPT>
void launch_sort_t(int ngroups, int cpb, int prows, int dstride, int xstride, int tstride, int need_c, const TDesc* td,
                   const K3Group* groups, double* tables, ColInfo* infos, cudaStream_t st) {
    auto k = k_qsort_tables<THREADS, IPT>;
    const size_t smem = sort_smem<THREADS, IPT>(cpb);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<ngroups, THREADS, smem, st>>>(td, groups, cpb, prows, dstride, xstride, tstride, need_c, tables, infos);
}

}  // namespace

int k3s_npad(int64_t rows) {
    if (rows > 4096 && rows <= 6144) return 6144;  // 384 threads x 16 (e.g. 12288- and 11008-row pieces)
    int n = 1024;
    while (n < rows) n <<= 1;
    return n;
}

int k3s_pieces(int64_t rows) {
    const int64_t p = (rows + kK3sPieceRows - 1) / kK3sPieceRows;
    return p <= kK3sMaxPieces ? static_cast<int>(std::max<int64_t>(p, 1)) : 0;
}

int64_t k3s_piece_rows(int64_t rows) {
    const int p = std::max(k3s_pieces(rows), 1);
    return (rows + p - 1) / p;
}

static int k3s_dstride(int64_t rows) { return static_cast<int>((rows + 2 + 1) & ~int64_t(1)); }
static int k3s_xstride(int64_t rows) { return static_cast<int>(std::max<int64_t>(k3s_npad(rows), rows + 16) + 3) & ~3; }
static int k3s_tstride(int64_t rows) { return k3s_dstride(rows) + k3s_xstride(rows) / 2; }

bool k3s_supported(int bits) { return bits >= 2 && bits <= 5; }

int k3s_cpb(int64_t rows) {
    // staged columns per sort CTA: ~32 KB of floats (coalesced row reads)
    const int npad = k3s_npad(rows);
    return std::max(1, std::min(8, (32 << 10) / (4 * npad)));
}

size_t k3s_slot_bytes(int64_t rows) { return sizeof(double) * k3s_tstride(rows) + sizeof(ColInfo); }

void launch_k3_sorted(int64_t rows, int cpb, const TDesc* td, const K3Group* groups, int ngroups, Scratch sc,
                      CfgDev cfg, void* work, size_t work_bytes, cudaStream_t st, int grid_points) {
    if (ngroups == 0) return;
    const int P = k3s_pieces(rows);
    const int64_t pr = k3s_piece_rows(rows);
    const int npad = k3s_npad(pr), dstride = k3s_dstride(pr);
    const int xstride = k3s_xstride(pr), tstride = k3s_tstride(pr);
    const int nb = cfg.lmax - cfg.lmin;
    // Waves of whole column groups (P consecutive groups each) whose tables
    // fit the work buffer, in stream order. (Overlapping a wave's sort with
    // the previous loop on side streams was measured slower on B200: 83.5 vs
    // 77.0 ms for the OPT-1.3B set.)
    const size_t per_group = k3s_slot_bytes(pr) * cpb;
    int wave = static_cast<int>(std::max<size_t>(P, std::min<size_t>(ngroups, work_bytes / per_group)));
    wave -= wave % P;
    double* tables = static_cast<double*>(work);
    ColInfo* infos = reinterpret_cast<ColInfo*>(tables + static_cast<size_t>(wave) * cpb * tstride);
    const SortShape sh = sort_shape(npad);
    const int ppl = (nb * P + 31) / 32;  // (threshold, piece) pairs per lane
    for (int g0 = 0; g0 < ngroups; g0 += wave) {
        const int ng = std::min(wave, ngroups - g0);
        const int64_t nslots = static_cast<int64_t>(ng) * cpb;
        const int ps = prof_begin("qsort", st);
        const int ipr = static_cast<int>(pr);
        switch (sh.threads * 100 + sh.ipt) {
            case 12808: launch_sort_t<128, 8>(ng, cpb, ipr, dstride, xstride, tstride, grid_points > 0, td, groups + g0, tables, infos, st); break;
            case 12816: launch_sort_t<128, 16>(ng, cpb, ipr, dstride, xstride, tstride, grid_points > 0, td, groups + g0, tables, infos, st); break;
            case 25616: launch_sort_t<256, 16>(ng, cpb, ipr, dstride, xstride, tstride, grid_points > 0, td, groups + g0, tables, infos, st); break;
            case 38416: launch_sort_t<384, 16>(ng, cpb, ipr, dstride, xstride, tstride, grid_points > 0, td, groups + g0, tables, infos, st); break;
            default: launch_sort_t<512, 16>(ng, cpb, ipr, dstride, xstride, tstride, grid_points > 0, td, groups + g0, tables, infos, st); break;
        }
        prof_end(ps, st, static_cast<double>(nslots) * static_cast<double>(pr));
        // work: column-steps (a step = one err/grad evaluation + Adam update)
        const int ncg = ng / P;
        if (grid_points > 0) {  // grid oracle instead of the Adam loop
            switch (ppl) {
                case 1: launch_grid_t<1>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, grid_points, st); break;
                case 2: launch_grid_t<2>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, grid_points, st); break;
                case 3: launch_grid_t<3>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, grid_points, st); break;
                case 4: launch_grid_t<4>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, grid_points, st); break;
                default: launch_grid_t<8>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, grid_points, st); break;
            }
            count_launch(2);
            continue;
        }
        const int pl = prof_begin("qrange", st);
        if (P == 1 && nb <= 15) {
            launch_loop_t<16, 1>(nslots, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st);
        } else {
            switch (ppl) {
                case 1: launch_pieces_t<1>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st); break;
                case 2: launch_pieces_t<2>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st); break;
                case 3: launch_pieces_t<3>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st); break;
                case 4: launch_pieces_t<4>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st); break;
                default: launch_pieces_t<8>(ncg, P, cpb, dstride, tstride, td, groups + g0, tables, infos, sc, cfg, st); break;
            }
        }
        prof_end(pl, st, static_cast<double>(ncg) * cpb * (cfg.mode == EZQ_MODE_EASYQUANT ? cfg.steps + 1 : 1));
        count_launch(2);
    }
}

}  // namespace ezq
