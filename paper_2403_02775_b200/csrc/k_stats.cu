// K1 (tensor statistics) and K2 (outlier detection + flat-ordered COO).
//
// K1 restates stats.cpp:27-100 bit-exactly: every 8192-element chunk is summed
// sequentially in fp64 by one thread (the reference's chunk order), partials
// are merged in chunk order by one thread per tensor, and the deviation pass
// uses separate multiply/add roundings (no FMA, stats.cpp:43-46). HBM-bound
// for large tensors, latency-bound (8192-long DADD chains) for small ones;
// batching many tensors into one launch hides the chain latency.
//
// K2 restates outliers.cpp:18-61: predicate |double(v) - mean| >= thr with
// thr = double(sigma_n) * stddev, empty when stddev == 0, output sorted by
// flat index = (row, col). Count -> per-tensor exclusive scan -> ordered
// write with warp-ballot compaction.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "ezq_kernels.cuh"

namespace ezq {

namespace {

__device__ __forceinline__ int find_tensor(const int64_t* base, int ntens, int64_t g) {
    int lo = 0, hi = ntens - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= g)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

struct P1 {
    double sum, max_abs;
    float mn, mx;
    unsigned long long bad;
};

__device__ __forceinline__ void p1_elem(P1& a, float v, unsigned long long flat) {
    const double dv = static_cast<double>(v);
    a.sum = __dadd_rn(a.sum, dv);
    const double av = fabs(dv);
    a.max_abs = (a.max_abs < av) ? av : a.max_abs;  // std::max(max_abs, fabs(v))
    a.mn = (v < a.mn) ? v : a.mn;                    // std::min(mn, v)
    a.mx = (a.mx < v) ? v : a.mx;                    // std::max(mx, v)
    if (!isfinite(v) && a.bad == ~0ull) a.bad = flat;
}

__global__ void __launch_bounds__(128) k_stats_pass1(const TDesc* __restrict__ td,
                                                     const int64_t* __restrict__ chunk_base,
                                                     int ntens, int64_t total, Scratch sc) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= total) return;
    const int t = find_tensor(chunk_base, ntens, g);
    const TDesc& d = td[t];
    const int64_t lo = (g - d.chunk_base) * kStatsChunk;
    const int64_t cnt = min(kStatsChunk, d.n - lo);
    const float* p = d.W + lo;

    P1 a;
    a.sum = 0.0;
    a.max_abs = 0.0;
    a.mn = p[0];
    a.mx = p[0];
    a.bad = ~0ull;
    int64_t i = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4* p4 = reinterpret_cast<const float4*>(p);
        const int64_t n4 = cnt >> 2;
#pragma unroll 8
        for (int64_t k = 0; k < n4; ++k) {
            const float4 v = __ldg(p4 + k);
            const unsigned long long f = lo + 4 * k;
            p1_elem(a, v.x, f);
            p1_elem(a, v.y, f + 1);
            p1_elem(a, v.z, f + 2);
            p1_elem(a, v.w, f + 3);
        }
        i = n4 << 2;
    }
    for (; i < cnt; ++i) p1_elem(a, p[i], lo + i);

    const int64_t c = d.chunk_base + (g - d.chunk_base);
    sc.p_sum[c] = a.sum;
    sc.p_max[c] = a.max_abs;
    sc.p_mn[c] = a.mn;
    sc.p_mx[c] = a.mx;
    if (a.bad != ~0ull) atomicMin(&d.st->bad_index, a.bad);
}

// One thread per tensor: chunk-ordered merge (stats.cpp:66-90).
__global__ void k_stats_fin1(const TDesc* __restrict__ td, int ntens, Scratch sc) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntens) return;
    const TDesc& d = td[t];
    TStats* st = d.st;
    const int64_t b = d.chunk_base;
    double sum = 0.0, mx_abs = 0.0;
    float mn = sc.p_mn[b], mx = sc.p_mx[b];
    for (int64_t c = 0; c < d.n_chunks; ++c) {
        sum = __dadd_rn(sum, sc.p_sum[b + c]);
        const double m = sc.p_max[b + c];
        mx_abs = (mx_abs < m) ? m : mx_abs;
        const float a = sc.p_mn[b + c], z = sc.p_mx[b + c];
        mn = (a < mn) ? a : mn;
        mx = (mx < z) ? z : mx;
    }
    st->sum = sum;
    st->max_abs = mx_abs;
    st->mn = mn;
    st->mx = mx;
    if (mn == mx) {
        st->constant = 1;
        st->mean = static_cast<double>(mn);
        st->stddev = 0.0;
    } else {
        st->constant = 0;
        st->mean = __ddiv_rn(sum, static_cast<double>(d.n));
    }
}

__global__ void __launch_bounds__(128) k_stats_pass2(const TDesc* __restrict__ td,
                                                     const int64_t* __restrict__ chunk_base,
                                                     int ntens, int64_t total, Scratch sc) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= total) return;
    const int t = find_tensor(chunk_base, ntens, g);
    const TDesc& d = td[t];
    if (d.st->constant) return;
    const double mean = d.st->mean;
    const int64_t lo = (g - d.chunk_base) * kStatsChunk;
    const int64_t cnt = min(kStatsChunk, d.n - lo);
    const float* p = d.W + lo;
    double acc = 0.0;
    int64_t i = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4* p4 = reinterpret_cast<const float4*>(p);
        const int64_t n4 = cnt >> 2;
#pragma unroll 8
        for (int64_t k = 0; k < n4; ++k) {
            const float4 v = __ldg(p4 + k);
            double dv = __dsub_rn(static_cast<double>(v.x), mean);
            acc = __dadd_rn(acc, __dmul_rn(dv, dv));
            dv = __dsub_rn(static_cast<double>(v.y), mean);
            acc = __dadd_rn(acc, __dmul_rn(dv, dv));
            dv = __dsub_rn(static_cast<double>(v.z), mean);
            acc = __dadd_rn(acc, __dmul_rn(dv, dv));
            dv = __dsub_rn(static_cast<double>(v.w), mean);
            acc = __dadd_rn(acc, __dmul_rn(dv, dv));
        }
        i = n4 << 2;
    }
    for (; i < cnt; ++i) {
        const double dv = __dsub_rn(static_cast<double>(p[i]), mean);
        acc = __dadd_rn(acc, __dmul_rn(dv, dv));
    }
    sc.p_dev[d.chunk_base + (g - d.chunk_base)] = acc;
}

__global__ void k_stats_fin2(const TDesc* __restrict__ td, int ntens, Scratch sc, float sigma_n,
                             int mask_mode) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntens) return;
    const TDesc& d = td[t];
    TStats* st = d.st;
    if (!st->constant) {
        double ss = 0.0;
        for (int64_t c = 0; c < d.n_chunks; ++c) ss = __dadd_rn(ss, sc.p_dev[d.chunk_base + c]);
        st->ss = ss;
        st->stddev = __dsqrt_rn(__ddiv_rn(ss, static_cast<double>(d.n)));
    }
    // detect_impl (outliers.cpp:33-40): no outliers when stddev == 0.
    st->mask = (mask_mode && st->stddev != 0.0) ? 1 : 0;
    st->thr = st->mask ? __dmul_rn(static_cast<double>(sigma_n), st->stddev)
                       : __longlong_as_double(0x7ff0000000000000ll);
    st->n_out = 0;
}

// ---- K2 -------------------------------------------------------------------
constexpr int kDT = 256;                     // detect CTA size
constexpr int kDRounds = kDetectBlock / (kDT * 4);  // float4 per thread per round

__device__ __forceinline__ float4 load4(const float* W, int64_t n, int64_t f, bool aligned) {
    if (aligned && f + 3 < n) return __ldg(reinterpret_cast<const float4*>(W + f));
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (f < n) v.x = W[f];
    if (f + 1 < n) v.y = W[f + 1];
    if (f + 2 < n) v.z = W[f + 2];
    if (f + 3 < n) v.w = W[f + 3];
    return v;
}

__device__ __forceinline__ unsigned pred4(const float4& v, int64_t f, int64_t n, double mean,
                                          double thr) {
    unsigned m = 0;
    if (f < n && is_outlier(v.x, mean, thr)) m |= 1u;
    if (f + 1 < n && is_outlier(v.y, mean, thr)) m |= 2u;
    if (f + 2 < n && is_outlier(v.z, mean, thr)) m |= 4u;
    if (f + 3 < n && is_outlier(v.w, mean, thr)) m |= 8u;
    return m;
}

__global__ void __launch_bounds__(kDT) k_detect_count(const TDesc* __restrict__ td,
                                                      const int64_t* __restrict__ dblk_base,
                                                      int ntens, int64_t total, Scratch sc) {
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    const int t = find_tensor(dblk_base, ntens, g);
    const TDesc& d = td[t];
    const TStats* st = d.st;
    int cnt = 0;
    if (st->mask) {
        const double mean = st->mean, thr = st->thr;
        const int64_t b0 = (g - d.dblk_base) * (int64_t)kDetectBlock;
        const bool al = (reinterpret_cast<uintptr_t>(d.W) & 15) == 0;
#pragma unroll 4
        for (int r = 0; r < kDRounds; ++r) {
            const int64_t f = b0 + 4 * ((int64_t)r * kDT + threadIdx.x);
            if (f >= d.n) break;
            cnt += __popc(pred4(load4(d.W, d.n, f, al), f, d.n, mean, thr));
        }
    }
    typedef cub::BlockReduce<int, kDT> BR;
    __shared__ typename BR::TempStorage tmp;
    const int tot = BR(tmp).Sum(cnt);
    if (threadIdx.x == 0) sc.blk_count[g] = tot;
}

// One CTA per tensor: exclusive scan of its block counts.
__global__ void __launch_bounds__(1024) k_detect_scan(const TDesc* __restrict__ td, Scratch sc) {
    const TDesc& d = td[blockIdx.x];
    typedef cub::BlockScan<long long, 1024> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < d.n_dblk; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const long long v = (i < d.n_dblk) ? sc.blk_count[d.dblk_base + i] : 0;
        long long ex, agg;
        BS(tmp).ExclusiveSum(v, ex, agg);
        if (i < d.n_dblk) sc.blk_offset[d.dblk_base + i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) d.st->n_out = carry;
}

__global__ void __launch_bounds__(kDT) k_detect_write(const TDesc* __restrict__ td,
                                                      const int64_t* __restrict__ dblk_base,
                                                      int ntens, int64_t total, Scratch sc) {
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    const int t = find_tensor(dblk_base, ntens, g);
    const TDesc& d = td[t];
    const TStats* st = d.st;
    if (!st->mask || sc.blk_count[g] == 0) return;
    const double mean = st->mean, thr = st->thr;
    const int64_t b0 = (g - d.dblk_base) * (int64_t)kDetectBlock;
    const bool al = (reinterpret_cast<uintptr_t>(d.W) & 15) == 0;
    long long out = sc.blk_offset[g];
    typedef cub::BlockScan<int, kDT> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int round_total;
    for (int r = 0; r < kDRounds; ++r) {
        const int64_t f = b0 + 4 * ((int64_t)r * kDT + threadIdx.x);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned m = 0;
        if (f < d.n) {
            v = load4(d.W, d.n, f, al);
            m = pred4(v, f, d.n, mean, thr);
        }
        if (!__syncthreads_or(m != 0)) continue;
        int ex, agg;
        BS(tmp).ExclusiveSum(__popc(m), ex, agg);
        if (threadIdx.x == 0) round_total = agg;
        long long pos = out + ex;
        const float vals[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (m & (1u << k)) {
                const uint64_t flat = static_cast<uint64_t>(f + k);
                ezq_outlier e;
                e.row = static_cast<uint32_t>(flat / static_cast<uint64_t>(d.cols));
                e.col = static_cast<uint32_t>(flat % static_cast<uint64_t>(d.cols));
                e.value = vals[k];
                d.outliers[pos++] = e;
            }
        }
        __syncthreads();
        out += round_total;
    }
}

}  // namespace

void launch_stats_pass1(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st) {
    if (total_chunks == 0) return;
    const int T = 128;
    k_stats_pass1<<<(unsigned)((total_chunks + T - 1) / T), T, 0, st>>>(td, chunk_base, ntens,
                                                                        total_chunks, sc);
    count_launch();
}

void launch_stats_fin1(const TDesc* td, int ntens, Scratch sc, cudaStream_t st) {
    k_stats_fin1<<<(ntens + 63) / 64, 64, 0, st>>>(td, ntens, sc);
    count_launch();
}

void launch_stats_pass2(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st) {
    if (total_chunks == 0) return;
    const int T = 128;
    k_stats_pass2<<<(unsigned)((total_chunks + T - 1) / T), T, 0, st>>>(td, chunk_base, ntens,
                                                                        total_chunks, sc);
    count_launch();
}

void launch_stats_fin2(const TDesc* td, int ntens, Scratch sc, float sigma_n, int mask_mode,
                       cudaStream_t st) {
    k_stats_fin2<<<(ntens + 63) / 64, 64, 0, st>>>(td, ntens, sc, sigma_n, mask_mode);
    count_launch();
}

void launch_detect_count(const TDesc* td, const int64_t* dblk_base, int ntens,
                         int64_t total_blocks, Scratch sc, cudaStream_t st) {
    if (total_blocks == 0) return;
    k_detect_count<<<(unsigned)total_blocks, kDT, 0, st>>>(td, dblk_base, ntens, total_blocks,
                                                           sc);
    count_launch();
}

void launch_detect_scan(const TDesc* td, int ntens, Scratch sc, cudaStream_t st) {
    k_detect_scan<<<ntens, 1024, 0, st>>>(td, sc);
    count_launch();
}

void launch_detect_write(const TDesc* td, const int64_t* dblk_base, int ntens,
                         int64_t total_blocks, Scratch sc, cudaStream_t st) {
    if (total_blocks == 0) return;
    k_detect_write<<<(unsigned)total_blocks, kDT, 0, st>>>(td, dblk_base, ntens, total_blocks,
                                                           sc);
    count_launch();
}

}  // namespace ezq
