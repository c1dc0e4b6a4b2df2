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

// ---- TMA-pipelined chunk passes -------------------------------------------
// One warp owns 32 consecutive global chunks (lane c <-> chunk c, so each
// lane runs exactly the reference's sequential chain for its chunk). The warp
// streams the chunks through SMEM in 64-element tiles: each lane's 256-byte
// tile row arrives by one cp.async.bulk on the stage's mbarrier (3-stage ring:
// 2 tiles in flight per warp, ~8 warps/SM; 16 cp.async per lane per tile, the
// previous fill, cost 0.7 ms per OPT-1.3B step), and every lane reads its own
// row with conflict-free LDS.128 (68-float row pitch). Partial tiles are read
// from global memory. Requires 16-byte aligned tensors (else the simple
// kernels run).
constexpr int kTile = 64;
constexpr int kPitch = kTile + 4;
constexpr int kStages = 3;  // 2 tiles in flight per warp (4 or 6 stages measured slower: fewer warps/SM)
constexpr int kWarpsPerCta = 1;
constexpr size_t kRingBytes = sizeof(float) * kStages * 32 * kPitch;  // per warp
constexpr size_t kStatsSmem = (kRingBytes + sizeof(unsigned long long) * kStages) * kWarpsPerCta;

// Ring fill: a lane's full 256-byte tile row is one cp.async.bulk (TMA)
// completing on the stage's mbarrier (lane 0 posts the expected bytes of the
// whole warp first); partial tiles are read from global memory by the
// consumer instead. All lanes call it (the byte count is a warp reduction).
__device__ __forceinline__ void issue_tile_bulk(float* row, unsigned bar, const float* my_ptr, int my_cnt, int t) {
    const bool full = my_ptr != nullptr && (t + 1) * kTile <= my_cnt;
    const unsigned total = __reduce_add_sync(0xffffffffu, full ? 256u : 0u);
    if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(total) : "memory");
    __syncwarp();
    if (full) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the row was read by this lane before
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(row))), "l"(my_ptr + t * kTile), "r"(bar)
                     : "memory");
    }
}

__device__ __forceinline__ void wait_bar(unsigned bar, unsigned phase) {
    unsigned ok = 0;
    for (long long spin = 0; !ok; ++spin) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
        if (spin > (1ll << 26)) __trap();  // never hang the device on a lost transfer
    }
}

// Pass 1: the reference-order fp64 sum chain (stats.cpp:31-37) plus the
// order-free parts of sum_chunk: max|x| (fmax of non-negative values is
// exact in any order), min / max (FMNMX; equal to the reference's ternaries
// for the mn == mx test given merge rules in k_stats_merge) and a
// non-finite probe (an fp32 running sum turns non-finite on any inf/NaN; a
// probe overflow only triggers the exact re-scan of that tile).
// Pass 2: the deviation chain (stats.cpp:43-46), separate roundings.
template <bool PASS2>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_stats_pipe(const TDesc* __restrict__ td,
                                                                  const int64_t* __restrict__ chunk_base,
                                                                  int ntens, int64_t total,
                                                                  Scratch sc) {
    extern __shared__ __align__(16) float sbuf[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* ring = sbuf + warp * kStages * 32 * kPitch;
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sbuf) + kRingBytes * kWarpsPerCta) +
        warp * kStages;
    const int64_t g = (static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp) * 32 + lane;
    const float* ptr = nullptr;
    int cnt = 0;
    int t = 0;
    double mean = 0.0;
    unsigned long long flat0 = 0;
    if (g < total) {
        t = find_tensor(chunk_base, ntens, g);
        const TDesc& d = td[t];
        const int64_t lo = (g - d.chunk_base) * kStatsChunk;
        cnt = static_cast<int>(min(kStatsChunk, d.n - lo));
        ptr = d.W + lo;
        flat0 = lo;
        if (PASS2) {
            mean = d.st->mean;
            if (d.st->constant) ptr = nullptr;  // stats.cpp:77-83 skips pass 2
        }
    }
    if (__all_sync(0xffffffffu, ptr == nullptr)) return;
    const int ntiles = ptr ? (cnt + kTile - 1) / kTile : 0;
    const int max_tiles = __reduce_max_sync(0xffffffffu, ntiles);
    float* myrow0 = ring + lane * kPitch;

    double acc = 0.0;
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000), amax = 0.f;
    unsigned long long bad = ~0ull;

    if (lane == 0) {
        for (int k = 0; k < kStages; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bars + k))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto bar_of = [&](int k) { return static_cast<unsigned>(__cvta_generic_to_shared(bars + k)); };
#pragma unroll
    for (int p = 0; p < kStages - 1; ++p) issue_tile_bulk(myrow0 + p * 32 * kPitch, bar_of(p), ptr, cnt, p);
    for (int tile = 0; tile < max_tiles; ++tile) {
        const int nt = tile + kStages - 1;
        issue_tile_bulk(myrow0 + (nt % kStages) * 32 * kPitch, bar_of(nt % kStages), ptr, cnt, nt);
        wait_bar(bar_of(tile % kStages), static_cast<unsigned>((tile / kStages) & 1));
        const float* r1 = myrow0 + (tile % kStages) * 32 * kPitch;
        const int e0 = tile * kTile;
        if (tile < ntiles) {
            const int n = min(kTile, cnt - e0);
            if (n == kTile) {
                const float4* row = reinterpret_cast<const float4*>(r1);
                if (PASS2) {
                    double sq[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const double dv = __dsub_rn(static_cast<double>(r1[j]), mean);
                        sq[j] = __dmul_rn(dv, dv);
                    }
#pragma unroll
                    for (int grp = 0; grp < kTile / 16; ++grp) {
                        double nx[16];
                        if (grp + 1 < kTile / 16) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const double dv =
                                    __dsub_rn(static_cast<double>(r1[16 * (grp + 1) + j]), mean);
                                nx[j] = __dmul_rn(dv, dv);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc = __dadd_rn(acc, sq[j]);
#pragma unroll
                        for (int j = 0; j < 16; ++j) sq[j] = nx[j];
                    }
                } else {
                    float probe = 0.f;
                    double xd[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) xd[j] = static_cast<double>(r1[j]);
#pragma unroll
                    for (int grp = 0; grp < kTile / 16; ++grp) {
                        double nx[16];
                        if (grp + 1 < kTile / 16) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                nx[j] = static_cast<double>(r1[16 * (grp + 1) + j]);
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc = __dadd_rn(acc, xd[j]);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 v = row[4 * grp + q];
                            mn = fminf(fminf(mn, v.x), fminf(fminf(v.y, v.z), v.w));
                            mx = fmaxf(fmaxf(mx, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
                            amax = fmaxf(fmaxf(amax, fabsf(v.x)),
                                         fmaxf(fmaxf(fabsf(v.y), fabsf(v.z)), fabsf(v.w)));
                            probe = __fadd_rn(probe, __fadd_rn(__fadd_rn(v.x, v.y),
                                                               __fadd_rn(v.z, v.w)));
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) xd[j] = nx[j];
                    }
                    if (!isfinite(probe) && bad == ~0ull) {
                        for (int k = 0; k < kTile; ++k)
                            if (!isfinite(r1[k])) {
                                bad = flat0 + e0 + k;
                                break;
                            }
                    }
                }
            } else {
                for (int k = 0; k < n; ++k) {
                    const float v = __ldg(ptr + e0 + k);  // partial tiles are not staged
                    if (PASS2) {
                        const double dv = __dsub_rn(static_cast<double>(v), mean);
                        acc = __dadd_rn(acc, __dmul_rn(dv, dv));
                    } else {
                        acc = __dadd_rn(acc, static_cast<double>(v));
                        mn = fminf(mn, v);
                        mx = fmaxf(mx, v);
                        amax = fmaxf(amax, fabsf(v));
                        if (!isfinite(v) && bad == ~0ull) bad = flat0 + e0 + k;
                    }
                }
            }
        }
    }
    if (ptr == nullptr) return;
    if (PASS2) {
        sc.p_dev[g] = acc;
    } else {
        sc.p_sum[g] = acc;
        sc.p_max[g] = static_cast<double>(amax);
        sc.p_mn[g] = mn;
        sc.p_mx[g] = mx;
        if (bad != ~0ull) atomicMin(&td[t].st->bad_index, bad);
    }
}

// The sigma_n-dependent part of the stats (outliers.cpp:18-27): the mask and
// the exact float bounds of the outlier predicate from mean and stddev.
__device__ __forceinline__ void set_outlier_threshold(TStats* st, float sigma_n, int mask_mode) {
    st->mask = (mask_mode && st->stddev != 0.0) ? 1 : 0;
    st->thr = st->mask ? __dmul_rn(static_cast<double>(sigma_n), st->stddev)
                       : __longlong_as_double(0x7ff0000000000000ll);
    st->olo = st->mask ? outlier_lo_bound(st->mean, st->thr) : -__int_as_float(0x7f800000);
    st->ohi = st->mask ? outlier_hi_bound(st->mean, st->thr) : __int_as_float(0x7f800000);
    st->n_out = 0;
}

__device__ __forceinline__ void set_constant_threshold(TStats* st) {
    st->mask = 0;
    st->thr = __longlong_as_double(0x7ff0000000000000ll);
    st->olo = -__int_as_float(0x7f800000);
    st->ohi = __int_as_float(0x7f800000);
    st->n_out = 0;
}

// One CTA per tensor. Order-free merges (max|x|, min, max) run as block
// reductions; the two sums are merged in chunk order by thread 0 from
// registers-prefetched SMEM (stats.cpp:66-76 / 96-98). Constant-tensor rule
// (stats.cpp:77-83): the reference keeps the first of equal values, so for a
// constant tensor mn == W[0]; a NaN at W[0] pins its mn/mx to NaN (never
// constant), NaNs elsewhere are skipped exactly like FMNMX skips them.
template <bool PASS2>
__global__ void __launch_bounds__(256) k_stats_merge(const TDesc* __restrict__ td, Scratch sc,
                                                     float sigma_n, int mask_mode) {
    const TDesc& d = td[blockIdx.x];
    TStats* st = d.st;
    __shared__ double bs[2048];
    if (PASS2 && st->constant) {
        if (threadIdx.x == 0) set_constant_threshold(st);
        return;
    }
    double sum = 0.0;
    float amax = 0.f, mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    for (int64_t base = 0; base < d.n_chunks; base += 2048) {
        const int cnt = static_cast<int>(min(static_cast<int64_t>(2048), d.n_chunks - base));
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int64_t c = d.chunk_base + base + i;
            bs[i] = PASS2 ? sc.p_dev[c] : sc.p_sum[c];
            if (!PASS2) {
                amax = fmaxf(amax, static_cast<float>(sc.p_max[c]));
                mn = fminf(mn, sc.p_mn[c]);
                mx = fmaxf(mx, sc.p_mx[c]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int i = 0;
            for (; i + 8 <= cnt; i += 8) {
                double v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = bs[i + j];
#pragma unroll
                for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, v[j]);
            }
            for (; i < cnt; ++i) sum = __dadd_rn(sum, bs[i]);
        }
        __syncthreads();
    }
    if (!PASS2) {
        typedef cub::BlockReduce<float, 256> BR;
        __shared__ typename BR::TempStorage tmp;
        amax = BR(tmp).Reduce(amax, cub::Max());
        __syncthreads();
        mn = BR(tmp).Reduce(mn, cub::Min());
        __syncthreads();
        mx = BR(tmp).Reduce(mx, cub::Max());
    }
    if (threadIdx.x != 0) return;
    if (PASS2) {
        st->ss = sum;
        st->stddev = __dsqrt_rn(__ddiv_rn(sum, static_cast<double>(d.n)));
        set_outlier_threshold(st, sigma_n, mask_mode);
    } else {
        st->sum = sum;
        st->max_abs = static_cast<double>(amax);
        st->mn = mn;
        st->mx = mx;
        const float w0 = d.W[0];
        if (mn == mx && !isnan(w0)) {
            st->constant = 1;
            st->mean = static_cast<double>(w0);
            st->stddev = 0.0;
        } else {
            st->constant = 0;
            st->mean = __ddiv_rn(sum, static_cast<double>(d.n));
        }
    }
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

__device__ __forceinline__ unsigned pred4(const float4& v, int64_t f, int64_t n, float olo,
                                          float ohi) {
    unsigned m = 0;
    if (f < n && is_outlier_f(v.x, olo, ohi)) m |= 1u;
    if (f + 1 < n && is_outlier_f(v.y, olo, ohi)) m |= 2u;
    if (f + 2 < n && is_outlier_f(v.z, olo, ohi)) m |= 4u;
    if (f + 3 < n && is_outlier_f(v.w, olo, ohi)) m |= 8u;
    return m;
}

// One CTA per 16384-element block, one warp per contiguous 2048-element
// segment (4 float4 per lane in flight): the block's outlier count, and each
// segment's offset inside the block for k_detect_write.
__global__ void __launch_bounds__(kDT) k_detect_count(const TDesc* __restrict__ td,
                                                      const int64_t* __restrict__ dblk_base,
                                                      int ntens, int64_t total, Scratch sc) {
    constexpr int kV = kDetectSeg / 128;  // float4 per lane
    constexpr int kB = 4;                 // in flight
    constexpr int NW = kDT / 32;
    static_assert(kDetectBlock == NW * kDetectSeg, "one segment per warp");
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    const int t = find_tensor(dblk_base, ntens, g);
    const TDesc& d = td[t];
    const TStats* st = d.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int cnt = 0;
    if (st->mask) {
        const float olo = st->olo, ohi = st->ohi;
        const int64_t s0 = (g - d.dblk_base) * (int64_t)kDetectBlock + (int64_t)warp * kDetectSeg;
        const bool al = (reinterpret_cast<uintptr_t>(d.W) & 15) == 0;
        for (int i0 = 0; i0 < kV; i0 += kB) {
            float4 v[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int64_t f = s0 + 4 * ((i0 + b) * 32 + lane);
                v[b] = f < d.n ? load4(d.W, d.n, f, al) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int64_t f = s0 + 4 * ((i0 + b) * 32 + lane);
                cnt += f < d.n ? __popc(pred4(v[b], f, d.n, olo, ohi)) : 0;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    __shared__ int wcnt[NW];
    if (lane == 0) wcnt[warp] = cnt;
    __syncthreads();
    if (threadIdx.x < NW) {
        int off = 0;
        for (int w = 0; w < static_cast<int>(threadIdx.x); ++w) off += wcnt[w];
        sc.seg_off[g * NW + threadIdx.x] = off;
        if (threadIdx.x == NW - 1) sc.blk_count[g] = off + wcnt[NW - 1];
    }
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

// Same geometry as k_detect_count: each warp writes its segment's outliers
// in flat order from its offset (block offset + k_detect_count's segment
// offset) with ballot ranks, reading W once; warps without outliers skip.
__global__ void __launch_bounds__(kDT) k_detect_write(const TDesc* __restrict__ td,
                                                      const int64_t* __restrict__ dblk_base,
                                                      int ntens, int64_t total, Scratch sc) {
    constexpr int kV = kDetectSeg / 128;  // float4 per lane
    constexpr int kB = 4;                 // in flight
    constexpr int NW = kDT / 32;
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    const int t = find_tensor(dblk_base, ntens, g);
    const TDesc& d = td[t];
    const TStats* st = d.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!st->mask) return;
    const int off = sc.seg_off[g * NW + warp];
    const int end = warp + 1 < NW ? sc.seg_off[g * NW + warp + 1] : static_cast<int>(sc.blk_count[g]);
    if (end == off) return;  // warp-uniform: no outliers in this segment
    const float olo = st->olo, ohi = st->ohi;
    const int64_t s0 = (g - d.dblk_base) * (int64_t)kDetectBlock + (int64_t)warp * kDetectSeg;
    const bool al = (reinterpret_cast<uintptr_t>(d.W) & 15) == 0;
    long long pos = sc.blk_offset[g] + off;
    const unsigned below = (1u << lane) - 1u;
    const uint64_t C = static_cast<uint64_t>(d.cols);
    for (int i0 = 0; i0 < kV; i0 += kB) {
        float4 v[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int64_t f = s0 + 4 * ((i0 + b) * 32 + lane);
            v[b] = f < d.n ? load4(d.W, d.n, f, al) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int64_t f = s0 + 4 * ((i0 + b) * 32 + lane);
            const unsigned m = f < d.n ? pred4(v[b], f, d.n, olo, ohi) : 0u;
            if (!__ballot_sync(0xffffffffu, m != 0u)) continue;  // warp-uniform
            int before = 0, total_i = 0;  // outliers of lower lanes / of the whole row of 128
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned bb = __ballot_sync(0xffffffffu, (m >> k) & 1u);
                before += __popc(bb & below);
                total_i += __popc(bb);
            }
            long long p = pos + before;
            const float vals[4] = {v[b].x, v[b].y, v[b].z, v[b].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if ((m >> k) & 1u) {
                    const uint64_t flat = static_cast<uint64_t>(f + k);
                    ezq_outlier e;
                    e.row = static_cast<uint32_t>(flat / C);
                    e.col = static_cast<uint32_t>(flat % C);
                    e.value = vals[k];
                    d.outliers[p++] = e;
                }
            }
            pos += total_i;
        }
    }
}

}  // namespace

void launch_stats_pass1(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st, bool aligned) {
    if (total_chunks == 0) return;
    if (aligned) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_stats_pipe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kStatsSmem);
            cudaFuncSetAttribute(k_stats_pipe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kStatsSmem);
            attr = true;
        }
        const int64_t per = 32 * kWarpsPerCta;
        k_stats_pipe<false><<<(unsigned)((total_chunks + per - 1) / per), 32 * kWarpsPerCta,
                              kStatsSmem, st>>>(td, chunk_base, ntens, total_chunks, sc);
    } else {
        const int T = 128;
        k_stats_pass1<<<(unsigned)((total_chunks + T - 1) / T), T, 0, st>>>(td, chunk_base, ntens,
                                                                            total_chunks, sc);
    }
    count_launch();
}

void launch_stats_fin1(const TDesc* td, int ntens, Scratch sc, cudaStream_t st) {
    k_stats_merge<false><<<ntens, 256, 0, st>>>(td, sc, 0.f, 0);
    count_launch();
}

void launch_stats_pass2(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st, bool aligned) {
    if (total_chunks == 0) return;
    if (aligned) {
        const int64_t per = 32 * kWarpsPerCta;
        k_stats_pipe<true><<<(unsigned)((total_chunks + per - 1) / per), 32 * kWarpsPerCta,
                             kStatsSmem, st>>>(td, chunk_base, ntens, total_chunks, sc);
    } else {
        const int T = 128;
        k_stats_pass2<<<(unsigned)((total_chunks + T - 1) / T), T, 0, st>>>(td, chunk_base, ntens,
                                                                            total_chunks, sc);
    }
    count_launch();
}

void launch_stats_fin2(const TDesc* td, int ntens, Scratch sc, float sigma_n, int mask_mode,
                       cudaStream_t st) {
    k_stats_merge<true><<<ntens, 256, 0, st>>>(td, sc, sigma_n, mask_mode);
    count_launch();
}

// Batched sigma sweep: the stats of an earlier call are reused and only the
// sigma_n-dependent threshold is recomputed (same device code as k_stats_merge).
__global__ void k_stats_rethreshold(const TDesc* __restrict__ td, int ntens, float sigma_n, int mask_mode) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntens) return;
    TStats* st = td[i].st;
    if (st->constant) set_constant_threshold(st);
    else set_outlier_threshold(st, sigma_n, mask_mode);
}

void launch_stats_rethreshold(const TDesc* td, int ntens, float sigma_n, int mask_mode, cudaStream_t st) {
    k_stats_rethreshold<<<(ntens + 127) / 128, 128, 0, st>>>(td, ntens, sigma_n, mask_mode);
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
