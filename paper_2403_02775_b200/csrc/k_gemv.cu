// K6: fused dequant + outlier GEMV / skinny GEMM on the tensor cores
// (the inference-side consumer of the EasyQuant
// artifact -- the reference itself stops at dequantize_tensor,
// pipeline.cpp:116-136, and leaves the product to the caller).
//
//   y[b, j] = scale_j * sum_i l_ij x[b, i]  +  sum_{(i,j) outlier} v_ij x[b, i]
//
// l_ij is the stored level (outlier slots hold level 0).
//
// Tensor-core formulation: mma.sync.m16n8k16 (bf16 or f16 operands, fp32
// accumulate) with A = a 16-column x 16-row tile of *levels* (integers in
// [-7, 8], exact in both bf16 and f16), B = 16 rows x 8 batch rows of x, D =
// the 16 x 8 output tile. The scale is applied once per column in the
// epilogue, so the products are exact and only the fp32 accumulation rounds.
// f32 activations are split x = hi + lo (two bf16 MMAs over the same A
// fragments), keeping ~16 mantissa bits. Batch 1..8 uses one n8 tile, 9..16
// two (sharing A); larger batches launch once per group of 16.
//
// Layout (built once by ezq_gemv_prepare): K is permuted inside every
// 64-row block so that lane (g, t) needs 16 *consecutive* x values for four
// consecutive k-steps (two 16-byte loads): logical (k-step s, k in {2t, 2t+1,
// 2t+8, 2t+9}) <-> physical row 64q + 16t + 4s + {0, 1, 2, 3}. The lane's
// word for k-step s holds the nibbles of (m, k) = (g,2t) (g,2t+1) (g+8,2t)
// (g+8,2t+1) (g,2t+8) (g,2t+9) (g+8,2t+8) (g+8,2t+9) at bits 0,16,4,20,8,24,
// 12,28, so every A register is (w >> 4r) & 0x000F000F | magic (one SHF + one
// LOP3) followed by one HSUB2 that removes (magic - lmin): exact levels.
// Words are stored T[tile][q][lane] as uint4 (4 k-steps): one fully
// coalesced 512-byte load per warp per 64 rows.
//
// Work split: a CTA (8 warps) owns one 16-column tile and a range of
// 64-row blocks; warps interleave the blocks, each keeping kUnroll 16-byte
// weight loads (and their x fragments) in flight. When there are too few
// tiles to fill 148 SMs the K range is split over several CTAs; one extra
// CTA per tile gathers the tile's outliers (CSC, lane-parallel, 256 entries
// per round) concurrently with the weight stream. Partials land in a
// workspace and the last CTA to arrive (atomic ticket, threadFenceReduction
// pattern -- no spinning) sums them in fixed split order, so results are
// deterministic. Without split and without outliers the CTA writes y
// directly.
//
// HBM-bound: algorithmic bytes = N/2 (codes) + 4 cols (scales) + 8 n_out
// (outlier row + value) + 8 (cols+1) (CSC pointers) + B rows |x| + 4 B cols.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr int kWarps = 16;         // consumer warps per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kTileCols = 16;      // MMA M
constexpr int kBlockRows = 64;     // rows per lane uint4 (4 k-steps of 16)
constexpr int kMaxGroup = 16;      // batch rows per launch (two n8 tiles)

enum XType { kF32 = 0, kBF16 = 1, kF16 = 2 };

__device__ __forceinline__ float load_x(const void* x, int xt, int64_t idx) {
    if (xt == kBF16)
        return __uint_as_float(static_cast<unsigned>(static_cast<const unsigned short*>(x)[idx]) << 16);
    if (xt == kF16) return __half2float(static_cast<const __half*>(x)[idx]);
    return static_cast<const float*>(x)[idx];
}

// Raw x fragment of one lane: 16 consecutive values of one batch row.
template <int XT>
struct XRaw {
    static constexpr int kWords = XT == kF32 ? 16 : 8;
    unsigned w[kWords];
};

template <int XT>
__device__ __forceinline__ void x_load(const void* __restrict__ x, int64_t rows, int n, int64_t r0,
                                       XRaw<XT>& o) {
    const int64_t base = static_cast<int64_t>(n) * rows + r0;
    if (XT == kF32) {
        const float* p = static_cast<const float*>(x) + base;
        if (r0 + 16 <= rows && (base & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + i);
                o.w[4 * i] = u.x, o.w[4 * i + 1] = u.y, o.w[4 * i + 2] = u.z, o.w[4 * i + 3] = u.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) o.w[i] = (r0 + i < rows) ? __float_as_uint(__ldg(p + i)) : 0u;
        }
    } else {
        const unsigned short* p = static_cast<const unsigned short*>(x) + base;
        if (r0 + 16 <= rows && (base & 7) == 0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + i);
                o.w[4 * i] = u.x, o.w[4 * i + 1] = u.y, o.w[4 * i + 2] = u.z, o.w[4 * i + 3] = u.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const unsigned a = (r0 + 2 * i < rows) ? p[2 * i] : 0u;
                const unsigned b = (r0 + 2 * i + 1 < rows) ? p[2 * i + 1] : 0u;
                o.w[i] = a | (b << 16);
            }
        }
    }
}

// B-fragment registers of k-step s: {x[4s], x[4s+1]} and {x[4s+2], x[4s+3]}.
// For f32, hi/lo bf16 pairs.
template <int XT>
__device__ __forceinline__ void x_frag(const XRaw<XT>& r, int s, unsigned (&hi)[2], unsigned (&lo)[2]) {
    if (XT == kF32) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float a = __uint_as_float(r.w[4 * s + 2 * h]), b = __uint_as_float(r.w[4 * s + 2 * h + 1]);
            const __nv_bfloat162 H = __floats2bfloat162_rn(a, b);
            const float2 Hf = __bfloat1622float2(H);
            const __nv_bfloat162 L = __floats2bfloat162_rn(a - Hf.x, b - Hf.y);
            hi[h] = *reinterpret_cast<const unsigned*>(&H);
            lo[h] = *reinterpret_cast<const unsigned*>(&L);
        }
    } else {
        hi[0] = r.w[2 * s];
        hi[1] = r.w[2 * s + 1];
        lo[0] = lo[1] = 0u;
    }
}

__device__ __forceinline__ unsigned lop_pair(unsigned w, int r, unsigned magic) {
    unsigned o;
    const unsigned v = w >> (4 * r);
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(o) : "r"(v), "r"(magic));  // (v & m) | magic
    return o;
}

template <bool F16>
__device__ __forceinline__ unsigned sub2(unsigned a, unsigned b) {
    unsigned o;
    if (F16)
        asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(b));
    else
        asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(b));
    return o;
}

template <bool F16>
__device__ __forceinline__ void mma16816(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    if (F16)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// ---- TMA bulk-copy ring (mbarrier producer/consumer) ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    const uint32_t addr = smem_u32(b);
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!ok);
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
        "[%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int kGemvThreads = kThreads;  // all warps consume; the last to release a stage refills it

struct GemvArgs {
    const uint4* T;
    int kq, tiles;
    int64_t rows, cols;
    int lmin;
    const float* scales;
    const void* x;
    int batch;         // rows of this group (1..16)
    float* y;
    int sb;            // 64-row blocks per ring stage (8 or 16)
    int stages;        // ring depth
    int stage_bytes;   // codes (sb * 512) + batch x slices (xstride each)
    int xstride;       // bytes per x slice in shared memory (padded: no bank conflicts)
    int dbg;
    unsigned long long* tl;  // debug timeline (dbg == 3)
};

// x fragment of lane (g, t) for local block lb from the staged slice.
template <int XT>
__device__ __forceinline__ void x_from_smem(const unsigned char* xs, int xstride, int n, int lb, int t,
                                            XRaw<XT>& o) {
    constexpr int es = XT == kF32 ? 4 : 2;
    const uint4* p = reinterpret_cast<const uint4*>(xs + n * xstride + (64 * lb + 16 * t) * es);
#pragma unroll
    for (int i = 0; i < XRaw<XT>::kWords / 4; ++i) {
        const uint4 u = p[i];
        o.w[4 * i] = u.x, o.w[4 * i + 1] = u.y, o.w[4 * i + 2] = u.z, o.w[4 * i + 3] = u.w;
    }
}

// Rows at or past `valid` (the matrix end inside the last stage) -> 0.
template <int XT>
__device__ __forceinline__ void x_mask_tail(int valid, XRaw<XT>& o) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (i < valid) continue;
        if (XT == kF32) o.w[i] = 0u;
        else o.w[i >> 1] &= (i & 1) ? 0x0000FFFFu : 0u;
    }
}

// Persistent CTAs (one per SM) walk tiles blockIdx.x, +gridDim.x, ...; the
// producer warp streams each tile's contiguous codes (kq x 512 B) *and* the
// matching x slices (one 1-D bulk copy per batch row) through a ring of
// `stages` stages with cp.async.bulk + mbarriers -- codes with an L2
// evict-first hint (read once), x slices from L2 (shared by every tile).
// The 8 consumer warps take the stage's 64-row blocks in turn (warp w:
// blocks w, w + 8, ...), so no global load sits on their critical path;
// stages are large (up to 64 blocks = 32 KB of codes) so the per-stage
// barrier work is amortised over many MMAs. Batch columns n >= batch read
// a valid x row and are never stored (D column n depends only on B column
// n), so the fragments need no predication. Two accumulator sets break
// the HMMA dependency chain. At the end of a tile the warps' fragments are
// reduced through shared memory in fixed order and y written (y = scale *
// D; the outlier term is added by k_gemv_outliers). XG: x is read straight
// from global memory (x rows not 16-byte aligned).
template <int NB, int XT, bool XG>
__global__ void __launch_bounds__(kGemvThreads, 1) k_gemv_mma(const GemvArgs a) {
    constexpr bool F16 = XT == kF16;
    constexpr int es = XT == kF32 ? 4 : 2;
    constexpr int kGroup = (XT == kF32 || NB == 2) ? 2 : 4;  // 64-row blocks in flight per warp
    constexpr int kChains = 4;  // independent accumulator sets (HMMA dependency chains)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float (*red)[kWarps][NB][32][4] = reinterpret_cast<float (*)[kWarps][NB][32][4]>(smem_raw);
    unsigned char* ring = smem_raw + sizeof(float) * 2 * kWarps * NB * 32 * 4;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(a.stages) * a.stage_bytes);
    uint64_t* red_done = full + a.stages;
    unsigned* red_cnt = reinterpret_cast<unsigned*>(red_done + 2);
    unsigned* slot_cnt = red_cnt + 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int stage_rows = a.sb * kBlockRows;
    const int nch = (a.kq + a.sb - 1) / a.sb;
    const int my_tiles = a.tiles > static_cast<int>(blockIdx.x)
                             ? (a.tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                             : 0;
    const int total = my_tiles * nch;
    auto gtime = []() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; };
    unsigned long long* tl = (a.dbg & 8) ? a.tl + blockIdx.x * 64 : nullptr;
    // Stage j of this CTA's sequence: chunk j % nch of tile blockIdx + (j / nch) * grid.
    auto issue_stage = [&](int j, uint64_t pol) {
        const int slot = j % a.stages;
        const int c = j % nch;
        const int tile = static_cast<int>(blockIdx.x) + (j / nch) * static_cast<int>(gridDim.x);
        unsigned char* st = ring + static_cast<size_t>(slot) * a.stage_bytes;
        const int blocks = min(a.sb, a.kq - c * a.sb);
        const unsigned wbytes = static_cast<unsigned>(blocks) * 512u;
        const int64_t r0 = static_cast<int64_t>(c) * stage_rows;
        const unsigned xbytes = XG ? 0u : static_cast<unsigned>(min(static_cast<int64_t>(stage_rows), a.rows - r0) * es);
        mbar_expect_tx(&full[slot], wbytes + ((a.dbg & 2) ? 0 : xbytes * a.batch));
        bulk_g2s(st, a.T + (static_cast<int64_t>(tile) * a.kq + static_cast<int64_t>(c) * a.sb) * 32, wbytes, &full[slot],
                 pol);
        if (!XG && !(a.dbg & 2))
            for (int n = 0; n < a.batch; ++n)
                bulk_g2s_keep(st + a.sb * 512 + n * a.xstride,
                              static_cast<const unsigned char*>(a.x) + (n * a.rows + r0) * es, xbytes, &full[slot]);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.stages; ++i) {
            mbar_init(&full[i], 1);
            slot_cnt[i] = 0u;
        }
        mbar_init(&red_done[0], 1);
        mbar_init(&red_done[1], 1);
        red_cnt[0] = red_cnt[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint64_t pol = evict_first_policy();
        for (int j = 0; j < min(a.stages, total); ++j) issue_stage(j, pol);
        if (tl) {
            tl[0] = gtime();
            unsigned smid;
            asm("mov.u32 %0, %smid;" : "=r"(smid));
            tl[1] = smid;
        }
    }
    __syncthreads();
    // Let a dependent launch (the outlier pass) start its gathers now.
    asm volatile("griddepcontrol.launch_dependents;");

    const int g = lane >> 2, t = lane & 3;
    const unsigned magic = F16 ? 0x64006400u : 0x43004300u;  // 1024 | 128 + nibble
    const unsigned off2 = F16 ? static_cast<unsigned>(__half_as_ushort(__int2half_rn(1024 - a.lmin))) * 0x10001u
                              : static_cast<unsigned>(__bfloat16_as_ushort(__int2bfloat16_rn(128 - a.lmin))) * 0x10001u;
    // x row served by this lane: batch columns past the end reuse a valid row.
    int nrow[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) nrow[nb] = min(nb * 8 + g, a.batch - 1);
    int buf = 0, c = 0, tile = blockIdx.x;
    float acc[kChains][NB][4];
    float sc[2] = {0.f, 0.f};
    int ntile = 0;  // tiles this warp has finished
    for (int it = 0; it < total; ++it) {
        const int slot = it % a.stages;
        if (c == 0) {
            // the epilogue's scales, loaded a whole tile ahead of their use
            if (!(a.dbg & 32)) {
                const int64_t j0 = static_cast<int64_t>(tile) * kTileCols + g;
                sc[0] = j0 < a.cols ? __ldg(a.scales + j0) : 0.f;
                sc[1] = j0 + 8 < a.cols ? __ldg(a.scales + j0 + 8) : 0.f;
            }
#pragma unroll
            for (int h = 0; h < kChains; ++h)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[h][nb][i] = 0.f;
        }
        const unsigned char* st = ring + static_cast<size_t>(slot) * a.stage_bytes;
        const int blocks = min(a.sb, a.kq - c * a.sb);
        // rows of the stage that exist (only the matrix's last stage is short)
        const int valid_rows = static_cast<int>(min(static_cast<int64_t>(stage_rows), a.rows - static_cast<int64_t>(c) * stage_rows));
        const bool tail = valid_rows < blocks * kBlockRows;
        mbar_wait(&full[slot], (it / a.stages) & 1);
        if (tl && threadIdx.x == 0 && it < 30) tl[2 + 2 * it] = gtime();
        // Groups of kGroup blocks per warp: all shared-memory loads of the
        // group are issued before its MMAs (ILP across blocks).
        for (int lb0 = warp; lb0 < ((a.dbg & 1) ? 0 : blocks); lb0 += kWarps * kGroup) {
            XRaw<XT> xr[kGroup][NB];
            uint4 w[kGroup];
#pragma unroll
            for (int u = 0; u < kGroup; ++u) {
                const int lb = lb0 + kWarps * u;
                if (lb >= blocks) break;
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    if (XG) x_load<XT>(a.x, a.rows, nrow[nb], static_cast<int64_t>(c) * stage_rows + 64 * lb + 16 * t, xr[u][nb]);
                    else x_from_smem<XT>(st + a.sb * 512, a.xstride, nrow[nb], lb, t, xr[u][nb]);
                    if (!XG && tail) x_mask_tail<XT>(valid_rows - (64 * lb + 16 * t), xr[u][nb]);
                }
                w[u] = reinterpret_cast<const uint4*>(st)[lb * 32 + lane];
            }
#pragma unroll
            for (int u = 0; u < kGroup; ++u) {
                if (lb0 + kWarps * u >= blocks) break;
                const unsigned ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    unsigned af[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) af[r] = sub2<F16>(lop_pair(ws[s], r, magic), off2);
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) {
                        unsigned hi[2], lo[2];
                        x_frag<XT>(xr[u][nb], s, hi, lo);
                        mma16816<F16>(acc[s % kChains][nb], af, hi);
                        if (XT == kF32) mma16816<F16>(acc[s % kChains][nb], af, lo);
                    }
                }
            }
        }
        // Release the slot; the last warp to release it refills it with
        // stage it + stages (no dedicated producer warp, no blocking).
        __syncwarp();
        if (lane == 0) {
            if (!(a.dbg & 16)) __threadfence_block();
            if (atomicAdd(&slot_cnt[slot], 1u) == kWarps - 1) {
                slot_cnt[slot] = 0u;
                if (it + a.stages < total) issue_stage(it + a.stages, evict_first_policy());
            }
        }
        if (tl && threadIdx.x == 0 && it < 30) tl[3 + 2 * it] = gtime();
        if (++c != nch) continue;
        c = 0;
        if (a.dbg & 4) { tile += gridDim.x; continue; }
        // Fixed-order reduction of the warps' fragments without a CTA
        // barrier: every warp deposits its fragment, the last to arrive
        // (shared-memory ticket) sums all of them in warp order and writes
        // y. Two buffers; a buffer is reused only after its reducer has
        // released it (red_done mbarrier).
        if (ntile >= 2) mbar_wait(&red_done[buf], ((ntile >> 1) - 1) & 1);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
        {
            float v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                v[i] = acc[0][nb][i];
#pragma unroll
                for (int h = 1; h < kChains; ++h) v[i] += acc[h][nb][i];
            }
            *reinterpret_cast<float4*>(red[buf][warp][nb][lane]) = make_float4(v[0], v[1], v[2], v[3]);
        }
        __syncwarp();
        unsigned ticket = 0;
        if (lane == 0) {
            if (!(a.dbg & 16)) __threadfence_block();
            ticket = atomicAdd(&red_cnt[buf], 1u);
            if (!(a.dbg & 16)) __threadfence_block();
        }
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket == kWarps - 1) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int w2 = 0; w2 < kWarps; ++w2) {
                    const float4 v = *reinterpret_cast<const float4*>(red[buf][w2][nb][lane]);
                    d[0] += v.x, d[1] += v.y, d[2] += v.z, d[3] += v.w;
                }
                // d0, d1: (m = g, n = 2t, 2t+1); d2, d3: (m = g + 8, ...)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = g + (i >= 2 ? 8 : 0);
                    const int n = nb * 8 + 2 * t + (i & 1);
                    const int64_t j = static_cast<int64_t>(tile) * kTileCols + m;
                    if (j < a.cols && n < a.batch) a.y[static_cast<int64_t>(n) * a.cols + j] = sc[i >> 1] * d[i];
                }
            }
            __syncwarp();
            if (lane == 0) {
                red_cnt[buf] = 0u;
                mbar_arrive(&red_done[buf]);
            }
        }
        ++ntile;
        buf ^= 1;
        tile += gridDim.x;
    }
    if (tl && threadIdx.x == 0) tl[62] = gtime(), tl[63] = total;
}

// Outlier term: y[n, j] += sum_{e in column j} x[n, row_e] * v_e. Eight
// lanes per column (a warp serves 4 columns, a CTA 32), each lane walking
// every 8th CSC entry with its loads unrolled; the 8 partials are combined
// by a fixed xor-butterfly. Launched as a programmatic dependent of
// k_gemv_mma: the gathers overlap the weight stream and griddepcontrol.wait
// orders the read-modify-write of y after the main kernel's stores.
template <int XT>
__global__ void __launch_bounds__(256) k_gemv_outliers(int64_t rows, int64_t cols, const int64_t* __restrict__ col_ptr,
                                                       const uint32_t* __restrict__ out_row,
                                                       const float* __restrict__ out_val, const void* __restrict__ x,
                                                       int batch, float* __restrict__ y) {
    const int sub = threadIdx.x & 7;
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 3;
    float part[kMaxGroup];
#pragma unroll
    for (int n = 0; n < kMaxGroup; ++n) part[n] = 0.f;
    int64_t e0 = 0, e1 = 0;
    if (j < cols) e0 = col_ptr[j], e1 = col_ptr[j + 1];
#pragma unroll 4
    for (int64_t e = e0 + sub; e < e1; e += 8) {
        const int64_t r = out_row[e];
        const float v = out_val[e];
#pragma unroll
        for (int n = 0; n < kMaxGroup; ++n)
            if (n < batch) part[n] = fmaf(load_x(x, XT, static_cast<int64_t>(n) * rows + r), v, part[n]);
    }
#pragma unroll
    for (int n = 0; n < kMaxGroup; ++n) {
        if (n >= batch) break;
#pragma unroll
        for (int o = 4; o; o >>= 1) part[n] += __shfl_xor_sync(0xffffffffu, part[n], o);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (e1 > e0) {
#pragma unroll
        for (int h = 0; h < kMaxGroup / 8; ++h) {
            const int n = sub + 8 * h;
            if (n >= batch) break;
            float v = 0.f;
#pragma unroll
            for (int k = 0; k < kMaxGroup; ++k)
                if (k == n) v = part[k];
            y[static_cast<int64_t>(n) * cols + j] += v;
        }
    }
}

// Repack the artifact's codes into the MMA fragment order (layout above).
// Rows past the end (and columns past the end of the last tile) hold level 0.
__global__ void k_gemv_repack(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                              int64_t kq, int lmin, uint4* __restrict__ T) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t tiles = (cols + kTileCols - 1) / kTileCols;
    if (i >= tiles * kq * 32) return;
    const int lane = static_cast<int>(i % 32);
    const int64_t q = (i / 32) % kq, tile = i / (32 * kq);
    const int g = lane >> 2, t = lane & 3;
    // (column offset, row offset) of nibble slots at bits 0,16,4,20,8,24,12,28
    constexpr int mo[8] = {0, 0, 8, 8, 0, 0, 8, 8};
    constexpr int eo[8] = {0, 1, 0, 1, 2, 3, 2, 3};
    constexpr int sh[8] = {0, 16, 4, 20, 8, 24, 12, 28};
    unsigned words[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        unsigned w = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t j = tile * kTileCols + g + mo[k];
            const int64_t r = kBlockRows * q + 16 * t + 4 * s + eo[k];
            unsigned nib = static_cast<unsigned>(-lmin);  // level 0
            if (r < rows && j < cols) {
                const int64_t f = r * cols + j;
                nib = bits == 4 ? ((f & 1) ? (packed[f >> 1] >> 4) : (packed[f >> 1] & 15)) : packed[f];
            }
            w |= nib << sh[k];
        }
        words[s] = w;
    }
    T[i] = make_uint4(words[0], words[1], words[2], words[3]);
}

}  // namespace
}  // namespace ezq

using namespace ezq;

static unsigned long long* g_tlbuf = nullptr;  // debug timeline (EZQ_GEMV_DBG=3)

struct ezq_gemv_plan {
    int64_t rows, cols, kq, tiles;
    int bits, lmin;
    uint4* T;             // repacked codes (owned)
    const float* scales;  // device (borrowed from the artifact)
    int64_t* col_ptr;     // CSC of the outliers (owned)
    uint32_t* out_row;
    float* out_val;
    int64_t n_out;
    int grid;             // unused (grid is chosen per launch)
    int dev;
};

extern "C" {

int ezq_gemv_prepare(const ezq_qweight* q, void* stream, ezq_gemv_plan** plan) {
    *plan = nullptr;
    if (q->mem != EZQ_MEM_DEVICE)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv needs a device-resident artifact");
    if (q->rows <= 0 || q->cols <= 0)
        return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    if (q->bits < 2 || q->bits > 4)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv supports 2- to 4-bit artifacts");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    // CSC view of the outliers (one-time): D2H the COO, bucket by column
    // (rows stay ascending: the COO is flat-ordered), H2D.
    std::vector<ezq_outlier> coo(q->n_outliers);
    if (q->n_outliers)
        EZQ_CK(cudaMemcpy(coo.data(), q->outliers, sizeof(ezq_outlier) * q->n_outliers,
                          cudaMemcpyDeviceToHost));
    std::vector<int64_t> ptr(q->cols + 1, 0);
    for (const auto& e : coo) {
        if (e.col >= static_cast<uint64_t>(q->cols) || e.row >= static_cast<uint64_t>(q->rows))
            return set_error(EZQ_ERR_INVALID_ARGUMENT, "outlier coordinate outside the matrix");
        ++ptr[e.col + 1];
    }
    for (int64_t c = 0; c < q->cols; ++c) ptr[c + 1] += ptr[c];
    std::vector<uint32_t> rr(q->n_outliers);
    std::vector<float> vv(q->n_outliers);
    {
        std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
        for (const auto& e : coo) {
            rr[pos[e.col]] = e.row;
            vv[pos[e.col]++] = e.value;
        }
    }
    auto* p = new ezq_gemv_plan{};
    p->rows = q->rows;
    p->cols = q->cols;
    p->bits = q->bits;
    p->lmin = -(1 << (q->bits - 1)) + 1;
    p->kq = (q->rows + kBlockRows - 1) / kBlockRows;
    p->tiles = (q->cols + kTileCols - 1) / kTileCols;
    p->scales = q->scales;
    p->n_out = q->n_outliers;
    p->dev = dev;
    EZQ_CK(cudaMalloc(&p->T, sizeof(uint4) * p->tiles * p->kq * 32));
    EZQ_CK(cudaMalloc(&p->col_ptr, sizeof(int64_t) * (q->cols + 1)));
    EZQ_CK(cudaMalloc(&p->out_row, sizeof(uint32_t) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->out_val, sizeof(float) * std::max<int64_t>(q->n_outliers, 1)));
    {
        static bool attr_done[64] = {};
        if (!attr_done[dev & 63]) {
            attr_done[dev & 63] = true;
            const int mx = device_info(dev).max_smem_optin;
#define EZQ_ATTR(NBT, X, G) \
    EZQ_CK(cudaFuncSetAttribute(k_gemv_mma<NBT, X, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx))
            EZQ_ATTR(1, kF32, false); EZQ_ATTR(2, kF32, false); EZQ_ATTR(1, kBF16, false);
            EZQ_ATTR(2, kBF16, false); EZQ_ATTR(1, kF16, false); EZQ_ATTR(2, kF16, false);
            EZQ_ATTR(1, kF32, true); EZQ_ATTR(2, kF32, true); EZQ_ATTR(1, kBF16, true);
            EZQ_ATTR(2, kBF16, true); EZQ_ATTR(1, kF16, true); EZQ_ATTR(2, kF16, true);
#undef EZQ_ATTR
        }
    }
    p->grid = 0;
    const int64_t nw = p->tiles * p->kq * 32;
    k_gemv_repack<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, st>>>(q->packed, q->rows, q->cols,
                                                                         q->bits, p->kq, p->lmin, p->T);
    count_launch();
    EZQ_CK(cudaMemcpyAsync(p->col_ptr, ptr.data(), sizeof(int64_t) * (q->cols + 1),
                           cudaMemcpyHostToDevice, st));
    if (q->n_outliers) {
        EZQ_CK(cudaMemcpyAsync(p->out_row, rr.data(), sizeof(uint32_t) * q->n_outliers,
                               cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(p->out_val, vv.data(), sizeof(float) * q->n_outliers,
                               cudaMemcpyHostToDevice, st));
    }
    EZQ_CK(cudaStreamSynchronize(st));
    *plan = p;
    return clear_error();
}

int ezq_gemv(const ezq_gemv_plan* p, const void* x, int x_dtype, int batch, float* y,
             void* stream) {
    if (!p) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null gemv plan");
    if (batch < 1) return set_error(EZQ_ERR_INVALID_ARGUMENT, "batch must be >= 1");
    if (x_dtype < 0 || x_dtype > 2) return set_error(EZQ_ERR_INVALID_ARGUMENT, "bad x dtype");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    const int pt = prof_begin("gemv", st);
    GemvArgs a{};
    a.T = p->T;
    a.kq = static_cast<int>(p->kq);
    a.tiles = static_cast<int>(p->tiles);
    a.rows = p->rows;
    a.cols = p->cols;
    a.lmin = p->lmin;
    a.scales = p->scales;
    const size_t xes = x_dtype == kF32 ? 4 : 2;
    // One launch per group of 16 batch rows (two n8 MMA tiles share the A
    // fragments); a group of <= 8 uses one n8 tile. The outlier pass is a
    // programmatic dependent launch (its gathers overlap the weight stream).
    const DeviceInfo& di = device_info(dev);
    a.dbg = std::getenv("EZQ_GEMV_DBG") ? std::atoi(std::getenv("EZQ_GEMV_DBG")) : 0;
    if ((a.dbg & 8) && !g_tlbuf) cudaMalloc(&g_tlbuf, 8 * 64 * 1024);
    a.tl = g_tlbuf;
    for (int b0 = 0; b0 < batch; b0 += kMaxGroup) {
        a.batch = std::min(batch - b0, kMaxGroup);
        a.x = static_cast<const char*>(x) + xes * static_cast<size_t>(b0) * p->rows;
        a.y = y + static_cast<int64_t>(b0) * p->cols;
        const bool two = a.batch > 8;
        // Ring geometry: one CTA per SM (16 consumer warps); the largest
        // stage (64, 32, 16 or 8 blocks of 64 rows) whose codes + x slices
        // fit 48 KB, as many stages (<= 8) as fit in shared memory.
        const bool xg = (p->rows * xes) % 16 != 0 || (reinterpret_cast<uintptr_t>(a.x) & 15) != 0;
        const int red = static_cast<int>(sizeof(float)) * 2 * kWarps * (two ? 2 : 1) * 32 * 4;
        static const int stage_cap = std::getenv("EZQ_GEMV_STAGE_KB") ? std::atoi(std::getenv("EZQ_GEMV_STAGE_KB")) * 1024 : 48 * 1024;
        a.sb = 64;
        for (;;) {
            a.xstride = a.sb * kBlockRows * static_cast<int>(xes) + 16;
            a.stage_bytes = a.sb * 512 + (xg ? 0 : a.batch * a.xstride);
            if (a.stage_bytes <= stage_cap || a.sb == 8) break;
            a.sb /= 2;
        }
        a.stages = std::max(2, std::min(8, (di.max_smem_optin - red - 8 * 8 - 64) / a.stage_bytes));
        const size_t smem = static_cast<size_t>(red) + static_cast<size_t>(a.stages) * a.stage_bytes + 8 * a.stages + 64;
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(p->tiles, di.sms));
        switch ((x_dtype * 2 + (two ? 1 : 0)) * 2 + (xg ? 1 : 0)) {
#define EZQ_L(K, NBT, X, G) \
    case K: k_gemv_mma<NBT, X, G><<<grid, kGemvThreads, smem, st>>>(a); break;
            EZQ_L(0, 1, kF32, false) EZQ_L(1, 1, kF32, true) EZQ_L(2, 2, kF32, false) EZQ_L(3, 2, kF32, true)
            EZQ_L(4, 1, kBF16, false) EZQ_L(5, 1, kBF16, true) EZQ_L(6, 2, kBF16, false) EZQ_L(7, 2, kBF16, true)
            EZQ_L(8, 1, kF16, false) EZQ_L(9, 1, kF16, true) EZQ_L(10, 2, kF16, false)
            default: k_gemv_mma<2, kF16, true><<<grid, kGemvThreads, smem, st>>>(a); break;
#undef EZQ_L
        }
        count_launch();
        if (p->n_out) {
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(static_cast<unsigned>((p->cols + 31) / 32));
            lc.blockDim = dim3(256);
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            const int64_t* cp = p->col_ptr;
            const uint32_t* orow = p->out_row;
            const float* oval = p->out_val;
            const void* xg = a.x;
            float* yg = a.y;
            const int bt = a.batch;
            cudaError_t e;
            if (x_dtype == kF32)
                e = cudaLaunchKernelEx(&lc, k_gemv_outliers<kF32>, p->rows, p->cols, cp, orow, oval, xg, bt, yg);
            else if (x_dtype == kBF16)
                e = cudaLaunchKernelEx(&lc, k_gemv_outliers<kBF16>, p->rows, p->cols, cp, orow, oval, xg, bt, yg);
            else
                e = cudaLaunchKernelEx(&lc, k_gemv_outliers<kF16>, p->rows, p->cols, cp, orow, oval, xg, bt, yg);
            EZQ_CK(e);
            count_launch();
        }
    }
    // Algorithmic bytes: the 4-bit codes (the repacked copy has the same
    // size as the artifact's nibbles), scales, CSC, x and y.
    const double bytes = static_cast<double>(p->rows * p->cols + 1) / 2 + 4.0 * p->cols +
                         8.0 * p->n_out + 8.0 * (p->cols + 1) +
                         batch * p->rows * static_cast<double>(xes) + 4.0 * batch * p->cols;
    prof_end(pt, st, bytes);
    EZQ_CK(cudaGetLastError());
    return clear_error();
}

// Debug: copy the last dbg==3 timeline (64 u64 per CTA) to host.
int ezq_gemv_debug_timeline(unsigned long long* out, int ctas) {
    if (!g_tlbuf) return 1;
    cudaDeviceSynchronize();
    return cudaMemcpy(out, g_tlbuf, 8 * 64 * static_cast<size_t>(ctas), cudaMemcpyDeviceToHost) != cudaSuccess;
}

void ezq_gemv_plan_free(ezq_gemv_plan* p) {
    if (!p) return;
    cudaFree(p->T);
    cudaFree(p->col_ptr);
    cudaFree(p->out_row);
    cudaFree(p->out_val);
    delete p;
}

}  // extern "C"
