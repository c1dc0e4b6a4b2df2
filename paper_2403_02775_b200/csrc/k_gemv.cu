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
// Work split: one CTA per 16-column tile (4, 8 or 16 warps, chosen so that
// about 16 warps per SM are resident in a single wave); its warps take the
// tile's 64-row blocks in turn with plain coalesced 16-byte loads,
// software-pipelined one block ahead. The warps' fragments are reduced
// through shared memory in fixed order (deterministic). The outlier term is
// a second, programmatic-dependent launch (k_gemv_outliers) whose gathers
// overlap the weight stream.
//
// Measured on B200 (tools/microbench/dequant_mma.cu): the dequant + MMA loop
// costs ~25 SM-cycles per 64-row block at 16 warps/SM (ALU-bound: 3 SHF + 4
// LOP3 + 4 HSUB2 per 8 codes), i.e. ~6 TB/s of int4 codes per GPU -- about
// the HBM rate, so the kernel sits on both limits at once. A persistent
// variant streaming the codes through a TMA bulk-copy/mbarrier ring was
// built and measured (git history) and was not faster at these sizes.
//
// HBM-bound: algorithmic bytes = N/2 (codes) + 4 cols (scales) + 8 n_out
// (outlier row + value) + 8 (cols+1) (CSC pointers) + B rows |x| + 4 B cols.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr int kMaxWarps = 16;      // warps per CTA (runtime: 4, 8 or 16)
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

// ---- K6 main kernel: persistent, TMA-fed ------------------------------------
// The codes of a tile are contiguous (T[tile][q][lane]), so the whole
// artifact is one array of 512-byte blocks in (tile, q) order. Each CTA owns
// a contiguous range of ~nblk/grid blocks and streams it through a ring of
// kRing stages x kStageBlocks blocks with cp.async.bulk (one elected producer
// lane, mbarrier full/empty pairs): ~100 KB of codes in flight per SM, which
// is what an HBM-latency-bound stream needs (Little's law: ~5 MB in flight
// GPU-wide at 6.5 TB/s), without holding them in registers. kCW consumer
// warps take the range's blocks round-robin (LDS.128 from the ring, x
// fragments from L1/L2 one block ahead), dequantize to exact levels and run
// the MMAs. At every tile boundary the warps' fragments meet in shared memory
// (fixed order); a tile cut by a range boundary is split across CTAs: each
// writes its partial to a workspace and the last to arrive (ticket) sums the
// partials in CTA order -- deterministic, bit-identical across calls.
constexpr int kCW = 4;            // consumer warps per CTA
constexpr int kStageBlocks = 16;  // 64-row blocks per ring stage (8 KB)
constexpr int kRing = 4;          // ring stages per CTA (32 KB)
constexpr int kStreamThreads = (kCW + 1) * 32;
constexpr int kStreamCtasPerSm = 3;

struct GemvArgs {
    const uint4* T;
    int64_t kq;    // 64-row blocks per tile
    int64_t nblk;  // tiles * kq
    int grid;      // CTAs (ranges)
    int64_t rows, cols;
    int lmin;
    const float* scales;
    const void* x;
    int batch;  // rows of this group (1..16)
    float* y;
    float* ws;     // split-tile partials [tiles][maxsplit][16 batch][16 cols]
    int* tickets;  // [tiles], self-resetting
    int maxsplit;
};

__host__ __device__ __forceinline__ int64_t range_begin(int64_t c, int64_t nblk, int64_t grid) {
    return c * nblk / grid;
}
// CTA whose range holds block b.
__device__ __forceinline__ int64_t range_of(int64_t b, int64_t nblk, int64_t grid) {
    int64_t c = (b * grid) / nblk;
    while (c > 0 && range_begin(c, nblk, grid) > b) --c;
    while (c + 1 < grid && range_begin(c + 1, nblk, grid) <= b) ++c;
    return c;
}

__device__ __forceinline__ void bar_wait(unsigned bar, unsigned phase) {
    unsigned ok = 0;
    for (long long spin = 0; !ok; ++spin) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
        if (spin > (1ll << 28)) __trap();  // never hang the device on a lost transfer
    }
}

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int NB, int XT>
__global__ void __launch_bounds__(kStreamThreads, kStreamCtasPerSm) k_gemv_stream(const GemvArgs a) {
    constexpr bool F16 = XT == kF16;
    constexpr int kChains = NB == 1 ? 4 : 2;
    extern __shared__ __align__(128) unsigned char smem[];
    uint4* ring = reinterpret_cast<uint4*>(smem);  // [kRing][kStageBlocks][32]
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + kRing * kStageBlocks * 512);
    float* red = reinterpret_cast<float*>(bars + 2 * kRing);  // [2][kCW][NB][32][4]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cta = blockIdx.x;
    const int64_t b0 = range_begin(cta, a.nblk, a.grid), b1 = range_begin(cta + 1, a.nblk, a.grid);
    const int64_t nb = b1 - b0;
    const int nst = static_cast<int>((nb + kStageBlocks - 1) / kStageBlocks);
    const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(bars));
    const unsigned empty0 = full0 + 8 * kRing;
    if (threadIdx.x == 0) {
        for (int k = 0; k < kRing; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * k));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * k), "r"(kCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");

    if (warp == kCW) {  // ---- producer: one elected lane streams the range
        if (lane == 0) {
            const uint4* src = a.T + b0 * 32;
            for (int k = 0; k < nst; ++k) {
                const int slot = k % kRing;
                if (k >= kRing) bar_wait(empty0 + 8 * slot, ((k / kRing) - 1) & 1);
                const unsigned bytes =
                    static_cast<unsigned>(min(static_cast<int64_t>(kStageBlocks), nb - k * kStageBlocks)) * 512u;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * slot),
                             "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        static_cast<unsigned>(__cvta_generic_to_shared(ring + slot * kStageBlocks * 32))),
                    "l"(src + static_cast<int64_t>(k) * kStageBlocks * 32), "r"(bytes), "r"(full0 + 8 * slot)
                    : "memory");
            }
        }
        return;
    }

    // ---- consumers
    const int g = lane >> 2, t = lane & 3;
    const unsigned magic = F16 ? 0x64006400u : 0x43004300u;
    const unsigned off2 = F16 ? static_cast<unsigned>(__half_as_ushort(__int2half_rn(1024 - a.lmin))) * 0x10001u
                              : static_cast<unsigned>(__bfloat16_as_ushort(__int2bfloat16_rn(128 - a.lmin))) * 0x10001u;
    int nrow[NB];
#pragma unroll
    for (int n8 = 0; n8 < NB; ++n8) nrow[n8] = min(n8 * 8 + g, a.batch - 1);
    const int64_t tile_first = b0 / a.kq, tile_last = nb > 0 ? (b1 - 1) / a.kq : tile_first - 1;
    int tcount = 0;
    for (int64_t tile = tile_first; tile <= tile_last; ++tile, ++tcount) {
        const int64_t ta = max(b0, tile * a.kq), tb = min(b1, (tile + 1) * a.kq);  // this CTA's blocks of the tile
        float acc[kChains][NB][4];
#pragma unroll
        for (int h = 0; h < kChains; ++h)
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[h][n8][i] = 0.f;
        // my blocks: i in [ta, tb) with (i - b0) % kCW == warp
        int64_t i = ta + ((warp - (ta - b0)) % kCW + kCW) % kCW;
        XRaw<XT> xc[NB];
        if (i < tb) {
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
                x_load<XT>(a.x, a.rows, nrow[n8], kBlockRows * (i - tile * a.kq) + 16 * t, xc[n8]);
        }
        for (; i < tb; i += kCW) {
            const int64_t j = i - b0;  // position in the range
            const int k = static_cast<int>(j / kStageBlocks), slot = k % kRing;
            bar_wait(full0 + 8 * slot, (k / kRing) & 1);
            const uint4 w = ring[(slot * kStageBlocks + static_cast<int>(j % kStageBlocks)) * 32 + lane];
            // release the stage after my last block in it (or my last block)
            if (j % kStageBlocks >= kStageBlocks - kCW || i + kCW >= b1) {
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
            }
            XRaw<XT> xn[NB];
            if (i + kCW < tb) {
#pragma unroll
                for (int n8 = 0; n8 < NB; ++n8)
                    x_load<XT>(a.x, a.rows, nrow[n8], kBlockRows * (i + kCW - tile * a.kq) + 16 * t, xn[n8]);
            }
            const unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                unsigned af[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) af[r] = sub2<F16>(lop_pair(ws[s], r, magic), off2);
#pragma unroll
                for (int n8 = 0; n8 < NB; ++n8) {
                    unsigned hi[2], lo[2];
                    x_frag<XT>(xc[n8], s, hi, lo);
                    mma16816<F16>(acc[s % kChains][n8], af, hi);
                    if (XT == kF32) mma16816<F16>(acc[s % kChains][n8], af, lo);
                }
            }
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8) xc[n8] = xn[n8];
        }
        // ---- flush the tile: warps meet in shared memory (fixed order)
        float* rb = red + (tcount & 1) * (kCW * NB * 32 * 4);
#pragma unroll
        for (int n8 = 0; n8 < NB; ++n8) {
            float v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                v[q] = acc[0][n8][q];
#pragma unroll
                for (int h = 1; h < kChains; ++h) v[q] += acc[h][n8][q];
            }
            *reinterpret_cast<float4*>(rb + ((warp * NB + n8) * 32 + lane) * 4) = make_float4(v[0], v[1], v[2], v[3]);
        }
        named_sync(1, kCW * 32);
        if (warp != static_cast<int>(tile % kCW)) continue;
        float d[NB][4];
#pragma unroll
        for (int n8 = 0; n8 < NB; ++n8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) d[n8][q] = 0.f;
            for (int w2 = 0; w2 < kCW; ++w2) {
                const float4 v = *reinterpret_cast<const float4*>(rb + ((w2 * NB + n8) * 32 + lane) * 4);
                d[n8][0] += v.x, d[n8][1] += v.y, d[n8][2] += v.z, d[n8][3] += v.w;
            }
        }
        const bool whole = ta == tile * a.kq && tb == (tile + 1) * a.kq;
        if (!whole) {
            // split tile: partial to the workspace, the last CTA to arrive sums
            const int64_t c_first = range_of(tile * a.kq, a.nblk, a.grid);
            const int64_t c_last = range_of((tile + 1) * a.kq - 1, a.nblk, a.grid);
            const int nsplit = static_cast<int>(c_last - c_first + 1);
            float* wsl = a.ws + (tile * a.maxsplit + (cta - c_first)) * 256;
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                for (int q = 0; q < 4; ++q) wsl[(n8 * 32 + lane) * 4 + q] = d[n8][q];
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(a.tickets + tile, 1) == nsplit - 1;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            const float* wst = a.ws + tile * a.maxsplit * 256;
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float sum = 0.f;
                    for (int sp = 0; sp < nsplit; ++sp) sum += __ldcg(wst + sp * 256 + (n8 * 32 + lane) * 4 + q);
                    d[n8][q] = sum;
                }
            if (lane == 0) a.tickets[tile] = 0;  // ready for the next call
        }
#pragma unroll
        for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int m = g + (q >= 2 ? 8 : 0);
                const int n = n8 * 8 + 2 * t + (q & 1);
                const int64_t jc = tile * kTileCols + m;
                if (jc < a.cols && n < a.batch) a.y[static_cast<int64_t>(n) * a.cols + jc] = a.scales[jc] * d[n8][q];
            }
    }
}

size_t stream_smem(int nb) {
    return static_cast<size_t>(kRing) * kStageBlocks * 512 + 2 * kRing * 8 + sizeof(float) * 2 * kCW * nb * 32 * 4;
}

// Outlier term: y[n, j] += sum_{e in column j} x[n, row_e] * v_e. One warp
// per column; the lanes take the column's CSC entries 32 apart, with kU
// entries per lane loaded independently per round (one round covers 128
// entries, i.e. a 1%-outlier column of up to 12.8k rows), and the partials
// are combined by a fixed xor-butterfly (deterministic). NBT = batch rows
// rounded up to 1, 8 or 16 (fully unrolled, predicated on `batch`).
// Launched as a programmatic dependent of k_gemv_mma: the gathers overlap
// the weight stream and griddepcontrol.wait orders the read-modify-write
// of y after the main kernel's stores.
// x [batch][rows] (any dtype) -> xt [rows][16] f32 (exact), so the outlier
// pass reads a row's batch values with NBT/4 16-byte loads instead of NBT
// scalar gathers.
__global__ void __launch_bounds__(256) k_gemv_xt(const void* __restrict__ x, int xt_type, int64_t rows, int batch,
                                                 float* __restrict__ xt) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 16 + (threadIdx.x >> 4);
    const int n = threadIdx.x & 15;
    if (r < rows) xt[r * 16 + n] = n < batch ? load_x(x, xt_type, static_cast<int64_t>(n) * rows + r) : 0.f;
}

template <int XT, int NBT>
__global__ void __launch_bounds__(256) k_gemv_outliers(int64_t rows, int64_t cols, const int64_t* __restrict__ col_ptr,
                                                       const uint32_t* __restrict__ out_row,
                                                       const float* __restrict__ out_val, const void* __restrict__ x,
                                                       int batch, float* __restrict__ y,
                                                       const float* __restrict__ xt) {
    constexpr int kU = 4;
    const int lane = threadIdx.x & 31;
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    float part[NBT];
#pragma unroll
    for (int n = 0; n < NBT; ++n) part[n] = 0.f;
    int64_t e0 = 0, e1 = 0;
    if (j < cols) e0 = __ldg(col_ptr + j), e1 = __ldg(col_ptr + j + 1);
    for (int64_t eb = e0; eb < e1; eb += 32 * kU) {
        uint32_t r[kU];
        float v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t e = eb + lane + 32 * u;
            r[u] = e < e1 ? __ldg(out_row + e) : 0u;
            v[u] = e < e1 ? __ldg(out_val + e) : 0.f;
        }
        if (NBT > 8) {  // transposed x: one 16-byte load per 4 batch rows
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int n4 = 0; n4 < NBT / 4; ++n4) {
                    const float4 xv = __ldg(reinterpret_cast<const float4*>(xt + static_cast<int64_t>(r[u]) * 16) + n4);
                    const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (4 * n4 + k < batch) part[4 * n4 + k] = fmaf(xs[k], v[u], part[4 * n4 + k]);
                }
        } else {
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int n = 0; n < NBT; ++n)
                    if (n < batch) part[n] = fmaf(load_x(x, XT, static_cast<int64_t>(n) * rows + r[u]), v[u], part[n]);
        }
    }
    const bool any = e1 > e0;
    if (any) {
#pragma unroll
        for (int n = 0; n < NBT; ++n) {
            if (n >= batch) break;
#pragma unroll
            for (int o = 16; o; o >>= 1) part[n] += __shfl_xor_sync(0xffffffffu, part[n], o);
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (any && lane < batch) {
        float add = part[0];
#pragma unroll
        for (int k = 1; k < NBT; ++k)
            if (k == lane) add = part[k];
        y[static_cast<int64_t>(lane) * cols + j] += add;
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

struct ezq_gemv_plan {
    int64_t rows, cols, kq, tiles;
    int bits, lmin;
    uint4* T;             // repacked codes (owned)
    const float* scales;  // device (borrowed from the artifact)
    int64_t* col_ptr;     // CSC of the outliers (owned)
    uint32_t* out_row;
    float* out_val;
    int64_t n_out;
    int dev;
    float* xt;            // batch > 1 with outliers: x transposed [rows][16] f32 (owned)
    int grid;             // persistent CTAs of k_gemv_stream (block ranges)
    int maxsplit;         // most ranges one tile is cut into
    float* ws;            // split-tile partials (owned)
    int* tickets;         // per tile (owned, self-resetting)
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
    p->xt = nullptr;
    if (q->n_outliers > 0) EZQ_CK(cudaMalloc(&p->xt, sizeof(float) * 16 * static_cast<size_t>(q->rows)));
    EZQ_CK(cudaMalloc(&p->out_row, sizeof(uint32_t) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->out_val, sizeof(float) * std::max<int64_t>(q->n_outliers, 1)));
    // Persistent ranges: kStreamCtasPerSm CTAs per SM, each a contiguous
    // range of 64-row blocks (never more ranges than blocks).
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nblk = p->tiles * p->kq;
    p->grid = static_cast<int>(std::min<int64_t>(nblk, static_cast<int64_t>(sms) * kStreamCtasPerSm));
    p->maxsplit = 1;
    for (int64_t tl = 0; tl < p->tiles; ++tl) {  // ranges cutting each tile (host mirror of range_of)
        auto rng = [&](int64_t b) {
            int64_t c = (b * p->grid) / nblk;
            while (c > 0 && range_begin(c, nblk, p->grid) > b) --c;
            while (c + 1 < p->grid && range_begin(c + 1, nblk, p->grid) <= b) ++c;
            return c;
        };
        p->maxsplit = std::max<int>(p->maxsplit, static_cast<int>(rng((tl + 1) * p->kq - 1) - rng(tl * p->kq) + 1));
    }
    EZQ_CK(cudaMalloc(&p->ws, sizeof(float) * 256 * static_cast<size_t>(p->tiles) * p->maxsplit));
    EZQ_CK(cudaMalloc(&p->tickets, sizeof(int) * static_cast<size_t>(p->tiles)));
    EZQ_CK(cudaMemsetAsync(p->tickets, 0, sizeof(int) * static_cast<size_t>(p->tiles), st));
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
    a.kq = p->kq;
    a.nblk = p->tiles * p->kq;
    a.grid = p->grid;
    a.ws = p->ws;
    a.tickets = p->tickets;
    a.maxsplit = p->maxsplit;
    a.rows = p->rows;
    a.cols = p->cols;
    a.lmin = p->lmin;
    a.scales = p->scales;
    const size_t xes = x_dtype == kF32 ? 4 : 2;
    // One launch per group of 16 batch rows (two n8 MMA tiles share the A
    // fragments); a group of <= 8 uses one n8 tile. The outlier pass is a
    // programmatic dependent launch (its gathers overlap the weight stream).
    for (int b0 = 0; b0 < batch; b0 += kMaxGroup) {
        a.batch = std::min(batch - b0, kMaxGroup);
        a.x = static_cast<const char*>(x) + xes * static_cast<size_t>(b0) * p->rows;
        a.y = y + static_cast<int64_t>(b0) * p->cols;
        const bool two = a.batch > 8;
        if (p->n_out && a.batch > 8) {  // transposed x for the outlier pass (pays off from 9 batch rows)
            k_gemv_xt<<<static_cast<unsigned>((p->rows + 15) / 16), 256, 0, st>>>(a.x, x_dtype, p->rows, a.batch,
                                                                                  p->xt);
            count_launch();
        }
        const unsigned grid = static_cast<unsigned>(p->grid);
        const size_t smem = stream_smem(two ? 2 : 1);
        switch (x_dtype * 2 + (two ? 1 : 0)) {
            case 0: k_gemv_stream<1, kF32><<<grid, kStreamThreads, smem, st>>>(a); break;
            case 1: k_gemv_stream<2, kF32><<<grid, kStreamThreads, smem, st>>>(a); break;
            case 2: k_gemv_stream<1, kBF16><<<grid, kStreamThreads, smem, st>>>(a); break;
            case 3: k_gemv_stream<2, kBF16><<<grid, kStreamThreads, smem, st>>>(a); break;
            case 4: k_gemv_stream<1, kF16><<<grid, kStreamThreads, smem, st>>>(a); break;
            default: k_gemv_stream<2, kF16><<<grid, kStreamThreads, smem, st>>>(a); break;
        }
        count_launch();
        if (p->n_out) {
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(static_cast<unsigned>((p->cols + 7) / 8));  // one warp per column
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
            const float* xtg = p->xt;
            cudaError_t e;
#define EZQ_OUT(X)                                                                                     \
    (bt == 1 ? cudaLaunchKernelEx(&lc, k_gemv_outliers<X, 1>, p->rows, p->cols, cp, orow, oval, xg, bt, yg, xtg) \
     : bt <= 8 ? cudaLaunchKernelEx(&lc, k_gemv_outliers<X, 8>, p->rows, p->cols, cp, orow, oval, xg, bt, yg, xtg) \
               : cudaLaunchKernelEx(&lc, k_gemv_outliers<X, 16>, p->rows, p->cols, cp, orow, oval, xg, bt, yg, xtg))
            if (x_dtype == kF32) e = EZQ_OUT(kF32);
            else if (x_dtype == kBF16) e = EZQ_OUT(kBF16);
            else e = EZQ_OUT(kF16);
#undef EZQ_OUT
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

void ezq_gemv_plan_free(ezq_gemv_plan* p) {
    if (!p) return;
    cudaFree(p->T);
    cudaFree(p->col_ptr);
    if (p->xt) cudaFree(p->xt);
    cudaFree(p->out_row);
    cudaFree(p->out_val);
    cudaFree(p->ws);
    cudaFree(p->tickets);
    delete p;
}

}  // extern "C"
