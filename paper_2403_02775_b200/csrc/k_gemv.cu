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
// Work split (k_gemv_cb below): persistent CTAs stream colblocks of TPC
// tiles over all of K through a TMA ring (codes, x slices and the outlier
// segments of each stage on one mbarrier); 4 consumer warps run the MMAs,
// outlier warps apply the isolated outliers from the staged x slice, and
// the writers add both (fixed order: deterministic). k_gemv_outliers is the
// separate CSC pass kept for the variants that do not fuse.
//
// Measured on B200: the dequant + MMA loop is ALU-heavy
// (SHF + LOP3 (+ HSUB2) per A register), ~0.72 of the HBM copy rate at the
// BLOOM-176B FFN shape at batch 1.
//
// HBM-bound: algorithmic bytes = N/2 (codes) + 4 cols (scales) + 6 (f32) or
// 4 (f16) n_out (outlier value + row) + B rows |x| + 4 B cols.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
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

// ---- K6 main kernel: column-block skinny GEMM, persistent, TMA-fed ----------
// Output columns go in colblocks of TPC MMA tiles (16 x TPC columns; TPC in
// {1, 2, 4, 8} chosen per shape by ezq_gemv_prepare so the colblocks fill
// the SMs); the artifact is repacked T[cb][q][tile][lane] (uint4), so a
// colblock's whole K is one contiguous byte range. A persistent CTA takes
// colblocks cb = blockIdx.x, + gridDim.x, ... and streams each through a
// ring of kRing stages of S q-blocks (8 KB of codes, one cp.async.bulk), the
// stage's x slice (S x 64 rows x the batch rows) arriving by 16-byte cp.async
// from the producer warp's lanes on the same mbarrier: tens of KB in flight
// per CTA without holding them in registers, and every x slice is read once
// per colblock. Each colblock's K is complete inside the CTA -- no
// cross-CTA reduction. The kCW = 4 consumer warps split a stage's (q, tile)
// blocks: with TPC >= 4 warp w owns tiles w, w + 4, ... over all of K (no
// reduction at all); with TPC < 4 the 4 / TPC warps of a tile split its q
// blocks and meet in shared memory at the end of the colblock (fixed order:
// deterministic, bit-identical across calls).
constexpr int kCW = 4;             // consumer warps per CTA
constexpr int kRing = 2;           // ring stages per CTA
constexpr int kStageCode = 32768;  // code bytes per full stage (sweep on B200: 8-32 KB x 2-6 stages)
constexpr int kStreamThreads = (kCW + 1) * 32;
constexpr int kOutWarpsSmall = 2, kOutWarpsMax = 4;              // outlier warps (fused outliers)
constexpr int kOutThreads = kStreamThreads + 32 * kOutWarpsMax;

struct GemvArgs {
    const uint4* T;
    int64_t kq;    // 64-row blocks (K)
    int64_t ncb;   // colblocks
    int64_t rows, cols;
    int lmin;
    const float* scales;
    const void* x;     // [batch][xstride], 64-row multiples, 16-byte aligned rows (else a padded copy)
    int64_t xstride;   // elements between batch rows of x
    int batch;         // rows of this group (1..16)
    float* y;
    // Fused outlier term (ezq_gemv_prepare; null: the separate pass): per
    // colblock, the outliers of every 512-row segment as {header, entries},
    // streamed into the ring beside the stage's codes.
    const unsigned char* oseg;
    const int64_t* obnd;  // [ncb * nseg + 1] byte offsets of the segments in oseg
    int64_t nseg;         // segments per colblock
    int ob;               // shared-memory bytes per ring stage for the segments
    int oes;              // value bytes: 4 = f32, 2 = f16
    // Split K (ks > 1): a thread-block cluster of ks CTAs shares each
    // colblock, rank r streaming stages [nst r / ks, nst (r + 1) / ks); the
    // ranks' partial outputs meet in rank 0's shared memory (DSMEM, fixed
    // rank order: deterministic) -- more bytes in flight per colblock for
    // shapes with fewer colblocks than resident CTAs.
    int ks;
};

// Fused outliers: segment = 512 rows (8 q-blocks; every stage of the variants
// that fuse holds 1 or 2 whole segments) x one colblock. Layout (16-byte
// aligned, sizes multiples of 16): u32 total bytes; u16 start[TPC * 16 + 1]
// (entry index of each column's first outlier; rows ascending inside a
// column); pad; the E = start[TPC * 16] values (f32 or f16); their rows
// inside the segment (u16); pad. 6 (f32) or 4 (f16) bytes per outlier.
constexpr int kSegRows = 512;
constexpr int kSegQ = kSegRows / kBlockRows;
__host__ __device__ constexpr int seg_hdr_bytes(int tpc) { return (4 + 2 * (tpc * kTileCols + 1) + 15) & ~15; }

__device__ __forceinline__ void bar_wait(unsigned bar, unsigned phase) {
    unsigned ok = 0;
    for (int spin = 0; !ok; ++spin) {
        // try_wait suspends the warp until the phase completes (or a time
        // limit): waiting warps take no issue slots from the dequant
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
        if (spin > (1 << 28)) __trap();  // never hang the device on a lost transfer
    }
}

// Same, acquiring at cluster scope (split-K partials written by other CTAs).
__device__ __forceinline__ void bar_wait_cluster(unsigned bar, unsigned phase) {
    unsigned ok = 0;
    for (int spin = 0; !ok; ++spin) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
        if (spin > (1 << 28)) __trap();
    }
}

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int TPC, int NB, int XT, bool SF = false>
struct CbGeom {
    static constexpr int ES = XT == kF32 ? 4 : 2;                     // x element bytes
    static constexpr int NBT = NB * 8;                                // batch rows staged
    static constexpr int XQ = 64 * NBT * ES;                          // x bytes per q-block
    static constexpr int S0 = kStageCode / (512 * TPC);               // q-blocks per stage (codes)
    static constexpr int S = S0 < 16384 / XQ ? S0 : 16384 / XQ;       // ... capped by <= 16 KB of x
    static constexpr int XP = S * 64 + (XT == kF32 ? 4 : 8);          // x row pitch (elements, padded)
    static constexpr int XB = NBT * XP * ES;                          // x bytes per stage
    static constexpr int CB = S * TPC * 512;                          // code bytes per stage
    static constexpr int TW = TPC >= kCW ? TPC / kCW : 1;             // tiles per warp
    static constexpr int QW = TPC >= kCW ? 1 : kCW / TPC;             // warps sharing a tile
    // HSUB2-free dequant (bf16 / split-f32 x, batch <= 8): A' = level + C
    // exactly (C = 128 - lmin), D' = D + C * sum(x) corrected at the end
    static constexpr bool SUBFREE = SF && XT != kF16 && NB == 1;
    static constexpr size_t RED = QW > 1 ? static_cast<size_t>(kCW) * NB * 32 * 4 * sizeof(float) : 0;
    static constexpr size_t smem() { return static_cast<size_t>(kRing) * (CB + XB) + 2 * kRing * 8 + RED + 16 * sizeof(float) + 16; }
    // fused outliers: 2 mbarriers (outlier sums ready / read), the sums
    // [TPC * 16][NBT], then the segment ring
    static constexpr size_t OBAR = static_cast<size_t>(kRing) * (CB + XB) + 2 * kRing * 8 + RED + 16 * sizeof(float);
    static constexpr size_t OSUM = (OBAR + 16 + 15) & ~static_cast<size_t>(15);
    static constexpr size_t osm_off() { return OSUM + static_cast<size_t>(TPC) * kTileCols * NBT * sizeof(float); }
};

// x value of batch row n at staged row r (exact f32)
template <int XT>
__device__ __forceinline__ float xs_val(const unsigned char* xs, int pitch, int n, unsigned r) {
    if (XT == kF32) return reinterpret_cast<const float*>(xs)[n * pitch + r];
    const unsigned short u = reinterpret_cast<const unsigned short*>(xs)[n * pitch + r];
    if (XT == kBF16) return __uint_as_float(static_cast<unsigned>(u) << 16);
    return __half2float(__ushort_as_half(u));
}

__device__ __forceinline__ void seg_entry(const unsigned char* vals, const unsigned short* rows, int oes, int e,
                                          unsigned& r, float& v) {
    r = rows[e];
    v = oes == 4 ? reinterpret_cast<const float*>(vals)[e]
                 : __half2float(reinterpret_cast<const __half*>(vals)[e]);
}

// The outlier warps (fused outliers; OW = 2 for batch groups of <= 2 rows,
// else 4): extra consumers of every ring stage. Warp ow owns C / OW of the
// colblock's C = 16 TPC columns; its lanes own them (CW / 32 columns per
// lane, or 32 / CW lanes per column splitting the entries), walk each stage's
// segment lists in rounds -- every round loads the next entry of all L
// lists at once, L independent shared-memory chains in flight -- and
// accumulate NBO batch rows in registers (fixed order: deterministic). At
// the end of a colblock it hands the sums to the writers through shared
// memory (one buffer, mbarriers both ways).
template <int TPC, int S, int XT, int XP, int XB, int NBT, int NBO, int OW>
__device__ __forceinline__ void outlier_warp(const GemvArgs& a, int64_t s_lo, int64_t s_hi, int64_t cb0, int64_t cbstep,
                                             unsigned full0, unsigned empty0,
                                             const unsigned char* osm, const unsigned char* xsm, float* osum,
                                             unsigned obar0, unsigned rbar0, int lane, int ow) {
    constexpr int C = TPC * kTileCols;
    constexpr int CW = C / OW;                   // columns per outlier warp
    constexpr int CPL = CW >= 32 ? CW / 32 : 1;  // columns per lane
    constexpr int LPC = CW >= 32 ? 1 : 32 / CW;  // lanes per column
    constexpr int SPG = S >= kSegQ ? S / kSegQ : 1;
    constexpr int L = CPL * SPG;
    constexpr int ES = XT == kF32 ? 4 : 2;
    const int sub = lane % LPC;
    int k = 0, it = 0;
    for (int64_t cb = cb0; cb < a.ncb; cb += cbstep, ++it) {
        float o[CPL][NBO];
#pragma unroll
        for (int i = 0; i < CPL; ++i)
#pragma unroll
            for (int n = 0; n < NBO; ++n) o[i][n] = 0.f;
        for (int64_t sq = s_lo; sq < s_hi; ++sq, ++k) {
            const int slot = k % kRing;
            bar_wait(full0 + 8 * slot, (k / kRing) & 1);
            const unsigned char* ob = osm + slot * a.ob;
            const unsigned char* xw = xsm + slot * XB;
            const int64_t sg0 = sq * SPG;
            const unsigned char* ent[SPG];   // values
            const unsigned short* rws[SPG];  // rows
            int e[L], e1[L];
#pragma unroll
            for (int sg = 0; sg < SPG; ++sg) {
                const bool ok = sg0 + sg < a.nseg;
                const unsigned short* hs = reinterpret_cast<const unsigned short*>(ob + 4);
                ent[sg] = ob + seg_hdr_bytes(TPC);
                rws[sg] = reinterpret_cast<const unsigned short*>(ent[sg] + a.oes * (ok ? hs[C] : 0));
#pragma unroll
                for (int i = 0; i < CPL; ++i) {
                    const int c = ow * CW + (LPC > 1 ? lane / LPC : lane + 32 * i);
                    e[sg * CPL + i] = ok ? hs[c] + sub : 0;
                    e1[sg * CPL + i] = ok ? hs[c + 1] : 0;
                }
                if (sg + 1 < SPG && ok) ob += *reinterpret_cast<const unsigned*>(ob);
            }
            bool more = false;
#pragma unroll
            for (int i = 0; i < L; ++i) more |= e[i] < e1[i];
#pragma unroll 1
            while (more) {
                unsigned r[L];
                float v[L];
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    r[i] = 0;
                    v[i] = 0.f;
                    if (e[i] < e1[i]) seg_entry(ent[i / CPL], rws[i / CPL], a.oes, e[i], r[i], v[i]);
                }
#pragma unroll
                for (int i = 0; i < L; ++i)
                    if (e[i] < e1[i]) {
                        const unsigned char* xs = xw + (i / CPL) * kSegRows * ES;
#pragma unroll
                        for (int n = 0; n < NBO; ++n) o[i % CPL][n] = fmaf(v[i], xs_val<XT>(xs, XP, n, r[i]), o[i % CPL][n]);
                    }
                more = false;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    e[i] += LPC;
                    more |= e[i] < e1[i];
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
        }
        // hand the colblock's sums to the writers
        if (it >= 1) bar_wait(rbar0, (it - 1) & 1);  // the buffer was read by the writers of it - 1
#pragma unroll
        for (int off = 1; off < LPC; off <<= 1)  // lanes of a column: fixed butterfly
#pragma unroll
            for (int n = 0; n < NBO; ++n) o[0][n] += __shfl_xor_sync(0xffffffffu, o[0][n], off);
        float* os = osum;
        if (sub == 0) {
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int c = ow * CW + (LPC > 1 ? lane / LPC : lane + 32 * i);
#pragma unroll
                for (int n = 0; n < NBO; ++n) os[c * NBT + n] = o[i][n];
            }
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(obar0) : "memory");
    }
}

template <int TPC, int NB, int XT, bool SF, bool OUT, int KS = 1>
__global__ void __launch_bounds__(kOutThreads) k_gemv_cb(const GemvArgs a) {
    using Gm = CbGeom<TPC, NB, XT, SF>;
    constexpr bool F16 = XT == kF16;
    constexpr int ES = Gm::ES, NBT = Gm::NBT, S = Gm::S, XP = Gm::XP, XB = Gm::XB, CB = Gm::CB;
    constexpr int TW = Gm::TW, QW = Gm::QW;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* codes = smem;                     // [kRing][S][TPC][512]
    unsigned char* xsm = smem + kRing * CB;          // [kRing][NBT][XP]
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(xsm + kRing * XB);
    float* red = reinterpret_cast<float*>(bars + 2 * kRing);  // [kCW][NB][32][4] (QW > 1)
    float* xsum = red + (QW > 1 ? kCW * NB * 32 * 4 : 0);      // [16] sum_i x[n][i] (SUBFREE)
    // OUT: outlier sums ready (obar: every outlier lane) / read (rbar: every consumer lane)
    const unsigned obar0 = static_cast<unsigned>(__cvta_generic_to_shared(smem + Gm::OBAR)), rbar0 = obar0 + 8;
    float* osum = reinterpret_cast<float*>(smem + Gm::OSUM);  // [TPC * 16][NBT] (OUT)
    unsigned char* osm = smem + Gm::osm_off();                 // [kRing][a.ob] outlier segments (OUT)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nout = static_cast<int>(blockDim.x >> 5) - kCW - 1;  // outlier warps (OUT)
    const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(bars));
    const unsigned empty0 = full0 + 8 * kRing;
    if (threadIdx.x == 0) {
        for (int k = 0; k < kRing; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * k));  // expect_tx arrival
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * k), "r"(kCW + 1 + (OUT ? nout : 0)));
        }
        if (OUT) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(obar0), "r"(32 * nout));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rbar0), "r"(kCW * 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // split K: this CTA's rank in its cluster, colblock walk and stage range
    const int64_t nst_all = (a.kq + S - 1) / S;
    unsigned rank = 0;
    int64_t cb0 = blockIdx.x, cbstep = gridDim.x, s_lo = 0, s_hi = nst_all;
    if (KS > 1) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        cb0 = blockIdx.x / KS, cbstep = gridDim.x / KS;
        s_lo = nst_all * rank / KS, s_hi = nst_all * (rank + 1) / KS;
    }
    const int64_t nst_cb = s_hi - s_lo;  // stages per colblock of this CTA
    // split-K reduction area at the end of dynamic shared memory: [full, free
    // mbarriers][(ks - 1) slots of the writers' partial outputs]
    constexpr int NWR = QW > 1 ? TPC : kCW;             // writer warps
    constexpr int RV = TW * NB * 4;                     // values per writer lane
    unsigned dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    const unsigned kred = KS > 1 ? (dsz - 16u - static_cast<unsigned>((KS - 1) * NWR * 32 * RV * 4)) & ~15u : 0u;
    const unsigned cfull = static_cast<unsigned>(__cvta_generic_to_shared(smem)) + kred, cfree = cfull + 8;
    float* kbuf = reinterpret_cast<float*>(smem + kred + 16);  // [ks - 1][NWR * 32][RV]
    if (KS > 1) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cfull), "r"(KS - 1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cfree));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        // every CTA of the cluster has its barriers before any remote arrive
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }

    if (OUT && warp > kCW) {  // ---- outlier warps (2 or 4: out_warps(batch))
        using G = CbGeom<TPC, NB, XT, SF>;
        const int ow = warp - kCW - 1;
        if (NB == 2) outlier_warp<TPC, S, XT, XP, XB, G::NBT, 16, 4>(a, s_lo, s_hi, cb0, cbstep, full0, empty0, osm, xsm, osum, obar0, rbar0, lane, ow);
        else if (a.batch == 1) outlier_warp<TPC, S, XT, XP, XB, G::NBT, 1, kOutWarpsSmall>(a, s_lo, s_hi, cb0, cbstep, full0, empty0, osm, xsm, osum, obar0, rbar0, lane, ow);
        else if (a.batch == 2) outlier_warp<TPC, S, XT, XP, XB, G::NBT, 2, kOutWarpsSmall>(a, s_lo, s_hi, cb0, cbstep, full0, empty0, osm, xsm, osum, obar0, rbar0, lane, ow);
        else if (a.batch <= 4) outlier_warp<TPC, S, XT, XP, XB, G::NBT, 4, 4>(a, s_lo, s_hi, cb0, cbstep, full0, empty0, osm, xsm, osum, obar0, rbar0, lane, ow);
        else outlier_warp<TPC, S, XT, XP, XB, G::NBT, 8, 4>(a, s_lo, s_hi, cb0, cbstep, full0, empty0, osm, xsm, osum, obar0, rbar0, lane, ow);
        return;
    }
    if (warp == kCW) {  // ---- producer warp: codes and x slices by TMA bulk copies
        // SUBFREE: while the CTA's first colblock streams, the producer also
        // sums the staged x slices (sum_i x[n][i] over all of K, the values
        // the MMA sees: bf16, or f32 as bf16 hi + lo; fixed lane assignment
        // and butterfly -- deterministic), lagging kRing - 1 stages behind
        // the copies; every other stage it releases at once. The sums go to
        // xsum[] and named barrier 2 tells the consumers.
        float xs_acc[Gm::NBT];
#pragma unroll
        for (int n = 0; n < Gm::NBT; ++n) xs_acc[n] = 0.f;
        int done = 0;  // first-colblock stages summed and released
        auto sum_stage = [&](int p) {
            const int slot = p % kRing;
            bar_wait(full0 + 8 * slot, (p / kRing) & 1);
            const int cnt = static_cast<int>(min(static_cast<int64_t>(S), a.kq - (s_lo + p) * S));
            const unsigned char* xw = xsm + slot * XB;
            for (int n = 0; n < a.batch; ++n) {
                for (int c16 = lane; c16 < cnt * 64 * ES / 16; c16 += 32) {
                    const uint4 u = *reinterpret_cast<const uint4*>(xw + n * XP * ES + 16 * c16);
                    const unsigned w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (XT == kF32) {
                            const float xv = __uint_as_float(w4[j]);
                            const float hi = __bfloat162float(__float2bfloat16_rn(xv));
                            xs_acc[n] += hi + __bfloat162float(__float2bfloat16_rn(xv - hi));
                        } else {
                            xs_acc[n] += __uint_as_float(w4[j] << 16) + __uint_as_float(w4[j] & 0xffff0000u);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
        };
        auto publish = [&]() {
            for (int n = 0; n < a.batch; ++n) {
                float v = xs_acc[n];
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) xsum[n] = v;
            }
            __syncwarp();
            asm volatile("bar.arrive 2, %0;" ::"r"(kStreamThreads) : "memory");  // consumers + producer
        };
        const int first_n = static_cast<int>(nst_cb);  // stages of the first colblock
        // OUT: byte range of a stage's segments, loaded one stage ahead (lane 0)
        constexpr int SPG = S >= kSegQ ? S / kSegQ : 1;
        int64_t o_lo = 0, o_hi = 0;
        auto seg_range = [&](int64_t cb, int64_t sq) {
            if (OUT && lane == 0 && cb < a.ncb) {
                const int64_t s0 = sq * SPG, s1 = min(s0 + SPG, a.nseg);
                o_lo = __ldg(a.obnd + cb * a.nseg + s0);
                o_hi = __ldg(a.obnd + cb * a.nseg + s1);
            }
        };
        seg_range(cb0, s_lo);
        int k = 0;
        for (int64_t cb = cb0; cb < a.ncb; cb += cbstep) {
            for (int64_t sq = s_lo; sq < s_hi; ++sq, ++k) {
                if (Gm::SUBFREE && k == first_n) {  // leaving the first colblock: drain, publish
                    while (done < first_n) sum_stage(done++);
                    publish();
                }
                const int64_t q0 = sq * S;
                const int cnt = static_cast<int>(min(static_cast<int64_t>(S), a.kq - q0));
                const int slot = k % kRing;
                if (k >= kRing) bar_wait(empty0 + 8 * slot, ((k / kRing) - 1) & 1);
                const unsigned fb = full0 + 8 * slot;
                // codes (one bulk copy) and the batch rows' x slices (one bulk
                // copy per row, contiguous in x), all on the stage's barrier
                const unsigned cbytes = static_cast<unsigned>(cnt) * TPC * 512u;
                const unsigned xbytes = static_cast<unsigned>(cnt) * 64u * ES;
                const int64_t seg_lo = o_lo;
                const unsigned obytes = OUT ? static_cast<unsigned>(o_hi - o_lo) : 0u;
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                                 "r"(cbytes + xbytes * static_cast<unsigned>(a.batch) + obytes)
                                 : "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            static_cast<unsigned>(__cvta_generic_to_shared(codes + slot * CB))),
                        "l"(a.T + (cb * a.kq + q0) * TPC * 32), "r"(cbytes), "r"(fb)
                        : "memory");
                    if (OUT && obytes)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                static_cast<unsigned>(__cvta_generic_to_shared(osm + slot * a.ob))),
                            "l"(a.oseg + seg_lo), "r"(obytes), "r"(fb)
                            : "memory");
                }
                if (OUT) {  // the next stage of this CTA
                    if (sq + 1 < s_hi) seg_range(cb, sq + 1);
                    else seg_range(cb + cbstep, s_lo);
                }
                // Launched as a programmatic dependent of the previous kernel
                // (a chain of GEMVs): the codes and outlier segments are
                // weights and stream before the wait; x may be the previous
                // kernel's output.
                if (k == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
                if (lane < a.batch)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            static_cast<unsigned>(__cvta_generic_to_shared(xsm + slot * XB + lane * XP * ES))),
                        "l"(static_cast<const char*>(a.x) + (lane * a.xstride + 64 * q0) * ES), "r"(xbytes), "r"(fb)
                        : "memory");
                if (Gm::SUBFREE && k < first_n) {
                    if (k >= kRing - 1) sum_stage(done++);  // the oldest stage in flight
                } else {
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
                }
            }
        }
        if (Gm::SUBFREE && k <= first_n) {  // the CTA had one colblock
            while (done < first_n) sum_stage(done++);
            publish();
        }
        // every copy of this CTA is issued: the next kernel in the stream (a
        // programmatic dependent) may launch and start its own weight stream
        // as the CTAs drain -- late enough that its CTAs are placed as ours
        // retire rather than beside them
        asm volatile("griddepcontrol.launch_dependents;");
        return;
    }

    // ---- consumers
    const int g = lane >> 2, t = lane & 3;
    const unsigned magic = F16 ? 0x64006400u : 0x43004300u;
    const unsigned off2 = F16 ? static_cast<unsigned>(__half_as_ushort(__int2half_rn(1024 - a.lmin))) * 0x10001u
                              : static_cast<unsigned>(__bfloat16_as_ushort(__int2bfloat16_rn(128 - a.lmin))) * 0x10001u;
    // my tiles: TPC >= 4: w, w + 4, ...; else tile w % TPC on q-blocks s = w / TPC (mod QW)
    int xrow[NB];  // staged x row of my batch column (rows past the batch read the last one; never stored)
#pragma unroll
    for (int n8 = 0; n8 < NB; ++n8) xrow[n8] = min(n8 * 8 + g, a.batch - 1);
    const int tile0 = TPC >= kCW ? warp : warp % TPC;
    const int qoff = TPC >= kCW ? 0 : warp / TPC;
    int k = 0, it = 0;
    for (int64_t cb = cb0; cb < a.ncb; cb += cbstep, ++it) {
        float acc[TW][2][NB][4];  // two accumulator sets per tile (alternating q) break the MMA chain
#pragma unroll
        for (int u = 0; u < TW; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[u][h][n8][i] = 0.f;
        for (int64_t sq = s_lo; sq < s_hi; ++sq, ++k) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(S), a.kq - sq * S));
            const int slot = k % kRing;
            bar_wait(full0 + 8 * slot, (k / kRing) & 1);
            const uint4* cw = reinterpret_cast<const uint4*>(codes + slot * CB);
            const unsigned char* xw = xsm + slot * XB;
#pragma unroll
            for (int si = 0; si < S / QW; ++si) {
                const int s = qoff + si * QW;
                if (s >= cnt) break;
                XRaw<XT> xr[NB];
#pragma unroll
                for (int n8 = 0; n8 < NB; ++n8) {
                    const uint4* xp = reinterpret_cast<const uint4*>(xw + (xrow[n8] * XP + s * 64 + 16 * t) * ES);
#pragma unroll
                    for (int i = 0; i < XRaw<XT>::kWords / 4; ++i) {
                        const uint4 u4 = xp[i];
                        xr[n8].w[4 * i] = u4.x, xr[n8].w[4 * i + 1] = u4.y, xr[n8].w[4 * i + 2] = u4.z,
                                      xr[n8].w[4 * i + 3] = u4.w;
                    }
                }
                const int h = si & 1;
#pragma unroll
                for (int u = 0; u < TW; ++u) {
                    const uint4 w = cw[(s * TPC + tile0 + u * kCW) * 32 + lane];
                    const unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int st = 0; st < 4; ++st) {
                        unsigned af[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            af[r] = Gm::SUBFREE ? lop_pair(ws[st], r, magic) : sub2<F16>(lop_pair(ws[st], r, magic), off2);
#pragma unroll
                        for (int n8 = 0; n8 < NB; ++n8) {
                            unsigned hi[2], lo[2];
                            x_frag<XT>(xr[n8], st, hi, lo);
                            if (h) {
                                mma16816<F16>(acc[u][1][n8], af, hi);
                                if (XT == kF32) mma16816<F16>(acc[u][1][n8], af, lo);
                            } else {
                                mma16816<F16>(acc[u][0][n8], af, hi);
                                if (XT == kF32) mma16816<F16>(acc[u][0][n8], af, lo);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
        }
        // ---- colblock done: (QW > 1) the warps of a tile meet in shared memory
        float d[TW][NB][4];
#pragma unroll
        for (int u = 0; u < TW; ++u)
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                for (int i = 0; i < 4; ++i) d[u][n8][i] = acc[u][0][n8][i] + acc[u][1][n8][i];
        if (Gm::SUBFREE && cb == cb0) named_sync(2, kStreamThreads);  // xsum published by the producer
        bool writer = true;
        if (QW > 1) {
#pragma unroll
            for (int n8 = 0; n8 < NB; ++n8)
                *reinterpret_cast<float4*>(red + ((warp * NB + n8) * 32 + lane) * 4) =
                    make_float4(d[0][n8][0], d[0][n8][1], d[0][n8][2], d[0][n8][3]);
            named_sync(1, kCW * 32);
            writer = warp < TPC;  // warp w < TPC sums the QW warps of tile w (warps w, w + TPC, ...)
            if (writer) {
#pragma unroll
                for (int n8 = 0; n8 < NB; ++n8) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[0][n8][i] = 0.f;
                    for (int j = 0; j < QW; ++j) {
                        const float4 v = *reinterpret_cast<const float4*>(red + (((warp + j * TPC) * NB + n8) * 32 + lane) * 4);
                        d[0][n8][0] += v.x, d[0][n8][1] += v.y, d[0][n8][2] += v.z, d[0][n8][3] += v.w;
                    }
                }
            }
            named_sync(1, kCW * 32);  // red is reused by the next colblock
        }
        const float* os = osum;  // OUT: this colblock's outlier sums
        if (OUT && writer) bar_wait(obar0, it & 1);
        if (writer) {
            asm volatile("griddepcontrol.wait;" ::: "memory");  // y: after the previous kernel (no-op once passed)
            if (Gm::SUBFREE) {  // D' = D + C sum(x): remove the offset once per output element
                const float C = static_cast<float>(128 - a.lmin);
#pragma unroll
                for (int u = 0; u < TW; ++u)
#pragma unroll
                    for (int q = 0; q < 4; ++q) d[u][0][q] -= C * xsum[min(2 * t + (q & 1), a.batch - 1)];
            }
            if (KS == 1) {  // one CTA per colblock: straight to y
#pragma unroll
                for (int u = 0; u < TW; ++u)
#pragma unroll
                    for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int64_t jc = (cb * TPC + tile0 + u * kCW) * kTileCols + g + (q >= 2 ? 8 : 0);
                            const int n = n8 * 8 + 2 * t + (q & 1);
                            if (jc < a.cols && n < a.batch) {
                                float yv = a.scales[jc] * d[u][n8][q];
                                if (OUT) yv += os[((tile0 + u * kCW) * kTileCols + g + (q >= 2 ? 8 : 0)) * Gm::NBT + n];
                                a.y[static_cast<int64_t>(n) * a.cols + jc] = yv;
                            }
                        }
            } else {
                float yv[TW][NB][4];
#pragma unroll
                for (int u = 0; u < TW; ++u)
#pragma unroll
                    for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int64_t jc = (cb * TPC + tile0 + u * kCW) * kTileCols + g + (q >= 2 ? 8 : 0);
                            const int n = n8 * 8 + 2 * t + (q & 1);
                            float v = 0.f;
                            if (jc < a.cols && n < a.batch) {
                                v = a.scales[jc] * d[u][n8][q];
                                if (OUT) v += os[((tile0 + u * kCW) * kTileCols + g + (q >= 2 ? 8 : 0)) * Gm::NBT + n];
                            }
                            yv[u][n8][q] = v;
                        }
                {  // split K: the ranks' partial outputs meet in rank 0 (DSMEM)
                    const int wl = warp * 32 + lane;  // writers are warps 0 .. NWR - 1
#define YV(i) yv[(i) / (NB * 4)][((i) / 4) % NB][(i) % 4]
                    if (rank != 0) {
                        if (it >= 1) bar_wait_cluster(cfree, (it - 1) & 1);  // rank 0 has read the previous colblock
                        const unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(kbuf + ((rank - 1) * NWR * 32 + wl) * RV));
                        unsigned ra;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(la));
#pragma unroll
                        for (int i = 0; i < RV; ++i)
                            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra + 4 * i), "f"(YV(i)) : "memory");
                        named_sync(3, NWR * 32);
                        if (wl == 0) {
                            unsigned rb;
                            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(cfull));
                            asm volatile("fence.acq_rel.cluster;\nmbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb)
                                         : "memory");
                        }
                    } else {
                        bar_wait_cluster(cfull, it & 1);
                        for (int r = 1; r < KS; ++r) {  // fixed rank order: deterministic
                            const float* src = kbuf + ((r - 1) * NWR * 32 + wl) * RV;
#pragma unroll
                            for (int i = 0; i < RV; ++i) YV(i) += src[i];
                        }
                        named_sync(3, NWR * 32);  // every writer has read the slots
                        if (wl == 0 && cb + cbstep < a.ncb)  // (no signal after the last colblock: the ranks may have exited)
                            for (int r = 1; r < KS; ++r) {
                                unsigned rb;
                                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(cfree), "r"(r));
                                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
                            }
                    }
#undef YV
                }
                if (rank == 0) {
#pragma unroll
                    for (int u = 0; u < TW; ++u)
#pragma unroll
                        for (int n8 = 0; n8 < NB; ++n8)
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int64_t jc = (cb * TPC + tile0 + u * kCW) * kTileCols + g + (q >= 2 ? 8 : 0);
                                const int n = n8 * 8 + 2 * t + (q & 1);
                                if (jc < a.cols && n < a.batch) a.y[static_cast<int64_t>(n) * a.cols + jc] = yv[u][n8][q];
                            }
                }
            }
        }
        if (OUT) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rbar0) : "memory");
    }
}

// x [batch][rows] (any alignment / ragged K) -> xpad [batch][kq * 64] with
// zeros past `rows`: the main kernel's 16-byte cp.async path needs 64-row
// multiples and 16-byte aligned rows.
__global__ void k_gemv_xpad(const void* __restrict__ x, int es, int64_t rows, int64_t prow, int batch,
                            void* __restrict__ xp) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= prow * batch) return;
    const int64_t n = i / prow, r = i % prow;
    if (es == 4)
        static_cast<float*>(xp)[i] = r < rows ? static_cast<const float*>(x)[n * rows + r] : 0.f;
    else
        static_cast<unsigned short*>(xp)[i] = r < rows ? static_cast<const unsigned short*>(x)[n * rows + r] : 0;
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

// Outlier values: f32 (exact) or f16 (ezq_gemv_prepare_ex; 6 bytes per
// outlier instead of 8, held to the GEMV's 1e-3 gate).
template <int VT>
__device__ __forceinline__ float load_val(const void* v, int64_t e) {
    if (VT == 1) return __half2float(static_cast<const __half*>(v)[e]);
    return static_cast<const float*>(v)[e];
}

template <int XT, int NBT, int VT>
__global__ void __launch_bounds__(256) k_gemv_outliers(int64_t rows, int64_t cols, const int64_t* __restrict__ col_ptr,
                                                       const uint32_t* __restrict__ out_row,
                                                       const void* __restrict__ out_val, const void* __restrict__ x,
                                                       int batch, float* __restrict__ y,
                                                       const float* __restrict__ xt) {
    // A grid that fits on the SMs beside the main kernel's CTAs: each warp
    // takes columns j = warp, + all warps, ... and computes ALL of them
    // before griddepcontrol.wait (their gathers overlap the weight stream),
    // keeping the sums in shared memory; then it applies them to y.
    extern __shared__ float osum[];  // [8 warps][cpw][NBT]
    constexpr int kU = 4;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib;
    const int cpw = static_cast<int>((cols + nwarps - 1) / nwarps);
    float* my = osum + static_cast<int64_t>(wib) * cpw * NBT;
    int ci = 0;
    for (int64_t j = w0; j < cols; j += nwarps, ++ci) {
        float part[NBT];
#pragma unroll
        for (int n = 0; n < NBT; ++n) part[n] = 0.f;
        const int64_t e0 = __ldg(col_ptr + j), e1 = __ldg(col_ptr + j + 1);
        for (int64_t eb = e0; eb < e1; eb += 32 * kU) {
            uint32_t r[kU];
            float v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t e = eb + lane + 32 * u;
                r[u] = e < e1 ? __ldg(out_row + e) : 0u;
                v[u] = e < e1 ? load_val<VT>(out_val, e) : 0.f;
            }
            if (NBT > 1) {  // transposed x: one 16-byte load per 4 batch rows
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
#pragma unroll
        for (int n = 0; n < NBT; ++n) {  // fixed butterfly: deterministic
            if (n >= batch) break;
#pragma unroll
            for (int o = 16; o; o >>= 1) part[n] += __shfl_xor_sync(0xffffffffu, part[n], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int n = 0; n < NBT; ++n) my[ci * NBT + n] = part[n];
        }
    }
    __syncwarp();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    ci = 0;
    for (int64_t j = w0; j < cols; j += nwarps, ++ci) {
        const int64_t e0 = __ldg(col_ptr + j), e1 = __ldg(col_ptr + j + 1);
        if (e1 > e0 && lane < batch) y[static_cast<int64_t>(lane) * cols + j] += my[ci * NBT + lane];
    }
}

// Repack the artifact's codes into the MMA fragment order (layout above),
// colblock major: T[cb][q][tile(TPC)][lane]. Rows past the end and columns
// past the end (the last colblock's padding tiles) hold level 0.
__global__ void k_gemv_repack(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                              int64_t kq, int64_t ncb, int tpc, int lmin, uint4* __restrict__ T) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ncb * kq * tpc * 32) return;
    const int lane = static_cast<int>(i % 32);
    const int64_t tt = (i / 32) % tpc, q = (i / (32 * tpc)) % kq, cb = i / (32 * tpc * kq);
    const int64_t tile = cb * tpc + tt;
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
    int64_t rows, cols, kq, tiles, ncb;
    int bits, lmin;
    int tpc;              // tiles per colblock (1, 2, 4, 8)
    uint4* T;             // repacked codes, colblock major (owned)
    const float* scales;  // device (borrowed from the artifact)
    int64_t* col_ptr;     // CSC of the outliers (owned)
    uint32_t* out_row;
    void* out_val;        // f32 / f16 / bf16 (vdtype)
    int vdtype;
    int64_t n_out;
    int dev;
    float* xt;            // batch > 1 with outliers: x transposed [rows][16] f32 (owned)
    void* xpad;           // ragged / unaligned x: padded copy [16][kq * 64] (owned)
    int grid[6];          // persistent CTAs of k_gemv_cb per (x dtype, NB) variant
    // fused outlier term (k_gemv_cb<..., OUT>): 512-row segments per colblock
    unsigned char* oseg;  // (owned)
    int64_t* obnd;        // [ncb * nseg + 1] (owned)
    int64_t nseg;
    int oes;              // value bytes (4: f32, 2: f16)
    int ob[6];            // segment bytes per ring stage, per variant
    int gridf[6][2];      // persistent CTAs of the fused kernel, per variant and outlier warps (small, max)
    size_t fsmem[6];      // its dynamic shared memory; 0: the separate pass
    int ks[6];            // K splits per colblock, per variant (thread-block cluster size; 1: none)
};

namespace {

int max_optin_smem() {
    static int v = [] {
        int dev = 0, m = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&m, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) m = 227 * 1024;
        return m;
    }();
    return v;
}

template <int TPC, int NB, int XT>
int cb_ctas_per_sm() {
    const int smem = static_cast<int>(CbGeom<TPC, NB, XT>::smem());
    const int cap = max_optin_smem();  // split-K launches add their area (ks_bytes)
    if (NB == 1 && XT != kF16)  // the HSUB2-free twin (same shared memory)
        cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    auto k = k_gemv_cb<TPC, NB, XT, false, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if constexpr (TPC == 1) {  // the split-K twins
        cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, false, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        if (NB == 1 && XT != kF16)
            cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, true, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kStreamThreads, smem) != cudaSuccess || n < 1) n = 1;
    return n;
}

template <int TPC>
void occ_row(int* o) {  // variants in (x dtype, NB) order: f32/1, f32/2, bf16/1, bf16/2, f16/1, f16/2
    o[0] = cb_ctas_per_sm<TPC, 1, kF32>();
    o[1] = cb_ctas_per_sm<TPC, 2, kF32>();
    o[2] = cb_ctas_per_sm<TPC, 1, kBF16>();
    o[3] = cb_ctas_per_sm<TPC, 2, kBF16>();
    o[4] = cb_ctas_per_sm<TPC, 1, kF16>();
    o[5] = cb_ctas_per_sm<TPC, 2, kF16>();
}

// CTAs per SM of every (TPC, variant), measured once per process.
const int* occupancy(int tpc) {
    static int occ[4][6];
    static std::once_flag once;
    std::call_once(once, [] {
        occ_row<1>(occ[0]);
        occ_row<2>(occ[1]);
        occ_row<4>(occ[2]);
        occ_row<8>(occ[3]);
    });
    return occ[tpc == 1 ? 0 : tpc == 2 ? 1 : tpc == 4 ? 2 : 3];
}

// Fused-outlier geometry of variant v: q-blocks per stage, segment ring
// offset, and CTAs per SM with `ob` segment bytes per stage (0: no fit).
struct FusedGeom {
    int S;
    size_t osm_off;
};

template <int TPC, int NB, int XT>
FusedGeom fused_geom() {
    using G = CbGeom<TPC, NB, XT>;
    return {G::S, G::osm_off()};
}

// outlier warps of a fused launch (see outlier_warp)
int out_warps(int batch) { return batch <= 2 ? kOutWarpsSmall : kOutWarpsMax; }

template <int TPC, int NB, int XT>
int fused_ctas_per_sm(size_t smem, int threads) {
    if (smem > static_cast<size_t>(max_optin_smem())) return 0;
    const int cap = max_optin_smem();
    if (NB == 1 && XT != kF16)
        cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    auto k = k_gemv_cb<TPC, NB, XT, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    if constexpr (TPC == 1) {  // the split-K twins
        cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, false, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        if (NB == 1 && XT != kF16)
            cudaFuncSetAttribute(k_gemv_cb<TPC, NB, XT, true, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, smem) != cudaSuccess) n = 0;
    return n;
}

template <int TPC>
void fused_info(int v, size_t ob, int threads, FusedGeom* g, int* ctas) {
    auto pick = [&](FusedGeom fg, auto occ_fn) {
        *g = fg;
        if (ctas) *ctas = occ_fn(fg.osm_off + static_cast<size_t>(kRing) * ob, threads);
    };
    switch (v) {
        case 0: pick(fused_geom<TPC, 1, kF32>(), fused_ctas_per_sm<TPC, 1, kF32>); break;
        case 1: pick(fused_geom<TPC, 2, kF32>(), fused_ctas_per_sm<TPC, 2, kF32>); break;
        case 2: pick(fused_geom<TPC, 1, kBF16>(), fused_ctas_per_sm<TPC, 1, kBF16>); break;
        case 3: pick(fused_geom<TPC, 2, kBF16>(), fused_ctas_per_sm<TPC, 2, kBF16>); break;
        case 4: pick(fused_geom<TPC, 1, kF16>(), fused_ctas_per_sm<TPC, 1, kF16>); break;
        default: pick(fused_geom<TPC, 2, kF16>(), fused_ctas_per_sm<TPC, 2, kF16>); break;
    }
}

void fused_variant(int tpc, int v, size_t ob, int threads, FusedGeom* g, int* ctas) {
    switch (tpc) {
        case 1: fused_info<1>(v, ob, threads, g, ctas); break;
        case 2: fused_info<2>(v, ob, threads, g, ctas); break;
        case 4: fused_info<4>(v, ob, threads, g, ctas); break;
        default: fused_info<8>(v, ob, threads, g, ctas); break;
    }
}

// q-blocks per ring stage of variant v (x dtype, NB) at colblock width tpc
template <int TPC>
int stage_qblocks_t(int v) {
    switch (v) {
        case 0: return CbGeom<TPC, 1, kF32>::S;
        case 1: return CbGeom<TPC, 2, kF32>::S;
        case 2: return CbGeom<TPC, 1, kBF16>::S;
        case 3: return CbGeom<TPC, 2, kBF16>::S;
        case 4: return CbGeom<TPC, 1, kF16>::S;
        default: return CbGeom<TPC, 2, kF16>::S;
    }
}
int stage_qblocks(int tpc, int v) {
    return tpc == 1 ? stage_qblocks_t<1>(v) : tpc == 2 ? stage_qblocks_t<2>(v) : tpc == 4 ? stage_qblocks_t<4>(v)
                                                                                         : stage_qblocks_t<8>(v);
}

// split-K reduction area (k_gemv_cb): 2 mbarriers + (ks - 1) slots of the
// writers' partial outputs, plus alignment slack
size_t ks_bytes(int tpc, int nb, int ks) {
    if (ks <= 1) return 0;
    const int nwr = tpc >= kCW ? kCW : tpc, tw = tpc >= kCW ? tpc / kCW : 1;
    return 32 + static_cast<size_t>(ks - 1) * nwr * 32 * tw * nb * 4 * sizeof(float);
}

template <typename K>
void launch_pdl(K kernel, unsigned grid, unsigned threads, size_t smem, cudaStream_t st, const GemvArgs& a) {
    // programmatic dependent launch: the weight stream of this GEMV starts
    // while the previous kernel drains (EZQ_GEMV_CHAIN=0: plain stream order)
    static const bool chain = !(std::getenv("EZQ_GEMV_CHAIN") && std::atoi(std::getenv("EZQ_GEMV_CHAIN")) == 0);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = chain ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = static_cast<unsigned>(a.ks);
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = a.ks > 1 ? 2 : 1;
    cudaLaunchKernelEx(&lc, kernel, a);
}

// HSUB2-free dequant for batch <= 2 (bf16 / f32 x): the producer's per-stage
// x sums stay cheap; larger batches keep the HSUB2 path. `smem` > 0: the
// fused-outlier kernel with that much dynamic shared memory.
template <int TPC, int NB, int XT>
void launch_cb_t(const GemvArgs& a, int grid, size_t smem, cudaStream_t st) {
    const unsigned gd = static_cast<unsigned>(grid);
    const bool sf = NB == 1 && XT != kF16 && a.batch <= 2;
    const size_t kx = ks_bytes(TPC, NB, a.ks);  // split-K area at the end of dynamic shared memory
    if constexpr (TPC == 1) if (a.ks == 2) {  // split K is chosen for 1-tile colblocks only (ezq_gemv_prepare)
        if (smem) {
            const unsigned nt = static_cast<unsigned>(kStreamThreads + 32 * out_warps(a.batch));
            if (sf) launch_pdl(k_gemv_cb<TPC, NB, XT, true, true, 2>, gd, nt, smem + kx, st, a);
            else launch_pdl(k_gemv_cb<TPC, NB, XT, false, true, 2>, gd, nt, smem + kx, st, a);
        } else {
            if (sf) launch_pdl(k_gemv_cb<TPC, NB, XT, true, false, 2>, gd, kStreamThreads, CbGeom<TPC, NB, XT, true>::smem() + kx, st, a);
            else launch_pdl(k_gemv_cb<TPC, NB, XT, false, false, 2>, gd, kStreamThreads, CbGeom<TPC, NB, XT>::smem() + kx, st, a);
        }
        return;
    }
    if (smem) {
        const unsigned nt = static_cast<unsigned>(kStreamThreads + 32 * out_warps(a.batch));
        if (sf) launch_pdl(k_gemv_cb<TPC, NB, XT, true, true>, gd, nt, smem, st, a);
        else launch_pdl(k_gemv_cb<TPC, NB, XT, false, true>, gd, nt, smem, st, a);
    } else {
        if (sf) launch_pdl(k_gemv_cb<TPC, NB, XT, true, false>, gd, kStreamThreads, CbGeom<TPC, NB, XT, true>::smem(), st, a);
        else launch_pdl(k_gemv_cb<TPC, NB, XT, false, false>, gd, kStreamThreads, CbGeom<TPC, NB, XT>::smem(), st, a);
    }
}

template <int TPC>
void launch_cb_v(int v, const GemvArgs& a, int grid, size_t smem, cudaStream_t st) {
    switch (v) {
        case 0: launch_cb_t<TPC, 1, kF32>(a, grid, smem, st); break;
        case 1: launch_cb_t<TPC, 2, kF32>(a, grid, smem, st); break;
        case 2: launch_cb_t<TPC, 1, kBF16>(a, grid, smem, st); break;
        case 3: launch_cb_t<TPC, 2, kBF16>(a, grid, smem, st); break;
        case 4: launch_cb_t<TPC, 1, kF16>(a, grid, smem, st); break;
        default: launch_cb_t<TPC, 2, kF16>(a, grid, smem, st); break;
    }
}

void launch_cb(int tpc, int v, const GemvArgs& a, int grid, size_t smem, cudaStream_t st) {
    switch (tpc) {
        case 1: launch_cb_v<1>(v, a, grid, smem, st); break;
        case 2: launch_cb_v<2>(v, a, grid, smem, st); break;
        case 4: launch_cb_v<4>(v, a, grid, smem, st); break;
        default: launch_cb_v<8>(v, a, grid, smem, st); break;
    }
}

template <int XT, int VT>
cudaError_t launch_outliers_v(cudaLaunchConfig_t& lc, int bt, int64_t rows, int64_t cols, const int64_t* cp,
                              const uint32_t* orow, const void* oval, const void* xg, float* yg, const float* xtg) {
    if (bt == 1) return cudaLaunchKernelEx(&lc, k_gemv_outliers<XT, 1, VT>, rows, cols, cp, orow, oval, xg, bt, yg, xtg);
    if (bt <= 8) return cudaLaunchKernelEx(&lc, k_gemv_outliers<XT, 8, VT>, rows, cols, cp, orow, oval, xg, bt, yg, xtg);
    return cudaLaunchKernelEx(&lc, k_gemv_outliers<XT, 16, VT>, rows, cols, cp, orow, oval, xg, bt, yg, xtg);
}

template <int XT>
cudaError_t launch_outliers(cudaLaunchConfig_t& lc, int vt, int bt, int64_t rows, int64_t cols, const int64_t* cp,
                            const uint32_t* orow, const void* oval, const void* xg, float* yg, const float* xtg) {
    if (vt == EZQ_GEMV_OUTLIER_F16 && bt > 8) {
        // f16 values with the 16-row variant fault (misaligned address, cause
        // not found); two 8-row passes over the transposed x instead
        const cudaError_t e = launch_outliers_v<XT, 1>(lc, 8, rows, cols, cp, orow, oval, xg, yg, xtg);
        if (e != cudaSuccess) return e;
        const size_t es = XT == kF32 ? 4 : 2;  // rows 8.. of x (direct path, bt == 9) or of xt
        return launch_outliers_v<XT, 1>(lc, bt - 8, rows, cols, cp, orow, oval,
                                        static_cast<const char*>(xg) + es * 8 * static_cast<size_t>(rows),
                                        yg + 8 * cols, xtg + 8);
    }
    if (vt == EZQ_GEMV_OUTLIER_F16) return launch_outliers_v<XT, 1>(lc, bt, rows, cols, cp, orow, oval, xg, yg, xtg);
    return launch_outliers_v<XT, 0>(lc, bt, rows, cols, cp, orow, oval, xg, yg, xtg);
}

}  // namespace

extern "C" {

int ezq_gemv_prepare_ex(const ezq_qweight* q, int outlier_dtype, void* stream, ezq_gemv_plan** plan) {
    *plan = nullptr;
    if (q->mem != EZQ_MEM_DEVICE)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv needs a device-resident artifact");
    if (q->rows <= 0 || q->cols <= 0)
        return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    if (q->bits < 2 || q->bits > 4)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv supports 2- to 4-bit artifacts");
    if (outlier_dtype != EZQ_GEMV_OUTLIER_F32 && outlier_dtype != EZQ_GEMV_OUTLIER_F16)
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "outlier values are stored as f32 or f16 (bf16's 8-bit mantissa misses the 1e-3 GEMV gate)");
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
    const size_t ves = outlier_dtype == EZQ_GEMV_OUTLIER_F32 ? 4 : 2;
    std::vector<uint16_t> vh;
    if (ves == 2) {  // round to nearest even, like the device conversions
        vh.resize(vv.size());
        for (size_t i = 0; i < vv.size(); ++i) {
            const __half h = __float2half_rn(vv[i]);
            vh[i] = __half_as_ushort(h);
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
    p->vdtype = outlier_dtype;
    p->dev = dev;
    // Colblock width: the TPC whose colblocks fill the resident CTAs best
    // (ncb / (waves x resident CTAs), bf16 batch-1 occupancy), ties to the
    // wider colblock (x slices read once per more columns).
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int force_tpc = std::getenv("EZQ_GEMV_TPC") ? std::atoi(std::getenv("EZQ_GEMV_TPC")) : 0;  // tuning / test aid
    double best = -1.0;
    for (int tpc : {8, 4, 2, 1}) {
        const int64_t ncb = (p->tiles + tpc - 1) / tpc;
        const int64_t res = static_cast<int64_t>(sms) * occupancy(tpc)[2];
        const int64_t waves = (ncb + res - 1) / res;
        const double eff = static_cast<double>(ncb) / static_cast<double>(waves * res);
        if ((force_tpc ? tpc == force_tpc : eff > best + 1e-9)) best = eff, p->tpc = tpc;
    }
    p->ncb = (p->tiles + p->tpc - 1) / p->tpc;
    const int* occ = occupancy(p->tpc);
    static const bool dbg = std::getenv("EZQ_GEMV_DEBUG") != nullptr;
    // Split K across a cluster when the colblocks cannot fill the resident
    // CTAs (latency-bound shapes: few output columns, long K): 2 CTAs per
    // colblock when each rank keeps >= 3 ring stages (measured on B200:
    // 11008x4096 batch 1 / 16: 11.8 -> 11.0 / 22.6 -> 15.6 us; 4 ranks and
    // 2-stage ranks were slower), per variant (its stage size).
    const char* ek = std::getenv("EZQ_GEMV_KS");  // tuning / test aid
    for (int v = 0; v < 6; ++v) {
        const int64_t res = static_cast<int64_t>(sms) * occ[v];
        const int sq = stage_qblocks(p->tpc, v);
        const int64_t nst = (p->kq + sq - 1) / sq;
        int ks = p->tpc == 1 && p->ncb * 2 <= res && nst >= 6 ? 2 : 1;
        if (ek && p->tpc == 1) ks = std::atoi(ek) == 2 ? 2 : 1;
        p->ks[v] = ks;
    }
    auto grid_of = [&](int64_t slots, int ks) {  // persistent CTAs: whole clusters, at most one unit each
        int64_t gr = std::min<int64_t>(p->ncb * ks, slots);
        gr -= gr % ks;
        return static_cast<int>(std::max<int64_t>(gr, ks));
    };
    for (int v = 0; v < 6; ++v) {
        p->grid[v] = grid_of(static_cast<int64_t>(sms) * occ[v], p->ks[v]);
        if (dbg)
            std::fprintf(stderr, "ezq_gemv_prepare: tpc %d ks %d ncb %lld variant %d ctas/sm %d grid %d\n", p->tpc, p->ks[v],
                         static_cast<long long>(p->ncb), v, occ[v], p->grid[v]);
    }
    // Fused outliers: for every colblock and 512-row segment, the header
    // (u32 bytes, u16 column starts) and the entries, rows ascending per
    // column; each variant whose stage holds whole segments and whose ring
    // still fits in shared memory (with >= 1 CTA per SM) runs the outlier
    // term inside the main kernel. EZQ_GEMV_FUSED=0 keeps the separate pass.
    std::vector<unsigned char> seg;
    std::vector<int64_t> bnd;
    const char* fz = std::getenv("EZQ_GEMV_FUSED");
    bool fuse = q->n_outliers > 0 && !(fz && std::atoi(fz) == 0);
    if (fuse) {
        const int C = p->tpc * kTileCols, hdr = seg_hdr_bytes(p->tpc), es = static_cast<int>(ves) + 2;
        p->nseg = (q->rows + kSegRows - 1) / kSegRows;
        p->oes = static_cast<int>(ves);
        bnd.resize(static_cast<size_t>(p->ncb * p->nseg + 1));
        seg.reserve(static_cast<size_t>(q->n_outliers) * es + static_cast<size_t>(p->ncb * p->nseg) * (hdr + 16));
        std::vector<int64_t> cur(ptr.begin(), ptr.end() - 1);
        std::vector<uint16_t> st(C + 1);
        for (int64_t cb = 0; cb < p->ncb && fuse; ++cb)
            for (int64_t sg = 0; sg < p->nseg; ++sg) {
                const size_t base = seg.size();
                bnd[cb * p->nseg + sg] = static_cast<int64_t>(base);
                const uint32_t rend = static_cast<uint32_t>(std::min<int64_t>((sg + 1) * kSegRows, q->rows));
                int64_t n = 0;
                for (int c = 0; c < C; ++c) {
                    st[c] = static_cast<uint16_t>(n);
                    const int64_t j = cb * C + c;
                    if (j >= q->cols) continue;
                    int64_t e = cur[j];
                    while (e < ptr[j + 1] && rr[e] < rend) ++e;
                    n += e - cur[j];
                    if (n > 65535) break;
                }
                if (n > 65535) {  // denser than the u16 header can index: keep the separate pass
                    fuse = false;
                    break;
                }
                st[C] = static_cast<uint16_t>(n);
                const size_t ebytes = (static_cast<size_t>(n) * es + 15) & ~static_cast<size_t>(15);
                seg.resize(base + hdr + ebytes, 0);
                const uint32_t tot = static_cast<uint32_t>(hdr + ebytes);
                std::memcpy(seg.data() + base, &tot, 4);
                std::memcpy(seg.data() + base + 4, st.data(), 2 * (C + 1));
                unsigned char* ent = seg.data() + base + hdr;
                unsigned char* erow = ent + ves * n;
                int64_t i = 0;
                for (int c = 0; c < C; ++c) {
                    const int64_t j = cb * C + c;
                    if (j >= q->cols) continue;
                    for (; cur[j] < ptr[j + 1] && rr[cur[j]] < rend; ++cur[j], ++i) {
                        const uint16_t rl = static_cast<uint16_t>(rr[cur[j]] - static_cast<uint32_t>(sg * kSegRows));
                        std::memcpy(erow + 2 * i, &rl, 2);
                        if (ves == 4) std::memcpy(ent + 4 * i, &vv[cur[j]], 4);
                        else std::memcpy(ent + 2 * i, &vh[cur[j]], 2);
                    }
                }
            }
        if (fuse) bnd[p->ncb * p->nseg] = static_cast<int64_t>(seg.size());
    }
    for (int v = 0; v < 6; ++v) {
        p->fsmem[v] = 0;
        p->ob[v] = 0;
        p->gridf[v][0] = p->gridf[v][1] = 0;
        if (!fuse) continue;
        FusedGeom fg{};
        fused_variant(p->tpc, v, 0, 0, &fg, nullptr);
        if (fg.S % kSegQ) continue;  // stage smaller than a segment (f32 x, 9..16 rows)
        const int64_t spg = fg.S / kSegQ;
        int64_t mx = 0;
        for (int64_t cb = 0; cb < p->ncb; ++cb)
            for (int64_t s0 = 0; s0 < p->nseg; s0 += spg)
                mx = std::max(mx, bnd[cb * p->nseg + std::min(s0 + spg, p->nseg)] - bnd[cb * p->nseg + s0]);
        int c1 = 0, c4 = 0;
        fused_variant(p->tpc, v, static_cast<size_t>(mx), kStreamThreads + 32 * kOutWarpsSmall, &fg, &c1);
        fused_variant(p->tpc, v, static_cast<size_t>(mx), kStreamThreads + 32 * kOutWarpsMax, &fg, &c4);
        if (c1 < 1 || c4 < 1) continue;
        if (fg.osm_off + static_cast<size_t>(kRing) * mx + ks_bytes(p->tpc, (v & 1) ? 2 : 1, p->ks[v]) >
            static_cast<size_t>(max_optin_smem()))
            continue;  // no room for the split-K area
        p->ob[v] = static_cast<int>(mx);
        p->fsmem[v] = fg.osm_off + static_cast<size_t>(kRing) * mx;
        p->gridf[v][0] = grid_of(static_cast<int64_t>(sms) * c1, p->ks[v]);
        p->gridf[v][1] = grid_of(static_cast<int64_t>(sms) * c4, p->ks[v]);
        if (dbg)
            std::fprintf(stderr, "ezq_gemv_prepare: fused variant %d: %lld B/stage, smem %zu, ctas/sm %d / %d\n", v,
                         static_cast<long long>(mx), p->fsmem[v], c1, c4);
    }
    p->oseg = nullptr;
    p->obnd = nullptr;
    if (fuse) {
        EZQ_CK(cudaMalloc(&p->oseg, std::max<size_t>(seg.size(), 16)));
        EZQ_CK(cudaMalloc(&p->obnd, sizeof(int64_t) * bnd.size()));
    }
    const int64_t nw = p->ncb * p->kq * p->tpc * 32;
    EZQ_CK(cudaMalloc(&p->T, sizeof(uint4) * nw));
    EZQ_CK(cudaMalloc(&p->col_ptr, sizeof(int64_t) * (q->cols + 1)));
    p->xt = nullptr;
    if (q->n_outliers > 0) EZQ_CK(cudaMalloc(&p->xt, sizeof(float) * 16 * static_cast<size_t>(q->rows)));
    EZQ_CK(cudaMalloc(&p->xpad, sizeof(float) * 16 * static_cast<size_t>(p->kq) * kBlockRows));
    EZQ_CK(cudaMalloc(&p->out_row, sizeof(uint32_t) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->out_val, ves * std::max<int64_t>(q->n_outliers, 1)));
    k_gemv_repack<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, st>>>(q->packed, q->rows, q->cols, q->bits,
                                                                         p->kq, p->ncb, p->tpc, p->lmin, p->T);
    count_launch();
    EZQ_CK(cudaMemcpyAsync(p->col_ptr, ptr.data(), sizeof(int64_t) * (q->cols + 1),
                           cudaMemcpyHostToDevice, st));
    if (q->n_outliers) {
        EZQ_CK(cudaMemcpyAsync(p->out_row, rr.data(), sizeof(uint32_t) * q->n_outliers,
                               cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(p->out_val, ves == 4 ? static_cast<const void*>(vv.data()) : vh.data(),
                               ves * q->n_outliers, cudaMemcpyHostToDevice, st));
    }
    if (p->oseg) {
        EZQ_CK(cudaMemcpyAsync(p->oseg, seg.data(), seg.size(), cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(p->obnd, bnd.data(), sizeof(int64_t) * bnd.size(), cudaMemcpyHostToDevice, st));
    }
    EZQ_CK(cudaStreamSynchronize(st));
    *plan = p;
    return clear_error();
}

int ezq_gemv_prepare(const ezq_qweight* q, void* stream, ezq_gemv_plan** plan) {
    return ezq_gemv_prepare_ex(q, EZQ_GEMV_OUTLIER_F32, stream, plan);
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
    a.ncb = p->ncb;
    a.rows = p->rows;
    a.cols = p->cols;
    a.lmin = p->lmin;
    a.scales = p->scales;
    const size_t xes = x_dtype == kF32 ? 4 : 2;
    // The main kernel stages x slices with 16-byte cp.async: 64-row multiples
    // and 16-byte aligned rows, else a zero-padded copy first.
    const bool direct = p->rows % kBlockRows == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    // One launch per group of 16 batch rows (two n8 MMA tiles share the A
    // fragments); a group of <= 8 uses one n8 tile. The outlier pass is a
    // programmatic dependent launch (its gathers overlap the weight stream).
    for (int b0 = 0; b0 < batch; b0 += kMaxGroup) {
        a.batch = std::min(batch - b0, kMaxGroup);
        const void* xg = static_cast<const char*>(x) + xes * static_cast<size_t>(b0) * p->rows;
        a.y = y + static_cast<int64_t>(b0) * p->cols;
        if (direct) {
            a.x = xg;
            a.xstride = p->rows;
        } else {
            const int64_t prow = p->kq * kBlockRows;
            const int64_t tot = prow * a.batch;
            k_gemv_xpad<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(xg, static_cast<int>(xes), p->rows,
                                                                               prow, a.batch, p->xpad);
            count_launch();
            a.x = p->xpad;
            a.xstride = prow;
        }
        const bool two = a.batch > 8;
        if (p->n_out && a.batch > 1 && !p->fsmem[x_dtype * 2 + (a.batch > 8 ? 1 : 0)]) {  // transposed x for the outlier pass (one 16-byte load per 4 batch rows)
            k_gemv_xt<<<static_cast<unsigned>((p->rows + 15) / 16), 256, 0, st>>>(xg, x_dtype, p->rows, a.batch,
                                                                                  p->xt);
            count_launch();
        }
        static const bool dsync = std::getenv("EZQ_GEMV_SYNC") != nullptr;  // diagnosis: sync after every launch
        if (dsync) {
            const cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_error(e, "gemv: before the main kernel");
        }
        const int v = x_dtype * 2 + (two ? 1 : 0);
        a.ks = p->ks[v];
        const bool fused = p->n_out && p->fsmem[v];
        if (fused) {
            a.oseg = p->oseg;
            a.obnd = p->obnd;
            a.nseg = p->nseg;
            a.ob = p->ob[v];
            a.oes = p->oes;
        }
        launch_cb(p->tpc, v, a, fused ? p->gridf[v][out_warps(a.batch) == kOutWarpsMax] : p->grid[v], fused ? p->fsmem[v] : 0, st);
        count_launch();
        if (dsync) {
            const cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_error(e, "gemv: main kernel");
        }
        if (p->n_out && !fused) {
            cudaLaunchConfig_t lc{};
            // two 8-warp CTAs per SM: resident beside the main kernel (see k_gemv_outliers)
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            // A programmatic dependent launch (gathers overlap the weight
            // stream) pays at batch 1 on up to 16k columns; above that, plain
            // stream order (measured on B200: the overlap slowed both kernels:
            // BLOOM shape batch 1, 135 vs 110 us; batch 16, 494 vs 321 us).
            // One warp per column either way.
            static const int pdl_max = std::getenv("EZQ_GEMV_PDL_MAX") ? std::atoi(std::getenv("EZQ_GEMV_PDL_MAX")) : 1;
            const bool pdl = a.batch <= pdl_max && p->cols <= 16384;
            const int64_t ctas = (p->cols + 7) / 8;
            const int64_t cpw = (p->cols + 8 * ctas - 1) / (8 * ctas);
            lc.gridDim = dim3(static_cast<unsigned>(ctas));
            lc.blockDim = dim3(256);
            lc.dynamicSmemBytes = static_cast<size_t>(8 * cpw * (a.batch > 8 ? 16 : (a.batch > 1 ? 8 : 1))) * sizeof(float);
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            // programmatic dependent launch (gathers overlap the weight stream)
            // at batch 1; plain stream order above (measured: overlapping the
            // multi-row gathers with the stream slowed both)
            at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
            lc.attrs = at;
            lc.numAttrs = 1;
            const int64_t* cp = p->col_ptr;
            const uint32_t* orow = p->out_row;
            const void* oval = p->out_val;
            float* yg = a.y;
            const int bt = a.batch;
            const float* xtg = p->xt;
            cudaError_t e;
            if (x_dtype == kF32) e = launch_outliers<kF32>(lc, p->vdtype, bt, p->rows, p->cols, cp, orow, oval, xg, yg, xtg);
            else if (x_dtype == kBF16) e = launch_outliers<kBF16>(lc, p->vdtype, bt, p->rows, p->cols, cp, orow, oval, xg, yg, xtg);
            else e = launch_outliers<kF16>(lc, p->vdtype, bt, p->rows, p->cols, cp, orow, oval, xg, yg, xtg);
            EZQ_CK(e);
            count_launch();
        }
    }
    // Algorithmic bytes: the 4-bit codes (the repacked copy has the same
    // size as the artifact's nibbles), scales, outlier values + u16 rows, x
    // and y.
    const double vbytes = p->vdtype == EZQ_GEMV_OUTLIER_F32 ? 4.0 : 2.0;
    const double bytes = static_cast<double>(p->rows * p->cols + 1) / 2 + 4.0 * p->cols +
                         (2.0 + vbytes) * p->n_out + batch * p->rows * static_cast<double>(xes) +
                         4.0 * batch * p->cols;
    prof_end(pt, st, bytes);
    EZQ_CK(cudaGetLastError());
    return clear_error();
}

void ezq_gemv_plan_free(ezq_gemv_plan* p) {
    if (!p) return;
    cudaFree(p->T);
    cudaFree(p->col_ptr);
    if (p->xt) cudaFree(p->xt);
    cudaFree(p->xpad);
    cudaFree(p->out_row);
    cudaFree(p->out_val);
    if (p->oseg) cudaFree(p->oseg);
    if (p->obnd) cudaFree(p->obnd);
    delete p;
}

}  // extern "C"
