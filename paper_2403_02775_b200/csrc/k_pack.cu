// K4 (final levels + packing) and K5 (dense restore + outlier scatter).
//
// K4 restates quantize_channel (rtn.cpp:88-99) at the stored float scale,
// the outlier-slot convention (level 0, pipeline.cpp:86) and pack_levels
// (rtn.cpp:123-149): k = 4 packs (level - lmin) nibbles with the even FLAT
// index in the low nibble (pairs straddle rows when cols is odd); any other
// k stores one offset byte per level. One thread owns 16 consecutive flat
// elements -> one 8-byte (k=4) or 16-byte store. HBM-bound: 4N bytes read,
// N/2 (or N) written.
//
// K5 restates dequantize_impl (pipeline.cpp:117-142): What_ij =
// float(double(s_j) * l_ij), which equals the correctly rounded fp32 product
// s_j * l_ij (the fp64 product is exact), then the stored outlier values are
// scattered back bit-exactly (outliers.cpp:106-114).
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

// Per-element path of k_pack (row wraps, ragged tails, unaligned columns).
__device__ __forceinline__ void pack_levels_slow(const float (&x)[kPackPerThread], uint8_t (&off)[kPackPerThread], int64_t col, int64_t cnt, int64_t C,
                                              const TDesc& d, const Scratch& sc, const CfgDev& cfg, float olo,
                                              float ohi) {
    const double dmin = cfg.lmin, dmax = cfg.lmax;
    const float fmin = static_cast<float>(cfg.lmin), fmax = static_cast<float>(cfg.lmax);
    const float guard = cfg.guard;
    // Per-column float 1/scale for the certified fp32 level (K3b wrote it);
    // the 16 columns are contiguous unless the run wraps a row.
    float invf[kPackPerThread];
    const float* ivp = sc.invf + d.col_base;
    if (col + kPackPerThread <= C && ((d.col_base + col) & 3) == 0) {
#pragma unroll
        for (int k = 0; k < kPackPerThread / 4; ++k) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(ivp + col) + k);
            invf[4 * k] = v.x, invf[4 * k + 1] = v.y, invf[4 * k + 2] = v.z, invf[4 * k + 3] = v.w;
        }
    } else {
        int64_t cc = col;
#pragma unroll
        for (int k = 0; k < kPackPerThread; ++k) {
            invf[k] = __ldg(ivp + cc);
            if (++cc == C) cc = 0;
        }
    }
#pragma unroll
    for (int k = 0; k < kPackPerThread; ++k) {
        int lvl = 0;
        if (k < cnt && !is_outlier_f(x[k], olo, ohi)) {
            const FastLevel fl{invf[k], fmin, fmax};
            float rm = 0.f;
            float q = level_fast(x[k], fl, rm);
            if (rm >= guard) q = static_cast<float>(level_exact(x[k], sc.inv[d.col_base + col], dmin, dmax));
            lvl = static_cast<int>(q);
        }
        off[k] = (k < cnt) ? static_cast<uint8_t>(lvl - cfg.lmin) : 0;
        if (++col == C) col = 0;
    }

}

__global__ void __launch_bounds__(kPackThreads) k_pack(const TDesc* __restrict__ td,
                                                       const int64_t* __restrict__ pblk_base,
                                                       int ntens, int64_t total, Scratch sc,
                                                       CfgDev cfg) {
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    const int t = find_tensor(pblk_base, ntens, g);
    const TDesc& d = td[t];
    if (d.pack_fused) return;  // K3b wrote this tensor's codes
    const int64_t e0 = ((g - d.pblk_base) * kPackThreads + threadIdx.x) * kPackPerThread;
    if (e0 >= d.n) return;
    const TStats* st = d.st;
    const float olo = st->olo, ohi = st->ohi;
    const int64_t C = d.cols;
    const int64_t col = e0 % C;
    const int64_t cnt = min(static_cast<int64_t>(kPackPerThread), d.n - e0);

    float x[kPackPerThread];
    if (cnt == kPackPerThread && (reinterpret_cast<uintptr_t>(d.W + e0) & 15) == 0) {
        const float4* p4 = reinterpret_cast<const float4*>(d.W + e0);
#pragma unroll
        for (int k = 0; k < kPackPerThread / 4; ++k) {
            const float4 v = __ldg(p4 + k);
            x[4 * k] = v.x;
            x[4 * k + 1] = v.y;
            x[4 * k + 2] = v.z;
            x[4 * k + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kPackPerThread; ++k) x[k] = (k < cnt) ? d.W[e0 + k] : 0.f;
    }

    uint8_t off[kPackPerThread];
    const float fmin = static_cast<float>(cfg.lmin), fmax = static_cast<float>(cfg.lmax);
    if (cnt == kPackPerThread && col + kPackPerThread <= C && ((d.col_base + col) & 3) == 0) {
        // Common case: 16 contiguous columns of one row. Certified fp32 levels
        // for the group (one guard test), the level's offset byte straight
        // from the magic-added bits (0x4B400000 + q), outlier slots -> level 0.
        const float4* iv4 = reinterpret_cast<const float4*>(sc.invf + d.col_base + col);
        float rmax = 0.f;
        unsigned tb[kPackPerThread];
#pragma unroll
        for (int k4 = 0; k4 < kPackPerThread / 4; ++k4) {
            const float4 v = __ldg(iv4 + k4);
            const float iv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * k4 + j;
                float u = __fmul_rn(x[k], iv[j]);
                u = fminf(fmaxf(u, fmin), fmax);
                const float t = __fadd_rn(u, kMagic);
                rmax = fmaxf(rmax, fabsf(__fsub_rn(u, __fsub_rn(t, kMagic))));
                tb[k] = __float_as_uint(t);
            }
        }
        if (rmax >= cfg.guard) {  // an element near a rounding boundary: reference fp64 levels
            const double dmin = cfg.lmin, dmax = cfg.lmax;
#pragma unroll
            for (int k = 0; k < kPackPerThread; ++k) {
                const double q = level_exact(x[k], sc.inv[d.col_base + col + k], dmin, dmax);
                tb[k] = __float_as_uint(__fadd_rn(static_cast<float>(q), kMagic));
            }
        }
        const unsigned base = __float_as_uint(kMagic) + static_cast<unsigned>(cfg.lmin);
#pragma unroll
        for (int k = 0; k < kPackPerThread; ++k)
            off[k] = is_outlier_f(x[k], olo, ohi) ? static_cast<uint8_t>(-cfg.lmin) : static_cast<uint8_t>(tb[k] - base);
    } else {
        pack_levels_slow(x, off, col, cnt, C, d, sc, cfg, olo, ohi);
    }
    if (cfg.bits == 4) {
        uint8_t b[kPackPerThread / 2];
#pragma unroll
        for (int k = 0; k < kPackPerThread / 2; ++k)
            b[k] = static_cast<uint8_t>(off[2 * k] | (off[2 * k + 1] << 4));
        uint8_t* dst = d.packed + e0 / 2;
        if (cnt == kPackPerThread) {
            uint2 w;
            w.x = b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<uint32_t>(b[3]) << 24);
            w.y = b[4] | (b[5] << 8) | (b[6] << 16) | (static_cast<uint32_t>(b[7]) << 24);
            *reinterpret_cast<uint2*>(dst) = w;
        } else {
            const int64_t nb = (cnt + 1) / 2;
            for (int64_t k = 0; k < nb; ++k) dst[k] = b[k];
        }
    } else {
        uint8_t* dst = d.packed + e0;
        if (cnt == kPackPerThread) {
            uint4 w;
            w.x = off[0] | (off[1] << 8) | (off[2] << 16) | (static_cast<uint32_t>(off[3]) << 24);
            w.y = off[4] | (off[5] << 8) | (off[6] << 16) | (static_cast<uint32_t>(off[7]) << 24);
            w.z = off[8] | (off[9] << 8) | (off[10] << 16) | (static_cast<uint32_t>(off[11]) << 24);
            w.w = off[12] | (off[13] << 8) | (off[14] << 16) |
                  (static_cast<uint32_t>(off[15]) << 24);
            *reinterpret_cast<uint4*>(dst) = w;
        } else {
            for (int64_t k = 0; k < cnt; ++k) dst[k] = off[k];
        }
    }
}

// A CTA's kPackBlock elements go as quads: thread t writes elements
// 4 (t + kPackThreads k) .. + 3 with one float4 each (consecutive lanes,
// consecutive 16-byte stores; the codes are read as one u16 (k = 4) or u32
// per quad, also coalesced).
__global__ void __launch_bounds__(kPackThreads) k_dequant(int64_t rows, int64_t cols, int bits,
                                                          const uint8_t* __restrict__ packed,
                                                          const float* __restrict__ scales,
                                                          float* __restrict__ out,
                                                          unsigned long long* bad_byte) {
    const int64_t n = rows * cols;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kPackBlock;
    const int cnt = static_cast<int>(min(kPackBlock, n - b0));
    const int lmin = -(1 << (bits - 1)) + 1;
    const int span = (1 << (bits - 1)) - lmin;
    // vector paths need aligned bases (b0 is a multiple of 4096)
    const bool vout = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const bool vin = (reinterpret_cast<uintptr_t>(packed) & (bits == 4 ? 1 : 3)) == 0;
#pragma unroll
    for (int k = 0; k < kPackPerThread / 4; ++k) {
        const int l = 4 * (threadIdx.x + kPackThreads * k);
        if (l >= cnt) break;
        const int64_t e = b0 + l;
        const int m = min(4, cnt - l);
        uint8_t off[4];
        if (bits == 4) {
            if (vin && m == 4) {
                const unsigned w = __ldg(reinterpret_cast<const unsigned short*>(packed + e / 2));
                off[0] = w & 0xf, off[1] = (w >> 4) & 0xf, off[2] = (w >> 8) & 0xf, off[3] = (w >> 12) & 0xf;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint8_t b = j < m ? packed[(e + j) / 2] : 0;
                    off[j] = ((e + j) & 1) ? (b >> 4) : (b & 0x0f);
                }
            }
        } else {
            if (vin && m == 4) {
                const unsigned w = __ldg(reinterpret_cast<const unsigned*>(packed + e));
#pragma unroll
                for (int j = 0; j < 4; ++j) off[j] = (w >> (8 * j)) & 0xff;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) off[j] = j < m ? packed[e + j] : 0;
            }
            // unpack_levels rejects offsets beyond the level span (rtn.cpp:173-178).
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < m && off[j] > span) atomicMin(bad_byte, static_cast<unsigned long long>(e + j));
        }
        // 32-bit modulo when the tensor has < 2^32 elements (a 64-bit IMOD per quad costs more than the quad)
        int64_t col = n < (int64_t(1) << 32) ? static_cast<int64_t>(static_cast<uint32_t>(e) % static_cast<uint32_t>(cols))
                                             : e % cols;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = __fmul_rn(__ldg(scales + col), static_cast<float>(lmin + off[j]));
            if (++col == cols) col = 0;
        }
        if (vout && m == 4) {
            *reinterpret_cast<float4*>(out + e) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < m) out[e + j] = v[j];
        }
    }
}

__global__ void k_scatter(int64_t rows, int64_t cols, const ezq_outlier* __restrict__ e,
                          int64_t n, float* __restrict__ out, unsigned long long* bad_entry) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ezq_outlier o = e[i];
    if (o.row >= static_cast<uint64_t>(rows) || o.col >= static_cast<uint64_t>(cols)) {
        atomicMin(bad_entry, static_cast<unsigned long long>(i));
        return;
    }
    out[static_cast<int64_t>(o.row) * cols + o.col] = o.value;
}

}  // namespace

void launch_pack(const TDesc* td, const int64_t* pblk_base, int ntens, int64_t total_blocks,
                 Scratch sc, CfgDev cfg, cudaStream_t st) {
    if (total_blocks == 0) return;
    k_pack<<<(unsigned)total_blocks, kPackThreads, 0, st>>>(td, pblk_base, ntens, total_blocks,
                                                            sc, cfg);
    count_launch();
}

void launch_dequant(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                    const float* scales, float* out, unsigned long long* bad_byte,
                    cudaStream_t st) {
    const int64_t n = rows * cols;
    const int64_t blocks = (n + kPackBlock - 1) / kPackBlock;
    if (blocks == 0) return;
    k_dequant<<<(unsigned)blocks, kPackThreads, 0, st>>>(rows, cols, bits, packed, scales, out,
                                                         bad_byte);
    count_launch();
}

void launch_scatter(int64_t rows, int64_t cols, const ezq_outlier* e, int64_t n, float* out,
                    unsigned long long* bad_entry, cudaStream_t st) {
    if (n == 0) return;
    k_scatter<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, cols, e, n, out, bad_entry);
    count_launch();
}

}  // namespace ezq
