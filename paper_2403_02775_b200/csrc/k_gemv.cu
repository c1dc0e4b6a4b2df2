// K6: fused dequant + outlier GEMV / skinny GEMM (the
// reference has no GEMV -- parity is against dequantize_tensor + an fp64
// GEMV, 1e-3 relative).
//
//   y[b, j] = s_j * sum_i x[b,i] * l_ij  +  sum_{(i, j, v) outlier} x[b,i] * v
//
// l_ij is the stored level (outlier slots hold level 0). ezq_gemv_prepare
// repacks the artifact's nibbles once into a K-contiguous word layout:
// T[j][w] (uint32) holds the 8 nibbles of rows 8w..8w+7 of column j, so one
// warp owns whole output columns, every load instruction reads 128
// contiguous bytes, and the K reduction is a register chain plus one warp
// shuffle tree -- no cross-CTA reduction, no workspace, one launch,
// deterministic. The level is produced directly as a float with the 2^23
// magic: float(0x4B000000 | nib) - (2^23 - lmin) = nib + lmin, exact.
// The column's outliers (CSC, rows ascending) are spread over the lanes and
// folded into the same shuffle reduction: the paper's "scatter the outliers
// back" costs 8 bytes per outlier of extra traffic and no extra pass.
//
// HBM-bound: algorithmic bytes = N/2 + 4 cols + 8 n_out + 8 (cols+1)
// + B rows (2|4) + 4 B cols.
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr int kWarps = 8;     // warps per CTA
constexpr int kColsPerWarp = 2;
constexpr int kMaxBatch = 16;
constexpr int kUnroll = 2;    // 16-byte loads per lane in flight per column

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t idx) {
    if (dtype == 1) {
        const unsigned short h = static_cast<const unsigned short*>(x)[idx];
        return __uint_as_float(static_cast<unsigned>(h) << 16);  // bf16
    }
    if (dtype == 2) return __half2float(static_cast<const __half*>(x)[idx]);
    return static_cast<const float*>(x)[idx];
}

// 8 consecutive x values (rows r0..r0+7) of batch row b; vectorised when the
// whole group is in range and aligned.
__device__ __forceinline__ void load_x8(const void* x, int dtype, int64_t rows, int b, int64_t r0,
                                        float (&v)[8]) {
    const int64_t base = static_cast<int64_t>(b) * rows + r0;
    if (r0 + 8 <= rows && (base & 7) == 0) {
        if (dtype == 0) {
            const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + base);
            const float4 a = __ldg(p), c = __ldg(p + 1);
            v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = c.x, v[5] = c.y, v[6] = c.z, v[7] = c.w;
        } else {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const unsigned short*>(x) + base));
            const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (dtype == 1) {
                    v[2 * k] = __uint_as_float(w[k] << 16);
                    v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
                } else {
                    const __half2 h = *reinterpret_cast<const __half2*>(&w[k]);
                    const float2 f = __half22float2(h);
                    v[2 * k] = f.x;
                    v[2 * k + 1] = f.y;
                }
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (r0 + k < rows) ? load_x(x, dtype, base + k) : 0.f;
    }
}

template <int B>
__global__ void __launch_bounds__(kWarps * 32) k_gemv(const unsigned* __restrict__ T, int64_t kw,
                                                      int64_t rows, int64_t cols, float bias,
                                                      const float* __restrict__ scales,
                                                      const int64_t* __restrict__ col_ptr,
                                                      const uint32_t* __restrict__ out_row,
                                                      const float* __restrict__ out_val,
                                                      const void* __restrict__ x, int dtype, int b0,
                                                      float* __restrict__ y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t j0 = (static_cast<int64_t>(blockIdx.x) * kWarps + warp) * kColsPerWarp;
    if (j0 >= cols) return;
    const int nc = static_cast<int>(min(static_cast<int64_t>(kColsPerWarp), cols - j0));
    float acc[kColsPerWarp][B];
#pragma unroll
    for (int c = 0; c < kColsPerWarp; ++c)
#pragma unroll
        for (int b = 0; b < B; ++b) acc[c][b] = 0.f;
    const unsigned* Tc[kColsPerWarp];
#pragma unroll
    for (int c = 0; c < kColsPerWarp; ++c) Tc[c] = T + (j0 + min(c, nc - 1)) * kw;

    // kw is a multiple of 4: lane l reads words 4(l + 32u) .. +3 (one 16-byte
    // load = 32 rows) for u < kUnroll; all loads of a round are in flight
    // before any is consumed.
    for (int64_t q0 = lane; 4 * q0 < kw; q0 += 32 * kUnroll) {
        uint4 wv[kUnroll][kColsPerWarp];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int c = 0; c < kColsPerWarp; ++c) {
                const int64_t q = q0 + 32 * u;
                wv[u][c] = 4 * q < kw ? __ldg(reinterpret_cast<const uint4*>(Tc[c]) + q)
                                      : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t q = q0 + 32 * u;
            if (4 * q >= kw) break;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int64_t r0 = 32 * q + 8 * h;
                if (r0 >= rows) break;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    float xv[8];
                    load_x8(x, dtype, rows, b0 + b, r0, xv);
#pragma unroll
                    for (int c = 0; c < kColsPerWarp; ++c) {
                        const unsigned w = h == 0 ? wv[u][c].x : h == 1 ? wv[u][c].y : h == 2 ? wv[u][c].z : wv[u][c].w;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float l = __uint_as_float(0x4B000000u | ((w >> (4 * e)) & 0xFu)) - bias;
                            acc[c][b] = fmaf(xv[e], l, acc[c][b]);
                        }
                    }
                }
            }
        }
    }
    // outliers of the warp's columns, spread over lanes (unscaled term)
    float oacc[kColsPerWarp][B];
#pragma unroll
    for (int c = 0; c < kColsPerWarp; ++c) {
#pragma unroll
        for (int b = 0; b < B; ++b) oacc[c][b] = 0.f;
        if (col_ptr && c < nc) {
            const int64_t e1 = col_ptr[j0 + c + 1];
            for (int64_t e = col_ptr[j0 + c] + lane; e < e1; e += 32) {
                const int64_t r = out_row[e];
                const float v = out_val[e];
#pragma unroll
                for (int b = 0; b < B; ++b)
                    oacc[c][b] = fmaf(load_x(x, dtype, static_cast<int64_t>(b0 + b) * rows + r), v, oacc[c][b]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < kColsPerWarp; ++c)
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc[c][b] += __shfl_xor_sync(0xffffffffu, acc[c][b], o);
                oacc[c][b] += __shfl_xor_sync(0xffffffffu, oacc[c][b], o);
            }
    if (lane < kColsPerWarp * B) {
        const int c = lane / B, b = lane % B;
        if (c < nc) {
            float a = 0.f, o = 0.f;
#pragma unroll
            for (int cc = 0; cc < kColsPerWarp; ++cc)
#pragma unroll
                for (int bb = 0; bb < B; ++bb)
                    if (cc == c && bb == b) a = acc[cc][bb], o = oacc[cc][bb];
            y[static_cast<int64_t>(b0 + b) * cols + j0 + c] = fmaf(scales[j0 + c], a, o);
        }
    }
}

// Repack: T[j][w] = nibbles of rows 8w..8w+7 of column j (row 8w+e at bits
// 4e); rows beyond the matrix get nibble -lmin (level 0, and x reads 0 there).
// Source addressing is the artifact's flat nibble order (rtn.cpp:136-141), any
// cols parity.
__global__ void k_gemv_repack(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols,
                              int bits, int64_t kw, int lmin, unsigned* __restrict__ T) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= cols * kw) return;
    const int64_t j = i / kw, w = i % kw;
    unsigned word = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t r = 8 * w + e;
        unsigned nib = static_cast<unsigned>(-lmin);
        if (r < rows) {
            const int64_t f = r * cols + j;
            // k = 4: nibbles; k < 4: one offset byte per level (rtn.cpp:143-147), < 16
            nib = bits == 4 ? ((f & 1) ? (packed[f >> 1] >> 4) : (packed[f >> 1] & 15)) : packed[f];
        }
        word |= nib << (4 * e);
    }
    T[i] = word;
}

}  // namespace
}  // namespace ezq

using namespace ezq;

struct ezq_gemv_plan {
    int64_t rows, cols, kw;
    int bits, lmin;
    unsigned* T;          // repacked codes (owned)
    const float* scales;  // device (borrowed from the artifact)
    int64_t* col_ptr;     // CSC of the outliers (owned)
    uint32_t* out_row;
    float* out_val;
    int64_t n_out;
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
    auto* p = new ezq_gemv_plan{};
    p->rows = q->rows;
    p->cols = q->cols;
    p->bits = q->bits;
    p->lmin = -(1 << (q->bits - 1)) + 1;
    p->kw = ((q->rows + 31) / 32) * 4;  // words per column, multiple of 4 (16 B)
    p->scales = q->scales;
    p->n_out = q->n_outliers;
    p->dev = dev;
    // CSC view of the outliers (one-time): D2H the COO, bucket by column
    // (rows stay ascending: the COO is flat-ordered), H2D.
    std::vector<ezq_outlier> coo(q->n_outliers);
    if (q->n_outliers)
        EZQ_CK(cudaMemcpy(coo.data(), q->outliers, sizeof(ezq_outlier) * q->n_outliers,
                          cudaMemcpyDeviceToHost));
    std::vector<int64_t> ptr(q->cols + 1, 0);
    for (const auto& e : coo) {
        if (e.col >= static_cast<uint64_t>(q->cols) || e.row >= static_cast<uint64_t>(q->rows)) {
            delete p;
            return set_error(EZQ_ERR_INVALID_ARGUMENT, "outlier coordinate outside the matrix");
        }
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
    EZQ_CK(cudaMalloc(&p->T, sizeof(unsigned) * q->cols * p->kw));
    EZQ_CK(cudaMalloc(&p->col_ptr, sizeof(int64_t) * (q->cols + 1)));
    EZQ_CK(cudaMalloc(&p->out_row, sizeof(uint32_t) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->out_val, sizeof(float) * std::max<int64_t>(q->n_outliers, 1)));
    const int64_t nw = q->cols * p->kw;
    k_gemv_repack<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, st>>>(q->packed, q->rows, q->cols,
                                                                         q->bits, p->kw, p->lmin, p->T);
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
    if (batch < 1 || batch > kMaxBatch)
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "batch must be in [1, " + std::to_string(kMaxBatch) + "]");
    if (x_dtype < 0 || x_dtype > 2) return set_error(EZQ_ERR_INVALID_ARGUMENT, "bad x dtype");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    const int pt = prof_begin("gemv", st);
    const unsigned grid =
        static_cast<unsigned>((p->cols + kWarps * kColsPerWarp - 1) / (kWarps * kColsPerWarp));
    const float bias = 8388608.0f - static_cast<float>(p->lmin);  // 2^23 - lmin (exact)
    const int64_t* cp = p->n_out ? p->col_ptr : nullptr;
    for (int b0 = 0; b0 < batch;) {
        const int used = std::min(batch - b0, 8);
        switch (used) {
#define EZQ_GEMV_B(BB)                                                                               \
    case BB:                                                                                         \
        k_gemv<BB><<<grid, kWarps * 32, 0, st>>>(p->T, p->kw, p->rows, p->cols, bias, p->scales, cp, \
                                                  p->out_row, p->out_val, x, x_dtype, b0, y);         \
        break;
            EZQ_GEMV_B(1)
            EZQ_GEMV_B(2)
            EZQ_GEMV_B(3)
            EZQ_GEMV_B(4)
            EZQ_GEMV_B(5)
            EZQ_GEMV_B(6)
            EZQ_GEMV_B(7)
            EZQ_GEMV_B(8)
#undef EZQ_GEMV_B
        }
        count_launch();
        b0 += used;
    }
    // Algorithmic bytes of the 4-bit codes the kernel streams (the repacked
    // copy has the same size as the artifact's nibbles).
    const double bytes = static_cast<double>(p->rows * p->cols + 1) / 2 + 4.0 * p->cols +
                         8.0 * p->n_out + 8.0 * (p->cols + 1) +
                         batch * p->rows * (x_dtype == 0 ? 4.0 : 2.0) + 4.0 * batch * p->cols;
    prof_end(pt, st, bytes);
    EZQ_CK(cudaGetLastError());
    return clear_error();
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
