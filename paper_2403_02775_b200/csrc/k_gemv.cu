// K6: fused dequant + outlier GEMV / skinny GEMM (the
// reference has no GEMV -- parity is against dequantize_tensor + an fp64
// GEMV, 1e-3 relative).
//
//   y[b, j] = s_j * ( sum_i x[b,i] * nib_ij  +  lmin * sum_i x[b,i] )
//           + sum_{(i, j, v) outlier} x[b,i] * v
//
// with nib_ij = l_ij - lmin the stored 4-bit offset (outlier slots hold level
// 0, so they add nothing to the first sum). The packed artifact is used as
// is: row-major [in = rows, out = cols] nibbles, so consecutive threads own
// consecutive columns and every warp load is a contiguous 512-byte row
// segment. HBM-bound: bytes = N/2 + 4 cols + 8 n_out + 4 (cols+1) + B rows
// (2|4) + 4 B cols.
//
// k_gemv_main: CTA = 128 threads x 32 columns (one 16-byte nibble word per
// thread per row), K split in chunks of `kc` rows; x chunk staged in SMEM;
// per-split partial sums go to a workspace (deterministic, no atomics).
// k_gemv_finish: sums the splits in fixed order, applies the scale, the lmin
// term and the column's outliers (CSC, rows ascending).
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr int kGT = 128;       // threads per CTA
constexpr int kGCols = 32;     // columns per thread (16 bytes of nibbles)
constexpr int kGTile = kGT * kGCols;
constexpr int kMaxBatch = 16;

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t idx) {
    if (dtype == 1) {
        const unsigned short h = static_cast<const unsigned short*>(x)[idx];
        return __uint_as_float(static_cast<unsigned>(h) << 16);  // bf16
    }
    if (dtype == 2) return __half2float(static_cast<const __half*>(x)[idx]);
    return static_cast<const float*>(x)[idx];
}

// nibble -> float via the 2^23 magic (exact): float(0x4B000000 | n) - 2^23.
__device__ __forceinline__ float nib_f(unsigned w, int shift) {
    return __uint_as_float(0x4B000000u | ((w >> shift) & 0xFu)) - 8388608.0f;
}

template <int B>
__global__ void __launch_bounds__(kGT) k_gemv_main(const uint8_t* __restrict__ packed,
                                                    int64_t rows, int64_t cols,
                                                    const void* __restrict__ x, int dtype, int b0,
                                                    int kc, float* __restrict__ part) {
    extern __shared__ float xs[];  // [kc][B]
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kc;
    const int nr = static_cast<int>(min(static_cast<int64_t>(kc), rows - r0));
    for (int i = threadIdx.x; i < nr * B; i += kGT) {
        const int r = i / B, b = i % B;
        xs[i] = load_x(x, dtype, static_cast<int64_t>(b0 + b) * rows + r0 + r);
    }
    __syncthreads();
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kGTile + threadIdx.x * kGCols;
    if (c0 >= cols) return;
    float acc[B][kGCols];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int c = 0; c < kGCols; ++c) acc[b][c] = 0.f;
    const uint8_t* base = packed + (r0 * cols + c0) / 2;
    const int64_t stride = cols / 2;
    int r = 0;
#pragma unroll 4
    for (; r < nr; ++r) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(base + r * stride));
        const unsigned ws[4] = {w.x, w.y, w.z, w.w};
        float xv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) xv[b] = xs[r * B + b];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float f = nib_f(ws[q], 4 * k);
#pragma unroll
                for (int b = 0; b < B; ++b) acc[b][q * 8 + k] = fmaf(xv[b], f, acc[b][q * 8 + k]);
            }
    }
    float* dst = part + (static_cast<int64_t>(blockIdx.y) * B) * cols + c0;
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int c = 0; c < kGCols; c += 4)
            *reinterpret_cast<float4*>(dst + static_cast<int64_t>(b) * cols + c) =
                make_float4(acc[b][c], acc[b][c + 1], acc[b][c + 2], acc[b][c + 3]);
}

// Generic path (any cols / alignment): one thread per column, flat nibble
// addressing exactly like unpack_levels (rtn.cpp:166-171).
__global__ void __launch_bounds__(256) k_gemv_generic(const uint8_t* __restrict__ packed,
                                                      int64_t rows, int64_t cols, int bits,
                                                      const void* __restrict__ x, int dtype,
                                                      int batch, int kc, float* __restrict__ part) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kc;
    const int64_t r1 = min(rows, r0 + kc);
    float acc[kMaxBatch];
    for (int b = 0; b < batch; ++b) acc[b] = 0.f;
    for (int64_t r = r0; r < r1; ++r) {
        const int64_t f = r * cols + j;
        const int nib = bits == 4 ? ((f & 1) ? (packed[f >> 1] >> 4) : (packed[f >> 1] & 15))
                                  : packed[f];
        for (int b = 0; b < batch; ++b)
            acc[b] = fmaf(load_x(x, dtype, static_cast<int64_t>(b) * rows + r),
                          static_cast<float>(nib), acc[b]);
    }
    for (int b = 0; b < batch; ++b) {
        const int g = b / 4, bb = b % 4, bg = min(4, batch - 4 * g);
        part[static_cast<int64_t>(g) * gridDim.y * 4 * cols +
             (static_cast<int64_t>(blockIdx.y) * bg + bb) * cols + j] = acc[b];
    }
}

__global__ void __launch_bounds__(256) k_gemv_finish(const float* __restrict__ part, int splits,
                                                     int64_t rows, int64_t cols, int batch,
                                                     int lmin, const float* __restrict__ scales,
                                                     const int64_t* __restrict__ col_ptr,
                                                     const uint32_t* __restrict__ out_row,
                                                     const float* __restrict__ out_val,
                                                     const void* __restrict__ x, int dtype,
                                                     const float* __restrict__ xsum,
                                                     float* __restrict__ y) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (j >= cols) return;
    // Partials of batch row b live in group g = b / 4 (width bg), laid out
    // [group][split][bg][cols] with a fixed group stride of splits*4*cols.
    const int g = b / 4, bb = b % 4, bg = min(4, batch - 4 * g);
    const float* pg = part + static_cast<int64_t>(g) * splits * 4 * cols;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += pg[(static_cast<int64_t>(k) * bg + bb) * cols + j];
    float v = scales[j] * fmaf(static_cast<float>(lmin), xsum[b], s);
    if (col_ptr) {
        for (int64_t e = col_ptr[j]; e < col_ptr[j + 1]; ++e)
            v = fmaf(load_x(x, dtype, static_cast<int64_t>(b) * rows + out_row[e]), out_val[e], v);
    }
    y[static_cast<int64_t>(b) * cols + j] = v;
}

// sum_i x[b, i] per batch row (fixed-order block reduction).
__global__ void __launch_bounds__(256) k_xsum(const void* __restrict__ x, int dtype, int64_t rows,
                                              float* __restrict__ xsum) {
    const int b = blockIdx.x;
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
        s += load_x(x, dtype, static_cast<int64_t>(b) * rows + i);
    __shared__ float red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) xsum[b] = red[0];
}

}  // namespace
}  // namespace ezq

using namespace ezq;

struct ezq_gemv_plan {
    int64_t rows, cols;
    int bits, lmin;
    const uint8_t* packed;  // device (borrowed from the artifact)
    const float* scales;    // device (borrowed)
    int64_t* col_ptr;       // CSC of the outliers (owned)
    uint32_t* out_row;
    float* out_val;
    int64_t n_out;
    int kc, splits;
    bool fast;
    float* part;  // [splits][kMaxBatch][cols]
    float* xsum;  // [kMaxBatch]
    int dev;
};

extern "C" {

int ezq_gemv_prepare(const ezq_qweight* q, void* stream, ezq_gemv_plan** plan) {
    *plan = nullptr;
    if (q->mem != EZQ_MEM_DEVICE)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv needs a device-resident artifact");
    if (q->rows <= 0 || q->cols <= 0)
        return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    auto* p = new ezq_gemv_plan{};
    p->rows = q->rows;
    p->cols = q->cols;
    p->bits = q->bits;
    p->lmin = -(1 << (q->bits - 1)) + 1;
    p->packed = q->packed;
    p->scales = q->scales;
    p->n_out = q->n_outliers;
    p->dev = dev;
    p->fast = q->bits == 4 && q->cols % 8 == 0 && (reinterpret_cast<uintptr_t>(q->packed) & 15) == 0 &&
              (q->cols / 2) % 16 == 0;
    // K split: enough CTAs for ~4 waves of 148 SMs, >= 64 rows per split.
    const int64_t col_tiles = p->fast ? (q->cols + kGTile - 1) / kGTile : (q->cols + 255) / 256;
    const DeviceInfo& di = device_info(dev);
    int64_t want = std::max<int64_t>(1, (4 * di.sms + col_tiles - 1) / col_tiles);
    int64_t kc = std::max<int64_t>(64, (q->rows + want - 1) / want);
    kc = ((kc + 7) / 8) * 8;
    p->kc = static_cast<int>(kc);
    p->splits = static_cast<int>((q->rows + kc - 1) / kc);
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
    EZQ_CK(cudaMalloc(&p->col_ptr, sizeof(int64_t) * (q->cols + 1)));
    EZQ_CK(cudaMalloc(&p->out_row, sizeof(uint32_t) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->out_val, sizeof(float) * std::max<int64_t>(q->n_outliers, 1)));
    EZQ_CK(cudaMalloc(&p->part, sizeof(float) * p->splits * kMaxBatch * q->cols));
    EZQ_CK(cudaMalloc(&p->xsum, sizeof(float) * kMaxBatch));
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
    k_xsum<<<batch, 256, 0, st>>>(x, x_dtype, p->rows, p->xsum);
    const dim3 grid_main(static_cast<unsigned>(p->fast ? (p->cols + kGTile - 1) / kGTile
                                                       : (p->cols + 255) / 256),
                         static_cast<unsigned>(p->splits));
    if (p->fast) {
        // Batch rows in groups of up to 4 (register-resident accumulators).
        for (int g = 0; 4 * g < batch; ++g) {
            const int bg = std::min(4, batch - 4 * g);
            const size_t smem = sizeof(float) * p->kc * bg;
            float* pg = p->part + static_cast<int64_t>(g) * p->splits * 4 * p->cols;
            switch (bg) {
                case 1: k_gemv_main<1><<<grid_main, kGT, smem, st>>>(p->packed, p->rows, p->cols, x, x_dtype, 4 * g, p->kc, pg); break;
                case 2: k_gemv_main<2><<<grid_main, kGT, smem, st>>>(p->packed, p->rows, p->cols, x, x_dtype, 4 * g, p->kc, pg); break;
                case 3: k_gemv_main<3><<<grid_main, kGT, smem, st>>>(p->packed, p->rows, p->cols, x, x_dtype, 4 * g, p->kc, pg); break;
                default: k_gemv_main<4><<<grid_main, kGT, smem, st>>>(p->packed, p->rows, p->cols, x, x_dtype, 4 * g, p->kc, pg); break;
            }
        }
    } else {
        k_gemv_generic<<<grid_main, 256, 0, st>>>(p->packed, p->rows, p->cols, p->bits, x, x_dtype,
                                                  batch, p->kc, p->part);
    }
    const dim3 grid_fin(static_cast<unsigned>((p->cols + 255) / 256), static_cast<unsigned>(batch));
    k_gemv_finish<<<grid_fin, 256, 0, st>>>(p->part, p->splits, p->rows, p->cols, batch, p->lmin,
                                            p->scales, p->n_out ? p->col_ptr : nullptr, p->out_row,
                                            p->out_val, x, x_dtype, p->xsum, y);
    const double bytes = static_cast<double>(p->bits == 4 ? (p->rows * p->cols + 1) / 2
                                                          : p->rows * p->cols) +
                         4.0 * p->cols + 8.0 * p->n_out + 8.0 * (p->cols + 1) +
                         batch * p->rows * (x_dtype == 0 ? 4.0 : 2.0) + 4.0 * batch * p->cols;
    prof_end(pt, st, bytes);
    count_launch(2 + (p->fast ? (batch + 3) / 4 : 1));
    EZQ_CK(cudaGetLastError());
    return clear_error();
}

void ezq_gemv_plan_free(ezq_gemv_plan* p) {
    if (!p) return;
    cudaFree(p->col_ptr);
    cudaFree(p->out_row);
    cudaFree(p->out_val);
    cudaFree(p->part);
    cudaFree(p->xsum);
    delete p;
}

}  // extern "C"
