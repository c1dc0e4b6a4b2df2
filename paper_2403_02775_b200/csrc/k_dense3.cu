// Dense 3-bit codes (a B200 extension -- the reference
// stores k = 3 one offset byte per level, rtn.cpp:119-147).
//
// Layout: the level offsets (level - lmin, 0..7) of the flat row-major
// elements as one little-endian bit stream, element e at bits 3e .. 3e + 2
// (eight elements per 3 bytes, 3 * ceil(n / 8) bytes, zero tail bits). The
// stream is position-independent: any 8-element group is 3 whole bytes, so a
// tensor's codes can be cut at multiples of 8 elements.
//
// Kernels (all HBM-bound byte work; one thread per 32 elements = 12 bytes of
// stream = three 4-byte words, so a warp moves 384 contiguous stream bytes):
//   k_pack_dense3    one byte per level (the reference's k = 3 payload) -> stream
//   k_unpack_dense3  stream -> one byte per level
//   k_dequant_dense3 stream + scales -> floats, What = float(double(s_j) * l)
//                    (dequantize_impl, pipeline.cpp:117-142; the outliers are
//                    scattered after it by k_scatter, outliers.cpp:106-114)
// Algorithmic bytes: pack 1 + 3/8 per element, unpack 3/8 + 1, dequant 3/8 +
// 4 (+ 4 per column for the scales).
#include <cstdint>
#include <string>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr int kD3Per = 32;  // elements per thread
constexpr unsigned long long kNoBad = ~0ull;
constexpr int kD3Threads = 256;

// the 12 stream bytes of elements [32 t, 32 t + 32) (fewer at the tail)
template <bool ALIGNED>
__device__ __forceinline__ void load_stream(const uint8_t* in, int64_t t, int nbytes, uint32_t (&w)[3]) {
    if (ALIGNED && nbytes == 12) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(in + 12 * t);
        w[0] = __ldg(p), w[1] = __ldg(p + 1), w[2] = __ldg(p + 2);
        return;
    }
    w[0] = w[1] = w[2] = 0u;
#pragma unroll
    for (int b = 0; b < 12; ++b)
        if (b < nbytes) w[b >> 2] |= static_cast<uint32_t>(in[12 * t + b]) << (8 * (b & 3));
}

__device__ __forceinline__ int field(const uint32_t (&w)[3], int j) {  // j: compile-time after unrolling
    const int p = 3 * j, q = p >> 5, s = p & 31;
    const uint64_t v = (static_cast<uint64_t>(q < 2 ? w[q + 1] : 0u) << 32) | w[q];
    return static_cast<int>((v >> s) & 7u);
}

template <bool ALIGNED>
__global__ void __launch_bounds__(kD3Threads) k_pack_dense3(const uint8_t* __restrict__ off, int64_t n,
                                                            uint8_t* __restrict__ out,
                                                            unsigned long long* __restrict__ bad) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kD3Threads + threadIdx.x;
    const int64_t e0 = t * kD3Per;
    if (e0 >= n) return;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kD3Per), n - e0));
    uint8_t b[kD3Per];
    if (ALIGNED && cnt == kD3Per) {
        const uint4* p = reinterpret_cast<const uint4*>(off + e0);
        const uint4 u0 = __ldg(p), u1 = __ldg(p + 1);
        const uint32_t ws[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int j = 0; j < kD3Per; ++j) b[j] = (ws[j >> 2] >> (8 * (j & 3))) & 0xffu;
    } else {
#pragma unroll
        for (int j = 0; j < kD3Per; ++j) b[j] = j < cnt ? off[e0 + j] : 0;
    }
    uint32_t w[3] = {0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < kD3Per; ++j) {
        if (b[j] > 7) atomicMin(bad, static_cast<unsigned long long>(e0 + j));  // unpack_levels' span check
        const uint64_t v = static_cast<uint64_t>(b[j] & 7u) << ((3 * j) & 31);
        const int q = (3 * j) >> 5;
        w[q] |= static_cast<uint32_t>(v);
        if (q < 2) w[q + 1] |= static_cast<uint32_t>(v >> 32);
    }
    const int nbytes = 3 * ((cnt + 7) >> 3);
    if (ALIGNED && nbytes == 12) {
        uint32_t* p = reinterpret_cast<uint32_t*>(out + 12 * t);
        p[0] = w[0], p[1] = w[1], p[2] = w[2];
    } else {
#pragma unroll
        for (int k = 0; k < 12; ++k)
            if (k < nbytes) out[12 * t + k] = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
    }
}

template <bool ALIGNED>
__global__ void __launch_bounds__(kD3Threads) k_unpack_dense3(const uint8_t* __restrict__ in, int64_t n,
                                                              uint8_t* __restrict__ out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kD3Threads + threadIdx.x;
    const int64_t e0 = t * kD3Per;
    if (e0 >= n) return;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kD3Per), n - e0));
    uint32_t w[3];
    load_stream<ALIGNED>(in, t, 3 * ((cnt + 7) >> 3), w);
    if (ALIGNED && cnt == kD3Per) {
        uint32_t o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            o[k] = field(w, 4 * k) | (field(w, 4 * k + 1) << 8) | (field(w, 4 * k + 2) << 16) |
                   (field(w, 4 * k + 3) << 24);
        uint4* p = reinterpret_cast<uint4*>(out + e0);
        p[0] = make_uint4(o[0], o[1], o[2], o[3]);
        p[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int j = 0; j < kD3Per; ++j)
            if (j < cnt) out[e0 + j] = static_cast<uint8_t>(field(w, j));
    }
}

// Dequant: a CTA's 8192 elements (3072 stream bytes) are staged in shared
// memory by coalesced word loads; then thread t writes elements 4 (t + 256 k)
// .. + 3 (k = 0..7) as one float4 each -- consecutive lanes, consecutive
// 16-byte stores (a whole-thread run of 32 floats per lane would put every
// store instruction of a warp on 32 different lines).
template <bool ALIGNED>
__global__ void __launch_bounds__(kD3Threads) k_dequant_dense3(int64_t rows, int64_t cols, const uint8_t* __restrict__ in,
                                                               const float* __restrict__ scales, int lmin,
                                                               float* __restrict__ out) {
    constexpr int kElems = kD3Per * kD3Threads;   // 8192
    constexpr int kWords = kElems * 3 / 32;       // 768 stream words
    __shared__ uint32_t sw[kWords + 1];
    const int64_t n = rows * cols;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kElems;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kElems), n - b0));
    const int nbytes = 3 * ((cnt + 7) >> 3);
    const uint8_t* src = in + b0 / 8 * 3;
    if (ALIGNED && nbytes == kWords * 4) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(src);
        for (int w = threadIdx.x; w < kWords; w += kD3Threads) sw[w] = __ldg(p + w);
    } else {
        for (int w = threadIdx.x; w < kWords; w += kD3Threads) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (4 * w + b < nbytes) v |= static_cast<uint32_t>(src[4 * w + b]) << (8 * b);
            sw[w] = v;
        }
    }
    if (threadIdx.x == 0) sw[kWords] = 0u;
    __syncthreads();
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (b0 & 3) == 0;
#pragma unroll 2
    for (int k = 0; k < kD3Per / 4; ++k) {
        const int l = 4 * (threadIdx.x + kD3Threads * k);  // local element of the quad
        if (l >= cnt) break;
        const int p = 3 * l, q = p >> 5, sh = p & 31;       // 12 bits at stream bit p
        const uint32_t f = static_cast<uint32_t>(((static_cast<uint64_t>(sw[q + 1]) << 32) | sw[q]) >> sh);
        // 32-bit modulo when the tensor has < 2^32 elements (a 64-bit IMOD per quad costs more than the quad)
        int64_t col = n < (int64_t(1) << 32) ? static_cast<int64_t>(static_cast<uint32_t>((b0 + l)) % static_cast<uint32_t>(cols))
                                             : (b0 + l) % cols;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // float(double(s) * l) == RN32(s * l): the fp64 product is exact
            v[j] = __fmul_rn(__ldg(scales + col), static_cast<float>(lmin + static_cast<int>((f >> (3 * j)) & 7u)));
            if (++col == cols) col = 0;
        }
        float* o = out + b0 + l;
        if (vec && l + 4 <= cnt) {
            *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (l + j < cnt) o[j] = v[j];
        }
    }
}

inline unsigned d3_blocks(int64_t n) {
    return static_cast<unsigned>((n + static_cast<int64_t>(kD3Per) * kD3Threads - 1) / (static_cast<int64_t>(kD3Per) * kD3Threads));
}

bool al4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) == 0; }
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Host/device staging shared by the entry points: `in` (in_bytes) and `out`
// (out_bytes) in `mem`; returns device pointers valid on `st`.
struct Staged {
    Arena ar;
    const uint8_t* din = nullptr;
    uint8_t* dout = nullptr;
    unsigned long long* bad = nullptr;
};

int stage_io(Staged& s, const uint8_t* in, size_t in_bytes, uint8_t* out, size_t out_bytes, int mem,
             cudaStream_t st) {
    s.ar.reserve(sizeof(unsigned long long));
    if (mem == EZQ_MEM_HOST) {
        s.ar.reserve(in_bytes);
        s.ar.reserve(out_bytes);
    }
    if (int r = s.ar.allocate(st)) return r;
    s.bad = s.ar.take<unsigned long long>(1);
    if (mem == EZQ_MEM_HOST) {
        uint8_t* a = s.ar.take<uint8_t>(in_bytes);
        s.dout = s.ar.take<uint8_t>(out_bytes);
        if (in_bytes) EZQ_CK(cudaMemcpyAsync(a, in, in_bytes, cudaMemcpyHostToDevice, st));
        s.din = a;
    } else {
        s.din = in;
        s.dout = out;
    }
    EZQ_CK(cudaMemsetAsync(s.bad, 0xff, sizeof(unsigned long long), st));
    return EZQ_OK;
}

}  // namespace
}  // namespace ezq

using namespace ezq;

extern "C" {

int64_t ezq_dense3_size(int64_t count) { return count <= 0 ? 0 : 3 * ((count + 7) / 8); }

int ezq_pack_dense3(const uint8_t* levels, int64_t count, uint8_t* out, int mem, void* stream) {
    if (count < 0) return set_error(EZQ_ERR_INVALID_ARGUMENT, "negative level count");
    if (mem != EZQ_MEM_HOST && mem != EZQ_MEM_DEVICE) return set_error(EZQ_ERR_INVALID_ARGUMENT, "unknown memory kind");
    if (count == 0) return clear_error();
    if (!levels || !out) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null buffer");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    const size_t ob = static_cast<size_t>(ezq_dense3_size(count));
    Staged s;
    if (int r = stage_io(s, levels, static_cast<size_t>(count), out, ob, mem, st)) return r;
    const int pd = prof_begin("dense3", st);
    if (al16(s.din) && al4(s.dout))
        k_pack_dense3<true><<<d3_blocks(count), kD3Threads, 0, st>>>(s.din, count, s.dout, s.bad);
    else
        k_pack_dense3<false><<<d3_blocks(count), kD3Threads, 0, st>>>(s.din, count, s.dout, s.bad);
    count_launch();
    prof_end(pd, st, static_cast<double>(count) + static_cast<double>(ob));
    EZQ_CK(cudaGetLastError());
    unsigned long long hb;
    EZQ_CK(cudaMemcpyAsync(&hb, s.bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    if (hb != kNoBad) {
        uint8_t byte = 0;
        EZQ_CK(cudaMemcpy(&byte, s.din + hb, 1, cudaMemcpyDeviceToHost));
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "packed byte " + std::to_string(byte) + " exceeds level span 7", static_cast<int64_t>(hb));
    }
    if (mem == EZQ_MEM_HOST) {
        EZQ_CK(cudaMemcpyAsync(out, s.dout, ob, cudaMemcpyDeviceToHost, st));
        EZQ_CK(cudaStreamSynchronize(st));
    }
    return clear_error();
}

int ezq_unpack_dense3(const uint8_t* dense, int64_t count, uint8_t* out, int mem, void* stream) {
    if (count < 0) return set_error(EZQ_ERR_INVALID_ARGUMENT, "negative level count");
    if (mem != EZQ_MEM_HOST && mem != EZQ_MEM_DEVICE) return set_error(EZQ_ERR_INVALID_ARGUMENT, "unknown memory kind");
    if (count == 0) return clear_error();
    if (!dense || !out) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null buffer");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    const size_t ib = static_cast<size_t>(ezq_dense3_size(count));
    Staged s;
    if (int r = stage_io(s, dense, ib, out, static_cast<size_t>(count), mem, st)) return r;
    const int pd = prof_begin("dense3", st);
    if (al4(s.din) && al16(s.dout))
        k_unpack_dense3<true><<<d3_blocks(count), kD3Threads, 0, st>>>(s.din, count, s.dout);
    else
        k_unpack_dense3<false><<<d3_blocks(count), kD3Threads, 0, st>>>(s.din, count, s.dout);
    count_launch();
    prof_end(pd, st, static_cast<double>(ib) + static_cast<double>(count));
    EZQ_CK(cudaGetLastError());
    if (mem == EZQ_MEM_HOST) EZQ_CK(cudaMemcpyAsync(out, s.dout, static_cast<size_t>(count), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    return clear_error();
}

int ezq_dequantize_dense3(const ezq_qweight* q, const uint8_t* dense, float* out, int out_mem, void* stream) {
    if (q->rows <= 0 || q->cols <= 0) return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    if (q->bits != 3) return set_error(EZQ_ERR_INVALID_ARGUMENT, "dense 3-bit codes need a 3-bit artifact");
    if (q->reserved) return set_error(EZQ_ERR_IO_FORMAT, "scale count does not match columns");
    if (!dense || !out || !q->scales) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null buffer");
    const int64_t N = q->rows * q->cols;
    const size_t db = static_cast<size_t>(ezq_dense3_size(N));
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    Arena ar;
    ar.reserve(sizeof(unsigned long long));
    const bool hin = q->mem == EZQ_MEM_HOST;
    if (hin) {
        ar.reserve(db);
        ar.reserve(sizeof(float) * q->cols);
        ar.reserve(sizeof(ezq_outlier) * q->n_outliers);
    }
    if (out_mem == EZQ_MEM_HOST) ar.reserve(sizeof(float) * N);
    if (int s = ar.allocate(st)) return s;
    unsigned long long* d_bad = ar.take<unsigned long long>(1);
    const uint8_t* pk = dense;
    const float* sc = q->scales;
    const ezq_outlier* oe = q->outliers;
    if (hin) {
        uint8_t* a = ar.take<uint8_t>(db);
        float* b = ar.take<float>(q->cols);
        ezq_outlier* c = ar.take<ezq_outlier>(q->n_outliers);
        EZQ_CK(cudaMemcpyAsync(a, dense, db, cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(b, q->scales, sizeof(float) * q->cols, cudaMemcpyHostToDevice, st));
        if (q->n_outliers)
            EZQ_CK(cudaMemcpyAsync(c, q->outliers, sizeof(ezq_outlier) * q->n_outliers, cudaMemcpyHostToDevice, st));
        pk = a, sc = b, oe = c;
    }
    float* dst = out_mem == EZQ_MEM_HOST ? ar.take<float>(N) : out;
    EZQ_CK(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), st));
    const int pd = prof_begin("dense3", st);
    if (al4(pk))
        k_dequant_dense3<true><<<d3_blocks(N), kD3Threads, 0, st>>>(q->rows, q->cols, pk, sc, -3, dst);
    else
        k_dequant_dense3<false><<<d3_blocks(N), kD3Threads, 0, st>>>(q->rows, q->cols, pk, sc, -3, dst);
    count_launch();
    launch_scatter(q->rows, q->cols, oe, q->n_outliers, dst, d_bad, st);
    prof_end(pd, st, static_cast<double>(db) + 4.0 * q->cols + 4.0 * N + 16.0 * q->n_outliers);
    EZQ_CK(cudaGetLastError());
    unsigned long long hb;
    EZQ_CK(cudaMemcpyAsync(&hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    if (hb != kNoBad) {
        ezq_outlier e;
        EZQ_CK(cudaMemcpy(&e, oe + hb, sizeof(e), cudaMemcpyDeviceToHost));
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "outlier coordinate (" + std::to_string(e.row) + ", " + std::to_string(e.col) + ") outside " +
                             std::to_string(q->rows) + "x" + std::to_string(q->cols),
                         static_cast<int64_t>(hb));
    }
    if (out_mem == EZQ_MEM_HOST) {
        EZQ_CK(cudaMemcpyAsync(out, dst, sizeof(float) * N, cudaMemcpyDeviceToHost, st));
        EZQ_CK(cudaStreamSynchronize(st));
    }
    return clear_error();
}

int ezq_gemv_prepare_dense3(const ezq_qweight* q, const uint8_t* dense, int outlier_dtype, void* stream,
                            ezq_gemv_plan** plan) {
    *plan = nullptr;
    if (q->mem != EZQ_MEM_DEVICE) return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv needs a device-resident artifact");
    if (q->bits != 3) return set_error(EZQ_ERR_INVALID_ARGUMENT, "dense 3-bit codes need a 3-bit artifact");
    if (q->rows <= 0 || q->cols <= 0) return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    if (!dense) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null buffer");
    const int64_t N = q->rows * q->cols;
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    // the plan's fragment repack reads one byte per level: unpack into a
    // transient buffer (prepare-time only; the plan keeps its own layout)
    uint8_t* tmp = nullptr;
    EZQ_CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), static_cast<size_t>(N), st));
    int r = ezq_unpack_dense3(dense, N, tmp, EZQ_MEM_DEVICE, st);
    if (r == EZQ_OK) {
        ezq_qweight v = *q;
        v.packed = tmp;
        v.packed_bytes = N;
        r = ezq_gemv_prepare_ex(&v, outlier_dtype, st, plan);
    }
    cudaStreamSynchronize(st);
    cudaFreeAsync(tmp, st);
    return r;
}

}  // extern "C"
