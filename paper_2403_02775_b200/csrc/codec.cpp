// .ezqt container codec (reference io.hpp:48-66,
// io.cpp:221-354). Host byte work behind the C-ABI: the artifact of
// ezq_quantize_* (once copied to host) encodes to exactly the bytes the
// reference writes, and decoding applies the reference's validation with the
// same error categories and byte offsets (EZQ_ERR_IO_* + ezq_last_error's
// index = offset). Layout, little-endian:
//   "EZQT" | version u32 = 1 | k u8 | pad u8[3] | sigma_n f32 | mean f64 |
//   std f64 | rows u64 | cols u64 | scales cols x f32 | count u64 |
//   outliers count x (row u32, col u32, value f32) | packed levels
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "runtime.hpp"

namespace ezq {
namespace {

constexpr char kEzqtMagic[4] = {'E', 'Z', 'Q', 'T'};
constexpr uint32_t kEzqtVersion = 1;
constexpr int64_t kHeaderBytes = 48;

struct Writer {
    uint8_t* p;
    void bytes(const void* src, size_t n) {
        std::memcpy(p, src, n);
        p += n;
    }
    void u8(uint8_t v) { *p++ = v; }
    void u32(uint32_t v) {
        for (int i = 0; i < 4; ++i) *p++ = static_cast<uint8_t>(v >> (8 * i));
    }
    void u64(uint64_t v) {
        for (int i = 0; i < 8; ++i) *p++ = static_cast<uint8_t>(v >> (8 * i));
    }
    void f32(float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u32(u);
    }
    void f64(double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
};

// Bounds-checked reader; a failure records the offset of the missing datum.
struct Reader {
    const uint8_t* b;
    int64_t len;
    int64_t pos = 0;
    bool need(int64_t n, const char* what, int* status) {
        if (pos + n > len) {
            *status = set_error(EZQ_ERR_IO_FORMAT, std::string("file truncated in ") + what, pos);
            return false;
        }
        return true;
    }
    uint32_t u32() {
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(b[pos + i]) << (8 * i);
        pos += 4;
        return v;
    }
    uint64_t u64() {
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[pos + i]) << (8 * i);
        pos += 8;
        return v;
    }
    float f32() {
        const uint32_t u = u32();
        float v;
        std::memcpy(&v, &u, 4);
        return v;
    }
    double f64() {
        const uint64_t u = u64();
        double v;
        std::memcpy(&v, &u, 8);
        return v;
    }
};

}  // namespace
}  // namespace ezq

using namespace ezq;

extern "C" {

int ezq_encode_quantized(const ezq_qweight* q, uint8_t** out, int64_t* out_len) {
    *out = nullptr;
    *out_len = 0;
    if (q->mem != EZQ_MEM_HOST)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "encode needs a host artifact (ezq_qweight_to_host)");
    // io.cpp:222-232, in order
    if (q->rows <= 0 || q->cols <= 0) return set_error(EZQ_ERR_INVALID_ARGUMENT, "cannot encode empty tensor shape");
    if (q->rows > UINT32_MAX || q->cols > UINT32_MAX)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "tensor dimensions exceed the 32-bit coordinate range");
    if (q->bits < 2 || q->bits > 8)
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "bit width " + std::to_string(q->bits) + " outside [2, 8]");
    if (q->reserved != 0)  // ezq_qweight_wrap flags n_scales != cols here
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "scale count does not match column count");
    if (q->packed_bytes != ezq_packed_size(q->rows * q->cols, q->bits))
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "packed level payload has the wrong length");
    for (int64_t j = 0; j < q->cols; ++j) {
        const float s = q->scales[j];
        if (!(s > 0.0f) || !std::isfinite(s))
            return set_error(EZQ_ERR_INVALID_ARGUMENT, "scales must be positive and finite");
    }
    for (int64_t i = 0; i < q->n_outliers; ++i) {
        const ezq_outlier& e = q->outliers[i];
        if (e.row >= static_cast<uint64_t>(q->rows) || e.col >= static_cast<uint64_t>(q->cols))
            return set_error(EZQ_ERR_INVALID_ARGUMENT, "outlier coordinate out of range");
        if (i > 0) {
            const ezq_outlier& p = q->outliers[i - 1];
            if (!(p.row < e.row || (p.row == e.row && p.col < e.col)))
                return set_error(EZQ_ERR_INVALID_ARGUMENT, "outliers must be strictly sorted by (row, col)");
        }
    }
    const int64_t len = kHeaderBytes + 4 * q->cols + 8 + 12 * q->n_outliers + q->packed_bytes;
    uint8_t* buf = static_cast<uint8_t*>(std::malloc(static_cast<size_t>(len)));
    if (!buf) return set_error(EZQ_ERR_OOM, "out of host memory encoding a quantized tensor");
    Writer w{buf};
    w.bytes(kEzqtMagic, 4);
    w.u32(kEzqtVersion);
    w.u8(static_cast<uint8_t>(q->bits));
    w.u8(0);
    w.u8(0);
    w.u8(0);
    w.f32(q->sigma_n);
    w.f64(q->mean);
    w.f64(q->stddev);
    w.u64(static_cast<uint64_t>(q->rows));
    w.u64(static_cast<uint64_t>(q->cols));
    for (int64_t j = 0; j < q->cols; ++j) w.f32(q->scales[j]);
    w.u64(static_cast<uint64_t>(q->n_outliers));
    for (int64_t i = 0; i < q->n_outliers; ++i) {
        w.u32(q->outliers[i].row);
        w.u32(q->outliers[i].col);
        w.f32(q->outliers[i].value);
    }
    if (q->packed_bytes) w.bytes(q->packed, static_cast<size_t>(q->packed_bytes));
    *out = buf;
    *out_len = len;
    return clear_error();
}

int ezq_decode_quantized(const uint8_t* bytes, int64_t len, ezq_qweight** out) {
    *out = nullptr;
    int status = EZQ_OK;
    Reader c{bytes, len};
    if (!c.need(4, "magic", &status)) return status;
    if (std::memcmp(bytes, kEzqtMagic, 4) != 0)
        return set_error(EZQ_ERR_IO_FORMAT, "bad magic, not a quantized tensor file", 0);
    c.pos = 4;
    if (!c.need(4, "version", &status)) return status;
    const uint32_t version = c.u32();
    if (version != kEzqtVersion)
        return set_error(EZQ_ERR_IO_VERSION,
                         "file version " + std::to_string(version) + ", reader supports 1", 4);
    const int64_t bits_off = c.pos;
    if (!c.need(1, "bits", &status)) return status;
    const int bits = c.b[c.pos++];
    if (bits < 2 || bits > 8)
        return set_error(EZQ_ERR_IO_FORMAT, "bit width " + std::to_string(bits) + " outside [2, 8]",
                         bits_off);
    for (int i = 0; i < 3; ++i) {
        if (!c.need(1, "padding", &status)) return status;
        ++c.pos;
    }
    if (!c.need(4, "sigma_n", &status)) return status;
    const float sigma_n = c.f32();
    if (!c.need(8, "mean", &status)) return status;
    const double mean = c.f64();
    if (!c.need(8, "std", &status)) return status;
    const double stddev = c.f64();
    const int64_t shape_off = c.pos;
    if (!c.need(8, "rows", &status)) return status;
    const uint64_t rows = c.u64();
    if (!c.need(8, "cols", &status)) return status;
    const uint64_t cols = c.u64();
    if (rows == 0 || cols == 0 || rows > UINT32_MAX || cols > UINT32_MAX)
        return set_error(EZQ_ERR_IO_FORMAT,
                         "shape " + std::to_string(rows) + "x" + std::to_string(cols) +
                             " outside the supported range",
                         shape_off);
    // Field-by-field like the reference's Cursor, so a truncation or a bad
    // value reports the same offset; nothing is allocated until the whole
    // buffer has been validated.
    const int64_t scales_off = c.pos;
    for (uint64_t j = 0; j < cols; ++j) {
        const int64_t off = c.pos;
        if (!c.need(4, "scales", &status)) return status;
        const float s = c.f32();
        if (!(s > 0.0f) || !std::isfinite(s))
            return set_error(EZQ_ERR_IO_FORMAT,
                             "scale " + std::to_string(j) + " is not positive and finite", off);
    }
    if (!c.need(8, "outlier count", &status)) return status;
    const uint64_t count = c.u64();
    if (count > rows * cols)
        return set_error(EZQ_ERR_IO_FORMAT, "outlier count exceeds element count", c.pos - 8);
    const int64_t outl_off = c.pos;
    uint32_t pr = 0, pc = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const int64_t off = c.pos;
        if (!c.need(4, "outliers", &status)) return status;
        const uint32_t r = c.u32();
        if (!c.need(4, "outliers", &status)) return status;
        const uint32_t col = c.u32();
        if (!c.need(4, "outliers", &status)) return status;
        c.pos += 4;
        if (r >= rows || col >= cols)
            return set_error(EZQ_ERR_IO_FORMAT, "outlier coordinate out of range", off);
        if (i > 0 && !(pr < r || (pr == r && pc < col)))
            return set_error(EZQ_ERR_IO_FORMAT, "outliers not strictly sorted by (row, col)", off);
        pr = r;
        pc = col;
    }
    const int64_t packed = ezq_packed_size(static_cast<int64_t>(rows * cols), bits);
    if (!c.need(packed, "packed levels", &status)) return status;
    const int64_t packed_off = c.pos;
    c.pos += packed;
    if (c.pos != len) return set_error(EZQ_ERR_IO_FORMAT, "trailing bytes after packed levels", c.pos);
    if (bits != 4) {
        // wider codes must stay inside the level span (unpack_levels, rtn.cpp:170-178)
        const int span = (1 << (bits - 1)) - (-(1 << (bits - 1)) + 1);
        for (int64_t i = 0; i < packed; ++i)
            if (bytes[packed_off + i] > span)
                return set_error(EZQ_ERR_INVALID_ARGUMENT,
                                 "packed byte " + std::to_string(bytes[packed_off + i]) +
                                     " exceeds level span " + std::to_string(span),
                                 i);
    }
    ezq_qweight* q = static_cast<ezq_qweight*>(std::calloc(1, sizeof(ezq_qweight)));
    q->rows = static_cast<int64_t>(rows);
    q->cols = static_cast<int64_t>(cols);
    q->bits = bits;
    q->mem = EZQ_MEM_HOST;
    q->owned = 1;
    q->packed_bytes = packed;
    q->packed = static_cast<uint8_t*>(host_alloc(static_cast<size_t>(std::max<int64_t>(packed, 1))));
    q->scales = static_cast<float*>(host_alloc(sizeof(float) * cols));
    q->n_outliers = static_cast<int64_t>(count);
    q->outliers = count ? static_cast<ezq_outlier*>(host_alloc(sizeof(ezq_outlier) * count)) : nullptr;
    if (!q->packed || !q->scales || (count && !q->outliers)) {
        ezq_qweight_free(q);
        return set_error(EZQ_ERR_OOM, "out of host memory decoding a quantized tensor");
    }
    std::memcpy(q->scales, bytes + scales_off, sizeof(float) * cols);  // little-endian host
    for (uint64_t i = 0; i < count; ++i) {
        const uint8_t* e = bytes + outl_off + 12 * i;
        std::memcpy(&q->outliers[i].row, e, 4);
        std::memcpy(&q->outliers[i].col, e + 4, 4);
        std::memcpy(&q->outliers[i].value, e + 8, 4);
    }
    std::memcpy(q->packed, bytes + packed_off, static_cast<size_t>(packed));
    q->mean = mean;
    q->stddev = stddev;
    q->sigma_n = sigma_n;
    q->has_errors = 0;  // rtn_error / final_error are not part of the file
    *out = q;
    return clear_error();
}

}  // extern "C"
