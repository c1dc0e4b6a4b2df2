// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (EasyQuant `ezquant`,
// /root/reference/proj), compiled out-of-tree from the reference's own
// sources by oracle/Makefile into oracle/_ref/libezq_ref.so. The namespace is
// renamed to `ezq_ref` at compile time (-Dezquant=ezq_ref) so the reference can
// share a process with the B200 drop-in without symbol clashes.
//
// Used by: tests/ (to pin the C restatement in oracle/ezq_oracle.c and to
// generate tests/golden/ fixtures) and bench.py --impl reference (the
// reference's own CPU implementation timed on the box's host cores).
#include <cstdint>
#include <cstring>
#include <set>
#include <span>
#include <string>
#include <vector>

#include "ezquant/error.hpp"
#include "ezquant/io.hpp"
#include "ezquant/model.hpp"
#include "ezquant/report.hpp"
#include "ezquant/optimize.hpp"
#include "ezquant/outliers.hpp"
#include "ezquant/pipeline.hpp"
#include "ezquant/rng.hpp"
#include "ezquant/rtn.hpp"
#include "ezquant/stats.hpp"
#include "ezquant/types.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace ezquant;  // expands to ezq_ref

namespace {
thread_local std::string g_err;

// Status codes mirror include/ezquant_c.h.
int fail(int code, const char* what) {
    g_err = what;
    return code;
}

#define GUARD_BEGIN try {
#define GUARD_END                                                      \
    }                                                                  \
    catch (const std::invalid_argument& e) { return fail(1, e.what()); } \
    catch (const invariant_error& e) { return fail(2, e.what()); }       \
    catch (const io_error& e) { return fail(3 + static_cast<int>(e.kind()), e.what()); } \
    catch (const std::exception& e) { return fail(9, e.what()); }

struct CCfg {
    int32_t bits;
    float sigma_n;
    double lr, beta1, beta2, eps;
    int32_t steps, select, select_step, pad;
    uint64_t seed;
};

QuantConfig to_cfg(const CCfg* c) {
    QuantConfig q;
    q.bits = c->bits;
    q.sigma_n = c->sigma_n;
    q.lr = c->lr;
    q.adam_beta1 = c->beta1;
    q.adam_beta2 = c->beta2;
    q.adam_eps = c->eps;
    q.steps = c->steps;
    q.select = c->select ? SelectPolicy::FixedStep : SelectPolicy::BestError;
    q.select_step = c->select_step;
    q.seed = c->seed;
    return q;
}

DenseMatrix to_mat(const float* W, int64_t rows, int64_t cols) {
    DenseMatrix m;
    m.rows = rows;
    m.cols = cols;
    if (rows > 0 && cols > 0) m.data.assign(W, W + rows * cols);
    return m;
}

OutlierSet to_set(const uint32_t* r, const uint32_t* c, const float* v, int64_t n) {
    OutlierSet s;
    for (int64_t i = 0; i < n; ++i) s.entries.push_back({r[i], c[i], v ? v[i] : 0.0f});
    return s;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n);
#endif
    (void)n;
}

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ---- synthetic inputs with the reference RNG (rng.hpp) -------------------
void ref_gaussian(float* out, int64_t n, uint64_t seed, double scale) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng.gaussian() * scale);
}

// plant_outliers recipe of tests/acceptance.cpp:92-102.
void ref_plant_outliers(float* W, int64_t n, int64_t count, double lo, double hi, uint64_t seed) {
    Rng rng(seed);
    std::set<int64_t> used;
    while (static_cast<int64_t>(used.size()) < count) {
        const int64_t flat = rng.uniform_int(0, n - 1);
        if (!used.insert(flat).second) continue;
        const double mag = rng.uniform(lo, hi);
        W[flat] = static_cast<float>(rng.uniform() < 0.5 ? -mag : mag);
    }
}

// ---- stats.hpp -----------------------------------------------------------
int ref_tensor_stats(const float* W, int64_t rows, int64_t cols, int serial, double* out3,
                     int64_t* count) {
    GUARD_BEGIN
    const DenseMatrix m = to_mat(W, rows, cols);
    const TensorStats st = serial ? serial::tensor_stats(m) : tensor_stats(m);
    out3[0] = st.mean;
    out3[1] = st.stddev;
    out3[2] = st.max_abs;
    *count = st.count;
    return 0;
    GUARD_END
}

// ---- outliers.hpp --------------------------------------------------------
// Two-call protocol: returns the count; fills arrays when non-null.
int ref_detect_outliers(const float* W, int64_t rows, int64_t cols, const CCfg* c, int serial,
                        int64_t* n_out, uint32_t* r, uint32_t* col, float* v, double* mean,
                        double* stddev) {
    GUARD_BEGIN
    const DenseMatrix m = to_mat(W, rows, cols);
    const OutlierSet s = serial ? serial::detect_outliers(m, to_cfg(c)) : detect_outliers(m, to_cfg(c));
    *n_out = s.size();
    *mean = s.mean;
    *stddev = s.stddev;
    if (r)
        for (int64_t i = 0; i < s.size(); ++i) {
            r[i] = s.entries[i].row;
            col[i] = s.entries[i].col;
            v[i] = s.entries[i].value;
        }
    return 0;
    GUARD_END
}

// ---- pipeline.hpp --------------------------------------------------------
void* ref_quantize(const float* W, int64_t rows, int64_t cols, const CCfg* c, int mode,
                   int serial, int* status) {
    try {
        const DenseMatrix m = to_mat(W, rows, cols);
        const QuantMode qm = static_cast<QuantMode>(mode);
        auto* q = new QuantizedWeight(serial ? serial::quantize_tensor(m, to_cfg(c), qm)
                                             : quantize_tensor(m, to_cfg(c), qm));
        *status = 0;
        return q;
    } catch (const std::invalid_argument& e) {
        *status = fail(1, e.what());
    } catch (const invariant_error& e) {
        *status = fail(2, e.what());
    } catch (const io_error& e) {
        *status = fail(3 + static_cast<int>(e.kind()), e.what());
    } catch (const std::exception& e) {
        *status = fail(9, e.what());
    }
    return nullptr;
}

void ref_q_free(void* h) { delete static_cast<QuantizedWeight*>(h); }

int64_t ref_q_packed(void* h, uint8_t* dst) {
    auto* q = static_cast<QuantizedWeight*>(h);
    if (dst) std::memcpy(dst, q->packed_levels.data(), q->packed_levels.size());
    return static_cast<int64_t>(q->packed_levels.size());
}

void ref_q_scales(void* h, float* dst) {
    auto* q = static_cast<QuantizedWeight*>(h);
    std::memcpy(dst, q->scales.scales.data(), q->scales.scales.size() * sizeof(float));
}

int64_t ref_q_outliers(void* h, uint32_t* r, uint32_t* c, float* v) {
    auto* q = static_cast<QuantizedWeight*>(h);
    if (r)
        for (int64_t i = 0; i < q->outliers.size(); ++i) {
            r[i] = q->outliers.entries[i].row;
            c[i] = q->outliers.entries[i].col;
            v[i] = q->outliers.entries[i].value;
        }
    return q->outliers.size();
}

// meta: mean, stddev, rtn_error, final_error (NaN when absent); sigma_n; bits.
void ref_q_meta(void* h, double* d4, float* sigma_n, int* bits) {
    auto* q = static_cast<QuantizedWeight*>(h);
    d4[0] = q->outliers.mean;
    d4[1] = q->outliers.stddev;
    d4[2] = q->rtn_error ? *q->rtn_error : __builtin_nan("");
    d4[3] = q->final_error ? *q->final_error : __builtin_nan("");
    *sigma_n = q->outliers.sigma_n;
    *bits = q->bits;
}

// Builds a QuantizedWeight from raw arrays (for dequant / codec checks).
void* ref_q_make(int64_t rows, int64_t cols, int bits, const uint8_t* packed, int64_t packed_n,
                 const float* scales, int64_t n_out, const uint32_t* r, const uint32_t* c,
                 const float* v, double mean, double stddev, float sigma_n) {
    auto* q = new QuantizedWeight();
    q->rows = rows;
    q->cols = cols;
    q->bits = bits;
    q->packed_levels.assign(packed, packed + packed_n);
    q->scales.scales.assign(scales, scales + (cols > 0 ? cols : 0));
    q->outliers = to_set(r, c, v, n_out);
    q->outliers.mean = mean;
    q->outliers.stddev = stddev;
    q->outliers.sigma_n = sigma_n;
    return q;
}

int ref_dequantize(void* h, float* out, int serial) {
    GUARD_BEGIN
    auto* q = static_cast<QuantizedWeight*>(h);
    const DenseMatrix m = serial ? serial::dequantize_tensor(*q) : dequantize_tensor(*q);
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    return 0;
    GUARD_END
}

// ---- io.hpp (.ezqt codec) -------------------------------------------------
int64_t ref_encode(void* h, uint8_t* dst) {
    auto* q = static_cast<QuantizedWeight*>(h);
    const std::vector<uint8_t> b = encode_quantized(*q);
    if (dst) std::memcpy(dst, b.data(), b.size());
    return static_cast<int64_t>(b.size());
}

void* ref_decode(const uint8_t* bytes, int64_t n, int* status, uint64_t* offset) {
    try {
        auto* q = new QuantizedWeight(decode_quantized(std::span<const uint8_t>(bytes, n)));
        *status = 0;
        return q;
    } catch (const io_error& e) {
        *status = fail(3 + static_cast<int>(e.kind()), e.what());
        *offset = e.offset();
    } catch (const std::exception& e) {
        *status = fail(9, e.what());
    }
    return nullptr;
}

// ---- optimize.hpp --------------------------------------------------------
int ref_channel_eval(const float* x, int64_t n, const uint32_t* mask, int64_t nmask, double s,
                     const CCfg* c, double* err, double* grad) {
    GUARD_BEGIN
    const ChannelEval ev = channel_eval(std::span<const float>(x, n),
                                        std::span<const uint32_t>(mask, nmask), s, to_cfg(c));
    *err = ev.error;
    *grad = ev.gradient;
    return 0;
    GUARD_END
}

double ref_adam_step(double* m, double* v, int64_t* t, double scale, double grad, const CCfg* c) {
    AdamState st{*m, *v, *t};
    const double r = adam_step(st, scale, grad, to_cfg(c));
    *m = st.m;
    *v = st.v;
    *t = st.t;
    return r;
}

// trace arrays (steps+1) may be null when keep_trace == 0.
int ref_optimize_channel(const float* x, int64_t n, const uint32_t* mask, int64_t nmask,
                         const CCfg* c, int keep_trace, float* scale, double* init_err,
                         double* final_err, int* best_step, double* best_scale, double* best_err,
                         int* n_trace, int* tr_step, double* tr_scale, double* tr_err) {
    GUARD_BEGIN
    const OptimizeResult r = optimize_channel_range(
        std::span<const float>(x, n), std::span<const uint32_t>(mask, nmask), to_cfg(c),
        keep_trace != 0);
    *scale = r.scale;
    *init_err = r.initial_error;
    *final_err = r.final_error;
    *best_step = r.trace.best_step;
    *best_scale = r.trace.best_scale;
    *best_err = r.trace.best_error;
    *n_trace = static_cast<int>(r.trace.points.size());
    if (tr_step)
        for (size_t i = 0; i < r.trace.points.size(); ++i) {
            tr_step[i] = r.trace.points[i].step;
            tr_scale[i] = r.trace.points[i].scale;
            tr_err[i] = r.trace.points[i].error;
        }
    return 0;
    GUARD_END
}

int ref_brute_force(const float* x, int64_t n, const uint32_t* mask, int64_t nmask,
                    const CCfg* c, int grid, double* scale, double* err) {
    GUARD_BEGIN
    const BruteForceResult r = brute_force_optimal_scale(
        std::span<const float>(x, n), std::span<const uint32_t>(mask, nmask), to_cfg(c), grid);
    *scale = r.scale;
    *err = r.error;
    return 0;
    GUARD_END
}

// ---- rtn.hpp -------------------------------------------------------------
double ref_initial_scale(const float* x, int64_t n, const CCfg* c) {
    return initial_scale(std::span<const float>(x, n), to_cfg(c));
}

int ref_quantize_channel(const float* x, int64_t n, double s, const CCfg* c, int16_t* out) {
    GUARD_BEGIN
    const LevelVector lv = quantize_channel(std::span<const float>(x, n), s, to_cfg(c));
    std::memcpy(out, lv.levels.data(), n * sizeof(int16_t));
    return 0;
    GUARD_END
}

int ref_dequantize_channel(const int16_t* l, int64_t n, int bits, double s, float* out) {
    GUARD_BEGIN
    LevelVector lv;
    lv.bits = bits;
    lv.levels.assign(l, l + n);
    const std::vector<float> o = dequantize_channel(lv, s);
    std::memcpy(out, o.data(), n * sizeof(float));
    return 0;
    GUARD_END
}

int64_t ref_packed_size(int64_t count, int bits) { return packed_size(count, bits); }

int ref_pack_levels(const int16_t* l, int64_t n, int bits, uint8_t* out) {
    GUARD_BEGIN
    LevelVector lv;
    lv.bits = bits;
    lv.levels.assign(l, l + n);
    const std::vector<uint8_t> b = pack_levels(lv);
    std::memcpy(out, b.data(), b.size());
    return 0;
    GUARD_END
}

int ref_unpack_levels(const uint8_t* b, int64_t nbytes, int64_t count, int bits, int16_t* out) {
    GUARD_BEGIN
    const LevelVector lv = unpack_levels(std::span<const uint8_t>(b, nbytes), count, bits);
    std::memcpy(out, lv.levels.data(), count * sizeof(int16_t));
    return 0;
    GUARD_END
}

int ref_reconstruction_error(const float* a, const float* b, int64_t rows, int64_t cols,
                             const uint32_t* r, const uint32_t* c, int64_t n_skip, int serial,
                             double* out) {
    GUARD_BEGIN
    const DenseMatrix A = to_mat(a, rows, cols);
    const DenseMatrix B = to_mat(b, rows, cols);
    const OutlierSet s = to_set(r, c, nullptr, n_skip);
    const OutlierSet* sp = r ? &s : nullptr;
    *out = serial ? serial::reconstruction_error(A, B, sp) : reconstruction_error(A, B, sp);
    return 0;
    GUARD_END
}

// ---- model.hpp (whole-model driver, for byte-identical output checks) ----
int ref_quantize_model(const char* manifest, const char* out_dir, const CCfg* c, int mode,
                       int workers, int* failures) {
    GUARD_BEGIN
    const ModelManifest m = load_manifest(manifest);
    *failures = quantize_model(m, to_cfg(c), static_cast<QuantMode>(mode), workers, out_dir).failures;
    return 0;
    GUARD_END
}

int ref_dequantize_model(const char* in_dir, const char* out_dir, int workers, int* failures) {
    GUARD_BEGIN
    *failures = dequantize_model(in_dir, workers, out_dir).failures;
    return 0;
    GUARD_END
}

// report.hpp sigma_sweep: JSON rows (sweep_to_json) into `out` (cap bytes).
int ref_sigma_sweep(const char* manifest, const CCfg* c, const float* sigmas, int n, int workers,
                    char* out, int64_t cap) {
    GUARD_BEGIN
    const std::vector<SweepRow> rows =
        sigma_sweep(load_manifest(manifest), to_cfg(c), std::vector<float>(sigmas, sigmas + n), workers);
    const std::string js = sweep_to_json(rows);
    if (static_cast<int64_t>(js.size()) + 1 > cap) return fail(1, "output buffer too small");
    std::memcpy(out, js.c_str(), js.size() + 1);
    return 0;
    GUARD_END
}

}  // extern "C"
