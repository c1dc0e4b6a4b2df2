// C++ drop-in (namespace ezquant, include/ezquant/*.hpp) over the C-ABI.
// Status codes from libezq_b200.so are mapped back onto the exact exception
// types the reference throws (error.hpp, <stdexcept>), with its messages.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ezquant/error.hpp"
#include "../../include/ezquant/optimize.hpp"
#include "../../include/ezquant/outliers.hpp"
#include "../../include/ezquant/pipeline.hpp"
#include "../../include/ezquant/rtn.hpp"
#include "../../include/ezquant/stats.hpp"
#include "../../include/ezquant/types.hpp"
#include "../../include/ezquant_c.h"

namespace ezquant {

namespace {

[[noreturn]] void raise(int code) {
    char msg[1024];
    int64_t idx = -1;
    ezq_last_error(msg, sizeof msg, &idx);
    switch (code) {
        case EZQ_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EZQ_ERR_INVARIANT: throw invariant_error(msg);
        case EZQ_ERR_IO_FAILURE: throw io_error(IoErrorKind::IoFailure, 0, msg);
        case EZQ_ERR_IO_FORMAT: throw io_error(IoErrorKind::FormatViolation, 0, msg);
        case EZQ_ERR_IO_VERSION: throw io_error(IoErrorKind::VersionMismatch, 0, msg);
        default: throw std::runtime_error(msg);
    }
}

inline void check(int code) {
    if (code != EZQ_OK) raise(code);
}

ezq_config to_c(const QuantConfig& c) {
    ezq_config o;
    ezq_config_default(&o);
    o.bits = c.bits;
    o.sigma_n = c.sigma_n;
    o.lr = c.lr;
    o.beta1 = c.adam_beta1;
    o.beta2 = c.adam_beta2;
    o.eps = c.adam_eps;
    o.steps = c.steps;
    o.select = c.select == SelectPolicy::FixedStep ? EZQ_SELECT_FIXED : EZQ_SELECT_BEST;
    o.select_step = c.select_step;
    o.seed = c.seed;
    return o;
}

void check_shape(const DenseMatrix& W) {
    if (W.rows <= 0 || W.cols <= 0)
        throw std::invalid_argument("matrix shape must be positive, got " + std::to_string(W.rows) +
                                    "x" + std::to_string(W.cols));
    if (static_cast<size_t>(W.rows) * static_cast<size_t>(W.cols) != W.data.size())
        throw std::invalid_argument("matrix data length " + std::to_string(W.data.size()) +
                                    " does not match shape " + std::to_string(W.rows) + "x" +
                                    std::to_string(W.cols));
}

QuantizedWeight from_c(const ezq_qweight* q) {
    QuantizedWeight w;
    w.rows = q->rows;
    w.cols = q->cols;
    w.bits = q->bits;
    w.packed_levels.assign(q->packed, q->packed + q->packed_bytes);
    w.scales.scales.assign(q->scales, q->scales + q->cols);
    w.outliers.entries.resize(static_cast<size_t>(q->n_outliers));
    for (int64_t i = 0; i < q->n_outliers; ++i)
        w.outliers.entries[i] = {q->outliers[i].row, q->outliers[i].col, q->outliers[i].value};
    w.outliers.mean = q->mean;
    w.outliers.stddev = q->stddev;
    w.outliers.sigma_n = q->sigma_n;
    if (q->has_errors) {
        w.rtn_error = q->rtn_error;
        w.final_error = q->final_error;
    }
    return w;
}

QuantizedWeight quantize_impl(const DenseMatrix& W, const QuantConfig& cfg, QuantMode mode) {
    check_shape(W);
    const ezq_config c = to_c(cfg);
    ezq_qweight* q = nullptr;
    check(ezq_quantize_tensor(W.data.data(), W.rows, W.cols, &c, static_cast<int>(mode),
                              EZQ_MEM_HOST, EZQ_MEM_HOST, nullptr, &q));
    QuantizedWeight w = from_c(q);
    ezq_qweight_free(q);
    return w;
}

DenseMatrix dequantize_impl(const QuantizedWeight& q) {
    std::vector<ezq_outlier> e(q.outliers.entries.size());
    for (size_t i = 0; i < e.size(); ++i)
        e[i] = {q.outliers.entries[i].row, q.outliers.entries[i].col, q.outliers.entries[i].value};
    ezq_qweight* w = nullptr;
    check(ezq_qweight_wrap(q.rows, q.cols, q.bits, q.packed_levels.data(),
                           static_cast<int64_t>(q.packed_levels.size()), q.scales.scales.data(),
                           q.scales.size(), e.data(), static_cast<int64_t>(e.size()),
                           q.outliers.mean, q.outliers.stddev, q.outliers.sigma_n, EZQ_MEM_HOST,
                           &w));
    DenseMatrix out;
    if (q.rows > 0 && q.cols > 0) out = DenseMatrix(q.rows, q.cols);
    const int s = ezq_dequantize_tensor(w, out.data.data(), EZQ_MEM_HOST, nullptr);
    ezq_qweight_free(w);
    check(s);
    return out;
}

double recon_impl(const DenseMatrix& a, const DenseMatrix& b, const OutlierSet* skip) {
    if (a.rows != b.rows || a.cols != b.cols)
        throw std::invalid_argument("shape mismatch: " + std::to_string(a.rows) + "x" +
                                    std::to_string(a.cols) + " vs " + std::to_string(b.rows) +
                                    "x" + std::to_string(b.cols));
    std::vector<uint32_t> r, c;
    if (skip && !skip->empty()) {
        for (const auto& e : skip->entries) {
            r.push_back(e.row);
            c.push_back(e.col);
        }
    }
    double out = 0.0;
    check(ezq_reconstruction_error(a.data.data(), b.data.data(), a.rows, a.cols,
                                   r.empty() ? nullptr : r.data(), c.empty() ? nullptr : c.data(),
                                   static_cast<int64_t>(r.size()), EZQ_MEM_HOST, nullptr, &out));
    return out;
}

OutlierSet detect_impl(const DenseMatrix& W, const QuantConfig& cfg) {
    const ezq_config c = to_c(cfg);
    ezq_outlier* e = nullptr;
    int64_t n = 0;
    OutlierSet s;
    check(ezq_detect_outliers(W.data.data(), W.rows, W.cols, &c, EZQ_MEM_HOST, nullptr, &e, &n,
                              &s.mean, &s.stddev));
    s.sigma_n = cfg.sigma_n;
    s.entries.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) s.entries[i] = {e[i].row, e[i].col, e[i].value};
    ezq_free(e);
    return s;
}

TensorStats stats_impl(const DenseMatrix& W) {
    ezq_stats st;
    check(ezq_tensor_stats(W.data.data(), W.rows, W.cols, EZQ_MEM_HOST, nullptr, &st));
    return {st.mean, st.stddev, st.max_abs, st.count};
}

ChannelEval eval_impl(std::span<const float> x, std::span<const uint32_t> mask, double s,
                      const QuantConfig& cfg) {
    const ezq_config c = to_c(cfg);
    ChannelEval ev;
    check(ezq_channel_eval(x.data(), static_cast<int64_t>(x.size()), mask.data(),
                           static_cast<int64_t>(mask.size()), s, &c, &ev.error, &ev.gradient));
    return ev;
}

}  // namespace

// ---- types.cpp -----------------------------------------------------------
void DenseMatrix::validate() const {
    check_shape(*this);
    for (size_t i = 0; i < data.size(); ++i)
        if (!std::isfinite(data[i]))
            throw std::invalid_argument("non-finite element at flat index " + std::to_string(i));
}

void QuantConfig::validate() const {
    const ezq_config c = to_c(*this);
    check(ezq_config_validate(&c));
}

// ---- stats ---------------------------------------------------------------
TensorStats tensor_stats(const DenseMatrix& W) { return stats_impl(W); }
namespace serial {
TensorStats tensor_stats(const DenseMatrix& W) { return stats_impl(W); }
}  // namespace serial

// ---- outliers ------------------------------------------------------------
OutlierSet detect_outliers(const DenseMatrix& W, const QuantConfig& cfg) {
    return detect_impl(W, cfg);
}
namespace serial {
OutlierSet detect_outliers(const DenseMatrix& W, const QuantConfig& cfg) {
    return detect_impl(W, cfg);
}
}  // namespace serial

std::vector<std::vector<uint32_t>> outlier_rows_by_column(const OutlierSet& outliers, int64_t cols) {
    std::vector<std::vector<uint32_t>> by_col(static_cast<size_t>(cols));
    for (const auto& e : outliers.entries) {
        if (e.col >= static_cast<uint64_t>(cols))
            throw std::invalid_argument("outlier column " + std::to_string(e.col) +
                                        " out of range for " + std::to_string(cols) + " columns");
        by_col[e.col].push_back(e.row);
    }
    return by_col;
}

MaskedChannel normal_mask_apply(std::span<const float> x, std::span<const uint32_t> outlier_rows) {
    MaskedChannel out;
    size_t k = 0;
    for (size_t i = 0; i < x.size(); ++i) {
        if (k < outlier_rows.size() && outlier_rows[k] == i) {
            ++k;
            continue;
        }
        out.values.push_back(x[i]);
        out.rows.push_back(static_cast<uint32_t>(i));
    }
    return out;
}

void scatter_outliers(DenseMatrix& m, const OutlierSet& outliers) {
    for (const auto& e : outliers.entries) {
        if (e.row >= static_cast<uint64_t>(m.rows) || e.col >= static_cast<uint64_t>(m.cols))
            throw std::invalid_argument("outlier coordinate (" + std::to_string(e.row) + ", " +
                                        std::to_string(e.col) + ") outside " +
                                        std::to_string(m.rows) + "x" + std::to_string(m.cols));
        m.at(e.row, e.col) = e.value;
    }
}

// ---- rtn -----------------------------------------------------------------
double initial_scale(std::span<const float> x, const QuantConfig& cfg) {
    const ezq_config c = to_c(cfg);
    return ezq_initial_scale(x.data(), static_cast<int64_t>(x.size()), &c);
}

LevelVector quantize_channel(std::span<const float> x, double scale, const QuantConfig& cfg) {
    const ezq_config c = to_c(cfg);
    LevelVector lv;
    lv.bits = cfg.bits;
    lv.levels.resize(x.size());
    check(ezq_quantize_channel(x.data(), static_cast<int64_t>(x.size()), scale, &c,
                               lv.levels.data()));
    return lv;
}

std::vector<float> dequantize_channel(const LevelVector& levels, double scale) {
    std::vector<float> out(levels.levels.size());
    check(ezq_dequantize_channel(levels.levels.data(), levels.size(), scale, out.data()));
    return out;
}

double reconstruction_error(const DenseMatrix& a, const DenseMatrix& b, const OutlierSet* skip) {
    return recon_impl(a, b, skip);
}
namespace serial {
double reconstruction_error(const DenseMatrix& a, const DenseMatrix& b, const OutlierSet* skip) {
    return recon_impl(a, b, skip);
}
}  // namespace serial

int64_t packed_size(int64_t count, int bits) { return ezq_packed_size(count, bits); }

std::vector<uint8_t> pack_levels(const LevelVector& lv) {
    std::vector<uint8_t> out(static_cast<size_t>(ezq_packed_size(lv.size(), lv.bits)));
    check(ezq_pack_levels(lv.levels.data(), lv.size(), lv.bits, out.data()));
    return out;
}

LevelVector unpack_levels(std::span<const uint8_t> bytes, int64_t count, int bits) {
    LevelVector lv;
    lv.bits = bits;
    lv.levels.resize(static_cast<size_t>(std::max<int64_t>(count, 0)));
    check(ezq_unpack_levels(bytes.data(), static_cast<int64_t>(bytes.size()), count, bits,
                            lv.levels.data()));
    return lv;
}

// ---- optimize --------------------------------------------------------------
double adam_step(AdamState& st, double scale, double grad, const QuantConfig& cfg) {
    const ezq_config c = to_c(cfg);
    double out = 0.0;
    check(ezq_adam_step(&st.m, &st.v, &st.t, scale, grad, &c, &out));
    return out;
}

double channel_error(std::span<const float> x, std::span<const uint32_t> mask, double s,
                     const QuantConfig& cfg) {
    return eval_impl(x, mask, s, cfg).error;
}
double range_gradient(std::span<const float> x, std::span<const uint32_t> mask, double s,
                      const QuantConfig& cfg) {
    return eval_impl(x, mask, s, cfg).gradient;
}
ChannelEval channel_eval(std::span<const float> x, std::span<const uint32_t> mask, double s,
                         const QuantConfig& cfg) {
    return eval_impl(x, mask, s, cfg);
}
namespace serial {
double channel_error(std::span<const float> x, std::span<const uint32_t> mask, double s,
                     const QuantConfig& cfg) {
    return eval_impl(x, mask, s, cfg).error;
}
}  // namespace serial

OptimizeResult optimize_channel_range(std::span<const float> x, std::span<const uint32_t> mask,
                                      const QuantConfig& cfg, bool keep_trace) {
    const ezq_config c = to_c(cfg);
    ezq_opt_result r;
    const size_t np = keep_trace ? static_cast<size_t>(std::max(cfg.steps, 0)) + 1 : 0;
    std::vector<int32_t> ts(np);
    std::vector<double> sc(np), er(np);
    check(ezq_optimize_channel(x.data(), static_cast<int64_t>(x.size()), mask.data(),
                               static_cast<int64_t>(mask.size()), &c, keep_trace ? 1 : 0, &r,
                               ts.data(), sc.data(), er.data()));
    OptimizeResult res;
    res.scale = r.scale;
    res.initial_error = r.initial_error;
    res.final_error = r.final_error;
    res.trace.best_step = r.best_step;
    res.trace.best_scale = r.best_scale;
    res.trace.best_error = r.best_error;
    for (int i = 0; i < r.n_trace; ++i) res.trace.points.push_back({ts[i], sc[i], er[i]});
    return res;
}

BruteForceResult brute_force_optimal_scale(std::span<const float> x,
                                           std::span<const uint32_t> mask,
                                           const QuantConfig& cfg, int grid_points) {
    const ezq_config c = to_c(cfg);
    BruteForceResult r;
    check(ezq_brute_force_scale(x.data(), static_cast<int64_t>(x.size()), mask.data(),
                                static_cast<int64_t>(mask.size()), &c, grid_points, &r.scale,
                                &r.error));
    return r;
}

// ---- pipeline ----------------------------------------------------------------
QuantMode parse_quant_mode(const std::string& s) {
    if (s == "easyquant") return QuantMode::Easyquant;
    if (s == "rtn") return QuantMode::Rtn;
    if (s == "outliers-only") return QuantMode::OutliersOnly;
    throw std::invalid_argument("unknown mode '" + s +
                                "' (expected easyquant, rtn, or outliers-only)");
}

const char* quant_mode_name(QuantMode m) {
    switch (m) {
        case QuantMode::Easyquant: return "easyquant";
        case QuantMode::Rtn: return "rtn";
        case QuantMode::OutliersOnly: return "outliers-only";
    }
    return "?";
}

QuantizedWeight quantize_tensor(const DenseMatrix& W, const QuantConfig& cfg, QuantMode mode) {
    return quantize_impl(W, cfg, mode);
}
QuantizedWeight easyquant_tensor(const DenseMatrix& W, const QuantConfig& cfg) {
    return quantize_impl(W, cfg, QuantMode::Easyquant);
}
QuantizedWeight rtn_tensor(const DenseMatrix& W, const QuantConfig& cfg) {
    return quantize_impl(W, cfg, QuantMode::Rtn);
}
DenseMatrix dequantize_tensor(const QuantizedWeight& q) { return dequantize_impl(q); }

std::vector<QuantizedWeight> quantize_tensors(const std::vector<const DenseMatrix*>& Ws,
                                              const QuantConfig& cfg, QuantMode mode) {
    std::vector<const float*> ptr;
    std::vector<int64_t> r, c;
    for (const DenseMatrix* W : Ws) {
        check_shape(*W);
        ptr.push_back(W->data.data());
        r.push_back(W->rows);
        c.push_back(W->cols);
    }
    const ezq_config cc = to_c(cfg);
    std::vector<ezq_qweight*> q(Ws.size(), nullptr);
    check(ezq_quantize_batch(ptr.data(), r.data(), c.data(), static_cast<int>(Ws.size()), &cc,
                             static_cast<int>(mode), EZQ_MEM_HOST, EZQ_MEM_HOST, nullptr, q.data(),
                             nullptr));
    std::vector<QuantizedWeight> out;
    for (ezq_qweight* w : q) {
        out.push_back(from_c(w));
        ezq_qweight_free(w);
    }
    return out;
}

namespace serial {
QuantizedWeight quantize_tensor(const DenseMatrix& W, const QuantConfig& cfg, QuantMode mode) {
    return quantize_impl(W, cfg, mode);
}
DenseMatrix dequantize_tensor(const QuantizedWeight& q) { return dequantize_impl(q); }
}  // namespace serial

}  // namespace ezquant
