// Compiled against include/ezquant/*.hpp and linked with libezquant.so: the
// reference's public C++ API used exactly as reference callers use it, now
// executed by the B200 engine. Prints "N checks, M failures".
#include <cmath>
#include <cstdio>
#include <set>
#include <stdexcept>
#include <vector>

#include "ezquant/error.hpp"
#include "ezquant/optimize.hpp"
#include "ezquant/outliers.hpp"
#include "ezquant/pipeline.hpp"
#include "ezquant/rng.hpp"
#include "ezquant/rtn.hpp"
#include "ezquant/stats.hpp"

using namespace ezquant;

static int g_checks = 0, g_fail = 0;
#define EXPECT(cond)                                                     \
    do {                                                                 \
        ++g_checks;                                                      \
        if (!(cond)) {                                                   \
            ++g_fail;                                                    \
            std::printf("FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond); \
        }                                                                \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static DenseMatrix normal(int64_t r, int64_t c, uint64_t seed, double sd) {
    DenseMatrix m(r, c);
    Rng g(seed);
    for (auto& v : m.data) v = static_cast<float>(g.gaussian() * sd);
    return m;
}

int main() {
    QuantConfig cfg;
    // stats
    TensorStats st = tensor_stats(DenseMatrix(1, 5, {0, 0, 0, 0, 100}));
    EXPECT(std::fabs(st.mean - 20.0) < 1e-12 && std::fabs(st.stddev - 40.0) < 1e-12);
    DenseMatrix g = normal(123, 217, 4, 0.05);
    TensorStats a = tensor_stats(g), b = serial::tensor_stats(g);
    EXPECT(a.mean == b.mean && a.stddev == b.stddev && a.max_abs == b.max_abs);
    // outliers
    QuantConfig two = cfg;
    two.sigma_n = 2.0f;
    OutlierSet os = detect_outliers(DenseMatrix(1, 5, {0, 0, 0, 0, 100}), two);
    EXPECT(os.size() == 1 && os.entries[0].col == 4 && os.entries[0].value == 100.0f);
    auto cols = outlier_rows_by_column(detect_outliers(normal(64, 16, 10, 1.0), two), 16);
    EXPECT(static_cast<int64_t>(cols.size()) == 16);
    MaskedChannel mc = normal_mask_apply(std::vector<float>{1.f, 9.f, 2.f}, std::vector<uint32_t>{1});
    EXPECT(mc.values == std::vector<float>({1.f, 2.f}) && mc.rows == std::vector<uint32_t>({0, 2}));
    // rtn / packing
    LevelVector lv = quantize_channel(std::vector<float>{0.5f, -0.25f, 1.0f, 2.5f}, 0.25, cfg);
    EXPECT(lv.levels == std::vector<int16_t>({2, -1, 4, 8}));
    EXPECT(quantize_channel(std::vector<float>{0.125f, -0.125f}, 0.25, cfg).levels ==
           std::vector<int16_t>({1, -1}));
    EXPECT(throws<std::invalid_argument>([&] { quantize_channel(std::vector<float>{1.f}, 0.0, cfg); }));
    LevelVector p;
    p.bits = 4;
    p.levels = {-7, 8};
    EXPECT(pack_levels(p) == std::vector<uint8_t>({0xF0}));
    EXPECT(unpack_levels(pack_levels(p), 2, 4).levels == p.levels);
    EXPECT(packed_size(3, 4) == 2 && packed_size(5, 3) == 5);
    // optimizer
    EXPECT(std::fabs(range_gradient(std::vector<float>{0.3f}, {}, 0.25, cfg) + 0.1) < 1e-6);
    std::vector<float> x(1024);
    Rng r7(7);
    for (auto& v : x) v = static_cast<float>(r7.gaussian());
    OptimizeResult o = optimize_channel_range(x, {}, cfg, true);
    EXPECT(o.trace.points.size() == 201 && o.final_error <= o.initial_error);
    EXPECT(static_cast<double>(o.scale) == o.trace.best_scale);
    BruteForceResult bf = brute_force_optimal_scale(x, {}, cfg, 2000);
    EXPECT(o.final_error <= 1.25 * bf.error);
    AdamState ad;
    EXPECT(adam_step(ad, 0.5, 0.0, cfg) == 0.5 && ad.t == 1);
    // pipeline
    DenseMatrix w = normal(96, 64, 71, 0.05);
    QuantizedWeight q = easyquant_tensor(w, cfg);
    QuantizedWeight qs = serial::quantize_tensor(w, cfg);
    EXPECT(q.packed_levels == qs.packed_levels && q.scales.scales == qs.scales.scales &&
           q.outliers.entries == qs.outliers.entries && q.rtn_error == qs.rtn_error &&
           q.final_error == qs.final_error);
    EXPECT(*q.final_error <= *q.rtn_error);
    DenseMatrix back = dequantize_tensor(q);
    for (const auto& e : q.outliers.entries) EXPECT(back.at(e.row, e.col) == w.at(e.row, e.col));
    double rec = reconstruction_error(w, back, &q.outliers);
    EXPECT(std::fabs(rec - *q.final_error) <= 1e-5 * *q.final_error);
    QuantizedWeight rt = rtn_tensor(w, cfg);
    EXPECT(rt.outliers.empty() && *rt.rtn_error == *rt.final_error);
    EXPECT(quant_mode_name(parse_quant_mode("outliers-only")) == std::string("outliers-only"));
    EXPECT(throws<std::invalid_argument>([] { parse_quant_mode("fp16"); }));
    DenseMatrix bad(2, 2, {1.f, 2.f, 3.f, INFINITY});
    EXPECT(throws<std::invalid_argument>([&] { easyquant_tensor(bad, cfg); }));
    EXPECT(throws<std::invalid_argument>([&] { easyquant_tensor(DenseMatrix(2, 2, {1.f, 2.f}), cfg); }));
    QuantConfig badcfg = cfg;
    badcfg.bits = 9;
    EXPECT(throws<std::invalid_argument>([&] { badcfg.validate(); }));
    QuantizedWeight empty;
    EXPECT(throws<io_error>([&] { dequantize_tensor(empty); }));
    std::vector<QuantizedWeight> many = quantize_tensors({&w, &g}, cfg);
    EXPECT(many.size() == 2 && many[0].packed_levels == q.packed_levels);
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
