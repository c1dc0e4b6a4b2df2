// Drop-in for ezquant/outliers.hpp (reference outliers.hpp:15-38).
// detect_outliers runs on the B200 (K1 + K2); the rest is host bookkeeping.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "ezquant/types.hpp"

namespace ezquant {

OutlierSet detect_outliers(const DenseMatrix& W, const QuantConfig& cfg);
std::vector<std::vector<uint32_t>> outlier_rows_by_column(const OutlierSet& outliers, int64_t cols);

struct MaskedChannel {
    std::vector<float> values;
    std::vector<uint32_t> rows;
};

MaskedChannel normal_mask_apply(std::span<const float> x, std::span<const uint32_t> outlier_rows);
void scatter_outliers(DenseMatrix& m, const OutlierSet& outliers);

namespace serial {
OutlierSet detect_outliers(const DenseMatrix& W, const QuantConfig& cfg);
}

}  // namespace ezquant
