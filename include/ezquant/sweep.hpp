// Threshold sweep (the sigma_sweep part of the reference's ezquant/report.hpp,
// /root/reference/proj/include/ezquant/report.hpp:82-99; SURVEY.md §8f next
// #2). Same declarations; the B200 implementation keeps the model's matrices
// resident in HBM across the sweep and quantizes all of them in one batched
// device call per sigma_n, keeping only the per-tensor scalars (outlier
// count, rtn_error, final_error) -- no artifact leaves the device.
// The rest of report.hpp (model_report, tensor_file_report, table/JSON
// renderers of a model directory) is presentation over the manifest and is
// out of scope.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "ezquant/io.hpp"
#include "ezquant/types.hpp"

namespace ezquant {

/// One sigma value of a threshold sweep over a model.
struct SweepRow {
    float sigma_n = 0.0f;
    int64_t outliers = 0;
    double outlier_fraction = 0.0;
    double rtn_error = 0.0;    // summed over tensors in manifest order, initial scales
    double final_error = 0.0;  // summed over tensors in manifest order, optimized scales
};

/// Quantizes every 2-D tensor of the model once per sigma (Easyquant mode,
/// nothing written) and aggregates outlier fractions and errors.
std::vector<SweepRow> sigma_sweep(const ModelManifest& manifest, const QuantConfig& base,
                                  const std::vector<float>& sigmas, int workers);

void print_sweep_table(const std::vector<SweepRow>& rows, std::ostream& os);
std::string sweep_to_json(const std::vector<SweepRow>& rows);

}  // namespace ezquant
