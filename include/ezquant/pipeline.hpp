// Drop-in for ezquant/pipeline.hpp (reference pipeline.hpp:12-49): the
// whole-tensor quantize / dequantize entry points, executed by the B200
// engine (K1-K5). serial:: twins run the same device path (bit-identical).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ezquant/types.hpp"

namespace ezquant {

enum class QuantMode { Easyquant, Rtn, OutliersOnly };

QuantMode parse_quant_mode(const std::string& s);
const char* quant_mode_name(QuantMode m);

QuantizedWeight quantize_tensor(const DenseMatrix& W, const QuantConfig& cfg,
                                QuantMode mode = QuantMode::Easyquant);
QuantizedWeight easyquant_tensor(const DenseMatrix& W, const QuantConfig& cfg);
QuantizedWeight rtn_tensor(const DenseMatrix& W, const QuantConfig& cfg);
DenseMatrix dequantize_tensor(const QuantizedWeight& q);

/// B200 extension: quantizes independent tensors in shared kernel launches.
std::vector<QuantizedWeight> quantize_tensors(const std::vector<const DenseMatrix*>& Ws,
                                              const QuantConfig& cfg,
                                              QuantMode mode = QuantMode::Easyquant);

namespace serial {
QuantizedWeight quantize_tensor(const DenseMatrix& W, const QuantConfig& cfg,
                                QuantMode mode = QuantMode::Easyquant);
DenseMatrix dequantize_tensor(const QuantizedWeight& q);
}  // namespace serial

}  // namespace ezquant
