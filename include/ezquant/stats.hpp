// Drop-in for ezquant/stats.hpp (reference stats.hpp:14-20). Runs on the
// B200 (K1): 8192-element fp64 chunks merged in chunk order, bit-identical to
// the reference for any thread count.
#pragma once

#include "ezquant/types.hpp"

namespace ezquant {
TensorStats tensor_stats(const DenseMatrix& W);
namespace serial {
TensorStats tensor_stats(const DenseMatrix& W);  // same device path, same bits
}
}  // namespace ezquant
