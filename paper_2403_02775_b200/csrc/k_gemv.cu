// K6: fused dequant + outlier GEMV / skinny GEMM (placeholder until the
// kernel lands; returns an explicit error, never a CPU fallback).
#include "runtime.hpp"

using namespace ezq;

struct ezq_gemv_plan {
    int dummy;
};

extern "C" {
int ezq_gemv_prepare(const ezq_qweight*, void*, ezq_gemv_plan** plan) {
    *plan = nullptr;
    return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv is not built yet");
}
int ezq_gemv(const ezq_gemv_plan*, const void*, int, int, float*, void*) {
    return set_error(EZQ_ERR_INVALID_ARGUMENT, "ezq_gemv is not built yet");
}
void ezq_gemv_plan_free(ezq_gemv_plan* plan) { delete plan; }
}
