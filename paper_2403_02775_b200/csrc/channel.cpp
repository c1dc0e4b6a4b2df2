// Channel-scale C-ABI (optimize.hpp:20-95, rtn.hpp:14-30). Host-side
// bookkeeping (mask gathering, grid construction, argmin) mirrors the
// reference line by line; every per-element evaluation runs on the device in
// the reference's sequential order (k_channel.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "runtime.hpp"

namespace ezq {
namespace {

// gather_normals (optimize.cpp:54-66): mask must be sorted ascending.
std::vector<float> gather(const float* x, int64_t n, const uint32_t* mask, int64_t nm) {
    std::vector<float> out;
    out.reserve(static_cast<size_t>(n));
    int64_t next = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (next < nm && mask[next] == static_cast<uint32_t>(i)) {
            ++next;
            continue;
        }
        out.push_back(x[i]);
    }
    return out;
}

int scale_error(double s) {
    return set_error(EZQ_ERR_INVALID_ARGUMENT, "scale must be finite and > 0, got " + fmt_double(s));
}

struct DevBuf {
    Arena ar;
    cudaStream_t st = nullptr;
};

// Evaluates err/grad of the (already gathered) channel at `scales` on the device.
int eval_scales(const std::vector<float>& v, const std::vector<double>& scales,
                const ezq_config* cfg, std::vector<double>& err, std::vector<double>* grad) {
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = thread_stream(dev);
    const size_t ns = scales.size();
    Arena ar;
    ar.reserve(sizeof(float) * std::max<size_t>(v.size(), 1));
    for (int k = 0; k < 3; ++k) ar.reserve(sizeof(double) * ns);
    if (int s = ar.allocate(st)) return s;
    float* dx = ar.take<float>(std::max<size_t>(v.size(), 1));
    double* ds = ar.take<double>(ns);
    double* de = ar.take<double>(ns);
    double* dg = ar.take<double>(ns);
    if (!v.empty())
        EZQ_CK(cudaMemcpyAsync(dx, v.data(), sizeof(float) * v.size(), cudaMemcpyHostToDevice, st));
    EZQ_CK(cudaMemcpyAsync(ds, scales.data(), sizeof(double) * ns, cudaMemcpyHostToDevice, st));
    const CfgDev cd = make_cfg(cfg, EZQ_MODE_EASYQUANT, nullptr);
    launch_channel_eval(dx, static_cast<int64_t>(v.size()), ds, static_cast<int>(ns), cd, de,
                        grad ? dg : nullptr, st);
    EZQ_CK(cudaGetLastError());
    err.resize(ns);
    EZQ_CK(cudaMemcpyAsync(err.data(), de, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    if (grad) {
        grad->resize(ns);
        EZQ_CK(cudaMemcpyAsync(grad->data(), dg, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    }
    EZQ_CK(cudaStreamSynchronize(st));
    return EZQ_OK;
}

}  // namespace
}  // namespace ezq

using namespace ezq;

extern "C" {

int ezq_channel_eval(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                     double scale, const ezq_config* cfg, double* error, double* gradient) {
    if (!(scale > 0.0) || !std::isfinite(scale)) return scale_error(scale);  // optimize.cpp:70
    const std::vector<float> v = gather(x, n, mask, n_mask);
    std::vector<double> e, g;
    if (int s = eval_scales(v, {scale}, cfg, e, &g)) return s;
    *error = e[0];
    *gradient = g[0];
    return clear_error();
}

int ezq_optimize_channel(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                         const ezq_config* cfg, int keep_trace, ezq_opt_result* res,
                         int32_t* trace_step, double* trace_scale, double* trace_error) {
    std::memset(res, 0, sizeof(*res));
    const std::vector<float> v = gather(x, n, mask, n_mask);
    if (v.empty()) {  // optimize.cpp:128-133
        res->scale = 1.0f;
        res->best_scale = 1.0;
        return clear_error();
    }
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = thread_stream(dev);
    std::vector<double> bc;
    bias_tables(cfg, bc);
    const int steps = cfg->steps > 0 ? cfg->steps : 0;
    const size_t ntr = keep_trace ? static_cast<size_t>(steps + 1) * 2 : 0;
    Arena ar;
    ar.reserve(sizeof(float) * v.size());
    ar.reserve(sizeof(int64_t) * 2);
    ar.reserve(sizeof(double) * bc.size());
    ar.reserve(sizeof(double) * 8);
    ar.reserve(sizeof(double) * ntr);
    if (int s = ar.allocate(st)) return s;
    float* dx = ar.take<float>(v.size());
    int64_t* doff = ar.take<int64_t>(2);
    double* dbc = ar.take<double>(bc.size());
    double* dout = ar.take<double>(8);
    double* dtr = ntr ? ar.take<double>(ntr) : nullptr;
    const int64_t offs[2] = {0, static_cast<int64_t>(v.size())};
    EZQ_CK(cudaMemcpyAsync(dx, v.data(), sizeof(float) * v.size(), cudaMemcpyHostToDevice, st));
    EZQ_CK(cudaMemcpyAsync(doff, offs, sizeof(offs), cudaMemcpyHostToDevice, st));
    EZQ_CK(cudaMemcpyAsync(dbc, bc.data(), sizeof(double) * bc.size(), cudaMemcpyHostToDevice, st));
    const CfgDev cd = make_cfg(cfg, EZQ_MODE_EASYQUANT, dbc);
    launch_optimize_channels(dx, doff, 1, cd, keep_trace, dout, dtr, st);
    EZQ_CK(cudaGetLastError());
    double o[8];
    std::vector<double> tr(ntr);
    EZQ_CK(cudaMemcpyAsync(o, dout, sizeof(o), cudaMemcpyDeviceToHost, st));
    if (ntr) EZQ_CK(cudaMemcpyAsync(tr.data(), dtr, sizeof(double) * ntr, cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    res->scale = static_cast<float>(o[0]);
    res->initial_error = o[1];
    res->final_error = o[2];
    res->best_step = static_cast<int32_t>(o[3]);
    res->best_scale = o[4];
    res->best_error = o[5];
    res->n_trace = keep_trace ? steps + 1 : 0;
    if (keep_trace) {
        for (int t = 0; t <= steps; ++t) {
            if (trace_step) trace_step[t] = t;
            if (trace_scale) trace_scale[t] = tr[2 * t];
            if (trace_error) trace_error[t] = tr[2 * t + 1];
        }
    }
    return clear_error();
}

int ezq_brute_force_scale(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                          const ezq_config* cfg, int grid_points, double* scale, double* error) {
    if (grid_points < 2) return set_error(EZQ_ERR_INVALID_ARGUMENT, "grid_points must be >= 2");
    const std::vector<float> v = gather(x, n, mask, n_mask);
    if (v.empty()) {
        *scale = 1.0;
        *error = 0.0;
        return clear_error();
    }
    // optimize.cpp:199-211: uniform grid over [s0/8, 1.25 s0] plus s0.
    const double s0 = ezq_initial_scale(v.data(), static_cast<int64_t>(v.size()), cfg);
    const double lo = s0 / 8.0;
    const double hi = s0 * 1.25;
    std::vector<double> grid;
    grid.reserve(static_cast<size_t>(grid_points) + 1);
    for (int i = 0; i < grid_points; ++i)
        grid.push_back(lo + (hi - lo) * static_cast<double>(i) / static_cast<double>(grid_points - 1));
    grid.push_back(s0);
    std::sort(grid.begin(), grid.end());
    grid.erase(std::unique(grid.begin(), grid.end()), grid.end());
    std::vector<double> err;
    if (int s = eval_scales(v, grid, cfg, err, nullptr)) return s;
    size_t best = 0;  // ascending scan, strict improvement (optimize.cpp:225-227)
    for (size_t i = 1; i < grid.size(); ++i)
        if (err[i] < err[best]) best = i;
    *scale = grid[best];
    *error = err[best];
    return clear_error();
}

int ezq_quantize_channel(const float* x, int64_t n, double scale, const ezq_config* cfg,
                         int16_t* levels) {
    if (!(scale > 0.0) || !std::isfinite(scale)) return scale_error(scale);  // rtn.cpp:89
    if (n == 0) return clear_error();
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = thread_stream(dev);
    Arena ar;
    ar.reserve(sizeof(float) * n);
    ar.reserve(sizeof(int16_t) * n);
    if (int s = ar.allocate(st)) return s;
    float* dx = ar.take<float>(n);
    int16_t* dl = ar.take<int16_t>(n);
    EZQ_CK(cudaMemcpyAsync(dx, x, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    launch_quantize_channel(dx, n, scale, make_cfg(cfg, EZQ_MODE_EASYQUANT, nullptr), dl, st);
    EZQ_CK(cudaGetLastError());
    EZQ_CK(cudaMemcpyAsync(levels, dl, sizeof(int16_t) * n, cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    return clear_error();
}

}  // extern "C"
