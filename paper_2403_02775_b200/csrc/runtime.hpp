// Host runtime shared by the C-ABI translation units: per-thread error slot,
// per-thread/per-device streams, device properties, a bump arena over
// stream-ordered device allocations, and QuantConfig validation.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ezquant_c.h"
#include "ezq_kernels.cuh"

namespace ezq {

int set_error(int code, const std::string& msg, int64_t index = -1);
int clear_error();
int cuda_error(cudaError_t e, const char* where);

#define EZQ_CK(expr)                                                \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return ::ezq::cuda_error(_e, #expr); \
    } while (0)

// Binds the calling thread's device; EZQ_ERR_NO_DEVICE when none exists.
int bind_device(int* dev);
cudaStream_t thread_stream(int dev);
cudaStream_t copy_stream(int dev);  // per-thread second stream for H2D staging
cudaStream_t d2h_stream(int dev);   // per-thread stream for deferred artifact copies
inline cudaStream_t pick_stream(void* user, int dev) {
    return user ? static_cast<cudaStream_t>(user) : thread_stream(dev);
}

struct DeviceInfo {
    int sms = 0;
    int max_smem_optin = 0;
    int smem_per_sm = 0;
    size_t total_mem = 0;
};
const DeviceInfo& device_info(int dev);

// QuantConfig::validate (types.cpp:23-40); returns status + message.
int validate_config(const ezq_config* cfg, std::string* msg);

// Builds the device-side config; the bias-correction tables must be uploaded
// by the caller into `bc` (4 * (steps + 1) doubles: bc1, bc2, 1/bc1, 1/bc2).
CfgDev make_cfg(const ezq_config* cfg, int mode, const double* bc_dev);
void bias_tables(const ezq_config* cfg, std::vector<double>& host);  // bc1 | bc2

// Recycled device scratch (see runtime.cpp): block_get waits on the block's
// last use; block_put records it on `st`.
void* block_get(size_t need, cudaStream_t st, size_t* got);
void block_put(void* p, size_t bytes, cudaStream_t st);

// Bump allocator over one recycled device block.
class Arena {
public:
    // Every take() realigns to 256 bytes; reserve() must be called once per
    // take() (or with enough slack) -- take() reports overflow via ok().
    void reserve(size_t bytes) { need_ += ((bytes + 255) & ~static_cast<size_t>(255)) + 256; }
    template <class T>
    void reserve_n(size_t count) {
        reserve(count * sizeof(T));
    }
    bool ok() const { return off_ <= need_; }
    int allocate(cudaStream_t st);
    template <class T>
    T* take(size_t count) {
        off_ = (off_ + 255) & ~static_cast<size_t>(255);
        T* p = reinterpret_cast<T*>(base_ + off_);
        off_ += count * sizeof(T);
        return off_ <= need_ ? p : nullptr;
    }
    void release(cudaStream_t st);
    ~Arena();

private:
    char* base_ = nullptr;
    size_t need_ = 0, off_ = 0, cap_ = 0;
    cudaStream_t owner_ = nullptr;
};

std::string fmt_double(double v);  // std::to_string(double) formatting

// EZQ_TRACE=1: host-side timestamps of the pipeline phases on stderr.
bool trace_on();
void trace(const char* what, long long a = -1);

// Pinned host memory for library-owned host outputs: blocks are recycled by
// exact size (repeat calls on the same shapes reuse them), so D2H copies run
// at full PCIe rate and asynchronously. host_free() accepts only pointers
// from host_alloc().
void* host_alloc(size_t bytes);
void host_free(void* p);

}  // namespace ezq
