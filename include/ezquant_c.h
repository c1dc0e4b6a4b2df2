/*
 * ezquant_c.h — C-ABI of the B200-native EasyQuant engine (the drop-in
 * boundary). Plain pointers and sizes only; no C++ or torch types.
 *
 * Every entry point replaces one function of the reference's public C++ API
 * (/root/reference/proj/include/ezquant/ headers, cited per function). The
 * C++ drop-in in include/ezquant/ (implemented by libezquant.so) is a thin
 * shim over these functions that maps status codes back onto the exact
 * reference exception types; INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Execution: tensor- and channel-scale work runs on the current CUDA device
 * (hand-written sm_100a kernels). There is NO CPU fallback: without a usable
 * device every compute entry point returns EZQ_ERR_NO_DEVICE.
 *
 * Threading: all entry points are reentrant. Each calling host thread gets
 * its own CUDA stream per device (or uses the `stream` argument when it is
 * non-null; pass cudaStreamLegacy, i.e. (void*)1, for the legacy default
 * stream) and its own last-error slot.
 */
#ifndef EZQUANT_C_H
#define EZQUANT_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception type -------------------- */
#define EZQ_OK 0
#define EZQ_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument                 */
#define EZQ_ERR_INVARIANT 2        /* ezquant::invariant_error (error.hpp:31) */
#define EZQ_ERR_IO_FAILURE 3       /* io_error{IoFailure}      (error.hpp:10) */
#define EZQ_ERR_IO_FORMAT 4        /* io_error{FormatViolation}               */
#define EZQ_ERR_IO_VERSION 5       /* io_error{VersionMismatch}               */
#define EZQ_ERR_CUDA 10            /* device-side failure                     */
#define EZQ_ERR_NO_DEVICE 11       /* no CUDA device: no CPU fallback exists  */
#define EZQ_ERR_OOM 12             /* device allocation failed                */

/* ---- memory spaces for pointer arguments --------------------------------- */
#define EZQ_MEM_HOST 0
#define EZQ_MEM_DEVICE 1

/* ---- quantization modes (pipeline.hpp:12-19, same numbering) ------------- */
#define EZQ_MODE_EASYQUANT 0
#define EZQ_MODE_RTN 1
#define EZQ_MODE_OUTLIERS_ONLY 2

/* ---- selection policies (types.hpp:31-34) -------------------------------- */
#define EZQ_SELECT_BEST 0
#define EZQ_SELECT_FIXED 1

/* QuantConfig (types.hpp:37-54). Defaults: ezq_config_default(). */
typedef struct ezq_config {
    int32_t bits;       /* k in [2, 8]                                   */
    float sigma_n;      /* outlier threshold multiplier, >= 0           */
    double lr;          /* Adam learning rate                            */
    double beta1;       /* Adam beta1                                    */
    double beta2;       /* Adam beta2                                    */
    double eps;         /* Adam epsilon                                  */
    int32_t steps;      /* optimisation steps, >= 0                      */
    int32_t select;     /* EZQ_SELECT_*                                  */
    int32_t select_step;
    int32_t reserved;
    uint64_t seed;
} ezq_config;

/* TensorStats (types.hpp:58-63). */
typedef struct ezq_stats {
    double mean;
    double stddev; /* population standard deviation */
    double max_abs;
    int64_t count;
} ezq_stats;

/* OutlierEntry (types.hpp:76-82): 12 bytes, same layout as the .ezqt record. */
typedef struct ezq_outlier {
    uint32_t row;
    uint32_t col;
    float value;
} ezq_outlier;

/* QuantizedWeight (types.hpp:103-113) plus the detection statistics of
 * OutlierSet (types.hpp:87-96). Arrays live in `mem` and are owned by the
 * library (free with ezq_qweight_free) unless built by ezq_qweight_wrap. */
typedef struct ezq_qweight {
    int64_t rows;
    int64_t cols;
    int32_t bits;
    int32_t mem;            /* EZQ_MEM_* of the arrays below            */
    int64_t packed_bytes;   /* packed_size(rows*cols, bits)             */
    uint8_t* packed;        /* k=4 nibbles (low = even flat index) or bytes */
    float* scales;          /* [cols]                                   */
    int64_t n_outliers;
    ezq_outlier* outliers;  /* sorted by (row, col)                     */
    double mean;            /* detection-time statistics                */
    double stddev;
    float sigma_n;
    int32_t has_errors;     /* rtn_error / final_error valid            */
    double rtn_error;       /* masked error at the initial scales       */
    double final_error;     /* masked error at the stored scales        */
    int32_t owned;          /* library owns the arrays                  */
    int32_t reserved;
} ezq_qweight;

/* OptimizeResult + OptimizeTrace (optimize.hpp:46-76). */
typedef struct ezq_opt_result {
    float scale;
    int32_t best_step;
    double initial_error;
    double final_error;
    double best_scale;
    double best_error;
    int32_t n_trace; /* points written to the trace arrays (0 if not kept) */
    int32_t reserved;
} ezq_opt_result;

/* ---- library / device ------------------------------------------------------ */
void ezq_config_default(ezq_config* cfg);
/* QuantConfig::validate (types.cpp:23-40). */
int ezq_config_validate(const ezq_config* cfg);
/* Last status of this thread, its message, and (for non-finite inputs and
 * bad coordinates) the offending flat index / entry index, else -1. */
int ezq_last_error(char* msg, size_t cap, int64_t* index);
int ezq_device_count(int* n);
/* Selects the device used by the calling thread (default: current device). */
int ezq_set_device(int device);
/* Blocks until all work issued by this thread on its stream has finished. */
int ezq_synchronize(void);
const char* ezq_version(void);
/* Number of kernels launched by this process (instrumentation for bench). */
int64_t ezq_kernel_launches(void);
/* Cumulative count of columns whose Adam-step selection was a near-tie the
 * exact evaluation could not certify against the reference's sequential fp64
 * sums, re-evaluated in reference order; `fallback`: of those, columns that
 * ran the whole reference loop (candidate slots overflowed). */
int ezq_tie_stats(int64_t* resolved, int64_t* fallback);

/* ---- instrumentation (bench / profiling) ------------------------------------ */
/* When enabled, every kernel launch of the named families is bracketed by
 * CUDA events on its own stream; ezq_profile_read synchronizes them and
 * returns the summed device time, launch count and algorithmic work (flop for
 * "qrange", bytes for the HBM-bound families). Families: "stats", "detect",
 * "qrange", "seqerr", "pack", "dequant", "gemv". */
int ezq_profile_enable(int on);
int ezq_profile_read(const char* family, double* ms, int64_t* launches, double* work);
/* FP64 DFMA peak of the current device (TFLOP/s), measured by a microkernel. */
int ezq_measure_fp64_peak(double* tflops);

/* ---- tensor statistics (stats.hpp:14-20; stats.cpp:27-108) ----------------- */
/* Bit-exact with the reference: 8192-element fp64 chunks, chunk-ordered merge.
 * `W` is host or device memory per `mem`. Also runs DenseMatrix::validate's
 * finiteness scan (types.cpp:17-20). */
int ezq_tensor_stats(const float* W, int64_t rows, int64_t cols, int mem, void* stream,
                     ezq_stats* out);

/* ---- outlier detection (outliers.hpp:15-38; outliers.cpp:29-73) ----------- */
/* Entries are returned in host memory allocated by the library (ezq_free). */
int ezq_detect_outliers(const float* W, int64_t rows, int64_t cols, const ezq_config* cfg,
                        int mem, void* stream, ezq_outlier** entries, int64_t* n,
                        double* mean, double* stddev);

/* ---- whole-tensor pipeline (pipeline.hpp:33-49; pipeline.cpp:65-115) ------- */
/* quantize_tensor / easyquant_tensor / rtn_tensor. `in_mem` says where W
 * lives, `out_mem` where the returned arrays should live. */
int ezq_quantize_tensor(const float* W, int64_t rows, int64_t cols, const ezq_config* cfg,
                        int mode, int in_mem, int out_mem, void* stream, ezq_qweight** out);
/* Batched form used by the whole-model driver: n independent tensors with
 * one config, grouped into shared kernel launches (model.cpp:154-192 runs the
 * same per-tensor calls on a worker pool). outs[i] receives tensor i. On the
 * first failing tensor the call stops and returns its status; `failed_index`
 * (nullable) receives its index. */
int ezq_quantize_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                       const ezq_config* cfg, int mode, int in_mem, int out_mem, void* stream,
                       ezq_qweight** outs, int* failed_index);
/* sigma_sweep's device loop (report.cpp:241-284): one EASYQUANT batch per
 * sigma_n over the same tensors; per point and tensor (point-major,
 * [nsig][n]) the outlier count, rtn_error and final_error (0 for tensors
 * without errors, as the reference's rows). With device-resident inputs the
 * tensor stats (K1) are computed by the first point only -- they do not
 * depend on sigma_n -- and reused, bit-identically, by the others. */
int ezq_sigma_sweep_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                          const ezq_config* cfg, int in_mem, void* stream, const float* sigmas, int nsig,
                          int64_t* n_outliers, double* rtn_error, double* final_error, int* failed_index);
/* brute_force_optimal_scale (optimize.cpp:186-229) for every column of a
 * batch, on the device: the reference's grid (grid_points scales in
 * [s0/8, 1.25 s0] plus s0) over each column's normals (outliers isolated
 * exactly as ezq_quantize_batch does). best_scale / best_error receive one
 * double per column, tensors in order. The errors are the exact values of the
 * grid objective (not the reference's sequential fp64 sums), so an argmin can
 * differ from the reference's only between near-equal grid points. k <= 5,
 * rows <= 65536. */
int ezq_grid_oracle_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                          const ezq_config* cfg, int grid_points, int in_mem, void* stream, double* best_scale,
                          double* best_error, int* failed_index);
/* dequantize_tensor (pipeline.cpp:117-142): unpack, rescale
 * float(double(s_j) * l), scatter outliers. `q` arrays may be host or device
 * (q->mem); `out` is rows*cols floats in `out_mem`. */
int ezq_dequantize_tensor(const ezq_qweight* q, float* out, int out_mem, void* stream);
/* Wraps caller-owned arrays (no copy) so they can be passed to
 * ezq_dequantize_tensor / ezq_gemv; ezq_qweight_free releases only the struct. */
int ezq_qweight_wrap(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                     int64_t packed_bytes, const float* scales, int64_t n_scales,
                     const ezq_outlier* outliers, int64_t n_outliers, double mean,
                     double stddev, float sigma_n, int mem, ezq_qweight** out);
void ezq_qweight_free(ezq_qweight* q);
/* Host copy (library-owned) of a device-resident artifact. */
int ezq_qweight_to_host(const ezq_qweight* q, ezq_qweight** out);
void ezq_free(void* p);

/* reconstruction_error (rtn.hpp:34-44; rtn.cpp:34-77): per-column sequential
 * fp64 sums merged in column order; coordinates in skip_rows/skip_cols
 * (nullable, n_skip entries) are excluded. */
int ezq_reconstruction_error(const float* a, const float* b, int64_t rows, int64_t cols,
                             const uint32_t* skip_rows, const uint32_t* skip_cols,
                             int64_t n_skip, int mem, void* stream, double* out);

/* ---- channel-scale entry points (optimize.hpp:20-95; rtn.hpp:14-30) ------- */
/* Host spans in, host results out; the work runs on the device with the
 * reference's sequential summation order, so results are bit-exact. */
int ezq_channel_eval(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                     double scale, const ezq_config* cfg, double* error, double* gradient);
/* optimize_channel_range; trace arrays (nullable) hold cfg->steps+1 points. */
int ezq_optimize_channel(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                         const ezq_config* cfg, int keep_trace, ezq_opt_result* res,
                         int32_t* trace_step, double* trace_scale, double* trace_error);
int ezq_brute_force_scale(const float* x, int64_t n, const uint32_t* mask, int64_t n_mask,
                          const ezq_config* cfg, int grid_points, double* scale, double* error);
int ezq_quantize_channel(const float* x, int64_t n, double scale, const ezq_config* cfg,
                         int16_t* levels);

/* ---- host scalar utilities (no meaningful GPU work; rtn.cpp, optimize.cpp) -- */
double ezq_initial_scale(const float* x, int64_t n, const ezq_config* cfg);
int ezq_adam_step(double* m, double* v, int64_t* t, double scale, double grad,
                  const ezq_config* cfg, double* out_scale);
int64_t ezq_packed_size(int64_t count, int bits);
int ezq_pack_levels(const int16_t* levels, int64_t n, int bits, uint8_t* out);
int ezq_unpack_levels(const uint8_t* bytes, int64_t n_bytes, int64_t count, int bits,
                      int16_t* out);
int ezq_dequantize_channel(const int16_t* levels, int64_t n, double scale, float* out);

/* ---- device buffers (for C/C++ callers without the CUDA runtime) ---------- */
/* Copies n floats from host memory into a new device buffer on the calling
 * thread's device; free with ezq_device_free. */
int ezq_device_upload(const float* host, int64_t n, float** dev);
void ezq_device_free(void* dev);
int ezq_device_mem_info(size_t* free_bytes, size_t* total_bytes);

/* ---- .ezqt container (io.hpp:48-66; io.cpp:221-354) ------------------------ */
/* encode_quantized: host artifact -> the reference's exact bytes (malloc'd;
 * free with ezq_free). Validation order and messages follow io.cpp:222-263;
 * failures are EZQ_ERR_INVALID_ARGUMENT. */
int ezq_encode_quantized(const ezq_qweight* q, uint8_t** out, int64_t* len);
/* decode_quantized: bytes -> library-owned host artifact. Failures are
 * EZQ_ERR_IO_FORMAT / EZQ_ERR_IO_VERSION with the byte offset the reference
 * reports in ezq_last_error's index (EZQ_ERR_INVALID_ARGUMENT for a k != 4
 * payload byte outside the level span, as unpack_levels). */
int ezq_decode_quantized(const uint8_t* bytes, int64_t len, ezq_qweight** out);

/* ---- fused dequant + outlier GEMV / skinny GEMM (new) ----- */
/* y[b, j] = sum_i x[b, i] * What[i, j] with What the dequantized `q`
 * (rows = in features, cols = out features). x: [batch, rows] (dtype 0 = f32,
 * 1 = bf16, 2 = f16), y: [batch, cols] f32. All pointers device memory;
 * q must be device-resident (ezq_gemv_prepare builds the CSR view). */
typedef struct ezq_gemv_plan ezq_gemv_plan;
int ezq_gemv_prepare(const ezq_qweight* q, void* stream, ezq_gemv_plan** plan);
/* Same, with the outlier values stored as f32 (exact, 8 bytes per outlier
 * with the u32 row) or f16 (6 bytes per outlier, round to nearest even; the
 * GEMV stays within its 1e-3 gate). */
#define EZQ_GEMV_OUTLIER_F32 0
#define EZQ_GEMV_OUTLIER_F16 1
int ezq_gemv_prepare_ex(const ezq_qweight* q, int outlier_dtype, void* stream, ezq_gemv_plan** plan);
int ezq_gemv(const ezq_gemv_plan* plan, const void* x, int x_dtype, int batch, float* y,
             void* stream);
void ezq_gemv_plan_free(ezq_gemv_plan* plan);

/* ---- dense 3-bit codes (new -- the reference stores k = 3
 * one offset byte per level, rtn.cpp:119-147) ------------------------------ */
/* Layout: the level offsets (level - lmin, 0..7) in flat row-major order as
 * one little-endian bit stream, element e at bits 3e..3e+2: 8 levels per 3
 * bytes, 3 * ceil(count / 8) bytes, zero tail bits. Buffers are all host or
 * all device memory (`mem`). */
int64_t ezq_dense3_size(int64_t count);
/* The reference's k = 3 payload (one offset byte per level, as pack_levels
 * writes it) -> dense stream. A byte > 7 fails like unpack_levels
 * (EZQ_ERR_INVALID_ARGUMENT, the element index in ezq_last_error). */
int ezq_pack_dense3(const uint8_t* levels, int64_t count, uint8_t* out, int mem, void* stream);
/* Dense stream -> one offset byte per level (the reference's k = 3 payload). */
int ezq_unpack_dense3(const uint8_t* dense, int64_t count, uint8_t* out, int mem, void* stream);
/* dequantize_tensor (pipeline.cpp:117-142) of a 3-bit artifact whose codes
 * are given as a dense stream (`dense`, in q->mem; q->packed is not read):
 * bit-identical to ezq_dequantize_tensor on the byte-per-level codes. */
int ezq_dequantize_dense3(const ezq_qweight* q, const uint8_t* dense, float* out, int out_mem, void* stream);
/* ezq_gemv_prepare_ex for a device-resident 3-bit artifact whose codes are a
 * dense stream (device memory); the plan is the one the byte codes give. */
int ezq_gemv_prepare_dense3(const ezq_qweight* q, const uint8_t* dense, int outlier_dtype, void* stream,
                            ezq_gemv_plan** plan);

#ifdef __cplusplus
}
#endif

#endif /* EZQUANT_C_H */
