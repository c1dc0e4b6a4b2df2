/*
 * ezq_oracle.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the EasyQuant reference hot path
 * (/root/reference/proj/src/{stats,outliers,rtn,optimize,pipeline}.cpp and
 * include/ezquant/rng.hpp), used by tests/ as the parity oracle, by
 * __graft_entry__.smoke() as the checker and by bench.py's cpu_baseline leg.
 * Each function cites the reference lines it restates. Pinned against the
 * reference's own known-answer tests and against oracle/_ref (the reference
 * compiled from its sources) -- see tests/test_oracle.py.
 *
 * Build: oracle/Makefile -> oracle/build/libezq_oracle.so (gcc -O2
 * -ffp-contract=off, the reference's non-contracted double arithmetic).
 */
#ifndef EZQ_ORACLE_H
#define EZQ_ORACLE_H

#include <stdint.h>

#include "../include/ezquant_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:11-68 (xoshiro256++ / splitmix64 / Box-Muller) -------------- */
typedef struct ezqo_rng {
    uint64_t s[4];
    double spare;
    int has_spare;
} ezqo_rng;
void ezqo_rng_init(ezqo_rng* r, uint64_t seed);
uint64_t ezqo_rng_next(ezqo_rng* r);
double ezqo_rng_uniform(ezqo_rng* r);
int64_t ezqo_rng_uniform_int(ezqo_rng* r, int64_t lo, int64_t hi);
double ezqo_rng_gaussian(ezqo_rng* r);
/* gaussian_matrix recipe of the reference tests (e.g. acceptance.cpp:61-66). */
void ezqo_gaussian(float* out, int64_t n, uint64_t seed, double scale);
/* plant_outliers recipe (acceptance.cpp:92-102). Returns 0, -1 on OOM. */
int ezqo_plant_outliers(float* W, int64_t n, int64_t count, double lo, double hi, uint64_t seed);

/* ---- stats.cpp:27-100 ---------------------------------------------------- */
void ezqo_tensor_stats(const float* W, int64_t n, double* mean, double* stddev, double* max_abs);

/* ---- outliers.cpp:18-61: returns the count; arrays filled when non-null -- */
int64_t ezqo_detect_outliers(const float* W, int64_t rows, int64_t cols, float sigma_n,
                             ezq_outlier* out, double* mean, double* stddev);

/* ---- rtn.cpp / optimize.cpp channel functions ---------------------------- */
double ezqo_initial_scale(const float* x, int64_t n, int bits);
int ezqo_level_of(double x, double inv_s, int lmin, int lmax);
void ezqo_eval_dense(const float* x, int64_t n, double s, int lmin, int lmax, double* err,
                     double* grad);
double ezqo_adam_step(double* m, double* v, int64_t* t, double scale, double grad,
                      const ezq_config* cfg);
/* optimize_channel_range over already-gathered normals; trace (steps+1
 * scale/error pairs) optional. Returns the stored f32 scale. */
float ezqo_optimize_channel(const float* v, int64_t n, const ezq_config* cfg, double* initial_error,
                            double* final_error, int* best_step, double* trace_scale,
                            double* trace_error);
void ezqo_brute_force(const float* v, int64_t n, const ezq_config* cfg, int grid_points,
                      double* scale, double* error);

/* ---- pipeline.cpp:29-115: full tensor quantization ------------------------
 * packed: packed_size(rows*cols, bits) bytes; scales: cols floats; outliers:
 * capacity `cap` entries. Returns the outlier count (> cap: nothing written
 * to outliers, call again), or -1 (non-finite input), -2 (invariant
 * violated), -3 (bad config). threads: OpenMP threads for the column loop
 * (results are identical for any count). */
int64_t ezqo_quantize(const float* W, int64_t rows, int64_t cols, const ezq_config* cfg, int mode,
                      int threads, uint8_t* packed, float* scales, ezq_outlier* outliers,
                      int64_t cap, double* mean, double* stddev, double* rtn_error,
                      double* final_error);

/* ---- pipeline.cpp:117-142 + rtn.cpp:151-182 + outliers.cpp:106-114 ------- */
int ezqo_dequantize(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                    const float* scales, const ezq_outlier* outliers, int64_t n_out, float* out);

/* ---- rtn.cpp:34-77 (skip list given as (row, col) pairs) ----------------- */
double ezqo_reconstruction_error(const float* a, const float* b, int64_t rows, int64_t cols,
                                 const ezq_outlier* skip, int64_t n_skip);

/* ---- rtn.cpp:119-182 ------------------------------------------------------ */
int64_t ezqo_packed_size(int64_t count, int bits);
int ezqo_pack_levels(const int16_t* levels, int64_t n, int bits, uint8_t* out);
int ezqo_unpack_levels(const uint8_t* bytes, int64_t nbytes, int64_t count, int bits,
                       int16_t* out);

/* fp32 matrix-vector reference for the GEMV parity tests (fp64 accumulate):
 * y[b, j] = sum_i x[b, i] * What[i, j]. */
void ezqo_gemv_f64(const float* What, int64_t rows, int64_t cols, const float* x, int batch,
                   double* y);

#ifdef __cplusplus
}
#endif

#endif
