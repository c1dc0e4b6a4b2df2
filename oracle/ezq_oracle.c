/*
 * ezq_oracle.c -- TEST INFRASTRUCTURE ONLY. Plain-C restatement of the
 * EasyQuant reference hot path; see ezq_oracle.h. Compiled with
 * -ffp-contract=off: every double operation below rounds exactly like the
 * reference's baseline x86-64 build (no FMA).
 */
#include "ezq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================= rng.hpp:11-68 ================================== */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void ezqo_rng_init(ezqo_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) { /* splitmix64 (rng.hpp:13-21) */
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        r->s[i] = z ^ (z >> 31);
    }
    r->spare = 0.0;
    r->has_spare = 0;
}

uint64_t ezqo_rng_next(ezqo_rng* r) { /* xoshiro256++ (rng.hpp:24-34) */
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

double ezqo_rng_uniform(ezqo_rng* r) { return (double)(ezqo_rng_next(r) >> 11) * 0x1.0p-53; }

int64_t ezqo_rng_uniform_int(ezqo_rng* r, int64_t lo, int64_t hi) { /* rng.hpp:42-45 */
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(ezqo_rng_next(r) % span);
}

double ezqo_rng_gaussian(ezqo_rng* r) { /* rng.hpp:48-60 */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - ezqo_rng_uniform(r);
    const double u2 = ezqo_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(th);
    r->has_spare = 1;
    return rad * cos(th);
}

void ezqo_gaussian(float* out, int64_t n, uint64_t seed, double scale) {
    ezqo_rng r;
    ezqo_rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(ezqo_rng_gaussian(&r) * scale);
}

int ezqo_plant_outliers(float* W, int64_t n, int64_t count, double lo, double hi, uint64_t seed) {
    uint8_t* used = (uint8_t*)calloc((size_t)((n + 7) / 8), 1);
    if (!used) return -1;
    ezqo_rng r;
    ezqo_rng_init(&r, seed);
    int64_t have = 0;
    while (have < count) { /* acceptance.cpp:92-102: distinct flat indices */
        const int64_t flat = ezqo_rng_uniform_int(&r, 0, n - 1);
        if (used[flat >> 3] & (1u << (flat & 7))) continue;
        used[flat >> 3] |= (uint8_t)(1u << (flat & 7));
        ++have;
        const double mag = lo + (hi - lo) * ezqo_rng_uniform(&r);
        W[flat] = (float)(ezqo_rng_uniform(&r) < 0.5 ? -mag : mag);
    }
    free(used);
    return 0;
}

/* ======================= stats.cpp:27-100 ================================ */
#define EZQO_CHUNK 8192 /* stats.cpp:18 */

void ezqo_tensor_stats(const float* W, int64_t n, double* mean, double* stddev, double* max_abs) {
    *mean = *stddev = *max_abs = 0.0;
    if (n <= 0) return;
    const int64_t chunks = (n + EZQO_CHUNK - 1) / EZQO_CHUNK;
    double sum = 0.0, mabs = 0.0;
    float mn = W[0], mx = W[0];
    for (int64_t c = 0; c < chunks; ++c) { /* sum_chunk, merged in chunk order */
        const int64_t lo = c * EZQO_CHUNK;
        const int64_t cnt = (n - lo) < EZQO_CHUNK ? (n - lo) : EZQO_CHUNK;
        double cs = 0.0, cm = 0.0;
        float cmn = W[lo], cmx = W[lo];
        for (int64_t i = 0; i < cnt; ++i) {
            const double v = (double)W[lo + i];
            cs += v;
            const double a = fabs(v);
            cm = (cm < a) ? a : cm;
            cmn = (W[lo + i] < cmn) ? W[lo + i] : cmn;
            cmx = (cmx < W[lo + i]) ? W[lo + i] : cmx;
        }
        sum += cs;
        mabs = (mabs < cm) ? cm : mabs;
        mn = (cmn < mn) ? cmn : mn;
        mx = (mx < cmx) ? cmx : mx;
    }
    *max_abs = mabs;
    if (mn == mx) { /* constant tensor (stats.cpp:77-83) */
        *mean = (double)mn;
        *stddev = 0.0;
        return;
    }
    const double m = sum / (double)n;
    double ss = 0.0;
    for (int64_t c = 0; c < chunks; ++c) { /* dev_chunk (stats.cpp:40-48) */
        const int64_t lo = c * EZQO_CHUNK;
        const int64_t cnt = (n - lo) < EZQO_CHUNK ? (n - lo) : EZQO_CHUNK;
        double acc = 0.0;
        for (int64_t i = 0; i < cnt; ++i) {
            const double dv = (double)W[lo + i] - m;
            acc += dv * dv;
        }
        ss += acc;
    }
    *mean = m;
    *stddev = sqrt(ss / (double)n);
}

/* ======================= outliers.cpp:18-61 ============================== */
int64_t ezqo_detect_outliers(const float* W, int64_t rows, int64_t cols, float sigma_n,
                             ezq_outlier* out, double* mean, double* stddev) {
    double mabs;
    ezqo_tensor_stats(W, rows * cols, mean, stddev, &mabs);
    if (*stddev == 0.0) return 0;
    const double thr = (double)sigma_n * *stddev;
    int64_t k = 0;
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            const float v = W[i * cols + j];
            if (fabs((double)v - *mean) >= thr) {
                if (out) {
                    out[k].row = (uint32_t)i;
                    out[k].col = (uint32_t)j;
                    out[k].value = v;
                }
                ++k;
            }
        }
    return k;
}

/* ======================= rtn.cpp / optimize.cpp ========================== */
double ezqo_initial_scale(const float* x, int64_t n, int bits) { /* rtn.cpp:81-86 */
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs((double)x[i]);
        m = (m < a) ? a : m;
    }
    if (m == 0.0) return 1.0;
    return m / (double)(1 << (bits - 1));
}

int ezqo_level_of(double x, double inv_s, int lmin, int lmax) { /* rtn.cpp:27-32 */
    const double u = x * inv_s;
    if (u >= (double)lmax) return lmax;
    if (u <= (double)lmin) return lmin;
    return (int)llround(u);
}

void ezqo_eval_dense(const float* x, int64_t n, double s, int lmin, int lmax, double* err,
                     double* grad) { /* optimize.cpp:30-51 */
    const double inv = 1.0 / s;
    double e = 0.0, g = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double xi = (double)x[i];
        const double q = (double)ezqo_level_of(xi, inv, lmin, lmax);
        const double d = s * q - xi;
        e += d * d;
        g += d * q;
    }
    *err = e;
    *grad = 2.0 * g;
}

static double snap(double s) { /* optimize.cpp:79-82 */
    const double v = (double)(float)s;
    return v < 1e-12 ? 1e-12 : v;
}

double ezqo_adam_step(double* m, double* v, int64_t* t, double scale, double grad,
                      const ezq_config* c) { /* optimize.cpp:86-94 */
    *t += 1;
    *m = c->beta1 * *m + (1.0 - c->beta1) * grad;
    *v = c->beta2 * *v + (1.0 - c->beta2) * grad * grad;
    const double mh = *m / (1.0 - pow(c->beta1, (double)*t));
    const double vh = *v / (1.0 - pow(c->beta2, (double)*t));
    const double upd = scale - c->lr * mh / (sqrt(vh) + c->eps);
    return upd < 1e-12 ? 1e-12 : upd;
}

float ezqo_optimize_channel(const float* v, int64_t n, const ezq_config* c, double* initial_error,
                            double* final_error, int* best_step, double* trace_scale,
                            double* trace_error) { /* optimize.cpp:118-184 */
    *initial_error = *final_error = 0.0;
    *best_step = 0;
    if (n == 0) return 1.0f;
    const int lmin = 1 - (1 << (c->bits - 1)), lmax = 1 << (c->bits - 1);
    double s = snap(ezqo_initial_scale(v, n, c->bits));
    double err, grad;
    ezqo_eval_dense(v, n, s, lmin, lmax, &err, &grad);
    *initial_error = err;
    if (trace_scale) {
        trace_scale[0] = s;
        trace_error[0] = err;
    }
    const double s0 = s, e0 = err;
    double best_e = err, best_s = s, fixed_s = s, fixed_e = err;
    const int fixed_at = c->select_step < c->steps ? c->select_step : c->steps;
    double m = 0.0, vv = 0.0;
    int64_t t = 0;
    for (int step = 1; step <= c->steps; ++step) {
        s = snap(ezqo_adam_step(&m, &vv, &t, s, grad, c));
        ezqo_eval_dense(v, n, s, lmin, lmax, &err, &grad);
        if (trace_scale) {
            trace_scale[step] = s;
            trace_error[step] = err;
        }
        if (err < best_e) {
            best_e = err;
            best_s = s;
            *best_step = step;
        }
        if (step == fixed_at) {
            fixed_s = s;
            fixed_e = err;
        }
    }
    if (c->select == EZQ_SELECT_FIXED) {
        if (fixed_e <= e0) {
            *final_error = fixed_e;
            return (float)fixed_s;
        }
        *final_error = e0;
        return (float)s0;
    }
    *final_error = best_e;
    return (float)best_s;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

void ezqo_brute_force(const float* v, int64_t n, const ezq_config* c, int grid_points,
                      double* scale, double* error) { /* optimize.cpp:186-229 */
    *scale = 1.0;
    *error = 0.0;
    if (n == 0 || grid_points < 2) return;
    const int lmin = 1 - (1 << (c->bits - 1)), lmax = 1 << (c->bits - 1);
    const double s0 = ezqo_initial_scale(v, n, c->bits);
    const double lo = s0 / 8.0, hi = s0 * 1.25;
    double* grid = (double*)malloc(sizeof(double) * (size_t)(grid_points + 1));
    int g = 0;
    for (int i = 0; i < grid_points; ++i)
        grid[g++] = lo + (hi - lo) * (double)i / (double)(grid_points - 1);
    grid[g++] = s0;
    qsort(grid, (size_t)g, sizeof(double), cmp_double);
    int u = 0;
    for (int i = 0; i < g; ++i)
        if (u == 0 || grid[i] != grid[u - 1]) grid[u++] = grid[i];
    double best_e = 0.0, gr;
    int best = 0;
    for (int i = 0; i < u; ++i) {
        double e;
        ezqo_eval_dense(v, n, grid[i], lmin, lmax, &e, &gr);
        if (i == 0 || e < best_e) {
            best_e = e;
            best = i;
        }
    }
    *scale = grid[best];
    *error = best_e;
    free(grid);
}

/* ======================= rtn.cpp:119-182 ================================= */
int64_t ezqo_packed_size(int64_t count, int bits) { return bits == 4 ? (count + 1) / 2 : count; }

int ezqo_pack_levels(const int16_t* lv, int64_t n, int bits, uint8_t* out) {
    const int lmin = 1 - (1 << (bits - 1)), lmax = 1 << (bits - 1);
    for (int64_t i = 0; i < n; ++i)
        if (lv[i] < lmin || lv[i] > lmax) return -1;
    memset(out, 0, (size_t)ezqo_packed_size(n, bits));
    for (int64_t i = 0; i < n; ++i) {
        const uint8_t off = (uint8_t)(lv[i] - lmin);
        if (bits != 4)
            out[i] = off;
        else if (i % 2 == 0)
            out[i / 2] = off; /* earlier element, low nibble */
        else
            out[i / 2] |= (uint8_t)(off << 4);
    }
    return 0;
}

int ezqo_unpack_levels(const uint8_t* b, int64_t nbytes, int64_t count, int bits, int16_t* out) {
    if (count < 0 || nbytes < ezqo_packed_size(count, bits)) return -1;
    const int lmin = 1 - (1 << (bits - 1)), span = (1 << (bits - 1)) - lmin;
    for (int64_t i = 0; i < count; ++i) {
        int off;
        if (bits == 4)
            off = (i % 2 == 0) ? (b[i / 2] & 0x0f) : (b[i / 2] >> 4);
        else {
            off = b[i];
            if (off > span) return -2;
        }
        out[i] = (int16_t)(lmin + off);
    }
    return 0;
}

/* ======================= pipeline.cpp:29-115 ============================= */
int64_t ezqo_quantize(const float* W, int64_t rows, int64_t cols, const ezq_config* c, int mode,
                      int threads, uint8_t* packed, float* scales, ezq_outlier* outliers,
                      int64_t cap, double* mean, double* stddev, double* rtn_error,
                      double* final_error) {
    const int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) /* DenseMatrix::validate (types.cpp:17-20) */
        if (!isfinite(W[i])) return -1;
    if (c->bits < 2 || c->bits > 8 || !(c->sigma_n >= 0.0f) || !(c->lr > 0.0) ||
        !(c->beta1 >= 0.0 && c->beta1 < 1.0) || !(c->beta2 >= 0.0 && c->beta2 < 1.0) ||
        !(c->eps > 0.0) || c->steps < 0 || c->select_step < 0)
        return -3;
    const int lmin = 1 - (1 << (c->bits - 1)), lmax = 1 << (c->bits - 1);

    /* outliers (or stats only for Rtn) */
    int64_t n_out = 0;
    ezq_outlier* set = NULL;
    if (mode == EZQ_MODE_RTN) {
        double ma;
        ezqo_tensor_stats(W, n, mean, stddev, &ma);
    } else {
        n_out = ezqo_detect_outliers(W, rows, cols, c->sigma_n, NULL, mean, stddev);
        set = (ezq_outlier*)malloc(sizeof(ezq_outlier) * (size_t)(n_out ? n_out : 1));
        ezqo_detect_outliers(W, rows, cols, c->sigma_n, set, mean, stddev);
    }
    if (outliers && n_out <= cap) memcpy(outliers, set, sizeof(ezq_outlier) * (size_t)n_out);

    /* per-column outlier row lists (outliers.cpp:75-87): flat order => rows
     * ascending per column */
    int64_t* start = (int64_t*)calloc((size_t)cols + 1, sizeof(int64_t));
    uint32_t* orow = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n_out ? n_out : 1));
    for (int64_t k = 0; k < n_out; ++k) start[set[k].col + 1]++;
    for (int64_t j = 0; j < cols; ++j) start[j + 1] += start[j];
    {
        int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cols ? cols : 1));
        memcpy(pos, start, sizeof(int64_t) * (size_t)cols);
        for (int64_t k = 0; k < n_out; ++k) orow[pos[set[k].col]++] = set[k].row;
        free(pos);
    }

    int16_t* grid = (int16_t*)calloc((size_t)n, sizeof(int16_t));
    double* col_rtn = (double*)calloc((size_t)cols, sizeof(double));
    double* col_fin = (double*)calloc((size_t)cols, sizeof(double));
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
#endif
    for (int64_t j = 0; j < cols; ++j) { /* quantize_column (pipeline.cpp:29-63) */
        float* v = (float*)malloc(sizeof(float) * (size_t)rows);
        uint32_t* vr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)rows);
        int64_t nv = 0, k = start[j];
        for (int64_t i = 0; i < rows; ++i) {
            if (k < start[j + 1] && orow[k] == (uint32_t)i) {
                ++k;
                continue;
            }
            v[nv] = W[i * cols + j];
            vr[nv++] = (uint32_t)i;
        }
        float s = 1.0f;
        if (nv > 0) {
            if (mode == EZQ_MODE_EASYQUANT) {
                int bs;
                s = ezqo_optimize_channel(v, nv, c, &col_rtn[j], &col_fin[j], &bs, NULL, NULL);
            } else {
                s = (float)ezqo_initial_scale(v, nv, c->bits);
                double g;
                ezqo_eval_dense(v, nv, (double)s, lmin, lmax, &col_rtn[j], &g);
                col_fin[j] = col_rtn[j];
            }
            const double inv = 1.0 / (double)s; /* quantize_channel (rtn.cpp:88-99) */
            for (int64_t t = 0; t < nv; ++t)
                grid[(int64_t)vr[t] * cols + j] = (int16_t)ezqo_level_of((double)v[t], inv, lmin, lmax);
        }
        scales[j] = s;
        free(v);
        free(vr);
    }
    double rtn = 0.0, fin = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
        rtn += col_rtn[j];
        fin += col_fin[j];
    }
    *rtn_error = rtn;
    *final_error = fin;
    ezqo_pack_levels(grid, n, c->bits, packed);
    free(grid);
    free(col_rtn);
    free(col_fin);
    free(start);
    free(orow);
    free(set);
    if (fin > rtn) return -2; /* pipeline.cpp:107-108 */
    return n_out;
}

/* ======================= pipeline.cpp:117-142 ============================ */
int ezqo_dequantize(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                    const float* scales, const ezq_outlier* outliers, int64_t n_out, float* out) {
    const int64_t n = rows * cols;
    const int lmin = 1 - (1 << (bits - 1));
    for (int64_t f = 0; f < n; ++f) {
        const int off = bits == 4 ? ((f % 2 == 0) ? (packed[f / 2] & 0x0f) : (packed[f / 2] >> 4))
                                  : packed[f];
        out[f] = (float)((double)scales[f % cols] * (double)(lmin + off));
    }
    for (int64_t k = 0; k < n_out; ++k) {
        if (outliers[k].row >= (uint64_t)rows || outliers[k].col >= (uint64_t)cols) return -1;
        out[(int64_t)outliers[k].row * cols + outliers[k].col] = outliers[k].value;
    }
    return 0;
}

/* ======================= rtn.cpp:34-77 =================================== */
double ezqo_reconstruction_error(const float* a, const float* b, int64_t rows, int64_t cols,
                                 const ezq_outlier* skip, int64_t n_skip) {
    double total = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
        /* column's skip rows in entry order (outlier_rows_by_column) */
        double acc = 0.0;
        int64_t k = 0;
        while (k < n_skip && skip[k].col != (uint32_t)j) ++k;
        for (int64_t i = 0; i < rows; ++i) {
            if (k < n_skip && skip[k].row == (uint32_t)i) {
                ++k;
                while (k < n_skip && skip[k].col != (uint32_t)j) ++k;
                continue;
            }
            const double d = (double)a[i * cols + j] - (double)b[i * cols + j];
            acc += d * d;
        }
        total += acc;
    }
    return total;
}

void ezqo_gemv_f64(const float* What, int64_t rows, int64_t cols, const float* x, int batch,
                   double* y) {
    for (int b = 0; b < batch; ++b)
        for (int64_t j = 0; j < cols; ++j) {
            double acc = 0.0;
            for (int64_t i = 0; i < rows; ++i)
                acc += (double)x[(int64_t)b * rows + i] * (double)What[i * cols + j];
            y[(int64_t)b * cols + j] = acc;
        }
}
