// CPU simulation of the K3s certification, an analysis tool.
//
// For every column of a synthetic N(0, std^2) matrix (n-sigma outliers
// removed as in outliers.cpp:18-73), run
//   (a) the reference q_range loop: eval_dense's sequential fp64 sums and
//       adam_step (optimize.cpp:30-51, 86-94, 118-184), and
//   (b) the K3s loop: err/grad from exact sums (double-double here), with the
//       rounding bounds of the certification -- a column is flagged when a
//       snap could land on the other side of a float rounding midpoint under
//       the reference's sequential rounding, or when the best-error selection
//       compares two steps whose exact errors lie within the reference's
//       rounding of each other.
// Reports: flagged columns (trajectory / selection), columns whose final
// scale differs between (a) and (b), and differing columns that were NOT
// flagged (the certification's soundness: must be 0).
//
//   gcc -O2 -fopenmp -o /tmp/cert_sim tools/cert_sim.c -lm
//   /tmp/cert_sim ROWS COLS [bits] [sigma_n] [std] [seed]
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double U = 1.1102230246251565e-16;  // 2^-53

static uint64_t sm64(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static double unif(uint64_t* s) { return (sm64(s) >> 11) * (1.0 / 9007199254740992.0); }
static double gauss(uint64_t* s) {
    double u1 = unif(s), u2 = unif(s);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2 * log(u1)) * cos(2 * M_PI * u2);
}

typedef struct { double hi, lo; } dd;
static dd two_sum(double a, double b) {
    double s = a + b, bb = s - a;
    return (dd){s, (a - (s - bb)) + (b - bb)};
}
static dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo += a.lo;
    return two_sum(s.hi, s.lo);
}
static dd dd_add_prod(dd a, double x, double y) {  // a + x*y
    double p = x * y, e = fma(x, y, -p);
    a = dd_add_d(a, p);
    return dd_add_d(a, e);
}

static double level_of(double x, double inv, int lmin, int lmax) {
    double u = x * inv;
    if (u >= lmax) return lmax;
    if (u <= lmin) return lmin;
    return (double)llround(u);
}
static double snap(double s) {
    double f = (double)(float)s;
    return f < 1e-12 ? 1e-12 : f;
}

typedef struct {
    double b1, b2, lr, eps;
} Adam;

static double adam(double* m, double* v, double s, double g, int t, const Adam* a) {
    *m = a->b1 * *m + (1.0 - a->b1) * g;
    *v = a->b2 * *v + (1.0 - a->b2) * g * g;
    double mh = *m / (1.0 - pow(a->b1, (double)t));
    double vh = *v / (1.0 - pow(a->b2, (double)t));
    double up = s - a->lr * mh / (sqrt(vh) + a->eps);
    return up < 1e-12 ? 1e-12 : up;
}

// (a) reference
static float ref_opt(const float* x, int n, int lmin, int lmax, int steps, const Adam* a) {
    double mx = 0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, fabs((double)x[i]));
    double s = snap(mx == 0 ? 1.0 : mx / lmax);
    double best = 0, bs = s, m = 0, v = 0, g = 0;
    for (int t = 0; t <= steps; ++t) {
        if (t) s = snap(adam(&m, &v, s, g, t, a));
        double inv = 1.0 / s, e = 0, gr = 0;
        for (int i = 0; i < n; ++i) {
            double xi = x[i], q = level_of(xi, inv, lmin, lmax), d = s * q - xi;
            e += d * d;
            gr += d * q;
        }
        g = 2.0 * gr;
        if (t == 0 || e < best) best = e, bs = s;
    }
    return (float)bs;
}

// Sequential reference error of a column at scale s (eval_dense's err).
static double seq_err(const float* x, int n, double s, int lmin, int lmax) {
    const double inv = 1.0 / s;
    double e = 0;
    for (int i = 0; i < n; ++i) {
        const double xi = x[i], q = level_of(xi, inv, lmin, lmax), d = s * q - xi;
        e += d * d;
    }
    return e;
}

// (b) K3s: exact sums, the gradient exactness predicate, and the selection
// candidates (steps whose exact error lies within the reference's rounding
// bound of the best), resolved with sequential errors. Returns the scale.
// *ncand: candidates left at the end; *gfail: steps where the predicate
// could not prove the sequential gradient exact.
static float cert_opt(const float* x, int n, int lmin, int lmax, int steps, const Adam* a, int* ncand,
                      int* gfail, int* gdiff) {
    double mx = 0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, fabs((double)x[i]));
    double s = snap(mx == 0 ? 1.0 : mx / lmax);
    const double gam = (n + 1) * U * (1 + 1e-9);
    const int L = lmax > -lmin ? lmax : -lmin;
    double m = 0, v = 0, g = 0;
    // candidate list (t order): scale, exact error
    double cs[256], ce[256];
    int nc = 0;
    double bestE = 0, bestS = s;
    *gfail = *gdiff = 0;
    for (int t = 0; t <= steps; ++t) {
        if (t) s = snap(adam(&m, &v, s, g, t, a));
        // exactness of the sequential gradient: every nonzero term d*q is a
        // multiple of D = 2^(floor(log2(s/2 (1-4u))) - 23) and sum |d q| <=
        // n L (s L + max|x|) < 2^53 D  =>  every partial sum is exact
        int e2;
        frexp(0.5 * s * (1 - 4 * U), &e2);
        const double D = ldexp(1.0, e2 - 1 - 23);
        if (!((double)n * L * (s * L + mx) < ldexp(D, 53))) ++*gfail;
        const double inv = 1.0 / s;
        dd E = {0, 0}, G = {0, 0};
        double gs = 0;
        for (int i = 0; i < n; ++i) {
            const double xi = x[i], q = level_of(xi, inv, lmin, lmax), d = s * q - xi;
            E = dd_add_prod(E, d, d);
            G = dd_add_prod(G, d, q);
            gs += d * q;
        }
        g = 2.0 * (G.hi + G.lo);
        if (g != 2.0 * gs) ++*gdiff;
        const double err = E.hi + E.lo;
        if (t == 0 || err < bestE) {
            // new best: keep the candidates whose error may still round below it
            int k = 0;
            for (int i = 0; i < nc; ++i)
                if (ce[i] - err <= gam * (ce[i] + err)) cs[k] = cs[i], ce[k] = ce[i], ++k;
            nc = k;
            bestE = err, bestS = s;
            cs[nc] = s, ce[nc] = err, ++nc;
        } else if (err - bestE <= gam * (err + bestE)) {
            int dup = 0;
            for (int i = 0; i < nc; ++i) dup |= cs[i] == s;
            if (!dup) cs[nc] = s, ce[nc] = err, ++nc;
        }
        if (nc > 250) nc = 250;
    }
    *ncand = nc;
    if (nc <= 1) return (float)bestS;
    double be = 0, bs = 0;
    for (int i = 0; i < nc; ++i) {
        const double e = seq_err(x, n, cs[i], lmin, lmax);
        if (i == 0 || e < be) be = e, bs = cs[i];
    }
    return (float)bs;
}

int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 4096, Cc = argc > 2 ? atoi(argv[2]) : 512;
    const int bits = argc > 3 ? atoi(argv[3]) : 4;
    const double sig = argc > 4 ? atof(argv[4]) : 3.0, sd = argc > 5 ? atof(argv[5]) : 0.02;
    const uint64_t seed = argc > 6 ? strtoull(argv[6], 0, 10) : 1;
    const int lmin = -(1 << (bits - 1)) + 1, lmax = 1 << (bits - 1), steps = 200;
    const Adam a = {0.9, 0.999, 1e-3, 1e-8};
    float* W = malloc(sizeof(float) * (size_t)R * Cc);
    uint64_t st = seed;
    double sum = 0, ss = 0;
    for (size_t i = 0; i < (size_t)R * Cc; ++i) W[i] = (float)(sd * gauss(&st)), sum += W[i];
    const double mean = sum / ((double)R * Cc);
    for (size_t i = 0; i < (size_t)R * Cc; ++i) ss += (W[i] - mean) * (W[i] - mean);
    const double thr = sig * sqrt(ss / ((double)R * Cc));
    long nflag = 0, ndiff = 0, ngfail = 0, ngdiff = 0, hist[18] = {0};
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : nflag, ndiff, ngfail, ngdiff) reduction(+ : hist[:18])
    for (int c = 0; c < Cc; ++c) {
        float* x = malloc(sizeof(float) * R);
        int n = 0;
        for (int r = 0; r < R; ++r) {
            const float v = W[(size_t)r * Cc + c];
            if (!(fabs((double)v - mean) >= thr)) x[n++] = v;
        }
        int nc, gf, gd;
        const float sr = ref_opt(x, n, lmin, lmax, steps, &a);
        const float sc = cert_opt(x, n, lmin, lmax, steps, &a, &nc, &gf, &gd);
        nflag += nc > 1;
        hist[nc > 17 ? 17 : nc]++;
        ndiff += sr != sc;
        ngfail += gf;
        ngdiff += gd;
        free(x);
    }
    printf("{\"rows\": %d, \"cols\": %d, \"bits\": %d, \"sigma_n\": %g, \"resolved_cols\": %ld, "
           "\"resolve_rate\": %.3g, \"cand_hist\": [", R, Cc, bits, sig, nflag, (double)nflag / Cc);
    for (int i = 0; i < 18; ++i) printf("%ld%s", hist[i], i < 17 ? ", " : "");
    printf("], \"grad_predicate_fail_steps\": %ld, \"grad_seq_ne_exact_steps\": %ld, \"scale_diff_vs_reference\": %ld}\n",
           ngfail, ngdiff, ndiff);
    return ndiff != 0;
}
