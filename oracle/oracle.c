/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY. Plain, slow, obviously-correct CPU
 * reference of the convolution arithmetic of Dryden et al., "Improving
 * Strong-Scaling of CNN Training by Exploiting Finer-Grained Parallelism"
 * (arXiv:1903.06681). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no
 * code, header or constant with the CUDA path (paper_1903_06681_b200/).
 *
 * Precision: IEEE fp64 throughout. Layout: NCHW activations and F x C x K x K
 * weights, the paper's layout ("We do not consider alternate
 * storage layouts (e.g. NHWC)").
 *
 * Generalisation to stride S and padding P ("these assumptions
 * are not necessary for our work"; reading R2): input index of
 * output (i, a) is S*i + a - P, output extent Ho = floor((H + 2P - K)/S) + 1,
 * out-of-range inputs read as zero. With S = 1 and P = O = floor(K/2) this is
 * exactly Eq. 1 (index i + a' with a' = a - O in [-O, O]).
 *
 * Pins (tests/test_oracle.py): worked values, the
 * cross-correlation asymmetric pin (R1), brute-force dependence,
 * adjoint identities, central finite differences, torch-CPU fp64 conv2d,
 * partition invariance.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

typedef int64_t i64;

static inline i64 out_extent(i64 H, i64 K, i64 S, i64 P) { return (H + 2 * P - K) / S + 1; }

#define X4(t, n, c, h, w, C, H, W) (t)[(((n) * (C) + (c)) * (H) + (h)) * (W) + (w)]

/* Eq. 1, generalised (reading R2):
 *   y[n,f,i,j] = sum_{c<C} sum_{a<K} sum_{b<K} x[n,c,S i+a-P, S j+b-P] * w[f,c,a,b]
 * Computes output rows i in [i0, i1) of every sample and filter (row range
 * exists only so bench.py can time a bounded sample and tests can check
 * sampled rows at full size). Summation order: c, then a, then b. */
void oracle_conv_fwd(i64 N, i64 C, i64 H, i64 W, i64 F, i64 K, i64 S, i64 P,
                     const double *x, const double *w, double *y, i64 i0, i64 i1)
{
    const i64 Ho = out_extent(H, K, S, P), Wo = out_extent(W, K, S, P);
#pragma omp parallel for collapse(2) schedule(static)
    for (i64 n = 0; n < N; ++n)
        for (i64 f = 0; f < F; ++f)
            for (i64 i = i0; i < i1; ++i)
                for (i64 j = 0; j < Wo; ++j) {
                    double acc = 0.0;
                    for (i64 c = 0; c < C; ++c)
                        for (i64 a = 0; a < K; ++a) {
                            const i64 h = S * i + a - P;
                            if (h < 0 || h >= H) continue;
                            for (i64 b = 0; b < K; ++b) {
                                const i64 v = S * j + b - P;
                                if (v < 0 || v >= W) continue;
                                acc += X4(x, n, c, h, v, C, H, W) * X4(w, f, c, a, b, C, K, K);
                            }
                        }
                    X4(y, n, f, i, j, F, Ho, Wo) = acc;
                }
}

/* Eq. 3, strided form = exact adjoint of the forward map
 * (reading R4):
 *   dx[n,c,u,v] = sum_f sum_a sum_b dy[n,f,(u+P-a)/S,(v+P-b)/S] * w[f,c,a,b]
 * where a term exists only if both divisions are exact and the quotient lies
 * in [0,Ho) x [0,Wo). With S=1, P=O this is Eq. 3 verbatim (dy index i-a').
 * Computes input rows u in [u0, u1). Order: f, then a, then b. */
void oracle_conv_bwd_data(i64 N, i64 C, i64 H, i64 W, i64 F, i64 K, i64 S, i64 P,
                          const double *dy, const double *w, double *dx, i64 u0, i64 u1)
{
    const i64 Ho = out_extent(H, K, S, P), Wo = out_extent(W, K, S, P);
#pragma omp parallel for collapse(2) schedule(static)
    for (i64 n = 0; n < N; ++n)
        for (i64 c = 0; c < C; ++c)
            for (i64 u = u0; u < u1; ++u)
                for (i64 v = 0; v < W; ++v) {
                    double acc = 0.0;
                    for (i64 f = 0; f < F; ++f)
                        for (i64 a = 0; a < K; ++a) {
                            const i64 ti = u + P - a;
                            if (ti < 0 || ti % S != 0) continue;
                            const i64 i = ti / S;
                            if (i >= Ho) continue;
                            for (i64 b = 0; b < K; ++b) {
                                const i64 tj = v + P - b;
                                if (tj < 0 || tj % S != 0) continue;
                                const i64 j = tj / S;
                                if (j >= Wo) continue;
                                acc += X4(dy, n, f, i, j, F, Ho, Wo) * X4(w, f, c, a, b, C, K, K);
                            }
                        }
                    X4(dx, n, c, u, v, C, H, W) = acc;
                }
}

/* Eq. 2, with the i, j range read as the output extent
 * (reading R3):
 *   dw[f,c,a,b] = sum_n sum_{i<Ho} sum_{j<Wo} dy[n,f,i,j] * x[n,c,S i+a-P, S j+b-P]
 * One entry; order n, then i, then j. */
double oracle_conv_bwd_filter_entry(i64 N, i64 C, i64 H, i64 W, i64 F, i64 K, i64 S, i64 P,
                                    const double *x, const double *dy, i64 f, i64 c, i64 a, i64 b)
{
    const i64 Ho = out_extent(H, K, S, P), Wo = out_extent(W, K, S, P);
    double acc = 0.0;
    for (i64 n = 0; n < N; ++n)
        for (i64 i = 0; i < Ho; ++i) {
            const i64 h = S * i + a - P;
            if (h < 0 || h >= H) continue;
            for (i64 j = 0; j < Wo; ++j) {
                const i64 v = S * j + b - P;
                if (v < 0 || v >= W) continue;
                acc += X4(dy, n, f, i, j, F, Ho, Wo) * X4(x, n, c, h, v, C, H, W);
            }
        }
    return acc;
}

/* All of dw (F x C x K x K), entry by entry. */
void oracle_conv_bwd_filter(i64 N, i64 C, i64 H, i64 W, i64 F, i64 K, i64 S, i64 P,
                            const double *x, const double *dy, double *dw)
{
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (i64 f = 0; f < F; ++f)
        for (i64 c = 0; c < C; ++c)
            for (i64 a = 0; a < K; ++a)
                for (i64 b = 0; b < K; ++b)
                    X4(dw, f, c, a, b, C, K, K) =
                        oracle_conv_bwd_filter_entry(N, C, H, W, F, K, S, P, x, dy, f, c, a, b);
}

/* Batch-norm statistics (reading R11):
 * per channel c, mean and biased variance over all (n, h, w) of t, two-pass:
 *   mu_c = sum t / (N H W);  var_c = sum (t - mu_c)^2 / (N H W). */
void oracle_bn_stats(i64 N, i64 C, i64 H, i64 W, const double *t, double *mean, double *var)
{
    const double cnt = (double)(N * H * W);
    for (i64 c = 0; c < C; ++c) {
        double s = 0.0;
        for (i64 n = 0; n < N; ++n)
            for (i64 h = 0; h < H; ++h)
                for (i64 w = 0; w < W; ++w) s += X4(t, n, c, h, w, C, H, W);
        const double mu = s / cnt;
        double q = 0.0;
        for (i64 n = 0; n < N; ++n)
            for (i64 h = 0; h < H; ++h)
                for (i64 w = 0; w < W; ++w) {
                    const double d = X4(t, n, c, h, w, C, H, W) - mu;
                    q += d * d;
                }
        mean[c] = mu;
        var[c] = q / cnt;
    }
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
