/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what arXiv 2509.20500 computes, written from
 * PAPER.md (= /root/reference/PAPER.md; "P:NN" is its line NN). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library. It shares no code,
 * header, table or constant with the CUDA product (paper_2509_20500_b200/), and the product never
 * calls it.
 *
 * What it computes (each function cites the passage it follows):
 *   - lambda(t), F(t): Eq. 1, S, B, Lambda, F(t) := int_0^t lambda (Thm 1),
 *     in closed form with erfc.
 *   - The transition matrix by the SEQUENTIAL definition the paper replaces: Eq. 3 bounds,
 *     the discretisation operator D and Eq. 4, one integral per entry, then
 *     row normalisation.  The paper's accelerated construction (Thm 2 / Eq. 6 / §3.4) is NOT
 *     used here; the GPU implements that one, so parity is a real check of Theorem 2.
 *   - pi with pi P~ = pi: dense Gaussian elimination, and plain power iteration.
 *   - A continuous-time Monte Carlo of the detection process of P:60 (inhomogeneous Poisson arrivals,
 *     SPAD dead time, X_k = T_k mod t_r), used only to pin the chain physically.
 *
 * Readings where the paper is silent (DESIGN.md §3 lists them all):
 *   R5  Lambda := F(t_r) (the integral of the one-period flux), so the periodic replica is exact.
 *   R6  lambda~ is the one-period lambda repeated (not a wrapped Gaussian).
 *   R4  x_d / Delta is evaluated as u = fmod(t_d, t_r) * N / t_r, read as the integer it is within
 *       8 ulps of (a dead time of whole bins in decimal lands on a bin centre); ceilings are taken in bin units
 *       so integer cases stay exact.
 *   R8  the 1/(1-exp(-Lambda)) prefactor of Eq. 3 is dropped: rows are divided by their sums.
 *   Parity pins: none unpinned (see tests/test_oracle_pins.py); the MC pin is statistical.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double t_r;          /* laser period                                  */
    int32_t n_bins;      /* n_b                                     */
    int32_t n_pulses;    /* K; Eq. 1 has K = 1, K > 1 sums pulses                */
    const double *tau;   /* pulse centres tau_k                           */
    const double *sigma; /* pulse widths sigma_t                          */
    const double *signal;/* S_k = alpha E                                 */
    double background;   /* B = t_r lambda_b                              */
} oracle_flux;

static const double kPi = 3.14159265358979323846;

/* Threads of the OpenMP row loops (timing only: the arithmetic does not depend on it). */
void oracle_set_threads(int32_t n) { omp_set_num_threads(n > 0 ? n : 1); }
int32_t oracle_max_threads(void) { return omp_get_max_threads(); }

/* Phi(z) standard normal CDF via erfc. */
static double std_cdf(double z) { return 0.5 * erfc(-z / sqrt(2.0)); }

/* Eq. 1 with s(t) = E N(t; 0, sigma^2), S = alpha E, lambda_b = B / t_r. */
double oracle_lambda(const oracle_flux *f, double t) {
    double v = f->background / f->t_r;
    for (int k = 0; k < f->n_pulses; ++k) {
        double z = (t - f->tau[k]) / f->sigma[k];
        v += f->signal[k] * exp(-0.5 * z * z) / (f->sigma[k] * sqrt(2.0 * kPi));
    }
    return v;
}

/* F(t) := int_0^t lambda(tau) dtau (Theorem 1), closed form, 0 <= t <= t_r. */
double oracle_F(const oracle_flux *f, double t) {
    double v = f->background * t / f->t_r;
    for (int k = 0; k < f->n_pulses; ++k)
        v += f->signal[k] * (std_cdf((t - f->tau[k]) / f->sigma[k]) - std_cdf(-f->tau[k] / f->sigma[k]));
    return v;
}

/* Lambda: total flux per period, read as F(t_r) (reading R5). */
double oracle_Lambda(const oracle_flux *f) { return oracle_F(f, f->t_r); }

/* Integral of the periodic replica lambda~ from 0 to q*t_r + t, 0 <= t <= t_r:
 * q whole periods plus F(t) (reading R6). */
double oracle_Ftilde(const oracle_flux *f, int64_t q, double t) {
    return (double)q * oracle_Lambda(f) + oracle_F(f, t);
}

/* Bin centre s_j = (j + 1/2) Delta for 0-based j, i.e. s_1..s_N of P:79 with Delta = t_r / n_b. */
static double centre(const oracle_flux *f, int64_t j) { return ((double)j + 0.5) * (f->t_r / f->n_bins); }

/* One UNNORMALISED entry of Eq. 4 with the bounds of Eq. 3:
 *   x_d = t_d mod t_r,  a = x_k + x_d,  b = ceil((x_k + x_d - x_{k+1}) / t_r) t_r + x_{k+1},
 *   D(t) = (ceil(t / Delta) - 1/2) Delta,
 *   E_ij = exp(- int_{D(a)}^{D(b)} lambda~),  P_ij = lambda(s_j) E_ij.
 * x_k = s_i, x_{k+1} = s_j. The ceilings are evaluated in bin units (a / Delta = i + 1/2 + u,
 * (a - s_j) / t_r = (i - j + u) / N with u = x_d / Delta), and each bound is carried as
 * (whole periods, bin index within the period), so period counts stay integers. */
double oracle_entry_eq4_unnorm(const oracle_flux *f, double t_d, int32_t i, int32_t j) {
    const int64_t N = f->n_bins;
    const double x_d = fmod(t_d, f->t_r);
    double u = x_d * (double)N / f->t_r;                  /* x_d / Delta (reading R4) */
    if (fabs(u - nearbyint(u)) <= 8.0 * 2.220446049250313e-16 * fmax(1.0, fabs(u))) u = nearbyint(u);
    /* lower limit D(a): a / Delta = i + 1/2 + u; ceil -> 1-based bin index k_a on the unrolled line */
    const int64_t k_a = (int64_t)ceil((double)i + 0.5 + u);   /* >= 1 since u >= 0 */
    const int64_t qa = (k_a - 1) / N;
    const int64_t ia = (k_a - 1) - qa * N;                /* D(a) = q_a t_r + s_ia */
    /* upper limit: b = m t_r + s_j with m = ceil((a - s_j) / t_r); b is a bin centre so D(b) = b */
    const int64_t m = (int64_t)ceil(((double)i - (double)j + u) / (double)N);
    const double upper = oracle_Ftilde(f, m, centre(f, j));
    const double lower = oracle_Ftilde(f, qa, centre(f, ia));
    const double integral = upper - lower;                /* int_{D(a)}^{D(b)} lambda~ */
    return oracle_lambda(f, centre(f, j)) * exp(-integral);
}

/* Row i of P~: Eq. 4 entries divided by their row sum (long double accumulation). */
int oracle_row_eq4(const oracle_flux *f, double t_d, int32_t i, double *row) {
    const int32_t N = f->n_bins;
    long double sum = 0.0L;
    for (int32_t j = 0; j < N; ++j) {
        row[j] = oracle_entry_eq4_unnorm(f, t_d, i, j);
        sum += row[j];
    }
    if (!(sum > 0.0L)) return 1;
    for (int32_t j = 0; j < N; ++j) row[j] = (double)((long double)row[j] / sum);
    return 0;
}

/* Rows [r0, r1) of P~ into out[(i - r0) * N + j]; OpenMP over rows only (no change in arithmetic). */
int oracle_rows_eq4(const oracle_flux *f, double t_d, int32_t r0, int32_t r1, double *out) {
    const int32_t N = f->n_bins;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
    for (int32_t i = r0; i < r1; ++i) bad |= oracle_row_eq4(f, t_d, i, out + (int64_t)(i - r0) * N);
    return bad;
}

/* Full N x N P~ (row-major). */
int oracle_build_eq4(const oracle_flux *f, double t_d, double *out) {
    return oracle_rows_eq4(f, t_d, 0, f->n_bins, out);
}

/* Y[v] = X[v]^T P~ for k vectors X[v] (k rows of N, row-major) and a row-streamed P~ (P~ never
 * stored): used to check pi P~ = pi at sizes where the dense matrix does not fit; each row
 * of P~ is recomputed once from Eq. 4 and applied to all k vectors. Y is accumulated in long
 * double per thread, then summed over threads in thread order. */
int oracle_left_matvec_streamed_multi(const oracle_flux *f, double t_d, int32_t k, const double *x,
                                      double *y) {
    const int32_t N = f->n_bins;
    const size_t nk = (size_t)N * (size_t)k;
    int bad = 0;
    long double *acc = (long double *)calloc(nk, sizeof(long double));
    if (!acc) return 2;
#pragma omp parallel reduction(| : bad)
    {
        long double *loc = (long double *)calloc(nk, sizeof(long double));
        double *row = (double *)malloc((size_t)N * sizeof(double));
        if (!loc || !row) bad |= 2;
        else {
#pragma omp for schedule(dynamic, 8)
            for (int32_t i = 0; i < N; ++i) {
                bad |= oracle_row_eq4(f, t_d, i, row);
                for (int32_t v = 0; v < k; ++v) {
                    const long double xi = x[(size_t)v * N + i];
                    long double *lv = loc + (size_t)v * N;
                    for (int32_t j = 0; j < N; ++j) lv[j] += xi * row[j];
                }
            }
#pragma omp critical
            for (size_t t = 0; t < nk; ++t) acc[t] += loc[t];
        }
        free(loc);
        free(row);
    }
    for (size_t t = 0; t < nk; ++t) y[t] = (double)acc[t];
    free(acc);
    return bad;
}

/* y = x^T P~ (one vector). */
int oracle_left_matvec_streamed(const oracle_flux *f, double t_d, const double *x, double *y) {
    return oracle_left_matvec_streamed_multi(f, t_d, 1, x, y);
}

/* pi P~ = pi, sum(pi) = 1 (leading left eigenvector of the stochastic matrix), by Gaussian
 * elimination with partial pivoting on (P~^T - I) with its last equation replaced by 1^T pi = 1. */
int oracle_stationary_dense(int32_t n, const double *Pt, double *pi) {
    double *A = (double *)malloc((size_t)n * n * sizeof(double));
    double *b = (double *)malloc((size_t)n * sizeof(double));
    if (!A || !b) { free(A); free(b); return 2; }
    for (int32_t r = 0; r < n; ++r) {          /* row r of A: equation for pi_r */
        for (int32_t c = 0; c < n; ++c) A[(int64_t)r * n + c] = Pt[(int64_t)c * n + r] - (r == c ? 1.0 : 0.0);
        b[r] = 0.0;
    }
    for (int32_t c = 0; c < n; ++c) A[(int64_t)(n - 1) * n + c] = 1.0;
    b[n - 1] = 1.0;
    for (int32_t k = 0; k < n; ++k) {
        int32_t p = k;
        for (int32_t r = k + 1; r < n; ++r)
            if (fabs(A[(int64_t)r * n + k]) > fabs(A[(int64_t)p * n + k])) p = r;
        if (A[(int64_t)p * n + k] == 0.0) { free(A); free(b); return 1; }
        if (p != k) {
            for (int32_t c = 0; c < n; ++c) {
                double t = A[(int64_t)k * n + c]; A[(int64_t)k * n + c] = A[(int64_t)p * n + c]; A[(int64_t)p * n + c] = t;
            }
            double t = b[k]; b[k] = b[p]; b[p] = t;
        }
        for (int32_t r = k + 1; r < n; ++r) {
            double l = A[(int64_t)r * n + k] / A[(int64_t)k * n + k];
            if (l == 0.0) continue;
            for (int32_t c = k; c < n; ++c) A[(int64_t)r * n + c] -= l * A[(int64_t)k * n + c];
            b[r] -= l * b[k];
        }
    }
    for (int32_t r = n - 1; r >= 0; --r) {
        long double s = b[r];
        for (int32_t c = r + 1; c < n; ++c) s -= (long double)A[(int64_t)r * n + c] * pi[c];
        pi[r] = (double)(s / A[(int64_t)r * n + r]);
    }
    free(A);
    free(b);
    return 0;
}

/* y = x^T A for R rows of A (row-major, N columns), accumulated in long double (the product used by
 * the power iteration below; exported so that bench.py can time a bounded sample of it). */
void oracle_left_matvec(int32_t R, int32_t n, const double *A, const double *x, long double *y) {
    for (int32_t j = 0; j < n; ++j) y[j] = 0.0L;
    for (int32_t i = 0; i < R; ++i) {
        long double xi = x[i];
        const double *row = A + (int64_t)i * n;
        for (int32_t j = 0; j < n; ++j) y[j] += xi * row[j];
    }
}

/* Power iteration (the solver BASELINE.json names for P:79): pi^0 = 1/N; pi^{k+1} = y / ||y||_1 with
 * y = pi^k P~; stop when ||pi^{k+1} - pi^k||_1 < tol. Returns 0 converged, 3 if max_iter reached.
 * iters = number of products y = pi P~ taken. */
int oracle_stationary_power(int32_t n, const double *Pt, double tol, int32_t max_iter,
                            double *pi, int32_t *iters, double *change) {
    long double *y = (long double *)malloc((size_t)n * sizeof(long double));
    if (!y) return 2;
    for (int32_t j = 0; j < n; ++j) pi[j] = 1.0 / n;
    double ch = INFINITY;
    int32_t it = 0;
    while (it < max_iter) {
        oracle_left_matvec(n, n, Pt, pi, y);
        long double s = 0.0L;
        for (int32_t j = 0; j < n; ++j) s += y[j];
        long double d = 0.0L;
        for (int32_t j = 0; j < n; ++j) {
            double v = (double)(y[j] / s);
            d += fabsl((long double)v - pi[j]);
            pi[j] = v;
        }
        ++it;
        ch = (double)d;
        if (ch < tol) break;
    }
    free(y);
    *iters = it;
    *change = ch;
    return ch < tol ? 0 : 3;
}

/* ---------------------------------------------------------------- Monte Carlo -------- */

static uint64_t splitmix64(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double unif01_open(uint64_t *s) {  /* (0, 1] */
    return ((double)(splitmix64(s) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}

/* Solve F(t) = y for t in [0, t_r] (F increasing): bisection on the closed form. */
static double F_inverse(const oracle_flux *f, double y) {
    double lo = 0.0, hi = f->t_r;
    for (int it = 0; it < 200 && hi - lo > 1e-13 * f->t_r; ++it) {
        double mid = 0.5 * (lo + hi);
        if (oracle_F(f, mid) < y) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

/* One registration of the continuous-time detection process: photons arrive as an
 * inhomogeneous Poisson process with the periodic rate lambda~ (Eq. 1 replicated); after
 * the registration at T_k = q t_r + t the SPAD is dead for t_d and re-arms at T_k + t_d; the
 * next registration is the first arrival after re-arming, T_{k+1} = Ftilde^{-1}(Ftilde(T_k + t_d) + E),
 * E ~ Exp(1) = -log U, U uniform on (0, 1] from splitmix64 (time change of a Poisson process). Time is
 * carried as (period q, offset t in [0, t_r)) to keep precision. */
static void mc_next(const oracle_flux *f, double Lam, double t_d, uint64_t *st, int64_t *q, double *t) {
    double tt = *t + t_d;
    int64_t qq = *q + (int64_t)floor(tt / f->t_r);
    tt = fmod(tt, f->t_r);
    if (tt < 0.0) tt += f->t_r;
    double target = oracle_F(f, tt) - log(unif01_open(st));
    int64_t extra = (int64_t)floor(target / Lam);
    double rem = target - (double)extra * Lam;
    if (rem < 0.0) { rem += Lam; extra -= 1; }
    if (rem >= Lam) { rem -= Lam; extra += 1; }
    *q = qq + extra;
    *t = F_inverse(f, rem);
    if (*t >= f->t_r) { *t -= f->t_r; *q += 1; }
}

/* The first n registrations of one chain started at (q, t) = (0, 0) with generator state `seed`:
 * q_out[k], t_out[k] (X_k = t_out[k] = T_k mod t_r). */
int oracle_mc_timestamps(const oracle_flux *f, double t_d, uint64_t seed, int64_t n, int64_t *q_out,
                         double *t_out) {
    const double Lam = oracle_Lambda(f);
    if (!(Lam > 0.0)) return 1;
    uint64_t st = seed;
    int64_t q = 0;
    double t = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        mc_next(f, Lam, t_d, &st, &q, &t);
        q_out[k] = q;
        t_out[k] = t;
    }
    return 0;
}

/* Histogram of the timestamps X_k = T_k mod t_r of one chain: n_hist bins
 * ((k-1) Delta_h, k Delta_h] with X = 0 read as t_r. The first n_burn registrations are discarded;
 * the rest are split into n_batches consecutive batches, hist[b * n_hist + k]. */
int oracle_mc(const oracle_flux *f, double t_d, uint64_t seed, int64_t n_burn, int64_t n_per_batch,
              int32_t n_batches, int32_t n_hist, int64_t *hist) {
    const double Lam = oracle_Lambda(f);
    if (!(Lam > 0.0)) return 1;
    uint64_t st = seed;
    int64_t q = 0;
    double t = 0.0;
    memset(hist, 0, sizeof(int64_t) * (size_t)n_batches * n_hist);
    const int64_t total = n_burn + n_per_batch * n_batches;
    for (int64_t k = 0; k < total; ++k) {
        mc_next(f, Lam, t_d, &st, &q, &t);
        if (k >= n_burn) {
            int64_t b = (k - n_burn) / n_per_batch;
            double dh = f->t_r / n_hist;
            int64_t bin = (int64_t)ceil(t / dh) - 1;   /* ((k-1)dh, k dh] */
            if (bin < 0) bin = n_hist - 1;             /* X = 0 is t_r */
            if (bin >= n_hist) bin = n_hist - 1;
            hist[b * n_hist + bin] += 1;
        }
    }
    return 0;
}
