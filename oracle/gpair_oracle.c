/*
 * gpair_oracle.c -- fp64 CPU ORACLE for the GPAIR closed-form forward operator
 * and its adjoint.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library.  The product path
 * (paper_2602_03893_b200/) never imports, links or executes anything under
 * oracle/, and this file shares no code, header, table or constant generator
 * with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited P:<line>):
 *
 *   Eq. 7, outgoing spherical wave of one Gaussian kernel:
 *       p(r, t) = A/(2r) * d * exp(-d^2 / (2 sigma^2)),   d = r - v t
 *   3-sigma truncation: "-3 sigma < d < 3 sigma"; k is a parameter,
 *       strict inequality (reading R1).
 *   Direct enumeration: "iterate over all source-detector pairs and
 *       evaluate the contribution at each temporal sampling point where d
 *       falls within the +-3 sigma range".
 *   Superposition (Eq. 2): y_j[n] = sum_i A_i a_ijn.
 *   Adjoint = exact transpose: g_i = sum_j sum_n a_ijn delta_j[n].
 *
 *   a_ijn = d * exp(-d^2/(2 sigma^2)) / (2 r_ij)   if |d| < k sigma, else 0,
 *   r_ij  = || c_i - s_j ||,  t_n = t0 + n / f_s  (reading R3), d = r_ij - v t_n.
 *
 * Plain definition, no blocking or reordering: fp64 throughout, libm exp/sqrt,
 * built with -O2 -fno-fast-math -ffp-contract=off.  Inputs are the fp32 values
 * the GPU receives, promoted exactly to fp64.  Forward accumulates each y_j[n]
 * in ascending kernel order i; adjoint accumulates each g_i in ascending j then
 * ascending n.  OpenMP only parallelises over independent outputs (sensors for
 * the forward, kernels for the adjoint), so results are bit-reproducible for
 * any thread count.
 *
 * Candidate samples: n from floor(((r - k s)/v - t0) f_s) - 2 to
 * ceil(((r + k s)/v - t0) f_s) + 2, clipped to [0, N_t); the membership test
 * |d| < k sigma is applied literally to each candidate (record-edge clipping:
 * reading R8).  Pairs with r_ij <= k sigma are rejected (reading R2: Eq. 7 is
 * a far-field model) with return code ORACLE_ERR_GEOMETRY.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_INVALID 1
#define ORACLE_ERR_GEOMETRY 2

static int g_threads = 0; /* 0 = OpenMP default */

void oracle_set_threads(int n) { g_threads = n; }

int oracle_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* Eq. 6: full pressure including the incoming term. */
double oracle_pressure_full(double A, double r, double t, double v, double sigma) {
    double a = r - v * t, b = r + v * t, s2 = 2.0 * sigma * sigma;
    return A / (2.0 * r) * (a * exp(-(a * a) / s2) + b * exp(-(b * b) / s2));
}

/* Eq. 7 with the P:291 truncation |d| < k sigma. */
double oracle_pressure_outgoing(double A, double r, double t, double v, double sigma, double k) {
    double d = r - v * t;
    if (!(fabs(d) < k * sigma)) return 0.0;
    return A / (2.0 * r) * d * exp(-(d * d) / (2.0 * sigma * sigma));
}

/* Distance r_ij from the fp32 inputs promoted to fp64 (differences exact). */
static double pair_distance(const float* centers, int64_t M, int64_t i,
                            const float* sensors, int32_t Nd, int32_t j) {
    double dx = (double)centers[i] - (double)sensors[j];
    double dy = (double)centers[M + i] - (double)sensors[Nd + j];
    double dz = (double)centers[2 * M + i] - (double)sensors[2 * Nd + j];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

/* Candidate sample range for one pair (generous; membership tested per n). */
static void candidate_range(double r, double ks, double v, double fs, double t0,
                            int32_t Nt, int64_t* n0, int64_t* n1) {
    double lo = floor(((r - ks) / v - t0) * fs) - 2.0;
    double hi = ceil(((r + ks) / v - t0) * fs) + 2.0;
    if (lo < 0.0) lo = 0.0;
    if (hi > (double)(Nt - 1)) hi = (double)(Nt - 1);
    *n0 = (int64_t)lo;
    *n1 = (int64_t)hi;
}

static int check_args(int64_t M, int32_t Nd, int32_t Nt, double sigma, double v,
                      double fs, double k) {
    if (M < 0 || Nd < 1 || Nt < 1) return ORACLE_ERR_INVALID;
    if (!(sigma > 0.0) || !(v > 0.0) || !(fs > 0.0) || !(k > 0.0)) return ORACLE_ERR_INVALID;
    return ORACLE_OK;
}

/*
 * Forward: y[j_out][n] = sum_i amp[i] * a_ijn for the sensors listed in
 * `rows` (n_rows entries; rows == NULL means all N_d sensors in order).
 * centers: [3][M] SoA fp32 metres; sensors: [3][N_d] SoA fp32 metres;
 * sigmas: optional per-kernel sigma (NULL -> sigma); y: [n_rows][N_t] fp64.
 */
int oracle_forward(int64_t M, const float* centers, const double* amp,
                   double sigma, const double* sigmas,
                   int32_t Nd, const float* sensors,
                   double v, double fs, double t0, int32_t Nt, double k,
                   const int32_t* rows, int32_t n_rows, double* y) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc) return rc;
    if (rows == NULL) n_rows = Nd;
    int err = ORACLE_OK;
    int nth = oracle_get_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nth)
    for (int32_t jo = 0; jo < n_rows; ++jo) {
        int32_t j = rows ? rows[jo] : jo;
        double* yj = y + (int64_t)jo * Nt;
        for (int32_t n = 0; n < Nt; ++n) yj[n] = 0.0;
        for (int64_t i = 0; i < M; ++i) {
            double s = sigmas ? sigmas[i] : sigma;
            double ks = k * s;
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            if (!(r > ks)) {
#pragma omp atomic write
                err = ORACLE_ERR_GEOMETRY;
                continue;
            }
            int64_t n0, n1;
            candidate_range(r, ks, v, fs, t0, Nt, &n0, &n1);
            for (int64_t n = n0; n <= n1; ++n) {
                double t = t0 + (double)n / fs;
                double d = r - v * t;
                if (fabs(d) < ks) {
                    double a = d * exp(-(d * d) / (2.0 * s * s)) / (2.0 * r);
                    yj[n] += amp[i] * a;
                }
            }
        }
    }
    return err;
}

/*
 * Adjoint: g[i_out] = sum_j sum_n a_ijn * delta[j][n] for the kernels listed
 * in `cols` (n_cols entries; cols == NULL means all M kernels in order).
 * delta: [N_d][N_t] fp64 row-major; g: [n_cols] fp64.
 */
int oracle_adjoint(int64_t M, const float* centers,
                   double sigma, const double* sigmas,
                   int32_t Nd, const float* sensors,
                   double v, double fs, double t0, int32_t Nt, double k,
                   const double* delta, const int64_t* cols, int64_t n_cols,
                   double* g) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc) return rc;
    if (cols == NULL) n_cols = M;
    int err = ORACLE_OK;
    int nth = oracle_get_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nth)
    for (int64_t io = 0; io < n_cols; ++io) {
        int64_t i = cols ? cols[io] : io;
        double s = sigmas ? sigmas[i] : sigma;
        double ks = k * s;
        double acc = 0.0;
        for (int32_t j = 0; j < Nd; ++j) {
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            if (!(r > ks)) {
#pragma omp atomic write
                err = ORACLE_ERR_GEOMETRY;
                continue;
            }
            const double* dj = delta + (int64_t)j * Nt;
            int64_t n0, n1;
            candidate_range(r, ks, v, fs, t0, Nt, &n0, &n1);
            for (int64_t n = n0; n <= n1; ++n) {
                double t = t0 + (double)n / fs;
                double d = r - v * t;
                if (fabs(d) < ks) {
                    double a = d * exp(-(d * d) / (2.0 * s * s)) / (2.0 * r);
                    acc += a * dj[n];
                }
            }
        }
        g[io] = acc;
    }
    return err;
}

/*
 * Exact count of in-window samples (useful pair-samples) over all pairs,
 * used by bench.py / tests for the algorithmic work count of one operator.
 */
int64_t oracle_count_pair_samples(int64_t M, const float* centers, double sigma,
                                  int32_t Nd, const float* sensors,
                                  double v, double fs, double t0, int32_t Nt, double k,
                                  const int64_t* cols, int64_t n_cols) {
    if (cols == NULL) n_cols = M;
    int64_t total = 0;
    double ks = k * sigma;
    int nth = oracle_get_threads();
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : total) num_threads(nth)
    for (int64_t io = 0; io < n_cols; ++io) {
        int64_t i = cols ? cols[io] : io;
        for (int32_t j = 0; j < Nd; ++j) {
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            int64_t n0, n1;
            candidate_range(r, ks, v, fs, t0, Nt, &n0, &n1);
            for (int64_t n = n0; n <= n1; ++n) {
                double t = t0 + (double)n / fs;
                double d = r - v * t;
                if (fabs(d) < ks) total += 1;
            }
        }
    }
    return total;
}

/* ------------------------------------------------------------------------
 * Near-field operator: Eq. 6 with BOTH terms,
 * the outgoing (r - v t) and the incoming (r + v t) wave, each truncated to
 * |.| < k sigma like P:291 (reading N1), with an optional
 * per-kernel sigma_i (reading N2):
 *   a_ijn = [dm exp(-dm^2/(2 s^2)) 1(|dm| < k s) + dp exp(-dp^2/(2 s^2)) 1(|dp| < k s)] / (2 r)
 *   dm = r - v t_n,  dp = r + v t_n,  s = sigma_i,  t_n = t0 + n / f_s.
 * Eq. 6 holds for every r > 0 (its 1/r is the only singularity), so pairs
 * need r > 0 instead of r > k sigma; r = 0 returns ORACLE_ERR_GEOMETRY
 * (reading N3).  When the incoming window of a pair is empty the entry is
 * bit-identical to oracle_forward's (an added +0.0 changes nothing).
 * Candidates: the union of the outgoing range and the incoming range
 * n in [floor(((-k s - r)/v - t0) f_s) - 2, ceil(((k s - r)/v - t0) f_s) + 2].
 * ---------------------------------------------------------------------- */
static double nf_entry(double r, double s, double ks, double v, double t) {
    double dm = r - v * t, dp = r + v * t;
    double tm = 0.0, tp = 0.0;
    if (fabs(dm) < ks) tm = dm * exp(-(dm * dm) / (2.0 * s * s));
    if (fabs(dp) < ks) tp = dp * exp(-(dp * dp) / (2.0 * s * s));
    return (tm + tp) / (2.0 * r);
}

static void nf_range(double r, double ks, double v, double fs, double t0, int32_t Nt, int64_t* n0, int64_t* n1) {
    candidate_range(r, ks, v, fs, t0, Nt, n0, n1);
    double lo = floor(((-ks - r) / v - t0) * fs) - 2.0;
    double hi = ceil(((ks - r) / v - t0) * fs) + 2.0;
    if (lo < 0.0) lo = 0.0;
    if (hi > (double)(Nt - 1)) hi = (double)(Nt - 1);
    if (lo <= hi) {  /* non-empty incoming range: take the union */
        if ((int64_t)lo < *n0) *n0 = (int64_t)lo;
        if ((int64_t)hi > *n1) *n1 = (int64_t)hi;
    }
}

int oracle_forward_nf(int64_t M, const float* centers, const double* amp,
                      double sigma, const double* sigmas,
                      int32_t Nd, const float* sensors,
                      double v, double fs, double t0, int32_t Nt, double k,
                      const int32_t* rows, int32_t n_rows, double* y) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc) return rc;
    if (rows == NULL) n_rows = Nd;
    int err = ORACLE_OK;
    int nth = oracle_get_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nth)
    for (int32_t jo = 0; jo < n_rows; ++jo) {
        int32_t j = rows ? rows[jo] : jo;
        double* yj = y + (int64_t)jo * Nt;
        for (int32_t n = 0; n < Nt; ++n) yj[n] = 0.0;
        for (int64_t i = 0; i < M; ++i) {
            double s = sigmas ? sigmas[i] : sigma;
            double ks = k * s;
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            if (!(r > 0.0)) {
#pragma omp atomic write
                err = ORACLE_ERR_GEOMETRY;
                continue;
            }
            int64_t n0, n1;
            nf_range(r, ks, v, fs, t0, Nt, &n0, &n1);
            for (int64_t n = n0; n <= n1; ++n) {
                double t = t0 + (double)n / fs;
                yj[n] += amp[i] * nf_entry(r, s, ks, v, t);
            }
        }
    }
    return err;
}

int oracle_adjoint_nf(int64_t M, const float* centers,
                      double sigma, const double* sigmas,
                      int32_t Nd, const float* sensors,
                      double v, double fs, double t0, int32_t Nt, double k,
                      const double* delta, const int64_t* cols, int64_t n_cols,
                      double* g) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc) return rc;
    if (cols == NULL) n_cols = M;
    int err = ORACLE_OK;
    int nth = oracle_get_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nth)
    for (int64_t io = 0; io < n_cols; ++io) {
        int64_t i = cols ? cols[io] : io;
        double s = sigmas ? sigmas[i] : sigma;
        double ks = k * s;
        double acc = 0.0;
        for (int32_t j = 0; j < Nd; ++j) {
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            if (!(r > 0.0)) {
#pragma omp atomic write
                err = ORACLE_ERR_GEOMETRY;
                continue;
            }
            const double* dj = delta + (int64_t)j * Nt;
            int64_t n0, n1;
            nf_range(r, ks, v, fs, t0, Nt, &n0, &n1);
            for (int64_t n = n0; n <= n1; ++n) {
                double t = t0 + (double)n / fs;
                acc += nf_entry(r, s, ks, v, t) * dj[n];
            }
        }
        g[io] = acc;
    }
    return err;
}

/* ------------------------------------------------------------------------
 * ASSA operator: the paper's discrete operator,
 * Eqs. 8-17 and Algorithm 1, stage by stage:
 *   Eq. 9 projection P_up:  k_ij = floor((r_ij/v - t0) f_s^up + 0.5)
 *          z_j[k] = sum_i x_i / r_ij 1(k = k_ij),  k = 0 .. N_t^up - 1
 *   Eq. 11 taps h[k] = C d[k] exp(-d[k]^2 / (2 sigma^2)),
 *          d[k] = -v k dt_up, k = -K .. K  (C = 1/2: reading A1)
 *   Eq. 10 transposed convolution zt_j[k] = sum_m z_j[m] h[k - m]
 *   Eq. 12 decimation y_j[n] = zt_j[alpha n]
 *   Eqs. 15-17 adjoint: zero-fill, correlation with the
 *          time-reversed taps, back-projection g_i = sum_j dconv_j[k_ij] / r_ij
 * t0 (reading R3) shifts the upsampled grid: t_k = t0 + k dt_up.  Impulses
 * with k_ij outside [0, N_t^up) do not exist (the indicator of Eq. 9 never
 * fires); convolution sums run over the record only (reading A3).
 * ---------------------------------------------------------------------- */

/* Eq. 11 taps, fp64, h[k + K] for k = -K..K. */
void oracle_assa_taps(double v, double fs_up, double sigma, int32_t K, double C, double* h) {
    double dt_up = 1.0 / fs_up;
    for (int32_t k = -K; k <= K; ++k) {
        double d = -v * (double)k * dt_up;
        h[k + K] = C * d * exp(-(d * d) / (2.0 * sigma * sigma));
    }
}

/* Eq. 9 aligned index. */
static int64_t assa_index(double r, double v, double t0, double fs_up) {
    return (int64_t)floor((r / v - t0) * fs_up + 0.5);
}

int oracle_assa_forward(int64_t M, const float* centers, const double* amp, int32_t Nd, const float* sensors,
                        double v, double fs, double t0, int32_t Nt, double sigma, double k, int32_t alpha,
                        int32_t K, const int32_t* rows, int32_t n_rows, double* y) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc || alpha < 1 || K < 0) return rc ? rc : ORACLE_ERR_INVALID;
    if (rows == NULL) n_rows = Nd;
    const double fs_up = (double)alpha * fs;
    const int64_t Nt_up = (int64_t)alpha * Nt;
    const double ks = k * sigma;
    double* h = (double*)malloc(sizeof(double) * (2 * K + 1));
    oracle_assa_taps(v, fs_up, sigma, K, 0.5, h);
    int err = ORACLE_OK;
    int nth = oracle_get_threads();
#pragma omp parallel num_threads(nth)
    {
        double* z = (double*)malloc(sizeof(double) * Nt_up);
#pragma omp for schedule(dynamic, 1)
        for (int32_t jo = 0; jo < n_rows; ++jo) {
            int32_t j = rows ? rows[jo] : jo;
            for (int64_t q = 0; q < Nt_up; ++q) z[q] = 0.0;
            /* 1. P_up (Eq. 9) */
            for (int64_t i = 0; i < M; ++i) {
                double r = pair_distance(centers, M, i, sensors, Nd, j);
                if (!(r > ks)) {
#pragma omp atomic write
                    err = ORACLE_ERR_GEOMETRY;
                    continue;
                }
                int64_t kij = assa_index(r, v, t0, fs_up);
                if (kij >= 0 && kij < Nt_up) z[kij] += amp[i] / r;
            }
            /* 2. transposed convolution (Eq. 10) at the decimated points (Eq. 12) */
            double* yj = y + (int64_t)jo * Nt;
            for (int32_t n = 0; n < Nt; ++n) {
                int64_t kk = (int64_t)alpha * n;
                double acc = 0.0;
                for (int64_t m = kk - K; m <= kk + K; ++m) {
                    if (m < 0 || m >= Nt_up) continue;
                    acc += z[m] * h[(kk - m) + K];
                }
                yj[n] = acc;
            }
        }
        free(z);
    }
    free(h);
    return err;
}

int oracle_assa_adjoint(int64_t M, const float* centers, int32_t Nd, const float* sensors, double v, double fs,
                        double t0, int32_t Nt, double sigma, double k, int32_t alpha, int32_t K,
                        const double* delta, const int64_t* cols, int64_t n_cols, double* g) {
    int rc = check_args(M, Nd, Nt, sigma, v, fs, k);
    if (rc || alpha < 1 || K < 0) return rc ? rc : ORACLE_ERR_INVALID;
    if (cols == NULL) n_cols = M;
    const double fs_up = (double)alpha * fs;
    const int64_t Nt_up = (int64_t)alpha * Nt;
    const double ks = k * sigma;
    double* h = (double*)malloc(sizeof(double) * (2 * K + 1));
    oracle_assa_taps(v, fs_up, sigma, K, 0.5, h);
    double* dconv = (double*)malloc(sizeof(double) * (size_t)Nd * Nt_up);
    int nth = oracle_get_threads();
    /* 1. zero-fill (Eq. 15) and 2. correlation with h-bar[k] = h[-k] (Eq. 16) */
#pragma omp parallel for schedule(dynamic, 1) num_threads(nth)
    for (int32_t j = 0; j < Nd; ++j) {
        double* dc = dconv + (int64_t)j * Nt_up;
        for (int64_t q = 0; q < Nt_up; ++q) {
            double acc = 0.0;
            for (int64_t m = q - K; m <= q + K; ++m) {
                if (m < 0 || m >= Nt_up || (m % alpha) != 0) continue;  /* delta_up[m] = 0 off-grid */
                acc += h[(m - q) + K] * delta[(int64_t)j * Nt + m / alpha];
            }
            dc[q] = acc;
        }
    }
    /* 3. back-projection (Eq. 17) */
    int err = ORACLE_OK;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nth)
    for (int64_t io = 0; io < n_cols; ++io) {
        int64_t i = cols ? cols[io] : io;
        double acc = 0.0;
        for (int32_t j = 0; j < Nd; ++j) {
            double r = pair_distance(centers, M, i, sensors, Nd, j);
            if (!(r > ks)) {
#pragma omp atomic write
                err = ORACLE_ERR_GEOMETRY;
                continue;
            }
            int64_t kij = assa_index(r, v, t0, fs_up);
            if (kij >= 0 && kij < Nt_up) acc += dconv[(int64_t)j * Nt_up + kij] / r;
        }
        g[io] = acc;
    }
    free(dconv);
    free(h);
    return err;
}
