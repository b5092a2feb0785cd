/*
 * gpair.h -- C ABI of the B200-native GPAIR hot path (libgpair.so).
 *
 * Implements the closed-form Gaussian-kernel forward operator, its exact
 * adjoint and the fused update of the iterative reconstruction of
 * "GPAIR: Gaussian-Kernel-Based Ultrafast 3D Photoacoustic Iterative
 * Reconstruction" (arXiv 2602.03893).  Citations P:<line> refer to that
 * paper's text; readings R<n> are listed in DESIGN.md.
 *
 * Operator (Eq. 7, with the 3-sigma truncation of P:291 and the
 * direct pair enumeration of P:295):
 *
 *   a_ijn = d exp(-d^2 / (2 sigma^2)) / (2 r_ij)  if |d| < k sigma, else 0
 *   r_ij  = |c_i - s_j|,  d = r_ij - v t_n,  t_n = t0 + n / f_s   (R3)
 *   forward:  y_j[n] = sum_i A_i a_ijn          (superposition)
 *   adjoint:  g_i    = sum_j sum_n a_ijn delta_j[n]   (transpose)
 *
 * Conventions (apply to every call unless stated):
 *   - Every array pointer is a DEVICE pointer (cudaMalloc / torch CUDA
 *     tensor) on the device current when gpair_create was called, fp32,
 *     contiguous, unless the comment says "host".
 *   - Layouts: kernel centres and sensor positions are SoA [3][n] (x row, y
 *     row, z row), metres.  Signals y, b, residuals are row-major
 *     [N_d][N_t] (detector-major).  Per-kernel vectors are [M_local]
 *     in the caller's kernel order; the spatial permutation is internal.
 *   - Ownership: the caller owns every buffer passed in.  gpair_create copies
 *     what it needs (centres, sensors) and keeps no caller pointer except the
 *     borrowed nccl_comm, which must outlive the context.
 *   - Outputs are overwritten, never accumulated into.
 *   - Asynchrony: calls other than gpair_create/gpair_destroy enqueue work
 *     on `stream` (a cudaStream_t; NULL = legacy default stream) and return
 *     without synchronising.  Argument and geometry validation errors are
 *     returned synchronously before anything is enqueued; asynchronous CUDA
 *     or NCCL faults are sticky and reported by the next call.
 *   - Errors: a non-GPAIR_OK status leaves outputs unspecified; the message
 *     is available from gpair_last_error(ctx).
 *   - Threading: a context is not thread-safe; use one context per rank
 *     (device).  The library never calls exit() or prints.
 */
#ifndef GPAIR_H
#define GPAIR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpair_ctx_s gpair_ctx;

typedef enum {
    GPAIR_OK = 0,
    GPAIR_ERR_INVALID_ARGUMENT = 1, /* bad size, NULL, non-positive or non-finite scalar */
    GPAIR_ERR_GEOMETRY = 2,         /* some r_ij <= k sigma (far-field Eq. 7 invalid), or
                                       kernel cloud too sparse for cell anchoring */
    GPAIR_ERR_RESOURCE = 3,         /* allocation failure, int32 index overflow, smem too small */
    GPAIR_ERR_NUMERICAL = 4,        /* non-finite loss when GPAIR_CHECK_FINITE is set */
    GPAIR_ERR_CUDA = 5,             /* CUDA runtime / launch error (no device, bad pointer, ...) */
    GPAIR_ERR_NCCL = 6              /* NCCL not loadable or a collective failed */
} gpair_status;

/* gpair_desc.flags */
enum {
    GPAIR_TOF_EXACT = 0,        /* Eq. 7 evaluated at the exact time of flight (this build) */
    GPAIR_TOF_ASSA = 1,         /* the paper's ASSA operator (Eqs. 8-17, Alg. 1):
                                   ToF snapped to the alpha-upsampled grid, k_ij =
                                   floor((r/v - t0) f_s^up + 0.5); taps h[k] = (1/2) d[k]
                                   exp(-d[k]^2/2 sigma^2), d[k] = -v k dt_up, |k| <= K;
                                   y_j[n] = sum_i (A_i / r_ij) h[alpha n - k_ij]; the adjoint
                                   is its exact transpose (zero-fill, correlation,
                                   back-projection).  Impulses with k_ij outside
                                   [0, alpha N_t) do not exist (reading A3). */
    GPAIR_NEAR_FIELD = 1 << 1,  /* near-field operator (N1-N3):
                                   Eq. 6 with BOTH terms, each truncated to
                                   |.| < k sigma_i:  a_ijn = [dm e^{-dm^2/2s^2} 1(|dm|<ks)
                                   + dp e^{-dp^2/2s^2} 1(|dp|<ks)] / (2 r),  dm = r - v t_n,
                                   dp = r + v t_n.  Pairs need only r > 0 (GEOMETRY if some
                                   r = 0).  Exact operator only (not with GPAIR_TOF_ASSA). */
    GPAIR_COLLECTIVE = 1 << 2,  /* take the kernel-sharded (collective) path even at world = 1:
                                   the NCCL all-reduce of y, the separate residual kernel, the
                                   per-group all-reduces of the pipeline and the R_VCR exchange
                                   run as at world > 1 (with a 1-rank communicator they are
                                   identities).  Implied by world > 1.  Needs nccl_comm. */
    GPAIR_CHECK_FINITE = 1 << 9 /* gpair_iterate syncs and checks the loss is finite */
};

/* Problem description (P:230-233 kernels, P:319 sensors, P:251 v, P:303-309 f_s, N_t). */
typedef struct {
    double sound_speed;    /* v [m/s] > 0                                         */
    double sampling_rate;  /* f_s [Hz] > 0                                 */
    int32_t n_samples;     /* N_t >= 1                                            */
    double t0;             /* time of sample 0 [s] (R3); t_n = t0 + n / f_s              */
    int64_t n_kernels;     /* M_local >= 1: kernels owned by this rank            */
    const float* centers;  /* DEVICE [3][M_local] SoA centres c_i [m], caller order      */
    double sigma;          /* Gaussian std-dev [m] > 0, shared by all kernels    */
    const float* sigmas;   /* DEVICE [M_local] per-kernel sigma_i > 0 [m] (row f4, N2), read
                              during create only; NULL -> `sigma` for every kernel.  Not
                              with GPAIR_TOF_ASSA.  With sigmas and without
                              GPAIR_NEAR_FIELD the r > k sigma check uses max sigma_i    */
    double window_k;       /* k in |d| < k sigma; paper: 3                        */
    int32_t n_sensors;     /* N_d >= 1                                                    */
    const float* sensors;  /* DEVICE [3][N_d] SoA point-detector positions [m]   */
    int32_t rank, world;   /* kernel-shard index / count; world >= 1                      */
    void* nccl_comm;       /* ncclComm_t over `world` ranks (borrowed), or NULL at world = 1
                              without GPAIR_COLLECTIVE.  Its size and rank must equal
                              world and rank (INVALID_ARGUMENT otherwise)               */
    int32_t flags;         /* GPAIR_TOF_EXACT or GPAIR_TOF_ASSA, | GPAIR_CHECK_FINITE      */
    int32_t assa_nmin;     /* ASSA N_min ("set to 25"); <= 0 -> 25; ignored unless ASSA */
} gpair_desc;

/* One IR iteration's hyper-parameters (Algorithm 2). */
typedef struct {
    float lr;          /* eta_t for this iteration (caller computes, e.g. gpair_cawr_lr) */
    float beta1;       /* Adam beta1, 0.9 (R11)                                          */
    float beta2;       /* Adam beta2, 0.999 (R11)                                        */
    float adam_eps;    /* Adam epsilon, 1e-8 (R11)                                       */
    float eps_npc;     /* NPC epsilon, 1e-8                                      */
    float grad_scale;  /* dL/dy = grad_scale (y - b); <= 0 -> 2/(N_d N_t) (R10)          */
    int32_t step;      /* 1-based Adam step count t >= 1 (bias correction)               */
    int32_t mode;      /* 0 = NPC x=(z+eps)^2 + Adam (paper);
                          1 = clamp: state z holds x, x <- max(x - lr g, 0) (R15)       */
    /* Vessel continuity regularisation (Eqs. 20-23; row f2).
     * lam = 0 disables it (the paper's lambda = 0 runs).  lam > 0 needs the
     * kernels in grid order i = ix + nx (iy + ny iz) (the order R_VCR's
     * differences use): at world == 1 grid[0] grid[1] grid[2] == M; at
     * world > 1 grid is the GLOBAL grid and each rank's M_local kernels are
     * the z planes [z0, z0 + M_local / (nx ny)) (>= 2 planes), ranks in z
     * order (rank 0 from z0 = 0, the last rank up to n_z), and every rank must
     * first call gpair_vcr_prepare(grid, z0) (INVALID_ARGUMENT otherwise).  The library then
     * exchanges 2 halo planes of z with ranks r-1 and r+1 (ncclSend/ncclRecv)
     * and all-reduces the fp64 value of R_VCR (8 bytes); the gradient stays
     * rank-local. */
    float lam;         /* lambda of Eq. 23 (>= 0)                                        */
    float beta;        /* beta of Eq. 20: R_VCR = R_H + beta R_TV                        */
    float eps_reg;     /* smoothing epsilon inside both square roots (V4), > 0           */
    int32_t grid[3];   /* (n_x, n_y, n_z) voxel grid of the kernel order                 */
    int32_t z0;        /* world > 1, lam > 0: first global z plane of this rank's slab    */
} gpair_step;

/* Accumulated device time of the library's own kernels (gpair_profile_*). */
enum {
    GPAIR_PROF_GATHER = 0,   /* amplitude gather (+NPC) into the spatial order      */
    GPAIR_PROF_FORWARD = 1,  /* forward pair evaluation (dominant)                  */
    GPAIR_PROF_REDUCE = 2,   /* region partials -> y (+ residual, loss partials)    */
    GPAIR_PROF_ALLREDUCE = 3,/* ncclAllReduce of y (world > 1)                      */
    GPAIR_PROF_RESIDUAL = 4, /* residual + loss (world > 1 only)                    */
    GPAIR_PROF_ADJOINT = 5,  /* adjoint gather (+ fused update) (dominant)          */
    GPAIR_PROF_LOSS = 6,     /* loss finalisation                                   */
    GPAIR_PROF_VCR = 7,      /* VCR terms + gradient (lam > 0 only)                 */
    GPAIR_PROF_N = 8
};
typedef struct {
    double ms[GPAIR_PROF_N];       /* summed CUDA-event durations [ms]                */
    int64_t launches[GPAIR_PROF_N];/* number of timed launches                        */
    int64_t kernels;               /* library kernels launched by the per-call entry
                                      points since gpair_profile_enable (counted whether
                                      or not events are recorded)                       */
} gpair_profile;

/* Static description of what gpair_create built (for benchmarks and tests). */
typedef struct {
    int64_t n_kernels;          /* M_local                                              */
    int64_t n_kernels_padded;   /* rounded up to whole 32-kernel cells                  */
    int32_t n_cells;            /* 32-kernel spatial cells                              */
    int32_t fwd_region_cells;   /* cells per forward region                              */
    int32_t fwd_regions;        /* forward regions                                      */
    int32_t fwd_window;         /* per-(region, sensor) window length (padded)          */
    int32_t fwd_warps;          /* sensor warps per forward CTA                         */
    int32_t adj_region_cells;   /* cells (= warps) per adjoint CTA                       */
    int32_t adj_regions;        /* adjoint CTAs                                         */
    int32_t adj_window;         /* per-(region, sensor) residual window length          */
    int32_t wmax;               /* max in-window samples per pair (unrolled length)      */
    int32_t grid_detected;      /* 1 if centres were recognised as a regular grid        */
    double max_eps;             /* max |q|/R^2 of the anchor expansion       */
    int64_t workspace_bytes;    /* device bytes owned by the context                    */
    int32_t assa;               /* 1 if the context implements the ASSA operator        */
    int32_t assa_alpha;         /* ASSA upsampling ratio alpha (Eq. 8)                  */
    int32_t assa_n_half;        /* ASSA N_half (Eq. 8)                                  */
    int32_t assa_K;             /* ASSA taps half-width K = alpha N_half (Eq. 11)       */
    int32_t general;            /* 1: per-kernel sigma and/or near-field path (row f4)   */
    int32_t near_rows;          /* sensors with near-field pairs                        */
    int64_t near_pairs;         /* pairs evaluated with both Eq. 6 terms (r < k sigma_i) */
    int32_t tab;                /* 1: factorised-Gaussian (TAB) forward path, 3 MUFU per pair */
    int32_t adj_kernel;         /* adjoint kernel: 0 = lane per kernel (k_adjoint),
                                   1 = sensor lanes + TAB (k_adjoint_t),
                                   2 = sensor lanes + lane-centred factorisation (k_adjoint_lcf),
                                   3 = sensor lanes + per-sample exponential (k_adjoint_sl),
                                   4 = lane per kernel + moment polynomial (k_adjoint_mp) */
    int32_t collective;         /* 1: kernel-sharded path (NCCL all-reduce of y, separate
                                   residual kernel): world > 1 or GPAIR_COLLECTIVE          */
    int32_t fwd_union;          /* 1: register-window forward (opt-in GPAIR_FWD_UNION=1) */
    double adj_fit_err;         /* moment-polynomial adjoint: max error of the degree-7 interpolants of the
                                   window weights / max |f| (create-time fit; 0 when not attempted)   */
    int32_t adj_row_bytes;      /* moment-polynomial adjoint: bytes per staged moment row (32 or 48; ASSA 4) */
} gpair_info;

/* Create a context: validates `d`, sorts the kernels into 32-kernel spatial
 * cells, builds per-(region, sensor) sample windows and allocates
 * workspaces.  Runs on `stream` and synchronises it before returning.
 * Errors: INVALID_ARGUMENT, GEOMETRY (r_ij <= k sigma_i for some pair: cells
 * whose bounding sphere comes within k sigma of a sensor are tested pair by
 * pair in fp64 with the oracle's operations, so exactly the geometries the
 * oracle rejects are rejected), RESOURCE, CUDA.  *out is NULL on error. */
gpair_status gpair_create(gpair_ctx** out, const gpair_desc* d, void* stream);

/* Forward operator (Eq. 7 summed over kernels).
 * amplitudes: DEVICE [M_local] A_i (caller order).
 * signals:    DEVICE [N_d][N_t] output y; with world > 1 the sum over all
 *             ranks (ncclAllReduce in place), identical on every rank. */
gpair_status gpair_forward(gpair_ctx* ctx, const float* amplitudes, float* signals, void* stream);

/* Adjoint operator (exact transpose of gpair_forward).
 * residual: DEVICE [N_d][N_t] delta (replicated on every rank).
 * grad:     DEVICE [M_local] output g_i = sum_j sum_n a_ijn delta_j[n]. */
gpair_status gpair_adjoint(gpair_ctx* ctx, const float* residual, float* grad, void* stream);

/* Vessel continuity regulariser R_VCR = R_H + beta R_TV (Eqs. 20-22,
 * P:457-481) with the difference operators of DESIGN.md readings V1-V3:
 *   R_TV = sum_i sqrt(sum_d (D_d x_i)^2 + eps),   D_d forward difference, 0 on
 *          the last index;
 *   R_H  = sum_i sqrt(sum_d (D_dd x_i)^2 + 2 sum_{p<q} (D_pq x_i)^2 + eps),
 *          D_dd = [1,-2,1] centred at clamp(i_d, 1, n_d - 2) (0 if n_d < 3),
 *          D_pq forward-forward cross difference, 0 on the last index of p or q.
 * grid:  HOST int32[3] (n_x, n_y, n_z) >= 1; M = n_x n_y n_z.
 * x:     DEVICE [M] image, index i = ix + n_x (iy + n_y iz).
 * grad:  DEVICE [M] output dR/dx, or NULL.
 * value: DEVICE float scalar R_VCR(x) (fp64-accumulated), or NULL.
 * Needs only a context for its workspace (any M; reallocated on change).
 * Errors: INVALID_ARGUMENT (NULL x, bad grid, eps <= 0, non-finite beta), CUDA. */
gpair_status gpair_vcr(gpair_ctx* ctx, const int32_t* grid, const float* x, float beta, float eps,
                       float* grad, float* value, void* stream);

/* R_VCR restricted to a z slab (the kernel-sharded form of gpair_vcr, row f2;
 * the same operators and readings V1-V4).  The own planes [z0, z0 + nz_own)
 * of the GLOBAL grid get their exact gradient entries of the whole-grid
 * R_VCR, and value receives the whole-grid sum restricted to the own voxels,
 * so the slabs' values add up to gpair_vcr's value and their gradients
 * concatenate to its gradient.
 * grid:   HOST int32[3] global (n_x, n_y, n_z).
 * x_ext:  DEVICE image on the planes [ext_z0, ext_z0 + ext_nz), which must
 *         contain [max(0, z0 - 2), min(n_z, z0 + nz_own + 2)) (the halo the
 *         stencils and their adjoints reach); index ix + n_x (iy + n_y (iz - ext_z0)).
 * grad:   DEVICE [n_x n_y nz_own] output, or NULL.  value: DEVICE float, or NULL.
 * Errors: INVALID_ARGUMENT (as gpair_vcr; slab outside the grid; halo not
 * covered), CUDA. */
gpair_status gpair_vcr_slab(gpair_ctx* ctx, const int32_t* grid, int32_t z0, int32_t nz_own,
                            const float* x_ext, int32_t ext_z0, int32_t ext_nz, float beta,
                            float eps, float* grad, float* value, void* stream);

/* Validate and set up the slab layout of R_VCR for gpair_iterate with lam > 0
 * (row f2).  Required on the collective path (world > 1
 * or GPAIR_COLLECTIVE), optional at world = 1 (it then only pre-allocates, so
 * the first iterate allocates nothing and stays CUDA-graph capturable).
 * grid: HOST int32[3] GLOBAL (n_x, n_y, n_z); z0: first global z plane of this
 * rank's kernels (M_local / (n_x n_y) whole planes, >= 2 at world > 1).
 * Collective on the collective path: every rank must call it; the ranks
 * exchange (z0, n_z,own, ok) in one all-reduce and all return the same
 * verdict, so a bad layout on one rank never leaves the others blocked in
 * the halo exchange.  Synchronises `stream`.  Allocates the halo buffer and
 * the R_VCR workspace.  Errors: INVALID_ARGUMENT (slabs not whole planes,
 * not contiguous in rank order, not covering n_z; bad grid), CUDA, NCCL. */
gpair_status gpair_vcr_prepare(gpair_ctx* ctx, const int32_t* grid, int32_t z0, void* stream);

/* One iteration of Algorithm 2:
 *   x = (z + eps)^2 (mode 0) or x = z (mode 1);  y = A x  [+ allreduce];
 *   L = (1/N) |y - b|^2 + lam R_VCR(x);
 *   g = A^T (grad_scale (y - b)) + lam grad R_VCR(x);
 *   mode 0: dz = g 2 (z + eps); Adam step on (z, m, v) with s->lr, s->step;
 *   mode 1: z = max(z - lr g, 0).
 * z, m, v:     DEVICE [M_local] in/out state (m, v unused in mode 1, may be NULL).
 * b:           DEVICE [N_d][N_t] measured signals.
 * signals_out: DEVICE [N_d][N_t] y of this iteration, or NULL.
 * x_out:       DEVICE [M_local] x of the UPDATED state, or NULL.
 * loss_out:    DEVICE float scalar L (of the pre-update state), or NULL. */
gpair_status gpair_iterate(gpair_ctx* ctx, float* z, float* m, float* v, const float* b,
                           const gpair_step* s, float* signals_out, float* x_out,
                           float* loss_out, void* stream);

/* Exact number of in-window pair-samples (|d| < k sigma, n in [0, N_t)) of
 * this rank's operator; for an ASSA context, the number of existing impulses
 * (pairs with k_ij in [0, alpha N_t)).  Synchronous.  Host output.
 * INVALID_ARGUMENT for per-kernel-sigma / near-field contexts. */
gpair_status gpair_count_pair_samples(gpair_ctx* ctx, int64_t* out_host, void* stream);

/* Fill *out (host struct) with the context's build parameters. */
gpair_status gpair_get_info(const gpair_ctx* ctx, gpair_info* out);

/* Release all device memory and events of the context (synchronises). NULL ok. */
gpair_status gpair_destroy(gpair_ctx* ctx);

/* Per-kernel device timing with CUDA events recorded on the launch stream.
 * enable != 0 starts accumulating (and resets the counters); read
 * synchronises the pending events and copies the totals to *out (host). */
gpair_status gpair_profile_enable(gpair_ctx* ctx, int enable);
gpair_status gpair_profile_read(gpair_ctx* ctx, gpair_profile* out);

/* CAWR learning rate, Eq. 24, host function.
 * printed_formula != 0: T_cur = t mod T0, T_i = T0 Tmult^floor(t/T0) as
 * printed (R13); 0: SGDR restarts (identical when Tmult = 1).
 * Returns NaN for T0 < 1 or Tmult < 1 or t < 0. */
double gpair_cawr_lr(int64_t t, double eta_min, double eta_max, int64_t T0, int64_t Tmult,
                     int printed_formula);

/* NCCL bootstrap helpers (host).  NCCL is loaded with dlopen("libnccl.so.2")
 * at first use.  unique_id: host buffer of 128 bytes (ncclUniqueId).
 * comm_out receives an ncclComm_t to pass as gpair_desc.nccl_comm. */
gpair_status gpair_nccl_unique_id(void* unique_id_host128);
gpair_status gpair_nccl_comm_init(void** comm_out, int32_t world, const void* unique_id_host128,
                                  int32_t rank);
gpair_status gpair_nccl_comm_destroy(void* comm);

/* Static strings; never NULL. */
const char* gpair_strerror(gpair_status s);
const char* gpair_last_error(const gpair_ctx* ctx); /* host string valid until the next call */
const char* gpair_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GPAIR_H */
