/*
 * splidar.h — C ABI of libsplidar.so, the B200 (sm_100a) hot path of arXiv 2509.20500
 * ("non-sequential Markov modelling of asynchronous SP-LiDAR timestamps under dead time").
 *
 * Citations: "P:NN" is line NN of the paper's text, with its section/equation.
 *
 * The path:
 *   1. flux vectors   lambda_j = lambda(s_j) (Eq. 1), the cumulative flux
 *                     F_j = F(s_j) = int_0^{s_j} lambda (Thm 1) by a warp+block prefix sum of
 *                     exact per-bin flux masses, Lambda = F(t_r), and the row normalisers.
 *   2. base matrix    P~0 = rownorm((1 lambda^T) . exp.(-Lambda L - D))   (§3.4):
 *                     P~0[r][j] = lambda_j exp(F_r - F_j - Lambda [r > j]) / Z_r.
 *   3. dead time      P~ = J_l P~0, row i of P~ is row (i + l) mod N of P~0, l = ceil(x_d / Delta),
 *                     x_d = t_d mod t_r (Thm 2). Folded into the solver's vector
 *                     gather; materialised only by splidar_apply_deadtime.
 *   4. stationary pdf pi P~ = pi by power iteration on the device.
 *
 * Conventions for every entry point:
 *   - Times (t_r, t_d, tau, sigma) share one unit (ns in the benchmarks). S and B are mean photons
 *     per laser period. Bins: Delta = t_r / n_bins, centres s_j = (j + 1/2) Delta,
 *     j = 0..N-1.
 *   - Matrices are row-major with leading dimension ld (elements), ld >= N, ld * sizeof(dtype) a
 *     multiple of 16 bytes and the base pointer 16-byte aligned (else SPLIDAR_ENOSPACE).
 *     Storage is fp64 or fp32 (splidar_dtype); every vector, every scan and every GEMV
 *     accumulation is fp64 regardless.
 *   - Device pointers are cudaMalloc'd / torch CUDA memory on the current device; host pointers
 *     are ordinary host memory. The caller owns every buffer; the library allocates nothing on
 *     the device, keeps no global state besides the last CUDA error code, and is re-entrant for
 *     distinct (stream, workspace) pairs.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Argument errors are returned synchronously, before anything is enqueued.
 *   - Entry points marked "async" only enqueue work on `stream`; the others synchronise `stream`
 *     exactly once at their end.
 */
#ifndef SPLIDAR_H
#define SPLIDAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPLIDAR_OK = 0,
    SPLIDAR_EINVAL = 1,   /* an argument violates an invariant (checked on the host, nothing enqueued) */
    SPLIDAR_ENOCONV = 2,  /* max_iter reached before the L1 change fell below tol; pi holds the last
                             iterate and info.l1_change the last change (not silently accepted) */
    SPLIDAR_EZEROROW = 3, /* a row normaliser D_r was zero or non-finite on the device */
    SPLIDAR_ENOSPACE = 4, /* workspace too small, ld < N, or a pointer / ld not 16-byte aligned */
    SPLIDAR_ECUDA = 5     /* CUDA runtime error; splidar_last_cuda_error() returns its code */
} splidar_status;

typedef enum { SPLIDAR_F64 = 0, SPLIDAR_F32 = 1 } splidar_dtype;   /* storage of P~0 / P~ */

/* How an entry of P~0 is evaluated (both compute the same matrix, §3.4):
 *   SPLIDAR_ENTRY_EXP:      lambda_j * exp(F_r - F_j - Lambda [r > j]) * (1 / Z_r), one exp per
 *                           entry (the paper's exp.(-Lambda L - D); fp64 exp for fp64 storage,
 *                           ex2.approx for fp32 storage).
 *   SPLIDAR_ENTRY_FACTORED: w_j * (r > j ? e^{-Lambda} : 1) * (1 / D_r), w_j = lambda_j e^{-F_j},
 *                           D_r = Z_r e^{-F_r}: the same product with e^{F_r} cancelled by the
 *                           row normalisation; no transcendental per entry. Default. */
typedef enum { SPLIDAR_ENTRY_FACTORED = 0, SPLIDAR_ENTRY_EXP = 1 } splidar_entry;

/* The problem statement theta without t_d: Eq. 1 generalised to K Gaussian pulses
 * lambda(t) = sum_k S_k N(t; tau_k, sigma_k^2) + B / t_r on [0, t_r); K = 1 is the paper.
 * All pointers are HOST pointers to K doubles. Invariants (else SPLIDAR_EINVAL): t_r > 0 finite;
 * 2 <= n_bins <= 2^20; 0 <= n_pulses <= SPLIDAR_MAX_PULSES; sigma_k > 0; S_k >= 0;
 * 0 <= tau_k < t_r; background B > 0 (a positive floor keeps the chain irreducible);
 * sum_k S_k + B <= 600 (keeps e^{-F} representable in fp64). */
#define SPLIDAR_MAX_PULSES 16
typedef struct {
    double t_r;            /* laser repetition period                  */
    int32_t n_bins;        /* N = n_b; bin width Delta = t_r / N       */
    int32_t n_pulses;      /* K                                               */
    const double *tau;     /* host [K] pulse centres (depth delay)      */
    const double *sigma;   /* host [K] pulse widths sigma_t            */
    const double *signal;  /* host [K] S_k = alpha E, photons / period */
    double background;     /* B = t_r lambda_b, photons / period       */
} splidar_flux;

typedef struct {
    int32_t iters;        /* power-iteration products pi P~ taken                          */
    int32_t converged;    /* 1 if the last L1 change was below tol                         */
    int32_t shift_l;      /* l = ceil(x_d / Delta) mod N used for the dead time (Thm 2)    */
    int32_t reserved;
    double l1_change;     /* last || pi^k P~ - pi^k ||_1                                   */
    double lambda_total;  /* Lambda = F(t_r) as computed on the device (0 if not computed) */
} splidar_solve_info;

/* Shift rule (Thm 2): l = ceil(u) mod N with u = fmod(t_d, t_r) * N / t_r in fp64
 * (the single definition used everywhere; l = N is the same as 0). Host only, synchronous.
 * t_r > 0, N >= 2, t_d >= 0, all finite, else SPLIDAR_EINVAL. */
splidar_status splidar_shift(double t_r, int32_t n_bins, double t_d, int32_t *l_out);

/* Device workspace (bytes) for n_matrices base matrices of N bins solved with up to n_vectors
 * dead times each (n_vectors <= 32). Any workspace at least this large, 256-byte aligned, may
 * be passed to every entry point below with the same or smaller sizes. */
size_t splidar_workspace_bytes(int32_t n_bins, int32_t n_matrices, int32_t n_vectors);

/* Steps 1a-1c of the path for one flux (async): writes the device vectors that the matrix is
 * built from. Any output pointer may be NULL. F[j] = F(s_j) (prefix sum of exact bin masses,
 * Thm 1), lam[j] = lambda(s_j) (Eq. 1), w[j] = lam[j] e^{-F[j]},
 * inv_d[j] = 1 / D_j with D_r = sum_{j>=r} w_j + e^{-Lambda} sum_{j<r} w_j (row sum of
 * exp.(-Lambda L - D) (1 lambda^T) divided by e^{F_r}), lambda_total[0] = Lambda = F(t_r).
 * All outputs are device fp64 arrays of N (lambda_total: 1). */
splidar_status splidar_flux_vectors(const splidar_flux *flux, double *F, double *lam, double *w,
                                    double *inv_d, double *lambda_total, void *ws, size_t ws_bytes,
                                    void *stream);

/* Step 2 (async): the normalised dead-time-free base matrix P~0 (§3.4, normalisation
 * P:79) into P0 (device, N x ld, dtype dt). Columns [N, ld) are not written. */
splidar_status splidar_build_base(const splidar_flux *flux, splidar_dtype dt, splidar_entry mode,
                                  void *P0, int64_t ld, void *ws, size_t ws_bytes, void *stream);

/* Step 2 for n_matrices fluxes at once (async): matrix m goes to P0 + m * matrix_stride
 * elements (matrix_stride >= N * ld, multiple of ld). All fluxes share n_bins. */
splidar_status splidar_build_base_batched(const splidar_flux *fluxes, int32_t n_matrices,
                                          splidar_dtype dt, splidar_entry mode, void *P0, int64_t ld,
                                          int64_t matrix_stride, void *ws, size_t ws_bytes,
                                          void *stream);

/* Step 3 materialised (async): P[i][:] = P0[(i + l) mod N][:] with l = splidar_shift(t_r, N, t_d)
 * (Thm 2). P and P0 are distinct device N x ld matrices of dtype dt (P == P0 is
 * SPLIDAR_EINVAL). The solvers never need this: they fold l into their vector gather. */
splidar_status splidar_apply_deadtime(const void *P0, void *P, int32_t n_bins, int64_t ld,
                                      splidar_dtype dt, double t_r, double t_d, void *stream);

/* P~ built ELEMENT BY ELEMENT from Eq. 4 -- the sequential
 * construction that Theorem 2 replaces -- for same-hardware comparisons: for every (i, j) on its own,
 * a = s_i + x_d, D(a) = (ceil(a / Delta) - 1/2) Delta, b = ceil((a - s_j) / t_r) t_r + s_j
 * (P:102), P_ij = lambda(s_j) exp(-int_{D(a)}^{b} lambda~) with the integral of the periodic replica in
 * closed form (erfc at both limits, no reuse between entries), then rows divided by their sums.
 * Same matrix as splidar_build_base + splidar_apply_deadtime up to rounding. P: device N x ld, dtype
 * dt. t_d >= 0 finite, flux as splidar_build_base, else SPLIDAR_EINVAL / SPLIDAR_ENOSPACE. */
splidar_status splidar_build_eq4(const splidar_flux *flux, double t_d, splidar_dtype dt, void *P, int64_t ld,
                                 void *stream);

/* Step 4 (synchronises stream once): pi P~ = pi for P~ = J_l P~0, by power iteration:
 * pi^0 = 1/N; y = pi^k P~ (fp64 accumulation, the row permutation applied as the gather
 * x_r = pi^k[(r - l) mod N] of a GEMV on P~0); pi^{k+1} = y / ||y||_1; stop after the first k with
 * ||pi^{k+1} - pi^k||_1 < tol or after max_iter products. The loop runs on the device (CUDA
 * graph with a conditional WHILE node): no host round trip per iteration.
 * pi: device fp64 [N]. info: host, may be NULL. tol > 0, max_iter >= 1. */
splidar_status splidar_stationary(const void *P0, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                  double t_r, double t_d, double tol, int32_t max_iter, double *pi,
                                  void *ws, size_t ws_bytes, splidar_solve_info *info, void *stream);
/* Step 4 for n_matrices matrices (P0 + m * matrix_stride) x n_vectors dead times each
 * (t_d[n_matrices * n_vectors], matrix-major), one multi-vector GEMV per matrix and pass; pi: device
 * fp64 [n_matrices * n_vectors * N]; info: host [n_matrices * n_vectors] or NULL; ws:
 * splidar_workspace_bytes(N, n_matrices, n_vectors). Synchronises stream once.
 * splidar_stationary is the case n_matrices = n_vectors = 1. Both keep the instantiated solver
 * (a plan) in a library cache keyed by (device, P0, strides, N, dtype, n_matrices, n_vectors, tol,
 * max_iter, pi, ws): a repeated call with the same buffers replays it (the shifts and output rows
 * go back into the workspace with one small upload, since the workspace is scratch between calls)
 * instead of building a CUDA graph per call. The cache holds at most 16 plans,
 * least recently used first out; splidar_plan_cache_clear() destroys them (call it before freeing
 * the CUDA context, or to return their pinned host memory). The same contract as plans applies:
 * one call at a time per workspace. */
splidar_status splidar_stationary_multi(const void *P0, int32_t n_matrices, int64_t matrix_stride,
                                        int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r,
                                        const double *t_d, int32_t n_vectors, double tol,
                                        int32_t max_iter, double *pi, void *ws, size_t ws_bytes,
                                        splidar_solve_info *info, void *stream);
/* As splidar_stationary_multi, and pi is also copied to pi_host (host [n_matrices * n_vectors * N],
 * pinned for an asynchronous copy) before the one stream synchronisation: host out in one call. */
splidar_status splidar_stationary_multi_host(const void *P0, int32_t n_matrices, int64_t matrix_stride,
                                             int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r,
                                             const double *t_d, int32_t n_vectors, double tol,
                                             int32_t max_iter, double *pi, double *pi_host, void *ws,
                                             size_t ws_bytes, splidar_solve_info *info, void *stream);
void splidar_plan_cache_clear(void);

/* Steps 1-4 for a batch of (signal, background, dead-time) triples (synchronises stream once):
 * item m has pulses (shape.tau, shape.sigma, S[m] * shape.signal[k]) and background B[m], dead time
 * t_d[m]; shape.signal are relative weights and shape.background is ignored. Items with equal
 * (S, B) share one P~0 (built once, solved with one multi-vector GEMV for all their dead times,
 * up to 32 per pass). P0_store: device, room for n_store matrices of N x ld (dtype dt) with
 * consecutive stride N * ld; unique (S, B) pairs are processed n_store at a time.
 * pi: device fp64 [n_items * N] (item-major). info: host [n_items], may be NULL.
 * P0_store == NULL: matrix-free, the items go to splidar_stationary_structured (same items, same pi to
 * rounding; dt, mode, n_store and ld are ignored; ws: splidar_structured_workspace_bytes(N, unique
 * (S, B) pairs, n_items) bytes).
 * Returns SPLIDAR_ENOCONV if any item did not converge (its pi is the last iterate). */
splidar_status splidar_sweep(const splidar_flux *shape, int32_t n_items, const double *S,
                             const double *B, const double *t_d, splidar_dtype dt, splidar_entry mode,
                             double tol, int32_t max_iter, double *pi, void *P0_store,
                             int32_t n_store, int64_t ld, void *ws, size_t ws_bytes,
                             splidar_solve_info *info, void *stream);

/* Plans: the solver of splidar_stationary / splidar_sweep captured once into an instantiated CUDA
 * graph and replayed. A plan binds the matrices, shifts, workspace and pi pointers; executing it
 * re-runs the whole power iteration from pi^0 (synchronises stream once). n_vectors dead times
 * t_d[n_matrices * n_vectors] (matrix-major) share each matrix. Destroy with splidar_plan_destroy. */
typedef struct splidar_plan_s *splidar_plan;
splidar_status splidar_plan_create(splidar_plan *plan, const void *P0, int32_t n_matrices,
                                   int64_t matrix_stride, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                   double t_r, const double *t_d, int32_t n_vectors, double tol,
                                   int32_t max_iter, double *pi, void *ws, size_t ws_bytes,
                                   void *stream);
splidar_status splidar_plan_execute(splidar_plan plan, splidar_solve_info *info /* host [M*V] */,
                                    void *stream);
/* A plan that also BUILDS its matrices: every launch runs steps 1-2 (flux vectors, entries of
 * P~0 for fluxes[m] into P0 + m * matrix_stride, as splidar_build_base_batched) and then the power
 * iteration. The build also sums the stored entries of every column: from the uniform start the
 * first product is x^0 P~ = (1/N) 1^T J_l P~0 = (1/N) 1^T P~0 -- the row permutation leaves column
 * sums unchanged (Thm 2) -- so iteration 1 of every dead time comes from those sums and the
 * GEMV passes start at iteration 2 (one matrix pass fewer per solve; same iterates up to the order
 * of the column sums). All fluxes share N and t_r. ws: splidar_workspace_bytes(N, n_matrices,
 * n_vectors); otherwise as splidar_plan_create.
 * Encoded storage: an fp32 plan with factored entries that runs the int8 GEMV (see splidar_plan_gemv)
 * and N <= 131072 first derives every column's largest exponent E_j from the row normalisers (the
 * column's extreme entries are w_j times the extremes of 1/D above and below the diagonal); when
 * every column passes the int8 range test it stores each entry of P0 not as fp32 but as its column's
 * scaled integer, the u32 word sig << (e - E_j + 8) (sig = the 24-bit significand, e = the biased
 * exponent; the same value, exactly), and the GEMV feeds those words to the tensor cores as they
 * arrive (no conversion pass). Such a P0 is an internal buffer: splidar_plan_storage tells which
 * form the last launch left; SPLIDAR_I8_ENC=0 at plan creation keeps fp32. */
splidar_status splidar_plan_create_build(splidar_plan *plan, const splidar_flux *fluxes, int32_t n_matrices,
                                         splidar_entry mode, splidar_dtype dt, void *P0, int64_t matrix_stride,
                                         int64_t ld, const double *t_d, int32_t n_vectors, double tol,
                                         int32_t max_iter, double *pi, void *ws, size_t ws_bytes,
                                         void *stream);
/* New flux parameters for a building plan's next launches (same N, same t_r as at creation, the same
 * number of matrices); enqueued on stream (a small upload), EINVAL otherwise. The dead times stay. */
splidar_status splidar_plan_set_fluxes(splidar_plan plan, const splidar_flux *fluxes, int32_t n_matrices,
                                       void *stream);
/* As execute, but only enqueues (async); read results later with splidar_plan_info. */
splidar_status splidar_plan_launch(splidar_plan plan, void *stream);
splidar_status splidar_plan_info(splidar_plan plan, splidar_solve_info *info, void *stream);
void splidar_plan_destroy(splidar_plan plan);
/* How a plan runs: SPLIDAR_PLAN_GRAPH (instantiated CUDA graph: [GEMV -> check] in a conditional WHILE
 * node; N > 2048), SPLIDAR_PLAN_LOOP (opt-in, SPLIDAR_PERSIST=1 at plan creation; N > 2048, GEMV not on
 * the int8 tensor cores: instantiated CUDA graph whose iterations are ONE cooperative launch of a
 * persistent kernel -- GEMV pass, grid barrier, convergence check, grid barrier, until every vector is
 * done (P:79 iterated on the device with no launch between iterations); same arithmetic in the same
 * order as the WHILE form, bit-identical results) or
 * SPLIDAR_PLAN_FUSED (N <= 2048: one clustered launch runs every iteration of every (matrix, dead
 * time) pair, P~0 rows staged in shared memory or streamed from L2; a single kernel launch, so
 * splidar_plan_launch may be captured into a caller's CUDA graph). -1 for NULL.
 * SPLIDAR_FUSED=0 in the environment at plan creation forces the graph forms. */
#define SPLIDAR_PLAN_GRAPH 0
#define SPLIDAR_PLAN_FUSED 1
#define SPLIDAR_PLAN_LOOP 2
int splidar_plan_kind(splidar_plan plan);
/* Which GEMV kernel ran the plan's last launch (synchronises the stream once):
 *   SPLIDAR_GEMV_TENSOR_I8 (2): the exact int8 split on the 5th-generation tensor cores
 *     (tcgen05.mma kind::i8, TMEM accumulators): P~0 in u8 planes with one exponent per column,
 *     x in 7 u8 slices (truncation < 2^-56 of the largest x); used for fp32 storage when the plan
 *     has 8..18 dead times per matrix, N % 128 == 0 and 1024 <= N <= 66048 (fp64 storage only with
 *     SPLIDAR_I8=2 in the environment at plan creation), and only if every column of every matrix
 *     passes the range test of each launch (every non-zero entry within 2^8 (fp32) / 2^11 (fp64) of
 *     its column's largest, no subnormal or negative entry) -- else the FP64 kernel runs;
 *   SPLIDAR_GEMV_FP64 (1): FP64 tensor cores (DMMA) / DFMA (k_power_step);
 *   SPLIDAR_GEMV_FUSED (0): the fused small-N solver (SPLIDAR_PLAN_FUSED);
 *   -1: NULL plan or CUDA error. SPLIDAR_I8=0 at plan creation disables the int8 kernel. */
#define SPLIDAR_GEMV_FUSED 0
#define SPLIDAR_GEMV_FP64 1
#define SPLIDAR_GEMV_TENSOR_I8 2
int splidar_plan_gemv(splidar_plan plan, void *stream);
/* The form of P0 after the plan's last launch (synchronises the stream once): SPLIDAR_STORAGE_IEEE
 * (the dtype's numbers) or SPLIDAR_STORAGE_ENCODED (a building plan's per-column scaled integers, see
 * splidar_plan_create_build); -1: NULL plan or CUDA error. */
/* Device time of the plan's GEMV launches since the last reset: each GEMV kernel stamps the device
 * clock (%globaltimer) when its first CTA starts and its last CTA ends, and the convergence check that
 * follows adds the difference, so *seconds / *launches is the GEMV kernel's own average launch duration
 * inside the CUDA-graph loop (where events cannot bracket a single kernel). The int8 plans' FP64
 * kernel returns at once without stamping; iteration 1 of a building plan has no GEMV launch. reset
 * != 0 zeroes the counters after reading. Synchronises the stream. Fused plans report 0 launches. */
splidar_status splidar_plan_gemv_time(splidar_plan plan, int32_t reset, double *seconds, int64_t *launches,
                                      void *stream);
#define SPLIDAR_STORAGE_IEEE 0
#define SPLIDAR_STORAGE_ENCODED 1
int splidar_plan_storage(splidar_plan plan, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Row shards of one matrix over several GPUs: the power iteration of P:79 with
 * P~ = J_l P~0 (Thm 2) split by rows. Rank g stores rows [row0, row0 + n_rows) of P~0
 * (n_rows x ld, row-major, built by splidar_build_base_rows: the same entries as rows row0.. of
 * splidar_build_base) and computes the partial product y_g^T = x^T P~0[rows, :], x_r = pi[(r - l) mod N]
 * gathered from the replicated iterate; the caller sums the partials over the ranks (one all-reduce of
 * N x n_vectors doubles per iteration, e.g. NCCL over NVLink) and every rank then runs the identical
 * normalisation / L1-change / next-gather step, so the iterate stays replicated and the dead-time
 * offset is applied after the collective. One iteration:
 *     splidar_plan_shard_gemv(plan)            -> ypart [n_vectors][N] fp64 holds this rank's partial
 *     all-reduce(ypart, SUM)                   (caller, same stream order)
 *     splidar_plan_shard_check(plan, &more)    -> more = 0 when every vector converged / stopped
 * preceded once by splidar_plan_shard_init and followed by splidar_plan_shard_finish (writes pi
 * [n_vectors][N] and info, synchronises). ypart: device fp64 [n_vectors * N], 16-byte aligned, owned
 * by the caller. ws: splidar_workspace_bytes(N, 1, n_vectors). The FP64 GEMV (DMMA / DFMA) runs the
 * shard. EINVAL for a row range outside [0, N) or a NULL ypart; other errors as splidar_plan_create. */
splidar_status splidar_build_base_rows(const splidar_flux *f, splidar_dtype dt, splidar_entry mode,
                                       void *P0_rows, int64_t ld, int32_t row0, int32_t n_rows, void *ws,
                                       size_t ws_bytes, void *stream);
splidar_status splidar_plan_create_rows(splidar_plan *plan, const void *P0_rows, int32_t row0,
                                        int32_t n_rows, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                        double t_r, const double *t_d, int32_t n_vectors, double tol,
                                        int32_t max_iter, double *pi, double *ypart, void *ws,
                                        size_t ws_bytes, void *stream);
splidar_status splidar_plan_shard_init(splidar_plan plan, void *stream);
splidar_status splidar_plan_shard_gemv(splidar_plan plan, void *stream);
splidar_status splidar_plan_shard_check(splidar_plan plan, int32_t *more, void *stream);
splidar_status splidar_plan_shard_finish(splidar_plan plan, splidar_solve_info *info, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Matrix-free (structured) operator: SURVEY §8(f) rows f2 and f1.
 *
 * From §3.4 (E_base = exp.(-Lambda L - D); P = (1 lambda^T) . E; row
 * normalisation P:79) every row of P~0 is the same column profile w_j = lambda_j e^{-F_j}
 * times a step (e^{-Lambda} below the diagonal, 1 on and above it) over the row normaliser D_r, so
 *     (x^T P~0)_j = w_j (C_j + e^{-Lambda} (T - C_j)),  C_j = sum_{r<=j} x_r / D_r,  T = C_{N-1}:
 * one prefix scan per product instead of a pass over N^2 stored entries. The dead time is the same
 * row permutation (Thm 2), x_r = v[(r - l) mod N]. These entry points never store P~0; they
 * compute exactly the matrix that splidar_build_base writes (up to rounding), so their results are
 * compared with the same oracle. N <= 65536 (a cluster of <= 16 CTAs x 4096 bins per item), else
 * SPLIDAR_EINVAL. Items follow splidar_sweep: item m has pulses (shape.tau, shape.sigma,
 * S[m] * shape.signal[k]), background B[m], dead time t_d[m]; items with equal (S, B) share their
 * step-1 vectors. All calls synchronise `stream` once at their end.
 *
 * Workspace: splidar_structured_workspace_bytes(N, n_profiles, n_items) bytes, 256-byte aligned
 * (n_profiles = number of distinct (S, B) pairs; n_items = items, or N for splidar_mixing_steps);
 * 0 if the sizes are invalid. */
size_t splidar_structured_workspace_bytes(int32_t n_bins, int32_t n_profiles, int32_t n_items);

/* f2: pi P~ = pi for every item by power iteration on the structured operator, with the same
 * definition as splidar_stationary (pi^0 = 1/N, 1-norm renormalisation, stop after the first product
 * with ||pi^{k+1} - pi^k||_1 < tol, or max_iter products -> SPLIDAR_ENOCONV with the last iterate).
 * pi: device fp64 [n_items * N]; info: host [n_items] or NULL. */
splidar_status splidar_stationary_structured(const splidar_flux *shape, int32_t n_items, const double *S,
                                             const double *B, const double *t_d, double tol, int32_t max_iter,
                                             double *pi, void *ws, size_t ws_bytes, splidar_solve_info *info,
                                             void *stream);

typedef struct {
    double lambda2_re, lambda2_im;  /* second eigenvalue of P~ (lambda2_im >= 0: the member of a
                                       conjugate pair with phase in [0, pi])                     */
    double modulus;                 /* |lambda_2| (§4)                                    */
    double phase;                   /* arg lambda_2 in [0, pi] (§4.2)                     */
    double gap;                     /* spectral gap 1 - |lambda_2| (§4.1)                 */
    double change;                  /* last move of the Ritz value                                */
    int32_t iters, converged;
} splidar_spectral_info;

/* f1: the second eigenvalue of P~ = J_l P~0 per item (§4). The leading pair (left pi,
 * right 1) is deflated, A = P~ - 1 pi, and a 2-D real subspace is iterated under v -> v A with Ritz
 * values from H = (W Q^T)(Q Q^T)^{-1} (a complex pair spans a real 2-D invariant subspace); stop
 * when the dominant Ritz value moves less than tol, else SPLIDAR_ENOCONV after max_iter products.
 * pi: device fp64 [n_items * N], the stationary vectors of the items (e.g. from
 * splidar_stationary_structured; accurate to << tol). info: host [n_items]. */
splidar_status splidar_second_eigenvalue(const splidar_flux *shape, int32_t n_items, const double *S,
                                         const double *B, const double *t_d, const double *pi, double tol,
                                         int32_t max_iter, void *ws, size_t ws_bytes, splidar_spectral_info *info,
                                         void *stream);

/* f1 on a STORED matrix (any row-stochastic P0 in HBM, fp64 or fp32: splidar_build_base's P~0,
 * splidar_build_eq4's matrix, or a user's): the second eigenvalue of P~ = J_l P0, l from t_r, t_d as in
 * splidar_shift (Thm 2; t_d = 0 gives P~ = P0), by the same deflated 2-D subspace iteration as
 * splidar_second_eigenvalue, each product y = q^T P~ being one pass of the multi-vector GEMV over P0
 * (two vectors, dead time folded into the gathered x). pi: device fp64 [N], the stationary vector of
 * P~ (e.g. from splidar_stationary; sum 1, accurate to << tol). info: host, may be NULL. The stored
 * matrix is read, never written. max_iter >= 2; SPLIDAR_ENOCONV if the Ritz value still moved by tol
 * or more after max_iter products. Workspace: splidar_spectral_dense_workspace_bytes(N), 256-aligned.
 * Synchronises `stream`. */
size_t splidar_spectral_dense_workspace_bytes(int32_t n_bins);
splidar_status splidar_second_eigenvalue_dense(const void *P0, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                               double t_r, double t_d, const double *pi, double tol,
                                               int32_t max_iter, void *ws, size_t ws_bytes,
                                               splidar_spectral_info *info, void *stream);

/* Structured plans: the items of splidar_stationary_structured (kind SPLIDAR_SPLAN_SOLVE) or
 * splidar_second_eigenvalue (kind SPLIDAR_SPLAN_LAMBDA2; pi is then the input) validated and uploaded
 * once; splidar_splan_launch only enqueues (step-1 vectors + the kernel, async, re-runnable; the
 * first launch is eager, the second captures the sequence into a CUDA graph on a private stream and
 * it and later launches replay it: one cudaGraphLaunch on `stream`; SPLIDAR_SPLAN_GRAPH=0 in the
 * environment keeps every launch eager; launches of one plan must not overlap);
 * splidar_splan_info synchronises `stream`, fills the per-item info (either pointer may be NULL)
 * and the device time of the last launch's kernel in ms (CUDA events recorded around it on
 * `stream`; may be NULL); SPLIDAR_ENOCONV if an item did not converge. The two calls above are
 * create + launch + info + destroy. */
#define SPLIDAR_SPLAN_SOLVE 0
#define SPLIDAR_SPLAN_LAMBDA2 1
typedef struct splidar_splan_s *splidar_splan;
splidar_status splidar_splan_create(splidar_splan *plan, int32_t kind, const splidar_flux *shape, int32_t n_items,
                                    const double *S, const double *B, const double *t_d, double tol,
                                    int32_t max_iter, double *pi, void *ws, size_t ws_bytes, void *stream);
splidar_status splidar_splan_launch(splidar_splan plan, void *stream);
splidar_status splidar_splan_info(splidar_splan plan, splidar_solve_info *solve_info,
                                  splidar_spectral_info *spectral_info, float *kernel_ms, void *stream);
void splidar_splan_destroy(splidar_splan plan);

/* f1: mixing steps (§4.1: "the number of steps n such that P~^n approaches the stationary
 * distribution"): the smallest n >= 1 with max_i 1/2 ||e_i^T P~^n - pi||_1 <= eps over all start
 * bins i (every row of P~^n), found per start as its first n_i (TV to stationarity is
 * non-increasing) and reduced as max_i n_i. pi: device fp64 [N]. steps_per_start: device int32 [N]
 * (n_i, -1 if max_steps was not enough) or NULL. mixing_steps: host, -1 with SPLIDAR_ENOCONV if
 * some start needs more than max_steps. Workspace: splidar_structured_workspace_bytes(N, 1, N). */
splidar_status splidar_mixing_steps(const splidar_flux *flux, double t_d, const double *pi, double eps,
                                    int32_t max_steps, int32_t *steps_per_start, int32_t *mixing_steps, void *ws,
                                    size_t ws_bytes, void *stream);

/* f1: the trajectory of one histogram bin (§4.2): traj[n] = (start^T P~^n)[bin] for
 * n = 0..steps (no renormalisation), and final_vec = start^T P~^steps (device [N], may be NULL).
 * start: device fp64 [N]; traj: device fp64 [steps + 1]. 0 <= bin < N, steps >= 0.
 * Workspace: splidar_structured_workspace_bytes(N, 1, 1). */
splidar_status splidar_bin_trajectory(const splidar_flux *flux, double t_d, const double *start, int32_t bin,
                                      int32_t steps, double *traj, double *final_vec, void *ws, size_t ws_bytes,
                                      void *stream);

/* ---------------------------------------------------------------------------------------------
 * Monte Carlo of the asynchronous detection process, the paper's ground
 * truth for the Markov model. Items as splidar_sweep (shape x S[m], B[m], t_d[m]); each
 * item runs n_runs independent chains ("runs", one histogram each). A chain starts at T = 0 as if a
 * photon had just been registered; after each registration at T_k the detector is dead for t_d and
 * the next registration is T_{k+1} = Ftilde^{-1}(Ftilde(T_k + t_d) - log U) (the first arrival of the
 * inhomogeneous Poisson process with rate lambda~, Eq. 1 replicated), U uniform on (0, 1]
 * from splitmix64 started at seed + c * 0xD1B54A32D192ED03 (mod 2^64) for chain c = m * n_runs + run
 * and advanced once per registration (the generator the CPU oracle implements, so chains can be
 * replayed). The first n_burn registrations are discarded; then X_k = T_k mod t_r goes into the
 * run's histogram of n_hist bins ((k-1) t_r/n_hist, k t_r/n_hist] (X = 0 read as t_r) until n_regs
 * registrations are counted, or, when n_cycles > 0 (n_regs ignored), until the first registration
 * n_cycles laser periods after the burn-in (the paper's "histograms of 50,000 laser cycles").
 * hist: device uint64 [n_items][n_runs][n_hist] (zeroed by the call). n_record > 0 also stores the
 * first n_record registrations of every chain: q_rec (period index) and t_rec (offset in [0, t_r)),
 * device [n_items * n_runs * n_split][n_record].
 * n_split >= 1: each run is n_split independent sub-chains (chain c = (m * n_runs + run) * n_split + sub,
 * seeded as above), each with its own n_burn and 1/n_split of the run's n_regs or n_cycles (which
 * must then be a multiple of n_split), all adding into the run's histogram: the same stationary
 * estimate with n_split times the parallelism; n_split = 1 is the paper's one-chain-per-histogram
 * protocol. Synchronises `stream` once.
 * Workspace: splidar_mc_workspace_bytes(n_profiles, n_items) (n_profiles = distinct (S, B) pairs). */
size_t splidar_mc_workspace_bytes(int32_t n_profiles, int32_t n_items);
splidar_status splidar_monte_carlo(const splidar_flux *shape, int32_t n_items, const double *S, const double *B,
                                   const double *t_d, uint64_t seed, int32_t n_runs, int32_t n_split, int64_t n_burn,
                                   int64_t n_regs, int64_t n_cycles, int32_t n_hist, uint64_t *hist, int32_t n_record,
                                   int64_t *q_rec, double *t_rec, void *ws, size_t ws_bytes, void *stream);

const char *splidar_strerror(splidar_status st);
int splidar_last_cuda_error(void);     /* cudaError_t of the last SPLIDAR_ECUDA, else 0 */
const char *splidar_build_info(void);  /* compile target and version string */

#ifdef __cplusplus
}
#endif
#endif /* SPLIDAR_H */
