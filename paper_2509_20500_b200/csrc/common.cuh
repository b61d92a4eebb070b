// Internal definitions shared by the libsplidar translation units (not part of the C ABI).
// Nothing here is shared with oracle/: the product and the oracle are independent.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/splidar.h"

namespace spl {

constexpr int kMaxPulses = SPLIDAR_MAX_PULSES;
constexpr int kMaxVectors = 32;      // dead times per matrix in one multi-vector GEMV pass
constexpr int kStripCols = 512;      // columns per GEMV / build CTA (4 KB of an fp64 row)
constexpr int kNumSMsDefault = 148; // B200; only used if the device query fails
constexpr int kMaxSMs = 160;        // workspace bound for the persistent GEMV grid (SM count queried per device)
constexpr int kCheckChunk = 2048;   // elements per CTA of the convergence-check kernel
constexpr int kGemvCtas = 2 * kMaxSMs;  // largest persistent GEMV grid (two 256-thread CTAs per SM)
constexpr int kMinRowsPerCta = 64;      // smallest row range a GEMV CTA is given

// theta without t_d, device copy. Eq. 1 with K pulses.
struct FluxDev {
    double t_r;
    int n;
    int k;
    double B;
    double tau[kMaxPulses];
    double sigma[kMaxPulses];
    double S[kMaxPulses];
};

// Per-matrix vectors of step 1 (all fp64, length N) + scalars.
struct VecPtrs {
    double *F;      // F(s_j), prefix sum of bin masses (Thm 1)
    double *lam;    // lambda(s_j)
    double *w;      // lambda_j e^{-F_j}
    double *invD;   // 1 / D_r
    double *invZ;   // e^{-F_r} / D_r  (= 1 / Z_r, row sum of the exp form)
    double *scal;   // [0] Lambda, [1] e^{-Lambda}, [2] bad-row flag (0 / 1), [3] tail mass m_N
    double *tiles;  // [5][M][ntile] per-1024-element-tile totals / offsets of the two-level scans
    int ntile;      // ceil((N + 1) / 1024)
};
constexpr int kScanTile = 1024;      // elements per tile of the two-level scans (256 threads x 4)

// Per (matrix, vector) power-iteration state.
struct __align__(16) SolveState {
    int l;          // row shift (Thm 2); < 0 marks an unused (padding) vector
    int iters;
    int done;
    int converged;
    int cur;        // which y buffer holds the current iterate
    int pad0, pad1, pad2;
    double s;       // ||y[cur]||_1: pi^k = y[cur] / s
    double change;  // last L1 change
};

// Workspace layout (offsets in bytes from the 256-aligned base).
struct WsLayout {
    int N, M, V;    // V padded to a power of two
    int strips, chunks, xstride, pieces;
    size_t flux, vec, lsh, oidx, y, X, part, ssum, l1part, state, strip_cnt, mv_cnt, act, glob;
    size_t ximg, colexp, colmin, smax, xtau, cpart, csum, epart, total;
};

WsLayout ws_layout(int N, int M, int V);
int pad_vectors(int V);

// ---- per-device host state (device.cu) -------------------------------------------------------
int current_device();
int device_sm_count();              // SMs of the current device (cached per device ordinal)
// Programmatic dependent launch between the library's own consecutive kernels (the build after the
// flux vectors, the fused solver after the build, the check after the GEMV in the iteration graph):
// on unless SPLIDAR_PDL=0 (read once per process).
bool pdl_enabled();
// cudaFuncSetAttribute once per (device, kernel, value): max dynamic shared memory (if > 0) and
// non-portable cluster sizes (if requested).
cudaError_t func_attrs_once(const void *fn, int max_dyn_smem, bool nonportable_cluster);

// ---- kernels launch wrappers (host) -------------------------------------------------------
// single (M = 1, N + 1 <= 8192): the profile by value, so d_flux need not be uploaded first
cudaError_t launch_flux_vectors(const FluxDev *d_flux, int M, int N, VecPtrs base, int64_t vstride,
                                cudaStream_t s, const FluxDev *single = nullptr);
constexpr int kSmallVecMax = 8192;   // N + 1 <= this: the one-launch vector kernel (k_vec_small)
// colsum_part ([M][colsum_chunks(N)][N]) / colsum ([M][N]): optional column sums of the stored
// entries (the first power-iteration product from the uniform start, fused into the build)
constexpr int kColsumChunks = 32;
int colsum_chunks(int N);
// optional (with colsum): the int8 GEMV's column exponents and range test from the build
struct ColStats {
    int *emax_part, *emin_part;   // [M][chunks][N] (null: not wanted)
    int *colexp;                  // [M][N]
    unsigned *flag;               // set to 1 by the build, cleared by a failing column
    int R, zero_col_exp;
    // encoded storage (fp32, factored entries; emax_part null): colexp and *flag come from
    // launch_enc_colexp before the build, which then stores every entry as its scaled integer
    // (fixpt.cuh) when *flag is set, and as fp32 otherwise
    int enc;
};
// Column exponents of the matrices a factored fp32 build is about to write, from the O(N) row
// normalisers (prefix / suffix extremes of 1/D), and the int8 range test: *flag = every column of
// every matrix in range (the condition for encoded storage).
cudaError_t launch_enc_colexp(const VecPtrs base, int64_t vstride, int M, int N, int *colexp, int *scratch,
                              unsigned *flag, cudaStream_t s);
cudaError_t launch_build(const VecPtrs base, int64_t vstride, int M, int N, int dtype, int mode,
                         void *P0, int64_t ld, int64_t mstride, cudaStream_t s, int row0 = 0, int nrows = -1,
                         double *colsum_part = nullptr, double *colsum = nullptr, ColStats cst = ColStats{});
cudaError_t launch_apply_deadtime(const void *P0, void *P, int N, int64_t ld, int dtype, int l,
                                  cudaStream_t s);
cudaError_t launch_build_eq4(const FluxDev &f, double u, int dtype, void *P, int64_t ld, cudaStream_t s);

constexpr int kGridBarWord = 32;   // glob[32..33]: k_power_loop's grid barrier (arrivals, generation)

struct PowerArgs {
    const void *P;
    int64_t ld;
    int64_t mstride;
    int N, M, V, strips, chunks, xstride;
    double *y;               // [M][V][2][N]       unnormalised iterates (ping-pong)
    double *X;               // [M][N][xstride]    gathered, normalised x_v[r] = pi_v[(r - l_v) mod N]
    double *part;            // [pieces][V][512]   per-CTA partial column sums
    double *ssum;            // [M][V][strips]     strip sums of y
    double *l1part;          // [M][V][chunks]     per-chunk L1 changes (check kernel)
    SolveState *st;          // [M][V]
    const int *lsh;          // [M][V] row shifts l (< 0: unused vector)
    unsigned *strip_cnt;     // [M * strips]       pieces finished per strip (active order)
    unsigned *mv_cnt;        // [M][V]             check-kernel CTA counters
    int *act;                // [M]                active matrices (any vector still running)
    unsigned *glob;          // [0] check CTA counter, [1] any-active flag, [2] number of active matrices,
                             // [3] int8 GEMV on, [kGridBarWord..+1] k_power_loop grid barrier
    double tol;
    int max_iter;
    int use_handle;
    cudaGraphConditionalHandle handle;
    // tcgen05 int8 GEMV (power_i8.cu); glob[3] = 1 when it runs (range test passed)
    int i8;                  // the plan has the int8 kernels in its loop
    int strips_i8;           // column tiles of the int8 GEMV (N / TN)
    unsigned char *ximg;     // [M][N / 64][8192]     x slices in the MMA's K-major image
    int *colexp;             // [M][N]                column exponents E_j
    int *colmin;             // [M][N]                smallest exponent of a non-zero entry (range test)
    double *smax;            // [M][V][N / 64]        tile maxima of y
    int *xtau;               // [M][V]                x scale exponents tau_v
    int i8_dbg;              // timing experiments only (SPLIDAR_I8_DBG): 1 skip conversion, 2 skip MMA
    // row shard: the stored block holds rows [row0, row0 + rows) of P~0; the GEMV
    // writes its partial y^T = x_g^T P~0[rows, :] to ypart [M][V][N] for the caller's all-reduce
    int rows, row0;
    double *ypart;
    int ypart_shared;        // ypart is [M][N], one y for every vector of a matrix (fused-build column sums)
    unsigned long long *ktime;   // GEMV launch timer (ptx.cuh): [0] first start, [1] last end, [2] sum of
                                 // launch durations (ns), [3] launches; null: not timed
};

// Kernel node parameters for the three solver kernels (for graph construction).
struct SolverKernels {
    void *init_fn;
    void *step_fn;
    void *check_fn;
    void *finish_fn;
    void *ssum_fn;           // row shard: strip sums of the all-reduced y
    void *loop_fn;           // k_power_loop: GEMV + check iterated in one cooperative launch (or null)
    dim3 init_grid, init_block;
    dim3 step_grid, step_block;
    dim3 check_grid, check_block;
    dim3 finish_grid, finish_block;
    size_t step_smem;
};
int solver_kernels(int dtype, int V, SolverKernels *out, const PowerArgs &a);
// int8 tensor-core GEMV (power_i8.cu)
struct I8Kernels {
    alignas(64) unsigned char tmap[128];   // CUtensorMap of the stored matrices (a kernel parameter)
    void *step_fn, *colexp_fn, *check_fn, *prep_fn;
    void *step_enc_fn;        // fp32 matrices stored encoded by a building plan (k_power_step_i8e)
    size_t step_enc_smem;
    dim3 step_grid, step_block, colexp_grid, colexp_block, small_grid;
    size_t step_smem;
    int rows_per_cta;
};
int i8_supported(int dtype, const PowerArgs &a);
cudaError_t i8_kernels(int dtype, I8Kernels *k, const PowerArgs &a);
int i8_tile_cols(int dtype);
int i8_range_bits(int dtype);      // R: non-zero entries within 2^R of their column maximum
size_t finish_args_size();
// pi output: out_idx[mv] >= 0 selects row out_idx[mv] of pi ([*, N]); < 0 skips the vector.
void make_finish_args(void *dst, const PowerArgs &a, double *pi, const int *out_idx);

// ---- structured (matrix-free) operator kernels (structured.cu) -----------
struct SpecOut {        // second eigenvalue of one item
    double re, im;      // lambda_2 (im >= 0)
    double change;      // last move of the dominant Ritz value
    int iters, converged;
};
struct StructArgs {
    int N, C, threads;          // cluster of C CTAs x threads, 8 positions per thread
    int64_t vstride;            // profile stride of the vectors
    const double *w, *invD, *scal;
    const int *prof, *lsh;      // [items] profile index and shift l
    double tol;
    int max_iter;               // solve / lambda2: max products; mixing: step cap; traj: steps
    double *pi;                 // solve: out [items][N]; lambda2: in [items][N]; mixing: in [N]
    SolveState *st;             // solve: [items]
    SpecOut *spec;              // lambda2: [items]
    double eps;                 // mixing: TV threshold
    int start_bin0;             // mixing: first start bin of this launch
    int *nsteps, *nmax;         // mixing: [N] per start, max over starts
    const double *start;        // traj: start distribution [N]
    int bin;                    // traj: recorded bin
    double *traj, *out;         // traj: [steps + 1], final vector [N] (may be null)
};
enum { kStructSolve = 0, kStructLambda2 = 1, kStructMixing = 2, kStructTraj = 3 };
int struct_shape(int N, int *C, int *threads);
cudaError_t launch_struct(int kind, const StructArgs &a, int n_units, cudaStream_t s);

// ---- fused small-N dense solve (fused.cu): all iterations of one (matrix, vector) in one cluster
constexpr int kFusedInline = 64;
struct FusedArgs {
    const void *P;
    int64_t ld, mstride;
    int N, M, V, C, R;
    int resident;               // rows of P~0 copied to shared memory once
    const int *lsh;             // [M][V]
    const int *out_idx;         // [M][V]
    int n_inline;               // M V <= kFusedInline: shifts / output rows passed in the parameters
    int lsh_in[64], oidx_in[64];
    double *pi;
    SolveState *st;             // [M][V]
    double tol;
    int max_iter;
    int p2p;                    // exchanges by st.async + per-CTA mbarriers (else barrier.cluster)
    int ldg;                    // non-resident rows: read-only global loads into registers (else TMA ring)
    int one_x;                  // one exchange per product: partials go straight to the CTA whose rows
                                // they feed (needs p2p); else owners sum and redistribute (two)
};
int fused_shape(int N, int *C, int *R);
int fused_resident(int N, int R, int dtype);
cudaError_t launch_fused(int dtype, const FusedArgs &a, cudaStream_t s);
cudaError_t fused_fn(int dtype, int N, void **fn);   // the kernel instance; sets its attributes (not in a capture)

// ---- second eigenvalue of a stored matrix (spectral_dense.cu; SURVEY §8(f) f1 on K6) -----------
struct SdState {
    double sig_w[2];            // the sigma the last w were formed with (update kernel)
    double al, be, ga;          // q1' = al w1, q2' = be (w2 - ga w1)
    double mu_re, mu_im, dmu;   // dominant Ritz value of the deflated operator, its last move
    int iters, converged, done, pad;
};
struct SdArgs {
    PowerArgs p;                // the GEMV's arguments (M = 1, V = 2; y buffer 0 holds q, 1 gets q P~)
    int l;                      // row shift of P~ = J_l P0
    const double *pi;           // [N]
    double *part;               // [chunks][10]
    double *qsum;               // [2][nq] per-CTA partial sums of the stored basis q_a
    int nq;                     // = sd_update_ctas(N)
    SdState *sd;
    unsigned *cnt;
    double tol;
    int max_iter;
    int use_handle;
    cudaGraphConditionalHandle handle;
};
struct SdKernels {
    void *init_fn, *dots_fn, *update_fn;
    dim3 block, dots_grid, update_grid;
};
int sd_chunks(int N);
int sd_update_ctas(int N);
constexpr int kSdDotsPerChunk = 10;
void sd_kernels(SdKernels *k, int N);

// ---- Monte Carlo of the detection process (mc.cu) ------------------------------
struct McArgs {
    const FluxDev *flux;        // [profiles]
    const int *prof;            // [items]
    const double *td;           // [items]
    int n_items, n_runs, n_split, n_hist, n_record;
    long long n_burn, n_regs, n_cycles;   // per chain (a run's budget / n_split)
    uint64_t seed;
    unsigned long long *hist;   // [items][runs][n_hist]
    long long *q_rec;           // [items * runs * n_split][n_record]
    double *t_rec;
};
cudaError_t launch_mc(const McArgs &a, cudaStream_t s);

}  // namespace spl
