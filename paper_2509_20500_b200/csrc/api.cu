// The C ABI of include/splidar.h: host validation, the shift rule, workspace layout, kernel
// dispatch and the CUDA-graph solver plans. No compute happens on the host: every step of the
// path runs in the kernels of flux_vectors.cu, build.cu and power.cu.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace spl {

// One NVTX range per public entry point, named after it (header-only NVTX3: a no-op unless a tool is
// attached; `ncu --nvtx --nvtx-include "splidar_plan_launch/"` profiles only the kernels one call
// launches, and a timeline tool shows host calls against their kernels).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
#define SPL_NVTX_RANGE() ::spl::NvtxRange spl_nvtx_range_(__func__)

static inline size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// Vector counts with a compiled GEMV: 1, 2, 4, 8, 16, 17, 18, 24, 32.
int pad_vectors(int V) {
    if (V <= 2) return V < 1 ? 1 : V;
    if (V <= 4) return 4;
    if (V <= 8) return 8;
    if (V <= 16) return 16;
    if (V <= 18) return V;   // 16 on tensor cores + 1-2 on DFMA
    return V <= 24 ? 24 : 32;
}

WsLayout ws_layout(int N, int M, int V) {
    WsLayout L;
    memset(&L, 0, sizeof(L));
    L.N = N;
    L.M = M;
    L.V = pad_vectors(V);
    L.strips = (N + kStripCols - 1) / kStripCols;
    L.chunks = (N + kCheckChunk - 1) / kCheckChunk;
    L.xstride = L.V < 2 ? 2 : (L.V + 1) / 2 * 2;
    L.pieces = kGemvCtas + M * L.strips;     // a CTA's k-th piece of strip g uses slot cta + g
    const size_t MV = (size_t)M * L.V;
    size_t o = 0;
    L.flux = o; o = a256(o + sizeof(FluxDev) * (size_t)M);
    const size_t ntile = ((size_t)N + 1 + kScanTile - 1) / kScanTile;
    L.vec = o;  o = a256(o + sizeof(double) * ((size_t)M * N * 5 + (size_t)M * 8 + 5 * (size_t)M * ntile));
    L.lsh = o;  o = a256(o + sizeof(int) * MV);
    L.oidx = o; o = a256(o + sizeof(int) * MV);
    L.y = o;    o = a256(o + sizeof(double) * MV * 2 * N);
    L.X = o;    o = a256(o + sizeof(double) * (size_t)M * N * L.xstride);
    L.part = o; o = a256(o + sizeof(double) * (size_t)L.pieces * L.V * kStripCols);
    const size_t tiles64 = ((size_t)N + 63) / 64;        // column tiles of the int8 GEMV (>= 64 columns)
    L.ssum = o; o = a256(o + sizeof(double) * MV * (tiles64 > (size_t)L.strips ? tiles64 : (size_t)L.strips));
    L.l1part = o; o = a256(o + sizeof(double) * MV * L.chunks);
    L.state = o; o = a256(o + sizeof(SolveState) * MV);
    L.strip_cnt = o; o = a256(o + sizeof(unsigned) * (size_t)M * (tiles64 > (size_t)L.strips ? tiles64 : (size_t)L.strips));
    L.mv_cnt = o; o = a256(o + sizeof(unsigned) * MV);
    L.act = o; o = a256(o + sizeof(int) * (size_t)M);
    L.glob = o; o = a256(o + sizeof(unsigned) * 4);
    // int8 tensor-core GEMV: x-slice image (128 bytes per row), column exponents, tile maxima, x scales
    L.ximg = o; o = a256(o + (size_t)M * tiles64 * 64 * 128);
    L.colexp = o; o = a256(o + sizeof(int) * (size_t)M * N);
    L.colmin = o; o = a256(o + sizeof(int) * (size_t)M * N);
    L.smax = o; o = a256(o + sizeof(double) * MV * tiles64);
    L.xtau = o; o = a256(o + sizeof(int) * MV);
    // plans that build their matrix: the build's partial column sums and the column sums (iteration 1)
    L.cpart = o; o = a256(o + sizeof(double) * (size_t)M * kColsumChunks * N);
    L.csum = o; o = a256(o + sizeof(double) * (size_t)M * N);
    L.epart = o; o = a256(o + 2 * sizeof(int) * (size_t)M * kColsumChunks * N);   // exponent max / min per chunk
    L.total = o;
    return L;
}

static VecPtrs vec_ptrs(char *ws, const WsLayout &L) {
    double *b = reinterpret_cast<double *>(ws + L.vec);
    const size_t MN = (size_t)L.M * L.N;
    VecPtrs v;
    v.F = b;
    v.lam = b + MN;
    v.w = b + 2 * MN;
    v.invD = b + 3 * MN;
    v.invZ = b + 4 * MN;
    v.scal = b + 5 * MN;
    v.ntile = (L.N + 1 + kScanTile - 1) / kScanTile;
    v.tiles = v.scal + (size_t)L.M * 8;
    return v;
}

// Small host arrays reach the device as kernel parameters (async, stream-ordered, capturable;
// no pageable-memcpy stream synchronisation). CUDA >= 12.1 allows 32764 bytes of parameters, so up to
// 32000 bytes (e.g. 76 flux records) go in one launch.
namespace {
constexpr int kUpChunk = 32000;
struct UpChunk {
    unsigned char data[kUpChunk];
    int n;
};
__global__ void k_upload(const UpChunk c, unsigned char *dst) {
    for (int i = threadIdx.x; i < c.n; i += blockDim.x) dst[i] = c.data[i];
}
}  // namespace

// Small uploads (one flux record, a plan's shifts) as a 1 KB parameter block: the launch copies its
// whole parameter block, so a 32 KB block for a few hundred bytes costs microseconds per call.
constexpr int kUpSmall = 1024;
struct UpSmall {
    unsigned char data[kUpSmall];
    int n;
};
__global__ void k_upload_small(const UpSmall c, unsigned char *dst) {
    for (int i = threadIdx.x; i < c.n; i += blockDim.x) dst[i] = c.data[i];
}

static cudaError_t upload_async(void *dst, const void *src, size_t n, cudaStream_t s) {
    const unsigned char *p = static_cast<const unsigned char *>(src);
    if (n <= (size_t)kUpSmall) {
        UpSmall c;
        c.n = (int)n;
        memcpy(c.data, p, n);
        k_upload_small<<<1, 128, 0, s>>>(c, static_cast<unsigned char *>(dst));
        return cudaGetLastError();
    }
    for (size_t o = 0; o < n; o += kUpChunk) {
        UpChunk c;
        c.n = (int)((n - o) < (size_t)kUpChunk ? (n - o) : (size_t)kUpChunk);
        memcpy(c.data, p + o, (size_t)c.n);
        k_upload<<<1, 256, 0, s>>>(c, static_cast<unsigned char *>(dst) + o);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace spl

using namespace spl;

static int g_last_cuda_error = 0;

static splidar_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return SPLIDAR_OK;
    g_last_cuda_error = (int)e;
    return SPLIDAR_ECUDA;
}
#define SPL_CUDA(x)                                              \
    do {                                                         \
        cudaError_t e_ = (x);                                    \
        if (e_ != cudaSuccess) return cuda_status(e_);           \
    } while (0)

static bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

static splidar_status check_flux(const splidar_flux *f, int expect_n = -1) {
    if (!f) return SPLIDAR_EINVAL;
    if (!finite_pos(f->t_r)) return SPLIDAR_EINVAL;
    if (f->n_bins < 2 || f->n_bins > (1 << 20)) return SPLIDAR_EINVAL;
    if (expect_n >= 0 && f->n_bins != expect_n) return SPLIDAR_EINVAL;
    if (f->n_pulses < 0 || f->n_pulses > kMaxPulses) return SPLIDAR_EINVAL;
    if (f->n_pulses > 0 && (!f->tau || !f->sigma || !f->signal)) return SPLIDAR_EINVAL;
    if (!finite_pos(f->background)) return SPLIDAR_EINVAL;
    double tot = f->background;
    for (int k = 0; k < f->n_pulses; ++k) {
        if (!finite_pos(f->sigma[k])) return SPLIDAR_EINVAL;
        if (!std::isfinite(f->signal[k]) || f->signal[k] < 0.0) return SPLIDAR_EINVAL;
        if (!std::isfinite(f->tau[k]) || f->tau[k] < 0.0 || f->tau[k] >= f->t_r) return SPLIDAR_EINVAL;
        tot += f->signal[k];
    }
    if (!(tot <= 600.0)) return SPLIDAR_EINVAL;
    return SPLIDAR_OK;
}

static FluxDev to_dev(const splidar_flux *f, double s_scale = 1.0, double B = -1.0) {
    FluxDev d;
    memset(&d, 0, sizeof(d));
    d.t_r = f->t_r;
    d.n = f->n_bins;
    d.k = f->n_pulses;
    d.B = B >= 0.0 ? B : f->background;
    for (int k = 0; k < f->n_pulses; ++k) {
        d.tau[k] = f->tau[k];
        d.sigma[k] = f->sigma[k];
        d.S[k] = s_scale * f->signal[k];
    }
    return d;
}

// Items (shape x S[m], B[m]): the shape's period, bins, pulse positions / widths and (non-negative)
// relative signal weights are validated once; each item then only needs S finite >= 0, B finite > 0
// and S * sum(weights) + B <= 600 -- the same conditions check_flux applies to the item's own flux,
// without building it (batches of 10^4 items are validated in microseconds).
static splidar_status check_shape(const splidar_flux *shape, double *sig_sum) {
    if (!shape || shape->n_pulses < 0 || shape->n_pulses > kMaxPulses) return SPLIDAR_EINVAL;
    if (shape->n_pulses > 0 && !shape->signal) return SPLIDAR_EINVAL;
    double zeros[kMaxPulses] = {0.0};
    splidar_flux f = *shape;
    f.background = 1.0;
    f.signal = zeros;                    // positions and widths only; weights checked below
    splidar_status st = check_flux(&f);
    if (st) return st;
    double sum = 0.0;
    for (int k = 0; k < shape->n_pulses; ++k) {
        if (!std::isfinite(shape->signal[k]) || shape->signal[k] < 0.0) return SPLIDAR_EINVAL;
        sum += shape->signal[k];
    }
    *sig_sum = sum;
    return SPLIDAR_OK;
}
static splidar_status check_item(double sig_sum, double S, double B) {
    if (!std::isfinite(S) || S < 0.0 || !finite_pos(B)) return SPLIDAR_EINVAL;
    if (!(S * sig_sum + B <= 600.0)) return SPLIDAR_EINVAL;
    return SPLIDAR_OK;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// u = x_d / Delta = fmod(t_d, t_r) N / t_r (x_d P:102, Thm 2; reading R4), snapped to the
// nearest integer when it is within a few ulps of one: a dead time that is a whole number of bins in
// decimal (t_d = 0.3 with Delta = 0.1) lands on a bin centre (l = u, E = 1 at zero distance), and
// binary rounding of t_d, Delta or the fmod must not push it a whole bin further.
static double shift_u(double t_r, int32_t n_bins, double t_d) {
    double u = std::fmod(t_d, t_r) * (double)n_bins / t_r;
    const double r = std::nearbyint(u);
    if (std::fabs(u - r) <= 8.0 * 2.220446049250313e-16 * std::fmax(1.0, std::fabs(u))) u = r;
    return u;
}

static splidar_status check_matrix(const void *P, int N, int64_t ld, int dt) {
    if (!P) return SPLIDAR_EINVAL;
    if (dt != SPLIDAR_F64 && dt != SPLIDAR_F32) return SPLIDAR_EINVAL;
    const int esz = dt == SPLIDAR_F64 ? 8 : 4;
    if (ld < N || ((ld * esz) & 15) != 0 || !aligned16(P)) return SPLIDAR_ENOSPACE;
    return SPLIDAR_OK;
}

static splidar_status check_ws(const void *ws, size_t ws_bytes, const WsLayout &L) {
    if (!ws || ((uintptr_t)ws & 255u) != 0 || ws_bytes < L.total) return SPLIDAR_ENOSPACE;
    return SPLIDAR_OK;
}

extern "C" {

splidar_status splidar_shift(double t_r, int32_t n_bins, double t_d, int32_t *l_out) {
    if (!l_out || !finite_pos(t_r) || n_bins < 2 || !std::isfinite(t_d) || t_d < 0.0) return SPLIDAR_EINVAL;
    const double u = shift_u(t_r, n_bins, t_d);   // x_d / Delta (Thm 2)
    long l = (long)std::ceil(u);
    l %= n_bins;
    *l_out = (int32_t)l;
    return SPLIDAR_OK;
}

size_t splidar_workspace_bytes(int32_t n_bins, int32_t n_matrices, int32_t n_vectors) {
    if (n_bins < 2 || n_matrices < 1 || n_vectors < 1 || n_vectors > kMaxVectors) return 0;
    return ws_layout(n_bins, n_matrices, n_vectors).total;
}

const char *splidar_strerror(splidar_status st) {
    switch (st) {
        case SPLIDAR_OK: return "ok";
        case SPLIDAR_EINVAL: return "invalid argument";
        case SPLIDAR_ENOCONV: return "power iteration did not converge within max_iter";
        case SPLIDAR_EZEROROW: return "zero or non-finite row normaliser";
        case SPLIDAR_ENOSPACE: return "workspace too small, ld < N, or misaligned pointer / ld";
        case SPLIDAR_ECUDA: return "CUDA runtime error";
    }
    return "unknown status";
}

int splidar_last_cuda_error(void) { return g_last_cuda_error; }

const char *splidar_build_info(void) {
    return "libsplidar sm_100a (nvcc " SPL_NVCC_VERSION "), fp64 vectors / fp64 accumulation";
}

// ---------------------------------------------------------------- steps 1-2 -----------------

static splidar_status vectors_and_build(const FluxDev *fl, int M, int N, int dt, int mode, void *P0,
                                        int64_t ld, int64_t mstride, char *ws, const WsLayout &L,
                                        cudaStream_t s) {
    const bool single = M == 1 && N + 1 <= kSmallVecMax;   // the profile travels in the parameters
    if (!single) SPL_CUDA(upload_async(ws + L.flux, fl, sizeof(FluxDev) * (size_t)M, s));
    VecPtrs vp = vec_ptrs(ws, L);
    SPL_CUDA(launch_flux_vectors(reinterpret_cast<const FluxDev *>(ws + L.flux), M, N, vp, N, s,
                                 single ? fl : nullptr));
    if (P0) SPL_CUDA(launch_build(vp, N, M, N, dt, mode, P0, ld, mstride, s));
    return SPLIDAR_OK;
}

splidar_status splidar_flux_vectors(const splidar_flux *flux, double *F, double *lam, double *w,
                                    double *inv_d, double *lambda_total, void *ws, size_t ws_bytes,
                                    void *stream) {
    SPL_NVTX_RANGE();
    splidar_status st = check_flux(flux);
    if (st) return st;
    const int N = flux->n_bins;
    const WsLayout L = ws_layout(N, 1, 1);
    if ((st = check_ws(ws, ws_bytes, L))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    char *wsb = static_cast<char *>(ws);
    FluxDev d = to_dev(flux);
    if ((st = vectors_and_build(&d, 1, N, SPLIDAR_F64, 0, nullptr, 0, 0, wsb, L, s))) return st;
    VecPtrs vp = vec_ptrs(wsb, L);
    const size_t nb = sizeof(double) * (size_t)N;
    if (F) SPL_CUDA(cudaMemcpyAsync(F, vp.F, nb, cudaMemcpyDeviceToDevice, s));
    if (lam) SPL_CUDA(cudaMemcpyAsync(lam, vp.lam, nb, cudaMemcpyDeviceToDevice, s));
    if (w) SPL_CUDA(cudaMemcpyAsync(w, vp.w, nb, cudaMemcpyDeviceToDevice, s));
    if (inv_d) SPL_CUDA(cudaMemcpyAsync(inv_d, vp.invD, nb, cudaMemcpyDeviceToDevice, s));
    if (lambda_total) SPL_CUDA(cudaMemcpyAsync(lambda_total, vp.scal, sizeof(double), cudaMemcpyDeviceToDevice, s));
    return SPLIDAR_OK;
}

splidar_status splidar_build_base_batched(const splidar_flux *fluxes, int32_t n_matrices, splidar_dtype dt,
                                          splidar_entry mode, void *P0, int64_t ld, int64_t matrix_stride,
                                          void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!fluxes || n_matrices < 1 || n_matrices > 65535) return SPLIDAR_EINVAL;
    if (mode != SPLIDAR_ENTRY_FACTORED && mode != SPLIDAR_ENTRY_EXP) return SPLIDAR_EINVAL;
    const int N = fluxes[0].n_bins;
    splidar_status st;
    for (int m = 0; m < n_matrices; ++m)
        if ((st = check_flux(&fluxes[m], N))) return st;
    if ((st = check_matrix(P0, N, ld, dt))) return st;
    if (n_matrices > 1 && (matrix_stride < (int64_t)N * ld || matrix_stride % ld != 0)) return SPLIDAR_EINVAL;
    const WsLayout L = ws_layout(N, n_matrices, 1);
    if ((st = check_ws(ws, ws_bytes, L))) return st;
    std::vector<FluxDev> d((size_t)n_matrices);
    for (int m = 0; m < n_matrices; ++m) d[(size_t)m] = to_dev(&fluxes[m]);
    return vectors_and_build(d.data(), n_matrices, N, dt, mode, P0, ld, matrix_stride,
                             static_cast<char *>(ws), L, (cudaStream_t)stream);
}

splidar_status splidar_build_base(const splidar_flux *flux, splidar_dtype dt, splidar_entry mode, void *P0,
                                  int64_t ld, void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    return splidar_build_base_batched(flux, 1, dt, mode, P0, ld, flux ? (int64_t)flux->n_bins * ld : 0, ws,
                                      ws_bytes, stream);
}

splidar_status splidar_apply_deadtime(const void *P0, void *P, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                      double t_r, double t_d, void *stream) {
    SPL_NVTX_RANGE();
    int32_t l;
    splidar_status st = splidar_shift(t_r, n_bins, t_d, &l);
    if (st) return st;
    if ((st = check_matrix(P0, n_bins, ld, dt))) return st;
    if ((st = check_matrix(P, n_bins, ld, dt))) return st;
    if (P == P0) return SPLIDAR_EINVAL;
    return cuda_status(launch_apply_deadtime(P0, P, n_bins, ld, dt, l, (cudaStream_t)stream));
}

// f4: the element-wise Eq. 4 construction, for same-hardware comparisons.
splidar_status splidar_build_eq4(const splidar_flux *flux, double t_d, splidar_dtype dt, void *P, int64_t ld,
                                 void *stream) {
    splidar_status st = check_flux(flux);
    if (st) return st;
    if (!std::isfinite(t_d) || t_d < 0.0) return SPLIDAR_EINVAL;
    if ((st = check_matrix(P, flux->n_bins, ld, dt))) return st;
    const double u = shift_u(flux->t_r, flux->n_bins, t_d);   // x_d / Delta (R4)
    return cuda_status(launch_build_eq4(to_dev(flux), u, dt, P, ld, (cudaStream_t)stream));
}

// ---------------------------------------------------------------- step 4: plans --------------

struct splidar_plan_s {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    WsLayout L;
    PowerArgs args;
    int M = 0, V = 0, Vreal = 0;
    std::vector<int> lsh;          // [M * V] (padded)
    std::vector<SolveState> host;  // [M * V]
    SolveState *host_pinned = nullptr;   // [M * V] page-locked copy target of splidar_plan_info (lazy)
    // fused building plans: steps 1-4 (flux vectors, build, fused solver) captured once as a graph,
    // replayed by launches on a stream that is not capturing; re-captured when fargs change
    cudaGraphExec_t fexec = nullptr;
    FusedArgs fargs_cap;
    std::vector<int> out_idx;      // [M * V]
    // eager mode (SPLIDAR_EAGER=1 at plan creation): the same kernels launched from a host loop that
    // reads the any-active flag after each iteration; for profilers that do not descend into
    // conditional graph bodies. Control only: every step still runs in the kernels.
    bool eager = false;
    SolverKernels k;
    PowerArgs eager_args;
    std::vector<unsigned char> fin_args;
    unsigned *host_flag = nullptr;
    // small N: every iteration of every (matrix, vector) in one clustered launch (fused.cu)
    bool fused = false;
    // graph plans: the iterations are one cooperative k_power_loop launch (else the WHILE node)
    bool persist = false;
    int dt = 0;
    FusedArgs fargs;
    I8Kernels q;       // int8 tensor-core GEMV (args.i8)
    bool shard = false;   // row shard (splidar_plan_create_rows): stepped by the caller
    // plans that build their matrices (splidar_plan_create_build): steps 1-2 run inside every launch,
    // and the build also reduces the column sums of the stored entries = the first power-iteration
    // product from the uniform start, shared by every dead time of a matrix (x^0 = 1/N is invariant
    // under the row permutation J_l): the solve starts at iteration 1 without a GEMV pass
    bool with_build = false;
    int bmode = 0;
    // fp32 factored building plans on the int8 GEMV store P~0 ENCODED when every column is in range:
    // each entry as its column's scaled integer (fixpt.cuh), so the GEMV needs no converters
    // (k_power_step_i8e); the column exponents come from launch_enc_colexp before the build
    bool enc = false;
    std::vector<FluxDev> bflux;
    char *ws = nullptr;
};

// Enqueue steps 1-2 of a building plan (flux vectors, entries + column sums) on s.
static cudaError_t plan_enqueue_build(const splidar_plan_s *p, int dt, cudaStream_t s) {
    const WsLayout &L = p->L;
    const int M = p->M, N = L.N;
    VecPtrs vp;
    {
        double *b = reinterpret_cast<double *>(p->ws + L.vec);
        const size_t MN = (size_t)L.M * L.N;
        vp.F = b; vp.lam = b + MN; vp.w = b + 2 * MN; vp.invD = b + 3 * MN; vp.invZ = b + 4 * MN;
        vp.scal = b + 5 * MN;
        vp.ntile = (L.N + 1 + kScanTile - 1) / kScanTile;
        vp.tiles = vp.scal + (size_t)L.M * 8;
    }
    // the fluxes are read from the plan's workspace (splidar_plan_set_fluxes replaces them there)
    cudaError_t e = launch_flux_vectors(reinterpret_cast<const FluxDev *>(p->ws + L.flux), M, N, vp, N, s, nullptr);
    if (e != cudaSuccess) return e;
    ColStats cst{};
    if (p->enc) {       // column exponents and range test first, then the build encodes (or not)
        e = launch_enc_colexp(vp, N, M, N, p->args.colexp, p->args.colmin, p->args.glob + 3, s);
        if (e != cudaSuccess) return e;
        cst.colexp = p->args.colexp;
        cst.flag = p->args.glob + 3;
        cst.R = i8_range_bits(dt);
        cst.enc = 1;
    } else if (p->args.i8) {   // the int8 GEMV's column exponents and range test come from the build too
        int *ep = reinterpret_cast<int *>(p->ws + L.epart);
        cst.emax_part = ep;
        cst.emin_part = ep + (size_t)M * colsum_chunks(N) * N;
        cst.colexp = p->args.colexp;
        cst.flag = p->args.glob + 3;
        cst.R = i8_range_bits(dt);
        cst.zero_col_exp = dt == SPLIDAR_F64 ? 2047 : 255;
    }
    return launch_build(vp, N, M, N, dt, p->bmode, const_cast<void *>(p->args.P), p->args.ld, p->args.mstride, s, 0,
                        N, p->fused ? nullptr : reinterpret_cast<double *>(p->ws + L.cpart),
                        p->fused ? nullptr : reinterpret_cast<double *>(p->ws + L.csum), cst);
}

static splidar_status plan_build(splidar_plan_s *p, int dt, double *pi, char *ws, cudaStream_t s) {
    const WsLayout &L = p->L;
    PowerArgs &a = p->args;
    p->ws = ws;
    p->dt = dt;
    if (p->with_build)   // the fluxes stay in the plan's workspace
        SPL_CUDA(spl::upload_async(ws + L.flux, p->bflux.data(), sizeof(FluxDev) * p->bflux.size(), s));
    a.y = reinterpret_cast<double *>(ws + L.y);
    a.X = reinterpret_cast<double *>(ws + L.X);
    a.part = reinterpret_cast<double *>(ws + L.part);
    a.ssum = reinterpret_cast<double *>(ws + L.ssum);
    a.l1part = reinterpret_cast<double *>(ws + L.l1part);
    a.st = reinterpret_cast<SolveState *>(ws + L.state);
    a.lsh = reinterpret_cast<const int *>(ws + L.lsh);
    a.strip_cnt = reinterpret_cast<unsigned *>(ws + L.strip_cnt);
    a.mv_cnt = reinterpret_cast<unsigned *>(ws + L.mv_cnt);
    a.act = reinterpret_cast<int *>(ws + L.act);
    a.glob = reinterpret_cast<unsigned *>(ws + L.glob);
    // GEMV launch timer in the glob block's spare bytes (ptx.cuh; read by splidar_plan_gemv_time)
    a.ktime = reinterpret_cast<unsigned long long *>(ws + L.glob + 64);
    SPL_CUDA(cudaMemsetAsync(a.ktime, 0, 4 * sizeof(unsigned long long), s));
    a.N = L.N;
    if (a.rows == 0) a.rows = L.N;      // a row shard sets rows / row0 / ypart before plan_build
    a.M = L.M;
    a.V = L.V;
    a.strips = L.strips;
    a.chunks = L.chunks;
    a.xstride = L.xstride;
    a.ximg = reinterpret_cast<unsigned char *>(ws + L.ximg);
    a.colexp = reinterpret_cast<int *>(ws + L.colexp);
    a.colmin = reinterpret_cast<int *>(ws + L.colmin);
    a.smax = reinterpret_cast<double *>(ws + L.smax);
    a.xtau = reinterpret_cast<int *>(ws + L.xtau);
    a.i8 = 0;
    if (!p->shard) {   // the int8 tensor-core GEMV (SPLIDAR_I8=0 keeps the DMMA / DFMA kernels only)
        const char *e = getenv("SPLIDAR_I8");
        const bool allow = !(e && e[0] == '0') && (dt == SPLIDAR_F32 || (e && e[0] == '2'));
        if (allow && i8_supported(dt, a)) {
            a.i8 = 1;
            const char *d = getenv("SPLIDAR_I8_DBG");
            a.i8_dbg = d ? atoi(d) : 0;
            a.strips_i8 = L.N / i8_tile_cols(dt);
            const char *ev = getenv("SPLIDAR_I8_ENC");
            p->enc = p->with_build && dt == SPLIDAR_F32 && p->bmode == SPLIDAR_ENTRY_FACTORED && L.N <= 131072 &&
                     !(ev && ev[0] == '0');
        }
    }

    SPL_CUDA(spl::upload_async(ws + L.lsh, p->lsh.data(), sizeof(int) * p->lsh.size(), s));
    SPL_CUDA(spl::upload_async(ws + L.oidx, p->out_idx.data(), sizeof(int) * p->out_idx.size(), s));

    {   // small N: the fused single-launch solver (SPLIDAR_FUSED=0 forces the general path)
        const char *e = getenv("SPLIDAR_FUSED");
        int C, R;
        if (!p->shard && !(e && e[0] == '0') && !fused_shape(L.N, &C, &R)) {
            p->fused = true;
            p->dt = dt;
            FusedArgs &f = p->fargs;
            memset(&f, 0, sizeof(f));
            f.P = a.P;
            f.ld = a.ld;
            f.mstride = a.mstride;
            f.N = L.N;
            f.M = L.M;
            f.V = L.V;
            f.C = C;
            f.R = R;
            f.resident = fused_resident(L.N, R, dt);
            f.lsh = reinterpret_cast<const int *>(ws + L.lsh);
            f.out_idx = reinterpret_cast<const int *>(ws + L.oidx);
            f.n_inline = (size_t)L.M * L.V <= (size_t)kFusedInline ? 1 : 0;
            for (size_t i = 0; f.n_inline && i < p->lsh.size(); ++i) {
                f.lsh_in[i] = p->lsh[i];
                f.oidx_in[i] = p->out_idx[i];
            }
            f.pi = pi;
            f.st = a.st;
            f.tol = a.tol;
            f.max_iter = a.max_iter;
            {
                const char *e2 = getenv("SPLIDAR_FUSED_P2P");
                f.p2p = (e2 && e2[0] == '0') ? 0 : 1;
                const char *e3 = getenv("SPLIDAR_FUSED_LDG");   // 0: rows not resident stream through a TMA ring
                f.ldg = (e3 && e3[0] == '0') ? 0 : 1;
                const char *e4 = getenv("SPLIDAR_FUSED_1X");    // 0: two exchanges per product
                // (the TMA ring leaves no shared memory for the double buffers at N = 2048)
                f.one_x = (f.p2p && (f.resident || f.ldg) && !(e4 && e4[0] == '0')) ? 1 : 0;
            }
            return SPLIDAR_OK;
        }
    }

    if (p->shard) {   // row shard: the caller steps the kernels around its all-reduce (no graph)
        if (solver_kernels(dt, L.V, &p->k, a)) return SPLIDAR_EINVAL;
        p->eager_args = a;
        p->eager_args.use_handle = 0;
        p->fin_args.resize(finish_args_size());
        make_finish_args(p->fin_args.data(), p->eager_args, pi, reinterpret_cast<const int *>(ws + L.oidx));
        return SPLIDAR_OK;
    }
    SPL_CUDA(cudaGraphCreate(&p->graph, 0));
    SolverKernels &k = p->k;
    if (solver_kernels(dt, L.V, &k, a)) return SPLIDAR_EINVAL;
    // SPLIDAR_PERSIST=1: the iterations as ONE cooperative launch of k_power_loop (GEMV + check fused,
    // grid barriers) when the plan is not on the int8 GEMV and the whole persistent grid can be
    // resident at once. Opt-in: measured against the conditional WHILE node of [k_power_step ->
    // k_power_check] (same box, alternating), it gained 0.3 % at c4 (DFMA) and lost 1.6 % at c5
    // (DMMA: the inlined GEMV pass itself runs ~1.8 % slower in the larger kernel), DESIGN.md §6.
    p->persist = false;
    if (!a.i8 && k.loop_fn) {
        const char *e = getenv("SPLIDAR_PERSIST");
        int nb = 0;
        if (e && e[0] == '1') {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k.loop_fn, (int)k.step_block.x, k.step_smem) !=
                cudaSuccess) {
                (void)cudaGetLastError();
                nb = 0;
            }
            p->persist = (long)nb * device_sm_count() >= (long)k.step_grid.x;
        }
    }
    if (p->persist) {
        a.use_handle = 0;
    } else {
        cudaGraphConditionalHandle h;
        SPL_CUDA(cudaGraphConditionalHandleCreate(&h, p->graph, 1, cudaGraphCondAssignDefault));
        a.use_handle = 1;
        a.handle = h;
    }
    p->eager_args = a;
    p->eager_args.use_handle = 0;
    {
        const char *e = getenv("SPLIDAR_EAGER");
        p->eager = e && e[0] == '1';
    }

    I8Kernels &q = p->q;
    if (a.i8) SPL_CUDA(i8_kernels(dt, &q, a));

    cudaKernelNodeParams kp;
    memset(&kp, 0, sizeof(kp));
    void *init_args[] = {&a};
    cudaGraphNode_t n_init, n_while, n_step, n_fin, n_prev = nullptr;
    if (p->with_build) {   // steps 1-2 as a child graph captured from the same launch code
        cudaStream_t cs;
        SPL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t bg = nullptr;
        cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            const cudaError_t eb = plan_enqueue_build(p, dt, cs);
            e = cudaStreamEndCapture(cs, &bg);
            if (e == cudaSuccess) e = eb;
        }
        if (e == cudaSuccess) e = cudaGraphAddChildGraphNode(&n_prev, p->graph, nullptr, 0, bg);
        if (bg) cudaGraphDestroy(bg);
        cudaStreamDestroy(cs);
        SPL_CUDA(e);
    }
    int rows_per_cta = q.rows_per_cta;
    void *colexp_args[] = {&a, &rows_per_cta};
    if (a.i8 && !p->with_build) {   // range test of the stored matrix: flag = 1, then every column may clear it
        cudaGraphNode_t n_prep, n_col, n_chk;
        kp.func = q.prep_fn;
        kp.gridDim = q.small_grid;
        kp.blockDim = dim3(256);
        kp.kernelParams = init_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_prep, p->graph, n_prev ? &n_prev : nullptr, n_prev ? 1 : 0, &kp));
        kp.func = q.colexp_fn;
        kp.gridDim = q.colexp_grid;
        kp.blockDim = q.colexp_block;
        kp.kernelParams = colexp_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_col, p->graph, &n_prep, 1, &kp));
        kp.func = q.check_fn;
        kp.gridDim = q.small_grid;
        kp.blockDim = dim3(256);
        kp.kernelParams = init_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_chk, p->graph, &n_col, 1, &kp));
        n_prev = n_chk;
    }
    kp.func = k.init_fn;
    kp.gridDim = k.init_grid;
    kp.blockDim = k.init_block;
    kp.kernelParams = init_args;
    SPL_CUDA(cudaGraphAddKernelNode(&n_init, p->graph, n_prev ? &n_prev : nullptr, n_prev ? 1 : 0, &kp));
    cudaGraphNode_t n_loop_dep = n_init;
    PowerArgs ac = a;      // iteration 1 from the build's column sums (no GEMV pass)
    if (p->with_build) {
        ac.ypart = reinterpret_cast<double *>(ws + L.csum);
        ac.ypart_shared = 1;
        void *cargs[] = {&ac};
        cudaGraphNode_t n_ss, n_ck;
        kp.func = k.ssum_fn;
        kp.gridDim = dim3((unsigned)(L.strips > a.strips_i8 ? L.strips : a.strips_i8), (unsigned)(L.M * L.V));
        kp.blockDim = dim3(256);
        kp.sharedMemBytes = 0;
        kp.kernelParams = cargs;
        SPL_CUDA(cudaGraphAddKernelNode(&n_ss, p->graph, &n_init, 1, &kp));
        kp.func = k.check_fn;
        kp.gridDim = k.check_grid;
        kp.blockDim = k.check_block;
        SPL_CUDA(cudaGraphAddKernelNode(&n_ck, p->graph, &n_ss, 1, &kp));
        n_loop_dep = n_ck;
    }

    if (p->persist) {
        void *loop_args[] = {&a};
        kp.func = k.loop_fn;
        kp.gridDim = k.step_grid;
        kp.blockDim = k.step_block;
        kp.sharedMemBytes = k.step_smem;
        kp.kernelParams = loop_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_while, p->graph, &n_loop_dep, 1, &kp));
        cudaKernelNodeAttrValue coop = {};
        coop.cooperative = 1;
        SPL_CUDA(cudaGraphKernelNodeSetAttribute(n_while, cudaLaunchAttributeCooperative, &coop));
        std::vector<unsigned char> &fa = p->fin_args;
        fa.resize(finish_args_size());
        make_finish_args(fa.data(), a, pi, reinterpret_cast<const int *>(ws + L.oidx));
        void *fin_args[] = {fa.data()};
        kp.func = k.finish_fn;
        kp.gridDim = k.finish_grid;
        kp.blockDim = k.finish_block;
        kp.sharedMemBytes = 0;
        kp.kernelParams = fin_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_fin, p->graph, &n_while, 1, &kp));
        SPL_CUDA(cudaGraphInstantiate(&p->exec, p->graph, 0));
        return SPLIDAR_OK;
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = a.handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    SPL_CUDA(cudaGraphAddNode(&n_while, p->graph, &n_loop_dep, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];

    void *step_args[] = {&a};
    cudaGraphNode_t n_i8 = nullptr;
    if (a.i8) {
        void *i8_args[] = {&a, q.tmap};
        kp.func = p->enc ? q.step_enc_fn : q.step_fn;
        kp.gridDim = q.step_grid;
        kp.blockDim = q.step_block;
        kp.sharedMemBytes = p->enc ? q.step_enc_smem : q.step_smem;
        kp.kernelParams = i8_args;
        SPL_CUDA(cudaGraphAddKernelNode(&n_i8, body, nullptr, 0, &kp));
    }
    kp.func = k.step_fn;
    kp.gridDim = k.step_grid;
    kp.blockDim = k.step_block;
    kp.sharedMemBytes = k.step_smem;
    kp.kernelParams = step_args;
    SPL_CUDA(cudaGraphAddKernelNode(&n_step, body, n_i8 ? &n_i8 : nullptr, n_i8 ? 1 : 0, &kp));
    void *check_args[] = {&a};
    kp.func = k.check_fn;
    kp.gridDim = k.check_grid;
    kp.blockDim = k.check_block;
    kp.sharedMemBytes = 0;
    kp.kernelParams = check_args;
    cudaGraphNode_t n_check;
    if (pdl_enabled()) {   // programmatic edge: the check's CTAs are scheduled while the GEMV runs
        SPL_CUDA(cudaGraphAddKernelNode(&n_check, body, nullptr, 0, &kp));
        cudaGraphEdgeData ed = {};
        ed.from_port = cudaGraphKernelNodePortProgrammatic;
        ed.type = cudaGraphDependencyTypeProgrammatic;
        SPL_CUDA(cudaGraphAddDependencies_v2(body, &n_step, &n_check, &ed, 1));
    } else {
        SPL_CUDA(cudaGraphAddKernelNode(&n_check, body, &n_step, 1, &kp));
    }

    std::vector<unsigned char> &fa = p->fin_args;
    fa.resize(finish_args_size());
    make_finish_args(fa.data(), a, pi, reinterpret_cast<const int *>(ws + L.oidx));
    void *fin_args[] = {fa.data()};
    kp.func = k.finish_fn;
    kp.gridDim = k.finish_grid;
    kp.blockDim = k.finish_block;
    kp.sharedMemBytes = 0;
    kp.kernelParams = fin_args;
    SPL_CUDA(cudaGraphAddKernelNode(&n_fin, p->graph, &n_while, 1, &kp));

    SPL_CUDA(cudaGraphInstantiate(&p->exec, p->graph, 0));
    return SPLIDAR_OK;
}

void splidar_plan_destroy(splidar_plan plan) {
    if (!plan) return;
    if (plan->exec) cudaGraphExecDestroy(plan->exec);
    if (plan->host_flag) cudaFreeHost(plan->host_flag);
    if (plan->host_pinned) cudaFreeHost(plan->host_pinned);
    if (plan->fexec) cudaGraphExecDestroy(plan->fexec);
    if (plan->graph) cudaGraphDestroy(plan->graph);
    delete plan;
}

// Internal: plan with explicit shifts (l < 0 = unused vector) and output rows.
static splidar_status plan_create_l(splidar_plan *out, const void *P0, int M, int64_t mstride, int N, int64_t ld,
                                    int dt, const int *l, int V, double tol, int max_iter, double *pi,
                                    const int *out_idx, void *ws, size_t ws_bytes, cudaStream_t s,
                                    int row0 = 0, int n_rows = -1, double *ypart = nullptr,
                                    const FluxDev *bflux = nullptr, int bmode = 0) {
    *out = nullptr;
    splidar_status st;
    if ((st = check_matrix(P0, N, ld, dt))) return st;
    if (M < 1 || M > 65535 || V < 1 || V > kMaxVectors || !pi) return SPLIDAR_EINVAL;
    if (M > 1 && (mstride < (int64_t)N * ld || mstride % ld != 0)) return SPLIDAR_EINVAL;
    if (!(tol > 0.0) || !std::isfinite(tol) || max_iter < 1) return SPLIDAR_EINVAL;
    splidar_plan_s *p = new splidar_plan_s();
    p->L = ws_layout(N, M, V);
    if ((st = check_ws(ws, ws_bytes, p->L))) { delete p; return st; }
    p->M = M;
    p->V = p->L.V;
    p->Vreal = V;
    p->lsh.assign((size_t)M * p->V, -1);
    p->out_idx.assign((size_t)M * p->V, -1);
    for (int m = 0; m < M; ++m)
        for (int v = 0; v < V; ++v) {
            p->lsh[(size_t)m * p->V + v] = l[(size_t)m * V + v];
            p->out_idx[(size_t)m * p->V + v] = out_idx ? out_idx[(size_t)m * V + v] : m * V + v;
        }
    p->host.resize((size_t)M * p->V);
    memset(&p->args, 0, sizeof(p->args));
    p->args.P = P0;
    p->args.ld = ld;
    p->args.mstride = mstride;
    p->args.tol = tol;
    p->args.max_iter = max_iter;
    if (bflux) {
        p->with_build = true;
        p->bmode = bmode;
        p->bflux.assign(bflux, bflux + M);
    }
    if (n_rows >= 0) {
        p->shard = true;
        p->args.rows = n_rows;
        p->args.row0 = row0;
        p->args.ypart = ypart;
    }
    if ((st = plan_build(p, dt, pi, static_cast<char *>(ws), s))) {
        splidar_plan_destroy(p);
        return st;
    }
    *out = p;
    return SPLIDAR_OK;
}

splidar_status splidar_plan_create(splidar_plan *plan, const void *P0, int32_t n_matrices, int64_t matrix_stride,
                                   int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r, const double *t_d,
                                   int32_t n_vectors, double tol, int32_t max_iter, double *pi, void *ws,
                                   size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan || !t_d || n_matrices < 1 || n_vectors < 1 || n_vectors > kMaxVectors) return SPLIDAR_EINVAL;
    std::vector<int> l((size_t)n_matrices * n_vectors);
    for (size_t i = 0; i < l.size(); ++i) {
        int32_t li;
        splidar_status st = splidar_shift(t_r, n_bins, t_d[i], &li);
        if (st) return st;
        l[i] = li;
    }
    return plan_create_l(plan, P0, n_matrices, matrix_stride, n_bins, ld, dt, l.data(), n_vectors, tol, max_iter,
                         pi, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

splidar_status splidar_plan_create_build(splidar_plan *plan, const splidar_flux *fluxes, int32_t n_matrices,
                                         splidar_entry mode, splidar_dtype dt, void *P0, int64_t matrix_stride,
                                         int64_t ld, const double *t_d, int32_t n_vectors, double tol,
                                         int32_t max_iter, double *pi, void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan || !fluxes || !t_d || n_matrices < 1 || n_matrices > 65535 || n_vectors < 1 ||
        n_vectors > kMaxVectors)
        return SPLIDAR_EINVAL;
    if (mode != SPLIDAR_ENTRY_FACTORED && mode != SPLIDAR_ENTRY_EXP) return SPLIDAR_EINVAL;
    const int N = fluxes[0].n_bins;
    splidar_status st;
    std::vector<FluxDev> d((size_t)n_matrices);
    for (int m = 0; m < n_matrices; ++m) {
        if ((st = check_flux(&fluxes[m], N))) return st;
        if (fluxes[m].t_r != fluxes[0].t_r) return SPLIDAR_EINVAL;     // one shift rule per plan
        d[(size_t)m] = to_dev(&fluxes[m]);
    }
    std::vector<int> l((size_t)n_matrices * n_vectors);
    for (size_t i = 0; i < l.size(); ++i) {
        int32_t li;
        if ((st = splidar_shift(fluxes[0].t_r, N, t_d[i], &li))) return st;
        l[i] = li;
    }
    return plan_create_l(plan, P0, n_matrices, n_matrices > 1 ? matrix_stride : (int64_t)N * ld, N, ld, dt, l.data(),
                         n_vectors, tol, max_iter, pi, nullptr, ws, ws_bytes, (cudaStream_t)stream, 0, -1, nullptr,
                         d.data(), mode);
}

splidar_status splidar_plan_set_fluxes(splidar_plan plan, const splidar_flux *fluxes, int32_t n_matrices,
                                       void *stream) {
    SPL_NVTX_RANGE();
    if (!plan || !plan->with_build || !fluxes || n_matrices != plan->M) return SPLIDAR_EINVAL;
    splidar_status st;
    for (int m = 0; m < n_matrices; ++m) {
        if ((st = check_flux(&fluxes[m], plan->L.N))) return st;
        if (fluxes[m].t_r != fluxes[0].t_r) return SPLIDAR_EINVAL;
        plan->bflux[(size_t)m] = to_dev(&fluxes[m]);
    }
    return cuda_status(spl::upload_async(plan->ws + plan->L.flux, plan->bflux.data(),
                                         sizeof(FluxDev) * plan->bflux.size(), (cudaStream_t)stream));
}

static splidar_status plan_launch_eager(splidar_plan_s *p, cudaStream_t s) {
    if (!p->host_flag) SPL_CUDA(cudaMallocHost(&p->host_flag, sizeof(unsigned)));
    const SolverKernels &k = p->k;
    const I8Kernels &q = p->q;
    void *args[] = {&p->eager_args};
    if (p->with_build) SPL_CUDA(plan_enqueue_build(p, p->dt, s));
    if (p->args.i8 && !p->with_build) {
        int rpc = q.rows_per_cta;
        void *cargs[] = {&p->eager_args, &rpc};
        SPL_CUDA(cudaLaunchKernel(q.prep_fn, q.small_grid, dim3(256), args, 0, s));
        SPL_CUDA(cudaLaunchKernel(q.colexp_fn, q.colexp_grid, q.colexp_block, cargs, 0, s));
        SPL_CUDA(cudaLaunchKernel(q.check_fn, q.small_grid, dim3(256), args, 0, s));
    }
    SPL_CUDA(cudaLaunchKernel(k.init_fn, k.init_grid, k.init_block, args, 0, s));
    bool more = true;
    if (p->with_build) {   // iteration 1 from the build's column sums
        PowerArgs ac = p->eager_args;
        ac.ypart = reinterpret_cast<double *>(p->ws + p->L.csum);
        ac.ypart_shared = 1;
        void *cargs[] = {&ac};
        const dim3 sgrid((unsigned)(p->L.strips > ac.strips_i8 ? p->L.strips : ac.strips_i8), (unsigned)(p->M * p->V));
        SPL_CUDA(cudaLaunchKernel(k.ssum_fn, sgrid, dim3(256), cargs, 0, s));
        SPL_CUDA(cudaLaunchKernel(k.check_fn, k.check_grid, k.check_block, cargs, 0, s));
        SPL_CUDA(cudaMemcpyAsync(p->host_flag, p->eager_args.glob + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        SPL_CUDA(cudaStreamSynchronize(s));
        more = *p->host_flag != 0;
    }
    void *i8_args[] = {&p->eager_args, const_cast<unsigned char *>(q.tmap)};
    for (int it = 0; more && it < p->args.max_iter; ++it) {
        if (p->args.i8)
            SPL_CUDA(cudaLaunchKernel(p->enc ? q.step_enc_fn : q.step_fn, q.step_grid, q.step_block, i8_args,
                                      p->enc ? q.step_enc_smem : q.step_smem, s));
        SPL_CUDA(cudaLaunchKernel(k.step_fn, k.step_grid, k.step_block, args, k.step_smem, s));
        SPL_CUDA(cudaLaunchKernel(k.check_fn, k.check_grid, k.check_block, args, 0, s));
        SPL_CUDA(cudaMemcpyAsync(p->host_flag, p->eager_args.glob + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        SPL_CUDA(cudaStreamSynchronize(s));
        if (!*p->host_flag && !p->args.i8_dbg) break;
    }
    void *fargs[] = {p->fin_args.data()};
    SPL_CUDA(cudaLaunchKernel(k.finish_fn, k.finish_grid, k.finish_block, fargs, 0, s));
    return SPLIDAR_OK;
}

int splidar_plan_kind(splidar_plan plan) {
    return !plan ? -1 : plan->fused ? SPLIDAR_PLAN_FUSED : plan->persist && !plan->eager ? SPLIDAR_PLAN_LOOP : SPLIDAR_PLAN_GRAPH;
}

int splidar_plan_gemv(splidar_plan plan, void *stream) {
    if (!plan) return -1;
    if (plan->fused) return SPLIDAR_GEMV_FUSED;
    if (!plan->args.i8) return SPLIDAR_GEMV_FP64;
    unsigned flag = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(&flag, plan->args.glob + 3, sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        g_last_cuda_error = (int)cudaGetLastError();
        return -1;
    }
    return flag ? SPLIDAR_GEMV_TENSOR_I8 : SPLIDAR_GEMV_FP64;
}

splidar_status splidar_plan_gemv_time(splidar_plan plan, int32_t reset, double *seconds, int64_t *launches,
                                      void *stream) {
    SPL_NVTX_RANGE();
    if (!plan || !seconds || !launches) return SPLIDAR_EINVAL;
    *seconds = 0.0;
    *launches = 0;
    if (plan->fused || !plan->args.ktime) return SPLIDAR_OK;
    unsigned long long h[2] = {0ull, 0ull};
    cudaStream_t s = (cudaStream_t)stream;
    SPL_CUDA(cudaMemcpyAsync(h, plan->args.ktime + 2, sizeof(h), cudaMemcpyDeviceToHost, s));
    if (reset) SPL_CUDA(cudaMemsetAsync(plan->args.ktime + 2, 0, sizeof(h), s));
    SPL_CUDA(cudaStreamSynchronize(s));
    *seconds = (double)h[0] * 1e-9;
    *launches = (int64_t)h[1];
    return SPLIDAR_OK;
}

int splidar_plan_storage(splidar_plan plan, void *stream) {
    if (!plan) return -1;
    if (!plan->enc) return SPLIDAR_STORAGE_IEEE;
    const int g = splidar_plan_gemv(plan, stream);   // encoded exactly when the range test passed
    return g < 0 ? -1 : g == SPLIDAR_GEMV_TENSOR_I8 ? SPLIDAR_STORAGE_ENCODED : SPLIDAR_STORAGE_IEEE;
}

splidar_status splidar_plan_launch(splidar_plan plan, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan) return SPLIDAR_EINVAL;
    if (plan->fused) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        SPL_CUDA(cudaStreamIsCapturing((cudaStream_t)stream, &cap));
        if (plan->with_build && cap == cudaStreamCaptureStatusNone && !plan->eager) {
            // one graph launch instead of three kernel launches (host cost of the small-N step)
            if (plan->fexec && memcmp(&plan->fargs_cap, &plan->fargs, sizeof(FusedArgs)) != 0) {
                cudaGraphExecDestroy(plan->fexec);
                plan->fexec = nullptr;
            }
            if (!plan->fexec) {
                void *fn = nullptr;   // kernel attributes are set outside the capture
                SPL_CUDA(fused_fn(plan->dt, plan->fargs.N, &fn));
                cudaStream_t cs;
                SPL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
                cudaGraph_t g = nullptr;
                cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
                if (e == cudaSuccess) {
                    cudaError_t eb = plan_enqueue_build(plan, plan->dt, cs);
                    if (eb == cudaSuccess) eb = launch_fused(plan->dt, plan->fargs, cs);
                    e = cudaStreamEndCapture(cs, &g);
                    if (e == cudaSuccess) e = eb;
                }
                if (e == cudaSuccess) e = cudaGraphInstantiate(&plan->fexec, g, 0);
                if (g) cudaGraphDestroy(g);
                cudaStreamDestroy(cs);
                if (e != cudaSuccess) plan->fexec = nullptr;
                SPL_CUDA(e);
                memcpy(&plan->fargs_cap, &plan->fargs, sizeof(FusedArgs));
            }
            return cuda_status(cudaGraphLaunch(plan->fexec, (cudaStream_t)stream));
        }
        if (plan->with_build) SPL_CUDA(plan_enqueue_build(plan, plan->dt, (cudaStream_t)stream));
        return cuda_status(launch_fused(plan->dt, plan->fargs, (cudaStream_t)stream));
    }
    if (plan->eager) return plan_launch_eager(plan, (cudaStream_t)stream);
    return cuda_status(cudaGraphLaunch(plan->exec, (cudaStream_t)stream));
}

splidar_status splidar_plan_info(splidar_plan plan, splidar_solve_info *info, void *stream) {
    if (!plan) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    // page-locked target: an asynchronous copy ordered behind the launch, then the one synchronisation
    // (a pageable target would stage through a driver buffer)
    if (!plan->host_pinned &&
        cudaMallocHost(reinterpret_cast<void **>(&plan->host_pinned), sizeof(SolveState) * plan->host.size()) != cudaSuccess) {
        (void)cudaGetLastError();
        plan->host_pinned = nullptr;
    }
    SolveState *hs = plan->host_pinned ? plan->host_pinned : plan->host.data();
    SPL_CUDA(cudaMemcpyAsync(hs, plan->args.st, sizeof(SolveState) * plan->host.size(), cudaMemcpyDeviceToHost, s));
    SPL_CUDA(cudaStreamSynchronize(s));
    bool all = true;
    for (int m = 0; m < plan->M; ++m)
        for (int v = 0; v < plan->Vreal; ++v) {
            const SolveState &h = hs[(size_t)m * plan->V + v];
            all = all && h.converged;
            if (info) {
                splidar_solve_info &o = info[(size_t)m * plan->Vreal + v];
                o.iters = h.iters;
                o.converged = h.converged;
                o.shift_l = h.l;
                o.reserved = 0;
                o.l1_change = h.change;
                o.lambda_total = 0.0;
            }
        }
    return all ? SPLIDAR_OK : SPLIDAR_ENOCONV;
}

splidar_status splidar_plan_execute(splidar_plan plan, splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    splidar_status st = splidar_plan_launch(plan, stream);
    if (st) return st;
    return splidar_plan_info(plan, info, stream);
}

// ---- plan cache of the one-shot calls (splidar_stationary, splidar_stationary_multi) ----------
// A plan binds pointers (P0, pi, workspace), sizes, dtype, tol and max_iter; the shifts l and output
// rows live in the workspace and are re-uploaded (one small upload) by every launch of a cached plan. A
// one-shot call with the same binding as an earlier one therefore replays that call's instantiated
// graph instead of building, instantiating and destroying one (the host cost that dominated small N).
// Keyed by the current device too. LRU of kPlanCache entries; splidar_plan_cache_clear frees them.
namespace {
struct PlanKey {
    int dev, M, N, V, dt, max_iter;
    const void *P0;
    int64_t mstride, ld;
    double tol;
    double *pi;
    void *ws;
    size_t ws_bytes;
    bool operator==(const PlanKey &o) const {
        return dev == o.dev && M == o.M && N == o.N && V == o.V && dt == o.dt && max_iter == o.max_iter &&
               P0 == o.P0 && mstride == o.mstride && ld == o.ld && tol == o.tol && pi == o.pi && ws == o.ws &&
               ws_bytes == o.ws_bytes;
    }
};
struct CachedPlan {
    PlanKey key;
    splidar_plan plan;
    std::vector<int> l;
};
constexpr size_t kPlanCache = 16;
std::mutex g_cache_mu;
std::list<CachedPlan> g_cache;   // most recently used first
}  // namespace

// Instantiated lambda_2 graphs of earlier calls, keyed by everything baked into their kernel
// parameters (device, matrix, sizes, shift, pi, tolerances, workspace); LRU of 8, cleared with the
// plan cache. A repeated call replays the graph instead of building and instantiating it again.
namespace {
struct SdCached {
    int dev, dt;
    SdArgs a;
    cudaGraphExec_t x;
};
std::list<SdCached> g_sd_cache;
bool sd_same(const SdArgs &u, const SdArgs &v) {
    return u.p.P == v.p.P && u.p.ld == v.p.ld && u.p.N == v.p.N && u.p.y == v.p.y && u.l == v.l && u.pi == v.pi &&
           u.tol == v.tol && u.max_iter == v.max_iter && u.sd == v.sd && u.part == v.part;
}
}  // namespace

static splidar_status cached_execute(const void *P0, int M, int64_t mstride, int N, int64_t ld, int dt,
                                     const int *l, int V, double tol, int max_iter, double *pi, void *ws,
                                     size_t ws_bytes, splidar_solve_info *info, cudaStream_t s,
                                     double *pi_host = nullptr) {
    PlanKey key{current_device(), M, N, V, dt, max_iter, P0, mstride, ld, tol, pi, ws, ws_bytes};
    const std::vector<int> lv(l, l + (size_t)M * V);
    splidar_plan plan = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
            if (it->key == key) {
                plan = it->plan;
                for (int m = 0; m < M; ++m)
                    for (int v = 0; v < V; ++v) plan->lsh[(size_t)m * plan->V + v] = lv[(size_t)m * V + v];
                it->l = lv;
                if (plan->fused && plan->fargs.n_inline) {   // small N: the shifts ride in the parameters
                    for (size_t i = 0; i < plan->lsh.size(); ++i) plan->fargs.lsh_in[i] = plan->lsh[i];
                    g_cache.splice(g_cache.begin(), g_cache, it);
                    break;
                }
                // the workspace is scratch between calls (the caller may have used it for anything):
                // the plan's shifts and output rows go back in with one upload per launch
                const WsLayout &L = plan->L;
                std::vector<unsigned char> blob(L.oidx + sizeof(int) * plan->out_idx.size() - L.lsh, 0);
                memcpy(blob.data(), plan->lsh.data(), sizeof(int) * plan->lsh.size());
                memcpy(blob.data() + (L.oidx - L.lsh), plan->out_idx.data(), sizeof(int) * plan->out_idx.size());
                SPL_CUDA(spl::upload_async(static_cast<char *>(ws) + L.lsh, blob.data(), blob.size(), s));
                g_cache.splice(g_cache.begin(), g_cache, it);
                break;
            }
    }
    if (!plan) {
        splidar_status st = plan_create_l(&plan, P0, M, mstride, N, ld, dt, l, V, tol, max_iter, pi, nullptr, ws,
                                          ws_bytes, s);
        if (st) return st;
        std::lock_guard<std::mutex> lock(g_cache_mu);
        g_cache.push_front(CachedPlan{key, plan, lv});
        while (g_cache.size() > kPlanCache) {
            splidar_plan_destroy(g_cache.back().plan);
            g_cache.pop_back();
        }
    }
    // the cached plan is used under the cache lock's protection only for lookup; like any plan it
    // must not be launched concurrently on two streams with the same workspace (the caller's contract)
    splidar_status st = splidar_plan_launch(plan, s);
    if (st) return st;
    if (pi_host)   // the result's copy to the host rides on the same stream sync as the info
        SPL_CUDA(cudaMemcpyAsync(pi_host, pi, sizeof(double) * (size_t)M * V * N, cudaMemcpyDeviceToHost, s));
    return splidar_plan_info(plan, info, s);
}

void splidar_plan_cache_clear(void) {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    for (auto &c : g_cache) splidar_plan_destroy(c.plan);
    g_cache.clear();
    for (auto &c : g_sd_cache) cudaGraphExecDestroy(c.x);
    g_sd_cache.clear();
}

splidar_status splidar_stationary(const void *P0, int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r,
                                  double t_d, double tol, int32_t max_iter, double *pi, void *ws,
                                  size_t ws_bytes, splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    return splidar_stationary_multi(P0, 1, (int64_t)n_bins * ld, n_bins, ld, dt, t_r, &t_d, 1, tol, max_iter, pi,
                                    ws, ws_bytes, info, stream);
}

splidar_status splidar_stationary_multi(const void *P0, int32_t n_matrices, int64_t matrix_stride, int32_t n_bins,
                                        int64_t ld, splidar_dtype dt, double t_r, const double *t_d,
                                        int32_t n_vectors, double tol, int32_t max_iter, double *pi, void *ws,
                                        size_t ws_bytes, splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    return splidar_stationary_multi_host(P0, n_matrices, matrix_stride, n_bins, ld, dt, t_r, t_d, n_vectors, tol,
                                         max_iter, pi, nullptr, ws, ws_bytes, info, stream);
}

splidar_status splidar_stationary_multi_host(const void *P0, int32_t n_matrices, int64_t matrix_stride,
                                             int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r,
                                             const double *t_d, int32_t n_vectors, double tol, int32_t max_iter,
                                             double *pi, double *pi_host, void *ws, size_t ws_bytes,
                                             splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    splidar_status st;
    if (!t_d || n_matrices < 1 || n_vectors < 1 || n_vectors > kMaxVectors) return SPLIDAR_EINVAL;
    if ((st = check_matrix(P0, n_bins, ld, dt))) return st;
    if (n_matrices > 1 && (matrix_stride < (int64_t)n_bins * ld || matrix_stride % ld != 0)) return SPLIDAR_EINVAL;
    if (!(tol > 0.0) || !std::isfinite(tol) || max_iter < 1 || !pi) return SPLIDAR_EINVAL;
    std::vector<int> l((size_t)n_matrices * n_vectors);
    for (size_t i = 0; i < l.size(); ++i) {
        int32_t li;
        if ((st = splidar_shift(t_r, n_bins, t_d[i], &li))) return st;
        l[i] = li;
    }
    if ((st = check_ws(ws, ws_bytes, ws_layout(n_bins, n_matrices, n_vectors)))) return st;
    return cached_execute(P0, n_matrices, n_matrices > 1 ? matrix_stride : (int64_t)n_bins * ld, n_bins, ld, dt,
                          l.data(), n_vectors, tol, max_iter, pi, ws, ws_bytes, info, (cudaStream_t)stream, pi_host);
}

// ------------------------------------------------ row shards ---------------

splidar_status splidar_build_base_rows(const splidar_flux *flux, splidar_dtype dt, splidar_entry mode, void *P0_rows,
                                       int64_t ld, int32_t row0, int32_t n_rows, void *ws, size_t ws_bytes,
                                       void *stream) {
    SPL_NVTX_RANGE();
    splidar_status st = check_flux(flux);
    if (st) return st;
    if (mode != SPLIDAR_ENTRY_FACTORED && mode != SPLIDAR_ENTRY_EXP) return SPLIDAR_EINVAL;
    const int N = flux->n_bins;
    if (row0 < 0 || n_rows < 1 || row0 + n_rows > N) return SPLIDAR_EINVAL;
    if ((st = check_matrix(P0_rows, N, ld, dt))) return st;
    const WsLayout L = ws_layout(N, 1, 1);
    if ((st = check_ws(ws, ws_bytes, L))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    char *wsb = static_cast<char *>(ws);
    FluxDev d = to_dev(flux);
    SPL_CUDA(upload_async(wsb + L.flux, &d, sizeof(FluxDev), s));
    VecPtrs vp = vec_ptrs(wsb, L);
    SPL_CUDA(launch_flux_vectors(reinterpret_cast<const FluxDev *>(wsb + L.flux), 1, N, vp, N, s));
    SPL_CUDA(launch_build(vp, N, 1, N, dt, mode, P0_rows, ld, (int64_t)n_rows * ld, s, row0, n_rows));
    return SPLIDAR_OK;
}

splidar_status splidar_plan_create_rows(splidar_plan *plan, const void *P0_rows, int32_t row0, int32_t n_rows,
                                        int32_t n_bins, int64_t ld, splidar_dtype dt, double t_r, const double *t_d,
                                        int32_t n_vectors, double tol, int32_t max_iter, double *pi, double *ypart,
                                        void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan || !t_d || !ypart || n_vectors < 1 || n_vectors > kMaxVectors) return SPLIDAR_EINVAL;
    if (row0 < 0 || n_rows < 1 || n_bins < 2 || row0 + n_rows > n_bins) return SPLIDAR_EINVAL;
    if (((uintptr_t)ypart & 15u) != 0) return SPLIDAR_ENOSPACE;
    std::vector<int> l((size_t)n_vectors);
    for (int v = 0; v < n_vectors; ++v) {
        int32_t li;
        splidar_status st = splidar_shift(t_r, n_bins, t_d[v], &li);
        if (st) return st;
        l[(size_t)v] = li;
    }
    return plan_create_l(plan, P0_rows, 1, (int64_t)n_rows * ld, n_bins, ld, dt, l.data(), n_vectors, tol, max_iter,
                         pi, nullptr, ws, ws_bytes, (cudaStream_t)stream, row0, n_rows, ypart);
}

splidar_status splidar_plan_shard_init(splidar_plan p, void *stream) {
    SPL_NVTX_RANGE();
    if (!p || !p->shard) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    void *args[] = {&p->eager_args};
    SPL_CUDA(cudaLaunchKernel(p->k.init_fn, p->k.init_grid, p->k.init_block, args, 0, s));
    return SPLIDAR_OK;
}

splidar_status splidar_plan_shard_gemv(splidar_plan p, void *stream) {
    SPL_NVTX_RANGE();
    if (!p || !p->shard) return SPLIDAR_EINVAL;
    void *args[] = {&p->eager_args};
    SPL_CUDA(cudaLaunchKernel(p->k.step_fn, p->k.step_grid, p->k.step_block, args, p->k.step_smem,
                              (cudaStream_t)stream));
    return SPLIDAR_OK;
}

splidar_status splidar_plan_shard_check(splidar_plan p, int32_t *more, void *stream) {
    SPL_NVTX_RANGE();
    if (!p || !p->shard || !more) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    void *args[] = {&p->eager_args};
    const dim3 sgrid((unsigned)p->L.strips, (unsigned)(p->M * p->V));
    SPL_CUDA(cudaLaunchKernel(p->k.ssum_fn, sgrid, dim3(256), args, 0, s));
    SPL_CUDA(cudaLaunchKernel(p->k.check_fn, p->k.check_grid, p->k.check_block, args, 0, s));
    if (!p->host_flag) SPL_CUDA(cudaMallocHost(&p->host_flag, sizeof(unsigned)));
    SPL_CUDA(cudaMemcpyAsync(p->host_flag, p->eager_args.glob + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    SPL_CUDA(cudaStreamSynchronize(s));
    *more = *p->host_flag ? 1 : 0;
    return SPLIDAR_OK;
}

splidar_status splidar_plan_shard_finish(splidar_plan p, splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    if (!p || !p->shard) return SPLIDAR_EINVAL;
    void *fargs[] = {p->fin_args.data()};
    SPL_CUDA(cudaLaunchKernel(p->k.finish_fn, p->k.finish_grid, p->k.finish_block, fargs, 0, (cudaStream_t)stream));
    return splidar_plan_info(p, info, stream);
}

// ------------------------------------------------ f1 on a stored matrix (spectral_dense.cu) ---

static size_t sd_extra(int N, size_t *o_part, size_t *o_qsum, size_t *o_state, size_t *o_cnt) {
    size_t o = 0;
    *o_part = o; o = a256(o + sizeof(double) * (size_t)sd_chunks(N) * kSdDotsPerChunk);
    *o_qsum = o; o = a256(o + sizeof(double) * 2 * (size_t)sd_update_ctas(N));
    *o_state = o; o = a256(o + sizeof(SdState));
    *o_cnt = o; o = a256(o + sizeof(unsigned) * 4);
    return o;
}

size_t splidar_spectral_dense_workspace_bytes(int32_t n_bins) {
    if (n_bins < 2) return 0;
    size_t a, b, c, d;
    return ws_layout(n_bins, 1, 2).total + sd_extra(n_bins, &a, &b, &c, &d);
}

static cudaGraphExec_t sd_cache_find(const SdArgs &a, int dt) {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    const int dev = current_device();
    for (auto it = g_sd_cache.begin(); it != g_sd_cache.end(); ++it)
        if (it->dev == dev && it->dt == dt && sd_same(it->a, a)) {
            g_sd_cache.splice(g_sd_cache.begin(), g_sd_cache, it);
            return it->x;
        }
    return nullptr;
}

static void sd_cache_put(const SdArgs &a, int dt, cudaGraphExec_t x) {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    g_sd_cache.push_front(SdCached{current_device(), dt, a, x});
    while (g_sd_cache.size() > 8) {
        cudaGraphExecDestroy(g_sd_cache.back().x);
        g_sd_cache.pop_back();
    }
}

splidar_status splidar_second_eigenvalue_dense(const void *P0, int32_t n_bins, int64_t ld, splidar_dtype dt,
                                               double t_r, double t_d, const double *pi, double tol,
                                               int32_t max_iter, void *ws, size_t ws_bytes,
                                               splidar_spectral_info *info, void *stream) {
    SPL_NVTX_RANGE();
    splidar_status st;
    if (n_bins < 2 || !pi) return SPLIDAR_EINVAL;
    if ((st = check_matrix(P0, n_bins, ld, dt))) return st;
    if (!(tol > 0.0) || !std::isfinite(tol) || max_iter < 2) return SPLIDAR_EINVAL;
    int32_t l;
    if ((st = splidar_shift(t_r, n_bins, t_d, &l))) return st;
    const int N = n_bins;
    const WsLayout L = ws_layout(N, 1, 2);
    size_t o_part, o_qsum, o_state, o_cnt;
    const size_t extra = sd_extra(N, &o_part, &o_qsum, &o_state, &o_cnt);
    if (!ws || ((uintptr_t)ws & 255u) != 0 || ws_bytes < L.total + extra) return SPLIDAR_ENOSPACE;
    char *wsb = static_cast<char *>(ws);
    cudaStream_t s = (cudaStream_t)stream;

    SdArgs a;
    memset(&a, 0, sizeof(a));
    PowerArgs &p = a.p;
    p.P = P0;
    p.ld = ld;
    p.mstride = (int64_t)N * ld;
    p.N = N;
    p.rows = N;
    p.M = 1;
    p.V = L.V;
    p.strips = L.strips;
    p.chunks = L.chunks;
    p.xstride = L.xstride;
    p.y = reinterpret_cast<double *>(wsb + L.y);
    p.X = reinterpret_cast<double *>(wsb + L.X);
    p.part = reinterpret_cast<double *>(wsb + L.part);
    p.ssum = reinterpret_cast<double *>(wsb + L.ssum);
    p.l1part = reinterpret_cast<double *>(wsb + L.l1part);
    p.st = reinterpret_cast<SolveState *>(wsb + L.state);
    p.lsh = reinterpret_cast<const int *>(wsb + L.lsh);
    p.strip_cnt = reinterpret_cast<unsigned *>(wsb + L.strip_cnt);
    p.mv_cnt = reinterpret_cast<unsigned *>(wsb + L.mv_cnt);
    p.act = reinterpret_cast<int *>(wsb + L.act);
    p.glob = reinterpret_cast<unsigned *>(wsb + L.glob);
    p.tol = tol;
    p.max_iter = max_iter;
    a.l = l;
    a.pi = pi;
    a.part = reinterpret_cast<double *>(wsb + L.total + o_part);
    a.qsum = reinterpret_cast<double *>(wsb + L.total + o_qsum);
    a.nq = sd_update_ctas(N);
    a.sd = reinterpret_cast<SdState *>(wsb + L.total + o_state);
    a.cnt = reinterpret_cast<unsigned *>(wsb + L.total + o_cnt);
    a.tol = tol;
    a.max_iter = max_iter;

    SolverKernels k;
    if (solver_kernels(dt, 2, &k, p)) return SPLIDAR_EINVAL;
    SdKernels q;
    sd_kernels(&q, N);
    const char *e = getenv("SPLIDAR_EAGER");
    if (e && e[0] == '1') {   // host loop (profilers); control only, every step runs in the kernels
        SdArgs ea = a;
        ea.use_handle = 0;
        void *args[] = {&ea};
        void *pargs[] = {&ea.p};
        SPL_CUDA(cudaLaunchKernel(q.init_fn, dim3(1), q.block, args, 0, s));
        SdState h;
        for (int it = 0; it < max_iter; ++it) {
            SPL_CUDA(cudaLaunchKernel(k.step_fn, k.step_grid, k.step_block, pargs, k.step_smem, s));
            SPL_CUDA(cudaLaunchKernel(q.dots_fn, q.dots_grid, q.block, args, 0, s));
            SPL_CUDA(cudaLaunchKernel(q.update_fn, q.update_grid, q.block, args, 0, s));
            SPL_CUDA(cudaMemcpyAsync(&h, a.sd, sizeof(h), cudaMemcpyDeviceToHost, s));
            SPL_CUDA(cudaStreamSynchronize(s));
            if (h.done) break;
        }
    } else if (cudaGraphExec_t cx = sd_cache_find(a, dt)) {   // the same call before: replay its graph
        SPL_CUDA(cudaGraphLaunch(cx, s));
    } else {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t x = nullptr;
        cudaError_t err = cudaSuccess;
        do {
            if ((err = cudaGraphCreate(&g, 0))) break;
            cudaGraphConditionalHandle h;
            if ((err = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault))) break;
            a.use_handle = 1;
            a.handle = h;
            cudaKernelNodeParams kp;
            memset(&kp, 0, sizeof(kp));
            void *args[] = {&a};
            void *pargs[] = {&a.p};
            cudaGraphNode_t n_init, n_while, n_step, n_dots, n_upd;
            kp.func = q.init_fn;
            kp.gridDim = dim3(1);
            kp.blockDim = q.block;
            kp.kernelParams = args;
            if ((err = cudaGraphAddKernelNode(&n_init, g, nullptr, 0, &kp))) break;
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            if ((err = cudaGraphAddNode(&n_while, g, &n_init, 1, &cp))) break;
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            kp.func = k.step_fn;
            kp.gridDim = k.step_grid;
            kp.blockDim = k.step_block;
            kp.sharedMemBytes = k.step_smem;
            kp.kernelParams = pargs;
            if ((err = cudaGraphAddKernelNode(&n_step, body, nullptr, 0, &kp))) break;
            kp.func = q.dots_fn;
            kp.gridDim = q.dots_grid;
            kp.blockDim = q.block;
            kp.sharedMemBytes = 0;
            kp.kernelParams = args;
            if ((err = cudaGraphAddKernelNode(&n_dots, body, &n_step, 1, &kp))) break;
            kp.func = q.update_fn;
            kp.gridDim = q.update_grid;
            if ((err = cudaGraphAddKernelNode(&n_upd, body, &n_dots, 1, &kp))) break;
            if ((err = cudaGraphInstantiate(&x, g, 0))) break;
            err = cudaGraphLaunch(x, s);
        } while (0);
        if (g) cudaGraphDestroy(g);
        if (err == cudaSuccess) sd_cache_put(a, dt, x);   // kept for the next identical call
        else if (x) cudaGraphExecDestroy(x);
        SPL_CUDA(err);
    }
    SdState h;
    SPL_CUDA(cudaMemcpyAsync(&h, a.sd, sizeof(h), cudaMemcpyDeviceToHost, s));
    SPL_CUDA(cudaStreamSynchronize(s));
    if (info) {
        info->lambda2_re = h.mu_re;
        info->lambda2_im = h.mu_im;
        info->modulus = std::hypot(h.mu_re, h.mu_im);
        info->phase = std::atan2(h.mu_im, h.mu_re);
        info->gap = 1.0 - info->modulus;
        info->change = h.dmu;
        info->iters = h.iters;
        info->converged = h.converged;
    }
    return h.converged ? SPLIDAR_OK : SPLIDAR_ENOCONV;
}

// ---------------------------------------------------------------- sweep ----------------------

splidar_status splidar_sweep(const splidar_flux *shape, int32_t n_items, const double *S, const double *B,
                             const double *t_d, splidar_dtype dt, splidar_entry mode, double tol, int32_t max_iter,
                             double *pi, void *P0_store, int32_t n_store, int64_t ld, void *ws, size_t ws_bytes,
                             splidar_solve_info *info, void *stream) {
    SPL_NVTX_RANGE();
    if (!shape || n_items < 1 || !S || !B || !t_d || !pi) return SPLIDAR_EINVAL;
    if (!P0_store)   // matrix-free: the same items on the structured operator (f2), no N^2 storage
        return splidar_stationary_structured(shape, n_items, S, B, t_d, tol, max_iter, pi, ws, ws_bytes, info,
                                             stream);
    if (n_store < 1) return SPLIDAR_EINVAL;
    if (mode != SPLIDAR_ENTRY_FACTORED && mode != SPLIDAR_ENTRY_EXP) return SPLIDAR_EINVAL;
    const int N = shape->n_bins;
    splidar_status st;
    if ((st = check_matrix(P0_store, N, ld, dt))) return st;
    // validate every item and compute its shift
    std::vector<int> l((size_t)n_items);
    double sig_sum;
    if ((st = check_shape(shape, &sig_sum))) return st;
    for (int i = 0; i < n_items; ++i) {
        if ((st = check_item(sig_sum, S[i], B[i]))) return st;
        int32_t li;
        if ((st = splidar_shift(shape->t_r, N, t_d[i], &li))) return st;
        l[(size_t)i] = li;
    }
    // group items by (S, B) in order of first appearance
    std::vector<std::pair<double, double>> keys;
    std::vector<std::vector<int>> members;
    {
        std::map<std::pair<double, double>, int> idx;
        for (int i = 0; i < n_items; ++i) {
            auto k = std::make_pair(S[i], B[i]);
            auto it = idx.find(k);
            if (it == idx.end()) {
                idx[k] = (int)keys.size();
                keys.push_back(k);
                members.emplace_back();
                members.back().push_back(i);
            } else {
                members[(size_t)it->second].push_back(i);
            }
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *wsb = static_cast<char *>(ws);
    const int64_t mstride = (int64_t)N * ld;
    const int G = (int)keys.size();
    bool all_conv = true;
    std::vector<splidar_solve_info> pinfo;
    for (int g0 = 0; g0 < G; g0 += n_store) {
        const int Mc = (G - g0) < n_store ? (G - g0) : n_store;
        size_t maxv = 1;
        for (int g = g0; g < g0 + Mc; ++g) maxv = members[(size_t)g].size() > maxv ? members[(size_t)g].size() : maxv;
        const int passes = (int)((maxv + kMaxVectors - 1) / kMaxVectors);
        const int Vp = (int)(maxv < (size_t)kMaxVectors ? maxv : (size_t)kMaxVectors);
        const WsLayout L = ws_layout(N, Mc, Vp);
        if ((st = check_ws(ws, ws_bytes, L))) return st;
        std::vector<FluxDev> fl((size_t)Mc);
        for (int g = 0; g < Mc; ++g) fl[(size_t)g] = to_dev(shape, keys[(size_t)(g0 + g)].first, keys[(size_t)(g0 + g)].second);
        if ((st = vectors_and_build(fl.data(), Mc, N, dt, mode, P0_store, ld, mstride, wsb, L, s))) return st;
        std::vector<double> lam_tot((size_t)Mc * 8);
        SPL_CUDA(cudaMemcpyAsync(lam_tot.data(), vec_ptrs(wsb, L).scal, sizeof(double) * lam_tot.size(),
                                 cudaMemcpyDeviceToHost, s));
        for (int pass = 0; pass < passes; ++pass) {
            std::vector<int> lp((size_t)Mc * Vp, -1), op((size_t)Mc * Vp, -1);
            for (int g = 0; g < Mc; ++g) {
                const std::vector<int> &mem = members[(size_t)(g0 + g)];
                for (int v = 0; v < Vp; ++v) {
                    const size_t k = (size_t)pass * kMaxVectors + v;
                    if (k < mem.size()) {
                        lp[(size_t)g * Vp + v] = l[(size_t)mem[k]];
                        op[(size_t)g * Vp + v] = mem[k];
                    }
                }
            }
            splidar_plan p;
            st = plan_create_l(&p, P0_store, Mc, mstride, N, ld, dt, lp.data(), Vp, tol, max_iter, pi, op.data(), ws,
                               ws_bytes, s);
            if (st) return st;
            pinfo.assign((size_t)Mc * Vp, splidar_solve_info());
            st = splidar_plan_execute(p, pinfo.data(), s);
            splidar_plan_destroy(p);
            if (st != SPLIDAR_OK && st != SPLIDAR_ENOCONV) return st;
            for (int g = 0; g < Mc; ++g)
                for (int v = 0; v < Vp; ++v) {
                    const int item = op[(size_t)g * Vp + v];
                    if (item < 0) continue;
                    splidar_solve_info o = pinfo[(size_t)g * Vp + v];
                    o.lambda_total = lam_tot[(size_t)g * 8];
                    if (lam_tot[(size_t)g * 8 + 2] != 0.0) return SPLIDAR_EZEROROW;
                    all_conv = all_conv && o.converged;
                    if (info) info[item] = o;
                }
        }
    }
    return all_conv ? SPLIDAR_OK : SPLIDAR_ENOCONV;
}

}  // extern "C"

// ---------------------------------------------------------------- structured operator (f1, f2) --
//
// Workspace: FluxDev[M] | the step-1 vectors of M profiles (as ws_layout) | prof[I] | lsh[I] |
// SolveState[I] | SpecOut[I] | nsteps[I] | nmax.

namespace spl {
struct SLayout {
    int N, M, I;
    size_t flux, vec, prof, lsh, st, spec, nsteps, nmax, total;
};
static SLayout struct_layout(int N, int M, int I) {
    SLayout L;
    L.N = N;
    L.M = M;
    L.I = I;
    size_t o = 0;
    L.flux = o; o = a256(o + sizeof(FluxDev) * (size_t)M);
    const size_t ntile = ((size_t)N + 1 + kScanTile - 1) / kScanTile;
    L.vec = o; o = a256(o + sizeof(double) * ((size_t)M * N * 5 + (size_t)M * 8 + 5 * (size_t)M * ntile));
    L.prof = o; o = a256(o + sizeof(int) * (size_t)I);
    L.lsh = o; o = a256(o + sizeof(int) * (size_t)I);
    L.st = o; o = a256(o + sizeof(SolveState) * (size_t)I);
    L.spec = o; o = a256(o + sizeof(SpecOut) * (size_t)I);
    L.nsteps = o; o = a256(o + sizeof(int) * (size_t)I);
    L.nmax = o; o = a256(o + sizeof(int) * 4);
    L.total = o;
    return L;
}
static VecPtrs svec_ptrs(char *ws, const SLayout &L) {
    WsLayout W;
    memset(&W, 0, sizeof(W));
    W.N = L.N;
    W.M = L.M;
    W.vec = L.vec;
    return vec_ptrs(ws, W);
}
}  // namespace spl

// Validates items (shape x S[m], B[m], t_d[m]), groups them by (S, B), enqueues the step-1 vectors of
// every distinct profile and uploads the per-item profile index and shift (n_items_ws: items the
// workspace must hold, >= n_items). Fills the kernel arguments with pointers into ws.
struct Prep {
    StructArgs a;
    SLayout L;
    const FluxDev *flux_dev;
    VecPtrs vp;
    std::vector<int> prof, l;
    std::vector<double> scal;   // [M][8] host copy (after read_scal)
};

static splidar_status struct_prepare(const splidar_flux *shape, int n_items, const double *S, const double *B,
                                     const double *t_d, int n_items_ws, void *ws, size_t ws_bytes, cudaStream_t s,
                                     Prep *p) {
    if (!shape || n_items < 1 || !S || !B || !t_d) return SPLIDAR_EINVAL;
    const int N = shape->n_bins;
    int C, T;
    if (N < 2 || struct_shape(N, &C, &T)) return SPLIDAR_EINVAL;
    splidar_status st;
    p->l.assign((size_t)n_items, 0);
    p->prof.assign((size_t)n_items, 0);
    std::vector<FluxDev> fl;
    std::map<std::pair<double, double>, int> idx;
    double sig_sum;
    if ((st = check_shape(shape, &sig_sum))) return st;
    for (int i = 0; i < n_items; ++i) {
        if ((st = check_item(sig_sum, S[i], B[i]))) return st;
        int32_t li;
        if ((st = splidar_shift(shape->t_r, N, t_d[i], &li))) return st;
        p->l[(size_t)i] = li;
        const auto key = std::make_pair(S[i], B[i]);
        if (i > 0 && S[i] == S[i - 1] && B[i] == B[i - 1]) {        // runs of equal (S, B): no lookup
            p->prof[(size_t)i] = p->prof[(size_t)i - 1];
            continue;
        }
        auto it = idx.find(key);
        if (it == idx.end()) {
            idx.emplace(key, (int)fl.size());
            p->prof[(size_t)i] = (int)fl.size();
            fl.push_back(to_dev(shape, S[i], B[i]));
        } else {
            p->prof[(size_t)i] = it->second;
        }
    }
    const int M = (int)fl.size();
    if (M > 65535) return SPLIDAR_EINVAL;
    p->L = struct_layout(N, M, n_items_ws > n_items ? n_items_ws : n_items);
    const SLayout &L = p->L;
    if (!ws || ((uintptr_t)ws & 255u) != 0 || ws_bytes < L.total) return SPLIDAR_ENOSPACE;
    char *wsb = static_cast<char *>(ws);
    SPL_CUDA(cudaMemcpyAsync(wsb + L.flux, fl.data(), sizeof(FluxDev) * (size_t)M, cudaMemcpyHostToDevice, s));
    VecPtrs vp = svec_ptrs(wsb, L);
    p->flux_dev = reinterpret_cast<const FluxDev *>(wsb + L.flux);
    p->vp = vp;
    SPL_CUDA(cudaMemcpyAsync(wsb + L.prof, p->prof.data(), sizeof(int) * (size_t)n_items, cudaMemcpyHostToDevice, s));
    SPL_CUDA(cudaMemcpyAsync(wsb + L.lsh, p->l.data(), sizeof(int) * (size_t)n_items, cudaMemcpyHostToDevice, s));
    StructArgs *a = &p->a;
    memset(a, 0, sizeof(*a));
    a->N = N;
    a->C = C;
    a->threads = T;
    a->vstride = N;
    a->w = vp.w;
    a->invD = vp.invD;
    a->scal = vp.scal;
    a->prof = reinterpret_cast<const int *>(wsb + L.prof);
    a->lsh = reinterpret_cast<const int *>(wsb + L.lsh);
    a->st = reinterpret_cast<SolveState *>(wsb + L.st);
    a->spec = reinterpret_cast<SpecOut *>(wsb + L.spec);
    a->nsteps = reinterpret_cast<int *>(wsb + L.nsteps);
    a->nmax = reinterpret_cast<int *>(wsb + L.nmax);
    return SPLIDAR_OK;
}

// After the kernels: the per-profile scalars (Lambda, e^{-Lambda}, bad-row flag) to the host; syncs s.
static splidar_status read_scal(Prep *p, cudaStream_t s) {
    p->scal.assign((size_t)p->L.M * 8, 0.0);
    SPL_CUDA(cudaMemcpyAsync(p->scal.data(), p->a.scal, sizeof(double) * p->scal.size(), cudaMemcpyDeviceToHost, s));
    SPL_CUDA(cudaStreamSynchronize(s));
    for (int m = 0; m < p->L.M; ++m)
        if (p->scal[(size_t)m * 8 + 2] != 0.0) return SPLIDAR_EZEROROW;
    return SPLIDAR_OK;
}

// Structured plans: items validated and uploaded once; each launch recomputes the step-1 vectors
// and runs the kernel (async); CUDA events around the kernel give its device time.
// The first launch runs eagerly (it also sets the kernels' attributes and caches the cluster
// residency query); a second launch captures the same sequence once into a CUDA graph, with the
// events as external event-record nodes, and it and later launches replay it (one cudaGraphLaunch instead of up to 6 kernel
// launches and 2 event records: the host gaps between them were ~1/4 of c5's structured step).
// SPLIDAR_SPLAN_GRAPH=0 keeps every launch eager.
struct splidar_splan_s {
    Prep p;
    int kind = 0;
    int n_items = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool graph_tried = false;
    long launches = 0;
    cudaGraphExec_t gexec = nullptr;
};

static splidar_status splan_launch_impl(splidar_splan_s *pl, cudaStream_t s, bool capture = false) {
    const Prep &p = pl->p;
    const unsigned fl = capture ? cudaEventRecordExternal : cudaEventRecordDefault;
    SPL_CUDA(launch_flux_vectors(p.flux_dev, p.L.M, p.a.N, p.vp, p.a.N, s));
    SPL_CUDA(cudaEventRecordWithFlags(pl->ev0, s, fl));
    SPL_CUDA(launch_struct(pl->kind == 0 ? kStructSolve : kStructLambda2, p.a, pl->n_items, s));
    SPL_CUDA(cudaEventRecordWithFlags(pl->ev1, s, fl));
    return SPLIDAR_OK;
}

// Capture the launch sequence on a private stream (nothing executes) and instantiate it.
static cudaError_t splan_capture(splidar_splan_s *pl) {
    cudaStream_t cs = nullptr;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        const splidar_status st = splan_launch_impl(pl, cs, true);
        const cudaError_t e2 = cudaStreamEndCapture(cs, &g);
        e = st != SPLIDAR_OK ? cudaErrorUnknown : e2;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&pl->gexec, g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess) pl->gexec = nullptr;
    return e;
}

extern "C" {

size_t splidar_structured_workspace_bytes(int32_t n_bins, int32_t n_profiles, int32_t n_items) {
    int C, T;
    if (n_bins < 2 || n_profiles < 1 || n_items < 1 || struct_shape(n_bins, &C, &T)) return 0;
    return struct_layout(n_bins, n_profiles, n_items).total;
}

void splidar_splan_destroy(splidar_splan plan) {
    if (!plan) return;
    if (plan->gexec) cudaGraphExecDestroy(plan->gexec);
    if (plan->ev0) cudaEventDestroy(plan->ev0);
    if (plan->ev1) cudaEventDestroy(plan->ev1);
    delete plan;
}

splidar_status splidar_splan_create(splidar_splan *plan, int32_t kind, const splidar_flux *shape, int32_t n_items,
                                    const double *S, const double *B, const double *t_d, double tol,
                                    int32_t max_iter, double *pi, void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan) return SPLIDAR_EINVAL;
    *plan = nullptr;
    if ((kind != SPLIDAR_SPLAN_SOLVE && kind != SPLIDAR_SPLAN_LAMBDA2) || !pi || !(tol > 0.0) ||
        !std::isfinite(tol) || max_iter < 1)
        return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    splidar_splan_s *pl = new splidar_splan_s();
    splidar_status st = struct_prepare(shape, n_items, S, B, t_d, n_items, ws, ws_bytes, s, &pl->p);
    if (st) { delete pl; return st; }
    pl->kind = kind;
    pl->n_items = n_items;
    pl->p.a.tol = tol;
    pl->p.a.max_iter = max_iter;
    pl->p.a.pi = pi;
    cudaError_t e = cudaEventCreate(&pl->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&pl->ev1);
    if (e != cudaSuccess) { splidar_splan_destroy(pl); return cuda_status(e); }
    *plan = pl;
    return SPLIDAR_OK;
}

splidar_status splidar_splan_launch(splidar_splan plan, void *stream) {
    SPL_NVTX_RANGE();
    if (!plan) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (!plan->gexec && plan->launches == 1 && !plan->graph_tried) {   // a reused plan: capture it once
        plan->graph_tried = true;
        const char *e = getenv("SPLIDAR_SPLAN_GRAPH");
        if (!(e && e[0] == '0') && splan_capture(plan) != cudaSuccess)
            (void)cudaGetLastError();   // stay eager: the graph is an optimisation only
    }
    ++plan->launches;
    if (plan->gexec) return cuda_status(cudaGraphLaunch(plan->gexec, s));
    return splan_launch_impl(plan, s);
}

splidar_status splidar_splan_info(splidar_splan plan, splidar_solve_info *solve_info,
                                  splidar_spectral_info *spectral_info, float *kernel_ms, void *stream) {
    if (!plan) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Prep &p = plan->p;
    const int n = plan->n_items;
    std::vector<SolveState> hs;
    std::vector<SpecOut> hp;
    if (plan->kind == SPLIDAR_SPLAN_SOLVE) {
        hs.resize((size_t)n);
        SPL_CUDA(cudaMemcpyAsync(hs.data(), p.a.st, sizeof(SolveState) * hs.size(), cudaMemcpyDeviceToHost, s));
    } else {
        hp.resize((size_t)n);
        SPL_CUDA(cudaMemcpyAsync(hp.data(), p.a.spec, sizeof(SpecOut) * hp.size(), cudaMemcpyDeviceToHost, s));
    }
    splidar_status st = read_scal(&p, s);
    if (st) return st;
    if (kernel_ms) SPL_CUDA(cudaEventElapsedTime(kernel_ms, plan->ev0, plan->ev1));
    bool all = true;
    for (int i = 0; i < n; ++i) {
        if (plan->kind == SPLIDAR_SPLAN_SOLVE) {
            const SolveState &h = hs[(size_t)i];
            all = all && h.converged;
            if (solve_info) {
                splidar_solve_info &o = solve_info[i];
                o.iters = h.iters;
                o.converged = h.converged;
                o.shift_l = h.l;
                o.reserved = 0;
                o.l1_change = h.change;
                o.lambda_total = p.scal[(size_t)p.prof[(size_t)i] * 8];
            }
        } else {
            const SpecOut &h = hp[(size_t)i];
            all = all && h.converged;
            if (spectral_info) {
                splidar_spectral_info &o = spectral_info[i];
                o.lambda2_re = h.re;
                o.lambda2_im = h.im;
                o.modulus = std::hypot(h.re, h.im);
                o.phase = std::atan2(h.im, h.re);
                o.gap = 1.0 - o.modulus;
                o.change = h.change;
                o.iters = h.iters;
                o.converged = h.converged;
            }
        }
    }
    return all ? SPLIDAR_OK : SPLIDAR_ENOCONV;
}

splidar_status splidar_stationary_structured(const splidar_flux *shape, int32_t n_items, const double *S,
                                             const double *B, const double *t_d, double tol, int32_t max_iter,
                                             double *pi, void *ws, size_t ws_bytes, splidar_solve_info *info,
                                             void *stream) {
    SPL_NVTX_RANGE();
    splidar_splan pl;
    splidar_status st = splidar_splan_create(&pl, SPLIDAR_SPLAN_SOLVE, shape, n_items, S, B, t_d, tol, max_iter,
                                             pi, ws, ws_bytes, stream);
    if (st) return st;
    st = splidar_splan_launch(pl, stream);
    if (!st) st = splidar_splan_info(pl, info, nullptr, nullptr, stream);
    splidar_splan_destroy(pl);
    return st;
}

splidar_status splidar_second_eigenvalue(const splidar_flux *shape, int32_t n_items, const double *S,
                                         const double *B, const double *t_d, const double *pi, double tol,
                                         int32_t max_iter, void *ws, size_t ws_bytes, splidar_spectral_info *info,
                                         void *stream) {
    SPL_NVTX_RANGE();
    splidar_splan pl;
    splidar_status st = splidar_splan_create(&pl, SPLIDAR_SPLAN_LAMBDA2, shape, n_items, S, B, t_d, tol,
                                             max_iter, const_cast<double *>(pi), ws, ws_bytes, stream);
    if (st) return st;
    st = splidar_splan_launch(pl, stream);
    if (!st) st = splidar_splan_info(pl, nullptr, info, nullptr, stream);
    splidar_splan_destroy(pl);
    return st;
}

splidar_status splidar_mixing_steps(const splidar_flux *flux, double t_d, const double *pi, double eps,
                                    int32_t max_steps, int32_t *steps_per_start, int32_t *mixing_steps, void *ws,
                                    size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!flux || !pi || !mixing_steps || !(eps > 0.0) || !std::isfinite(eps) || max_steps < 1) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const double one = 1.0, bg = flux->background;
    const int N = flux->n_bins;
    Prep p;
    splidar_status st = struct_prepare(flux, 1, &one, &bg, &t_d, N, ws, ws_bytes, s, &p);
    if (st) return st;
    SPL_CUDA(launch_flux_vectors(p.flux_dev, p.L.M, N, p.vp, N, s));
    p.a.pi = const_cast<double *>(pi);
    p.a.eps = eps;
    p.a.max_iter = max_steps;
    p.a.start_bin0 = 0;
    SPL_CUDA(cudaMemsetAsync(p.a.nmax, 0, sizeof(int), s));
    SPL_CUDA(launch_struct(kStructMixing, p.a, N, s));
    if (steps_per_start)
        SPL_CUDA(cudaMemcpyAsync(steps_per_start, p.a.nsteps, sizeof(int) * (size_t)N, cudaMemcpyDeviceToDevice, s));
    int hmax = 0;
    SPL_CUDA(cudaMemcpyAsync(&hmax, p.a.nmax, sizeof(int), cudaMemcpyDeviceToHost, s));
    if ((st = read_scal(&p, s))) return st;
    if (hmax == 0x7fffffff) {
        *mixing_steps = -1;
        return SPLIDAR_ENOCONV;
    }
    *mixing_steps = hmax;
    return SPLIDAR_OK;
}

splidar_status splidar_bin_trajectory(const splidar_flux *flux, double t_d, const double *start, int32_t bin,
                                      int32_t steps, double *traj, double *final_vec, void *ws, size_t ws_bytes,
                                      void *stream) {
    SPL_NVTX_RANGE();
    if (!flux || !start || !traj || steps < 0 || bin < 0 || bin >= flux->n_bins) return SPLIDAR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const double one = 1.0, bg = flux->background;
    Prep p;
    splidar_status st = struct_prepare(flux, 1, &one, &bg, &t_d, 1, ws, ws_bytes, s, &p);
    if (st) return st;
    SPL_CUDA(launch_flux_vectors(p.flux_dev, p.L.M, flux->n_bins, p.vp, flux->n_bins, s));
    p.a.start = start;
    p.a.bin = bin;
    p.a.max_iter = steps;
    p.a.traj = traj;
    p.a.out = final_vec;
    SPL_CUDA(launch_struct(kStructTraj, p.a, 1, s));
    return read_scal(&p, s);
}

}  // extern "C"

// ---------------------------------------------------------------- Monte Carlo (f3) -------------
static size_t mc_layout(int M, int I, size_t *o_prof, size_t *o_td) {
    size_t o = a256(sizeof(FluxDev) * (size_t)M);
    *o_prof = o;
    o = a256(o + sizeof(int) * (size_t)I);
    *o_td = o;
    return a256(o + sizeof(double) * (size_t)I);
}

extern "C" {

size_t splidar_mc_workspace_bytes(int32_t n_profiles, int32_t n_items) {
    if (n_profiles < 1 || n_items < 1) return 0;
    size_t a, b;
    return mc_layout(n_profiles, n_items, &a, &b);
}

splidar_status splidar_monte_carlo(const splidar_flux *shape, int32_t n_items, const double *S, const double *B,
                                   const double *t_d, uint64_t seed, int32_t n_runs, int32_t n_split, int64_t n_burn,
                                   int64_t n_regs, int64_t n_cycles, int32_t n_hist, uint64_t *hist, int32_t n_record,
                                   int64_t *q_rec, double *t_rec, void *ws, size_t ws_bytes, void *stream) {
    SPL_NVTX_RANGE();
    if (!shape || n_items < 1 || n_items > 65535 || !S || !B || !t_d || !hist) return SPLIDAR_EINVAL;
    if (n_runs < 1 || n_split < 1 || (int64_t)n_runs * n_split > (1 << 30) || n_hist < 1 || n_burn < 0 ||
        n_record < 0 || (n_regs < 1 && n_cycles < 1))
        return SPLIDAR_EINVAL;
    if ((n_cycles > 0 && n_cycles % n_split) || (n_cycles < 1 && n_regs % n_split)) return SPLIDAR_EINVAL;
    if (n_record > 0 && (!q_rec || !t_rec)) return SPLIDAR_EINVAL;
    splidar_status st;
    std::vector<FluxDev> fl;
    std::vector<int> prof((size_t)n_items);
    std::map<std::pair<double, double>, int> idx;
    double sig_sum;
    if ((st = check_shape(shape, &sig_sum))) return st;
    for (int i = 0; i < n_items; ++i) {
        if ((st = check_item(sig_sum, S[i], B[i]))) return st;
        if (!std::isfinite(t_d[i]) || t_d[i] < 0.0) return SPLIDAR_EINVAL;
        const auto key = std::make_pair(S[i], B[i]);
        auto it = idx.find(key);
        if (it == idx.end()) {
            idx.emplace(key, (int)fl.size());
            prof[(size_t)i] = (int)fl.size();
            fl.push_back(to_dev(shape, S[i], B[i]));
        } else {
            prof[(size_t)i] = it->second;
        }
    }
    size_t o_prof, o_td;
    const size_t need = mc_layout((int)fl.size(), n_items, &o_prof, &o_td);
    if (!ws || ((uintptr_t)ws & 255u) != 0 || ws_bytes < need) return SPLIDAR_ENOSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    char *wsb = static_cast<char *>(ws);
    SPL_CUDA(cudaMemcpyAsync(wsb, fl.data(), sizeof(FluxDev) * fl.size(), cudaMemcpyHostToDevice, s));
    SPL_CUDA(cudaMemcpyAsync(wsb + o_prof, prof.data(), sizeof(int) * prof.size(), cudaMemcpyHostToDevice, s));
    SPL_CUDA(cudaMemcpyAsync(wsb + o_td, t_d, sizeof(double) * (size_t)n_items, cudaMemcpyHostToDevice, s));
    SPL_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint64_t) * (size_t)n_items * n_runs * n_hist, s));
    McArgs a;
    memset(&a, 0, sizeof(a));
    a.flux = reinterpret_cast<const FluxDev *>(wsb);
    a.prof = reinterpret_cast<const int *>(wsb + o_prof);
    a.td = reinterpret_cast<const double *>(wsb + o_td);
    a.n_items = n_items;
    a.n_runs = n_runs;
    a.n_split = n_split;
    a.n_hist = n_hist;
    a.n_record = n_record;
    a.n_burn = n_burn;
    a.n_regs = n_cycles > 0 ? 0 : n_regs / n_split;
    a.n_cycles = n_cycles > 0 ? n_cycles / n_split : 0;
    a.seed = seed;
    a.hist = reinterpret_cast<unsigned long long *>(hist);
    a.q_rec = reinterpret_cast<long long *>(q_rec);
    a.t_rec = t_rec;
    SPL_CUDA(launch_mc(a, s));
    SPL_CUDA(cudaStreamSynchronize(s));
    return SPLIDAR_OK;
}

}  // extern "C"
