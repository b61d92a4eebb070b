// Step 1 of the path (K1-K3): discretised flux, prefix sums, row normalisers.
// Everything fp64; every sum is tree-shaped (thread-local run of 4, warp __shfl_up_sync scan,
// fixed-order combination of the 8 warp totals, then a scan of the 1024-element tile totals),
// never a long sequential chain (a sequential fp64 cumsum drifts ~1e-12 at N = 32768).
//
//   masses   m_0 = int_0^{s_0} lambda, m_j = int_{s_{j-1}}^{s_j} lambda (1 <= j < N),
//            m_N = int_{s_{N-1}}^{t_r} lambda, each exact (erfc differences, Eq. 1)
//   F_j      = sum_{i <= j} m_i = F(s_j)  (Thm 1: F(t) := int_0^t lambda)
//   Lambda   = sum_{i <= N} m_i = F(t_r)  (reading R5)
//   lambda_j = lambda(s_j)
//   w_j      = lambda_j e^{-F_j}
//   L_r      = sum_{j < r} w_j, U_r = sum_{j >= r} w_j
//   D_r      = U_r + e^{-Lambda} L_r = e^{-F_r} sum_j lambda_j exp(F_r - F_j - Lambda [r > j])
//            (the row sum of (1 lambda^T) . exp.(-Lambda L - D), §3.4, over e^{F_r})
//   invD_r   = 1 / D_r, invZ_r = e^{-F_r} / D_r (normalisation)
//
// N < 8192: one launch, one 1024-thread CTA per profile (k_vec_small, the same three scans in one CTA).
// Larger N: five grid-wide launches per batch of profiles (grid = tiles x profiles):
//   A  masses + lambda, tile-local inclusive scan of the masses, tile totals
//   B  exclusive scan of the tile totals (one CTA per profile) -> tile offsets, Lambda
//   C  F = local + offset, w, tile-local exclusive prefix / inclusive suffix of w, tile totals of w
//   D  exclusive prefix and suffix of the w tile totals (one CTA per profile)
//   E  L, U, D, 1/D, 1/Z
// tiles[5][M][ntile]: 0 mass tile totals, 1 mass tile offsets, 2 w tile totals, 3 w tile
// prefix offsets, 4 w tile suffix offsets.
#include <mutex>

#include <cstring>

#include "common.cuh"
#include "ptx.cuh"

namespace spl {
namespace {

constexpr int kT = 1024;                // threads per tile CTA (one element each: the erfc / exp chains of
                                        // a tile run in parallel; 256 x 4 left 8 warps per tile, k_vec_a 19 us at N = 32768)
constexpr int kE = kScanTile / kT;      // consecutive elements per thread

__device__ __forceinline__ double bin_centre(const FluxDev &f, int j) {
    return ((double)j + 0.5) * (f.t_r / (double)f.n);
}

// Phi(zh) - Phi(zl) for zl <= zh without cancellation: both tails use erfc of the same sign,
// the straddling case uses erf of both halves (all terms positive).
__device__ __forceinline__ double phi_diff(double zl, double zh) {
    const double r2 = 0.70710678118654752440;  // 1/sqrt(2)
    if (zl >= 0.0) return 0.5 * (erfc(zl * r2) - erfc(zh * r2));
    if (zh <= 0.0) return 0.5 * (erfc(-zh * r2) - erfc(-zl * r2));
    return 0.5 * (erf(zh * r2) + erf(-zl * r2));
}

// int_lo^hi lambda(t) dt for 0 <= lo <= hi <= t_r (Eq. 1; S = alpha E, lambda_b = B/t_r). The
// reference form of the masses k_vec_a / k_vec_small compute with shared bin-edge erfc evaluations.
[[maybe_unused]] __device__ double flux_mass(const FluxDev &f, double lo, double hi) {
    double v = f.B * ((hi - lo) / f.t_r);
    for (int k = 0; k < f.k; ++k) {
        const double is = 1.0 / f.sigma[k];
        v += f.S[k] * phi_diff((lo - f.tau[k]) * is, (hi - f.tau[k]) * is);
    }
    return v;
}

// lambda(t) (Eq. 1).
__device__ double flux_rate(const FluxDev &f, double t) {
    const double inv_sqrt_2pi = 0.39894228040143267794;
    double v = f.B / f.t_r;
    for (int k = 0; k < f.k; ++k) {
        const double z = (t - f.tau[k]) / f.sigma[k];
        v += f.S[k] * inv_sqrt_2pi / f.sigma[k] * exp(-0.5 * z * z);
    }
    return v;
}

// Inclusive scan of a 1024-element tile held as kE consecutive values per thread (kT threads);
// returns the tile total. warp_tot: kT / 32 doubles of shared memory.
__device__ double tile_scan(double (&v)[kE], double *warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 1; i < kE; ++i) v[i] += v[i - 1];
    double x = v[kE - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    // exclusive prefix of the thread totals by a shuffle, never as (inclusive - own): with values
    // spanning hundreds of decades (w = lambda e^{-F} at large Lambda) the subtraction would leave
    // an error of ulp(own) on a much smaller prefix
    double xe = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) xe = 0.0;
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    double wex = 0.0, total = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < kT / 32; ++w2) {       // the warp totals: a short fixed-order sum
        const double wt = warp_tot[w2];
        if (w2 < warp) wex += wt;
        total += wt;
    }
    const double ex = xe + wex;
#pragma unroll
    for (int i = 0; i < kE; ++i) v[i] += ex;
    __syncthreads();
    return total;
}

// Exclusive prefix and suffix scans of n <= 4096 tile totals by one 1024-thread CTA, fixed tree
// order: pre[i] = sum_{k<i} in[k], suf[i] = sum_{k>i} in[k]; returns the total (pre or suf may
// be null).
__device__ double totals_scan(const double *in, int n, double *pre, double *suf) {
    __shared__ double wt_f[65], wt_b[65];
    constexpr int EPT = 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double f[EPT], bk[EPT];
    const int e0 = threadIdx.x * EPT;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        f[i] = e0 + i < n ? in[e0 + i] : 0.0;
        bk[i] = e0 + i < n ? in[n - 1 - (e0 + i)] : 0.0;   // reversed sequence for the suffix
    }
    // thread-local EXCLUSIVE running sums (no subtraction anywhere: see tile_scan)
    double fe[EPT], be[EPT];
    fe[0] = 0.0;
    be[0] = 0.0;
#pragma unroll
    for (int i = 1; i < EPT; ++i) { fe[i] = fe[i - 1] + f[i - 1]; be[i] = be[i - 1] + bk[i - 1]; }
    double xf = fe[EPT - 1] + f[EPT - 1], xb = be[EPT - 1] + bk[EPT - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double yf = __shfl_up_sync(0xffffffffu, xf, o);
        const double yb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= o) { xf += yf; xb += yb; }
    }
    double xfe = __shfl_up_sync(0xffffffffu, xf, 1), xbe = __shfl_up_sync(0xffffffffu, xb, 1);
    if (lane == 0) { xfe = 0.0; xbe = 0.0; }
    if (lane == 31) { wt_f[warp] = xf; wt_b[warp] = xb; }
    __syncthreads();
    if (warp == 0) {
        double sf = wt_f[lane], sb = wt_b[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double yf = __shfl_up_sync(0xffffffffu, sf, o);
            const double yb = __shfl_up_sync(0xffffffffu, sb, o);
            if (lane >= o) { sf += yf; sb += yb; }
        }
        double sfe = __shfl_up_sync(0xffffffffu, sf, 1), sbe = __shfl_up_sync(0xffffffffu, sb, 1);
        if (lane == 0) { sfe = 0.0; sbe = 0.0; }
        wt_f[32 + lane] = sfe;                  // exclusive prefix of the warp totals
        wt_b[32 + lane] = sbe;
        if (lane == 31) { wt_f[64] = sf; wt_b[64] = sb; }
    }
    __syncthreads();
    const double exf = xfe + wt_f[32 + warp];
    const double exb = xbe + wt_b[32 + warp];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = e0 + i;
        if (e < n) {
            if (pre) pre[e] = exf + fe[i];                       // exclusive prefix
            if (suf) suf[n - 1 - e] = exb + be[i];               // exclusive suffix
        }
    }
    return wt_f[64];
}

__device__ __forceinline__ double *tile_row(const VecPtrs &b, int M, int which, int m) {
    return b.tiles + ((size_t)which * M + m) * b.ntile;
}

// (A) masses + lambda; tile-local inclusive scan of the masses -> F (local), tile total.
__global__ void __launch_bounds__(kT) k_vec_a(const FluxDev *__restrict__ fluxes, int N, int M, VecPtrs b,
                                              int64_t vstride) {
    static_assert(kE == 1, "one element per thread: the edge sharing below assumes it");
    __shared__ double warp_tot[kT / 32];
    __shared__ double eh[kT];                  // erfc(|z| / sqrt 2) of each thread's upper bin edge
    const int m = blockIdx.y, tile = blockIdx.x;
    const FluxDev &f = fluxes[m];
    const int e0 = tile * kScanTile + threadIdx.x * kE;
    // flux_mass(lo, hi) with each bin edge's erfc evaluated once and shared by the two masses it
    // bounds (as k_vec_small; the tile's first mass evaluates its lower edge itself): bitwise the
    // same masses with half the erfc evaluations
    double v[kE];
    const int e = e0;
    const double lo = e == 0 ? 0.0 : bin_centre(f, e - 1);
    const double hi = e == N ? f.t_r : bin_centre(f, e);
    v[0] = e <= N ? f.B * ((hi - lo) / f.t_r) : 0.0;
    const double r2 = 0.70710678118654752440;  // 1/sqrt(2)
    for (int k = 0; k < f.k; ++k) {
        const double is = 1.0 / f.sigma[k];
        const double zl = (lo - f.tau[k]) * is, zh = (hi - f.tau[k]) * is;
        __syncthreads();                         // eh[] of the previous pulse consumed
        eh[threadIdx.x] = e <= N ? erfc((zh >= 0.0 ? zh : -zh) * r2) : 0.0;
        __syncthreads();
        if (e <= N) {
            const double el = threadIdx.x > 0 ? eh[threadIdx.x - 1] : erfc((zl >= 0.0 ? zl : -zl) * r2);
            double ph;
            if (zl >= 0.0) ph = 0.5 * (el - eh[threadIdx.x]);
            else if (zh <= 0.0) ph = 0.5 * (eh[threadIdx.x] - el);
            else ph = 0.5 * (erf(zh * r2) + erf(-zl * r2));
            v[0] += f.S[k] * ph;
        }
    }
    const double tot = tile_scan(v, warp_tot);
    double *F = b.F + m * vstride, *lam = b.lam + m * vstride;
#pragma unroll
    for (int i = 0; i < kE; ++i) {
        const int e = e0 + i;
        if (e < N) {
            F[e] = v[i];
            lam[e] = flux_rate(f, bin_centre(f, e));
        }
    }
    if (threadIdx.x == 0) tile_row(b, M, 0, m)[tile] = tot;
}

// (B) exclusive scan of the mass tile totals -> tile offsets; Lambda = the total; e^{-Lambda}.
__global__ void __launch_bounds__(1024) k_vec_b(int M, int nt, VecPtrs b) {
    const int m = blockIdx.x;
    const double Lam = totals_scan(tile_row(b, M, 0, m), nt, tile_row(b, M, 1, m), nullptr);
    if (threadIdx.x == 0) {
        b.scal[m * 8 + 0] = Lam;
        b.scal[m * 8 + 1] = exp(-Lam);
        b.scal[m * 8 + 2] = 0.0;
    }
}

// (C) F = local + offset; w = lambda e^{-F}; tile-local exclusive prefix of w (into invD, temp)
// and inclusive suffix of w (into invZ, temp); tile total of w.
__global__ void __launch_bounds__(kT) k_vec_c(int N, int M, VecPtrs b, int64_t vstride) {
    __shared__ double warp_tot[kT / 32];
    __shared__ double rev[kScanTile];
    const int m = blockIdx.y, tile = blockIdx.x;
    const double off = tile_row(b, M, 1, m)[tile];
    double *F = b.F + m * vstride, *lam = b.lam + m * vstride, *w = b.w + m * vstride;
    double *Lt = b.invD + m * vstride, *Ut = b.invZ + m * vstride;
    const int e0 = tile * kScanTile + threadIdx.x * kE;
    double wv[kE], pf[kE], sf[kE];
#pragma unroll
    for (int i = 0; i < kE; ++i) {
        const int e = e0 + i;
        if (e < N) {
            const double Fe = F[e] + off;
            F[e] = Fe;
            wv[i] = lam[e] * exp(-Fe);
            w[e] = wv[i];
        } else {
            wv[i] = 0.0;
        }
        pf[i] = wv[i];
        rev[threadIdx.x * kE + i] = wv[i];
    }
    const double tot = tile_scan(pf, warp_tot);   // (its barriers also publish rev[])
#pragma unroll
    for (int i = 0; i < kE; ++i) {
        const int e = e0 + i;
        if (e < N) Lt[e] = pf[i] - wv[i];          // exclusive prefix within the tile
    }
    // inclusive suffix within the tile = inclusive scan of the reversed tile
#pragma unroll
    for (int i = 0; i < kE; ++i) sf[i] = rev[kScanTile - 1 - (threadIdx.x * kE + i)];
    tile_scan(sf, warp_tot);
#pragma unroll
    for (int i = 0; i < kE; ++i) {
        const int e = tile * kScanTile + kScanTile - 1 - (threadIdx.x * kE + i);
        if (e < N) Ut[e] = sf[i];
    }
    if (threadIdx.x == 0) tile_row(b, M, 2, m)[tile] = tot;
}

// (D) exclusive prefix and suffix of the w tile totals.
__global__ void __launch_bounds__(1024) k_vec_d(int M, int nt, VecPtrs b) {
    const int m = blockIdx.x;
    totals_scan(tile_row(b, M, 2, m), nt, tile_row(b, M, 3, m), tile_row(b, M, 4, m));
}

// (E) L_r, U_r, D_r = U_r + e^{-Lambda} L_r, 1/D_r, 1/Z_r; flags a non-positive / non-finite D_r.
__global__ void __launch_bounds__(kT) k_vec_e(int N, int M, VecPtrs b, int64_t vstride) {
    const int m = blockIdx.y, tile = blockIdx.x;
    const double lpre = tile_row(b, M, 3, m)[tile];
    const double usuf = tile_row(b, M, 4, m)[tile];
    const double eL = b.scal[m * 8 + 1];
    const double *F = b.F + m * vstride;
    double *invD = b.invD + m * vstride, *invZ = b.invZ + m * vstride;
    int bad = 0;
    const int e0 = tile * kScanTile + threadIdx.x * kE;
#pragma unroll
    for (int i = 0; i < kE; ++i) {
        const int r = e0 + i;
        if (r < N) {
            const double L = invD[r] + lpre;
            const double U = invZ[r] + usuf;
            const double D = U + eL * L;
            bad |= !(D > 0.0 && isfinite(D));
            const double id = 1.0 / D;
            invD[r] = id;
            invZ[r] = id * exp(-F[r]);
        }
    }
    if (bad) b.scal[m * 8 + 2] = 1.0;
}

// ---- N < 8192: the five launches above as ONE CTA per profile (1024 threads x 8 consecutive slots;
// same sums: thread-local run, warp __shfl_up_sync scan, scan of the 32 warp totals).
constexpr int kST = 1024, kSEl = 8;

// inclusive scan of 8 consecutive values per thread over the block; returns the block total
__device__ double small_scan(double (&v)[kSEl], double *wt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 1; i < kSEl; ++i) v[i] += v[i - 1];
    const double t = v[kSEl - 1];
    double x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    double ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = 0.0;
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const double a = lane < (int)(blockDim.x >> 5) ? wt[lane] : 0.0;   // blockDim may be < 1024
        double z = a;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        double ze = __shfl_up_sync(0xffffffffu, z, 1);   // exclusive prefix, not z - a (see tile_scan)
        if (lane == 0) ze = 0.0;
        wt[32 + lane] = ze;
        if (lane == 31) wt[64] = z;       // block total
    }
    __syncthreads();
    const double off = wt[32 + warp] + ex;
#pragma unroll
    for (int i = 0; i < kSEl; ++i) v[i] += off;
    const double tot = wt[64];
    __syncthreads();
    return tot;
}

// small_scan of two arrays at once (the same sums in the same order for each, one set of barriers)
__device__ void small_scan2(double (&v)[kSEl], double (&u)[kSEl], double *wt, double *wu) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 1; i < kSEl; ++i) {
        v[i] += v[i - 1];
        u[i] += u[i - 1];
    }
    double x = v[kSEl - 1], y = u[kSEl - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xffffffffu, x, o), c = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) { x += a; y += c; }
    }
    double ex = __shfl_up_sync(0xffffffffu, x, 1), ey = __shfl_up_sync(0xffffffffu, y, 1);
    if (lane == 0) { ex = 0.0; ey = 0.0; }
    if (lane == 31) { wt[warp] = x; wu[warp] = y; }
    __syncthreads();
    if (warp == 0) {
        const bool in = lane < (int)(blockDim.x >> 5);
        double z = in ? wt[lane] : 0.0, q = in ? wu[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double a = __shfl_up_sync(0xffffffffu, z, o), c = __shfl_up_sync(0xffffffffu, q, o);
            if (lane >= o) { z += a; q += c; }
        }
        double ze = __shfl_up_sync(0xffffffffu, z, 1), qe = __shfl_up_sync(0xffffffffu, q, 1);
        if (lane == 0) { ze = 0.0; qe = 0.0; }
        wt[32 + lane] = ze;
        wu[32 + lane] = qe;
    }
    __syncthreads();
    const double ov = wt[32 + warp] + ex, ou = wu[32 + warp] + ey;
#pragma unroll
    for (int i = 0; i < kSEl; ++i) {
        v[i] += ov;
        u[i] += ou;
    }
}

__global__ void __launch_bounds__(kST) k_vec_small(const FluxDev *__restrict__ fluxes, int N, VecPtrs b,
                                                   int64_t vstride, const __grid_constant__ FluxDev single,
                                                   int use_single) {
    __shared__ double wt[65], wu[65];
    __shared__ FluxDev fs;               // the profile's parameters: shared-memory loads in the erfc loops
    extern __shared__ double rev[];      // [blockDim * 8]: w reversed, then its inclusive scan; then
                                         // [blockDim * 8]: lambda_j (own slots)
    const int nslot = (int)blockDim.x * kSEl;
    double *lams = rev + nslot;
    pdl_trigger();     // the build (a PDL secondary) may be scheduled while the vectors are computed
    const int m = blockIdx.x;
    {   // the profile's parameters (one profile: passed by value), one 8-byte word per thread
        static_assert(sizeof(FluxDev) % 8 == 0, "FluxDev is copied as 8-byte words");
        const unsigned long long *src = use_single ? reinterpret_cast<const unsigned long long *>(&single)
                                                   : reinterpret_cast<const unsigned long long *>(fluxes + m);
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(&fs);
        for (int i = threadIdx.x; i < (int)(sizeof(FluxDev) / 8); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const FluxDev &f = fs;
    const int e0 = threadIdx.x * kSEl;
    double *F = b.F + m * vstride, *lam = b.lam + m * vstride, *w = b.w + m * vstride;
    double *invD = b.invD + m * vstride, *invZ = b.invZ + m * vstride;
    // The erfc / exp evaluations run in rolled loops STRIDED over the CTA's threads (one element per
    // thread and round, coalesced stores; the CTA has up to 1024 threads, more than the (N + 1) / 8 the
    // scans need) through shared memory; the scans then take 8 consecutive slots per thread. Unrolled
    // 8x per thread the inlined fp64 erfc / exp stalled on instruction fetch, and 8 serial evaluations
    // per thread were the latency of the whole kernel (35 us for c3's profiles).
    // masses (N + 1 of them) and their inclusive scan: F_j = F(s_j), Lambda = F(t_r).
    // Each mass is flux_mass(lo, hi) (B term, then the pulses in order) with every bin edge's erfc
    // evaluated once and shared by the two masses it bounds: per pulse, erfc(|z| / sqrt 2) of the upper
    // edge of mass e goes to lams[e] (free until the lambda loop), and mass e adds the tail-aware
    // difference of phi_diff from lams[e - 1] and lams[e] (the straddling mass calls erf as phi_diff
    // does): bitwise the same masses with half the erfc evaluations.
#pragma unroll 1
    for (int e = threadIdx.x; e < nslot; e += blockDim.x) {
        double mv = 0.0;
        if (e <= N) {
            const double lo = e == 0 ? 0.0 : bin_centre(f, e - 1);
            const double hi = e == N ? f.t_r : bin_centre(f, e);
            mv = f.B * ((hi - lo) / f.t_r);
        }
        rev[e] = mv;
    }
    const double r2 = 0.70710678118654752440;  // 1/sqrt(2)
#pragma unroll 1
    for (int k = 0; k < f.k; ++k) {
        const double is = 1.0 / f.sigma[k];
        __syncthreads();                         // lams[] of the previous pulse consumed
#pragma unroll 1
        for (int e = threadIdx.x; e <= N; e += blockDim.x) {
            const double hi = e == N ? f.t_r : bin_centre(f, e);
            const double zh = (hi - f.tau[k]) * is;
            lams[e] = erfc((zh >= 0.0 ? zh : -zh) * r2);
        }
        __syncthreads();
#pragma unroll 1
        for (int e = threadIdx.x; e <= N; e += blockDim.x) {
            const double lo = e == 0 ? 0.0 : bin_centre(f, e - 1);
            const double hi = e == N ? f.t_r : bin_centre(f, e);
            const double zl = (lo - f.tau[k]) * is, zh = (hi - f.tau[k]) * is;
            double ph;
            if (zl >= 0.0) {
                ph = 0.5 * ((e == 0 ? erfc(zl * r2) : lams[e - 1]) - lams[e]);
            } else if (zh <= 0.0) {
                ph = 0.5 * (lams[e] - (e == 0 ? erfc(-zl * r2) : lams[e - 1]));
            } else {
                ph = 0.5 * (erf(zh * r2) + erf(-zl * r2));
            }
            rev[e] += f.S[k] * ph;
        }
    }
    __syncthreads();
    double wv[kSEl];
#pragma unroll
    for (int i = 0; i < kSEl; ++i) wv[i] = rev[e0 + i];
    const double Lam = small_scan(wv, wt);       // its barriers: every thread has read its slots
    const double eL = exp(-Lam);
#pragma unroll
    for (int i = 0; i < kSEl; ++i) rev[e0 + i] = wv[i];   // F_j (own slots)
    __syncthreads();
    // lambda_j, w_j = lambda_j e^{-F_j} (strided, as the masses)
#pragma unroll 1
    for (int e = threadIdx.x; e < nslot; e += blockDim.x) {
        double wj = 0.0;
        if (e < N) {
            const double Fe = rev[e];
            const double lm = flux_rate(f, bin_centre(f, e));
            const double ef = exp(-Fe);
            F[e] = Fe;
            lam[e] = lm;
            lams[e] = ef;                        // e^{-F_j}: 1/Z_j = e^{-F_j} / D_j below
            wj = lm * ef;
            w[e] = wj;
        }
        rev[e] = wj;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSEl; ++i) wv[i] = rev[e0 + i];
    __syncthreads();                             // own slots read: rev[] now takes w reversed
#pragma unroll
    for (int i = 0; i < kSEl; ++i) rev[nslot - 1 - (e0 + i)] = wv[i];
    double pf[kSEl], sf[kSEl];
#pragma unroll
    for (int i = 0; i < kSEl; ++i) pf[i] = wv[i];
    __syncthreads();                             // the reversed w is in rev[]
#pragma unroll
    for (int i = 0; i < kSEl; ++i) sf[i] = rev[e0 + i];
    small_scan2(pf, sf, wt, wu);                 // prefix of w and inclusive scan of the reversed w
#pragma unroll
    for (int i = 0; i < kSEl; ++i) rev[e0 + i] = sf[i];
    __syncthreads();
    // D_r = U_r + e^{-Lambda} L_r at the owner's slots (rev[nslot - 1 - r] held U_r: only this thread
    // reads it), then 1/D and 1/Z with one division per element strided over all threads (the
    // owner-slot form ran up to 16 dependent divisions in the 32 threads that own the positions)
#pragma unroll
    for (int i = 0; i < kSEl; ++i) {
        const int r = e0 + i;
        if (r < N) {
            const double L = pf[i] - wv[i];                   // sum_{j < r} w_j (exclusive prefix)
            const double U = rev[nslot - 1 - r];              // sum_{j >= r} w_j (inclusive suffix)
            rev[nslot - 1 - r] = U + eL * L;
        }
    }
    __syncthreads();
    int bad = 0;
#pragma unroll 1
    for (int r = threadIdx.x; r < N; r += blockDim.x) {
        const double D = rev[nslot - 1 - r];
        bad |= !(D > 0.0 && isfinite(D));
        const double id = 1.0 / D;
        invD[r] = id;
        invZ[r] = id * lams[r];                               // e^{-F_r} / D_r
    }
    if (threadIdx.x == 0) {
        b.scal[m * 8 + 0] = Lam;
        b.scal[m * 8 + 1] = eL;
        b.scal[m * 8 + 2] = 0.0;
    }
    __syncthreads();
    if (bad) b.scal[m * 8 + 2] = 1.0;
}

}  // namespace

cudaError_t launch_flux_vectors(const FluxDev *d_flux, int M, int N, VecPtrs base, int64_t vstride,
                                cudaStream_t s, const FluxDev *single) {
    const int nt = base.ntile;                         // tiles over the N + 1 masses
    const int ntN = (N + kScanTile - 1) / kScanTile;   // tiles over the N bins
    if (nt > 4096) return cudaErrorInvalidValue;
    if (N + 1 <= kST * kSEl) {                         // one CTA per profile, one launch
        int threads = N + 1 < kST ? N + 1 : kST;     // one element per thread for the transcendentals
        threads = (threads + 31) / 32 * 32;          // (the scans need only (N + 1) / 8 of them)
        const int smem = (int)(sizeof(double) * threads * kSEl * 2);
        // once per device (thread-safe; not in captured launches)
        const cudaError_t attr = func_attrs_once((const void *)k_vec_small, (int)(sizeof(double) * kST * kSEl * 2), false);
        if (attr != cudaSuccess) return attr;
        FluxDev one;
        if (single) one = *single;
        else memset(&one, 0, sizeof(one));
        k_vec_small<<<M, threads, smem, s>>>(d_flux, N, base, vstride, one, single ? 1 : 0);
        return cudaGetLastError();
    }
    k_vec_a<<<dim3(nt, M), kT, 0, s>>>(d_flux, N, M, base, vstride);
    k_vec_b<<<M, 1024, 0, s>>>(M, nt, base);
    k_vec_c<<<dim3(ntN, M), kT, 0, s>>>(N, M, base, vstride);
    k_vec_d<<<M, 1024, 0, s>>>(M, ntN, base);
    k_vec_e<<<dim3(ntN, M), kT, 0, s>>>(N, M, base, vstride);
    return cudaGetLastError();
}

}  // namespace spl
