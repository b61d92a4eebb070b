// Step 1 of the path (K1-K3): discretised flux, warp+block prefix sums, row
// normalisers; everything fp64, the sums tree-shaped. The transcendental work (erfc differences,
// exp) runs grid-wide in pointwise kernels (A, C, E); the scans (B, D) run one 1024-thread CTA per
// profile (warp __shfl_up_sync scan + block scan of warp totals + a carry across 8192-element tiles).
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
#include "common.cuh"

namespace spl {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kEPT = 8;                       // consecutive elements per thread per tile
constexpr int kTile = kThreads * kEPT;        // 8192 elements per tile

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

// int_lo^hi lambda(t) dt for 0 <= lo <= hi <= t_r (Eq. 1; S = alpha E, lambda_b = B/t_r).
__device__ double flux_mass(const FluxDev &f, double lo, double hi) {
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

// Block-wide inclusive scan of a tile: each thread holds kEPT consecutive values in v[].
// Thread-local running sums, then a warp scan of thread totals (__shfl_up_sync, 5 steps), then
// a scan of the 32 warp totals by warp 0, then offsets. `carry` (the sum of all previous
// tiles) is added. Returns the tile total. Summation depth: kEPT + 5 + 5 + 1 per tile.
__device__ double block_scan_tile(double (&v)[kEPT], double *warp_tot, double carry) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 1; i < kEPT; ++i) v[i] += v[i - 1];
    const double t = v[kEPT - 1];
    double x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        double s = warp_tot[lane];  // kWarps == 32
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s;
    }
    __syncthreads();
    const double excl = (x - t) + (warp > 0 ? warp_tot[warp - 1] : 0.0);
    const double total = warp_tot[kWarps - 1];
#pragma unroll
    for (int i = 0; i < kEPT; ++i) v[i] = carry + (excl + v[i]);
    __syncthreads();  // warp_tot is reused by the next tile
    return total;
}

// (A) pointwise, grid-wide: bin masses m_e (e = 0..N) into F[] (m_N into scal[3]) and lambda_j.
__global__ void __launch_bounds__(256) k_vec_pointwise(const FluxDev *__restrict__ fluxes, int N, VecPtrs base,
                                                       int64_t vstride) {
    const int m = blockIdx.y;
    const FluxDev &f = fluxes[m];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e > N) return;
    const double lo = e == 0 ? 0.0 : bin_centre(f, e - 1);
    const double hi = e == N ? f.t_r : bin_centre(f, e);
    const double mass = flux_mass(f, lo, hi);
    if (e < N) {
        base.F[m * vstride + e] = mass;
        base.lam[m * vstride + e] = flux_rate(f, bin_centre(f, e));
    } else {
        base.scal[m * 8 + 3] = mass;
    }
}

// (B) one CTA per profile: F = inclusive prefix sum of the masses (in place), Lambda = F_{N-1} + m_N.
__global__ void __launch_bounds__(kThreads) k_vec_scan_F(int N, VecPtrs base, int64_t vstride) {
    __shared__ double warp_tot[kWarps];
    const int m = blockIdx.x;
    double *F = base.F + m * vstride;
    double *scal = base.scal + m * 8;
    double carry = 0.0;
    for (int t0 = 0; t0 < N; t0 += kTile) {
        double v[kEPT];
        const int e0 = t0 + threadIdx.x * kEPT;
#pragma unroll
        for (int i = 0; i < kEPT; ++i) v[i] = e0 + i < N ? F[e0 + i] : 0.0;
        const double tot = block_scan_tile(v, warp_tot, carry);
#pragma unroll
        for (int i = 0; i < kEPT; ++i)
            if (e0 + i < N) F[e0 + i] = v[i];
        carry += tot;
    }
    if (threadIdx.x == 0) {
        const double Lam = carry + scal[3];   // the tail mass int_{s_{N-1}}^{t_r} lambda closes the period
        scal[0] = Lam;
        scal[1] = exp(-Lam);
    }
}

// (C) pointwise: w_j = lambda_j e^{-F_j}.
__global__ void __launch_bounds__(256) k_vec_w(int N, VecPtrs base, int64_t vstride) {
    const int m = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N) base.w[m * vstride + j] = base.lam[m * vstride + j] * exp(-base.F[m * vstride + j]);
}

// (D) one CTA per profile: L_r = sum_{j<r} w_j (exclusive prefix), U_r = sum_{j>=r} w_j (suffix),
// D_r = U_r + e^{-Lambda} L_r, invD_r = 1 / D_r; a bad-row flag if some D_r is not positive and finite.
__global__ void __launch_bounds__(kThreads) k_vec_scan_D(int N, VecPtrs base, int64_t vstride) {
    __shared__ double warp_tot[kWarps];
    const int m = blockIdx.x;
    const double *w = base.w + m * vstride;
    double *invD = base.invD + m * vstride;
    double *scal = base.scal + m * 8;
    const double eL = scal[1];
    // prefix: scan of w shifted by one (element r holds w_{r-1}) = exclusive prefix L_r, kept in invD
    double carry = 0.0;
    for (int t0 = 0; t0 < N; t0 += kTile) {
        double v[kEPT];
        const int e0 = t0 + threadIdx.x * kEPT;
#pragma unroll
        for (int i = 0; i < kEPT; ++i) {
            const int e = e0 + i;
            v[i] = (e >= 1 && e < N) ? w[e - 1] : 0.0;
        }
        const double tot = block_scan_tile(v, warp_tot, carry);
#pragma unroll
        for (int i = 0; i < kEPT; ++i)
            if (e0 + i < N) invD[e0 + i] = v[i];
        carry += tot;
    }
    __syncthreads();
    // suffix: scan of the reversed sequence, element e holds w_{N-1-e}
    carry = 0.0;
    int bad = 0;
    for (int t0 = 0; t0 < N; t0 += kTile) {
        double v[kEPT];
        const int e0 = t0 + threadIdx.x * kEPT;
#pragma unroll
        for (int i = 0; i < kEPT; ++i) {
            const int e = e0 + i;
            v[i] = e < N ? w[N - 1 - e] : 0.0;
        }
        const double tot = block_scan_tile(v, warp_tot, carry);
#pragma unroll
        for (int i = 0; i < kEPT; ++i) {
            const int e = e0 + i;
            if (e < N) {
                const int r = N - 1 - e;
                const double D = v[i] + eL * invD[r];   // U_r + e^{-Lambda} L_r
                bad |= !(D > 0.0 && isfinite(D));
                invD[r] = 1.0 / D;
            }
        }
        carry += tot;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) scal[2] = bad ? 1.0 : 0.0;
}

// (E) pointwise: invZ_r = e^{-F_r} / D_r (row normaliser of the exp form).
__global__ void __launch_bounds__(256) k_vec_invz(int N, VecPtrs base, int64_t vstride) {
    const int m = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N) base.invZ[m * vstride + j] = base.invD[m * vstride + j] * exp(-base.F[m * vstride + j]);
}

}  // namespace

cudaError_t launch_flux_vectors(const FluxDev *d_flux, int M, int N, VecPtrs base, int64_t vstride,
                                cudaStream_t s) {
    const dim3 gp((N + 1 + 255) / 256, M), gv((N + 255) / 256, M);
    k_vec_pointwise<<<gp, 256, 0, s>>>(d_flux, N, base, vstride);
    k_vec_scan_F<<<M, kThreads, 0, s>>>(N, base, vstride);
    k_vec_w<<<gv, 256, 0, s>>>(N, base, vstride);
    k_vec_scan_D<<<M, kThreads, 0, s>>>(N, base, vstride);
    k_vec_invz<<<gv, 256, 0, s>>>(N, base, vstride);
    return cudaGetLastError();
}

}  // namespace spl
