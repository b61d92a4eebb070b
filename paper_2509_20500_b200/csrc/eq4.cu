// the transition matrix built element by element from Eq. 4 (the sequential
// construction the paper replaces), on the GPU, so that Theorem 2's construction can be
// timed against it on the same hardware (the paper's Fig. 3a comparison).
//
// For every entry, independently (no reuse of integrals between entries, as in the element-wise
// method):
//   x_d = t_d mod t_r, u = x_d / Delta                        (reading R4: u in fp64)
//   a = s_i + x_d, D(a) = (ceil(a / Delta) - 1/2) Delta       (Eq. 3 bounds P:102, D P:104)
//   b = ceil((a - s_j) / t_r) t_r + s_j                       (a bin centre, so D(b) = b)
//   I_ij = int_{D(a)}^{b} lambda~ = (m_b - q_a) Lambda + F(s_j) - F(s_ia)   (periodic replica)
//   P_ij = lambda(s_j) exp(-I_ij)                             (Eq. 4)
// with F(t) = B t / t_r + sum_k S_k (Phi((t - tau_k) / sigma_k) - Phi(-tau_k / sigma_k)) evaluated in
// closed form (erfc) at both limits of every entry, then the row divided by its sum.
// One CTA per row: a pass that writes the unnormalised row and reduces its sum (fixed order), a
// second pass that rescales it in place (the row is L2-resident).
#include "common.cuh"

namespace spl {
namespace {

constexpr int kEqThreads = 256;

// Phi(z) standard normal CDF.
__device__ __forceinline__ double eq_cdf(double z) { return 0.5 * erfc(-z * 0.70710678118654752440); }

// Per-flux constants (not per-entry work): 1 / sigma_k, Phi(-tau_k / sigma_k), the Gaussian
// amplitudes S_k / (sigma_k sqrt(2 pi)), B / t_r.
struct EqConst {
    double is[kMaxPulses], c0[kMaxPulses], amp[kMaxPulses], rate_b;
};

// F(t) of one period (Thm 1), closed form: one erfc per pulse.
__device__ __forceinline__ double eq_F(const FluxDev &f, const EqConst &q, double t) {
    double v = q.rate_b * t;
    for (int k = 0; k < f.k; ++k) v += f.S[k] * (eq_cdf((t - f.tau[k]) * q.is[k]) - q.c0[k]);
    return v;
}

// lambda(t) (Eq. 1): one exp per pulse.
__device__ __forceinline__ double eq_lambda(const FluxDev &f, const EqConst &q, double t) {
    double v = q.rate_b;
    for (int k = 0; k < f.k; ++k) {
        const double z = (t - f.tau[k]) * q.is[k];
        v += q.amp[k] * exp(-0.5 * z * z);
    }
    return v;
}

template <typename T>
__global__ void __launch_bounds__(kEqThreads) k_build_eq4(const FluxDev f, double u, T *__restrict__ P, int64_t ld) {
    __shared__ double red[kEqThreads / 32];
    const int N = f.n;
    const int i = blockIdx.x;
    const double delta = f.t_r / (double)N;
    T *row = P + (int64_t)i * ld;
    EqConst q;
    q.rate_b = f.B / f.t_r;
    for (int k = 0; k < f.k; ++k) {
        q.is[k] = 1.0 / f.sigma[k];
        q.c0[k] = eq_cdf(-f.tau[k] / f.sigma[k]);
        q.amp[k] = f.S[k] / (f.sigma[k] * 2.50662827463100050242);
    }
    const double Lam = eq_F(f, q, f.t_r);   // Lambda = F(t_r) (reading R5)
    double sum = 0.0;
    for (int j = threadIdx.x; j < N; j += kEqThreads) {
        // every entry's integral from scratch: both limits in closed form, lambda(s_j), one exp
        const long long ka = (long long)ceil((double)i + 0.5 + u);     // 1-based bin of D(a), unrolled
        const long long qa = (ka - 1) / N;
        const int ia = (int)((ka - 1) - qa * N);
        const long long mb = (long long)ceil(((double)i - (double)j + u) / (double)N);
        const double sj = ((double)j + 0.5) * delta;
        const double sa = ((double)ia + 0.5) * delta;
        const double I = (double)(mb - qa) * Lam + (eq_F(f, q, sj) - eq_F(f, q, sa));
        const double p = eq_lambda(f, q, sj) * exp(-I);
        row[j] = (T)p;
        sum += p;
    }
    // fixed-order block reduction of the row sum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kEqThreads / 32; ++w) tot += red[w];
    const double inv = 1.0 / tot;
    for (int j = threadIdx.x; j < N; j += kEqThreads) row[j] = (T)((double)row[j] * inv);
}

}  // namespace

cudaError_t launch_build_eq4(const FluxDev &f, double u, int dtype, void *P, int64_t ld, cudaStream_t s) {
    if (dtype == SPLIDAR_F64) k_build_eq4<double><<<f.n, kEqThreads, 0, s>>>(f, u, (double *)P, ld);
    else k_build_eq4<float><<<f.n, kEqThreads, 0, s>>>(f, u, (float *)P, ld);
    return cudaGetLastError();
}

}  // namespace spl
