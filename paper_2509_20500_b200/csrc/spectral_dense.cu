// SURVEY §8(f) row f1 on a STORED matrix: the second eigenvalue of P~ = J_l P0 (§4) for
// any row-stochastic P0 in HBM (fp64 or fp32; e.g. splidar_build_base's P~0, splidar_build_eq4's
// matrix, or a user's), reusing the multi-vector GEMV k_power_step<T, 2> (K6) for the products.
//
// Deflated two-dimensional real subspace iteration, as the structured kernel (structured.cu):
//   A = P~ - 1 pi (left pi, right 1: v A = v P~ - (v 1) pi), Q = [q1; q2], W = Q A,
//   H = (W Q^T)(Q Q^T)^{-1}, lambda_2 = the dominant eigenvalue of H (a complex pair spans a real plane),
//   q1' = w1 / |w1|, q2' = (w2 - (w1.w2 / w1.w1) w1) / |w2|.
// One iteration = three kernels in the body of a CUDA-graph WHILE node:
//   k_power_step<T, 2>  y_a = x_a^T P0 with the gathered x_a[r] = q_a[(r - l) mod N]   (y into buffer 1)
//   k_sd_dots           w_a = y_a - sigma_a pi (sigma_a = q_a 1, summed from the update kernel's per-CTA
//                       partials of the basis actually stored); per chunk the 7 dots w_a.q_b, w_a.w_b
//                       and the Gram dots q_a.q_b; the last CTA adds the chunks in fixed order, forms
//                       H, its dominant eigenvalue, the convergence test, the next basis coefficients
//                       and sets the WHILE condition
//   k_sd_update         q_a' at the natural positions (buffer 0) and gathered (x rows) for the next GEMV,
//                       with per-CTA partial sums of q_a'
// sigma is summed from the stored q, never carried analytically: in the degenerate cases (|w| at
// rounding level, q' = w / |w|) an analytic sigma' = (sum y - sigma) / |w| is all cancellation.
// Deterministic (fixed-order sums, no floating-point atomics).
#include <mutex>

#include "common.cuh"

namespace spl {
namespace {

constexpr int kSdT = 256;
constexpr int kSdChunk = 512;     // 64 CTAs at N = 32768 (4096: 8 CTAs, 17.7 us per launch)
constexpr int kSdDots = kSdDotsPerChunk;

__device__ __forceinline__ double sd_hash(uint32_t j, uint32_t salt) {   // deterministic in [-1, 1)
    uint32_t x = j * 0x9E3779B1u + salt * 0x85EBCA77u + 0x165667B1u;
    x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12; x *= 0x297A2D39u; x ^= x >> 15;
    return (double)x * (2.0 / 4294967296.0) - 1.0;
}

__device__ __forceinline__ double sd_warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// block sum of K values (fixed order); thread 0 gets the totals
template <int K>
__device__ __forceinline__ void sd_block_sum(double (&v)[K], double (*red)[kSdT / 32]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double x = sd_warp_sum(v[k]);
        if (lane == 0) red[k][warp] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < kSdT / 32; ++w) s += red[k][w];
            v[k] = s;
        }
    }
    __syncthreads();
}

// q at the natural positions: y[a][0] (buffer 0; the GEMV writes y into buffer 1, st.cur stays 0)
__device__ __forceinline__ double *sd_q(const SdArgs &s, int a) { return s.p.y + ((size_t)a * 2 + 0) * s.p.N; }
__device__ __forceinline__ double *sd_y(const SdArgs &s, int a) { return s.p.y + ((size_t)a * 2 + 1) * s.p.N; }

// one CTA: initial basis (hash vectors), gathered x rows, sigma; GEMV state and counters
__global__ void __launch_bounds__(kSdT) k_sd_init(const SdArgs s) {
    __shared__ double red[2][kSdT / 32];
    const PowerArgs &a = s.p;
    const int N = a.N, l = s.l;
    double acc[2] = {0.0, 0.0};   // sum q1, sum q2
    for (int j = threadIdx.x; j < N; j += kSdT) {
        const double q1 = sd_hash((uint32_t)j, 1u), q2 = sd_hash((uint32_t)j, 2u);
        sd_q(s, 0)[j] = q1;
        sd_q(s, 1)[j] = q2;
        int r = j + l;
        if (r >= N) r -= N;
        a.X[(size_t)r * a.xstride + 0] = q1;      // x_a[r] = q_a[(r - l) mod N]
        a.X[(size_t)r * a.xstride + 1] = q2;
        acc[0] += q1; acc[1] += q2;
    }
    for (int i = threadIdx.x; i < a.strips; i += kSdT) a.strip_cnt[i] = 0u;
    sd_block_sum<2>(acc, red);
    for (int k = threadIdx.x; k < s.nq; k += kSdT) {     // partials of sum q: the total in slot 0
        s.qsum[k] = k == 0 ? acc[0] : 0.0;
        s.qsum[s.nq + k] = k == 0 ? acc[1] : 0.0;
    }
    if (threadIdx.x == 0) {
        SdState st = {};
        st.al = 1.0; st.be = 1.0; st.ga = 0.0;
        st.dmu = __longlong_as_double(0x7ff0000000000000ll);
        *s.sd = st;
        for (int v = 0; v < 2; ++v) {
            SolveState ps = {};
            ps.l = l;
            ps.s = 1.0;
            a.st[v] = ps;                          // both vectors run; cur stays 0
        }
        a.act[0] = 0;
        a.glob[0] = 0u;
        a.glob[1] = 1u;
        a.glob[2] = 1u;
        *s.cnt = 0u;
    }
}

// w = y - sigma pi; the 10 dots per chunk; the last CTA decides
__global__ void __launch_bounds__(kSdT) k_sd_dots(const SdArgs s) {
    __shared__ double red[kSdDots][kSdT / 32];
    __shared__ int s_last;
    __shared__ double s_sig[2];
    const PowerArgs &a = s.p;
    const int N = a.N, c = blockIdx.x;
    const SdState st = *s.sd;
    {   // sigma_a = sum of the update kernel's partials, in the same fixed order in every CTA
        double sg[2] = {0.0, 0.0};
        for (int k = threadIdx.x; k < s.nq; k += kSdT) {
            sg[0] += __ldcg(s.qsum + k);
            sg[1] += __ldcg(s.qsum + s.nq + k);
        }
        sd_block_sum<2>(sg, red);
        if (threadIdx.x == 0) { s_sig[0] = sg[0]; s_sig[1] = sg[1]; }
        __syncthreads();
    }
    const double sig0 = s_sig[0], sig1 = s_sig[1];
    const double *y0 = sd_y(s, 0), *y1 = sd_y(s, 1), *q0 = sd_q(s, 0), *q1 = sd_q(s, 1);
    double acc[kSdDots];   // h11 h12 h21 h22 (w_a.q_b), g11 g12 g22 (w_a.w_b), G11 G12 G22 (q_a.q_b)
#pragma unroll
    for (int k = 0; k < kSdDots; ++k) acc[k] = 0.0;
    const int j1 = min(N, (c + 1) * kSdChunk);
    for (int j = c * kSdChunk + threadIdx.x; j < j1; j += kSdT) {
        const double pj = s.pi[j];
        const double w0 = __ldcg(y0 + j) - sig0 * pj, w1 = __ldcg(y1 + j) - sig1 * pj;
        const double a0 = __ldcg(q0 + j), a1 = __ldcg(q1 + j);
        acc[0] += w0 * a0; acc[1] += w0 * a1; acc[2] += w1 * a0; acc[3] += w1 * a1;
        acc[4] += w0 * w0; acc[5] += w0 * w1; acc[6] += w1 * w1;
        acc[7] += a0 * a0; acc[8] += a0 * a1; acc[9] += a1 * a1;
    }
    sd_block_sum<kSdDots>(acc, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kSdDots; ++k) s.part[(size_t)c * kSdDots + k] = acc[k];
        __threadfence();
        s_last = atomicAdd(s.cnt, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    {   // the last CTA: dot k summed over the chunks by warp k % 8 (lanes strided, then a fixed tree)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int k = warp; k < kSdDots; k += kSdT / 32) {
            double t = 0.0;
            for (int cc = lane; cc < (int)gridDim.x; cc += 32) t += __ldcg(s.part + (size_t)cc * kSdDots + k);
            t = sd_warp_sum(t);
            if (lane == 0) red[k][0] = t;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    double h[kSdDots];
#pragma unroll
    for (int k = 0; k < kSdDots; ++k) h[k] = red[k][0];
    SdState n = st;
    n.iters += 1;
    // Ritz values: H = M G^{-1}, M = W Q^T = [[h11, h12], [h21, h22]], G = Q Q^T
    double nre, nim;
    const double G11 = h[7], G12 = h[8], G22 = h[9];
    const double detG = G11 * G22 - G12 * G12;
    if (!(h[4] > 1e-280) || !(G11 > 0.0)) {
        nre = 0.0; nim = 0.0;
    } else if (detG > 1e-24 * G11 * G22) {
        const double id = 1.0 / detG;
        const double H11 = (h[0] * G22 - h[1] * G12) * id, H12 = (-h[0] * G12 + h[1] * G11) * id;
        const double H21 = (h[2] * G22 - h[3] * G12) * id, H22 = (-h[2] * G12 + h[3] * G11) * id;
        const double tr = 0.5 * (H11 + H22), det = H11 * H22 - H12 * H21, disc = tr * tr - det;
        if (disc < 0.0) { nre = tr; nim = sqrt(-disc); }
        else {
            const double sq = sqrt(disc), r1 = tr + sq, r2 = tr - sq;
            nre = fabs(r1) >= fabs(r2) ? r1 : r2;
            nim = 0.0;
        }
    } else {
        nre = h[0] / G11; nim = 0.0;
    }
    n.dmu = hypot(nre - st.mu_re, nim - st.mu_im);
    n.mu_re = nre;
    n.mu_im = nim;
    bool stop = false;
    if (!(h[4] > 1e-280)) { n.converged = 1; stop = true; }
    else if (n.iters > 1 && n.dmu < s.tol) { n.converged = 1; stop = true; }
    else if (n.iters >= s.max_iter || !isfinite(n.dmu)) stop = true;
    // next basis q1' = al w1, q2' = be (w2 - ga w1)
    n.al = h[4] > 1e-280 ? 1.0 / sqrt(h[4]) : 1.0;
    n.ga = h[4] > 1e-280 ? h[5] / h[4] : 0.0;
    n.be = h[6] > 1e-280 ? 1.0 / sqrt(h[6]) : 0.0;
    n.sig_w[0] = sig0;                             // the sigma these w were formed with (update kernel)
    n.sig_w[1] = sig1;
    n.done = stop;
    *s.sd = n;
    *s.cnt = 0u;
    __threadfence();
    if (s.use_handle) cudaGraphSetConditional(s.handle, stop ? 0u : 1u);
    else a.glob[1] = stop ? 0u : 1u;
}

// q' at the natural positions and gathered into the x rows of the next GEMV
__global__ void __launch_bounds__(kSdT) k_sd_update(const SdArgs s) {
    __shared__ double red[2][kSdT / 32];
    const PowerArgs &a = s.p;
    const int N = a.N, l = s.l;
    const SdState st = *s.sd;
    if (st.done) return;
    const double *y0 = sd_y(s, 0), *y1 = sd_y(s, 1);
    double *q0 = sd_q(s, 0), *q1 = sd_q(s, 1);
    double acc[2] = {0.0, 0.0};
    for (int j = blockIdx.x * kSdT + threadIdx.x; j < N; j += gridDim.x * kSdT) {
        const double pj = s.pi[j];
        const double w0 = __ldcg(y0 + j) - st.sig_w[0] * pj, w1 = __ldcg(y1 + j) - st.sig_w[1] * pj;
        const double n0 = st.al * w0, n1 = st.be * (w1 - st.ga * w0);
        q0[j] = n0;
        q1[j] = n1;
        int r = j + l;
        if (r >= N) r -= N;
        a.X[(size_t)r * a.xstride + 0] = n0;
        a.X[(size_t)r * a.xstride + 1] = n1;
        acc[0] += n0;
        acc[1] += n1;
    }
    sd_block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        s.qsum[blockIdx.x] = acc[0];
        s.qsum[s.nq + blockIdx.x] = acc[1];
    }
}

}  // namespace

int sd_chunks(int N) { return (N + kSdChunk - 1) / kSdChunk; }

void sd_kernels(SdKernels *k, int N) {
    k->init_fn = (void *)k_sd_init;
    k->dots_fn = (void *)k_sd_dots;
    k->update_fn = (void *)k_sd_update;
    k->block = dim3(kSdT);
    k->dots_grid = dim3((unsigned)sd_chunks(N));
    k->update_grid = dim3((unsigned)sd_update_ctas(N));
}

int sd_update_ctas(int N) {
    const int ug = (N + kSdT - 1) / kSdT;
    return ug < 1184 ? ug : 1184;
}

}  // namespace spl
