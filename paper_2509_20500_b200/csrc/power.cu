// Step 4 (K6 + K7): power iteration for pi P~ = pi with P~ = J_l P~0 (Thm 2),
// one kernel per iteration, looped on the device by a CUDA-graph conditional WHILE node.
//
// One iteration for NV dead times sharing one P~0 (NV = 1 for a single solve):
//   x_v[r]   = pi_v^k[(r - l_v) mod N]              (row permutation folded into the gather)
//   y_v[j]   = sum_r x_v[r] P~0[r][j]               (left GEMV, fp64 accumulation)
//   s_v = sum_j y_v[j],  pi_v^{k+1} = y_v / s_v,  change_v = ||pi_v^{k+1} - pi_v^k||_1
//   (pi is kept as (y, s): the next iteration gathers y_v * (1 / s_v))
//
// Grid (strips, splits, matrices). CTA (c, s, m) reads the 512-column strip c of rows
// [s * rows_per_split, ...) of matrix m once (128-bit loads, 8 rows in flight per thread), multiplies by
// the NV gathered vectors staged in shared memory, and writes fp64 partial sums [v][s][j].
// The last CTA of a strip (atomic counter) adds the splits' partials in fixed order
// (deterministic) and writes y and the strip's sum of y. A second, small kernel (k_power_check)
// forms s, the normalised L1 change and the per-vector state, and its last CTA sets the WHILE
// condition (any vector still running and below max_iter). Converged vectors are frozen; a matrix
// whose vectors are all done is skipped by all of its CTAs.
#include "common.cuh"

namespace spl {
namespace {

constexpr int kSub = 64;      // rows of x staged in shared memory at a time
constexpr int kUnroll = 8;    // rows of P~0 in flight per thread

template <typename T> struct Ld16;
template <> struct Ld16<double> {
    static constexpr int n = 2;
    __device__ static __forceinline__ void load(const double *p, double (&o)[2]) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
        o[0] = v.x; o[1] = v.y;
    }
};
template <> struct Ld16<float> {
    static constexpr int n = 4;
    __device__ static __forceinline__ void load(const float *p, double (&o)[4]) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

template <typename T, int NV>
__global__ void __launch_bounds__(kStripCols / Ld16<T>::n) k_power_step(const PowerArgs a) {
    constexpr int VEC = Ld16<T>::n;
    constexpr int THREADS = kStripCols / VEC;
    constexpr int NWARPS = THREADS / 32;
    __shared__ double xs[kSub * NV];
    __shared__ double s_inv[NV];
    __shared__ int s_l[NV], s_cur[NV], s_done[NV];
    __shared__ int s_active, s_last_strip;
    __shared__ double red_sum[NWARPS][NV];

    const int m = blockIdx.z, split = blockIdx.y, strip = blockIdx.x, tid = threadIdx.x;
    const int N = a.N;
    SolveState *st = a.st + (size_t)m * NV;
    if (tid < NV) {
        const SolveState s = st[tid];
        s_inv[tid] = 1.0 / s.s;
        s_l[tid] = s.l < 0 ? 0 : s.l;
        s_cur[tid] = s.cur;
        s_done[tid] = s.done;
    }
    __syncthreads();
    if (tid == 0) {
        int act = 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) act |= !s_done[v];
        s_active = act;
    }
    __syncthreads();

    if (s_active) {
        const T *__restrict__ P = reinterpret_cast<const T *>(a.P) + (size_t)m * a.mstride;
        double *ybase = a.y + (size_t)m * NV * 2 * N;
        const int j0 = strip * kStripCols + tid * VEC;
        const bool full = j0 + VEC <= N;
        double acc[NV][VEC];
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[v][e] = 0.0;

        const int r0 = split * a.rows_per_split;
        const int r1 = min(N, r0 + a.rows_per_split);
        for (int rb = r0; rb < r1; rb += kSub) {
            const int nr = min(kSub, r1 - rb);
            for (int idx = tid; idx < nr * NV; idx += THREADS) {
                const int rr = idx / NV, v = idx % NV;
                int src = rb + rr - s_l[v];
                if (src < 0) src += N;
                xs[idx] = ybase[(size_t)(v * 2 + s_cur[v]) * N + src] * s_inv[v];
            }
            __syncthreads();
            if (full) {
                const T *prow = P + (size_t)rb * a.ld + j0;
                int rr = 0;
                for (; rr + kUnroll <= nr; rr += kUnroll) {
                    double p[kUnroll][VEC];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) Ld16<T>::load(prow + (size_t)(rr + u) * a.ld, p[u]);
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const double x = xs[(rr + u) * NV + v];
#pragma unroll
                            for (int e = 0; e < VEC; ++e) acc[v][e] = fma(x, p[u][e], acc[v][e]);
                        }
                }
                for (; rr < nr; ++rr) {
                    double p[VEC];
                    Ld16<T>::load(prow + (size_t)rr * a.ld, p);
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double x = xs[rr * NV + v];
#pragma unroll
                        for (int e = 0; e < VEC; ++e) acc[v][e] = fma(x, p[e], acc[v][e]);
                    }
                }
            } else if (j0 < N) {
                for (int rr = 0; rr < nr; ++rr) {
                    const T *prow = P + (size_t)(rb + rr) * a.ld + j0;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        if (j0 + e < N) {
                            const double pe = (double)prow[e];
#pragma unroll
                            for (int v = 0; v < NV; ++v) acc[v][e] = fma(xs[rr * NV + v], pe, acc[v][e]);
                        }
                    }
                }
            }
            __syncthreads();
        }

        // partial sums of this split: part[m][v][split][j]
        double *part = a.part + (size_t)m * NV * a.splits * N;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e)
                if (j0 + e < N) part[((size_t)v * a.splits + split) * N + j0 + e] = acc[v][e];
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(&a.strip_cnt[(size_t)m * a.strips + strip], 1u);
            s_last_strip = prev == (unsigned)(a.splits - 1);
        }
        __syncthreads();

        if (s_last_strip) {
            // ---- strip finalisation: y = sum over splits (fixed order) and the strip's sum of y
            __threadfence();
            double lsum[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) lsum[v] = 0.0;
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const int j = j0 + e;
                if (j < N) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double *pp = part + (size_t)v * a.splits * N + j;
                        // fixed-order sum over splits: 4 interleaved partial sums, then (a0+a1)+(a2+a3)
                        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                        int s = 0;
                        for (; s + 4 <= a.splits; s += 4) {
                            a0 += __ldcg(pp + (size_t)(s + 0) * N);
                            a1 += __ldcg(pp + (size_t)(s + 1) * N);
                            a2 += __ldcg(pp + (size_t)(s + 2) * N);
                            a3 += __ldcg(pp + (size_t)(s + 3) * N);
                        }
                        for (; s < a.splits; ++s) a0 += __ldcg(pp + (size_t)s * N);
                        const double y = (a0 + a1) + (a2 + a3);
                        ybase[((size_t)v * 2 + (1 - s_cur[v])) * N + j] = y;
                        lsum[v] += y;
                    }
                }
            }
            const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double t = warp_sum(lsum[v]);
                if (lane == 0) red_sum[warp][v] = t;
            }
            __syncthreads();
            if (tid < NV) {
                double ssum = 0.0;
#pragma unroll
                for (int w = 0; w < NWARPS; ++w) ssum += red_sum[w][tid];
                a.ssum[((size_t)m * NV + tid) * a.strips + strip] = ssum;
            }
            if (tid == 0) a.strip_cnt[(size_t)m * a.strips + strip] = 0u;
        }
    }
}

// Convergence check of one iteration (runs after k_power_step in the WHILE body).
// CTA (c, mv): s = sum of the strip sums (fixed order), then the chunk's part of
// ||y / s - pi^k||_1; the last CTA of each (matrix, vector) adds the chunks in fixed order and updates
// the state (iters, s, change, cur, converged / done); the last CTA of the grid sets the WHILE
// condition. Done vectors are skipped (their pi stays frozen).
__global__ void __launch_bounds__(256) k_power_check(const PowerArgs a) {
    __shared__ double red[8];
    __shared__ int s_last;
    const int c = blockIdx.x, mv = blockIdx.y, tid = threadIdx.x;
    const int N = a.N;
    const SolveState st = a.st[mv];
    if (!st.done) {
        double S = 0.0;
        const double *ss = a.ssum + (size_t)mv * a.strips;
        for (int k = 0; k < a.strips; ++k) S += __ldcg(ss + k);
        const double inv_new = 1.0 / S, inv_old = 1.0 / st.s;
        const double *yn = a.y + ((size_t)mv * 2 + (1 - st.cur)) * N;
        const double *yo = a.y + ((size_t)mv * 2 + st.cur) * N;
        double l1 = 0.0;
        const int j1 = min(N, (c + 1) * kCheckChunk);
        for (int j = c * kCheckChunk + tid; j < j1; j += 256) l1 += fabs(__ldcg(yn + j) * inv_new - yo[j] * inv_old);
        l1 = warp_sum(l1);
        if ((tid & 31) == 0) red[tid >> 5] = l1;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t += red[w];
            a.l1part[(size_t)mv * a.chunks + c] = t;
            __threadfence();
            const unsigned prev = atomicAdd(&a.mv_cnt[mv], 1u);
            s_last = prev == (unsigned)(a.chunks - 1);
        }
        __syncthreads();
        if (s_last && tid == 0) {
            __threadfence();
            double L1 = 0.0;
            for (int k = 0; k < a.chunks; ++k) L1 += __ldcg(a.l1part + (size_t)mv * a.chunks + k);
            SolveState s = st;
            s.iters += 1;
            s.change = L1;
            s.s = S;
            s.cur ^= 1;
            if (L1 < a.tol) { s.converged = 1; s.done = 1; }
            else if (s.iters >= a.max_iter || !(S > 0.0) || !isfinite(L1)) { s.done = 1; }
            a.st[mv] = s;
            a.mv_cnt[mv] = 0u;
            __threadfence();
        }
    }
    // grid completion: the last CTA decides whether the WHILE loop runs again
    if (tid == 0) {
        __threadfence();
        const unsigned total = gridDim.x * gridDim.y;
        const unsigned prev = atomicAdd(&a.glob[0], 1u);
        if (prev == total - 1) {
            __threadfence();
            int any = 0;
            const int n = a.M * a.V;
            for (int i = 0; i < n; ++i) any |= !__ldcg(&a.st[i].done);
            a.glob[0] = 0u;
            a.glob[1] = (unsigned)any;
            if (a.use_handle) cudaGraphSetConditional(a.handle, any ? 1u : 0u);
        }
    }
}

// pi^0 = 1/N for every (matrix, vector); state reset; counters zeroed.
__global__ void k_power_init(const PowerArgs a) {
    const int mv = blockIdx.y;
    const int N = a.N;
    double *y = a.y + (size_t)mv * 2 * N;
    const double u = 1.0 / (double)N;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) y[j] = u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        SolveState s;
        const int l = a.lsh[mv];
        s.l = l;
        s.iters = 0;
        s.done = l < 0 ? 1 : 0;
        s.converged = 0;
        s.cur = 0;
        s.pad0 = s.pad1 = s.pad2 = 0;
        s.s = 1.0;
        s.change = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        a.st[mv] = s;
    }
    if (mv == 0) {
        const int ncnt = a.M * a.strips;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncnt; i += gridDim.x * blockDim.x)
            a.strip_cnt[i] = 0u;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.M * a.V; i += gridDim.x * blockDim.x)
            a.mv_cnt[i] = 0u;
        if (blockIdx.x == 0 && threadIdx.x == 0) { a.glob[0] = 0u; a.glob[1] = 1u; }
    }
}

// pi = y[cur] / s, written to row out_idx[mv] of pi (skipped when out_idx[mv] < 0).
struct FinishArgs {
    PowerArgs p;
    double *pi;
    const int *out_idx;
};
__global__ void k_power_finish(const FinishArgs f) {
    const PowerArgs &a = f.p;
    const int mv = blockIdx.y;
    const int o = f.out_idx[mv];
    if (o < 0) return;
    const SolveState s = a.st[mv];
    const double *y = a.y + ((size_t)mv * 2 + s.cur) * a.N;
    double *out = f.pi + (size_t)o * a.N;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.N; j += gridDim.x * blockDim.x)
        out[j] = y[j] / s.s;
}

template <typename T>
void *step_fn(int V) {
    switch (V) {
        case 1: return (void *)k_power_step<T, 1>;
        case 2: return (void *)k_power_step<T, 2>;
        case 4: return (void *)k_power_step<T, 4>;
        case 8: return (void *)k_power_step<T, 8>;
        case 16: return (void *)k_power_step<T, 16>;
        default: return nullptr;
    }
}

}  // namespace

// Describes the three solver kernels (function, grid, block) for graph construction.
int solver_kernels(int dtype, int V, SolverKernels *out, const PowerArgs &a) {
    out->init_fn = (void *)k_power_init;
    out->step_fn = dtype == SPLIDAR_F64 ? step_fn<double>(V) : step_fn<float>(V);
    out->check_fn = (void *)k_power_check;
    out->finish_fn = (void *)k_power_finish;
    if (!out->step_fn) return 1;
    const int gx = (a.N + 255) / 256 < 64 ? (a.N + 255) / 256 : 64;
    out->init_grid = dim3(gx, a.M * a.V);
    out->init_block = dim3(256);
    out->finish_grid = dim3(gx, a.M * a.V);
    out->finish_block = dim3(256);
    out->step_grid = dim3(a.strips, a.splits, a.M);
    out->step_block = dim3(dtype == SPLIDAR_F64 ? kStripCols / 2 : kStripCols / 4);
    out->step_smem = 0;
    out->check_grid = dim3(a.chunks, a.M * a.V);
    out->check_block = dim3(256);
    return 0;
}

size_t finish_args_size() { return sizeof(FinishArgs); }
void make_finish_args(void *dst, const PowerArgs &a, double *pi, const int *out_idx) {
    FinishArgs *f = reinterpret_cast<FinishArgs *>(dst);
    f->p = a;
    f->pi = pi;
    f->out_idx = out_idx;
}

}  // namespace spl
