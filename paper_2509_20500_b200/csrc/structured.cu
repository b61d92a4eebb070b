// SURVEY §8(f) rows f2 + f1: the structured (matrix-free) transition operator, with the stationary
// solve, the second eigenvalue, the mixing steps and the bin trajectories built on it.
//
// The left product with the base matrix never needs the matrix. From §3.4 (E_base = exp.(-Lambda L - D),
// P:172-174; P = (1 lambda^T) . E; row normalisation P:79):
//   P~0[r][j] = w_j (r > j ? e^{-Lambda} : 1) / D_r,   w_j = lambda_j e^{-F_j}
// so for a row vector x (already gathered by the dead-time permutation of Thm 2, x_r = v[(r - l) mod N]):
//   y_j = sum_r x_r P~0[r][j] = w_j (C_j + e^{-Lambda} (T - C_j)),   z_r = x_r / D_r,
//   C_j = sum_{r <= j} z_r (inclusive prefix), T = sum_r z_r.
// One product is one prefix scan: O(N) instead of the N^2 b bytes of the dense GEMV.
//
// Teams: the threads that own one item's N positions, E consecutive positions per thread:
//   kWarp     one warp, E = 8 (N <= 256): shuffles only, __syncwarp orders the pushes
//   kBlock    one CTA, E = 8 (N <= 4096): block scan / sums through shared memory, __syncthreads
//   kCluster  a thread-block cluster of C CTAs x 512 threads, E = 8 (C = ceil(N / 4096)) for the solve,
//             lambda_2 and mixing, E = 16 (C = ceil(N / 8192)) for trajectories; CTA totals
//             exchanged over DSMEM, barrier.cluster between phases. (E = 16 solves fit c5's 17 items in
//             one wave of 4-CTA clusters but measured slower: 460 vs 361 us; per-CTA work dominates.)
// w and 1/D of a thread's positions stay in registers (solve) or are staged once in shared memory;
// the gathered iterate lives in
// shared memory (xbuf) and each product's result is pushed straight into the owner's xbuf at
// (j + l) mod N (DSMEM across CTAs), so the permutation costs one store per element and no extra pass.
// Per product: scan -> publish the CTA totals -> barrier -> outputs + push + publish the next sums ->
// barrier. Every CTA adds the published values in the same fixed order, so all CTAs take the same
// control-flow decisions and the result does not depend on timing (deterministic). Exclusive prefixes
// are formed by shuffles, never by subtraction.
#include <cooperative_groups.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spl {
namespace {

constexpr int kSMaxT = 512;                   // threads per CTA
constexpr int kSMaxWarps = kSMaxT / 32;
constexpr int kSMaxC = 16;                    // cluster size (> 8 is non-portable)
constexpr int kSExK = 8;                      // values published per CTA per exchange
constexpr int kSChunkB = kSMaxT * 8;          // positions per CTA at E = 8 (one-CTA limit)

enum { kWarp = 0, kBlock = 1, kCluster = 2 };

// padded shared-memory index of a position (E consecutive per thread: <= 2-way bank conflicts)
template <int E>
__device__ __forceinline__ int sidx(int p) { return p + p / E; }

struct SShared {
    double exA[kSExK * kSMaxC];
    double exB[kSExK * kSMaxC];
    double scr[kSExK * kSMaxWarps];
};

__device__ __forceinline__ double warp_allsum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Lane-parallel sums over the (<= 16) warps of a CTA, replacing 16-long dependent loops that every
// thread ran (ncu: ~860 of the lambda_2 kernel's ~2280 SASS instructions per warp per product).
// Fixed trees: every warp of every CTA computes bitwise-identical results from the same values.
// src[w] for w < nw (the CTA's warps); lanes >= nw contribute 0.
__device__ __forceinline__ double lanes_total(const double *src, int nw) {
    const int lane = threadIdx.x & 31;
    double x = lane < nw ? src[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
// exclusive prefix over the warps before `warp` and the total, of src[w] (w < nw)
__device__ __forceinline__ void lanes_scan(const double *src, int nw, int warp, double &before, double &total) {
    const int lane = threadIdx.x & 31;
    double inc = lane < nw ? src[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < kSMaxWarps; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const double exc = __shfl_up_sync(0xffffffffu, inc, 1);
    before = __shfl_sync(0xffffffffu, lane == 0 ? 0.0 : exc, warp);
    total = __shfl_sync(0xffffffffu, inc, kSMaxWarps - 1);
}

// Transposed butterfly: the warp sums of 8 values in 9 double shuffles (8 separate xor trees take 40).
// Each xor step exchanges half of the lane's remaining values with its partner, so after offsets
// 16, 8, 4 lane l holds one value index k8(l) = 4 b4 + 2 b3 + b2 (bits of l) summed over 8 lanes, and
// offsets 2, 1 finish it. Fixed order: every warp gets bitwise-identical totals for the same inputs.
__device__ __forceinline__ int k8_of_lane(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }
__device__ __forceinline__ int lane_of_k8(int k) { return ((k >> 2) & 1) * 16 + ((k >> 1) & 1) * 8 + (k & 1) * 4; }
__device__ __forceinline__ double warp_sum8(const double (&v)[8]) {
    const int lane = threadIdx.x & 31;
    const bool h4 = (lane >> 4) & 1, h3 = (lane >> 3) & 1, h2 = (lane >> 2) & 1;
    double w4[4], w2[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double keep = h4 ? v[i + 4] : v[i], send = h4 ? v[i] : v[i + 4];
        w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double keep = h3 ? w4[i + 2] : w4[i], send = h3 ? w4[i] : w4[i + 2];
        w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double x = (h2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, h2 ? w2[0] : w2[1], 4);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}
// per-warp sums of K <= 8 values, written by lane lane_of_k8(k) to dst[k * kSMaxWarps + warp]
template <int K>
__device__ __forceinline__ void warp_sums_to(const double (&v)[K], double *dst) {
    static_assert(K <= 8, "at most 8 values");
    double u[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k] = k < K ? v[k] : 0.0;
    const double t = warp_sum8(u);
    const int lane = threadIdx.x & 31, k = k8_of_lane(lane);
    if ((lane & 3) == 0 && k < K) dst[k * kSMaxWarps + (threadIdx.x >> 5)] = t;
}
// totals over the nw warps of K <= 8 per-warp values src[k * kSMaxWarps + w], in every thread
template <int K>
__device__ __forceinline__ void lanes_totals(const double *src, int nw, double (&out)[K]) {
    const int lane = threadIdx.x & 31;
    double u[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k] = (k < K && lane < nw) ? src[k * kSMaxWarps + lane] : 0.0;
    const double t = warp_sum8(u);
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = __shfl_sync(0xffffffffu, t, lane_of_k8(k));
}

template <int MODE>
struct Team {
    cg::cluster_group cl;
    int c, C;          // CTA rank in the cluster, cluster size
    double *exA, *exB, *scr;

    __device__ Team(SShared &sh, int C_) : cl(cg::this_cluster()) {
        c = MODE == kCluster ? (int)cl.block_rank() : 0;
        C = MODE == kCluster ? C_ : 1;
        exA = sh.exA;
        exB = sh.exB;
        scr = sh.scr;
    }
    __device__ __forceinline__ void barrier() {
        if constexpr (MODE == kWarp) __syncwarp();
        else if constexpr (MODE == kBlock) __syncthreads();
        else cl.sync();
    }
    // sum over the team-local threads (warp or CTA) of K values; every thread gets the totals
    template <int K>
    __device__ __forceinline__ void sum(double (&v)[K]) {
        if constexpr (MODE == kWarp) {
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = warp_allsum(v[k]);
        } else {
            const int nw = blockDim.x >> 5;
            if constexpr (K <= 8) {
                warp_sums_to<K>(v, scr);
                __syncthreads();
                lanes_totals<K>(scr, nw, v);
            } else {
                const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double x = warp_allsum(v[k]);
                    if (lane == 0) scr[k * kSMaxWarps + warp] = x;
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < K; ++k) v[k] = lanes_total(scr + k * kSMaxWarps, nw);
            }
            __syncthreads();
        }
    }
    // inclusive scan over the team-local positions of V vectors (E consecutive per thread);
    // tot[a] = team-local total
    template <int V, int E>
    __device__ __forceinline__ void scan(double (&v)[V][E], double (&tot)[V]) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double x[V], ex[V];
#pragma unroll
        for (int a = 0; a < V; ++a) {
#pragma unroll
            for (int i = 1; i < E; ++i) v[a][i] += v[a][i - 1];
            x[a] = v[a][E - 1];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int a = 0; a < V; ++a) {
                const double y = __shfl_up_sync(0xffffffffu, x[a], o);
                if (lane >= o) x[a] += y;
            }
#pragma unroll
        for (int a = 0; a < V; ++a) {
            ex[a] = __shfl_up_sync(0xffffffffu, x[a], 1);
            if (lane == 0) ex[a] = 0.0;
        }
        if constexpr (MODE == kWarp) {
#pragma unroll
            for (int a = 0; a < V; ++a) {
                tot[a] = __shfl_sync(0xffffffffu, x[a], 31);
#pragma unroll
                for (int i = 0; i < E; ++i) v[a][i] += ex[a];
            }
        } else {
            const int nw = blockDim.x >> 5;
#pragma unroll
            for (int a = 0; a < V; ++a)
                if (lane == 31) scr[a * kSMaxWarps + warp] = x[a];
            __syncthreads();
#pragma unroll
            for (int a = 0; a < V; ++a) {
                double wex, tt;
                lanes_scan(scr + a * kSMaxWarps, nw, warp, wex, tt);
                tot[a] = tt;
                const double e = wex + ex[a];
#pragma unroll
                for (int i = 0; i < E; ++i) v[a][i] += e;
            }
            __syncthreads();
        }
    }
    // as scan<V, E>, and in the same barrier the per-warp partials wp[k * kSMaxWarps + w] (written by
    // lane 0 of each warp before the call) are added in fixed order: part[k] = their sum over the
    // team-local warps
    template <int V, int E, int K>
    __device__ __forceinline__ void scan_sum(double (&v)[V][E], double (&tot)[V], const double *wp, double (&part)[K]) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double x[V], ex[V];
#pragma unroll
        for (int a = 0; a < V; ++a) {
#pragma unroll
            for (int i = 1; i < E; ++i) v[a][i] += v[a][i - 1];
            x[a] = v[a][E - 1];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int a = 0; a < V; ++a) {
                const double y = __shfl_up_sync(0xffffffffu, x[a], o);
                if (lane >= o) x[a] += y;
            }
#pragma unroll
        for (int a = 0; a < V; ++a) {
            ex[a] = __shfl_up_sync(0xffffffffu, x[a], 1);
            if (lane == 0) ex[a] = 0.0;
        }
        if constexpr (MODE == kWarp) {
#pragma unroll
            for (int a = 0; a < V; ++a) {
                tot[a] = __shfl_sync(0xffffffffu, x[a], 31);
#pragma unroll
                for (int i = 0; i < E; ++i) v[a][i] += ex[a];
            }
#pragma unroll
            for (int k = 0; k < K; ++k) part[k] = wp[k * kSMaxWarps];
        } else {
            const int nw = blockDim.x >> 5;
#pragma unroll
            for (int a = 0; a < V; ++a)
                if (lane == 31) scr[a * kSMaxWarps + warp] = x[a];
            __syncthreads();
#pragma unroll
            for (int a = 0; a < V; ++a) {
                double wex, tt;
                lanes_scan(scr + a * kSMaxWarps, nw, warp, wex, tt);
                tot[a] = tt;
                const double e = wex + ex[a];
#pragma unroll
                for (int i = 0; i < E; ++i) v[a][i] += e;
            }
            lanes_totals<K>(wp, nw, part);
            __syncthreads();
        }
    }
    // sum over the team-local warps of per-warp partials (after a barrier that ordered their writes)
    template <int K>
    __device__ __forceinline__ void warp_partials(const double *wp, double (&part)[K]) const {
        if constexpr (MODE == kWarp) {
#pragma unroll
            for (int k = 0; k < K; ++k) part[k] = wp[k * kSMaxWarps];
        } else {
            const int nw = (int)(blockDim.x >> 5);
            lanes_totals<K>(wp, nw, part);
        }
    }
    // exchange K per-CTA values through area ex (A or B) and synchronise the team; afterwards
    // total(k) gives the sum over all CTAs and over the CTAs before this one. For a single-CTA
    // team only the barrier remains (and the values are already the totals).
    template <int K>
    __device__ __forceinline__ void exchange(double *ex, const double (&v)[K]) {
        if constexpr (MODE == kCluster) {
            const int t = threadIdx.x;
            if (t < C * K) {
                const int dst = t / K, k = t - dst * K;
                double val = v[0];                 // select by unrolled compares: v[k] with a runtime k
#pragma unroll                                    // would put v in local memory
                for (int kk = 1; kk < K; ++kk) val = k == kk ? v[kk] : val;
                cl.map_shared_rank(ex, dst)[k * kSMaxC + c] = val;
            }
            cl.sync();
        } else {
            barrier();
        }
    }
    // totals only (no prefix) of K exchange values k0 .. k0 + K - 1, two per pass (lanes 0-15 and
    // 16-31, C <= 16, fixed xor trees); single-CTA teams: the own values
    template <int K>
    __device__ __forceinline__ void totals_only(const double *ex, int k0, const double (&own)[K], double (&tot)[K]) const {
        if constexpr (MODE == kCluster) {
            const int lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
#pragma unroll
            for (int k = 0; k < K; k += 2) {
                const int kk = k + half;
                double x = (sl < C && kk < K) ? ex[(k0 + kk) * kSMaxC + sl] : 0.0;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                tot[k] = __shfl_sync(0xffffffffu, x, 0);
                if (k + 1 < K) tot[k + 1] = __shfl_sync(0xffffffffu, x, 16);
            }
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) tot[k] = own[k];
        }
    }
    __device__ __forceinline__ void total(const double *ex, int k, double own, double &tot, double &before) const {
        if constexpr (MODE == kCluster) {   // lane-parallel over the C <= 16 CTAs (fixed shfl-up tree)
            const int lane = threadIdx.x & 31;
            double inc = lane < C ? ex[k * kSMaxC + lane] : 0.0;
#pragma unroll
            for (int o = 1; o < kSMaxC; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const double exc = __shfl_up_sync(0xffffffffu, inc, 1);
            tot = __shfl_sync(0xffffffffu, inc, kSMaxC - 1);
            before = __shfl_sync(0xffffffffu, lane == 0 ? 0.0 : exc, c);
        } else {
            tot = own;
            before = 0.0;
        }
    }

};

// Positions of this thread: p0 .. p0 + E - 1 (global), local index tid * E + e in its CTA's chunk.
template <int MODE, int E>
struct Pos {
    int N, p0, l;
    __device__ Pos(int N_, int c, int l_) : N(N_), l(l_) {
        p0 = (MODE == kCluster ? c * (int)blockDim.x * E : 0) + (int)threadIdx.x * E;
    }
    __device__ bool valid(int e) const { return p0 + e < N; }
    __device__ int loc(int e) const { return sidx<E>((int)threadIdx.x * E + e); }
};

// Push y (natural positions p0 + e) into the gathered xbuf of the owner of (p + l) mod N.
template <int MODE, int E>
__device__ __forceinline__ void push(Team<MODE> &tm, double *xbuf, const Pos<MODE, E> &P, const double (&y)[E]) {
    const int chunk = (int)blockDim.x * E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int p = P.p0 + e;
        if (p < P.N) {
            int r = p + P.l;
            if (r >= P.N) r -= P.N;
            if constexpr (MODE == kCluster) {
                const int dst = r / chunk;
                tm.cl.map_shared_rank(xbuf, dst)[sidx<E>(r - dst * chunk)] = y[e];
            } else {
                xbuf[sidx<E>(r)] = y[e];
            }
        }
    }
}

// Cluster push through a staging buffer: the warp's 32 E consecutive y values are written to its
// slice of ybuf (blocked, as held), then read back lane-contiguous, so every remote store instruction
// of the warp writes 32 consecutive positions of the destination (the blocked layout scattered each
// store over 32 lines of DSMEM; DSMEM moves ~20 B/clk per SM).
template <int E>
__device__ __forceinline__ void push_cl(Team<kCluster> &tm, double *xbuf, double *ybuf, const Pos<kCluster, E> &P,
                                        const double (&y)[E]) {
    constexpr int chunk = kSMaxT * E;                   // cluster teams are 512 threads (power of two)
    const int lane = threadIdx.x & 31, wbase = (int)(threadIdx.x & ~31u) * E;
#pragma unroll
    for (int e = 0; e < E; ++e) ybuf[P.loc(e)] = y[e];
    __syncwarp();
    const int cbase = tm.c * chunk;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const int q = wbase + k * 32 + lane;
        const int p = cbase + q;
        if (p < P.N) {
            int r = p + P.l;
            if (r >= P.N) r -= P.N;
            const int dst = r / chunk;                  // a shift: chunk is a compile-time power of two
            tm.cl.map_shared_rank(xbuf, dst)[sidx<E>(r & (chunk - 1))] = ybuf[sidx<E>(q)];
        }
    }
    __syncwarp();   // the slice may be restaged at once (two vectors per product)
}

// stage the thread's E values of src (global) in shared memory at its padded local indices
template <int MODE, int E>
__device__ __forceinline__ void stage(double *dst, const double *src, const Pos<MODE, E> &P) {
#pragma unroll
    for (int e = 0; e < E; ++e) dst[P.loc(e)] = P.valid(e) ? __ldg(src + P.p0 + e) : 0.0;
}

template <int MODE>
__device__ __forceinline__ int item_index(int C) {
    if constexpr (MODE == kCluster) return blockIdx.x / C;
    else return blockIdx.x;
}

template <int E>
__device__ __forceinline__ int xsize(int threads) { const int ch = threads * E; return ch + ch / E; }

// ---------------------------------------------------------------------------------------------
// f2: stationary solve. pi^0 = 1/N; v^{k+1} = v^k P~; pi^k = v^k / ||v^k||_1; stop after the first k
// with ||pi^{k+1} - pi^k||_1 < tol. P~ is row-stochastic, so ||v^k||_1 = ||v^0||_1 = 1 up to rounding
// (|1 - ||v^k||| ~ sqrt(k) eps): the iterates are not renormalised, the change is ||v^{k+1} - v^k||_1
// (differs from the normalised change by ~1e-15 << tol) and pi is normalised once at the end
// (R25). Per product: scan (its first barrier also adds the previous product's change
// partials) -> publish (scan total, change) -> barrier -> y, push, change partial -> barrier.
// Shared memory: xbuf | w | 1/D (each xsize; w and 1/D in registers at E = 8).
template <int MODE, int E>
// Warp and CTA teams (cluster teams run k_struct_solve_c1 below).
__global__ void __launch_bounds__(kSMaxT, 1) k_struct_solve(const StructArgs a) {
    static_assert(MODE != kCluster, "cluster teams: k_struct_solve_c1");
    extern __shared__ double xbuf[];
    __shared__ SShared sh;
    __shared__ double dwarp[kSMaxWarps];              // per-warp change partials of the last product
    Team<MODE> tm(sh, a.C);
    const int item = item_index<MODE>(a.C);
    const int m = a.prof[item], l = a.lsh[item];
    const Pos<MODE, E> P(a.N, tm.c, l);
    // w and 1/D: registers at E = 8 (measured faster), shared memory at E = 16
    constexpr bool REG = E <= 8;
    const int xs = xsize<E>(blockDim.x);
    double *ws = xbuf + xs, *ids = xbuf + 2 * xs;
    double wr[REG ? E : 1], idr[REG ? E : 1];
    if constexpr (REG) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            wr[e] = P.valid(e) ? __ldg(a.w + (size_t)m * a.vstride + P.p0 + e) : 0.0;
            idr[e] = P.valid(e) ? __ldg(a.invD + (size_t)m * a.vstride + P.p0 + e) : 0.0;
        }
    } else {
        stage(ws, a.w + (size_t)m * a.vstride, P);
        stage(ids, a.invD + (size_t)m * a.vstride, P);
    }
    const double eL = a.scal[m * 8 + 1];
    double yp[E];
    const double u = 1.0 / (double)P.N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        yp[e] = P.valid(e) ? u : 0.0;
        xbuf[P.loc(e)] = yp[e];                        // the gathered uniform vector is uniform
    }
    if ((threadIdx.x & 31) == 0) dwarp[threadIdx.x >> 5] = 0.0;
    double change = __longlong_as_double(0x7ff0000000000000ll);
    int k = 0, conv = 0;
    tm.barrier();
    for (;;) {
        // phase 1: z = x / D, scan (+ the change partials of product k - 1); publish both
        double v[1][E], tt[1], dp[1];
#pragma unroll
        for (int e = 0; e < E; ++e) v[0][e] = xbuf[P.loc(e)] * (REG ? idr[REG ? e : 0] : ids[P.loc(e)]);
        tm.template scan_sum<1, E, 1>(v, tt, dwarp, dp);   // its closing barrier also orders the xbuf
        const double tot = tt[0], dpart = dp[0];           // reads before this product's pushes
        double T, off, dummy;
        tm.total(tm.exA, 0, tot, T, off);
        if (k > 0) {
            tm.total(tm.exA, 1, dpart, change, dummy);
            if (change < a.tol) { conv = 1; break; }
            if (k >= a.max_iter || !isfinite(change)) break;
        }
        // phase 2: y = w (C + e^{-Lambda} (T - C)) at the natural positions (in place of the scan);
        // push; the change partial ||y - y_prev||_1 of this warp
        double d = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double Cj = off + v[0][e];
            v[0][e] = P.valid(e) ? (REG ? wr[REG ? e : 0] : ws[P.loc(e)]) * (Cj + eL * (T - Cj)) : 0.0;
            d += fabs(v[0][e] - yp[e]);
            yp[e] = v[0][e];
        }
        push<MODE, E>(tm, xbuf, P, v[0]);
        d = warp_allsum(d);
        if ((threadIdx.x & 31) == 0) dwarp[threadIdx.x >> 5] = d;
        tm.barrier();   // pushes complete (and dwarp written) before the next product reads them
        ++k;
    }
    // pi^k = v^k / ||v^k||_1 at the natural positions
    double sv[1] = {0.0};
#pragma unroll
    for (int e = 0; e < E; ++e) sv[0] += yp[e];
    tm.template sum<1>(sv);
    tm.template exchange<1>(tm.exB, sv);
    double s_k, dm;
    tm.total(tm.exB, 0, sv[0], s_k, dm);
    double *out = a.pi + (size_t)item * P.N;
    const double is = 1.0 / s_k;
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (P.valid(e)) out[P.p0 + e] = yp[e] * is;
    if (tm.c == 0 && threadIdx.x == 0) {
        SolveState st;
        st.l = l;
        st.iters = k;
        st.done = 1;
        st.converged = conv && s_k > 0.0;
        st.cur = 0;
        st.pad0 = st.pad1 = st.pad2 = 0;
        st.s = s_k;
        st.change = change;
        a.st[item] = st;
    }
}

// f2 on a cluster team with ONE cluster barrier per product. The two-barrier order exchanges the CTA
// totals of z = x / D after the scan (for every CTA's prefix offset and T), then pushes y. Here the
// pushing CTA also sends, per destination CTA, the sum of the z values it delivers there,
// z_r = y_j / D_r with r = (j + l) mod N (1/D at the shifted positions is staged once), and its change
// partial. After one barrier every CTA has its gathered x AND every CTA total: it scans its own chunk
// (one block barrier) and adds the offsets. Gathered x and the table are double-buffered by the
// parity of the product: a CTA can only be one product ahead (its next write needs everyone's
// arrival at the barrier that follows the current read).
// A CTA's chunk maps to a contiguous range of r (mod N) of one chunk's length, so its pushes land in
// at most 3 runs of destination CTAs (one chunk boundary and the wrap at N; the ragged last chunk ends
// at N): run boundaries are per-CTA constants, each thread keeps one accumulator per run.
// Issue-bound (~700 SASS instructions per warp per product in the first version): the table totals,
// the run sums and the table rows are done by warp 0 only, warp offsets by a lane-parallel scan,
// chunk = 512 E is a compile-time power of two (no integer division).
constexpr int kSeg = 3;
struct C1Shared {
    double tab[2][kSMaxC][kSMaxC + 1];   // [parity][source CTA][destination CTA | change]
    double wrun[kSeg + 1][kSMaxWarps];   // per run (and change partial), per warp: z delivered
    double scr[kSMaxWarps];              // block scan: warp totals
    double off, T, change;               // this product's offset of the CTA, total, last change
};

template <int E>
__global__ void __launch_bounds__(kSMaxT, 1) k_struct_solve_c1(const StructArgs a) {
    constexpr int kChunk = kSMaxT * E;                  // cluster teams are 512 threads
    constexpr int kLog = E == 4 ? 11 : (E == 8 ? 12 : 13);
    static_assert((1 << kLog) == kChunk, "chunk must be a power of two");
    extern __shared__ double dyn[];
    __shared__ C1Shared sh;
    __shared__ SShared shT;                             // epilogue sum (Team exchange)
    Team<kCluster> tm(shT, a.C);
    const int C = a.C, c = tm.c;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int item = blockIdx.x / C;
    const int m = a.prof[item], l = a.lsh[item];
    const Pos<kCluster, E> P(a.N, c, l);
    const int N = P.N, cbase = c * kChunk;
    const int nval = min(kChunk, N - cbase);            // valid positions of this CTA
    const int xs = xsize<E>(blockDim.x);
    double *stg = dyn + 2 * xs, *idsh = dyn + 3 * xs;   // push staging; 1/D at (j + l) mod N, lane order
    // gathered x of product parity b: dyn + b * xs (arithmetic, not a pointer array: a runtime-indexed
    // array of pointers lives in local memory)
    const double *wv = a.w + (size_t)m * a.vstride, *iv = a.invD + (size_t)m * a.vstride;
    // destination runs of this CTA's pushes: local q in [0, q1) -> dst0, [q1, q2) -> dst1, [q2, ..) -> dst2
    int q1, q2, dstr[kSeg];
    {
        int r = cbase + l;
        r = r >= N ? r - N : r;
        int q = 0;
        int qb[kSeg];
#pragma unroll
        for (int s2 = 0; s2 < kSeg; ++s2) {
            const int d = r >> kLog;
            const int end = min((d + 1) << kLog, N);    // first r past this run
            dstr[s2] = d;
            q += end - r;
            qb[s2] = q;
            r = end >= N ? 0 : end;
        }
        q1 = qb[0];
        q2 = qb[1];
    }
    double wr[E], idr[E], yp[E];
    const double u = 1.0 / (double)N;
    double own = 0.0;                                   // this CTA's total of z^0 = u / D
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const bool ok = P.valid(e);
        wr[e] = ok ? __ldg(wv + P.p0 + e) : 0.0;
        idr[e] = ok ? __ldg(iv + P.p0 + e) : 0.0;
        yp[e] = ok ? u : 0.0;
        dyn[P.loc(e)] = yp[e];                          // x^0: the uniform vector is its own gather
        dyn[xs + P.loc(e)] = 0.0;                       // positions >= N stay 0 in both buffers
        own += yp[e] * idr[e];
    }
    const int wq = (int)(tid & ~31u) * E + lane;        // lane-order local index for kk = 0
    int sgk[E];                                         // run of this lane's kk-th pushed position
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const int q = wq + k * 32;
        int r = cbase + q + l;
        if (r >= N) r -= N;
        idsh[sidx<E>(q)] = q < nval ? __ldg(iv + r) : 0.0;
        sgk[k] = (q >= q1) + (q >= q2);
    }
    const double eL = a.scal[m * 8 + 1];
    {   // table of product 0: own total on the diagonal
        double v[1] = {own};
        tm.template sum<1>(v);
        if (tid < C * (C + 1)) {
            const int dst = tid / (C + 1), col = tid - dst * (C + 1);
            tm.cl.map_shared_rank(&sh.tab[0][0][0], dst)[c * (kSMaxC + 1) + col] = col == c ? v[0] : 0.0;
        }
    }
    tm.cl.sync();
    double change = __longlong_as_double(0x7ff0000000000000ll);
    int k = 0, conv = 0;
    for (;;) {
        const int b = k & 1;
        const double *xcur = dyn + b * xs;
        double *xnext = dyn + (b ^ 1) * xs;
        if (warp == 0) {   // CTA totals (lane d: sum over sources, fixed order), offset, T, change
            double tot_d = 0.0, chg = 0.0;
            if (lane < C) {
                for (int src = 0; src < C; ++src) tot_d += sh.tab[b][src][lane];
                chg = sh.tab[b][lane][C];
            }
            double inc = tot_d;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const double exc = __shfl_up_sync(0xffffffffu, inc, 1);
            chg = warp_allsum(chg);
            if (lane == c) sh.off = c == 0 ? 0.0 : exc;
            if (lane == C - 1) sh.T = inc;
            if (lane == 0) sh.change = chg;
        }
        // local inclusive scan of z = x / D over the chunk
        double v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = xcur[P.loc(e)] * idr[e];
#pragma unroll
        for (int e = 1; e < E; ++e) v[e] += v[e - 1];
        double x = v[E - 1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        double ex = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) ex = 0.0;
        if (lane == 31) sh.scr[warp] = x;
        __syncthreads();
        if (k > 0) {
            change = sh.change;
            if (change < a.tol) { conv = 1; break; }
            if (k >= a.max_iter || !isfinite(change)) break;
        }
        double wt = lane < kSMaxWarps ? sh.scr[lane] : 0.0;   // exclusive prefix of the warp totals
#pragma unroll
        for (int o = 1; o < kSMaxWarps; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, wt, o);
            if (lane >= o) wt += y;
        }
        const double wexc = __shfl_sync(0xffffffffu, wt, warp == 0 ? 0 : warp - 1);
        const double base = sh.off + (warp == 0 ? 0.0 : wexc) + ex;
        const double T = sh.T;
        // y = w (C + e^{-Lambda} (T - C)); change partial
        double d = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double Cj = base + v[e];
            const double y = P.valid(e) ? wr[e] * (Cj + eL * (T - Cj)) : 0.0;
            d += fabs(y - yp[e]);
            yp[e] = y;
            stg[P.loc(e)] = y;
        }
        __syncwarp();
        // push y (lane-contiguous) into the other buffer; z delivered per run
        double acc[kSeg + 1] = {0.0, 0.0, 0.0, d};
#pragma unroll
        for (int kk = 0; kk < E; ++kk) {
            const int q = wq + kk * 32;
            if (q < nval) {
                int r = cbase + q + l;
                if (r >= N) r -= N;
                const int dst = r >> kLog;
                const double y = stg[sidx<E>(q)];
                tm.cl.map_shared_rank(xnext, dst)[sidx<E>(r & (kChunk - 1))] = y;
                const double z = y * idsh[sidx<E>(q)];
                acc[0] += sgk[kk] == 0 ? z : 0.0;
                acc[1] += sgk[kk] == 1 ? z : 0.0;
                acc[2] += sgk[kk] == 2 ? z : 0.0;
            }
        }
        warp_sums_to<kSeg + 1>(acc, &sh.wrun[0][0]);
        __syncthreads();
        if (warp == 0) {   // run sums and change partial of the CTA; its table row to every CTA
            double rs[kSeg + 1];
            lanes_totals<kSeg + 1>(&sh.wrun[0][0], kSMaxWarps, rs);
            if (lane <= C) {
                double val = rs[kSeg];                           // column C: change partial
                if (lane < C) {
                    val = 0.0;
#pragma unroll
                    for (int s2 = 0; s2 < kSeg; ++s2) val += dstr[s2] == lane ? rs[s2] : 0.0;
                }
                for (int dst = 0; dst < C; ++dst)
                    tm.cl.map_shared_rank(&sh.tab[b ^ 1][0][0], dst)[c * (kSMaxC + 1) + lane] = val;
            }
        }
        tm.cl.sync();   // pushes and table rows visible; everyone is done reading buffer b
        ++k;
    }
    // pi^k = v^k / ||v^k||_1 at the natural positions
    double sv[1] = {0.0};
#pragma unroll
    for (int e = 0; e < E; ++e) sv[0] += yp[e];
    tm.template sum<1>(sv);
    tm.template exchange<1>(tm.exB, sv);
    double s_k, dm;
    tm.total(tm.exB, 0, sv[0], s_k, dm);
    double *out = a.pi + (size_t)item * N;
    const double is = 1.0 / s_k;
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (P.valid(e)) out[P.p0 + e] = yp[e] * is;
    if (c == 0 && tid == 0) {
        SolveState st;
        st.l = l;
        st.iters = k;
        st.done = 1;
        st.converged = conv && s_k > 0.0;
        st.cur = 0;
        st.pad0 = st.pad1 = st.pad2 = 0;
        st.s = s_k;
        st.change = change;
        a.st[item] = st;
    }
}

// ---------------------------------------------------------------------------------------------
// f1: the second eigenvalue of P~ (§4). The known leading pair (left pi, right 1) is
// deflated: A = P~ - 1 pi, v A = v P~ - (v 1) pi. A two-dimensional real subspace Q = [q1; q2] is
// iterated, W = Q A, and the Ritz values are the eigenvalues of H = (W Q^T)(Q Q^T)^{-1}; a complex
// pair lambda2, conj(lambda2) spans a real 2-D invariant subspace, so real arithmetic suffices. Basis
// update: q1 = w1 / |w1|, q2 = (w2 - (w1.w2 / w1.w1) w1) / |w2| (applied as coefficients to the pushed
// w, so the product needs two team exchanges). Stop when the dominant Ritz value moves < tol.
// Shared memory: xbuf0 | xbuf1 | w | 1/D | pi.

__device__ __forceinline__ double hash_unit(uint32_t j, uint32_t salt) {   // deterministic in [-1, 1)
    uint32_t x = j * 0x9E3779B1u + salt * 0x85EBCA77u + 0x165667B1u;
    x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12; x *= 0x297A2D39u; x ^= x >> 15;
    return (double)x * (2.0 / 4294967296.0) - 1.0;
}

template <int MODE, int E>
__global__ void __launch_bounds__(kSMaxT, 1) k_struct_lambda2(const StructArgs a) {
    extern __shared__ double xbuf[];
    __shared__ SShared sh;
    Team<MODE> tm(sh, a.C);
    const int item = item_index<MODE>(a.C);
    const int m = a.prof[item], l = a.lsh[item];
    const Pos<MODE, E> P(a.N, tm.c, l);
    const int xs = xsize<E>(blockDim.x);
    double *xb0 = xbuf, *xb1 = xbuf + xs, *ws = xbuf + 2 * xs, *ids = xbuf + 3 * xs, *pis = xbuf + 4 * xs;
    __shared__ double wpart[7 * kSMaxWarps];          // per-warp partial dot products
    stage(ws, a.w + (size_t)m * a.vstride, P);
    stage(ids, a.invD + (size_t)m * a.vstride, P);
    stage(pis, a.pi + (size_t)item * P.N, P);
    const double eL = a.scal[m * 8 + 1];
    double wn[2][E];   // last W at the natural positions (q = combination of these)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int p = P.p0 + e;
        wn[0][e] = P.valid(e) ? hash_unit((uint32_t)p, 1u) : 0.0;
        wn[1][e] = P.valid(e) ? hash_unit((uint32_t)p, 2u) : 0.0;
        double g0 = 0.0, g1 = 0.0;       // gathered copies: xbuf[r] = q[(r - l) mod N]
        if (p < P.N) {
            int src = p - l;
            if (src < 0) src += P.N;
            g0 = hash_unit((uint32_t)src, 1u);
            g1 = hash_unit((uint32_t)src, 2u);
        }
        xb0[P.loc(e)] = g0;
        xb1[P.loc(e)] = g1;
    }
    double al = 1.0, be = 1.0, ga = 0.0;           // q1 = al w1, q2 = be (w2 - ga w1)
    double mu_re = 0.0, mu_im = 0.0, dmu = __longlong_as_double(0x7ff0000000000000ll);
    int k = 0, conv = 0;
    tm.barrier();
    for (;;) {
        // phase 1: current basis (gathered and natural), z = x / D, scans; sums and Gram Q Q^T
        double v[2][E], tot[2];
        double pp[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // sum q1, sum q2, q1.q1, q1.q2, q2.q2
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double idr = ids[P.loc(e)];
            const double g0 = xb0[P.loc(e)], g1 = xb1[P.loc(e)];
            v[0][e] = al * g0 * idr;
            v[1][e] = be * (g1 - ga * g0) * idr;
            wn[1][e] = be * (wn[1][e] - ga * wn[0][e]);   // q2 (natural)
            wn[0][e] = al * wn[0][e];                      // q1
            pp[0] += wn[0][e];
            pp[1] += wn[1][e];
            pp[2] += wn[0][e] * wn[0][e];
            pp[3] += wn[0][e] * wn[1][e];
            pp[4] += wn[1][e] * wn[1][e];
        }
        warp_sums_to<5>(pp, wpart);
        if constexpr (MODE == kWarp) __syncwarp();
        tm.template scan_sum<2, E, 5>(v, tot, wpart, pp);   // its first barrier also adds the pp partials
        {
            const double pv[7] = {tot[0], tot[1], pp[0], pp[1], pp[2], pp[3], pp[4]};
            tm.template exchange<7>(tm.exA, pv);
        }
        double T[2], off[2], sig[2], G11, G12, G22;
        tm.total(tm.exA, 0, tot[0], T[0], off[0]);
        tm.total(tm.exA, 1, tot[1], T[1], off[1]);
        {
            double tt[5];
            tm.template totals_only<5>(tm.exA, 2, pp, tt);
            sig[0] = tt[0]; sig[1] = tt[1]; G11 = tt[2]; G12 = tt[3]; G22 = tt[4];
        }
        // phase 2: W = Q P~ - (Q 1) pi; dots with Q (held in wn) and W; push W (into v)
        double hp[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};   // h11 h12 h21 h22 g11 g12 g22
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double y0 = 0.0, y1 = 0.0;
            if (P.valid(e)) {
                const double wj = ws[P.loc(e)], pj = pis[P.loc(e)];
                const double C0 = off[0] + v[0][e], C1 = off[1] + v[1][e];
                y0 = wj * (C0 + eL * (T[0] - C0)) - sig[0] * pj;
                y1 = wj * (C1 + eL * (T[1] - C1)) - sig[1] * pj;
            }
            hp[0] += y0 * wn[0][e];
            hp[1] += y0 * wn[1][e];
            hp[2] += y1 * wn[0][e];
            hp[3] += y1 * wn[1][e];
            hp[4] += y0 * y0;
            hp[5] += y0 * y1;
            hp[6] += y1 * y1;
            wn[0][e] = y0;
            wn[1][e] = y1;
        }
        if constexpr (MODE == kCluster) {            // staging buffer: the 6th (cluster launches only)
            push_cl<E>(tm, xb0, xbuf + 5 * xs, P, wn[0]);
            push_cl<E>(tm, xb1, xbuf + 5 * xs, P, wn[1]);
        } else {
            push<MODE, E>(tm, xb0, P, wn[0]);
            push<MODE, E>(tm, xb1, P, wn[1]);
        }
        double h[7];
        if constexpr (MODE == kCluster) {
            tm.template sum<7>(hp);
            tm.template exchange<7>(tm.exB, hp);
            tm.template totals_only<7>(tm.exB, 0, hp, h);
        } else {                                      // one barrier orders the pushes and the partials
            warp_sums_to<7>(hp, wpart);
            tm.barrier();
            tm.template warp_partials<7>(wpart, h);
            tm.barrier();                             // wpart is rewritten in the next phase 1
        }
        ++k;
        // Ritz values: H = M G^{-1}, M = W Q^T = [[h11, h12], [h21, h22]], G = Q Q^T
        double nre, nim;
        const double detG = G11 * G22 - G12 * G12;
        const bool two = detG > 1e-24 * G11 * G22 && G11 > 0.0;
        if (!(h[4] > 1e-280) || !(G11 > 0.0)) {        // the deflated operator annihilates the subspace
            nre = 0.0; nim = 0.0;
        } else if (two) {
            const double id = 1.0 / detG;
            const double H11 = (h[0] * G22 - h[1] * G12) * id, H12 = (-h[0] * G12 + h[1] * G11) * id;
            const double H21 = (h[2] * G22 - h[3] * G12) * id, H22 = (-h[2] * G12 + h[3] * G11) * id;
            const double tr = 0.5 * (H11 + H22);
            const double det = H11 * H22 - H12 * H21;
            const double disc = tr * tr - det;
            if (disc < 0.0) {
                nre = tr; nim = sqrt(-disc);
            } else {
                const double sq = sqrt(disc);
                const double r1 = tr + sq, r2 = tr - sq;
                nre = fabs(r1) >= fabs(r2) ? r1 : r2;
                nim = 0.0;
            }
        } else {
            nre = h[0] / G11;   // one-dimensional subspace: Rayleigh quotient
            nim = 0.0;
        }
        dmu = hypot(nre - mu_re, nim - mu_im);
        mu_re = nre;
        mu_im = nim;
        if (!(h[4] > 1e-280)) { conv = 1; break; }
        if (k > 1 && dmu < a.tol) { conv = 1; break; }
        if (k >= a.max_iter || !isfinite(dmu)) break;
        al = 1.0 / sqrt(h[4]);
        ga = h[5] / h[4];
        be = h[6] > 1e-280 ? 1.0 / sqrt(h[6]) : 0.0;
    }
    if (tm.c == 0 && threadIdx.x == 0) {
        SpecOut o;
        o.re = mu_re;
        o.im = fabs(mu_im);   // the member of a conjugate pair with phase in [0, pi]
        o.iters = k;
        o.converged = conv;
        o.change = dmu;
        a.spec[item] = o;
    }
}

// ---------------------------------------------------------------------------------------------
// f1: mixing steps (§4.1): for each start bin i, the first n with
// 1/2 || e_i P~^n - pi ||_1 <= eps (no renormalisation: P~ is stochastic). TV to stationarity is
// non-increasing in n for every start, so the smallest n with max_i TV_i(n) <= eps is max_i n_i.
// Item = one start bin; n_i written to a.nsteps[i] (-1: max_iter steps not enough).
// Shared memory: xbuf | w | 1/D | pi.
template <int MODE, int E>
__global__ void __launch_bounds__(kSMaxT, 1) k_struct_mixing(const StructArgs a) {
    extern __shared__ double xbuf[];
    __shared__ SShared sh;
    __shared__ double twarp[kSMaxWarps];              // per-warp TV partials of the last product
    Team<MODE> tm(sh, a.C);
    const int start = a.start_bin0 + item_index<MODE>(a.C);
    const int m = a.prof[0], l = a.lsh[0];
    const Pos<MODE, E> P(a.N, tm.c, l);
    const int xs = xsize<E>(blockDim.x);
    double *ws = xbuf + xs, *ids = xbuf + 2 * xs, *pis = xbuf + 3 * xs;
    stage(ws, a.w + (size_t)m * a.vstride, P);
    stage(ids, a.invD + (size_t)m * a.vstride, P);
    stage(pis, a.pi, P);
    const double eL = a.scal[m * 8 + 1];
    int r0 = start + l;
    if (r0 >= P.N) r0 -= P.N;
#pragma unroll
    for (int e = 0; e < E; ++e) xbuf[P.loc(e)] = (P.p0 + e == r0) ? 1.0 : 0.0;
    if ((threadIdx.x & 31) == 0) twarp[threadIdx.x >> 5] = 0.0;
    int n = 0, hit = -1;
    tm.barrier();
    for (;;) {
        // phase 1: scan of x / D (+ the TV partials of product n, decided one exchange later)
        double v[1][E], tt[1], tp[1];
#pragma unroll
        for (int e = 0; e < E; ++e) v[0][e] = xbuf[P.loc(e)] * ids[P.loc(e)];
        tm.template scan_sum<1, E, 1>(v, tt, twarp, tp);
        const double tot = tt[0], tvpart = tp[0];
        if constexpr (MODE == kCluster) {   // warp / CTA teams: scan_sum's closing barrier suffices
            const double pv[2] = {tot, tvpart};
            tm.template exchange<2>(tm.exA, pv);
        }
        double T, off, TV, dm;
        tm.total(tm.exA, 0, tot, T, off);
        if (n > 0) {
            tm.total(tm.exA, 1, tvpart, TV, dm);
            if (0.5 * TV <= a.eps) { hit = n; break; }
            if (n >= a.max_iter) break;
        }
        // phase 2: product n + 1, push, its TV partial
        double tv = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double Cj = off + v[0][e];
            v[0][e] = P.valid(e) ? ws[P.loc(e)] * (Cj + eL * (T - Cj)) : 0.0;
            tv += fabs(v[0][e] - pis[P.loc(e)]);
        }
        if constexpr (MODE == kCluster) push_cl<E>(tm, xbuf, xbuf + 4 * xs, P, v[0]);   // 5th buffer (cluster)
        else push<MODE, E>(tm, xbuf, P, v[0]);
        tv = warp_allsum(tv);
        if ((threadIdx.x & 31) == 0) twarp[threadIdx.x >> 5] = tv;
        tm.barrier();
        ++n;
    }
    if (tm.c == 0 && threadIdx.x == 0) {
        a.nsteps[start] = hit;
        atomicMax(a.nmax, hit < 0 ? 0x7fffffff : hit);
    }
}

// ---------------------------------------------------------------------------------------------
// f1: bin trajectory (§4.2): (start P~^n)[bin] for n = 0..steps (no renormalisation),
// and the final vector start P~^steps. Shared memory: xbuf | w | 1/D.
template <int MODE, int E>
__global__ void __launch_bounds__(kSMaxT, 1) k_struct_traj(const StructArgs a) {
    extern __shared__ double xbuf[];
    __shared__ SShared sh;
    Team<MODE> tm(sh, a.C);
    const int m = a.prof[0], l = a.lsh[0];
    const Pos<MODE, E> P(a.N, tm.c, l);
    const int xs = xsize<E>(blockDim.x);
    double *ws = xbuf + xs, *ids = xbuf + 2 * xs;
    stage(ws, a.w + (size_t)m * a.vstride, P);
    stage(ids, a.invD + (size_t)m * a.vstride, P);
    const double eL = a.scal[m * 8 + 1];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = P.p0 + e;
        double g = 0.0;
        if (r < P.N) {
            int src = r - l;
            if (src < 0) src += P.N;
            g = a.start[src];
        }
        xbuf[P.loc(e)] = g;
    }
    if (tm.c == 0 && threadIdx.x == 0) a.traj[0] = a.start[a.bin];
    tm.barrier();
    double v[1][E];
    for (int n = 1; n <= a.max_iter; ++n) {
        double tot[1];
#pragma unroll
        for (int e = 0; e < E; ++e) v[0][e] = xbuf[P.loc(e)] * ids[P.loc(e)];
        tm.template scan<1, E>(v, tot);
        tm.template exchange<1>(tm.exA, tot);
        double T, off;
        tm.total(tm.exA, 0, tot[0], T, off);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double Cj = off + v[0][e];
            v[0][e] = P.valid(e) ? ws[P.loc(e)] * (Cj + eL * (T - Cj)) : 0.0;
            if (P.p0 + e == a.bin) a.traj[n] = v[0][e];
        }
        if (n < a.max_iter) push<MODE, E>(tm, xbuf, P, v[0]);
        tm.barrier();   // pushes visible; the xbuf reads of this product are done everywhere
    }
    if (a.out) {
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (P.valid(e)) a.out[P.p0 + e] = a.max_iter > 0 ? v[0][e] : a.start[P.p0 + e];
    }
}

// Team shape for N positions and E positions per thread: C CTAs of `threads` threads.
int shape_for(int N, int E, int *C, int *threads) {
    if (N <= kSChunkB) {                         // one warp or one CTA (E = 8)
        int t = (N + 7) / 8;
        t = (t + 31) / 32 * 32;
        *C = 1;
        *threads = t < 32 ? 32 : t;
        return 0;
    }
    *threads = kSMaxT;
    *C = (N + kSMaxT * E - 1) / (kSMaxT * E);
    return *C <= kSMaxC ? 0 : 1;
}

// nbuf = shared-memory vectors of xsize doubles the kernel uses
// Kernel attributes once per kernel (keyed by its address: every team kernel has the same type), at
// the largest dynamic shared memory it can request; thread-safe, never inside a captured launch.
cudaError_t team_attrs_once(const void *fn, size_t max_smem) {
    return func_attrs_once(fn, (int)max_smem, true);   // once per (device, kernel)
}

template <typename K>
cudaError_t launch_team(K kernel, StructArgs a, int n_units, int E, int nbuf, cudaStream_t s) {
    int C, T;
    if (shape_for(a.N, E, &C, &T)) return cudaErrorInvalidValue;
    a.C = C;
    a.threads = T;
    const int chunk = T * E;
    const size_t smem = sizeof(double) * (size_t)nbuf * (chunk + chunk / E);
    const int cmax = kSMaxT * E;
    cudaError_t e = team_attrs_once((const void *)kernel, sizeof(double) * (size_t)nbuf * (cmax + cmax / E));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_units * C));
    cfg.blockDim = dim3((unsigned)T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = C > 1 ? 1 : 0;   // single-CTA teams launch without a cluster (no residency cap)
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// Clusters of C CTAs x T threads with `smem` dynamic bytes resident at once (cached per kernel, C).
int resident_clusters(const void *fn, int C, int T, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, int, size_t>, int> cache;   // per device
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, fn, C, T, smem);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3((unsigned)T);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        n = 0;
    }
    cache[key] = n;
    return n;
}

// Team width: 4 bins per thread (clusters of twice as many CTAs, half the DSMEM bytes per SM per
// product: c4's single item -15%) when every item's cluster is resident at once; else 8 (c5's 17
// items: two waves of 8-CTA clusters beat two of 16-CTA ones, 0.223 vs 0.356 ms).
bool one_wave_at_e4(const void *fn, int N, int n_units, int nbuf) {
    int C, T;
    if (shape_for(N, 4, &C, &T) || C < 2) return false;
    const size_t smem = sizeof(double) * (size_t)nbuf * (T * 4 + T);
    if (team_attrs_once(fn, sizeof(double) * (size_t)nbuf * (kSMaxT * 4 + kSMaxT)) != cudaSuccess) return false;
    const int cap = resident_clusters(fn, C, T, smem);
    return cap > 0 && n_units <= cap;
}

}  // namespace

// Valid N for every structured kernel (the lambda_2 kernel, at 4096 bins per CTA, is the tightest).
int struct_shape(int N, int *C, int *threads) {
    if (N < 2) return 1;
    return shape_for(N, 8, C, threads);
}

// NBUF_CL: shared-memory vectors of the cluster variant (+1 staging buffer for push_cl)
#define SPL_TEAM_LAUNCH(KERNEL, EC, NBUF, NBUF_CL)                                              \
    (a.N > kSChunkB ? launch_team(KERNEL<kCluster, EC>, a, n_units, EC, NBUF_CL, s)             \
                    : (a.N <= 256 ? launch_team(KERNEL<kWarp, 8>, a, n_units, 8, NBUF, s)       \
                                  : launch_team(KERNEL<kBlock, 8>, a, n_units, 8, NBUF, s)))

cudaError_t launch_struct(int kind, const StructArgs &a, int n_units, cudaStream_t s) {
    switch (kind) {
        case kStructSolve:
            if (a.N > kSChunkB) {   // cluster teams: one barrier.cluster per product
                if (one_wave_at_e4((const void *)k_struct_solve_c1<4>, a.N, n_units, 4))
                    return launch_team(k_struct_solve_c1<4>, a, n_units, 4, 4, s);
                return launch_team(k_struct_solve_c1<8>, a, n_units, 8, 4, s);
            }
            return a.N <= 256 ? launch_team(k_struct_solve<kWarp, 8>, a, n_units, 8, 3, s)
                              : launch_team(k_struct_solve<kBlock, 8>, a, n_units, 8, 3, s);
        case kStructLambda2:                                                       // 221 KB at E = 8
            if (a.N > kSChunkB && one_wave_at_e4((const void *)k_struct_lambda2<kCluster, 4>, a.N, n_units, 6))
                return launch_team(k_struct_lambda2<kCluster, 4>, a, n_units, 4, 6, s);
            return SPL_TEAM_LAUNCH(k_struct_lambda2, 8, 5, 6);
        case kStructMixing: return SPL_TEAM_LAUNCH(k_struct_mixing, 8, 4, 5);     // 184 KB at E = 8
        case kStructTraj: n_units = 1; return SPL_TEAM_LAUNCH(k_struct_traj, 16, 3, 3);
    }
    return cudaErrorInvalidValue;
}

}  // namespace spl
