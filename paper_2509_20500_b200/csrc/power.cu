// Step 4 (K6 + K7): power iteration for pi P~ = pi with P~ = J_l P~0 (Thm 2),
// looped on the device by a CUDA-graph conditional WHILE node whose body is two kernels.
//
// One iteration for V dead times sharing one P~0 (V = 1 for a single solve):
//   x_v[r]   = pi_v^k[(r - l_v) mod N]              (row permutation folded into the gather; the
//                                                     check kernel writes x in this gathered form)
//   y_v[j]   = sum_r x_v[r] P~0[r][j]               (left GEMV, fp64 accumulation)
//   s_v = sum_j y_v[j],  pi_v^{k+1} = y_v / s_v,  change_v = ||pi_v^{k+1} - pi_v^k||_1
//
// k_power_step (the GEMV, the dominant kernel): a persistent grid of kGemvCtas CTAs splits the
// row-segments (matrix, 512-column strip, row) of all still-active matrices into equal contiguous
// ranges (stream-K style, so the grid stays full when only a few matrices of a batch are still
// iterating). Each CTA streams its rows through a 3-stage shared-memory ring filled by TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx): per stage, RS row segments of 4 KB (fp64) or 2 KB
// (fp32) plus the matching RS rows of gathered x. Threads read their 2 columns per row from
// shared memory and accumulate all running vectors in fp64 registers; x of converged vectors is
// compacted away per stage so frozen vectors cost no FMAs. At the end of a strip piece a CTA writes
// its partial column sums; the last piece of a strip (atomic counter) adds the pieces in fixed order
// (deterministic), writes y and the strip's sum of y.
// k_power_check: s, the normalised L1 change, the state, the next gathered x, the active-matrix
// list, and (last CTA) the WHILE condition.
#include "common.cuh"
#include "ptx.cuh"

namespace spl {
namespace {

constexpr int kThreads = 256;           // 2 columns per thread across a 512-column strip

// RS rows per stage; SROW = shared-memory row stride in elements (512 + pad, 16-byte multiple) so that
// the k-rows of an MMA B fragment fall in different banks.
template <typename T> struct GemvCfg;
template <> struct GemvCfg<double> { static constexpr int RS = 8, SROW = kStripCols + 4; };   // 8 x 4 KB
template <> struct GemvCfg<float> { static constexpr int RS = 16, SROW = kStripCols + 8; };   // 16 x 2 KB

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

template <typename T> __device__ __forceinline__ void lds2(const T *p, double &a, double &b);
template <> __device__ __forceinline__ void lds2<double>(const double *p, double &a, double &b) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    a = v.x; b = v.y;
}
template <> __device__ __forceinline__ void lds2<float>(const float *p, double &a, double &b) {
    const float2 v = *reinterpret_cast<const float2 *>(p);
    a = v.x; b = v.y;
}

// acc[a][0..1] += sum_{rr < nr} xs[rr][a] * seg[rr][2 tid .. 2 tid + 1] for slots a < NA.
template <typename T, int NV, int NA, int RS>
__device__ __forceinline__ void stage_fma(double (&acc)[NV][2], const T *seg, const double *xs, int xst, int nr,
                                          int tid) {
    constexpr int SROW = GemvCfg<T>::SROW;   // shared-memory row stride
    if (nr == RS) {
#pragma unroll
        for (int rr = 0; rr < RS; ++rr) {
            double p0, p1;
            lds2<T>(seg + rr * SROW + 2 * tid, p0, p1);
            const double *xr = xs + rr * xst;
            if constexpr (NA == 1) {
                const double x = xr[0];
                acc[0][0] = fma(x, p0, acc[0][0]);
                acc[0][1] = fma(x, p1, acc[0][1]);
            } else {
#pragma unroll
                for (int v = 0; v < NA; v += 2) {
                    const double2 x = *reinterpret_cast<const double2 *>(xr + v);
                    acc[v][0] = fma(x.x, p0, acc[v][0]);
                    acc[v][1] = fma(x.x, p1, acc[v][1]);
                    acc[v + 1][0] = fma(x.y, p0, acc[v + 1][0]);
                    acc[v + 1][1] = fma(x.y, p1, acc[v + 1][1]);
                }
            }
        }
    } else {
        for (int rr = 0; rr < nr; ++rr) {
            double p0, p1;
            lds2<T>(seg + rr * SROW + 2 * tid, p0, p1);
            const double *xr = xs + rr * xst;
#pragma unroll
            for (int v = 0; v < NA; ++v) {
                acc[v][0] = fma(xr[v], p0, acc[v][0]);
                acc[v][1] = fma(xr[v], p1, acc[v][1]);
            }
        }
    }
}

// DMMA (FP64 tensor core, mma.sync) form of a stage for NV = 8, 16, 24, 32 vectors held as NV/8
// groups of 8. Per warp, the 64-column slice [64 w, 64 w + 64) as 8 n-tiles of 8 columns;
// D[v][col] += sum_k X[k][v] P[k][col] with A = X^T, B = 4 rows of P (4 x 8), D in registers:
// acc[q][nt][e] = D[8 q + g][64 w + 8 nt + 2 t + e] (g = lane / 4, t = lane % 4). A pair of active
// groups is one m16n8k4; a single active group is one m8n8k4; a converged group costs nothing.
// Rows k >= nr of a partial stage are zeroed in both operands (stale shared memory may hold NaN).
// One n-tile for vector groups Q, Q+1 of the compile-time running mask GM: one m16n8k4 when both
// run, one m8n8k4 when one does, nothing when neither does; then the next pair.
template <int NG, int Q, unsigned GM>
__device__ __forceinline__ void mma_groups(double (&acc)[NG][8][2], const double (&a)[NG], double bv, int nt) {
    if constexpr (Q < NG) {
        constexpr bool lo = (GM >> Q) & 1u;
        constexpr bool hi = Q + 1 < NG && ((GM >> (Q + 1)) & 1u);
        if constexpr (lo && hi) {
            asm volatile(
                "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                : "+d"(acc[Q][nt][0]), "+d"(acc[Q][nt][1]), "+d"(acc[Q + 1][nt][0]), "+d"(acc[Q + 1][nt][1])
                : "d"(a[Q]), "d"(a[Q + 1]), "d"(bv));
        } else if constexpr (lo) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[Q][nt][0]), "+d"(acc[Q][nt][1])
                         : "d"(a[Q]), "d"(bv));
        } else if constexpr (hi) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[Q + 1][nt][0]), "+d"(acc[Q + 1][nt][1])
                         : "d"(a[Q + 1]), "d"(bv));
        }
        mma_groups<NG, Q + 2, GM>(acc, a, bv, nt);
    }
}

// NVM slots on tensor cores (groups of 8, running mask GM bits [0, NVM/8)) and NVF <= 2 leftover
// slots on DFMA (running mask bits [NVM/8, NVM/8 + NVF)) that reuse the B fragments already in
// registers: lane (g, t) accumulates x_f[k = t] * P[t][64 w + 8 nt + g] into accf[f][nt]; the 4 t-lanes
// of a column are added with shuffles when the piece ends. Slots are the running vectors in
// compacted order: slot s reads the x column xc of vector s_vmap[s] (xc < 0: an empty slot of the
// last, partly filled group, fed zeros), so converged vectors free their tensor-core group.
template <typename T, int NVM, int NVF, int RS, int XST, unsigned GM>
__device__ __forceinline__ void stage_mma_fixed(double (&acc)[NVM / 8][8][2], double (&accf)[NVF > 0 ? NVF : 1][8],
                                                const T *seg, const double *xs, int nr, int lane, int warp,
                                                const int (&xc)[NVM / 8], const int (&fc)[NVF > 0 ? NVF : 1]) {
    constexpr int SROW = GemvCfg<T>::SROW;
    constexpr int NG = NVM / 8;
    const int g = lane >> 2, t = lane & 3;
    const T *sb = seg + warp * 64 + g;
#pragma unroll
    for (int kb = 0; kb < RS; kb += 4) {
        const int k = kb + t;
        const bool kin = k < nr;
        double a[NG];                                   // A fragments: X[k][slot 8 q + g]
#pragma unroll
        for (int q = 0; q < NG; ++q)
            a[q] = (kin && ((GM >> q) & 1u) && xc[q] >= 0) ? xs[k * XST + xc[q]] : 0.0;
        double xf[NVF > 0 ? NVF : 1];
#pragma unroll
        for (int f = 0; f < NVF; ++f) xf[f] = (kin && ((GM >> (NG + f)) & 1u)) ? xs[k * XST + fc[f]] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const double bv = kin ? (double)sb[k * SROW + nt * 8] : 0.0;
            mma_groups<NG, 0, GM>(acc, a, bv, nt);
#pragma unroll
            for (int f = 0; f < NVF; ++f)
                if ((GM >> (NG + f)) & 1u) accf[f][nt] = fma(xf[f], bv, accf[f][nt]);
        }
    }
}

// Running masks of compacted slots: the first G groups, and leftovers only behind all NG groups.
template <int NG, int NVF>
__host__ __device__ constexpr unsigned slot_mask(int nact) {
    const int G = nact >= 8 * NG ? NG : (nact + 7) / 8;
    const int F = nact > 8 * NG ? (nact - 8 * NG < NVF ? nact - 8 * NG : NVF) : 0;
    return ((1u << G) - 1u) | (((1u << F) - 1u) << NG);
}
template <int NG, int NVF>
__host__ __device__ constexpr bool is_slot_mask(unsigned m) {
    for (int n = 1; n <= 8 * NG + NVF; ++n)
        if (slot_mask<NG, NVF>(n) == m) return true;
    return false;
}

// Runtime running mask -> the compile-time specialisation (one per reachable slot mask; uniform branch).
template <typename T, int NVM, int NVF, int RS, int XST, unsigned GM = 1>
__device__ __forceinline__ void stage_mma(double (&acc)[NVM / 8][8][2], double (&accf)[NVF > 0 ? NVF : 1][8],
                                          const T *seg, const double *xs, int nr, int lane, int warp, unsigned mask,
                                          const int (&xc)[NVM / 8], const int (&fc)[NVF > 0 ? NVF : 1]) {
    if constexpr (GM < (1u << (NVM / 8 + NVF))) {
        if constexpr (is_slot_mask<NVM / 8, NVF>(GM)) {
            if (mask == GM) {
                stage_mma_fixed<T, NVM, NVF, RS, XST, GM>(acc, accf, seg, xs, nr, lane, warp, xc, fc);
                return;
            }
        }
        stage_mma<T, NVM, NVF, RS, XST, GM + 1>(acc, accf, seg, xs, nr, lane, warp, mask, xc, fc);
    }
}

template <typename T, int NV>
struct StepSmem {
    // DMMA path for NV >= 8: NVM = the multiple of 8 on FP64 tensor cores, NVF = 0..2 leftover
    // vectors on plain DFMA (so 17 dead times cost 17 FMAs per entry, not 24)
    static constexpr int NVM = NV >= 8 ? NV / 8 * 8 : 0;
    static constexpr int NVF = NV - NVM;
    static constexpr bool MMA = NVM > 0;
    // up to 16 vectors: 2 CTAs per SM with a 3-stage ring; 24 / 32 vectors need the registers of one
    // CTA per SM, which gets a 5-stage ring instead
    static constexpr int STAGES = NV >= 32 ? 5 : 3;
    static constexpr int MINB = NV >= 32 ? 1 : 2;
    static constexpr int RS = GemvCfg<T>::RS;
    static constexpr int XST = NV < 2 ? 2 : (NV + 1) / 2 * 2;           // == PowerArgs::xstride (16-B rows)
    static constexpr int SROW = GemvCfg<T>::SROW;
    static constexpr size_t SEG = (size_t)RS * SROW * sizeof(T);        // matrix bytes per stage
    static constexpr size_t XB = (size_t)RS * XST * sizeof(double);     // x bytes per stage
    static constexpr size_t BYTES = STAGES * (SEG + XB) + STAGES * sizeof(uint64_t);
};

// The state of (matrix, vector) mv through L2 (never a stale L1 line: the persistent loop kernel
// reads states other CTAs wrote in the same launch).
template <bool CG>
__device__ __forceinline__ SolveState load_state(const SolveState *p) {
    static_assert(sizeof(SolveState) == 48, "SolveState is three 16-byte words");
    if constexpr (!CG) return *p;   // a kernel of its own: states from earlier launches only
    SolveState s;
    const int4 *q = reinterpret_cast<const int4 *>(p);
    int4 *d = reinterpret_cast<int4 *>(&s);
    d[0] = __ldcg(q);
    d[1] = __ldcg(q + 1);
    d[2] = __ldcg(q + 2);
    return s;
}

// A load that bypasses L1 in the persistent loop kernel (CG: values other CTAs wrote in the same
// launch) and is a plain load in the two-kernel form.
template <bool CG, typename V>
__device__ __forceinline__ V ld_x(const V *p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
}

// One GEMV pass of every active (matrix, vector) over the stored P~0 (the body of k_power_step and of
// each iteration of k_power_loop). full[]: the CTA's ring mbarriers, initialised by the caller;
// q_issue / q_cons: the ring's stage sequence numbers, continued across passes. Every cross-CTA
// input (active list, states, partials) is read through L2.
template <typename T, int NV, bool CG>
__device__ __forceinline__ void gemv_pass(const PowerArgs &a, unsigned char *smem, uint32_t &q_issue,
                                          uint32_t &q_cons) {
    using SM = StepSmem<T, NV>;
    constexpr int RS = SM::RS;
    constexpr int kStages = SM::STAGES;
    constexpr int NWARPS = kThreads / 32;
    T *segs = reinterpret_cast<T *>(smem);                                             // [S][RS][512]
    double *xbuf = reinterpret_cast<double *>(smem + kStages * SM::SEG);               // [S][RS][XST]
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * (SM::SEG + SM::XB));   // TMA landed
    __shared__ int s_vmap[NV], s_cur[NV], s_nact, s_last;
    __shared__ unsigned s_gmask, s_vmask;
    __shared__ double red_sum[NWARPS][NV];

    const int tid = threadIdx.x, b = blockIdx.x, G = gridDim.x;
    const int N = a.N, S = a.strips;
    const int n_act = (int)ld_x<CG>(a.glob + 2);
    const int R = a.rows;                           // rows of the stored block (N, or a row shard)
    const int64_t T_units = (int64_t)n_act * S * R;
    if (T_units == 0) return;
    int64_t U = (T_units + G - 1) / G;
    if (U < kMinRowsPerCta) U = kMinRowsPerCta;
    const int64_t u_begin = (int64_t)b * U;
    if (u_begin >= T_units) return;
    const int64_t u_end = u_begin + U < T_units ? u_begin + U : T_units;
    if (tid == 0) ktime_start(a.ktime);

    int64_t u = u_begin;
    while (u < u_end) {
        const int64_t g64 = u / R;                       // strip index in active order
        const int g = (int)g64;
        const int ai = g / S, c = g % S;
        const int m = ld_x<CG>(a.act + ai);
        const int r_lo = (int)(u - g64 * R);
        const int64_t strip_end = (g64 + 1) * R;
        const int r_hi = (int)((u_end < strip_end ? u_end : strip_end) - g64 * R);
        u = g64 * R + r_hi;

        // running vectors of matrix m, compacted into slots (slot s = the s-th running vector)
        if (tid == 0) {
            int n = 0;
            unsigned vm = 0;
            for (int v = 0; v < NV; ++v) {
                const SolveState s = load_state<CG>(a.st + (size_t)m * NV + v);
                if (!s.done) {
                    s_vmap[n] = v; s_cur[n] = s.cur; ++n;
                    vm |= 1u << v;
                }
            }
            s_nact = n;
            // MMA path: the first ceil(n / 8) groups of 8 slots, DFMA leftovers only behind all groups
            s_gmask = SM::MMA ? slot_mask<SM::NVM / 8, SM::NVF>(n) : 0u;
            s_vmask = vm;
        }
        __syncthreads();
        const int nact = s_nact;
        const unsigned gmask = s_gmask;             // running MMA groups + DFMA leftovers
        const unsigned vmask = s_vmask;             // running vectors
        constexpr int NGX = SM::MMA ? SM::NVM / 8 : 1;
        constexpr int NFX = SM::NVF > 0 ? SM::NVF : 1;
        int xc[NGX];                                // x column of this lane's slot 8 q + (lane / 4)
        int fc[NFX];                                // x column of leftover slot NVM + f
        {
            const int gl = (tid & 31) >> 2;
#pragma unroll
            for (int q = 0; q < NGX; ++q) xc[q] = q * 8 + gl < nact ? s_vmap[q * 8 + gl] : -1;
#pragma unroll
            for (int f = 0; f < NFX; ++f) fc[f] = SM::NVM + f < nact ? s_vmap[SM::NVM + f] : 0;
        }

        const int cols = min(kStripCols, N - c * kStripCols);
        const uint32_t seg_bytes = (uint32_t)(((size_t)cols * sizeof(T) + 15) & ~(size_t)15);
        const T *pbase = reinterpret_cast<const T *>(a.P) + (size_t)m * a.mstride + (size_t)c * kStripCols;
        const double *xg = a.X + ((size_t)m * N + a.row0) * SM::XST;   // gathered x of the block's rows
        const int nstages = (r_hi - r_lo + RS - 1) / RS;

        auto issue = [&](int k) {   // stage k of this piece into buffer q_issue % S (thread 0)
            const int rs = r_lo + k * RS;
            const int nr = min(RS, r_hi - rs);
            const int buf = q_issue % kStages;
            mbar_expect_tx(&full[buf], nr * seg_bytes + (uint32_t)(nr * SM::XST * sizeof(double)));
            for (int rr = 0; rr < nr; ++rr)
                bulk_g2s(segs + ((size_t)buf * RS + rr) * SM::SROW, pbase + (size_t)(rs + rr) * a.ld, seg_bytes,
                         &full[buf]);
            bulk_g2s(xbuf + (size_t)buf * RS * SM::XST, xg + (size_t)rs * SM::XST,
                     (uint32_t)(nr * SM::XST * sizeof(double)), &full[buf]);
            ++q_issue;
        };
        if (tid == 0)
            for (int k = 0; k < kStages - 1 && k < nstages; ++k) issue(k);

        // MMA path: accm[group][n-tile][2]; FMA path: acc[vector][2]; MMA leftovers: acc[i][2]
        constexpr int NG = SM::MMA ? SM::NVM / 8 : 1;
        constexpr int NF = SM::MMA ? 1 : NV;
        constexpr int NL = SM::NVF > 0 ? SM::NVF : 1;
        double accm[NG][8][2];
        double accf[NL][8];   // MMA path leftovers: per lane, columns 64 w + 8 nt + g, rows k = t
        double acc[NF][2];    // FMA path (NV <= 4): vector v, columns 2 tid, 2 tid + 1
#pragma unroll
        for (int q = 0; q < NG; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) accm[q][i][0] = accm[q][i][1] = 0.0;
#pragma unroll
        for (int v = 0; v < NF; ++v) acc[v][0] = acc[v][1] = 0.0;
#pragma unroll
        for (int f = 0; f < NL; ++f)
#pragma unroll
            for (int i = 0; i < 8; ++i) accf[f][i] = 0.0;

        const int lane = tid & 31, warp = tid >> 5;
        for (int k = 0; k < nstages; ++k) {
            const int buf = q_cons % kStages;
            mbar_wait(&full[buf], (q_cons / kStages) & 1);
            const int nr = min(RS, r_hi - (r_lo + k * RS));
            const double *xs = xbuf + (size_t)buf * RS * SM::XST;
            const T *segb = segs + (size_t)buf * RS * SM::SROW;
            // every warp is done with stage k - 1: its ring slot takes stage k + S - 1 (measured
            // faster here than per-warp empty mbarriers: the block barrier keeps warps in step)
            __syncthreads();
            if (tid == 0 && k + kStages - 1 < nstages) issue(k + kStages - 1);
            if constexpr (SM::MMA) {
                stage_mma<T, SM::NVM, SM::NVF, RS, SM::XST>(accm, accf, segb, xs, nr, lane, warp, gmask, xc, fc);
            } else {
                if (2 * tid < cols) stage_fma<T, NV, NV, RS>(acc, segb, xs, SM::XST, nr, tid);
            }
            ++q_cons;
        }

        // ---- piece done: partial column sums into slot (b + g); the last piece of the strip reduces
        const int64_t gN = g64 * R;
        const int first = (int)(gN / U);
        const int last = (int)((gN + R - 1) / U);
        double *part = a.part + (size_t)(b + g) * NV * kStripCols;
        if constexpr (SM::MMA) {
            // rows of D of the running groups (converged vectors are never read back)
            const int lane = tid & 31, w = tid >> 5, gq = lane >> 2, tq = lane & 3;
            // slot rows go to their vector's partial row
#pragma unroll
            for (int q = 0; q < NG; ++q) {
                if (!((gmask >> q) & 1u) || xc[q] < 0) continue;
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
                    *reinterpret_cast<double2 *>(part + (size_t)xc[q] * kStripCols + w * 64 + nt * 8 + 2 * tq) =
                        make_double2(accm[q][nt][0], accm[q][nt][1]);
            }
            if constexpr (SM::NVF > 0) {
                // leftovers: add the 4 k-lanes (t) of each column, lane t = 0 writes
#pragma unroll
                for (int f = 0; f < SM::NVF; ++f) {
                    if (!((gmask >> (SM::NVM / 8 + f)) & 1u)) continue;
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) {
                        double v = accf[f][nt];
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        if (tq == 0) part[(size_t)fc[f] * kStripCols + w * 64 + nt * 8 + gq] = v;
                    }
                }
            }
        } else if (2 * tid < cols) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if ((vmask >> v) & 1u)
                    *reinterpret_cast<double2 *>(part + (size_t)v * kStripCols + 2 * tid) =
                        make_double2(acc[v][0], acc[v][1]);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(&a.strip_cnt[g], 1u);
            s_last = prev == (unsigned)(last - first);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            double lsum[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) lsum[v] = 0.0;
            if (2 * tid < cols) {
#pragma unroll
                for (int sl = 0; sl < NV; ++sl) {
                    if (sl >= nact) break;
                    const int v = s_vmap[sl];
                    double y0 = 0.0, y1 = 0.0;
                    for (int pc = first; pc <= last; ++pc) {   // fixed order over the pieces
                        const double2 t = __ldcg(reinterpret_cast<const double2 *>(
                            a.part + ((size_t)(pc + g) * NV + v) * kStripCols + 2 * tid));
                        y0 += t.x;
                        y1 += t.y;
                    }
                    // row shard: the partial y goes to the contiguous buffer the caller all-reduces
                    double *yv = (a.ypart ? a.ypart + ((size_t)m * NV + v) * N
                                          : a.y + (((size_t)m * NV + v) * 2 + (1 - s_cur[sl])) * N) +
                                 c * kStripCols + 2 * tid;
                    yv[0] = y0;
                    if (2 * tid + 1 < cols) yv[1] = y1;
                    else y1 = 0.0;
                    lsum[sl] = y0 + y1;
                }
            }
            const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
            for (int sl = 0; sl < NV; ++sl) {
                if (sl >= nact) break;
                const double t = warp_sum(lsum[sl]);
                if (lane == 0) red_sum[warp][sl] = t;
            }
            __syncthreads();
            if (tid < nact) {
                double ssum = 0.0;
#pragma unroll
                for (int w = 0; w < NWARPS; ++w) ssum += red_sum[w][tid];
                a.ssum[((size_t)m * NV + s_vmap[tid]) * S + c] = ssum;
            }
            if (tid == 0) a.strip_cnt[g] = 0u;
        }
        __syncthreads();
    }
    if (tid == 0) ktime_end(a.ktime);
}

template <typename T, int NV>
__device__ __forceinline__ void ring_init(unsigned char *smem) {
    using SM = StepSmem<T, NV>;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + SM::STAGES * (SM::SEG + SM::XB));
    if (threadIdx.x == 0) {
        for (int i = 0; i < SM::STAGES; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
}

template <typename T, int NV>
__global__ void __launch_bounds__(kThreads, StepSmem<T, NV>::MINB) k_power_step(const PowerArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_trigger();                                  // the check (programmatic graph edge) may be scheduled
    if (a.i8 && a.glob[3]) return;                  // the int8 tensor-core GEMV runs this plan
    ring_init<T, NV>(smem);
    uint32_t q_issue = 0, q_cons = 0;               // stage sequence numbers (buffer q % S, parity (q / S) & 1)
    gemv_pass<T, NV, false>(a, smem, q_issue, q_cons);
}

// Convergence check of one iteration (after k_power_step in the WHILE body). CTA (chunk, mv):
// s = sum of strip sums (fixed order); the chunk's part of ||y / s - pi^k||_1; the next gathered
// x: X[m][(j + l) mod N][v] = y_j / s; the last CTA of each (matrix, vector) adds the chunks in
// fixed order and updates the state; the last CTA of the grid rebuilds the active-matrix list and
// sets the WHILE condition. Done vectors are skipped (their pi stays frozen).
// check_item: the work of CTA (chunk c, vector mv); n_items = chunks x M x V, the count after which the
// last item rebuilds the active list (one item per CTA in k_power_check, grid-strided in k_power_loop).
template <bool CG>
__device__ __forceinline__ void check_item(const PowerArgs &a, int c, int mv, unsigned n_items) {
    __shared__ double red[8];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int N = a.N;
    const SolveState st = load_state<CG>(a.st + mv);
    if (st.done && a.ypart && !a.ypart_shared) {   // row shard: a frozen vector's partial stays zero
        const int j1 = min(N, (c + 1) * kCheckChunk);
        for (int j = c * kCheckChunk + tid; j < j1; j += 256) a.ypart[(size_t)mv * N + j] = 0.0;
    }
    if (!st.done) {
        const int m = mv / a.V, v = mv % a.V;
        // s = the strip sums added by every warp in the same fixed order (lane-strided, xor tree), so
        // all CTAs of (matrix, vector) hold the bitwise-same s
        const bool i8 = a.i8 && a.glob[3];
        const int nstrips = i8 ? a.strips_i8 : a.strips;
        // row shard: y = the all-reduced partial products (a.ypart); it is also kept in y[1 - cur] as
        // the next iterate (finish kernel, next change)
        const double *yn = a.ypart ? a.ypart + (size_t)(a.ypart_shared ? m : mv) * N
                                   : a.y + ((size_t)mv * 2 + (1 - st.cur)) * N;
        const double *yo = a.y + ((size_t)mv * 2 + st.cur) * N;
        // the chunk's y loads (E per thread) go out before the strip-sum reduction and stay in flight
        // together (the X stores below could alias them as far as the compiler knows)
        constexpr int E = kCheckChunk / 256;
        double yv[E], ov[E];
        if (!i8) {
            const int j1 = min(N, (c + 1) * kCheckChunk);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = c * kCheckChunk + tid + e * 256;
                yv[e] = j < j1 ? __ldcg(yn + j) : 0.0;
                ov[e] = j < j1 ? ld_x<CG>(yo + j) : 0.0;
            }
        }
        double S = 0.0;
        const double *ss = a.ssum + (size_t)mv * nstrips;
        for (int k = tid & 31; k < nstrips; k += 32) S += __ldcg(ss + k);
        S = warp_sum(S);
        const double inv_new = 1.0 / S, inv_old = 1.0 / st.s;
        if (a.ypart) {
            double *yw = a.y + ((size_t)mv * 2 + (1 - st.cur)) * N;
            const int j1 = min(N, (c + 1) * kCheckChunk);
            for (int j = c * kCheckChunk + tid; j < j1; j += 256) yw[j] = __ldcg(yn + j);
        }
        const int l = st.l < 0 ? 0 : st.l;
        double l1 = 0.0;
        if (i8) {
            // next x in the int8 GEMV's form: x~ = floor(pi^{k+1} 2^tau) in 7 bytes (power_i8.cu),
            // tau from the largest y (tile maxima), written at the gathered row r = (j + l) mod N
            double ym = 0.0;
            const double *sm = a.smax + (size_t)mv * nstrips;
            for (int k = tid & 31; k < nstrips; k += 32) ym = fmax(ym, __ldcg(sm + k));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ym = fmax(ym, __shfl_xor_sync(0xffffffffu, ym, o));
            const double pmax = ym * inv_new;
            const int tau = pmax > 0.0 ? 55 - ilogb(pmax) : 0;
            if (c == 0 && tid == 0) a.xtau[mv] = tau;
            const int r0 = c * kCheckChunk + tid * 8;         // 8 consecutive gathered rows
            if (r0 < N) {
                uint64_t wq[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    int j = r0 + e - l;
                    if (j < 0) j += N;
                    const double pn = __ldcg(yn + j) * inv_new;
                    l1 += fabs(pn - ld_x<CG>(yo + j) * inv_old);
                    const uint64_t xt = (uint64_t)ldexp(pn, tau);
#pragma unroll
                    for (int q = 0; q < 7; ++q) wq[q] |= ((xt >> (8 * (6 - q))) & 0xFFull) << (8 * e);
                }
                unsigned char *img = a.ximg + ((size_t)m * (N / 64) + r0 / 64) * 8192 + ((r0 % 64) / 16) * 128 + (r0 % 16);
#pragma unroll
                for (int q = 0; q < 7; ++q) {
                    const int row = q * a.V + v;
                    *reinterpret_cast<uint64_t *>(img + (row / 8) * 512 + (row % 8) * 16) = wq[q];
                }
            }
        } else {
            double *X = a.X + (size_t)m * N * a.xstride + v;
            const int j1 = min(N, (c + 1) * kCheckChunk);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = c * kCheckChunk + tid + e * 256;
                if (j < j1) {
                    const double pn = yv[e] * inv_new;
                    l1 += fabs(pn - ov[e] * inv_old);
                    int r = j + l;
                    if (r >= N) r -= N;
                    X[(size_t)r * a.xstride] = pn;
                }
            }
        }
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
        if (s_last && tid < 32) {   // the last CTA: chunk partials added lane-strided, fixed xor tree
            __threadfence();
            double L1 = 0.0;
            for (int k = tid; k < a.chunks; k += 32) L1 += __ldcg(a.l1part + (size_t)mv * a.chunks + k);
            L1 = warp_sum(L1);
            if (tid == 0) {
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
    }
    if (tid < 32) {   // the last CTA of the grid: active-matrix list (warp 0, 32 matrices per ballot)
        unsigned prev = 0;
        if (tid == 0) {
            __threadfence();
            prev = atomicAdd(&a.glob[0], 1u);
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == n_items - 1) {
            __threadfence();
            int n_act = 0;
            for (int m0 = 0; m0 < a.M; m0 += 32) {
                const int m = m0 + tid;
                int any = 0;
                if (m < a.M)
                    for (int v = 0; v < a.V; ++v) any |= !__ldcg(&a.st[(size_t)m * a.V + v].done);
                const unsigned b = __ballot_sync(0xffffffffu, any);
                if (any) a.act[n_act + __popc(b & ((1u << tid) - 1u))] = m;
                n_act += __popc(b);
            }
            if (tid == 0) {
                if (a.ktime) {   // the GEMV launch of this iteration (none before iteration 2 of a building plan)
                    const unsigned long long t0 = __ldcg(a.ktime), t1 = __ldcg(a.ktime + 1);
                    if (t1 > t0) {
                        a.ktime[2] += t1 - t0;
                        a.ktime[3] += 1ull;
                    }
                    a.ktime[0] = ~0ull;
                    a.ktime[1] = 0ull;
                }
                a.glob[0] = 0u;
                a.glob[1] = n_act > 0 ? 1u : 0u;
                a.glob[2] = (unsigned)n_act;
                if (a.use_handle) cudaGraphSetConditional(a.handle, n_act > 0 ? 1u : 0u);
            }
        }
    }
    __syncthreads();   // red / s_last free for the CTA's next item
}

__global__ void __launch_bounds__(256) k_power_check(const PowerArgs a) {
    pdl_wait();        // PDL secondary of the GEMV in the iteration graph; no-op otherwise
    check_item<false>(a, blockIdx.x, blockIdx.y, gridDim.x * gridDim.y);
}

// Grid-wide barrier of a co-resident (cooperatively launched) grid: bar[0] arrivals, bar[1] the
// generation. Generic-proxy global writes before it are made visible to the async proxy (the next
// pass's TMA reads of the gathered x) and to every CTA's L2 reads after it.
__device__ __forceinline__ void grid_sync(unsigned *bar) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // this thread's x writes -> later TMA reads
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = *reinterpret_cast<volatile unsigned *>(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned *>(bar + 1) == gen) {
            }
        }
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}

// The whole power iteration of a plan in ONE launch (a6 with the convergence check fused): a
// cooperatively launched persistent grid (every CTA resident) runs, while any vector is running,
// the GEMV pass (gemv_pass, as k_power_step), a grid barrier, the check of every (chunk, vector)
// item grid-strided over the CTAs (check_item, as k_power_check: normalisation, L1 change, next
// gathered x, states, active list), and a second grid barrier -- no launches, no graph nodes and
// no host round trips between iterations. Same arithmetic in the same order as the two-kernel loop.
template <typename T, int NV>
__global__ void __launch_bounds__(kThreads, StepSmem<T, NV>::MINB) k_power_loop(const PowerArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    ring_init<T, NV>(smem);
    uint32_t q_issue = 0, q_cons = 0;
    unsigned *bar = a.glob + kGridBarWord;
    const unsigned n_items = (unsigned)(a.chunks * a.M * a.V);
    while (__ldcg(a.glob + 1) != 0u) {
        gemv_pass<T, NV, true>(a, smem, q_issue, q_cons);
        grid_sync(bar);
        for (unsigned it = blockIdx.x; it < n_items; it += gridDim.x)
            check_item<true>(a, (int)(it % (unsigned)a.chunks), (int)(it / (unsigned)a.chunks), n_items);
        grid_sync(bar);
    }
}

// Strip sums (and, for the int8 GEMV, tile maxima) of an externally supplied y (a.ypart): the
// all-reduced partial products of a row shard, or the column sums the fused build produced (the
// first power-iteration product from the uniform start, shared by every vector of a matrix:
// a.ypart_shared). The GEMV's own strip sums do not exist for such a y. CTA (strip, mv), fixed order;
// the strip width follows the GEMV that runs this plan (512 columns, or the int8 GEMV's tiles).
__global__ void __launch_bounds__(256) k_shard_ssum(const PowerArgs a) {
    __shared__ double red[8], mx[8];
    const int c = blockIdx.x, mv = blockIdx.y, tid = threadIdx.x;
    const int N = a.N;
    const bool i8 = a.i8 && a.glob[3];
    const int nstrips = i8 ? a.strips_i8 : a.strips;
    if (c >= nstrips) return;
    const int width = i8 ? N / a.strips_i8 : kStripCols;
    const int m = mv / a.V;
    const double *yp = a.ypart + (size_t)(a.ypart_shared ? m : mv) * N + (size_t)c * width;
    const int cols = min(width, N - c * width);
    double t = 0.0, x = 0.0;
    for (int j = tid; j < cols; j += 256) {
        const double v = __ldcg(yp + j);
        t += v;
        x = fmax(x, v);
    }
    t = warp_sum(t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((tid & 31) == 0) { red[tid >> 5] = t; mx[tid >> 5] = x; }
    __syncthreads();
    if (tid == 0) {
        double sum = 0.0, smx = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { sum += red[w]; smx = fmax(smx, mx[w]); }
        a.ssum[(size_t)mv * nstrips + c] = sum;
        if (i8) a.smax[(size_t)mv * nstrips + c] = smx;
    }
}

// pi^0 = 1/N (y and gathered x), state reset, counters zeroed, all matrices with a real vector active.
__global__ void k_power_init(const PowerArgs a) {
    const int mv = blockIdx.y;
    const int m = mv / a.V, v = mv % a.V;
    const int N = a.N;
    double *y = a.y + (size_t)mv * 2 * N;
    double *X = a.X + (size_t)m * N * a.xstride;
    const double u = 1.0 / (double)N;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        y[j] = u;
        X[(size_t)j * a.xstride + v] = u;
        if (a.V == 1) X[(size_t)j * a.xstride + 1] = 0.0;   // padding column of the 16-byte x row
    }
    if (a.i8 && a.glob[3]) {
        // x^0 = 1/N in the int8 GEMV's slices (rows q V + v; zero for unused vectors), and v = 0
        // zeroes the image rows 7 V .. 127 that no vector owns
        const int tau = 55 - ilogb(u);
        const uint64_t xt = a.lsh[mv] >= 0 ? (uint64_t)ldexp(u, tau) : 0ull;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.xtau[mv] = tau;
        for (int r0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8; r0 < N; r0 += gridDim.x * blockDim.x * 8) {
            unsigned char *img = a.ximg + ((size_t)m * (N / 64) + r0 / 64) * 8192 + ((r0 % 64) / 16) * 128 + (r0 % 16);
            for (int q = 0; q < 7; ++q) {
                const uint64_t b = (xt >> (8 * (6 - q))) & 0xFFull;
                const int row = q * a.V + v;
                *reinterpret_cast<uint64_t *>(img + (row / 8) * 512 + (row % 8) * 16) = b * 0x0101010101010101ull;
            }
            if (v == 0)
                for (int row = 7 * a.V; row < 128; ++row)
                    *reinterpret_cast<uint64_t *>(img + (row / 8) * 512 + (row % 8) * 16) = 0ull;
        }
    }
    if (mv == 0 && blockIdx.x == 0 && threadIdx.x == 0 && a.ktime) {
        a.ktime[0] = ~0ull;
        a.ktime[1] = 0ull;
    }
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
        a.mv_cnt[mv] = 0u;
    }
    if (mv == 0) {
        const int ncnt = a.M * (a.i8 && a.strips_i8 > a.strips ? a.strips_i8 : a.strips);   // int8 GEMV: column tiles
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncnt; i += gridDim.x * blockDim.x)
            a.strip_cnt[i] = 0u;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            int n = 0;
            for (int mm = 0; mm < a.M; ++mm) {
                int any = 0;
                for (int vv = 0; vv < a.V; ++vv) any |= a.lsh[(size_t)mm * a.V + vv] >= 0;
                if (any) a.act[n++] = mm;
            }
            a.glob[0] = 0u;
            a.glob[1] = n > 0 ? 1u : 0u;
            a.glob[2] = (unsigned)n;
            a.glob[kGridBarWord] = 0u;        // k_power_loop's grid barrier: no arrivals
        }
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

template <typename T, int NV>
void *step_entry(size_t *smem, int *ctas_per_sm, void **loop) {
    *smem = StepSmem<T, NV>::BYTES;
    *ctas_per_sm = StepSmem<T, NV>::MINB;
    void *fn = (void *)k_power_step<T, NV>;
    if (func_attrs_once(fn, (int)*smem, false) != cudaSuccess) return nullptr;
    *loop = (void *)k_power_loop<T, NV>;
    if (func_attrs_once(*loop, (int)*smem, false) != cudaSuccess) *loop = nullptr;
    return fn;
}

void *step_fn(int dtype, int V, size_t *smem, int *cps, void **loop) {
    if (dtype == SPLIDAR_F64) {
        switch (V) {
            case 1: return step_entry<double, 1>(smem, cps, loop);
            case 2: return step_entry<double, 2>(smem, cps, loop);
            case 4: return step_entry<double, 4>(smem, cps, loop);
            case 8: return step_entry<double, 8>(smem, cps, loop);
            case 16: return step_entry<double, 16>(smem, cps, loop);
            case 17: return step_entry<double, 17>(smem, cps, loop);
            case 18: return step_entry<double, 18>(smem, cps, loop);
            case 24: return step_entry<double, 24>(smem, cps, loop);
            case 32: return step_entry<double, 32>(smem, cps, loop);
        }
    } else {
        switch (V) {
            case 1: return step_entry<float, 1>(smem, cps, loop);
            case 2: return step_entry<float, 2>(smem, cps, loop);
            case 4: return step_entry<float, 4>(smem, cps, loop);
            case 8: return step_entry<float, 8>(smem, cps, loop);
            case 16: return step_entry<float, 16>(smem, cps, loop);
            case 17: return step_entry<float, 17>(smem, cps, loop);
            case 18: return step_entry<float, 18>(smem, cps, loop);
            case 24: return step_entry<float, 24>(smem, cps, loop);
            case 32: return step_entry<float, 32>(smem, cps, loop);
        }
    }
    return nullptr;
}

}  // namespace

// Describes the solver kernels (function, grid, block, shared memory) for graph construction.
int solver_kernels(int dtype, int V, SolverKernels *out, const PowerArgs &a) {
    out->init_fn = (void *)k_power_init;
    int cps = 2;
    out->loop_fn = nullptr;
    out->step_fn = step_fn(dtype, V, &out->step_smem, &cps, &out->loop_fn);
    out->check_fn = (void *)k_power_check;
    out->finish_fn = (void *)k_power_finish;
    out->ssum_fn = (void *)k_shard_ssum;
    if (!out->step_fn) return 1;
    const int gx = (a.N + 255) / 256 < 64 ? (a.N + 255) / 256 : 64;
    out->init_grid = dim3(gx, a.M * a.V);
    out->init_block = dim3(256);
    out->finish_grid = dim3(gx, a.M * a.V);
    out->finish_block = dim3(256);
    // persistent: every resident CTA slot of the current device once (<= kGemvCtas, the workspace's
    // partial-sum slots)
    const int sms = device_sm_count() < kMaxSMs ? device_sm_count() : kMaxSMs;
    out->step_grid = dim3(sms * cps);
    out->step_block = dim3(kThreads);
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
