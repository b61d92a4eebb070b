// Step 4 for small N (N <= 2048): the whole power iteration of one (matrix, dead time) pair in ONE
// launch, on one thread-block cluster, reading the STORED P~0 (the same GEMV as k_power_step, without
// its per-iteration launches). At these sizes the matrices are L2-resident and the general path is
// bound by launch and graph latency (c1: ~30 us per iteration), not by bandwidth.
//
// Cluster of C CTAs (C = min(16, ceil(N / 32))): CTA c owns the rows [c R, (c + 1) R) of P~0 and the
// output columns [c W, (c + 1) W) (R = W = ceil(N / C)). Its rows of P~0 are copied to shared memory
// once when they fit in 96 KB (N <= 384 fp64 / 512 fp32 at R = 32), else read from L2 straight into
// registers (16 rows of 16-byte loads in flight per thread; SPLIDAR_FUSED_LDG=0: a 3-stage
// shared-memory ring of TMA bulk copies, 64 KB per stage). One product pi P~ = x P~0 with the
// gathered x_r = v[(r - l) mod N] (Thm 2), default form (ONE exchange per product):
//   A  partial y over the CTA's rows (x_r from shared memory, fp64 FMA) -> the partial of column j
//      pushed (st.async, completing the receiver's mbarrier) to the CTA owning row (j + l) mod N, with
//      the CTA's partial total and its change partial of the previous product
//   B  every CTA adds the C partials of each of its rows in fixed CTA order -> x_r = y_{r-l}
//      (unnormalised); s = sum of the C totals; the L1 change over its rows (published with the next A)
// SPLIDAR_FUSED_1X=0: the two-exchange form (owners of columns add the partials, then push y_j to
// row (j + l) mod N and the sums; barrier.cluster or st.async per exchange). Same y in the same order;
// s is summed in another order, so the two forms agree to rounding.
// Same definition as the general path: pi^0 = 1/N, pi^{k+1} = y / ||y||_1, stop after the first
// product with ||pi^{k+1} - pi^k||_1 < tol (decided one exchange later, on identical sums in every
// CTA), or after max_iter products. Deterministic: fixed-order sums, no atomics.
#include <cooperative_groups.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace spl {
namespace {

constexpr int kFT = 256;          // threads per CTA
constexpr int kRing = 3;          // stages of the TMA row ring (rows not resident in shared memory)
constexpr int kRingBytes = 64 * 1024;   // per stage
constexpr int kFMaxC = 16;
constexpr int kFMaxN = 2 * kFT * 4;   // N <= 2048: at most 4 column pairs per thread

struct FusedShared {
    double exA[2 * kFMaxC];       // scan of nothing: [0] unused, change partials
    double exB[kFMaxC];           // sum partials
    double red[kFT / 32];
    double tx[2][kFMaxC];         // one-exchange form: every CTA's partial-y total, by product parity
    double dx[2][kFMaxC];         // and its change partial of the previous product
};

__device__ __forceinline__ double fwarp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// block sum, every thread gets the total (fixed order)
__device__ __forceinline__ double fblock_sum(double v, double *red) {
    v = fwarp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kFT / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

// Q = column pairs per thread (N <= 512 Q), RS = rows whose loads are in flight together.
template <typename T, int Q>
__global__ void __launch_bounds__(kFT, 1) k_power_fused(const FusedArgs a) {
    constexpr int NC = 2 * Q;
    constexpr int RS = Q <= 2 ? 8 : 4;
    // direct global loads: twice the rows in flight at Q = 2 (N = 513..1024, the c2 shape); at Q = 1
    // (mostly rows resident in shared memory) the register budget of RS keeps 2x more clusters resident
    constexpr int RSG = Q == 2 ? 16 : 8;
    pdl_wait();        // PDL secondary of the build (launch_fused); no-op otherwise
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double fsm[];
    __shared__ FusedShared sh;
    const int C = a.C, c = (int)cl.block_rank();
    const int mv = blockIdx.x / C;
    const int N = a.N, R = a.R;                      // rows / owned columns per CTA
    const int m = mv / a.V;
    const int l = a.n_inline ? a.lsh_in[mv] : a.lsh[mv];
    double *xb = fsm;                                // [R]      gathered x of my rows
    double *recv = fsm + R;                          // [C][R]   partials of my columns from every CTA
    double *yp = recv + (size_t)C * R;               // [R]      previous y of my columns
    const int NP = (N + 3) & ~3;                     // row stride: 16-byte aligned rows for both dtypes
    // one-exchange form: [2][C][R] partials of my rows' x from every CTA in place of recv / yp
    const size_t head = (size_t)R * (a.one_x ? 2 * C + 1 : C + 2);
    T *slice = reinterpret_cast<T *>(fsm + ((head + 1) & ~(size_t)1));   // [R][NP] (a.resident)
    if (l < 0) {                                     // padding vector: nothing to solve
        if (c == 0 && threadIdx.x == 0) {
            SolveState st = {};
            st.l = -1;
            st.done = 1;
            a.st[mv] = st;
        }
        return;
    }
    const int r0 = c * R, r1 = min(N, r0 + R);
    const T *P = reinterpret_cast<const T *>(a.P) + (size_t)m * a.mstride;
    const int nrow = r1 - r0;
    // non-resident rows: the TMA ring (after the small buffers, where the resident slice would be)
    T *ring = slice;
    const uint32_t row_bytes = (uint32_t)(((size_t)N * sizeof(T) + 15) & ~(size_t)15);   // <= ld bytes
    int ring_rows = kRingBytes / (int)(NP * sizeof(T));
    ring_rows = ring_rows < 1 ? 1 : (ring_rows > 8 ? 8 : ring_rows);
    __shared__ uint64_t rbar[kRing];
    uint32_t q_issue = 0, q_cons = 0;
    const double *xrow = nullptr;
    if (!a.resident && !a.ldg && threadIdx.x == 0) {
        for (int i = 0; i < kRing; ++i) mbar_init(&rbar[i], 1);
        fence_mbar_init();
    }
    if (a.resident) {                                // my rows, once, by TMA bulk copies; then smem only
        __shared__ uint64_t bar;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_expect_tx(&bar, row_bytes * (uint32_t)nrow);
            for (int r = 0; r < nrow; ++r) bulk_g2s(slice + (size_t)r * NP, P + (size_t)(r0 + r) * a.ld, row_bytes, &bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
    }
    const double u = 1.0 / (double)N;
    for (int i = threadIdx.x; i < R; i += kFT) {
        xb[i] = r0 + i < N ? u : 0.0;                // gathered uniform vector
        yp[i] = c * R + i < N ? u : 0.0;
    }
    double s_prev = 1.0, dpart = 0.0, change = __longlong_as_double(0x7ff0000000000000ll);
    int k = 0, conv = 0;
    // p2p exchanges: every value another CTA delivers is an st.async whose bytes complete a phase of
    // my mbarrier xbar[0] (partials + change partials, A) or xbar[1] (y + sums, B); thread 0 arms each
    // phase with the bytes it will receive, everyone waits on its parity. Single buffers suffice: a
    // CTA only sends phase-A data of the next product after it has every CTA's phase-B data of this
    // one, which each sends after it has read its own buffers (and the same for phase B).
    __shared__ uint64_t xbar[2];
    const int ncols = min(N, (c + 1) * R) - c * R;           // my owned columns == my rows
    const uint32_t bytesA = 8u * (uint32_t)C * (uint32_t)(ncols + 1), bytesB = 8u * (uint32_t)(ncols + C);
    if ((a.p2p || a.one_x) && threadIdx.x == 0) {
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        fence_mbar_init();
    }
    cl.sync();
    // one product: acc[2 q + e] = partial y of column j = 2 t + 2 kFT q + e over my rows (x = xb)
    auto gemv = [&](double (&acc)[NC]) {
#pragma unroll
        for (int i = 0; i < NC; ++i) acc[i] = 0.0;
        // ---- A: partial y over my rows; column j = 2 t + 512 q + e. Resident rows: from shared
        // memory, RS rows per step. Otherwise rows stream through a 3-stage shared-memory ring filled by
        // TMA bulk copies (thread 0 issues, mbarrier complete_tx), so ~kRing x 64 KB are in flight.
        // from_global: read-only loads from L2 straight into registers (no shared-memory staging)
        // rows_c: rows whose loads are in flight together
        auto rows_fma = [&](auto from_global, auto rows_c, const T *base, int64_t rs, int n) {
            constexpr int RS = decltype(rows_c)::value;
            for (int r = 0; r < n; r += RS) {
                double xr[RS];
                double pv[RS][NC];
#pragma unroll
                for (int rr = 0; rr < RS; ++rr) {
                    const bool rin = r + rr < n;
                    xr[rr] = rin ? xrow[r + rr] : 0.0;
                    const T *row = base + (size_t)(rin ? r + rr : r) * rs;
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const int j = 2 * threadIdx.x + 2 * kFT * q;
                        pv[rr][2 * q] = pv[rr][2 * q + 1] = 0.0;
                        if (j < N) {
                            if constexpr (sizeof(T) == 8) {
                                const double2 v = decltype(from_global)::value
                                                      ? __ldg(reinterpret_cast<const double2 *>(row + j))
                                                      : *reinterpret_cast<const double2 *>(row + j);
                                pv[rr][2 * q] = v.x; pv[rr][2 * q + 1] = v.y;
                            } else {
                                const float2 v = decltype(from_global)::value
                                                     ? __ldg(reinterpret_cast<const float2 *>(row + j))
                                                     : *reinterpret_cast<const float2 *>(row + j);
                                pv[rr][2 * q] = v.x; pv[rr][2 * q + 1] = v.y;
                            }
                        }
                    }
                }
#pragma unroll
                for (int rr = 0; rr < RS; ++rr)
#pragma unroll
                    for (int i = 0; i < NC; ++i) acc[i] = fma(xr[rr], pv[rr][i], acc[i]);
            }
        };
        if (a.resident) {
            xrow = xb;
            rows_fma(std::false_type{}, std::integral_constant<int, RS>{}, slice, NP, nrow);
        } else if (a.ldg) {
            xrow = xb;
            rows_fma(std::true_type{}, std::integral_constant<int, RSG>{}, P + (size_t)r0 * a.ld, a.ld, nrow);
        } else {
            const int nst = (nrow + ring_rows - 1) / ring_rows;
            auto issue = [&](int st) {                 // thread 0: stage st into buffer q_issue % kRing
                const int rs0 = st * ring_rows;
                const int nr = min(ring_rows, nrow - rs0);
                const int buf = (int)(q_issue % kRing);
                mbar_expect_tx(&rbar[buf], row_bytes * (uint32_t)nr);
                for (int rr = 0; rr < nr; ++rr)
                    bulk_g2s(ring + ((size_t)buf * ring_rows + rr) * NP, P + (size_t)(r0 + rs0 + rr) * a.ld, row_bytes,
                             &rbar[buf]);
                ++q_issue;
            };
            if (threadIdx.x == 0)
                for (int st = 0; st < kRing - 1 && st < nst; ++st) issue(st);
            for (int st = 0; st < nst; ++st) {
                const int buf = (int)(q_cons % kRing);
                mbar_wait(&rbar[buf], (q_cons / kRing) & 1u);
                __syncthreads();                       // every thread is done with stage st - 1's buffer
                if (threadIdx.x == 0 && st + kRing - 1 < nst) issue(st + kRing - 1);
                xrow = xb + st * ring_rows;
                rows_fma(std::false_type{}, std::integral_constant<int, RS>{}, ring + (size_t)buf * ring_rows * NP, NP, min(ring_rows, nrow - st * ring_rows));
                ++q_cons;
            }
        }
    };

    if (a.one_x) {
        // One exchange per product (st.async + mbarrier, double-buffered by product parity b): every
        // CTA pushes its partial of column j straight to the CTA owning row r = (j + l) mod N (whose
        // next x_r is y_j, Theorem 2's gather), with its partial total (-> s) and its change partial of
        // the previous product. The owner sums the C partials of each row in CTA order. A CTA sends
        // product k + 2 into buffer b only after it has every CTA's product k + 1, which each sends
        // after reading its buffer b of product k, so two buffers suffice.
        double *rx = fsm + R;
        const uint32_t bytesX = 8u * ((uint32_t)C * (uint32_t)nrow + 2u * (uint32_t)C);
        for (;;) {
            double acc[NC];
            gemv(acc);
            double tp = 0.0;                            // (a pair's odd column may be row padding)
            const int b = k & 1;
            double *rb = rx + (size_t)b * C * R;
            if (threadIdx.x == 0) mbar_expect_tx(&xbar[b], bytesX);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 2 * threadIdx.x + 2 * kFT * q + e;
                    if (j < N) {
                        int r = j + l;
                        if (r >= N) r -= N;
                        const uint32_t ow = (uint32_t)(r / R);
                        st_async_f64(mapa_u32(smem_u32(rb + (size_t)c * R + (r - (int)ow * R)), ow), acc[2 * q + e],
                                     mapa_u32(smem_u32(&xbar[b]), ow));
                        tp += acc[2 * q + e];
                    }
                }
            }
            const double tot = fblock_sum(tp, sh.red);  // after the partials are on their way
            if (threadIdx.x < C) {
                const uint32_t bar = mapa_u32(smem_u32(&xbar[b]), threadIdx.x);
                st_async_f64(mapa_u32(smem_u32(&sh.tx[b][c]), threadIdx.x), tot, bar);
                st_async_f64(mapa_u32(smem_u32(&sh.dx[b][c]), threadIdx.x), dpart, bar);
            }
            mbar_wait(&xbar[b], (uint32_t)(k >> 1) & 1u);
            if (k > 0) {
                double t = 0.0;
                for (int cc = 0; cc < C; ++cc) t += sh.dx[b][cc];
                change = t;
                if (change < a.tol) { conv = 1; break; }
                if (k >= a.max_iter || !(s_prev > 0.0) || !isfinite(change)) break;
            }
            double s = 0.0;
            for (int cc = 0; cc < C; ++cc) s += sh.tx[b][cc];
            double d = 0.0;
            if ((int)threadIdx.x < nrow) {              // y of the column feeding my row, its change
                double yj = 0.0;
                for (int cc = 0; cc < C; ++cc) yj += rb[(size_t)cc * R + threadIdx.x];
                d = fabs(yj / s - xb[threadIdx.x] / s_prev);
                xb[threadIdx.x] = yj;
            }
            dpart = fblock_sum(d, sh.red);
            s_prev = s;
            ++k;
        }
        cl.sync();   // nothing is in flight to a CTA that exits
        const int o = a.n_inline ? a.oidx_in[mv] : a.out_idx[mv];
        if (o >= 0 && (int)threadIdx.x < nrow) {     // pi^k over the columns feeding my rows
            int j = r0 + (int)threadIdx.x - l;
            if (j < 0) j += N;
            a.pi[(size_t)o * N + j] = xb[threadIdx.x] / s_prev;
        }
    } else {
        for (;;) {
            double acc[NC];
            gemv(acc);
            // push partials to the owners of the columns: recv[c][j - owner R] in the owner's smem
            if (a.p2p) {
                if (threadIdx.x == 0) mbar_expect_tx(&xbar[0], bytesA);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = 2 * threadIdx.x + 2 * kFT * q + e;
                        if (j < N) {
                            const uint32_t ow = (uint32_t)(j / R);
                            st_async_f64(mapa_u32(smem_u32(recv + (size_t)c * R + (j - (int)ow * R)), ow), acc[2 * q + e],
                                         mapa_u32(smem_u32(&xbar[0]), ow));
                        }
                    }
                }
                if (threadIdx.x < C)
                    st_async_f64(mapa_u32(smem_u32(&sh.exA[kFMaxC + c]), threadIdx.x), dpart,
                                 mapa_u32(smem_u32(&xbar[0]), threadIdx.x));
                mbar_wait(&xbar[0], (uint32_t)k & 1u);
            } else {
#pragma unroll
                for (int q = 0; q < Q; ++q) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = 2 * threadIdx.x + 2 * kFT * q + e;
                        if (j < N) {
                            const int ow = j / R;
                            cl.map_shared_rank(recv, ow)[(size_t)c * R + (j - ow * R)] = acc[2 * q + e];
                        }
                    }
                }
                if (threadIdx.x < C) cl.map_shared_rank(sh.exA, threadIdx.x)[kFMaxC + c] = dpart;
                cl.sync();   // A
            }
            if (k > 0) {
                double t = 0.0;
                for (int cc = 0; cc < C; ++cc) t += sh.exA[kFMaxC + cc];
                change = t;
                if (change < a.tol) { conv = 1; break; }
                if (k >= a.max_iter || !(s_prev > 0.0) || !isfinite(change)) break;
            }
            // ---- B: owners add the partials (fixed order); push y to the x buffers; publish sum(y)
            double ys = 0.0, yj = 0.0;
            const int j = c * R + (int)threadIdx.x;
            const bool own = (int)threadIdx.x < R && j < N;
            if (a.p2p && threadIdx.x == 0) mbar_expect_tx(&xbar[1], bytesB);
            if (own) {
                for (int cc = 0; cc < C; ++cc) yj += recv[(size_t)cc * R + threadIdx.x];
                ys = yj;
                int r = j + l;
                if (r >= N) r -= N;
                const int ow = r / R;
                if (a.p2p)
                    st_async_f64(mapa_u32(smem_u32(xb + (r - ow * R)), (uint32_t)ow), yj,
                                 mapa_u32(smem_u32(&xbar[1]), (uint32_t)ow));
                else
                    cl.map_shared_rank(xb, ow)[r - ow * R] = yj;
            }
            ys = fblock_sum(ys, sh.red);
            if (a.p2p) {
                if (threadIdx.x < C)
                    st_async_f64(mapa_u32(smem_u32(&sh.exB[c]), threadIdx.x), ys, mapa_u32(smem_u32(&xbar[1]), threadIdx.x));
                mbar_wait(&xbar[1], (uint32_t)k & 1u);
            } else {
                if (threadIdx.x < C) cl.map_shared_rank(sh.exB, threadIdx.x)[c] = ys;
                cl.sync();   // B
            }
            double s = 0.0;
            for (int cc = 0; cc < C; ++cc) s += sh.exB[cc];
            // ---- C: L1 change of the normalised iterates over my columns
            double d = 0.0;
            if (own) {
                d = fabs(yj / s - yp[threadIdx.x] / s_prev);
                yp[threadIdx.x] = yj;
            }
            dpart = fblock_sum(d, sh.red);
            s_prev = s;
            ++k;
        }
        if (a.p2p) cl.sync();   // nothing is in flight to a CTA that exits (every phase was waited for)
        // pi^k = y / s over my columns
        const int o = a.n_inline ? a.oidx_in[mv] : a.out_idx[mv];
        if (o >= 0) {
            const int j = c * R + (int)threadIdx.x;
            if ((int)threadIdx.x < R && j < N) a.pi[(size_t)o * N + j] = yp[threadIdx.x] / s_prev;
        }
    }
    if (c == 0 && threadIdx.x == 0) {
        SolveState st;
        st.l = l;
        st.iters = k;
        st.done = 1;
        st.converged = conv;
        st.cur = 0;
        st.pad0 = st.pad1 = st.pad2 = 0;
        st.s = s_prev;
        st.change = change;
        a.st[mv] = st;
    }
}

}  // namespace

int fused_shape(int N, int *C, int *R) {
    if (N > kFMaxN) return 1;
    int c = (N + 31) / 32;
    if (c > kFMaxC) c = kFMaxC;
    if (c < 1) c = 1;
    int r = (N + c - 1) / c;
    if (r > kFT) return 1;
    *C = c;
    *R = r;
    return 0;
}

constexpr size_t kFResidentMax = 96 * 1024;   // largest row slice kept in shared memory

size_t fused_slice_bytes(int N, int R, int dtype) {
    return (size_t)R * ((N + 3) & ~3) * (dtype == SPLIDAR_F64 ? 8 : 4);
}
size_t fused_ring_bytes(int N, int dtype) {
    const size_t row = (size_t)((N + 3) & ~3) * (dtype == SPLIDAR_F64 ? 8 : 4);
    size_t rows = kRingBytes / row;
    rows = rows < 1 ? 1 : (rows > 8 ? 8 : rows);
    return kRing * rows * row;
}
size_t fused_smem(const FusedArgs &a, int dtype) {
    return sizeof(double) * (((size_t)a.R * (a.one_x ? 2 * a.C + 1 : a.C + 2) + 1) & ~(size_t)1) +
           (a.resident ? fused_slice_bytes(a.N, a.R, dtype) : a.ldg ? 0 : fused_ring_bytes(a.N, dtype));
}

template <typename T>
void *fused_fn_q(int N) {
    const int q = (N + 2 * kFT - 1) / (2 * kFT);
    if (q <= 1) return (void *)k_power_fused<T, 1>;
    if (q <= 2) return (void *)k_power_fused<T, 2>;
    return (void *)k_power_fused<T, 4>;
}

// the kernel instance for (dtype, N); its attributes are set once per device for all instances
// (thread-safe; never inside a captured launch)
cudaError_t fused_fn(int dtype, int N, void **fn) {
    const void *all[] = {(void *)k_power_fused<double, 1>, (void *)k_power_fused<double, 2>,
                         (void *)k_power_fused<double, 4>, (void *)k_power_fused<float, 1>,
                         (void *)k_power_fused<float, 2>, (void *)k_power_fused<float, 4>};
    for (const void *f : all) {
        const cudaError_t e = func_attrs_once(f, 220 * 1024, true);
        if (e != cudaSuccess) return e;
    }
    *fn = dtype == SPLIDAR_F64 ? fused_fn_q<double>(N) : fused_fn_q<float>(N);
    return cudaSuccess;
}

int fused_resident(int N, int R, int dtype) { return fused_slice_bytes(N, R, dtype) <= kFResidentMax; }

cudaError_t launch_fused(int dtype, const FusedArgs &a, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.M * a.V * a.C));
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = fused_smem(a, dtype);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL secondary of the build
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    void *fn = nullptr;
    cudaError_t e = fused_fn(dtype, a.N, &fn);
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<FusedArgs *>(&a)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace spl
