// Step 2 (K4): the normalised base matrix P~0 and step 3 materialised (K5): the row permutation.
//
// P~0[r][j] = lambda_j exp(F_r - F_j - Lambda [r > j]) / Z_r            (mode EXP)
//           = w_j (r > j ? e^{-Lambda} / D_r : 1 / D_r)                  (mode FACTORED)
// from E_base = exp.(-Lambda L - D), L_rj = 1{s_r > s_j}, D_rj = F(s_j) - F(s_r),
// P = (1 lambda^T) . E, row-normalised (§3.4).
//
// Layout: a CTA owns a 512-column strip and a chunk of rows; each thread owns 16 bytes of columns
// (2 fp64 or 4 fp32) for every row of the chunk, keeps its column vectors (w, w e^{-Lambda} or
// lambda, F) in registers and streams 128-bit stores down the rows. Per row it reads one
// broadcast scalar (1/D_r or 1/Z_r, F_r). The kernel is a pure HBM write stream: N^2 * b bytes.
#include "common.cuh"
#include "fixpt.cuh"
#include "ptx.cuh"

namespace spl {
namespace {

constexpr int kRowsPerCta = 32;

template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };

template <typename T, int MODE>
__global__ void __launch_bounds__(kStripCols / Vec16<T>::n)
k_build(const VecPtrs base, int64_t vstride, int N, T *__restrict__ P0, int64_t ld, int64_t mstride, int row0,
        int nrows, int rows_per_cta, double *__restrict__ colsum_part, const ColStats cst) {
    constexpr int VEC = Vec16<T>::n;
    using V = typename Vec16<T>::type;
    pdl_wait();        // PDL secondary of the flux-vector kernel (launch_build); no-op otherwise
    pdl_trigger();     // the consumer (fused solver / iteration graph) may be scheduled now
    const int m = blockIdx.z;
    const double *__restrict__ w = base.w + m * vstride;
    const double *__restrict__ lam = base.lam + m * vstride;
    const double *__restrict__ F = base.F + m * vstride;
    const double *__restrict__ invD = base.invD + m * vstride;
    const double *__restrict__ invZ = base.invZ + m * vstride;
    const double Lam = base.scal[m * 8 + 0];
    const double eL = base.scal[m * 8 + 1];
    T *__restrict__ out = P0 + m * mstride;

    const int j0 = blockIdx.x * kStripCols + threadIdx.x * VEC;
    if (j0 >= N) return;
    // rows [row0, row0 + nrows) of P~0 (a row shard); stored from row 0 of P0
    const int r0 = row0 + blockIdx.y * rows_per_cta;
    const int r1 = min(row0 + nrows, r0 + rows_per_cta);
    const bool full = j0 + VEC <= N;

    // column operands in registers
    double a[VEC], b[VEC];   // FACTORED: a = w_j;  EXP: a = lambda_j, b = F_j
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
        const int j = j0 + e;
        if (MODE == SPLIDAR_ENTRY_FACTORED) {
            a[e] = j < N ? w[j] : 0.0;
            b[e] = 0.0;
        } else {
            a[e] = j < N ? lam[j] : 0.0;
            b[e] = j < N ? F[j] : 0.0;
        }
    }

    double cs[VEC];              // column sums of the STORED entries over this CTA's rows (colsum_part)
    int emx[VEC], emn[VEC];      // largest / smallest exponent of a non-zero stored entry (cst: the int8
                                 // GEMV's range test; -1: a subnormal or negative entry)
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
        cs[e] = 0.0;
        emx[e] = 0;
        emn[e] = 1 << 20;
    }
    if (cst.emax_part && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *cst.flag = 1u;
    // encoded storage: entry -> scaled integer of its column (fixpt.cuh; launch_enc_colexp set E_j)
    bool enc = false;
    int base23[VEC];
    uint64_t csi[VEC];           // encoded storage: column sums of the stored integers (exact)
#pragma unroll
    for (int e = 0; e < VEC; ++e) csi[e] = 0;
    if constexpr (sizeof(T) == 4 && MODE == SPLIDAR_ENTRY_FACTORED) {
        enc = cst.enc && *cst.flag;
        if (enc) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) base23[e] = j0 + e < N ? cst.colexp[(size_t)m * N + j0 + e] - cst.R - 23 : 255;
        }
    }
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        T val[VEC];
        if (MODE == SPLIDAR_ENTRY_FACTORED) {
            // row multipliers 1/D_r (j >= r) and e^{-Lambda}/D_r (j < r): forming w_j e^{-Lambda} first
            // would underflow (~e^{-2 Lambda}) for Lambda > ~350, while e^{-Lambda}/D_r stays O(1)
            const double inv_hi = __ldg(invD + r);
            const double inv_lo = eL * inv_hi;
#pragma unroll
            for (int e = 0; e < VEC; ++e) val[e] = (T)(a[e] * (j0 + e < r ? inv_lo : inv_hi));
        } else {
            const double iz = __ldg(invZ + r);
            const double Fr = __ldg(F + r);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const double arg = Fr - b[e] - (j0 + e < r ? Lam : 0.0);   // in [-Lambda, 0]
                if constexpr (sizeof(T) == 8) {
                    val[e] = a[e] * exp(arg) * iz;
                } else {
                    // fp32 storage: ex2.approx on the fp64-formed exponent (|rel err| ~ 1e-6)
                    val[e] = (float)(a[e] * iz) * __expf((float)arg);
                }
            }
        }
        if (colsum_part && !enc) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) cs[e] += (double)val[e];
        }
        if (cst.emax_part) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                int ex;
                bool nz, bad;
                if constexpr (sizeof(T) == 4) {
                    const uint32_t u = __float_as_uint(val[e]);
                    ex = (int)((u >> 23) & 0xFF);
                    nz = (u & 0x7FFFFFFFu) != 0;
                    bad = (ex == 0 && nz) || (u >> 31);
                } else {
                    const uint64_t u = (uint64_t)__double_as_longlong(val[e]);
                    ex = (int)((u >> 52) & 0x7FF);
                    nz = (u & 0x7FFFFFFFFFFFFFFFull) != 0;
                    bad = (ex == 0 && nz) || (u >> 63);
                }
                if (nz) {
                    emx[e] = max(emx[e], ex);
                    emn[e] = min(emn[e], ex);
                }
                if (bad) emn[e] = -1;
            }
        }
        T *row = out + (int64_t)(r - row0) * ld + j0;
        if constexpr (sizeof(T) == 4 && MODE == SPLIDAR_ENTRY_FACTORED) {
            if (enc) {
                uint32_t wd[VEC];
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    wd[e] = fx32(__float_as_uint((float)val[e]), base23[e]);
                    csi[e] += wd[e];
                }
                if (full) {
                    *reinterpret_cast<uint4 *>(row) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e)
                        if (j0 + e < N) reinterpret_cast<uint32_t *>(row)[e] = wd[e];
                }
                continue;
            }
        }
        if (full) {
            V v;
            if constexpr (VEC == 2) { v.x = val[0]; v.y = val[1]; }
            else { v.x = val[0]; v.y = val[1]; v.z = val[2]; v.w = val[3]; }
            *reinterpret_cast<V *>(row) = v;
        } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e)
                if (j0 + e < N) row[e] = val[e];
        }
    }
    if (colsum_part) {           // [M][row chunk][N]: summed over the chunks in fixed order later
        double *cp = colsum_part + ((size_t)m * gridDim.y + blockIdx.y) * N;
        if (enc) {   // stored value = integer x 2^(base23 - 127) (fixpt.cuh); a chunk's sum < 2^53: exact
#pragma unroll
            for (int e = 0; e < VEC; ++e) cs[e] = ldexp((double)csi[e], base23[e] - 127);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (j0 + e < N) cp[j0 + e] = cs[e];
    }
    if (cst.emax_part) {
        const size_t o = ((size_t)m * gridDim.y + blockIdx.y) * N;
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (j0 + e < N) {
                cst.emax_part[o + j0 + e] = emx[e];
                cst.emin_part[o + j0 + e] = emn[e];
            }
    }
}

// colsum[m][j] = sum over the row chunks (fixed order) of the build's partial column sums.
// With cst: E_j (the column's largest exponent; all-zero columns get the largest representable, so
// every shift of the int8 GEMV is negative) and the range test of the int8 GEMV (power_i8.cu): clear
// *cst.flag if a non-zero entry lies more than 2^R below its column maximum, the maximum is <= R, or an
// entry is subnormal / negative. The same test as k_i8_colexp / k_i8_colcheck, from the build's
// registers instead of a second read of the matrix.
__global__ void __launch_bounds__(256) k_colsum_reduce(const double *__restrict__ part, int nch, int N, int M,
                                                       double *__restrict__ colsum, const ColStats cst) {
    const int m = blockIdx.y;
    bool bad = false;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        double t = 0.0;
#pragma unroll 8
        for (int c = 0; c < nch; ++c) t += __ldcg(part + ((size_t)m * nch + c) * N + j);   // loads in flight, fixed-order adds
        colsum[(size_t)m * N + j] = t;
        if (cst.emax_part) {
            int mx = 0, mn = 1 << 20;
            for (int c = 0; c < nch; ++c) {
                const size_t o = ((size_t)m * nch + c) * N + j;
                mx = max(mx, cst.emax_part[o]);
                mn = min(mn, cst.emin_part[o]);
            }
            const bool any = mn < (1 << 20);
            cst.colexp[(size_t)m * N + j] = any ? mx : cst.zero_col_exp;
            bad |= mn < 0 || (any && (mx - mn > cst.R || mx <= cst.R));
        }
    }
    if (cst.emax_part && __syncthreads_or(bad) && threadIdx.x == 0) atomicAnd(cst.flag, 0u);
}

// Column exponents for encoded storage, before the build writes anything. Factored entries are
// P~0[r][j] = fl32(w_j * h_r) with h_r = 1/D_r for r <= j and fl(e^{-Lambda} / D_r) for r > j (k_build),
// and fl(w * x) is non-decreasing in x, so column j's largest / smallest entries are w_j times the
// extremes of 1/D over r <= j (prefix) and e^{-Lambda} times those over r > j (suffix). Grid
// (column blocks of 1024, matrices); a thread per column. Every CTA first reduces the extremes of all
// blocks (one warp per block, coalesced: the 1/D vector is L2-resident), then a warp-shuffle scan plus
// the warp and block totals give its columns the inclusive prefix and exclusive suffix extremes. The
// range test is k_i8_colcheck's (a column fails if its smallest entry is not a normal fp32 number, lies
// more than 2^R below the largest, or the largest exponent is <= R); an all-zero column (w_j = 0) gets
// E_j = 255. Each CTA writes whether one of its columns failed; k_enc_flag folds those into the flag.
constexpr int kEncBlock = 1024;
constexpr int kEncMaxBlocks = 128;        // N <= 131072

__global__ void __launch_bounds__(kEncBlock) k_enc_colexp(const VecPtrs base, int64_t vstride, int N, int R,
                                                          int *__restrict__ colexp, int *__restrict__ bad_out) {
    __shared__ double s_bmx[kEncMaxBlocks], s_bmn[kEncMaxBlocks], s_wmx[32], s_wmn[32];
    const int m = blockIdx.y, nb = gridDim.x, bk = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    const double *__restrict__ invD = base.invD + m * vstride;
    const double *__restrict__ w = base.w + m * vstride;
    const double eL = base.scal[m * 8 + 1];
    for (int b2 = wp; b2 < nb; b2 += kEncBlock / 32) {          // extremes of every block
        double mx = 0.0, mn = INFINITY;
        const int jend = min(N, (b2 + 1) * kEncBlock);
#pragma unroll 8
        for (int j = b2 * kEncBlock + lane; j < jend; j += 32) {    // 8 loads in flight per lane
            const double h = invD[j];
            mx = fmax(mx, h);
            mn = fmin(mn, h);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (lane == 0) { s_bmx[b2] = mx; s_bmn[b2] = mn; }
    }
    const int j = bk * kEncBlock + t;
    const double h = j < N ? invD[j] : 0.0;
    double pmx = h, pmn = j < N ? h : INFINITY, smx = pmx, smn = pmn;   // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xffffffffu, pmx, o), b2 = __shfl_up_sync(0xffffffffu, pmn, o);
        const double c = __shfl_down_sync(0xffffffffu, smx, o), d = __shfl_down_sync(0xffffffffu, smn, o);
        if (lane >= o) { pmx = fmax(pmx, a); pmn = fmin(pmn, b2); }
        if (lane + o < 32) { smx = fmax(smx, c); smn = fmin(smn, d); }
    }
    if (lane == 31) { s_wmx[wp] = pmx; s_wmn[wp] = pmn; }       // warp totals
    double xsmx = __shfl_down_sync(0xffffffffu, smx, 1), xsmn = __shfl_down_sync(0xffffffffu, smn, 1);
    if (lane == 31) { xsmx = 0.0; xsmn = INFINITY; }            // exclusive suffix within the warp
    __syncthreads();
    for (int k = 0; k < 32; ++k) {
        if (k < wp) { pmx = fmax(pmx, s_wmx[k]); pmn = fmin(pmn, s_wmn[k]); }
        if (k > wp) { xsmx = fmax(xsmx, s_wmx[k]); xsmn = fmin(xsmn, s_wmn[k]); }
    }
    for (int k = 0; k < nb; ++k) {
        if (k < bk) { pmx = fmax(pmx, s_bmx[k]); pmn = fmin(pmn, s_bmn[k]); }
        if (k > bk) { xsmx = fmax(xsmx, s_bmx[k]); xsmn = fmin(xsmn, s_bmn[k]); }
    }
    bool bad = false;
    if (j < N) {
        float vmx = (float)(w[j] * pmx), vmn = (float)(w[j] * pmn);    // rows r <= j
        if (j + 1 < N) {                                                 // rows r > j
            vmx = fmaxf(vmx, (float)(w[j] * (eL * xsmx)));
            vmn = fminf(vmn, (float)(w[j] * (eL * xsmn)));
        }
        const uint32_t ux = __float_as_uint(vmx), un = __float_as_uint(vmn);
        const int ex = (int)(ux >> 23), en = (int)(un >> 23);           // biased exponents (entries >= 0)
        if (ux == 0u && un == 0u) {
            colexp[(size_t)m * N + j] = 255;                             // all-zero column
        } else {
            bad = !(en >= 1 && ex <= 254 && ex - en <= R && ex > R);     // +0 / subnormal / inf / NaN fail
            colexp[(size_t)m * N + j] = ex;
        }
    }
    bad = __syncthreads_or(bad);
    if (t == 0) bad_out[m * nb + bk] = bad ? 1 : 0;
}

// flag = no CTA of k_enc_colexp saw a failing column.
__global__ void k_enc_flag(const int *__restrict__ bad, int n, unsigned *__restrict__ flag) {
    int any = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) any |= bad[i];
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) *flag = any ? 0u : 1u;
}

// P[i][:] = P0[(i + l) mod N][:] (Thm 2; J_l), 16-byte vectors, one row per CTA row.
__global__ void __launch_bounds__(256) k_apply_deadtime(const uint4 *__restrict__ P0, uint4 *__restrict__ P,
                                                        int N, int64_t ld_vec, int row_vecs, int l) {
    const int i = blockIdx.x;
    const int src = (int)(((int64_t)i + l) % N);
    const uint4 *s = P0 + (int64_t)src * ld_vec;
    uint4 *d = P + (int64_t)i * ld_vec;
#pragma unroll 4
    for (int c = threadIdx.x; c < row_vecs; c += blockDim.x) d[c] = __ldcs(s + c);
}

}  // namespace

int colsum_chunks(int N) { return N / kRowsPerCta < kColsumChunks ? (N + kRowsPerCta - 1) / kRowsPerCta : kColsumChunks; }

cudaError_t launch_build(const VecPtrs base, int64_t vstride, int M, int N, int dtype, int mode,
                         void *P0, int64_t ld, int64_t mstride, cudaStream_t s, int row0, int nrows,
                         double *colsum_part, double *colsum, ColStats cst) {
    if (nrows < 0) nrows = N;
    // with column sums: at most kColsumChunks row chunks per matrix (deterministic fixed-order sum);
    // without: chunks of 32 rows, or fewer rows per CTA when that leaves the grid below two CTAs per
    // SM (small N: c1's N = 256 was 8 CTAs of 32 rows)
    int nch = colsum_part ? colsum_chunks(nrows) : (nrows + kRowsPerCta - 1) / kRowsPerCta;
    if (!colsum_part) {
        const int strips = (N + kStripCols - 1) / kStripCols;
        const int want = (2 * device_sm_count() + strips * M - 1) / (strips * M);
        if (nch < want) nch = want < nrows ? want : nrows;
    }
    const int rpc = (nrows + nch - 1) / nch;
    dim3 grid((N + kStripCols - 1) / kStripCols, nch, M);
    // a PDL secondary of the kernel before it on s (k_build waits for it before any global access)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kStripCols / (dtype == SPLIDAR_F64 ? 2 : 4));
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e;
    if (dtype == SPLIDAR_F64) {
        if (mode == SPLIDAR_ENTRY_EXP)
            e = cudaLaunchKernelEx(&cfg, k_build<double, SPLIDAR_ENTRY_EXP>, base, vstride, N, (double *)P0, ld, mstride, row0, nrows, rpc, colsum_part, cst);
        else
            e = cudaLaunchKernelEx(&cfg, k_build<double, SPLIDAR_ENTRY_FACTORED>, base, vstride, N, (double *)P0, ld, mstride, row0, nrows, rpc, colsum_part, cst);
    } else {
        if (mode == SPLIDAR_ENTRY_EXP)
            e = cudaLaunchKernelEx(&cfg, k_build<float, SPLIDAR_ENTRY_EXP>, base, vstride, N, (float *)P0, ld, mstride, row0, nrows, rpc, colsum_part, cst);
        else
            e = cudaLaunchKernelEx(&cfg, k_build<float, SPLIDAR_ENTRY_FACTORED>, base, vstride, N, (float *)P0, ld, mstride, row0, nrows, rpc, colsum_part, cst);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess && colsum_part) {
        k_colsum_reduce<<<dim3((N + 255) / 256 < 64 ? (N + 255) / 256 : 64, M), 256, 0, s>>>(colsum_part, nch, N, M,
                                                                                          colsum, cst);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_enc_colexp(const VecPtrs base, int64_t vstride, int M, int N, int *colexp, int *scratch,
                              unsigned *flag, cudaStream_t s) {
    const int nb = (N + kEncBlock - 1) / kEncBlock;
    if (nb > kEncMaxBlocks) return cudaErrorInvalidValue;
    k_enc_colexp<<<dim3(nb, M), kEncBlock, 0, s>>>(base, vstride, N, 8, colexp, scratch);
    k_enc_flag<<<1, 256, 0, s>>>(scratch, nb * M, flag);
    return cudaGetLastError();
}

cudaError_t launch_apply_deadtime(const void *P0, void *P, int N, int64_t ld, int dtype, int l,
                                  cudaStream_t s) {
    const int esz = dtype == SPLIDAR_F64 ? 8 : 4;
    const int64_t ld_vec = ld * esz / 16;
    const int row_vecs = (int)(((int64_t)N * esz + 15) / 16);
    k_apply_deadtime<<<N, 256, 0, s>>>((const uint4 *)P0, (uint4 *)P, N, ld_vec, row_vecs, l);
    return cudaGetLastError();
}

}  // namespace spl
