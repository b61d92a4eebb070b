// Step 4's GEMV on the 5th-generation tensor cores: y_v = x_v^T P~0 for up to 18 dead times,
// computed EXACTLY in integers (an Ozaki-style split) on tcgen05.mma kind::i8 with TMEM
// accumulators, instead of on the FP64 tensor cores (DMMA), whose rate -- not HBM -- bounds the
// multi-vector pass (17 FMAs per 4- or 8-byte entry).
//
// Split (per plan launch, per matrix):
//   column scale   E_j = the largest biased exponent in column j of P~0 (k_i8_colexp). If every
//                  non-zero entry of the column lies within 2^R of it (R = 8 for fp32, 11 for fp64
//                  storage), a_rj 2^(BIAS + MBITS + R - E_j) is an integer of <= 32 (fp32) / 64
//                  (fp64) bits, i.e. NP = 4 / 8 unsigned bytes A_p (A_0 most significant):
//                    a~_rj = sum_p A_p[r][j] 2^(8 (NP - 1 - p))                      (exact)
//   vector scale   tau_v = 55 - floor(log2(max_r x_v[r])): x~_v[r] = floor(x_v[r] 2^tau_v) < 2^56,
//                  7 bytes X_q (q = 0 most significant), truncation error < 2^-56 max_r x_v[r]
//   product        sum_r x~ a~ = sum_{p,q} D_pq 2^(8 (NP - 1 - p) + 8 (6 - q)),
//                  D_pq[v][j] = sum_r X_q[v][r] A_p[r][j]   (u8 x u8 -> s32 on the tensor core: exact)
//   y_v[j]       = 2^(E_j - BIAS - MBITS - R - tau_v) sum_{p,q} ...   (fp64, fixed order)
// If any column of any matrix fails the range test the plan's WHILE body runs the DMMA kernel
// instead (both kernels are in the body; each returns at once when the flag says it is not the one).
//
// k_power_step_i8<T>: persistent, one CTA per SM (TMEM: NP x TN = 512 columns). Work units are
// (active matrix, column tile of TN = 128 (fp32) / 64 (fp64) columns, k-block of 64 rows), split
// into equal contiguous ranges (stream-K). Warp roles:
//   warp 3      TMA producer: the unit's 64 x 512-byte tile of P~0 as 4 tensor-map boxes of 64 rows
//               x 128 B (cp.async.bulk.tensor, 128-byte swizzle) into a 3-stage ring;
//   warp 0      x-slice producer: the unit's 8 KB image (written by k_power_check) with one
//               cp.async.bulk into the MMA buffer, once the MMA has freed it (3 buffers);
//   warp 1      MMA issuer (one thread): per unit 2 k-steps x 2 tcgen05.mma of M = 128 rows (q, v)
//               of x slices, N = 256 bytes of scaled integers (64 fp32 / 32 fp64 columns, byte n =
//               W j + p of column j's word), K = 32; D in TMEM column (W j + p) of the tile;
//   warp 2      TMEM allocator;
//   warps 4-11  converters: each unit's tile -> its scaled integers in the canonical MN-major layout
//               (the tensor core reads every byte as its own u8 column: no transposes); shared-memory bandwidth (TMA write, converter read and
//               write, MMA operand reads: ~152 KB per 32 KB unit) is the budget the layout is cut
//               for -- N = 256 MMAs read the x slices once per 2 (fp32) / 4 (fp64) planes. At the
//               end of a piece the epilogue:
//               TMEM -> registers (tcgen05.ld), sum over p and q in fp64, per-piece partial sums;
//               the last piece of a tile adds the pieces in fixed order (deterministic), writes y,
//               the tile's sum and max of y (the next x scale).
// k_power_step_i8e: fp32 matrices a building plan stored already ENCODED (each entry its scaled
// integer; build.cu): the TMA boxes are the MMA's B operand as they land, so it has no converters
// (4 stages of tile + x image, the same MMA issue and epilogue).
#include <climits>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "fixpt.cuh"
#include "ptx.cuh"
#include "tc05.cuh"

namespace spl {
namespace {

constexpr int kI8Threads = 384;          // 12 warps
constexpr int kI8Conv0 = 4;              // first converter warp
constexpr int kI8ConvThreads = 256;      // 8 converter warps
constexpr int kKB = 64;                  // rows per unit
constexpr int kRowBytes = 512;           // bytes of a row segment per unit (128 fp32 / 64 fp64)
constexpr int kSBuf = 3;                 // slice + x buffers between the converters and the MMA
constexpr int kSBytes = kKB * kRowBytes;     // byte planes of one unit: NP x 64 x TN = 32 KB
constexpr int kXBytes = 128 * kKB;           // x-slice image of one unit: 8 KB
constexpr int kXQ = 7;                       // x slices

template <typename T> struct I8Cfg;
template <> struct I8Cfg<float> {
    static constexpr int NP = 4, TN = 128, R = 8, BIAS_MBITS = 150;
};
template <> struct I8Cfg<double> {
    static constexpr int NP = 8, TN = 64, R = 11, BIAS_MBITS = 1075;
};

constexpr int kEStages = 4;              // encoded-storage kernel: TMA stages (tile + x image)

struct __align__(8) I8Bars {
    uint64_t a_full[kEStages], a_empty[kEStages];
    uint64_t s_full[kSBuf], x_full[kSBuf], s_empty[kSBuf];
    uint64_t t_full, t_empty;
};

constexpr size_t kI8Smem = 1024 + 3 * 32768 + kSBuf * (size_t)kSBytes + kSBuf * (size_t)kXBytes + 1024;


__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Walks the units (active matrix ai, column tile c, k-block kb) of a CTA's range without divisions.
struct UnitCursor {
    int64_t g;     // ai * tiles + c
    int kb, ai, c;
    __device__ __forceinline__ UnitCursor(int64_t u, int kbs, int tiles) {
        g = u / kbs;
        kb = (int)(u - g * kbs);
        ai = (int)(g / tiles);
        c = (int)(g - (int64_t)ai * tiles);
    }
    __device__ __forceinline__ void next(int kbs, int tiles) {
        if (++kb == kbs) {
            kb = 0;
            ++g;
            if (++c == tiles) { c = 0; ++ai; }
        }
    }
};
// ring slot / phase of a k-stage ring, advanced once per unit
template <int K>
struct Ring {
    int i = 0;
    uint32_t ph = 0;
    __device__ __forceinline__ void next() {
        if (++i == K) { i = 0; ph ^= 1u; }
    }
};

// Byte image of a unit (the MMA's B operand, MN-major SWIZZLE_NONE) in the "word layout": B column
// n = W j + p is byte p (little-endian) of column j's scaled integer, so a row of B is the row of
// scaled integers as they sit in memory. Core matrices of 8 rows x 16 bytes:
//   offset(r, n) = (r / 8) * 4096 + (n / 16) * 128 + (r % 8) * 16 + n % 16,
// LBO (next 8 rows) = 4096 B, SBO (next 16 bytes of n) = 128 B; one MMA with N = 256 spans 64 fp32 /
// 32 fp64 columns (their accumulators are adjacent in TMEM).
constexpr int kKGroup = 4096;

// The unit's tile arrives in shared memory as 4 tensor-map boxes of [64 rows][128 B] with the
// 128-byte swizzle (the 16-byte chunk c of row r sits at chunk c ^ (r % 8), so the 8 rows of one
// core matrix read their chunks from 8 different bank groups). Converter item = (row r, 16-column
// block jb): 16 entries -> NP plane rows of 16 bytes (one 16-byte store each; the 8 rows of a
// core matrix are 8 consecutive lanes: conflict-free).
constexpr int kBoxBytes = kKB * 128;
constexpr int kAStages = 3;
constexpr int kABytes = 4 * kBoxBytes;       // 32 KB
constexpr int kEStaging = 2 * 16 * 129 * 8 + 1024;   // the epilogue's staging (stage[2][16][129] doubles)
constexpr size_t kI8eSmem = 1024 + kEStages * (size_t)(kABytes + kXBytes) + kEStaging + 1024;

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

template <typename T>
__device__ __forceinline__ void convert_item(const unsigned char *tile, unsigned char *sw_img, int r, int jb,
                                             const int (&base)[16]) {
    // the 16 scaled integers of row r, columns 16 jb .. 16 jb + 15, little-endian, as they are:
    // byte n = sizeof(T) j + p of the MMA's B row is byte p of column j (4 / 8 core-matrix rows of
    // 16 bytes; the 8 rows r % 8 of one core matrix are 8 consecutive lanes: conflict-free stores)
    constexpr int W = sizeof(T);                     // bytes (planes) per entry
    unsigned char *dst = sw_img + (r >> 3) * kKGroup + jb * W * 128 + (r & 7) * 16;
    const int sw = r & 7;
    if constexpr (sizeof(T) == 4) {
        // columns 16 jb .. 16 jb + 15: box jb / 2, chunks 4 (jb % 2) .. + 3
        const unsigned char *row = tile + (jb >> 1) * kBoxBytes + r * 128;
        const int c0 = (jb & 1) * 4;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + (((c0 + g) ^ sw) << 4));
            *reinterpret_cast<uint4 *>(dst + g * 128) =
                make_uint4(fx32(v.x, base[4 * g]), fx32(v.y, base[4 * g + 1]), fx32(v.z, base[4 * g + 2]),
                           fx32(v.w, base[4 * g + 3]));
        }
    } else {
        // columns 16 jb .. 16 jb + 15: box jb, chunks 0 .. 7 (2 entries each)
        const unsigned char *row = tile + jb * kBoxBytes + r * 128;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + ((g ^ sw) << 4));
            uint4 o;
            fx64(v.x, v.y, base[2 * g], o.x, o.y);
            fx64(v.z, v.w, base[2 * g + 1], o.z, o.w);
            *reinterpret_cast<uint4 *>(dst + g * 128) = o;
        }
    }
}

struct PieceCtx {
    int m, c;
    int64_t g;
};

// Epilogue of a piece (matrix m, tile c): TMEM -> fp64 partial sums of y per running vector; the
// last piece of the tile adds the pieces in fixed order (deterministic), writes y and the tile's
// sum and maximum of y. Executed by the 256 converter threads.
template <typename T>
__device__ __forceinline__ void epilogue(const PowerArgs &a, const PieceCtx &pc, uint32_t tmem, unsigned char *sS,
                                         I8Bars *bars, int piece, int64_t U, int b, int *s_vmap, int *s_cur,
                                         int *s_tau, int *s_nact, int *s_last) {
    using C = I8Cfg<T>;
    constexpr int NP = C::NP, TN = C::TN;
    const int ct = threadIdx.x - kI8Conv0 * 32, cw = ct >> 5, lane = threadIdx.x & 31;
    const int N = a.N, kbs = N / kKB, VP = a.V, m = pc.m, c = pc.c;
    const int64_t g = pc.g;
    if (ct == 0) {
        int n = 0;
        for (int v = 0; v < VP; ++v) {
            const SolveState st = a.st[(size_t)m * VP + v];
            if (!st.done) { s_vmap[n] = v; s_cur[n] = st.cur; ++n; }
            s_tau[v] = a.xtau[(size_t)m * VP + v];
        }
        *s_nact = n;
    }
    mbar_wait(&bars->t_full, piece & 1);
    tc05::fence_after();
    named_sync(1, kI8ConvThreads);
    const int quad = cw & 3, half = cw >> 2;
    const int row = 32 * quad + lane;                       // TMEM lane = x-slice row (q, v)
    const int q = row / VP;
    const bool live = q < kXQ;
    double *stage = reinterpret_cast<double *>(sS);         // [2 halves][16 cols][SROW]
    constexpr int CW = 16;                                  // columns per chunk
    constexpr int SROW = 129;   // odd row stride: the q-sum below reads 16 columns at once, conflict-free
    constexpr int CHUNKS = TN / 2 / CW;                     // chunks per warp (its half of the tile)
    const int64_t gN = g * kbs;
    double *part = a.part + (size_t)(b + g) * VP * TN;
    const int nact = *s_nact;
    for (int ch = 0; ch < CHUNKS; ++ch) {
        const int col0 = half * (TN / 2) + ch * CW;
        // D column n = NP j + p holds byte p (weight 2^(8 p)) of column j's scaled integers
        double acc[CW];
        const double wq = ldexp(1.0, 8 * (kXQ - 1 - (live ? q : 0)));
#pragma unroll
        for (int c4 = 0; c4 < CW * NP / 16; ++c4) {
            uint32_t r[16];
            tc05::ld32x16(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(NP * col0 + 16 * c4), r);
            tc05::wait_ld();
            // D is read as UNSIGNED: every product is >= 0 and a column's sum over <= 66048 rows is
            // < 2^32 (i8_supported bounds N), so the s32 accumulator's wrap-around is exact mod 2^32
#pragma unroll
            for (int e = 0; e < 16 / NP; ++e) {
                double t;
                if constexpr (NP == 4) {     // fp32: sum_p D_p 2^(8p) < 2^56, exact in 64-bit integers
                    const uint64_t t64 = (uint64_t)r[e * 4] + ((uint64_t)r[e * 4 + 1] << 8) +
                                         ((uint64_t)r[e * 4 + 2] << 16) + ((uint64_t)r[e * 4 + 3] << 24);
                    t = (double)t64;
                } else {                     // fp64: 8 planes (up to 2^88): fp64, most significant last
                    t = 0.0;
#pragma unroll
                    for (int p = NP - 1; p >= 0; --p) t = fma((double)r[e * NP + p], ldexp(1.0, 8 * p), t);
                }
                acc[c4 * (16 / NP) + e] = t * wq;
            }
        }
        double *st = stage + (size_t)half * CW * SROW;
#pragma unroll
        for (int i = 0; i < CW; ++i) st[i * SROW + row] = live ? acc[i] : 0.0;
        named_sync(2 + half, 128);
        // y partial for (v, col0 + i): sum over q (fixed order, largest slice first)
        const int t = ct & 127;
        for (int o = t; o < nact * CW; o += 128) {
            const int sl = o / CW, i = o % CW;
            const int v = s_vmap[sl];
            double ysum = 0.0;
#pragma unroll
            for (int qq = 0; qq < kXQ; ++qq) ysum += st[i * SROW + qq * VP + v];
            const int j = c * TN + col0 + i;
            const int ex = a.colexp[(size_t)m * N + j] - C::BIAS_MBITS - C::R - s_tau[v];
            // ysum 2^ex: a multiply by the exact power of two (same rounding as ldexp) when 2^ex is normal
            part[(size_t)v * TN + col0 + i] =
                ex >= -1022 && ex <= 1023 ? ysum * __longlong_as_double((long long)(ex + 1023) << 52) : ldexp(ysum, ex);
        }
        named_sync(2 + half, 128);
    }
    tc05::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->t_empty);
    // ---- last piece of the tile: add the pieces in fixed order, write y, tile sum / max ----
    __threadfence();
    named_sync(1, kI8ConvThreads);
    const int first_p = (int)(gN / U), last_p = (int)((gN + kbs - 1) / U);
    if (ct == 0) {
        const unsigned prev = atomicAdd(&a.strip_cnt[g], 1u);
        *s_last = prev == (unsigned)(last_p - first_p);
    }
    named_sync(1, kI8ConvThreads);
    if (*s_last) {
        __threadfence();
        double *red = reinterpret_cast<double *>(sS);                  // [8 warps][2][32] (stage is free)
        for (int sl = 0; sl < nact; ++sl) {
            const int v = s_vmap[sl];
            double ysum = 0.0, ymax = 0.0;
            if (ct < TN) {
                double yv = 0.0;
                for (int pcs = first_p; pcs <= last_p; ++pcs)
                    yv += __ldcg(a.part + ((size_t)(pcs + g) * VP + v) * TN + ct);
                a.y[(((size_t)m * VP + v) * 2 + (1 - s_cur[sl])) * N + (size_t)c * TN + ct] = yv;
                ysum = yv;
                ymax = yv;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ysum += __shfl_xor_sync(0xffffffffu, ysum, o);
                ymax = fmax(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
            }
            if (lane == 0) {
                red[(cw * 2 + 0) * kMaxVectors + sl] = ysum;
                red[(cw * 2 + 1) * kMaxVectors + sl] = ymax;
            }
        }
        named_sync(1, kI8ConvThreads);
        if (ct < nact) {
            double ssum = 0.0, smax = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                ssum += red[(w * 2 + 0) * kMaxVectors + ct];
                smax = fmax(smax, red[(w * 2 + 1) * kMaxVectors + ct]);
            }
            const size_t mv = (size_t)m * VP + s_vmap[ct];
            a.ssum[mv * a.strips_i8 + c] = ssum;
            a.smax[mv * a.strips_i8 + c] = smax;
        }
        if (ct == 0) a.strip_cnt[g] = 0u;
    }
    named_sync(1, kI8ConvThreads);
}

template <typename T>
__global__ void __launch_bounds__(kI8Threads, 1) k_power_step_i8(const PowerArgs a, const __grid_constant__ CUtensorMap tmap) {
    using C = I8Cfg<T>;
    constexpr int NP = C::NP, TN = C::TN;
    if (!a.glob[3]) return;                             // range test failed: the DMMA kernel runs
    const int N = a.N;
    const int tiles = N / TN, kbs = N / kKB;
    const int n_act = a.i8_dbg ? a.M : (int)a.glob[2];      // timing experiments: every matrix, always
    const int64_t T_units = (int64_t)n_act * tiles * kbs;
    if (T_units == 0) return;
    const int G = gridDim.x, b = blockIdx.x;
    int64_t U = (T_units + G - 1) / G;
    if (U < 2) U = 2;
    const int64_t u_begin = (int64_t)b * U;
    if (u_begin >= T_units) return;
    const int64_t u_end = u_begin + U < T_units ? u_begin + U : T_units;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char *sA = smem;                                       // [3][4 boxes][64][128]
    unsigned char *sS = sA + kAStages * kABytes;                    // [kSBuf][64 rows x NP planes x TN]
    unsigned char *sX = sS + kSBuf * kSBytes;                       // [kSBuf][8 KB]
    I8Bars *bars = reinterpret_cast<I8Bars *>(sX + kSBuf * kXBytes);
    __shared__ uint32_t s_tmem;
    __shared__ int s_vmap[kMaxVectors], s_cur[kMaxVectors], s_tau[kMaxVectors], s_nact, s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&bars->a_full[i], 1);
            mbar_init(&bars->a_empty[i], 8);
        }
        for (int i = 0; i < kSBuf; ++i) {
            mbar_init(&bars->s_full[i], 8);
            mbar_init(&bars->x_full[i], 1);
            mbar_init(&bars->s_empty[i], 1);
        }
        mbar_init(&bars->t_full, 1);
        mbar_init(&bars->t_empty, 8);
        fence_mbar_init();
    }
    if (warp == 2) tc05::alloc<512>(&s_tmem);
    if (threadIdx.x == 0) ktime_start(a.ktime);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 3) {
        // ------------------------------------------------------------------ TMA producer of P~0 tiles
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kAStages> ra;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), ra.next()) {
                const int m = a.i8_dbg ? cu.ai : a.act[cu.ai];
                mbar_wait(&bars->a_empty[ra.i], ra.ph ^ 1);
                mbar_expect_tx(&bars->a_full[ra.i], kABytes);
                unsigned char *dst = sA + ra.i * kABytes;
                constexpr int BOXC = 128 / sizeof(T);      // columns per box
#pragma unroll
                for (int bx = 0; bx < 4; ++bx)
                    tma_load_3d(dst + bx * kBoxBytes, &tmap, cu.c * TN + bx * BOXC, cu.kb * kKB, m, &bars->a_full[ra.i]);
            }
        }
    } else if (warp == 0) {
        // ------------------------------------------------------------------ x-slice producer
        if (lane == 0) {
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kSBuf> rb;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), rb.next()) {
                const int m = a.i8_dbg ? cu.ai : a.act[cu.ai];
                mbar_wait(&bars->s_empty[rb.i], rb.ph ^ 1);
                mbar_expect_tx(&bars->x_full[rb.i], kXBytes);
                bulk_g2s(sX + rb.i * kXBytes, a.ximg + ((size_t)m * kbs + cu.kb) * kXBytes, kXBytes, &bars->x_full[rb.i]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc05::idesc_i8(128, 256, true);
            const uint32_t sS_u = smem_u32(sS), sX_u = smem_u32(sX);
            int piece = 0;
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kSBuf> rb;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), rb.next()) {
                const bool first = u == u_begin || cu.kb == 0;
                const bool last = u + 1 == u_end || cu.kb + 1 == kbs;
                const int sb = rb.i;
                if (first) {
                    mbar_wait(&bars->t_empty, (piece & 1) ^ 1);
                    tc05::fence_after();
                }
                mbar_wait(&bars->x_full[sb], rb.ph);
                mbar_wait(&bars->s_full[sb], rb.ph);
                tc05::fence_after();
                // per k-step of 32 rows, NP * TN / 256 = 2 MMAs of N = 256 (2 fp32 / 4 fp64 planes each)
#pragma unroll
                for (int h = 0; h < NP * TN / 256; ++h) {
                    if (a.i8_dbg & 2) break;
#pragma unroll
                    for (int s = 0; s < kKB / 32; ++s) {
                        const uint64_t ad = tc05::smem_desc(sX_u + sb * kXBytes + s * 256, 128, 512);
                        const uint64_t bd = tc05::smem_desc(sS_u + sb * kSBytes + s * 4 * kKGroup + h * 256 / 16 * 128,
                                                            kKGroup, 128);
                        tc05::mma_i8(tmem + (uint32_t)(h * 256), ad, bd, idesc, (first && s == 0) ? 0u : 1u);
                    }
                }
                tc05::commit(&bars->s_empty[sb]);
                if (last) {
                    tc05::commit(&bars->t_full);
                    ++piece;
                }
            }
        }
    } else if (warp >= kI8Conv0) {
        // ------------------------------------------------------------------ converters + epilogue
        const int ct = threadIdx.x - kI8Conv0 * 32;                // 0..255
        constexpr int JB = TN / 16;                                 // 16-column blocks per row
        constexpr int ITEMS = kKB * JB / kI8ConvThreads;            // 2 (fp32) / 1 (fp64)
        const int jb = (ct >> 3) % JB;
        int base[16];
        int piece = 0;
        UnitCursor cc(u_begin, kbs, tiles);
        Ring<kAStages> ra;
        Ring<kSBuf> rb;
        for (int64_t u = u_begin; u < u_end; ++u, cc.next(kbs, tiles), ra.next(), rb.next()) {
            const int m = a.i8_dbg ? cc.ai : a.act[cc.ai];
            const bool last = u + 1 == u_end || cc.kb + 1 == kbs;
            if (u == u_begin || cc.kb == 0) {                       // new piece: column bases
                const int4 *E = reinterpret_cast<const int4 *>(a.colexp + (size_t)m * N + (size_t)cc.c * TN + jb * 16);
                constexpr int OFF = C::R + (sizeof(T) == 4 ? 23 : 0);   // fp32 funnel: s = e - E + R + 23
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int4 e4 = E[i];
                    base[4 * i] = e4.x - OFF;
                    base[4 * i + 1] = e4.y - OFF;
                    base[4 * i + 2] = e4.z - OFF;
                    base[4 * i + 3] = e4.w - OFF;
                }
            }
            mbar_wait(&bars->a_full[ra.i], ra.ph);
            mbar_wait(&bars->s_empty[rb.i], rb.ph ^ 1);
            const unsigned char *At = sA + ra.i * kABytes;
#pragma unroll
            for (int h = 0; h < ITEMS; ++h) {
                if (a.i8_dbg & 1) break;
                const int it = ct + kI8ConvThreads * h;
                const int r = (it & 7) + 8 * (it / (8 * JB));
                convert_item<T>(At, sS + rb.i * kSBytes, r, jb, base);
            }
            tc05::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bars->a_empty[ra.i]);
                mbar_arrive(&bars->s_full[rb.i]);
            }
            if (last) {
                const PieceCtx pc{m, cc.c, cc.g};
                epilogue<T>(a, pc, tmem, sS, bars, piece, U, b, s_vmap, s_cur, s_tau, &s_nact, &s_last);
                ++piece;
            }
        }
    }
    tc05::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) ktime_end(a.ktime);
    if (warp == 2) {
        tc05::fence_after();
        tc05::dealloc<512>(tmem);
    }
}

// k_power_step_i8e: the same GEMV for a matrix a building plan stored ENCODED (build.cu, fp32 storage
// with every column in range): each 4-byte entry already holds its scaled integer a~_rj (fixpt.cuh),
// so the TMA boxes of a unit ARE the MMA's B operand -- MN-major with the 128-byte swizzle the tensor
// map applies (CuTe's canonical ((T,8,m),(8,k)):((1,T,LBO),(8T,SBO)) layout: LBO = the next 128-byte
// column span = the next box, SBO = the next 8 rows = 1024 B; tools/probe/umma_sw128_probe.cu). No
// converters: per unit the producer loads the tile and the x-slice image into one of 4 stages, the MMA
// issuer consumes it, and the epilogue is the converter kernel's. Warps 4-11 only run the epilogue.
__global__ void __launch_bounds__(kI8Threads, 1) k_power_step_i8e(const PowerArgs a, const __grid_constant__ CUtensorMap tmap) {
    using T = float;
    using C = I8Cfg<T>;
    constexpr int NP = C::NP, TN = C::TN;
    if (!a.glob[3]) return;                             // range test failed: stored as fp32, DMMA runs
    const int N = a.N;
    const int tiles = N / TN, kbs = N / kKB;
    const int n_act = a.i8_dbg ? a.M : (int)a.glob[2];
    const int64_t T_units = (int64_t)n_act * tiles * kbs;
    if (T_units == 0) return;
    const int G = gridDim.x, b = blockIdx.x;
    int64_t U = (T_units + G - 1) / G;
    if (U < 2) U = 2;
    const int64_t u_begin = (int64_t)b * U;
    if (u_begin >= T_units) return;
    const int64_t u_end = u_begin + U < T_units ? u_begin + U : T_units;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char *sA = smem;                                       // [4][4 boxes][64][128]
    unsigned char *sX = sA + kEStages * kABytes;                    // [4][8 KB]
    unsigned char *sS = sX + kEStages * kXBytes;                    // epilogue staging
    I8Bars *bars = reinterpret_cast<I8Bars *>(sS + kEStaging);
    __shared__ uint32_t s_tmem;
    __shared__ int s_vmap[kMaxVectors], s_cur[kMaxVectors], s_tau[kMaxVectors], s_nact, s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kEStages; ++i) {
            mbar_init(&bars->a_full[i], 1);
            mbar_init(&bars->a_empty[i], 1);
        }
        mbar_init(&bars->t_full, 1);
        mbar_init(&bars->t_empty, 8);
        fence_mbar_init();
    }
    if (warp == 2) tc05::alloc<512>(&s_tmem);
    if (threadIdx.x == 0) ktime_start(a.ktime);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 3) {
        // ------------------------------------------------------------------ TMA producer (tile + x)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kEStages> ra;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), ra.next()) {
                const int m = a.i8_dbg ? cu.ai : a.act[cu.ai];
                mbar_wait(&bars->a_empty[ra.i], ra.ph ^ 1);
                mbar_expect_tx(&bars->a_full[ra.i], kABytes + kXBytes);
                unsigned char *dst = sA + ra.i * kABytes;
#pragma unroll
                for (int bx = 0; bx < 4; ++bx)
                    tma_load_3d(dst + bx * kBoxBytes, &tmap, cu.c * TN + bx * 32, cu.kb * kKB, m, &bars->a_full[ra.i]);
                bulk_g2s(sX + ra.i * kXBytes, a.ximg + ((size_t)m * kbs + cu.kb) * kXBytes, kXBytes, &bars->a_full[ra.i]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc05::idesc_i8(128, 256, true);
            const uint32_t sA_u = smem_u32(sA), sX_u = smem_u32(sX);
            int piece = 0;
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kEStages> ra;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), ra.next()) {
                const bool first = u == u_begin || cu.kb == 0;
                const bool last = u + 1 == u_end || cu.kb + 1 == kbs;
                if (first) {
                    mbar_wait(&bars->t_empty, (piece & 1) ^ 1);
                    tc05::fence_after();
                }
                mbar_wait(&bars->a_full[ra.i], ra.ph);
                tc05::fence_after();
                // per k-step of 32 rows, 2 MMAs of N = 256 bytes (64 columns = boxes 2h, 2h + 1)
#pragma unroll
                for (int h = 0; h < NP * TN / 256; ++h) {
                    if (a.i8_dbg & 2) break;
#pragma unroll
                    for (int s = 0; s < kKB / 32; ++s) {
                        const uint64_t ad = tc05::smem_desc(sX_u + ra.i * kXBytes + s * 256, 128, 512);
                        const uint64_t bd = tc05::smem_desc(sA_u + ra.i * kABytes + 2 * h * kBoxBytes + s * 32 * 128,
                                                            kBoxBytes, 1024) | (2ull << 61);   // SWIZZLE_128B
                        tc05::mma_i8(tmem + (uint32_t)(h * 256), ad, bd, idesc, (first && s == 0) ? 0u : 1u);
                    }
                }
                tc05::commit(&bars->a_empty[ra.i]);
                if (last) {
                    tc05::commit(&bars->t_full);
                    ++piece;
                }
            }
        }
    } else if (warp >= kI8Conv0) {
        // ------------------------------------------------------------------ epilogue
        int piece = 0;
        UnitCursor cc(u_begin, kbs, tiles);
        for (int64_t u = u_begin; u < u_end; ++u, cc.next(kbs, tiles)) {
            if (u + 1 == u_end || cc.kb + 1 == kbs) {
                const int m = a.i8_dbg ? cc.ai : a.act[cc.ai];
                const PieceCtx pc{m, cc.c, cc.g};
                epilogue<T>(a, pc, tmem, sS, bars, piece, U, b, s_vmap, s_cur, s_tau, &s_nact, &s_last);
                ++piece;
            }
        }
    }
    tc05::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) ktime_end(a.ktime);
    if (warp == 2) {
        tc05::fence_after();
        tc05::dealloc<512>(tmem);
    }
}

// Column exponents E_j (largest biased exponent of column j) and the range test, in three steps:
// k_i8_prep (flag = 1, E_j = 0, e_min_j = INT_MAX), k_i8_colexp (a CTA per 128 columns x a chunk of
// rows: one warp reads 512 B / 1 KB of a row, every lane 4 consecutive columns; atomicMax / atomicMin
// per column), k_i8_colcheck (per column: the range test clears glob[3] when some non-zero entry
// lies more than 2^R below its column maximum, or the maximum itself is <= R; all-zero columns get
// E_j = the largest exponent so that every shift is negative). Subnormal or negative entries clear
// the flag in k_i8_colexp.
template <typename T>
__global__ void __launch_bounds__(256) k_i8_colexp(const PowerArgs a, int rows_per_cta) {
    const int N = a.N, m = blockIdx.z;
    const int j0 = blockIdx.x * 128 + (threadIdx.x & 31) * 4;
    const int r0 = blockIdx.y * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
    const int w = threadIdx.x >> 5;
    int emax[4] = {0, 0, 0, 0}, emin[4] = {1 << 20, 1 << 20, 1 << 20, 1 << 20};
    bool bad = false;
    const T *P = reinterpret_cast<const T *>(a.P) + (size_t)m * a.mstride + j0;
#pragma unroll 4
    for (int r = r0 + w; r < r1; r += 8) {
        if constexpr (sizeof(T) == 4) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(P + (size_t)r * a.ld));
            const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = (int)((x[i] >> 23) & 0xFF);
                bad |= (e == 0 && (x[i] & 0x7FFFFFu)) || (x[i] >> 31);      // subnormal or negative
                if (x[i] & 0x7FFFFFFFu) { emax[i] = max(emax[i], e); emin[i] = min(emin[i], e); }
            }
        } else {
            const uint4 v0 = __ldcs(reinterpret_cast<const uint4 *>(P + (size_t)r * a.ld));
            const uint4 v1 = __ldcs(reinterpret_cast<const uint4 *>(P + (size_t)r * a.ld + 2));
            const uint64_t x[4] = {((uint64_t)v0.y << 32) | v0.x, ((uint64_t)v0.w << 32) | v0.z,
                                   ((uint64_t)v1.y << 32) | v1.x, ((uint64_t)v1.w << 32) | v1.z};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = (int)((x[i] >> 52) & 0x7FF);
                bad |= (e == 0 && (x[i] & 0xFFFFFFFFFFFFFull)) || (x[i] >> 63);
                if (x[i] & 0x7FFFFFFFFFFFFFFFull) { emax[i] = max(emax[i], e); emin[i] = min(emin[i], e); }
            }
        }
    }
    __shared__ int s_max[8][128], s_min[8][128];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        s_max[w][(threadIdx.x & 31) * 4 + i] = emax[i];
        s_min[w][(threadIdx.x & 31) * 4 + i] = emin[i];
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAnd(&a.glob[3], 0u);
    if (threadIdx.x < 128) {
        int mx = 0, mn = 1 << 20;
#pragma unroll
        for (int k = 0; k < 8; ++k) { mx = max(mx, s_max[k][threadIdx.x]); mn = min(mn, s_min[k][threadIdx.x]); }
        const size_t j = (size_t)m * N + blockIdx.x * 128 + threadIdx.x;
        if (mx > 0) atomicMax(&a.colexp[j], mx);
        if (mn < (1 << 20)) atomicMin(&a.colmin[j], mn);
    }
}

template <typename T>
__global__ void k_i8_colcheck(const PowerArgs a) {
    using C = I8Cfg<T>;
    const size_t n = (size_t)a.M * a.N;
    bool bad = false;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const int mx = a.colexp[j], mn = a.colmin[j];
        if (mn == INT_MAX) a.colexp[j] = sizeof(T) == 4 ? 255 : 2047;   // all-zero column
        else bad |= mx - mn > C::R || mx <= C::R;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAnd(&a.glob[3], 0u);
}

__global__ void k_i8_prep(const PowerArgs a) {
    const size_t n = (size_t)a.M * a.N;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        a.colexp[j] = 0;
        a.colmin[j] = INT_MAX;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.glob[3] = 1u;
}


}  // namespace

// Host side: the i8 kernels of a plan (nullptr when the plan cannot use them).
int i8_supported(int dtype, const PowerArgs &a) {
    const int TN = dtype == SPLIDAR_F64 ? I8Cfg<double>::TN : I8Cfg<float>::TN;
    // N <= 66048: a column's u8 x u8 sum over N rows stays below 2^32 (the accumulator read unsigned)
    return a.V >= 8 && 7 * a.V <= 128 && a.N % 128 == 0 && a.N % TN == 0 && a.N >= 1024 && a.N <= 66048;
}

// Tensor map of the stored matrices: dims {N columns, N rows, M matrices}, strides {ld, mstride}
// elements; boxes of 128 B x 64 rows x 1 matrix with the 128-byte swizzle.
static cudaError_t make_tmap(CUtensorMap *map, int dtype, const PowerArgs &a) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const bool f64 = dtype == SPLIDAR_F64;
    const size_t esz = f64 ? 8 : 4;
    const cuuint64_t dims[3] = {(cuuint64_t)a.N, (cuuint64_t)a.N, (cuuint64_t)a.M};
    const cuuint64_t strides[2] = {(cuuint64_t)a.ld * esz, (cuuint64_t)(a.M > 1 ? a.mstride : (int64_t)a.N * a.ld) * esz};
    const cuuint32_t box[3] = {(cuuint32_t)(128 / esz), (cuuint32_t)kKB, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                              const_cast<void *>(a.P), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t i8_kernels(int dtype, I8Kernels *k, const PowerArgs &a) {
    const bool f64 = dtype == SPLIDAR_F64;
    cudaError_t e = make_tmap(reinterpret_cast<CUtensorMap *>(k->tmap), dtype, a);
    if (e != cudaSuccess) return e;
    k->step_fn = f64 ? (void *)k_power_step_i8<double> : (void *)k_power_step_i8<float>;
    k->colexp_fn = f64 ? (void *)k_i8_colexp<double> : (void *)k_i8_colexp<float>;
    k->check_fn = f64 ? (void *)k_i8_colcheck<double> : (void *)k_i8_colcheck<float>;
    k->prep_fn = (void *)k_i8_prep;
    k->step_smem = kI8Smem;
    k->step_enc_fn = f64 ? nullptr : (void *)k_power_step_i8e;
    k->step_enc_smem = kI8eSmem;
    k->step_block = dim3(kI8Threads);
    const int sms = device_sm_count() < kMaxSMs ? device_sm_count() : kMaxSMs;
    k->step_grid = dim3(sms);
    // colexp: column tiles x row chunks, about 8 CTAs per SM in all
    const int ct = a.N / 128;
    int rc = (8 * sms + ct * a.M - 1) / (ct * a.M);
    rc = rc < 1 ? 1 : (rc > a.N / 8 ? a.N / 8 : rc);
    k->rows_per_cta = (a.N + rc - 1) / rc;
    k->colexp_grid = dim3(ct, rc, a.M);
    k->colexp_block = dim3(256);
    k->small_grid = dim3(2 * sms);
    e = func_attrs_once(k->step_fn, (int)kI8Smem, false);
    if (e == cudaSuccess && k->step_enc_fn) e = func_attrs_once(k->step_enc_fn, (int)kI8eSmem, false);
    return e;
}

int i8_range_bits(int dtype) { return dtype == SPLIDAR_F64 ? I8Cfg<double>::R : I8Cfg<float>::R; }

int i8_tile_cols(int dtype) { return dtype == SPLIDAR_F64 ? I8Cfg<double>::TN : I8Cfg<float>::TN; }

}  // namespace spl
