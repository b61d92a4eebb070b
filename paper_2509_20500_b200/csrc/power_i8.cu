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
//   warp 0      TMA producer: the unit's 64 x 512-byte tile of P~0 as 4 tensor-map boxes of 64 rows
//               x 128 B (cp.async.bulk.tensor, 128-byte swizzle) into a 3-stage ring, and its 8 KB
//               x-slice image (written by k_power_check, cp.async.bulk) into the MMA buffer;
//   warp 1      MMA issuer (one thread): per unit 2 k-steps x NP tcgen05.mma (M = 128 rows
//               (q, v) of x slices, N = TN columns, K = 32), D_p in TMEM columns [p TN, (p+1) TN);
//   warp 2      TMEM allocator;
//   warps 4-11  converters: each unit's fp32/fp64 tile -> NP byte planes in the canonical MN-major
//               layout (byte transposes with PRMT), then at the end of a piece the epilogue:
//               TMEM -> registers (tcgen05.ld), sum over p and q in fp64, per-piece partial sums;
//               the last piece of a tile adds the pieces in fixed order (deterministic), writes y,
//               the tile's sum and max of y (the next x scale).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tc05.cuh"

namespace spl {
namespace {

constexpr int kI8Threads = 384;          // 12 warps
constexpr int kI8Conv0 = 4;              // first converter warp
constexpr int kI8ConvThreads = 256;      // 8 converter warps
constexpr int kKB = 64;                  // rows per unit
constexpr int kRowBytes = 512;           // bytes of a row segment per unit (128 fp32 / 64 fp64)
constexpr int kBoxBytes = kKB * 128;     // one tensor-map box: 64 rows x 128 B (128-byte swizzle)
constexpr int kAStages = 3;
constexpr int kABytes = kKB * kRowBytes;     // 4 boxes = 32 KB
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

struct __align__(8) I8Bars {
    uint64_t a_full[kAStages], a_empty[kAStages];
    uint64_t s_full[2], x_full[2], s_empty[2];
    uint64_t t_full, t_empty;
};

constexpr size_t kI8Smem = 1024 + (size_t)kAStages * kABytes + 2 * (size_t)kSBytes + 2 * (size_t)kXBytes + 1024;

// 2-D / 3-D tensor-map copy global -> shared (box at coordinates {c0 elements, c1 rows, c2 matrix}).
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}
// 4 x 32-bit words -> 4 byte planes: out[k] = byte k of (w0, w1, w2, w3) (w0 in the low byte)
__device__ __forceinline__ void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
    const uint32_t t0 = prmt(w0, w1, 0x5140), t1 = prmt(w2, w3, 0x5140);   // b0: w0 w1 | b1: w0 w1
    const uint32_t t2 = prmt(w0, w1, 0x7362), t3 = prmt(w2, w3, 0x7362);   // b2 | b3
    o[0] = prmt(t0, t1, 0x5410);
    o[1] = prmt(t0, t1, 0x7632);
    o[2] = prmt(t2, t3, 0x5410);
    o[3] = prmt(t2, t3, 0x7632);
}

// Scaled integer of one entry: mantissa << (e - base); zero stays zero (the range test guarantees
// 0 <= e - base <= R for every non-zero entry when the plan runs this kernel).
// PTX shl clamps the shift amount to the register width, so a zero entry (e = 0, shift e - base
// < 0, i.e. huge as unsigned) gives 0 without a select; k_i8_colexp guarantees base > 0 for every
// column with a non-zero entry and sets E_j = 255 / 2047 (base > 0 as well) for all-zero columns.
__device__ __forceinline__ uint32_t fx32(uint32_t u, int base) {
    const uint32_t m = (u & 0x7FFFFFu) | 0x800000u;
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(m), "r"((uint32_t)((int)(u >> 23) - base)));
    return r;
}
__device__ __forceinline__ uint64_t fx64(uint64_t u, int base) {
    const uint64_t m = (u & 0xFFFFFFFFFFFFFull) | (1ull << 52);
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(m), "r"((uint32_t)((int)(u >> 52) - base)));
    return r;
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

// Byte-plane image of a unit: plane p at p * (64 TN); within a plane the MN-major canonical
// layout: (r / 8) * (TN / 16) * 128 + (j / 16) * 128 + (r % 8) * 16 + j % 16.
// The unit's tile in shared memory is 4 boxes of [64 rows][128 B] with the 128-byte swizzle: the
// 16-byte chunk c of row r sits at chunk c ^ (r % 8) (so the 8 rows of one core matrix read
// their chunks from 8 different bank groups).
template <typename T>
__device__ __forceinline__ void convert_item(const unsigned char *tile, unsigned char *splanes, int r, int jb,
                                             const int (&base)[16]) {
    using C = I8Cfg<T>;
    constexpr int PLANE = kKB * C::TN;
    unsigned char *dst = splanes + (r >> 3) * (C::TN / 16) * 128 + jb * 128 + (r & 7) * 16;
    const int sw = r & 7;
    if constexpr (sizeof(T) == 4) {
        // columns 16 jb .. 16 jb + 15: box jb / 2, chunks 4 (jb % 2) .. + 3
        const unsigned char *row = tile + (jb >> 1) * kBoxBytes + r * 128;
        const int c0 = (jb & 1) * 4;
        uint32_t pw[4][4];                              // [plane byte k][word g]
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + (((c0 + g) ^ sw) << 4));
            uint32_t o[4];
            transpose4(fx32(v.x, base[4 * g]), fx32(v.y, base[4 * g + 1]), fx32(v.z, base[4 * g + 2]),
                       fx32(v.w, base[4 * g + 3]), o);
#pragma unroll
            for (int k = 0; k < 4; ++k) pw[k][g] = o[k];
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)                    // plane p = byte 3 - p
            *reinterpret_cast<uint4 *>(dst + p * PLANE) = make_uint4(pw[3 - p][0], pw[3 - p][1], pw[3 - p][2], pw[3 - p][3]);
    } else {
        // columns 16 jb .. 16 jb + 15: box jb, chunks 0 .. 7
        const unsigned char *row = tile + jb * kBoxBytes + r * 128;
        uint32_t pw[8][4];                              // [byte k][word g]
#pragma unroll
        for (int g = 0; g < 4; ++g) {                   // 4 entries per word group
            const uint4 v0 = *reinterpret_cast<const uint4 *>(row + (((2 * g) ^ sw) << 4));
            const uint4 v1 = *reinterpret_cast<const uint4 *>(row + (((2 * g + 1) ^ sw) << 4));
            const uint64_t e0 = fx64(((uint64_t)v0.y << 32) | v0.x, base[4 * g]);
            const uint64_t e1 = fx64(((uint64_t)v0.w << 32) | v0.z, base[4 * g + 1]);
            const uint64_t e2 = fx64(((uint64_t)v1.y << 32) | v1.x, base[4 * g + 2]);
            const uint64_t e3 = fx64(((uint64_t)v1.w << 32) | v1.z, base[4 * g + 3]);
            uint32_t lo[4], hi[4];
            transpose4((uint32_t)e0, (uint32_t)e1, (uint32_t)e2, (uint32_t)e3, lo);
            transpose4((uint32_t)(e0 >> 32), (uint32_t)(e1 >> 32), (uint32_t)(e2 >> 32), (uint32_t)(e3 >> 32), hi);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                pw[k][g] = lo[k];
                pw[4 + k][g] = hi[k];
            }
        }
#pragma unroll
        for (int p = 0; p < 8; ++p)                    // plane p = byte 7 - p
            *reinterpret_cast<uint4 *>(dst + p * PLANE) = make_uint4(pw[7 - p][0], pw[7 - p][1], pw[7 - p][2], pw[7 - p][3]);
    }
}

template <typename T>
__global__ void __launch_bounds__(kI8Threads, 1) k_power_step_i8(const PowerArgs a, const __grid_constant__ CUtensorMap tmap) {
    using C = I8Cfg<T>;
    constexpr int NP = C::NP, TN = C::TN;
    if (!a.glob[3]) return;                             // range test failed: the DMMA kernel runs
    const int N = a.N;
    const int tiles = N / TN, kbs = N / kKB;
    const int n_act = (int)a.glob[2];
    const int64_t T_units = (int64_t)n_act * tiles * kbs;
    if (T_units == 0) return;
    const int G = gridDim.x, b = blockIdx.x;
    int64_t U = (T_units + G - 1) / G;
    if (U < 2) U = 2;
    const int64_t u_begin = (int64_t)b * U;
    if (u_begin >= T_units) return;
    const int64_t u_end = u_begin + U < T_units ? u_begin + U : T_units;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);   // swizzle atoms: 1 KB aligned
    unsigned char *sA = smem;                                       // [3][4 boxes][64][128]
    unsigned char *sS = sA + kAStages * kABytes;                    // [2][NP planes][64 x TN]
    unsigned char *sX = sS + 2 * kSBytes;                           // [2][8 KB]
    I8Bars *bars = reinterpret_cast<I8Bars *>(sX + 2 * kXBytes);
    __shared__ uint32_t s_tmem;
    __shared__ int s_vmap[kMaxVectors], s_cur[kMaxVectors], s_tau[kMaxVectors], s_nact, s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&bars->a_full[i], 1);
            mbar_init(&bars->a_empty[i], 8);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 8);
            mbar_init(&bars->x_full[i], 1);
            mbar_init(&bars->s_empty[i], 1);
        }
        mbar_init(&bars->t_full, 1);
        mbar_init(&bars->t_empty, 8);
        fence_mbar_init();
    }
    if (warp == 2) tc05::alloc<512>(&s_tmem);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<kAStages> ra;
            Ring<2> rb;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), ra.next(), rb.next()) {
                const int m = a.act[cu.ai];
                mbar_wait(&bars->a_empty[ra.i], ra.ph ^ 1);
                mbar_expect_tx(&bars->a_full[ra.i], kABytes);
                unsigned char *dst = sA + ra.i * kABytes;
                constexpr int BOXC = 128 / sizeof(T);      // columns per box
#pragma unroll
                for (int bx = 0; bx < 4; ++bx)
                    tma_load_3d(dst + bx * kBoxBytes, &tmap, cu.c * TN + bx * BOXC, cu.kb * kKB, m, &bars->a_full[ra.i]);
                mbar_wait(&bars->s_empty[rb.i], rb.ph ^ 1);
                mbar_expect_tx(&bars->x_full[rb.i], kXBytes);
                bulk_g2s(sX + rb.i * kXBytes, a.ximg + ((size_t)m * kbs + cu.kb) * kXBytes, kXBytes, &bars->x_full[rb.i]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc05::idesc_i8(128, TN, true);
            const uint32_t sS_u = smem_u32(sS), sX_u = smem_u32(sX);
            int piece = 0;
            UnitCursor cu(u_begin, kbs, tiles);
            Ring<2> rb;
            for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), rb.next()) {
                const bool first = u == u_begin || cu.kb == 0;
                const bool last = u + 1 == u_end || cu.kb + 1 == kbs;
                const int sb = rb.i;
                const uint32_t ph = rb.ph;
                if (first) {
                    mbar_wait(&bars->t_empty, (piece & 1) ^ 1);
                    tc05::fence_after();
                }
                mbar_wait(&bars->x_full[sb], ph);
                mbar_wait(&bars->s_full[sb], ph);
                tc05::fence_after();
#pragma unroll
                for (int s = 0; s < kKB / 32; ++s) {
                    const uint64_t ad = tc05::smem_desc(sX_u + sb * kXBytes + s * 256, 128, 512);
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        const uint64_t bd = tc05::smem_desc(sS_u + sb * kSBytes + p * (kKB * TN) + s * 4 * (TN / 16) * 128,
                                                            (TN / 16) * 128, 128);
                        tc05::mma_i8(tmem + (uint32_t)(p * TN), ad, bd, idesc, (first && s == 0) ? 0u : 1u);
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
        const int cw = ct >> 5;                                     // converter warp 0..7
        constexpr int JB = TN / 16;                                 // 16-column blocks per row
        constexpr int ITEMS = kKB * JB / kI8ConvThreads;            // 2 (fp32) / 1 (fp64)
        const int jb = (ct >> 3) % JB;
        int base[16];
        int piece = 0;
        const int VP = a.V;
        UnitCursor cu(u_begin, kbs, tiles);
        Ring<kAStages> ra;
        Ring<2> rb;
        for (int64_t u = u_begin; u < u_end; ++u, cu.next(kbs, tiles), ra.next(), rb.next()) {
            const int64_t g = cu.g;
            const int c = cu.c;
            const int m = a.act[cu.ai];
            const bool last = u + 1 == u_end || cu.kb + 1 == kbs;
            if (u == u_begin || cu.kb == 0) {                       // new piece: column bases
                const int4 *E = reinterpret_cast<const int4 *>(a.colexp + (size_t)m * N + (size_t)c * TN + jb * 16);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int4 e4 = E[i];
                    base[4 * i] = e4.x - C::R;
                    base[4 * i + 1] = e4.y - C::R;
                    base[4 * i + 2] = e4.z - C::R;
                    base[4 * i + 3] = e4.w - C::R;
                }
            }
            const int sa = ra.i, sb = rb.i;
            mbar_wait(&bars->a_full[sa], ra.ph);
            mbar_wait(&bars->s_empty[sb], rb.ph ^ 1);
            const unsigned char *At = sA + sa * kABytes;
#pragma unroll
            for (int h = 0; h < ITEMS; ++h) {
                const int it = ct + kI8ConvThreads * h;
                const int r = (it & 7) + 8 * (it / (8 * JB));
                convert_item<T>(At, sS + sb * kSBytes, r, jb, base);
            }
            tc05::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bars->a_empty[sa]);
                mbar_arrive(&bars->s_full[sb]);
            }
            if (!last) continue;

            // ---- epilogue of the piece (matrix m, tile c): TMEM -> fp64 partial sums ----------
            if (ct == 0) {
                int n = 0;
                for (int v = 0; v < VP; ++v) {
                    const SolveState s = a.st[(size_t)m * VP + v];
                    if (!s.done) { s_vmap[n] = v; s_cur[n] = s.cur; ++n; }
                    s_tau[v] = a.xtau[(size_t)m * VP + v];
                }
                s_nact = n;
            }
            mbar_wait(&bars->t_full, piece & 1);
            tc05::fence_after();
            named_sync(1, kI8ConvThreads);
            const int quad = cw & 3, half = cw >> 2;
            const int row = 32 * quad + lane;                       // TMEM lane = x-slice row (q, v)
            const int q = row / VP;
            const bool live = q < kXQ;
            double *stage = reinterpret_cast<double *>(sS);         // [2 halves][32 cols][128 rows]
            constexpr int CHUNKS = TN / 64;                         // 32-column chunks per warp
            const int64_t gN = g * kbs;
            double *part = a.part + (size_t)(b + g) * VP * TN;
            for (int ch = 0; ch < CHUNKS; ++ch) {
                const int col0 = half * (TN / 2) + ch * 32;
                double acc[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] = 0.0;
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    uint32_t r[32];
                    tc05::ld32x32(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(p * TN + col0), r);
                    tc05::wait_ld();
                    const double w = ldexp(1.0, 8 * (NP - 1 - p) + 8 * (kXQ - 1 - (live ? q : 0)));
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = fma((double)(int)r[i], w, acc[i]);
                }
                double *st = stage + (size_t)half * 32 * 128;
#pragma unroll
                for (int i = 0; i < 32; ++i) st[i * 128 + row] = live ? acc[i] : 0.0;
                named_sync(2 + half, 128);
                // y partial for (v, col0 + i): sum over q (fixed order, largest slice first)
                const int t = ct & 127;
                for (int o = t; o < s_nact * 32; o += 128) {
                    const int sl = o >> 5, i = o & 31;
                    const int v = s_vmap[sl];
                    double ysum = 0.0;
#pragma unroll
                    for (int qq = 0; qq < kXQ; ++qq) ysum += st[i * 128 + qq * VP + v];
                    const int j = c * TN + col0 + i;
                    const int ex = a.colexp[(size_t)m * N + j] - C::BIAS_MBITS - C::R - s_tau[v];
                    part[(size_t)v * TN + col0 + i] = ldexp(ysum, ex);
                }
                named_sync(2 + half, 128);
            }
            tc05::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->t_empty);
            ++piece;
            // ---- last piece of the tile: add the pieces in fixed order, write y, tile sum / max --
            __threadfence();
            named_sync(1, kI8ConvThreads);
            if (ct == 0) {
                const int first_p = (int)(gN / U), last_p = (int)((gN + kbs - 1) / U);
                const unsigned prev = atomicAdd(&a.strip_cnt[g], 1u);
                s_last = prev == (unsigned)(last_p - first_p);
            }
            named_sync(1, kI8ConvThreads);
            if (s_last) {
                __threadfence();
                const int first_p = (int)(gN / U), last_p = (int)((gN + kbs - 1) / U);
                double *red = reinterpret_cast<double *>(sS);                  // [8 warps][2][32] (stage is free)
                for (int sl = 0; sl < s_nact; ++sl) {
                    const int v = s_vmap[sl];
                    double ysum = 0.0, ymax = 0.0;
                    if (ct < TN) {
                        double yv = 0.0;
                        for (int pc = first_p; pc <= last_p; ++pc)
                            yv += __ldcg(a.part + ((size_t)(pc + g) * VP + v) * TN + ct);
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
                if (ct < s_nact) {
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
    }
    tc05::fence_before();
    __syncthreads();
    if (warp == 2) {
        tc05::fence_after();
        tc05::dealloc<512>(tmem);
    }
}

// Column exponents E_j (largest biased exponent of column j) and the range test, one CTA per
// 32 columns of one matrix; flag glob[3] is cleared if some non-zero entry lies more than 2^R
// below its column maximum, or is subnormal.
template <typename T>
__global__ void __launch_bounds__(256) k_i8_colexp(const PowerArgs a) {
    using C = I8Cfg<T>;
    const int N = a.N, m = blockIdx.y;
    const int j0 = blockIdx.x * 32;
    const int tid = threadIdx.x;
    constexpr int PER = 16 / sizeof(T);              // entries per 16-byte load
    constexpr int LANES = 32 / PER;                  // threads per row segment of 32 columns
    const int jl = (tid % LANES) * PER, rl = tid / LANES, RSTEP = 256 / LANES;
    int emax[PER], emin[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) { emax[i] = 0; emin[i] = 1 << 20; }
    const T *P = reinterpret_cast<const T *>(a.P) + (size_t)m * a.mstride + j0 + jl;
    bool sub = false;
#pragma unroll 4
    for (int r = rl; r < N; r += RSTEP) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(P + (size_t)r * a.ld));
        if constexpr (sizeof(T) == 4) {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = (int)((w[i] >> 23) & 0xFF);
                sub |= (e == 0 && (w[i] & 0x7FFFFFu)) || (w[i] >> 31);      // subnormal or negative
                if (w[i] & 0x7FFFFFFFu) { emax[i] = max(emax[i], e); emin[i] = min(emin[i], e); }
            }
        } else {
            const uint64_t w[2] = {((uint64_t)v.y << 32) | v.x, ((uint64_t)v.w << 32) | v.z};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int e = (int)((w[i] >> 52) & 0x7FF);
                sub |= (e == 0 && (w[i] & 0xFFFFFFFFFFFFFull)) || (w[i] >> 63);   // subnormal or negative
                if (w[i] & 0x7FFFFFFFFFFFFFFFull) { emax[i] = max(emax[i], e); emin[i] = min(emin[i], e); }
            }
        }
    }
    __shared__ int s_max[256][PER], s_min[256][PER];
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) { s_max[tid][i] = emax[i]; s_min[tid][i] = emin[i]; }
    __syncthreads();
    if (sub) s_bad = 1;
    if (tid < 32) {
        const int l = tid / PER, i = tid % PER;       // column j0 + tid = lane l's entry i
        int mx = 0, mn = 1 << 20;
        for (int t = l; t < 256; t += LANES) { mx = max(mx, s_max[t][i]); mn = min(mn, s_min[t][i]); }
        // all-zero column: E_j = the largest exponent, so that every shift is negative (zero out);
        // a column whose largest exponent is <= R (entries ~ the subnormal range) fails the test
        const bool any = mn < (1 << 20);
        a.colexp[(size_t)m * N + j0 + tid] = any ? mx : (sizeof(T) == 4 ? 255 : 2047);
        if (any && (mx - mn > C::R || mx <= C::R)) s_bad = 1;
    }
    __syncthreads();
    if (tid == 0 && s_bad) atomicAnd(&a.glob[3], 0u);
}

__global__ void k_i8_flag_set(const PowerArgs a) { a.glob[3] = 1u; }

}  // namespace

// Host side: the i8 kernels of a plan (nullptr when the plan cannot use them).
int i8_supported(int dtype, const PowerArgs &a) {
    const int TN = dtype == SPLIDAR_F64 ? I8Cfg<double>::TN : I8Cfg<float>::TN;
    return a.V >= 8 && 7 * a.V <= 128 && a.N % 128 == 0 && a.N % TN == 0 && a.N >= 1024;
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
    k->flag_fn = (void *)k_i8_flag_set;
    k->step_smem = kI8Smem;
    k->step_block = dim3(kI8Threads);
    const int sms = device_sm_count() < kMaxSMs ? device_sm_count() : kMaxSMs;
    k->step_grid = dim3(sms);
    k->colexp_grid = dim3(a.N / 32, a.M);
    k->colexp_block = dim3(256);
    return func_attrs_once(k->step_fn, (int)kI8Smem, false);
}

int i8_tile_cols(int dtype) { return dtype == SPLIDAR_F64 ? I8Cfg<double>::TN : I8Cfg<float>::TN; }

}  // namespace spl
