// Per-column fixed point of the int8 GEMV (power_i8.cu) and of the encoded fp32 storage a building
// plan writes (build.cu): with E_j the largest biased exponent of column j and R headroom bits, an
// entry a = 1.m x 2^(e - bias) of column j is the integer
//   a~ = significand << (e - E_j + R)        (exact when E_j - R <= e <= E_j; 0 for a = 0)
// i.e. a 2^(BIAS + MBITS + R - E_j), of <= 32 (fp32, R = 8) / 64 (fp64, R = 11) bits.
// Internal; not shared with oracle/.
#pragma once
#include <stdint.h>

namespace spl {

// PTX shl clamps the shift amount to the register width, so a zero entry (e = 0, shift e - base
// < 0, i.e. huge as unsigned) gives 0 without a select; the callers guarantee base > 0 for every
// column with a non-zero entry and set E_j = 255 / 2047 (base > 0 as well) for all-zero columns.
// fp32: the significand 1.m left-aligned as the 64-bit value (1 : m << 9) = 2^9 sig, shifted left
// by s = sh + 23 with a clamping funnel shift; the high word is sig << sh (3 integer ops per entry).
// For a zero entry s < 0 (huge as unsigned) clamps to 32 and the funnel returns the low word, 0.
// base23 = E_j - R - 23.
__device__ __forceinline__ uint32_t fx32(uint32_t u, int base23) {
    const uint32_t s = (uint32_t)((int)(u >> 23) - base23);          // e - base + 23
    uint32_t r;
    asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(u << 9), "r"(1u), "r"(s));
    return r;
}
// fp64: 53-bit significand (hi 21 bits : lo 32 bits) << sh, sh <= 11, as two clamping shifts; a zero
// entry has sh < 0: both clamp to 0 (the funnel returns the zero low word). base = E_j - R.
__device__ __forceinline__ void fx64(uint32_t lo, uint32_t hi, int base, uint32_t &rlo, uint32_t &rhi) {
    const uint32_t sh = (uint32_t)((int)(hi >> 20) - base);
    const uint32_t sig_hi = (hi & 0xFFFFFu) | 0x100000u;
    asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(rhi) : "r"(lo), "r"(sig_hi), "r"(sh));
    asm("shl.b32 %0, %1, %2;" : "=r"(rlo) : "r"(lo), "r"(sh));
}

}  // namespace spl
