// tc_common.cuh -- code unpacking into UMMA (tcgen05) K-major smem tiles.
//
// Codes are packed LSB-first.  A 32-bit word of 2-bit codes holds 16
// consecutive codes; (w >> 2k) & 0x03030303 (k = 0..3) yields 4 bytes holding the
// codes at positions {k, k+4, k+8, k+12}.  Writing the four results consecutively
// stores the 16 codes in a fixed permutation pi2 inside every 16-group; 4-bit words
// (8 codes) use (w >> 4k) & 0x0F0F0F0F, a permutation pi4 inside every 8-group.
// A dot product is invariant when both operands are permuted alike, and Pi-aligned
// partitions are unions of 16-groups, so the other operand (Q' or P', which the
// kernels write themselves) is simply stored in the same permuted order.
#pragma once
#include <stdint.h>

#include "tc_ptx.cuh"

namespace hack {

// Byte position p (0..15) of a permuted 16-byte chunk -> original index in the chunk.
template <int BITS>
HACK_DEV constexpr int perm_src(int p) {
  return BITS == 2 ? (p >> 2) + 4 * (p & 3) : 8 * (p >> 3) + ((p & 7) >> 2) + 2 * (p & 3);
}

// 16 codes (2-bit) -> 16 bytes in pi2 order.
HACK_DEV uint4 unpack16_2b(uint32_t w) {
  return make_uint4(w & 0x03030303u, (w >> 2) & 0x03030303u, (w >> 4) & 0x03030303u, (w >> 6) & 0x03030303u);
}
// 8 codes (4-bit) -> 8 bytes in pi4 order.
HACK_DEV uint2 unpack8_4b(uint32_t w) { return make_uint2(w & 0x0F0F0F0Fu, (w >> 4) & 0x0F0F0F0Fu); }

// Doubled codes 2c (u8) in the same orders: the B operand of the centered kernels, so that
// sum (a - 128)(2c) + offsets gives the exact integer 2 x sum (a - 128)(c - (2^b - 1)/2).
HACK_DEV uint4 unpack16_2b_x2(uint32_t w) {
  return make_uint4((w << 1) & 0x06060606u, (w >> 1) & 0x06060606u, (w >> 3) & 0x06060606u, (w >> 5) & 0x06060606u);
}
HACK_DEV uint2 unpack8_4b_x2(uint32_t w) { return make_uint2((w << 1) & 0x1E1E1E1Eu, (w >> 3) & 0x1E1E1E1Eu); }

// Offset of (row, k-byte) in a K-major no-swizzle tile: [row/8][k/16][row%8][16 B].
HACK_DEV uint32_t kmaj_off(int row, int kbyte, int sbo) {
  return (uint32_t)((row >> 3) * sbo + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15));
}

}  // namespace hack
