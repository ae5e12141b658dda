// hist16.cuh -- the packed 65536-bin shared-memory histogram used by the
// 16-bit kernels (k_u16_3d.cu, k_batch16.cu).
//
// Bin k's running change sum lives in half (k & 1) of word k >> 1, biased
// by 32768.  A half is "in band" while its biased value lies in
// [16384, 49151] (bit 15 XOR bit 14 of the half set).  Every update is an
// atomic add that returns the old word; an update that changes the band of
// its half (either direction) hands exactly the value it saw to the caller's
// spill target and subtracts it from the half, so (half + spills) is always
// the exact sum and halves stay far from the carry boundary: a half would
// need thousands more updates of the same bin between the crossing atomic
// and the fix a few instructions later to wrap.  Updates are issued in
// groups so their atomic latencies overlap; one warp vote per group decides
// whether any lane has a fix to make (rare), and the fix itself is
// predicated, so the common path has no divergent branches.
#pragma once
#include <cstdint>

namespace eccb {
namespace hist16 {

constexpr uint32_t BIAS = 0x80008000u;

struct Upd {
  uint32_t key, add, old;
};

// add the signed change chu (two's complement; 0 = no-op) to bin `key`.
// chu << (16 * (key & 1)) is one wrap-mode funnel shift by key << 4 (the
// shift amount is taken mod 32).
__device__ __forceinline__ void issue(uint32_t hbase, uint32_t key, uint32_t chu, Upd& u) {
  u.key = key;
  u.add = __funnelshift_l(0u, chu, key << 4);
  // unconditional: a zero add is cheaper than the branch ptxas makes of a
  // predicated atomic with a return value (ISETP + BSSY + BRA + BSYNC)
  asm volatile("atom.shared.add.u32 %0, [%1], %2;"
               : "=r"(u.old)
               : "r"(hbase + (key >> 1) * 4u), "r"(u.add)
               : "memory");
}

// Band change of the updated half.  Only that half can differ between the
// old and new word (the band keeps the low half from carrying into the high
// one), so one constant mask covers both halves.
__device__ __forceinline__ uint32_t crossed(const Upd& u) {
  const uint32_t d = u.old ^ (u.old + u.add);
  return (d ^ (d << 1)) & 0x80008000u;
}

// the rare fix: predicated shared add of -after, and `spill(key, after)`
template <class Spill>
__device__ __forceinline__ void fix(uint32_t hbase, const Upd& u, uint32_t cross, Spill& spill) {
  if (cross) {
    const uint32_t sh = (u.key & 1u) << 4;
    const int after = (int)(((u.old + u.add) >> sh) & 0xFFFFu) - 32768;
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hbase + (u.key >> 1) * 4u),
                 "r"((uint32_t)(-after) << sh)
                 : "memory");
    spill(u.key, after);
  }
}

// occupancy bit of `key` when `own` (0 or 1): an unconditional shared OR
// (OR-ing 0 is a no-op); cheaper than testing the bit first, which ptxas
// turns into a load, a compare and a branch per pixel.
__device__ __forceinline__ void mark(uint32_t pbase, uint32_t key, uint32_t own) {
  const uint32_t pa = pbase + (key >> 5) * 4u;
  const uint32_t bit = __funnelshift_l(0u, own, key);  // own << (key & 31)
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(pa), "r"(bit) : "memory");
}

}  // namespace hist16
}  // namespace eccb
