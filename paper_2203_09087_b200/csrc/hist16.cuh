// hist16.cuh -- the packed 65536-bin shared-memory histogram used by the
// 16-bit kernels (k_u16_3d.cu, k_batch16.cu).
//
// Bin k's running change sum lives in half (k & 1) of word k >> 1, biased
// by 32768.  A half is "in band" while its unbiased value lies in
// [-BAND, BAND) = [-4096, 4095] (biased bits 15..12 = 0111 or 1000).  Every update is an
// atomic add that returns the old word; an update that leaves its half out
// of band moves the half's whole current value to the caller's spill target
// with a compare-and-swap on the word (retried while other updates race it,
// and dropped once the half is back in band), so (half + spills) is always
// the exact sum and a half is reset to exactly 0 -- never over-corrected, so
// it stays tens of thousands of updates away from the 16-bit wrap however
// hot the bin (an earlier version subtracted the value each crossing thread
// had seen, and several crossings racing on one bin of a 2-valued image
// could push the half past the wrap; tests/test_gpu_parity.py now covers
// that).  Updates are issued in groups so their atomic latencies overlap;
// one warp vote per group decides whether any lane has a fix to make
// (rare), and the common path has no divergent branches.
//
// Why a half never wraps (the static bound every user asserts).  Take the
// moment a half leaves the band.  Every update applied after that, until a
// fix resets it, leaves it out of band, so its issuing thread will fix it
// once its group's results are in -- and a thread issues its next group only
// after fixing the previous one (the fix loop ends only when the half is
// back in band or reset to 0).  So before the first fix lands, each thread
// of the CTA adds at most its one outstanding group: the half can move at
// most THREADS x GROUP x MAX|change| past the band edge, which must stay
// below HEADROOM = 32768 - BAND to keep the 16 bits unambiguous:
//   k_u16_3d   384 threads x 10 voxels x 7 = 26880 < 28672
//   k_u16_2d   512 x 8 x 3 = 12288;  k_batch16  512 x 8 x 3 = 12288;
//   k_batch (wide u16 batched)  1024 x 1 x 3 = 3072.
#pragma once
#include <cstdint>

namespace eccb {
namespace hist16 {

constexpr uint32_t BIAS = 0x80008000u;
constexpr int BAND = 4096;                 // in band: [-BAND, BAND)
constexpr int HEADROOM = 32768 - BAND;     // distance from the band edge to the wrap

// the no-wrap condition for `threads` threads with `group` updates in flight
// each, every update of magnitude <= `max_change`
constexpr bool no_wrap(int threads, int group, int max_change) {
  return (long long)threads * group * max_change < HEADROOM;
}

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

// Nonzero when the updated half is out of band after this update.  Only
// that half can differ between the old and the new word (no half ever
// reaches its wrap, so the low half never carries into the high one); the
// mask restricts the test to it.  In band: biased bits 15..12 = 0111 or
// 1000, i.e. t = w ^ (w << 1) has bit 15 set and bits 14, 13 clear.
__device__ __forceinline__ uint32_t crossed(const Upd& u) {
  const uint32_t w = u.old + u.add;
  const uint32_t t = w ^ (w << 1);
  const uint32_t half = __funnelshift_l(0u, 0xE000u, u.key << 4);  // this half's bits 15..13
  return ((~t & 0x80008000u) | (t & 0x60006000u)) & half;
}

// the rare fix: move the half's current value to `spill(key, value)` with a
// compare-and-swap that leaves the half at exactly 0 (biased 32768)
template <class Spill>
__device__ __forceinline__ void fix(uint32_t hbase, const Upd& u, uint32_t cross, Spill& spill) {
  if (cross) {
    const uint32_t addr = hbase + (u.key >> 1) * 4u;
    const uint32_t sh = (u.key & 1u) << 4;
    uint32_t cur = u.old + u.add;
    for (;;) {
      const int h = (int)((cur >> sh) & 0xFFFFu) - 32768;
      if (h >= -BAND && h < BAND) break;  // back in band: another update moved it
      const uint32_t want = cur - ((uint32_t)h << sh);
      uint32_t prev;
      asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;"
                   : "=r"(prev)
                   : "r"(addr), "r"(cur), "r"(want)
                   : "memory");
      if (prev == cur) {
        spill(u.key, h);
        break;
      }
      cur = prev;
    }
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
