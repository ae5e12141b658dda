// hist16.cuh -- the packed 65536-bin shared-memory histogram used by the
// 16-bit kernels (k_u16_3d.cu, k_u16_2d.cu, k_batch16.cu, k_batch.cu).
//
// Bin k's running change sum v lives in half (k & 1) of word k >> 1, stored
// as v + 0x1000: the word is the integer  H * 65536 + L  (mod 2^32) with
// H = v_hi + 0x1000 and L = v_lo + 0x1000, so an update is one plain 32-bit
// add of  change << (16 * (k & 1))  -- a low half below -4096 borrows from
// the high half, which unpack() undoes exactly as long as every |v| stays
// below 32768.  A half is "in band" while v lies in [-BAND, BAND) =
// [-4096, 4095], i.e. while its stored 16 bits lie in [0, 0x2000): the top
// three bits are zero, so ONE mask over the new word (old + add) flags an
// out-of-band half.  The mask tests both halves: the other half's flag is a
// harmless false alarm (the fix re-reads its own half exactly), and the high
// half's bits read one low while the low half is below the band (the
// borrow), so its flag may lag by one count at the band's upper edge.
// An update that leaves its half out of band moves the half's whole current
// value to the caller's spill target with a compare-and-swap on the word
// (retried while other updates race it, dropped once the half is back in
// band), so (half + spills) is always the exact sum and a half is reset to
// exactly 0 -- never over-corrected, so it stays tens of thousands of
// updates away from the wrap however hot the bin (an earlier version
// subtracted the value each crossing thread had seen, and several crossings
// racing on one bin of a 2-valued image could push the half past the wrap;
// tests/test_gpu_parity.py covers that).  Updates are issued in groups so
// their atomic latencies overlap; one warp vote per group decides whether
// any lane has a fix to make (rare), and the common path has no divergent
// branches.  Per update the common path is: two PRMTs (key, change), one
// SHF (the half shift), the atomic, and the flag test (one IMAD + one LOP3
// folded into the group's vote word); the addresses are IMADs, off the
// integer ALU pipe that bounds these kernels.
//
// Why a half never wraps (the static bound every user asserts).  Take the
// moment a half leaves the band widened by one count (the flag's lag).
// Every update applied after that, until a fix resets it, leaves it out of
// band and is flagged, so its issuing thread will fix it once its group's
// results are in -- and a thread issues its next group only after fixing
// the previous one (the fix loop ends only when the half is back in band or
// reset to 0).  So before the first fix lands, each thread of the CTA adds
// at most its one outstanding group: the half can move at most THREADS x
// GROUP x MAX|change| past the widened band edge, which must stay below
// HEADROOM = 32768 - BAND - 1 to keep |v| < 32768:
//   k_u16_3d   384 threads x 10 voxels x 7 = 26880 < 28671
//   k_u16_2d   512 x 8 x 3 = 12288;  k_batch16  512 x 16 x 3 = 24576;
//   k_batch (wide u16 batched)  1024 x 1 x 3 = 3072.
#pragma once
#include <cstdint>

namespace eccb {
namespace hist16 {

constexpr uint32_t BIAS = 0x10001000u;     // both halves at 0
constexpr int BAND = 4096;                 // in band: [-BAND, BAND)
constexpr int HEADROOM = 32768 - BAND - 1; // distance from the widened band edge to the wrap
constexpr uint32_t FLAG = 0xE000E000u;     // top three bits of each stored half

// the no-wrap condition for `threads` threads with `group` updates in flight
// each, every update of magnitude <= `max_change`
constexpr bool no_wrap(int threads, int group, int max_change) {
  return (long long)threads * group * max_change < HEADROOM;
}

// the signed sums of a word's two halves (exact while both |v| < 32768)
__host__ __device__ __forceinline__ int lo_value(uint32_t w) {
  return (int16_t)(uint16_t)(w - 0x1000u);
}
__host__ __device__ __forceinline__ int hi_value(uint32_t w) {
  return (int16_t)(uint16_t)((w - (uint32_t)lo_value(w) - BIAS) >> 16);
}
__host__ __device__ __forceinline__ int half_value(uint32_t w, uint32_t hi) {
  return hi ? hi_value(w) : lo_value(w);
}

#ifdef __CUDACC__  // the device side (the encoding above is also checked on the CPU, tests/cpp/test_bits.cpp)
struct Upd {
  uint32_t key, add, old;
};

// byte address of word (key >> 1) / (key >> 5): IMAD.HI + IMAD, both on the
// FMA pipe (the shift-and-mask form is two integer-ALU ops)
__device__ __forceinline__ uint32_t word_addr(uint32_t base, uint32_t key) {
  uint32_t a;
  asm("{\n\t.reg .u32 t;\n\tmul.hi.u32 t, %1, 0x80000000;\n\tmad.lo.u32 %0, t, 4, %2;\n\t}"
      : "=r"(a)
      : "r"(key), "r"(base));
  return a;
}
__device__ __forceinline__ uint32_t bit_word_addr(uint32_t base, uint32_t key) {
  uint32_t a;
  asm("{\n\t.reg .u32 t;\n\tmul.hi.u32 t, %1, 0x08000000;\n\tmad.lo.u32 %0, t, 4, %2;\n\t}"
      : "=r"(a)
      : "r"(key), "r"(base));
  return a;
}

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
               : "r"(word_addr(hbase, key)), "r"(u.add)
               : "memory");
}

// Nonzero when a half of the updated word is out of band (see the header:
// both halves are tested; the fix re-checks its own half exactly).
__device__ __forceinline__ uint32_t crossed(const Upd& u) { return (u.old + u.add) & FLAG; }

// the rare fix: move the half's current value to `spill(key, value)` with a
// compare-and-swap that leaves the half at exactly 0
template <class Spill>
__device__ __forceinline__ void fix(uint32_t hbase, const Upd& u, Spill& spill) {
  if (crossed(u)) {
    const uint32_t addr = word_addr(hbase, u.key);
    const uint32_t hi = u.key & 1u, sh = hi << 4;
    uint32_t cur = u.old + u.add;
    for (;;) {
      const int h = half_value(cur, hi);
      if (h >= -BAND && h < BAND) break;  // in band (another update moved it, or a false alarm)
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
  const uint32_t bit = __funnelshift_l(0u, own, key);  // own << (key & 31)
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(bit_word_addr(pbase, key)), "r"(bit) : "memory");
}

#endif  // __CUDACC__

}  // namespace hist16
}  // namespace eccb
