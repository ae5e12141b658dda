// f2s.cuh -- shortest round-trip decimal text of a float, byte-identical to
// std::to_chars(char*, char*, float) (the reference's format_value,
// curve.hpp:56-66): the shortest digit string that parses back to the same
// float -- Ulf Adams' Ryu algorithm ("Ryu: fast float-to-string conversion",
// PLDI 2018; its two float tables are generated from their definition by
// tools/gen_f2s_tables.py) -- then the C++17 layout rule: fixed notation
// unless scientific is strictly shorter.  __host__ __device__: the curve
// writers run it on the GPU (k_format.cu); tests/cpp/test_f2s.cpp checks it
// against std::to_chars.
#pragma once
#include <cstdint>

namespace eccb {
namespace f2s {

constexpr int INV_BITS = 59, POW5_BITS = 61;

// ceil(2^(pow5bits(i) - 1 + 59) / 5^i) for i < 31, and the top 61 bits of 5^i for i < 47
#ifdef __CUDA_ARCH__
#define ECC_F2S_SPACE static __constant__
#else
#define ECC_F2S_SPACE static constexpr
#endif
ECC_F2S_SPACE uint64_t kInv[31] = {
    576460752303423489ull, 461168601842738791ull, 368934881474191033ull,
    295147905179352826ull, 472236648286964522ull, 377789318629571618ull,
    302231454903657294ull, 483570327845851670ull, 386856262276681336ull,
    309485009821345069ull, 495176015714152110ull, 396140812571321688ull,
    316912650057057351ull, 507060240091291761ull, 405648192073033409ull,
    324518553658426727ull, 519229685853482763ull, 415383748682786211ull,
    332306998946228969ull, 531691198313966350ull, 425352958651173080ull,
    340282366920938464ull, 544451787073501542ull, 435561429658801234ull,
    348449143727040987ull, 557518629963265579ull, 446014903970612463ull,
    356811923176489971ull, 570899077082383953ull, 456719261665907162ull,
    365375409332725730ull,
};
ECC_F2S_SPACE uint64_t kPow5[47] = {
    1152921504606846976ull, 1441151880758558720ull, 1801439850948198400ull,
    2251799813685248000ull, 1407374883553280000ull, 1759218604441600000ull,
    2199023255552000000ull, 1374389534720000000ull, 1717986918400000000ull,
    2147483648000000000ull, 1342177280000000000ull, 1677721600000000000ull,
    2097152000000000000ull, 1310720000000000000ull, 1638400000000000000ull,
    2048000000000000000ull, 1280000000000000000ull, 1600000000000000000ull,
    2000000000000000000ull, 1250000000000000000ull, 1562500000000000000ull,
    1953125000000000000ull, 1220703125000000000ull, 1525878906250000000ull,
    1907348632812500000ull, 1192092895507812500ull, 1490116119384765625ull,
    1862645149230957031ull, 1164153218269348144ull, 1455191522836685180ull,
    1818989403545856475ull, 2273736754432320594ull, 1421085471520200371ull,
    1776356839400250464ull, 2220446049250313080ull, 1387778780781445675ull,
    1734723475976807094ull, 2168404344971008868ull, 1355252715606880542ull,
    1694065894508600678ull, 2117582368135750847ull, 1323488980084844279ull,
    1654361225106055349ull, 2067951531382569187ull, 1292469707114105741ull,
    1615587133892632177ull, 2019483917365790221ull,
};
#undef ECC_F2S_SPACE

__host__ __device__ __forceinline__ int pow5bits(int e) { return (int)(((uint32_t)e * 1217359u) >> 19) + 1; }
__host__ __device__ __forceinline__ int log10pow2(int e) { return (int)(((uint32_t)e * 78913u) >> 18); }
__host__ __device__ __forceinline__ int log10pow5(int e) { return (int)(((uint32_t)e * 732923u) >> 20); }

__host__ __device__ __forceinline__ int pow5factor(uint32_t v) {
  int n = 0;
  for (;;) {
    const uint32_t q = v / 5, r = v - 5 * q;
    if (r != 0) break;
    v = q;
    ++n;
  }
  return n;
}
__host__ __device__ __forceinline__ bool mult_pow5(uint32_t v, int p) { return pow5factor(v) >= p; }
__host__ __device__ __forceinline__ bool mult_pow2(uint32_t v, int p) {
  return (v & ((1u << p) - 1)) == 0;
}

__host__ __device__ __forceinline__ uint32_t mulshift(uint32_t m, uint64_t f, int shift) {
  const uint64_t lo = (uint64_t)m * (uint32_t)f, hi = (uint64_t)m * (uint32_t)(f >> 32);
  const uint64_t sum = (lo >> 32) + hi;
  return (uint32_t)(sum >> (shift - 32));
}

// shortest (digits, exponent) with value = digits * 10^exponent for a finite
// nonzero float given by its biased exponent and mantissa fields
__host__ __device__ inline void shortest(uint32_t mant, uint32_t bexp, uint32_t& digits, int& exponent) {
  int e2;
  uint32_t m2;
  if (bexp == 0) {
    e2 = 1 - 127 - 23 - 2;
    m2 = mant;
  } else {
    e2 = (int)bexp - 127 - 23 - 2;
    m2 = (1u << 23) | mant;
  }
  const bool even = (m2 & 1) == 0, accept = even;
  const uint32_t mv = 4 * m2, mp = 4 * m2 + 2;
  const uint32_t mmshift = (mant != 0 || bexp <= 1) ? 1u : 0u;
  const uint32_t mm = 4 * m2 - 1 - mmshift;
  uint32_t vr, vp, vm;
  int e10;
  bool vm_tz = false, vr_tz = false;
  uint32_t last = 0;
  if (e2 >= 0) {
    const int q = log10pow2(e2);
    e10 = q;
    const int k = INV_BITS + pow5bits(q) - 1;
    const int i = -e2 + q + k;
    vr = mulshift(mv, kInv[q], i);
    vp = mulshift(mp, kInv[q], i);
    vm = mulshift(mm, kInv[q], i);
    if (q != 0 && (vp - 1) / 10 <= vm / 10) {
      const int l = INV_BITS + pow5bits(q - 1) - 1;
      last = mulshift(mv, kInv[q - 1], -e2 + q - 1 + l) % 10;
    }
    if (q <= 9) {
      if (mv % 5 == 0)
        vr_tz = mult_pow5(mv, q);
      else if (accept)
        vm_tz = mult_pow5(mm, q);
      else
        vp -= mult_pow5(mp, q) ? 1u : 0u;
    }
  } else {
    const int q = log10pow5(-e2);
    e10 = q + e2;
    const int i = -e2 - q;
    const int k = pow5bits(i) - POW5_BITS;
    int j = q - k;
    vr = mulshift(mv, kPow5[i], j);
    vp = mulshift(mp, kPow5[i], j);
    vm = mulshift(mm, kPow5[i], j);
    if (q != 0 && (vp - 1) / 10 <= vm / 10) {
      j = q - 1 - (pow5bits(i + 1) - POW5_BITS);
      last = mulshift(mv, kPow5[i + 1], j) % 10;
    }
    if (q <= 1) {
      vr_tz = true;
      if (accept)
        vm_tz = mmshift == 1;
      else
        --vp;
    } else if (q < 31) {
      vr_tz = mult_pow2(mv, q - 1);
    }
  }
  int removed = 0;
  uint32_t out;
  if (vm_tz || vr_tz) {
    while (vp / 10 > vm / 10) {
      vm_tz &= vm % 10 == 0;
      vr_tz &= last == 0;
      last = vr % 10;
      vr /= 10;
      vp /= 10;
      vm /= 10;
      ++removed;
    }
    if (vm_tz) {
      while (vm % 10 == 0) {
        vr_tz &= last == 0;
        last = vr % 10;
        vr /= 10;
        vp /= 10;
        vm /= 10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;  // round half to even
    out = vr + (((vr == vm && (!accept || !vm_tz)) || last >= 5) ? 1u : 0u);
  } else {
    while (vp / 10 > vm / 10) {
      last = vr % 10;
      vr /= 10;
      vp /= 10;
      vm /= 10;
      ++removed;
    }
    out = vr + ((vr == vm || last >= 5) ? 1u : 0u);
  }
  digits = out;
  exponent = e10 + removed;
}

__host__ __device__ __forceinline__ int ndigits(uint32_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// Writes std::to_chars(float)'s text of the float with bits `u` at `p` (when
// non-null) and returns its length (at most 15 bytes).
__host__ __device__ inline int format(uint32_t u, char* p) {
  const bool neg = u >> 31;
  const uint32_t bexp = (u >> 23) & 0xFF, mant = u & 0x7FFFFF;
  int n = 0;
  auto put = [&](char c) {
    if (p) p[n] = c;
    ++n;
  };
  if (bexp == 0xFF) {
    if (mant) {  // NaN (libstdc++ prints the sign of a NaN too)
      if (neg) put('-');
      put('n'); put('a'); put('n');
    } else {
      if (neg) put('-');
      put('i'); put('n'); put('f');
    }
    return n;
  }
  if (neg) put('-');
  if (bexp == 0 && mant == 0) {
    put('0');
    return n;
  }
  uint32_t d;
  int e;
  shortest(mant, bexp, d, e);
  const int len = ndigits(d);
  // value = d * 10^e; scientific exponent x = e + len - 1
  const int x = e + len - 1;
  const int xl = (x < 0 ? -x : x) >= 100 ? 3 : 2;
  const int sci = len + (len > 1 ? 1 : 0) + 2 + xl;
  int fixed;
  if (e >= 0)
    fixed = len + e;
  else if (len + e > 0)
    fixed = len + 1;
  else
    fixed = 2 - e;  // "0." then -e digits: leading zeros and the digits
  char buf[10];
  for (int k = len - 1; k >= 0; --k) {
    buf[k] = (char)('0' + d % 10);
    d /= 10;
  }
  if (fixed <= sci) {
    if (e > 0) {
      // an integer value: of the len + e character strings the EXACT digits
      // are the closest to the value (C++17 [charconv.to.chars]/2: smallest
      // difference among the shortest), so print the float's exact integer
      // (it has len + e digits; < 10^15 whenever fixed wins)
      const uint32_t m2 = bexp ? ((1u << 23) | mant) : mant;
      const int sh = (int)(bexp ? bexp : 1) - 150;
      uint64_t v = sh >= 0 ? ((uint64_t)m2 << sh) : ((uint64_t)m2 >> -sh);
      char ib[20];
      int ni = 0;
      do {
        ib[ni++] = (char)('0' + v % 10);
        v /= 10;
      } while (v);
      while (ni) put(ib[--ni]);
    } else if (e == 0) {
      for (int k = 0; k < len; ++k) put(buf[k]);
    } else if (len + e > 0) {
      for (int k = 0; k < len + e; ++k) put(buf[k]);
      put('.');
      for (int k = len + e; k < len; ++k) put(buf[k]);
    } else {
      put('0');
      put('.');
      for (int k = 0; k < -(len + e); ++k) put('0');
      for (int k = 0; k < len; ++k) put(buf[k]);
    }
  } else {
    put(buf[0]);
    if (len > 1) {
      put('.');
      for (int k = 1; k < len; ++k) put(buf[k]);
    }
    put('e');
    put(x < 0 ? '-' : '+');
    int ax = x < 0 ? -x : x;
    if (ax >= 100) {
      put((char)('0' + ax / 100));
      ax %= 100;
    }
    put((char)('0' + ax / 10));
    put((char)('0' + ax % 10));
  }
  return n;
}

}  // namespace f2s
}  // namespace eccb
