// fin_u8.cuh -- the end of every u8 bit-sliced kernel (k_u8_3d.cu,
// k_u8_2d.cu): reduce the CTA's (code, value) shared-memory table to
// per-value change sums and pixel counts, flush them with int64 global
// atomics, and -- when a finalize workspace is passed -- let the last CTA
// to finish turn the global histogram into the curve in the same launch
// (merge_local + vcec_to_ecc, vcec.hpp:35-66, curve.hpp:28-35), re-zeroing
// the histogram and the ticket for the next launch.
#pragma once
#include <cstdint>

#include <cub/cub.cuh>

namespace eccb {
namespace u8fin {

struct Fin {
  uint32_t* ticket;    // zero before the launch, zero again after it
  uint32_t* bins;      // [256] occurring values, ascending
  int64_t* changes;    // [256] their VCEC entries
  int64_t* chi;        // [256] the curve
  uint64_t* count;     // number of occurring values
};

// Code: static constexpr int n (codes per value in the table);
//       static __device__ bool live(int c) (a real change, not "not emitted");
//       static __device__ int change(int c).
// ghist: [256] change sums then [256] pixel counts.
template <int NT, class Code>
__device__ __forceinline__ void flush_and_finalize(const uint32_t* hist, int64_t* ghist,
                                                   const Fin& fin) {
  static_assert(256 % NT == 0 || NT % 256 == 0, "NT must divide 256 or be a multiple of it");
  __syncthreads();
  for (int v = threadIdx.x; v < 256; v += NT) {
    long long sum = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < Code::n; ++c) {
      if (!Code::live(c)) continue;
      const long long n = hist[c * 256 + v];
      cnt += n;
      sum += n * Code::change(c);
    }
    if (cnt != 0) {
      if (sum != 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[v]),
                  static_cast<unsigned long long>(sum));
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[256 + v]),
                static_cast<unsigned long long>(cnt));
    }
  }
  if (!fin.ticket) return;
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(fin.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // thread t owns values [VPT t, VPT (t + 1)) (VPT = 0 for threads past 256)
  constexpr int VPT = NT >= 256 ? 1 : 256 / NT;
  struct Add {
    __device__ longlong2 operator()(const longlong2& a, const longlong2& b) const {
      return make_longlong2(a.x + b.x, a.y + b.y);
    }
  };
  using Scan = cub::BlockScan<longlong2, NT>;
  __shared__ typename Scan::TempStorage tmp;
  const int v0 = VPT * threadIdx.x;
  const bool mine = v0 < 256;
  long long s[VPT], n[VPT];
  longlong2 in = make_longlong2(0, 0);
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    s[j] = mine ? __ldcg(&ghist[v0 + j]) : 0;
    n[j] = mine ? __ldcg(&ghist[256 + v0 + j]) : 0;
    in.x += (n[j] != 0);
    in.y += s[j];
  }
  longlong2 ex, total;
  Scan(tmp).ExclusiveScan(in, ex, make_longlong2(0, 0), Add(), total);
  long long pos = ex.x, acc = ex.y;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    acc += s[j];
    if (n[j] != 0) {
      fin.bins[pos] = v0 + j;
      fin.changes[pos] = s[j];
      fin.chi[pos] = acc;
      ++pos;
    }
    if (mine) {
      ghist[v0 + j] = 0;
      ghist[256 + v0 + j] = 0;
    }
  }
  if (threadIdx.x == 0) {
    *fin.count = (uint64_t)total.x;
    *fin.ticket = 0;
  }
}

}  // namespace u8fin
}  // namespace eccb
