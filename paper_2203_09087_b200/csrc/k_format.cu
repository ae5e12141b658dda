// k_format.cu -- curve serialisation on the device:
// write_curve's CSV and JSON layouts (curve.hpp:87-121) and write_vcec's CSV
// (curve.hpp:154-169), byte-identical to the reference writers, for
//   * every image of a dense batch (ecc_batch2d output: int32
//     chi[count][nbins] + presence bitmaps; integer thresholds), and
//   * one sparse curve / VCEC of any value type (u8 / u16 / f32 thresholds,
//     int64 chi or changes): f32 thresholds through f2s.cuh, the shortest
//     round-trip text std::to_chars prints (format_value, curve.hpp:56-66).
//
// Two passes, one CTA per image: k_format_sizes sums the bytes of the
// image's occurring points (block reduction); after an exclusive scan over
// images, k_format_write block-scans the per-thread byte counts and entry
// counts and each thread writes its run of lines.
#include <cub/cub.cuh>

#include "f2s.cuh"
#include "internal.h"

namespace eccb {
namespace fmt {

constexpr int NT = 512;

__device__ __forceinline__ int ndigits_u(uint32_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

__device__ __forceinline__ int len_i(int32_t v) {
  const uint32_t a = v < 0 ? (uint32_t)(-(int64_t)v) : (uint32_t)v;
  return ndigits_u(a) + (v < 0);
}

__device__ __forceinline__ char* put_u(char* p, uint32_t v) {
  const int n = ndigits_u(v);
  for (int i = n - 1; i >= 0; --i) {
    p[i] = (char)('0' + v % 10);
    v /= 10;
  }
  return p + n;
}

__device__ __forceinline__ char* put_i(char* p, int32_t v) {
  if (v < 0) {
    *p++ = '-';
    return put_u(p, (uint32_t)(-(int64_t)v));
  }
  return put_u(p, (uint32_t)v);
}

__device__ __forceinline__ char* put_s(char* p, const char* s) {
  while (*s) *p++ = *s++;
  return p;
}

// bytes of one point: CSV "t,chi\n"; JSON "{"t":T,"chi":C}" (+ "," before
// every point but the first, counted by the writer)
__device__ __forceinline__ int point_bytes(int json, uint32_t t, int32_t c) {
  return json ? 5 + ndigits_u(t) + 7 + len_i(c) + 1 : ndigits_u(t) + 1 + len_i(c) + 1;
}

constexpr int CSV_HEADER = 31;  // "threshold,euler_characteristic\n"

__global__ void __launch_bounds__(NT) k_format_sizes(const int32_t* __restrict__ chi,
                                                     const uint32_t* __restrict__ pres,
                                                     uint32_t nbins, int json,
                                                     uint64_t* __restrict__ sizes) {
  const int32_t* row = chi + (size_t)blockIdx.x * nbins;
  const uint32_t* prow = pres + (size_t)blockIdx.x * (nbins / 32);
  const uint32_t per = (nbins + NT - 1) / NT;
  const uint32_t b0 = min(nbins, threadIdx.x * per), b1 = min(nbins, b0 + per);
  uint64_t bytes = 0, pts = 0;
  for (uint32_t b = b0; b < b1; ++b)
    if ((prow[b >> 5] >> (b & 31)) & 1u) {
      bytes += point_bytes(json, b, row[b]);
      ++pts;
    }
  using Red = cub::BlockReduce<ulonglong2, NT>;
  __shared__ typename Red::TempStorage tmp;
  struct Add {
    __device__ ulonglong2 operator()(const ulonglong2& a, const ulonglong2& b) const {
      return make_ulonglong2(a.x + b.x, a.y + b.y);
    }
  };
  const ulonglong2 tot = Red(tmp).Reduce(make_ulonglong2(bytes, pts), Add());
  if (threadIdx.x == 0) {
    uint64_t total = tot.x;
    if (json)
      total += 1 + (tot.y > 1 ? tot.y - 1 : 0) + 2;  // '[' , commas , "]\n"
    else
      total += CSV_HEADER;
    sizes[blockIdx.x] = total;
  }
}

__global__ void __launch_bounds__(NT) k_format_write(const int32_t* __restrict__ chi,
                                                     const uint32_t* __restrict__ pres,
                                                     uint32_t nbins, int json,
                                                     const uint64_t* __restrict__ offsets,
                                                     char* __restrict__ out) {
  const int32_t* row = chi + (size_t)blockIdx.x * nbins;
  const uint32_t* prow = pres + (size_t)blockIdx.x * (nbins / 32);
  const uint32_t per = (nbins + NT - 1) / NT;
  const uint32_t b0 = min(nbins, threadIdx.x * per), b1 = min(nbins, b0 + per);
  uint64_t bytes = 0, pts = 0;
  for (uint32_t b = b0; b < b1; ++b)
    if ((prow[b >> 5] >> (b & 31)) & 1u) {
      bytes += point_bytes(json, b, row[b]);
      ++pts;
    }
  using Scan = cub::BlockScan<ulonglong2, NT>;
  __shared__ typename Scan::TempStorage tmp;
  struct Add {
    __device__ ulonglong2 operator()(const ulonglong2& a, const ulonglong2& b) const {
      return make_ulonglong2(a.x + b.x, a.y + b.y);
    }
  };
  ulonglong2 ex;
  Scan(tmp).ExclusiveScan(make_ulonglong2(bytes, pts), ex, make_ulonglong2(0, 0), Add());
  char* base = out + offsets[blockIdx.x];
  const uint64_t head = json ? 1 : CSV_HEADER;
  if (threadIdx.x == 0) {
    if (json)
      base[0] = '[';
    else
      put_s(base, "threshold,euler_characteristic\n");
  }
  // every point but the image's first is preceded by a comma in JSON: the
  // ex.y - 1 commas before this thread's first point lie ahead of it (that
  // point's own comma is written below)
  char* p = base + head + ex.x + ((json && ex.y > 0) ? ex.y - 1 : 0);
  uint64_t idx = ex.y;
  for (uint32_t b = b0; b < b1; ++b)
    if ((prow[b >> 5] >> (b & 31)) & 1u) {
      if (json) {
        if (idx > 0) *p++ = ',';
        p = put_s(p, "{\"t\":");
        p = put_u(p, b);
        p = put_s(p, ",\"chi\":");
        p = put_i(p, row[b]);
        *p++ = '}';
      } else {
        p = put_u(p, b);
        *p++ = ',';
        p = put_i(p, row[b]);
        *p++ = '\n';
      }
      ++idx;
    }
  if (json && threadIdx.x == NT - 1) {
    char* end = out + offsets[blockIdx.x + 1];
    end[-2] = ']';
    end[-1] = '\n';
  }
}

// zero_crossings (curve.hpp:36-50) of every image: bit t of the output row is
// set iff occurring bin t is a zero crossing -- chi == 0, or a strict sign
// change from the previous occurring point (which may lie in another
// thread's range: a block scan carries the last occurring chi forward).
// Thread ranges are whole bitmap words (>= 32 bins).
__global__ void __launch_bounds__(NT) k_zero_crossings(const int32_t* __restrict__ chi,
                                                       const uint32_t* __restrict__ pres,
                                                       uint32_t nbins, uint32_t* __restrict__ zc) {
  const int32_t* row = chi + (size_t)blockIdx.x * nbins;
  const uint32_t* prow = pres + (size_t)blockIdx.x * (nbins / 32);
  uint32_t* zrow = zc + (size_t)blockIdx.x * (nbins / 32);
  const uint32_t per = max(32u, (nbins + NT - 1) / NT / 32 * 32);
  const uint32_t b0 = min(nbins, threadIdx.x * per), b1 = min(nbins, b0 + per);
  // (has a point, chi of the last point) of this thread's range
  int2 last = make_int2(0, 0);
  for (uint32_t b = b0; b < b1; ++b)
    if ((prow[b >> 5] >> (b & 31)) & 1u) last = make_int2(1, row[b]);
  struct Last {
    __device__ int2 operator()(const int2& a, const int2& b) const { return b.x ? b : a; }
  };
  using Scan = cub::BlockScan<int2, NT>;
  __shared__ typename Scan::TempStorage tmp;
  int2 prev;
  Scan(tmp).ExclusiveScan(last, prev, make_int2(0, 0), Last());
  for (uint32_t w = b0; w < b1; w += 32) {
    uint32_t bits = 0;
    const uint32_t pw = prow[w >> 5];
    for (uint32_t j = 0; j < 32 && w + j < b1; ++j)
      if ((pw >> j) & 1u) {
        const int32_t c = row[w + j];
        const bool z = c == 0 || (prev.x && prev.y != 0 && ((c > 0) != (prev.y > 0)));
        bits |= (uint32_t)z << j;
        prev = make_int2(1, c);
      }
    zrow[w >> 5] = bits;
  }
}

}  // namespace fmt

cudaError_t launch_zero_crossings(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                  uint32_t nbins, uint32_t* zc, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  fmt::k_zero_crossings<<<(unsigned)count, fmt::NT, 0, st>>>(chi, pres, nbins, zc);
  return cudaGetLastError();
}

cudaError_t launch_format_sizes(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                uint32_t nbins, int json, uint64_t* sizes, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  fmt::k_format_sizes<<<(unsigned)count, fmt::NT, 0, st>>>(chi, pres, nbins, json, sizes);
  return cudaGetLastError();
}

cudaError_t launch_format_write(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                uint32_t nbins, int json, const uint64_t* offsets, char* out,
                                cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  fmt::k_format_write<<<(unsigned)count, fmt::NT, 0, st>>>(chi, pres, nbins, json, offsets, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- one sparse curve / VCEC
namespace fmt1 {

__device__ __forceinline__ int ndigits_u64(uint64_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// text of an int64 (std::to_chars)
__device__ __forceinline__ int put_i64(char* p, int64_t v) {
  const bool neg = v < 0;
  uint64_t a = neg ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
  const int n = ndigits_u64(a) + (neg ? 1 : 0);
  if (p) {
    int i = n - 1;
    do {
      p[i--] = (char)('0' + a % 10);
      a /= 10;
    } while (a);
    if (neg) p[0] = '-';
  }
  return n;
}

// text of threshold i (format_value): integers for u8 / u16, f2s for f32
__device__ __forceinline__ int put_t(char* p, const void* t, int dtype, uint64_t i) {
  if (dtype == 2) return f2s::format(__float_as_uint(static_cast<const float*>(t)[i]), p);
  const int64_t v = dtype == 0 ? (int64_t) static_cast<const uint8_t*>(t)[i]
                               : (int64_t) static_cast<const uint16_t*>(t)[i];
  return put_i64(p, v);
}

// mode 0 CSV curve ("t,chi\n"), 1 JSON curve ("{\"t\":T,\"chi\":C}", comma
// before all but the first), 2 VCEC CSV ("value,change\n")
__device__ __forceinline__ int point(char* p, int mode, const void* t, int dtype, const int64_t* c,
                                     uint64_t i) {
  int n = 0;
  if (mode == 1) {
    if (i) {
      if (p) p[n] = ',';
      ++n;
    }
    const char* a = "{\"t\":";
    for (int k = 0; a[k]; ++k, ++n)
      if (p) p[n] = a[k];
  }
  n += put_t(p ? p + n : nullptr, t, dtype, i);
  if (mode == 1) {
    const char* b = ",\"chi\":";
    for (int k = 0; b[k]; ++k, ++n)
      if (p) p[n] = b[k];
  } else {
    if (p) p[n] = ',';
    ++n;
  }
  n += put_i64(p ? p + n : nullptr, c[i]);
  if (mode == 1) {
    if (p) p[n] = '}';
    ++n;
  } else {
    if (p) p[n] = '\n';
    ++n;
  }
  return n;
}

__global__ void k_point_sizes(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                              uint32_t* sizes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    sizes[i] = (uint32_t)point(nullptr, mode, t, dtype, c, i);
}

__global__ void k_point_write(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                              const uint64_t* offsets, uint64_t head, char* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    point(out + head + offsets[i], mode, t, dtype, c, i);
}

}  // namespace fmt1

cudaError_t launch_point_sizes(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                               uint32_t* sizes, int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fmt1::k_point_sizes<<<sms * 4, 256, 0, st>>>(mode, t, dtype, c, n, sizes);
  return cudaGetLastError();
}

cudaError_t launch_point_write(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                               const uint64_t* offsets, uint64_t head, char* out, int sms,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fmt1::k_point_write<<<sms * 4, 256, 0, st>>>(mode, t, dtype, c, n, offsets, head, out);
  return cudaGetLastError();
}

}  // namespace eccb
