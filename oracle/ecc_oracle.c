/*
 * ecc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the ECC hot path
 * (per-voxel Euler change -> histogram by value -> prefix sum).  It exists so
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
 * check the CUDA product path; nothing in paper_2203_09087_b200/ links,
 * imports or calls it.
 *
 * Parity of this restatement is pinned against the reference itself (compiled
 * from /root/reference by oracle/Makefile into oracle/_ref/) and against the
 * golden curve hashes in tests/golden/ (SURVEY.md Appendix B).
 *
 * Reference citations are relative to /root/reference/proj/include/ecc/.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* Synthetic inputs: datagen.hpp:18-27 (splitmix64, counter_hash).         */

uint64_t ecc_oracle_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t ecc_oracle_counter_hash(uint64_t seed, uint64_t i) {
  return ecc_oracle_splitmix64(seed + i * 0x9E3779B97F4A7C15ull);
}

/* SURVEY.md 8(d) inputs: u8 v = H>>56, u16 v = H>>48, f32 v = (H>>48)*2^-16,
 * counter = base + i. */
void ecc_oracle_fill_u8(uint8_t* dst, uint64_t n, uint64_t seed, uint64_t base) {
  for (uint64_t i = 0; i < n; ++i)
    dst[i] = (uint8_t)(ecc_oracle_counter_hash(seed, base + i) >> 56);
}
void ecc_oracle_fill_u16(uint16_t* dst, uint64_t n, uint64_t seed, uint64_t base) {
  for (uint64_t i = 0; i < n; ++i)
    dst[i] = (uint16_t)(ecc_oracle_counter_hash(seed, base + i) >> 48);
}
void ecc_oracle_fill_f32q(float* dst, uint64_t n, uint64_t seed, uint64_t base) {
  for (uint64_t i = 0; i < n; ++i)
    dst[i] = (float)(ecc_oracle_counter_hash(seed, base + i) >> 48) * 0x1p-16f;
}

/* ---------------------------------------------------------------------- */
/* Float order key: value_index.hpp:95-105.                                */

uint32_t ecc_oracle_float_order_key(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if (u == 0x80000000u) u = 0; /* -0.0 and +0.0 share a bin */
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

float ecc_oracle_float_from_order_key(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* ---------------------------------------------------------------------- */
/* The stencil.  The image is viewed through a padded 3-plane window whose
 * collar holds the sentinel (chunk.hpp:50-63, 193-220): sentinel 256 for
 * u8 (common.hpp:54-59), +inf for f32 (common.hpp:61-66).  u16 is carried
 * as float (exact), matching the reference's f32 path.
 *
 * change_2d: kernel.hpp:81-94.  change_3d: kernel.hpp:99-137.  Offsets
 * toward an earlier voxel (first nonzero component negative,
 * kernel.hpp:21-27) compare strictly, later offsets non-strictly.        */

#define ECC_CHANGE_2D(E)                                                    \
  static int change_2d_##E(const E* p, ptrdiff_t s0, ptrdiff_t s1) {        \
    const E c = p[0];                                                       \
    const unsigned am = c < p[-s0], ap = c <= p[s0];                        \
    const unsigned bm = c < p[-s1], bp = c <= p[s1];                        \
    unsigned verts = 0;                                                     \
    verts += am & bm & (unsigned)(c < p[-s0 - s1]);                         \
    verts += am & bp & (unsigned)(c < p[-s0 + s1]);                         \
    verts += ap & bm & (unsigned)(c <= p[s0 - s1]);                         \
    verts += ap & bp & (unsigned)(c <= p[s0 + s1]);                         \
    return 1 + (int)verts - (int)(am + ap + bm + bp);                       \
  }

#define ECC_CHANGE_3D(E)                                                     \
  static int change_3d_##E(const E* p, ptrdiff_t s0, ptrdiff_t s1) {         \
    const E c = p[0];                                                        \
    const unsigned xm = c < p[-s0], xp = c <= p[s0];                         \
    const unsigned ym = c < p[-s1], yp = c <= p[s1];                         \
    const unsigned zm = c < p[-1], zp = c <= p[1];                           \
    const unsigned exy_mm = xm & ym & (unsigned)(c < p[-s0 - s1]);           \
    const unsigned exy_mp = xm & yp & (unsigned)(c < p[-s0 + s1]);           \
    const unsigned exy_pm = xp & ym & (unsigned)(c <= p[s0 - s1]);           \
    const unsigned exy_pp = xp & yp & (unsigned)(c <= p[s0 + s1]);           \
    const unsigned exz_mm = xm & zm & (unsigned)(c < p[-s0 - 1]);            \
    const unsigned exz_mp = xm & zp & (unsigned)(c < p[-s0 + 1]);            \
    const unsigned exz_pm = xp & zm & (unsigned)(c <= p[s0 - 1]);            \
    const unsigned exz_pp = xp & zp & (unsigned)(c <= p[s0 + 1]);            \
    const unsigned eyz_mm = ym & zm & (unsigned)(c < p[-s1 - 1]);            \
    const unsigned eyz_mp = ym & zp & (unsigned)(c < p[-s1 + 1]);            \
    const unsigned eyz_pm = yp & zm & (unsigned)(c <= p[s1 - 1]);            \
    const unsigned eyz_pp = yp & zp & (unsigned)(c <= p[s1 + 1]);            \
    unsigned v = 0;                                                          \
    v += exy_mm & exz_mm & eyz_mm & (unsigned)(c < p[-s0 - s1 - 1]);         \
    v += exy_mm & exz_mp & eyz_mp & (unsigned)(c < p[-s0 - s1 + 1]);         \
    v += exy_mp & exz_mm & eyz_pm & (unsigned)(c < p[-s0 + s1 - 1]);         \
    v += exy_mp & exz_mp & eyz_pp & (unsigned)(c < p[-s0 + s1 + 1]);         \
    v += exy_pm & exz_pm & eyz_mm & (unsigned)(c <= p[s0 - s1 - 1]);         \
    v += exy_pm & exz_pp & eyz_mp & (unsigned)(c <= p[s0 - s1 + 1]);         \
    v += exy_pp & exz_pm & eyz_pm & (unsigned)(c <= p[s0 + s1 - 1]);         \
    v += exy_pp & exz_pp & eyz_pp & (unsigned)(c <= p[s0 + s1 + 1]);         \
    const unsigned sq = xm + xp + ym + yp + zm + zp;                         \
    const unsigned ed = exy_mm + exy_mp + exy_pm + exy_pp + exz_mm + exz_mp + \
                        exz_pm + exz_pp + eyz_mm + eyz_mp + eyz_pm + eyz_pp; \
    return -1 + (int)sq - (int)ed + (int)v;                                  \
  }

ECC_CHANGE_2D(int32_t)
ECC_CHANGE_3D(int32_t)
ECC_CHANGE_2D(float)
ECC_CHANGE_3D(float)

/* Per-voxel changes of a whole image, owned row-major order (the same
 * output compute_changes produces, kernel.hpp:244-265).  `T` is the input
 * element type, `E` the extended type.  A padded 3-plane ring plays the
 * role of PaddedChunk with the one-plane halo of fill_padded_chunk.      */
#define ECC_CHANGES(NAME, T, E, SENT, CH2, CH3)                                \
  int NAME(const T* img, uint64_t w0, uint64_t w1, uint64_t w2,               \
           int8_t* out) {                                                     \
    const int is2d = (w2 == 1);                                               \
    const uint64_t P1 = w1 + 2, P2 = is2d ? 3 : w2 + 2;                       \
    const uint64_t plane = P1 * P2;                                           \
    E* win = (E*)malloc(sizeof(E) * plane * 3);                               \
    if (!win) return -1;                                                      \
    /* slot s holds image plane (i - 1 + s) */                                \
    for (uint64_t i = 0; i < w0; ++i) {                                       \
      for (int s = 0; s < 3; ++s) {                                           \
        E* dst = win + s * plane;                                             \
        for (uint64_t q = 0; q < plane; ++q) dst[q] = SENT;                   \
        const int64_t r = (int64_t)i - 1 + s;                                 \
        if (r < 0 || (uint64_t)r >= w0) continue;                             \
        for (uint64_t j = 0; j < w1; ++j)                                     \
          for (uint64_t k = 0; k < w2; ++k)                                   \
            dst[(j + 1) * P2 + (k + 1)] =                                     \
                (E)img[((uint64_t)r * w1 + j) * w2 + k];                      \
      }                                                                       \
      const E* mid = win + plane;                                             \
      for (uint64_t j = 0; j < w1; ++j)                                       \
        for (uint64_t k = 0; k < w2; ++k) {                                   \
          const E* p = mid + (j + 1) * P2 + (k + 1);                          \
          const int ch = is2d ? CH2(p, (ptrdiff_t)plane, (ptrdiff_t)P2)       \
                              : CH3(p, (ptrdiff_t)plane, (ptrdiff_t)P2);      \
          out[(i * w1 + j) * w2 + k] = (int8_t)ch;                            \
        }                                                                     \
    }                                                                         \
    free(win);                                                                \
    return 0;                                                                 \
  }

/* In 2D the reference stencil runs over axes 0 and 1 (kernel.hpp:81-94,
 * 202-207): strides s0 = padded plane, s1 = padded row of width 3 -> here
 * the row stride of the (w1+2) x 3 padded plane is P2 = 3, and the centre
 * sits at column 1, so p[+-s1] moves along axis 1.                        */
ECC_CHANGES(ecc_oracle_changes_u8, uint8_t, int32_t, 256, change_2d_int32_t,
            change_3d_int32_t)
ECC_CHANGES(ecc_oracle_changes_u16_as_f32, uint16_t, float, INFINITY,
            change_2d_float, change_3d_float)
ECC_CHANGES(ecc_oracle_changes_f32, float, float, INFINITY, change_2d_float,
            change_3d_float)

/* ---------------------------------------------------------------------- */
/* Dense histogram for integer images: accumulate_dense_u8 (kernel.hpp:
 * 268-277) generalised to 2^bits bins; `count` records occupancy
 * (ValueIndex<uint8_t>::build, value_index.hpp:63-71).                   */

int ecc_oracle_vcec_u8(const uint8_t* img, uint64_t w0, uint64_t w1,
                       uint64_t w2, int64_t* hist /*256*/,
                       int64_t* count /*256*/) {
  const uint64_t n = w0 * w1 * w2;
  int8_t* ch = (int8_t*)malloc(n ? n : 1);
  if (!ch) return -1;
  if (ecc_oracle_changes_u8(img, w0, w1, w2, ch)) { free(ch); return -1; }
  memset(hist, 0, 256 * sizeof(int64_t));
  memset(count, 0, 256 * sizeof(int64_t));
  for (uint64_t i = 0; i < n; ++i) { hist[img[i]] += ch[i]; count[img[i]]++; }
  free(ch);
  return 0;
}

int ecc_oracle_vcec_u16(const uint16_t* img, uint64_t w0, uint64_t w1,
                        uint64_t w2, int64_t* hist /*65536*/,
                        int64_t* count /*65536*/) {
  const uint64_t n = w0 * w1 * w2;
  int8_t* ch = (int8_t*)malloc(n ? n : 1);
  if (!ch) return -1;
  if (ecc_oracle_changes_u16_as_f32(img, w0, w1, w2, ch)) { free(ch); return -1; }
  memset(hist, 0, 65536 * sizeof(int64_t));
  memset(count, 0, 65536 * sizeof(int64_t));
  for (uint64_t i = 0; i < n; ++i) { hist[img[i]] += ch[i]; count[img[i]]++; }
  free(ch);
  return 0;
}

/* f32: build_index_counts (value_index.hpp:159-197): records
 * (order_key << 32 | position) sorted by key, runs reduced to
 * (distinct value, summed change), -0 folded into +0.  qsort replaces the
 * LSD radix sort; the result is identical because only the key order and
 * the per-key sums matter.  Returns the number of distinct values.       */
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

int64_t ecc_oracle_vcec_f32(const float* img, uint64_t w0, uint64_t w1,
                            uint64_t w2, float* values, int64_t* changes) {
  const uint64_t n = w0 * w1 * w2;
  if (n == 0) return -1;
  for (uint64_t i = 0; i < n; ++i)
    if (isnan(img[i])) return -2; /* ValueIndex<float>::build rejects NaN */
  int8_t* ch = (int8_t*)malloc(n);
  uint64_t* rec = (uint64_t*)malloc(n * 8);
  if (!ch || !rec) { free(ch); free(rec); return -1; }
  ecc_oracle_changes_f32(img, w0, w1, w2, ch);
  for (uint64_t i = 0; i < n; ++i)
    rec[i] = ((uint64_t)ecc_oracle_float_order_key(img[i]) << 32) |
             (uint64_t)(uint8_t)(ch[i] + 16);
  qsort(rec, n, 8, cmp_u64);
  int64_t m = -1;
  uint32_t prev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t key = (uint32_t)(rec[i] >> 32);
    const int c = (int)(rec[i] & 0xFF) - 16;
    if (m < 0 || key != prev) {
      ++m;
      values[m] = ecc_oracle_float_from_order_key(key);
      changes[m] = 0;
      prev = key;
    }
    changes[m] += c;
  }
  free(ch);
  free(rec);
  return m + 1;
}

/* vcec_to_ecc: curve.hpp:28-35 (sequential int64 prefix sum). */
void ecc_oracle_prefix_sum(const int64_t* changes, int64_t* chi, uint64_t m) {
  int64_t acc = 0;
  for (uint64_t i = 0; i < m; ++i) { acc += changes[i]; chi[i] = acc; }
}

/* ---------------------------------------------------------------------- */
/* Pipeline inputs: uniform_noise datagen.hpp:57-62
 * with counter_uniform :30-32; gaussian_smooth :108-122 = gaussian_kernel
 * :66-79 + convolve_axis :80-105 along axes 0, 1, 2 (skipped when the axis
 * extent or the width is 1), edge-clamped, double accumulation in tap order,
 * rounded to float.  Built as ISO C (no FMA contraction), like the reference. */

void ecc_oracle_uniform_noise(float* dst, uint64_t n, uint64_t seed) {
  for (uint64_t i = 0; i < n; ++i)
    dst[i] = (float)(ecc_oracle_counter_hash(seed, i) >> 40) * 0x1p-24f;
}

/* returns -1 for an invalid width (even or < 1) */
int ecc_oracle_gaussian_smooth(const float* in, float* out, uint64_t w0, uint64_t w1,
                               uint64_t w2, double sigma, int width) {
  if (width < 1 || width % 2 == 0) return -1;
  const int half = width / 2;
  double* kern = (double*)malloc(sizeof(double) * (size_t)width);
  double sum = 0;
  for (int i = -half; i <= half; ++i) {
    const double v = width == 1 ? 1.0 : exp(-((double)i * i) / (2.0 * sigma * sigma));
    kern[i + half] = v;
    sum += v;
  }
  for (int i = 0; i < width; ++i) kern[i] /= sum;
  const uint64_t n = w0 * w1 * w2;
  const uint64_t ext[3] = {w0, w1, w2};
  const uint64_t stride[3] = {w1 * w2, w2, 1};
  float* cur = (float*)malloc(sizeof(float) * (n ? n : 1));
  float* nxt = (float*)malloc(sizeof(float) * (n ? n : 1));
  memcpy(cur, in, sizeof(float) * n);
  for (int axis = 0; axis < 3; ++axis) {
    const uint64_t aw = ext[axis], as = stride[axis];
    if (!(aw > 1 && width > 1)) continue;
    for (uint64_t i = 0; i < n; ++i) {
      const int64_t pos = (int64_t)((i / as) % aw);
      double acc = 0;
      for (int k = -half; k <= half; ++k) {
        int64_t q = pos + k;
        if (q < 0) q = 0;
        if (q > (int64_t)aw - 1) q = (int64_t)aw - 1;
        acc += kern[k + half] * (double)cur[i + (uint64_t)(q - pos) * as];
      }
      nxt[i] = (float)acc;
    }
    float* t = cur;
    cur = nxt;
    nxt = t;
  }
  memcpy(out, cur, sizeof(float) * n);
  free(cur);
  free(nxt);
  free(kern);
  return 0;
}
