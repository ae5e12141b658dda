// fin_u8.cuh -- the end of every u8 bit-sliced kernel (k_u8_3d.cu,
// k_u8_2d.cu): reduce the CTA's (code, value) shared-memory table to
// per-value change sums and pixel counts, flush them with int64 global
// atomics, and -- when a finalize workspace is passed -- let the last CTA
// to finish turn the global histogram into the curve in the same launch
// (merge_local + vcec_to_ecc, vcec.hpp:35-66, curve.hpp:28-35), re-zeroing
// the histogram and the ticket for the next launch.
#pragma once
#include <cstdint>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

namespace eccb {
namespace u8fin {

// Rank exchange over peer memory (multi-GPU z-slab sharding, SURVEY.md
// 8(e)): the last CTA of every rank stores its rank's 512-entry histogram
// into slot [parity][rank] of EVERY rank's exchange buffer (NVLink P2P
// stores through CUDA-IPC mappings), releases a per-(parity, rank) flag
// there, waits for all ranks' flags in its own buffer, and runs K3 on the
// sum -- the all-reduce fused into the stencil launch.  The parity double
// buffer keeps a rank that is one step ahead from overwriting slots a
// slower rank is still reading.
struct Xchg {
  int world = 1, rank = 0;
  uint32_t epoch = 0;           // this launch's step number (flags hold it)
  int64_t* const* slots = nullptr;   // [world] -> peer's int64[2][world][512]
  uint32_t* const* flags = nullptr;  // [world] -> peer's uint32[2][world]
  const int64_t* my_slots = nullptr;
  const uint32_t* my_flags = nullptr;
  uint32_t* err = nullptr;      // mapped host word: set when a peer never arrives (timeout)
};

struct Fin {
  uint32_t* ticket;    // zero before the launch, zero again after it
  uint32_t* bins;      // [256] occurring values, ascending
  int64_t* changes;    // [256] their VCEC entries
  int64_t* chi;        // [256] the curve
  uint64_t* count;     // number of occurring values
  Xchg x;              // world > 1: fused rank exchange
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Code: static constexpr int n (codes per value in the table);
//       static __device__ bool live(int c) (a real change, not "not emitted");
//       static __device__ int change(int c).
// ghist: [256] change sums then [256] pixel counts.
// REP: the table is replicated REP times (entry e at words e * REP .. + REP-1,
// one replica per group of 32 / REP lanes, to spread the shared-memory banks).
template <int NT, class Code, int REP = 1>
__device__ __forceinline__ void flush_and_finalize(const uint32_t* hist, int64_t* ghist,
                                                   const Fin& fin) {
  static_assert(256 % NT == 0 || NT >= 256, "NT must divide 256 or be at least 256");
  __syncthreads();
  for (int v = threadIdx.x; v < 256; v += NT) {
    long long sum = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < Code::n; ++c) {
      if (!Code::live(c)) continue;
      long long n = 0;
#pragma unroll
      for (int r = 0; r < REP; ++r) n += hist[(c * 256 + v) * REP + r];
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
  const Xchg& x = fin.x;
  const int par = (int)(x.epoch & 1u);
  if (x.world > 1) {
    // publish this rank's histogram into every rank's slot [par][rank]
    for (int r = 0; r < x.world; ++r) {
      int64_t* dst = x.slots[r] + ((size_t)par * x.world + x.rank) * 512;
      for (int v = threadIdx.x; v < 512; v += NT) dst[v] = __ldcg(&ghist[v]);
    }
    __threadfence_system();
    __syncthreads();
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
      timed_out = 0;
      for (int r = 0; r < x.world; ++r) st_release_sys(x.flags[r] + par * x.world + x.rank, x.epoch);
      // wait for every rank's data in our own buffer (10 s guard: never hang)
      const uint64_t t0 = globaltimer();
      for (int r = 0; r < x.world && !timed_out; ++r)
        while (ld_acquire_sys(x.my_flags + par * x.world + r) != x.epoch) {
          if (globaltimer() - t0 > 10000000000ull) {
            timed_out = 1;
            break;
          }
        }
    }
    __syncthreads();
    if (timed_out) {
      // no partial curve: the count is poisoned (the host API rejects a
      // count above 256), the flag is raised in mapped host memory so the
      // NEXT ecc_curve_sharded call fails without a device round trip, and
      // the workspace is re-zeroed like on the normal path
      for (int v = threadIdx.x; v < 512; v += NT) ghist[v] = 0;
      if (threadIdx.x == 0) {
        *fin.count = ~0ull;
        *reinterpret_cast<volatile uint32_t*>(x.err) = 1u;
        __threadfence_system();
        *fin.ticket = 0;
      }
      return;
    }
  }
  // the global histogram: this launch's (one rank) or the sum of all ranks'
  auto gsum = [&](int v) -> long long {
    if (x.world <= 1) return __ldcg(&ghist[v]);
    long long t = 0;
    for (int r = 0; r < x.world; ++r)
      t += __ldcg(&x.my_slots[((size_t)par * x.world + r) * 512 + v]);
    return t;
  };
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
    s[j] = mine ? gsum(v0 + j) : 0;
    n[j] = mine ? gsum(256 + v0 + j) : 0;
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

// Small images in ONE thread-block cluster (k_u8_2d's cluster path, one
// GPU): every CTA reduces its table to per-value (sum, count) and stores
// them straight into CTA 0's shared memory (distributed shared memory,
// fire-and-forget stores); after one cluster barrier CTA 0 sums the rows
// and writes the curve -- no global histogram, no atomics, no ticket, no
// L2 round trip.  `fin.ticket` and the global histogram stay untouched (zero).
constexpr int kMaxCluster = 16;
// first half of the "every CTA of the cluster has started" barrier; called
// by every thread at the kernel's start, completed in cluster_finalize
__device__ __forceinline__ void cluster_started_arrive() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
// rows: kMaxCluster x 256 sums then kMaxCluster x 256 counts (dynamic shared
// memory, cluster_rows_bytes).
constexpr int cluster_rows_bytes = 2 * kMaxCluster * 256 * 4;
template <int NT, class Code, int REP = 1>
__device__ __forceinline__ void cluster_finalize(const uint32_t* hist, int* rows, const Fin& fin) {
  static_assert(NT >= 256, "one thread per value");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  // rows [rank][value] of CTA 0's copy; int32: a cluster holds < 2^31 / 7 pixels
  int(*rows_s)[256] = reinterpret_cast<int(*)[256]>(rows);
  int(*rows_c)[256] = reinterpret_cast<int(*)[256]>(rows + kMaxCluster * 256);
  const unsigned rank = cluster.block_rank(), nb = cluster.num_blocks();
  __syncthreads();
  // CTA 0 must have started before its shared memory is written remotely:
  // the kernel arrived on the cluster barrier at its start
  // (cluster_started_arrive); this wait completes that phase
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  for (int v = threadIdx.x; v < 256; v += NT) {
    int sum = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < Code::n; ++c) {
      if (!Code::live(c)) continue;
      int n = 0;
#pragma unroll
      for (int r = 0; r < REP; ++r) n += (int)hist[(c * 256 + v) * REP + r];
      cnt += n;
      sum += n * Code::change(c);
    }
    *cluster.map_shared_rank(&rows_s[rank][v], 0) = sum;
    *cluster.map_shared_rank(&rows_c[rank][v], 0) = cnt;
  }
  cluster.sync();  // release / acquire: every CTA's row is in CTA 0
  if (rank != 0) return;
  struct Add {
    __device__ longlong2 operator()(const longlong2& a, const longlong2& b) const {
      return make_longlong2(a.x + b.x, a.y + b.y);
    }
  };
  using Scan = cub::BlockScan<longlong2, NT>;
  __shared__ typename Scan::TempStorage tmp;
  const int v = threadIdx.x;
  long long s = 0, n = 0;
  if (v < 256) {
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r)
      if (r < (int)nb) {
        s += rows_s[r][v];
        n += rows_c[r][v];
      }
  }
  longlong2 ex, total;
  Scan(tmp).ExclusiveScan(make_longlong2(n != 0, s), ex, make_longlong2(0, 0), Add(), total);
  if (n != 0) {
    fin.bins[ex.x] = v;
    fin.changes[ex.x] = s;
    fin.chi[ex.x] = ex.y + s;
  }
  if (threadIdx.x == 0) *fin.count = (uint64_t)total.x;
}

// A batch of images, one thread-block cluster per image (k_u8_2d's BATCH
// path): the same reduction into CTA 0, which writes the image's dense row
// chi[v] = sum_{v' <= v} change sums (int32, every value 0..255) and its
// occupancy bitmap -- the batched output format of k_batch.cu.
template <int NT, class Code, int REP = 1>
__device__ __forceinline__ void batch_finalize(const uint32_t* hist, int* rows, int32_t* chi_row,
                                               uint32_t* pres_row) {
  static_assert(NT >= 256, "one thread per value");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  int(*rows_s)[256] = reinterpret_cast<int(*)[256]>(rows);
  int(*rows_c)[256] = reinterpret_cast<int(*)[256]>(rows + kMaxCluster * 256);
  const unsigned rank = cluster.block_rank(), nb = cluster.num_blocks();
  __syncthreads();
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // CTA 0 has started
  for (int v = threadIdx.x; v < 256; v += NT) {
    int sum = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < Code::n; ++c) {
      if (!Code::live(c)) continue;
      int n = 0;
#pragma unroll
      for (int r = 0; r < REP; ++r) n += (int)hist[(c * 256 + v) * REP + r];
      cnt += n;
      sum += n * Code::change(c);
    }
    *cluster.map_shared_rank(&rows_s[rank][v], 0) = sum;
    *cluster.map_shared_rank(&rows_c[rank][v], 0) = cnt;
  }
  cluster.sync();
  if (rank != 0) return;
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  const int v = threadIdx.x;
  int32_t s = 0, n = 0;
  if (v < 256) {
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r)
      if (r < (int)nb) {
        s += rows_s[r][v];
        n += rows_c[r][v];
      }
  }
  int32_t incl;
  Scan(tmp).InclusiveSum(s, incl);
  if (v < 256) {
    chi_row[v] = incl;
    const uint32_t word = __ballot_sync(0xFFFFFFFFu, n != 0);
    if ((v & 31) == 0) pres_row[v >> 5] = word;
  }
}

}  // namespace u8fin
}  // namespace eccb
