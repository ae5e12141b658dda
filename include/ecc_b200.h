/*
 * ecc_b200.h -- C ABI of the B200-native Euler-characteristic-curve engine.
 *
 * This is the drop-in boundary for the reference's hot path.
 * The reference (/root/reference/proj/include/ecc) has no C ABI: it is a
 * header-only C++20 library.  Every entry point below replaces one reference
 * call (cited as file:line relative to proj/include/ecc/), and the C++
 * drop-in headers in include/ecc/ re-expose the reference signatures on top
 * of these functions.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers documented as "device" are CUDA
 *    device pointers on the context's GPU; "host" pointers may be pageable or
 *    pinned.  `stream` is a cudaStream_t passed as void* (NULL = the
 *    context's own stream).
 *  - Every function returns ECC_OK (0) or a negative status; the message of
 *    the last failure on the calling thread is available from
 *    ecc_last_error().  The C++ headers rethrow it as ecc::error with the
 *    reference's wording (common.hpp:11-14).
 *  - Axis 0 (w0) is the slowest axis, axis 2 (w2) the contiguous one; a 2D
 *    image is w2 == 1 (common.hpp:16-31).
 *  - There is no CPU fallback: if the CUDA library or a GPU is missing the
 *    calls fail with ECC_ECUDA.
 */
#ifndef ECC_B200_H_
#define ECC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECC_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define ECC_API __attribute__((visibility("default")))
#else
#define ECC_API
#endif

enum {
  ECC_OK = 0,
  ECC_EINVAL = -1,   /* bad argument / invalid plan (streaming.hpp:186-195) */
  ECC_ECUDA = -2,    /* CUDA runtime or launch failure, or no device */
  ECC_ENOMEM = -3,   /* device or pinned allocation failed */
  ECC_ESOURCE = -4,  /* read_rows callback failed (streaming.hpp:250-259) */
  ECC_EBINMAP = -5,  /* a value does not fit the requested bin map */
  ECC_ENAN = -6      /* NaN input (value_index.hpp:29-30, image.hpp:45-48) */
};

/* Element type of the image.  u8 and f32 are the reference's ValueKind
 * (common.hpp:43); u16 is the extension BASELINE config 3 needs, with the
 * reference f32 path as its parity target. */
typedef enum { ECC_U8 = 0, ECC_U16 = 1, ECC_F32 = 2 } ecc_dtype;

typedef struct {
  uint64_t w0, w1, w2;
} ecc_dims;

/* Value -> histogram-bin map; replaces ValueIndex (value_index.hpp:23-85).
 *  ECC_BIN_IDENTITY : u8/u16, bin = value (256 / 65536 bins).
 *  ECC_BIN_AFFINE   : f32 quantised to a grid, bin = (v - lo) / step, which
 *                     must be an exact integer in [0, nbins) and map back to
 *                     v (checked on the device; failure -> ECC_EBINMAP).
 *  ECC_BIN_SORTED   : general f32: distinct values found by a device radix
 *                     sort + reduce-by-key (build_index_counts,
 *                     value_index.hpp:159-197). */
enum { ECC_BIN_IDENTITY = 0, ECC_BIN_AFFINE = 1, ECC_BIN_SORTED = 2 };

typedef struct {
  int32_t kind;
  uint32_t nbins; /* AFFINE only */
  float lo;       /* AFFINE only */
  float step;     /* AFFINE only */
} ecc_binmap;

/* Per-chunk phase times in seconds since the call began (ChunkTiming,
 * streaming.hpp:83-89).  ingest = read_rows + H2D, kernel = stencil +
 * histogram on the device, merge = device histogram reduction. */
typedef struct {
  uint64_t begin, end;
  double ingest_begin, ingest_end;
  double index_begin, index_end;
  double kernel_begin, kernel_end;
  double merge_begin, merge_end;
} ecc_chunk_timing;

typedef struct ecc_ctx ecc_ctx;

/* ------------------------------------------------------------ context */
ECC_API int ecc_abi_version(void);
ECC_API const char* ecc_last_error(void);
/* One context per GPU; it owns a stream, scratch and pinned staging. */
ECC_API int ecc_ctx_create(int device, ecc_ctx** out);
ECC_API void ecc_ctx_destroy(ecc_ctx* ctx);
/* The context's own stream (cudaStream_t). */
ECC_API void* ecc_ctx_stream(ecc_ctx* ctx);
/* Number of my kernels launched by this context since creation. */
ECC_API uint64_t ecc_ctx_launch_count(ecc_ctx* ctx);

/* Number of histogram bins for (dtype, binmap); ECC_BIN_SORTED -> 0. */
ECC_API int ecc_bin_count(ecc_dtype dtype, const ecc_binmap* bm, uint64_t* nbins);

/* ------------------------------------------------------------ L2: slab kernels
 * A slab is the reference's PaddedChunk (chunk.hpp:50-127): owned rows
 * [own0, own1) along axis 0 plus one halo plane on each side when it exists
 * inside the image; outside the image the collar sentinel applies
 * (common.hpp:49-66).  `d_planes` holds image planes [plane0,
 * plane0 + nplanes) contiguously and must cover
 * [max(own0,1)-1, min(own1+1, w0)). */

/* Stencil + histogram (K1+K2): adds the slab's per-bin change sums to
 * d_hist[0..nbins) and per-bin voxel counts to d_hist[nbins..2*nbins)
 * (int64, device).  Replaces accumulate_dense_u8 (kernel.hpp:268-277),
 * run_chunk_kernel_u8 (streaming.hpp:146-174) and accumulate_chunk
 * (kernel.hpp:229-239).  Not valid for ECC_BIN_SORTED. */
ECC_API int ecc_accumulate_slab(ecc_ctx* ctx, const void* d_planes, ecc_dtype dtype,
                        ecc_dims image, uint64_t plane0, uint64_t nplanes,
                        uint64_t own0, uint64_t own1, const ecc_binmap* bm,
                        int64_t* d_hist, void* stream);

/* Per-voxel Euler changes of the owned rows, int8, owned row-major order
 * (compute_changes, kernel.hpp:244-265 with change_2d/change_3d/
 * change_row_3d, kernel.hpp:81-188).  d_out: device. */
ECC_API int ecc_compute_changes(ecc_ctx* ctx, const void* d_planes, ecc_dtype dtype,
                        ecc_dims image, uint64_t plane0, uint64_t nplanes,
                        uint64_t own0, uint64_t own1, int8_t* d_out,
                        void* stream);

/* ------------------------------------------------------------ L3: merge + curve
 * K3: compacts the occurring bins of a dense histogram (merge_local,
 * vcec.hpp:35-66) and prefix-sums them (vcec_to_ecc, curve.hpp:28-35).
 * Outputs are device arrays of capacity nbins; *d_count (device uint64) gets
 * the number of occurring bins. */
ECC_API int ecc_finalize(ecc_ctx* ctx, const int64_t* d_hist, uint64_t nbins,
                 uint32_t* d_bins, int64_t* d_changes, int64_t* d_chi,
                 uint64_t* d_count, void* stream);

/* Device-resident whole image -> curve in device buffers: process_image
 * (streaming.hpp:332-338) + vcec_to_ecc (curve.hpp:28-35) for an image that
 * is already in HBM.  3D u8 volumes whose rows are a multiple of 16 bytes
 * take ONE fused launch (stencil + histogram + compaction + prefix sum in
 * the last CTA); other shapes take memset + K1/K2 + K3.  d_bins (uint32),
 * d_changes / d_chi (int64) have capacity ecc_bin_count(); *d_count (device
 * uint64) receives the number of occurring values.  Not valid for
 * ECC_BIN_SORTED.  One call in flight per context. */
ECC_API int ecc_curve_device(ecc_ctx* ctx, const void* d_data, ecc_dtype dtype, ecc_dims dims,
                     const ecc_binmap* bm, uint32_t* d_bins, int64_t* d_changes,
                     int64_t* d_chi, uint64_t* d_count, void* stream);

/* ------------------------------------------------------------ L4: whole images
 * process_image(const Image<T>&, plan) (streaming.hpp:332-338) + the VCEC
 * result.  `data` is host (where = 0) or device (where = 1).  Outputs are
 * host arrays: values_out (dtype elements) and changes_out (int64), capacity
 * `cap`; *n_out = number of occurring values.  The result is independent of
 * any chunking (acceptance.cpp:203-227), so no plan is taken. */
ECC_API int ecc_vcec(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype,
             ecc_dims dims, const ecc_binmap* bm, void* values_out,
             int64_t* changes_out, uint64_t cap, uint64_t* n_out);

/* Same, returning the curve (vcec_to_ecc): thresholds + chi. */
ECC_API int ecc_curve(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype,
              ecc_dims dims, const ecc_binmap* bm, void* thresholds_out,
              int64_t* chi_out, uint64_t cap, uint64_t* n_out);

/* ------------------------------------------------------------ L4: streaming
 * process_image(ChunkSource<T>&, const ChunkPlan&, ...) (streaming.hpp:
 * 181-329).  Rows arrive through `read_rows` (ChunkSource::read_rows,
 * chunk.hpp:131-137), which fills `dst` (pinned host staging) with image
 * rows [r0, r1) and returns 0, or nonzero with a message in errbuf.
 * `bounds` holds nchunks+1 ascending row indices (the plan's ranges).
 * Ingestion of chunk k+1 overlaps the device work of chunk k. */
typedef int (*ecc_read_rows_fn)(void* user, uint64_t r0, uint64_t r1,
                                void* dst, char* errbuf, size_t errlen);

ECC_API int ecc_process_stream(ecc_ctx* ctx, ecc_read_rows_fn read_rows, void* user,
                       ecc_dtype dtype, ecc_dims dims, const uint64_t* bounds,
                       size_t nchunks, const ecc_binmap* bm,
                       ecc_chunk_timing* timings, void* values_out,
                       int64_t* changes_out, uint64_t cap, uint64_t* n_out);

/* process_image over a plan for an image that is already in HOST memory
 * (streaming.hpp:181-338 with a MemorySource, chunk.hpp:139-152): each
 * chunk's rows [own0 - 1, own1 + 1) are copied by DMA straight from `host`
 * (page-locked memory gives full-speed asynchronous copies; pageable memory
 * works but each copy then blocks) on the copy stream into one of three
 * device slab buffers while the previous chunks' kernels run.  No
 * read_rows callback and no staging copy.  Not valid for ECC_BIN_SORTED. */
ECC_API int ecc_process_host(ecc_ctx* ctx, const void* host, ecc_dtype dtype, ecc_dims dims,
                     const uint64_t* bounds, size_t nchunks, const ecc_binmap* bm,
                     ecc_chunk_timing* timings, void* values_out, int64_t* changes_out,
                     uint64_t cap, uint64_t* n_out);

/* process_image over a FileSource (chunk.hpp:154-189, image.hpp:39-52): a
 * raw row-major file of dtype elements with `dims` (size checked with the
 * reference's message), read chunk by chunk (pread into pinned staging,
 * overlapped with the previous chunk's device work).  For f32 the byte swap
 * of big-endian files and the NaN check run on the device after the copy; a
 * NaN fails the call with "ingestion of chunk k failed: NaN value at linear
 * index i" (the first chunk, in plan order, whose rows hold one). */
ECC_API int ecc_process_file(ecc_ctx* ctx, const char* path, ecc_dtype dtype, ecc_dims dims,
                     int big_endian, const uint64_t* bounds, size_t nchunks,
                     const ecc_binmap* bm, ecc_chunk_timing* timings, void* values_out,
                     int64_t* changes_out, uint64_t cap, uint64_t* n_out);

/* ------------------------------------------------------------ sharded streaming
 * a rank's share of a host image (C5 on several GPUs).
 * Accumulates the owned planes [bounds[0], bounds[nchunks]) into the device
 * histogram d_hist (int64[2 * nbins] as in ecc_accumulate_slab; NOT zeroed
 * here) chunk by chunk with the pipelined DMA of ecc_process_host: chunk k
 * owns [bounds[k], bounds[k+1]) and its halo planes come from the same host
 * buffer, which holds image planes [plane0, plane0 + nplanes).  The bounds
 * must increase within [0, w0] but need not start at 0 or end at w0 (each
 * rank passes its own range); combine ranks with one all-reduce of d_hist and
 * ecc_finalize.  Synchronous.  Replaces, per rank, the reference's
 * process_image over a chunk plan (streaming.hpp:181-329). */
ECC_API int ecc_accumulate_host(ecc_ctx* ctx, const void* host_planes, uint64_t plane0,
                                uint64_t nplanes, ecc_dtype dtype, ecc_dims image,
                                const uint64_t* bounds, size_t nchunks, const ecc_binmap* bm,
                                int64_t* d_hist);

/* ------------------------------------------------------------ fused multi-GPU exchange
 * z-slab sharding with the all-reduce fused into the stencil
 * launch.  Each rank creates an exchange buffer (ecc_xchg_create; the 64-byte
 * CUDA-IPC handle it returns is all-gathered by the caller, e.g. through
 * torch.distributed), opens its peers' buffers (ecc_xchg_open), then
 * ecc_curve_sharded runs K1+K2 over its slab and, in the same launch, the
 * last CTA stores the rank's histogram into every peer's buffer over NVLink,
 * waits for all ranks and runs K3 on the sum: every rank ends with the
 * global curve in d_bins / d_changes / d_chi / d_count (as ecc_curve_device).
 * 3D u8 slabs (the C2 path).  All ranks must call ecc_curve_sharded the same
 * number of times; ecc_xchg_status reports a peer that never arrived (10 s
 * guard inside the kernel instead of a hang).  Replaces the reference's
 * per-chunk merge_local (vcec.hpp:35-66) across devices. */
typedef struct ecc_xchg ecc_xchg;
ECC_API int ecc_xchg_create(ecc_ctx* ctx, int rank, int world, ecc_xchg** out,
                            void* handle_out /* 64 bytes */);
ECC_API int ecc_xchg_open(ecc_xchg* x, const void* handles /* world x 64 bytes */);
ECC_API void ecc_xchg_destroy(ecc_xchg* x);
ECC_API int ecc_xchg_status(ecc_xchg* x);
ECC_API int ecc_curve_sharded(ecc_ctx* ctx, ecc_xchg* x, const void* d_planes, ecc_dims image,
                              uint64_t plane0, uint64_t nplanes, uint64_t own0, uint64_t own1,
                              uint32_t* d_bins, int64_t* d_changes, int64_t* d_chi,
                              uint64_t* d_count, void* stream);

/* ------------------------------------------------------------ batched 2D
 * New entry point (the reference has none): `count` images of
 * h x w (axis 0 = h), stored back to back.  For each image b, writes the
 * dense curve chi[b][t] = chi(K_<=t) for every bin t (int32; 256 or 65536
 * bins) and a presence bitmap presence[b][t/32] (bit t%32 set iff value t
 * occurs).  data/chi/presence are all device (where = 1) or all host
 * (where = 0). */
ECC_API int ecc_batch2d(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype,
                uint64_t count, uint64_t h, uint64_t w, int32_t* chi,
                uint32_t* presence, void* stream);

/* ------------------------------------------------------------ batched curve files
 * write_curve (curve.hpp:87-121) for every image of a
 * dense batch (ecc_batch2d's device outputs d_chi / d_presence, dtype u8 or
 * u16 thresholds), formatted on the device: format 0 = CSV
 * ("threshold,euler_characteristic\n" + "t,chi\n" per occurring bin),
 * 1 = JSON ("[{"t":T,"chi":C},...]\n"), byte-identical to the reference
 * writer.  offsets (host, count + 1) gets each image's byte range in the
 * output and *total the size; with out == NULL the call only sizes,
 * otherwise out (host, cap >= *total) receives the bytes. */
ECC_API int ecc_batch_format(ecc_ctx* ctx, const int32_t* d_chi, const uint32_t* d_presence,
                             uint64_t count, ecc_dtype dtype, int format, char* out,
                             uint64_t cap, uint64_t* offsets, uint64_t* total);

/* zero_crossings (curve.hpp:36-50) of every image of a dense batch, on the
 * device: bit t of d_out[b] (uint32[count][nbins/32]) is set iff occurring
 * bin t of image b has chi == 0 or a strict sign change from the image's
 * previous occurring point. */
ECC_API int ecc_batch_zero_crossings(ecc_ctx* ctx, const int32_t* d_chi,
                                     const uint32_t* d_presence, uint64_t count, ecc_dtype dtype,
                                     uint32_t* d_out, void* stream);

/* ------------------------------------------------------------ synthetic inputs
 * Device fill with the reference generator (datagen.hpp:18-27): element i
 * gets counter_hash(seed, base + i) >> 56 (u8), >> 48 (u16) or
 * float(H >> 48) * 2^-16 (f32).  Used by the bench and tests. */
ECC_API int ecc_fill_synthetic(ecc_ctx* ctx, void* d_data, ecc_dtype dtype,
                       uint64_t n, uint64_t seed, uint64_t base, void* stream);

/* ------------------------------------------------------------ pipeline
 * The reference's in-memory benchmark, GPU-resident.
 *
 * ecc_uniform_noise: d_out[i] = counter_uniform(seed, i) = (counter_hash(seed, i) >> 40) * 2^-24
 *   (uniform_noise, datagen.hpp:57-62; counter_uniform :30-32), bit-identical.
 * ecc_gaussian_smooth: separable Gaussian smoothing with a normalised sampled
 *   kernel and edge clamping (gaussian_smooth datagen.hpp:108-122, convolve_axis
 *   :80-105, gaussian_kernel :66-79), bit-identical floats; d_in may equal d_out.
 *   Errors: "Gaussian kernel width must be odd and >= 1".
 * ecc_bench_run: bench_run (pipeline.hpp:236-291): uniform noise once, then
 *   `iterations` x {gaussian_smooth; process_image + vcec_to_ecc of the f32
 *   volume on the sorted (exact) path}, everything in device memory.  The
 *   report mirrors BenchReport (pipeline.hpp:212-233); smoothing / ECC times
 *   are CUDA-event device times, generate / total host wall time.  Errors:
 *   "bench needs at least one iteration". */
typedef struct {
  uint64_t iterations, voxels;
  double generate_s, total_s, per_iteration_s, ecc_avg_s, smooth_avg_s, ecc_gvox_per_s;
  uint64_t last_points;    /* points of the last iteration's curve */
  int64_t last_chi_first;  /* its chi at the lowest threshold */
  int64_t last_chi_last;   /* and at the highest (1 for any non-empty image) */
} ecc_bench_report;

ECC_API int ecc_uniform_noise(ecc_ctx* ctx, float* d_out, uint64_t n, uint64_t seed,
                              void* stream);
ECC_API int ecc_gaussian_smooth(ecc_ctx* ctx, const float* d_in, float* d_out, ecc_dims dims,
                                double sigma, int width, void* stream);
ECC_API int ecc_bench_run(ecc_ctx* ctx, ecc_dims dims, uint64_t iterations, uint64_t seed,
                          double sigma, int width, ecc_bench_report* report);

/* ------------------------------------------------------------ L1/L2: padded chunks
 * The reference's chunk-level API (kernel.hpp:32-74, 229-277,
 * value_index.hpp:23-197, vcec.hpp:35-66) on the device.  `padded` is a
 * PaddedChunk's host storage (chunk.hpp:50-127): (len+2) x (w1+2) x (w2+2)
 * extended values -- int16 for u8 (sentinel 256), int32 for u16 (65536),
 * float for f32 (+inf) -- with the one-voxel collar and the padding rows
 * begin-1 / end, len = end - begin.  The device evaluates the stencil on
 * exactly the stored values (collar and padding rows included), so a chunk
 * built by hand with set_padded behaves as in the reference.  Rows
 * [row_begin, row_end) are relative to the chunk (0 = row `begin`).  Host
 * outputs; synchronous. */
typedef struct {
  ecc_dims image;      /* the image the chunk belongs to */
  uint64_t begin, end; /* owned rows [begin, end) along axis 0 */
} ecc_chunk;

/* Per-voxel Euler changes of the owned voxels of rows [row_begin, row_end),
 * owned row-major order (compute_changes, kernel.hpp:244-265). */
ECC_API int ecc_chunk_changes(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                              uint64_t row_begin, uint64_t row_end, int8_t* out);

/* Per owned voxel, the FaceOffsets o it introduces (introduced(),
 * kernel.hpp:32-53): bit (o0+1)*9 + (o1+1)*3 + (o2+1), bit 13 never set.
 * 2D chunks are evaluated over their padded axis 2 as well, so offsets with
 * o2 != 0 meet the collar exactly as in the reference. */
ECC_API int ecc_chunk_faces(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                            uint64_t row_begin, uint64_t row_end, uint32_t* out);

/* Change sums per bin over the owned voxels of rows [row_begin, row_end):
 * index_values == NULL -> identity bins of the (narrowed) value, nbins = 256
 * (u8; accumulate_dense_u8, kernel.hpp:268-277) or 65536 (u16); otherwise the
 * bins of a value index (ValueIndex<float>, value_index.hpp:23-58): bin b is
 * index_values[b] (ascending, distinct, nbins of them) and every voxel value
 * must be one of them (accumulate_chunk, kernel.hpp:229-239; else
 * ECC_EBINMAP "value not present in index").  hist_out: nbins int64. */
ECC_API int ecc_chunk_accumulate(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                                 uint64_t row_begin, uint64_t row_end, const float* index_values,
                                 uint64_t nbins, int64_t* hist_out);

/* The occurring values of `values` (n elements of dtype, host), ascending and
 * distinct (f32: -0 folds onto +0, NaN -> ECC_ENAN "cannot build a value
 * index: NaN input"), and -- when `changes` (n int8, host) is given -- the
 * summed change of each (ValueIndex::build value_index.hpp:23-71,
 * build_index_counts :159-197: device radix sort + reduce-by-key).
 * values_out / sums_out: host, capacity cap; *n_out = distinct count (also
 * when it exceeds cap, with ECC_EINVAL). */
ECC_API int ecc_value_index(ecc_ctx* ctx, ecc_dtype dtype, const void* values, uint64_t n,
                            const int8_t* changes, void* values_out, int64_t* sums_out,
                            uint64_t cap, uint64_t* n_out);

/* Same over the owned voxels of a padded chunk (build_index_counts on its
 * owned voxels in owned row-major order, changes as compute_changes wrote
 * them). */
ECC_API int ecc_chunk_index_counts(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                                   const int8_t* changes, void* values_out, int64_t* sums_out,
                                   uint64_t cap, uint64_t* n_out);

/* merge_local (vcec.hpp:35-66) on the device: the global VCEC (gvals /
 * gchg, gn entries, ascending) plus, for every occurring value ivals[i] of a
 * chunk index (in entries, ascending), local[bin] where bin = the value for
 * u8 / u16 and i for f32; values new to the global list are inserted (zero
 * changes included).  Host arrays; out_* capacity cap (gn + in suffices). */
ECC_API int ecc_merge_local(ecc_ctx* ctx, ecc_dtype dtype, const void* gvals,
                            const int64_t* gchg, uint64_t gn, const int64_t* local,
                            uint64_t nlocal, const void* ivals, uint64_t in, void* out_vals,
                            int64_t* out_chg, uint64_t cap, uint64_t* n_out);

/* ------------------------------------------------------------ host-buffer helpers
 * The reference's host-facing generators and raw-file fixup with host arrays
 * in and out; the work runs on the device (the C++ headers' datagen.hpp,
 * image.hpp, FileSource::read_rows).  Synchronous.
 * ecc_uniform_noise_host: uniform_noise (datagen.hpp:57-62) into host memory.
 * ecc_gaussian_smooth_host: gaussian_smooth (datagen.hpp:108-122); in may equal out.
 * ecc_fixup_f32_host: fixup_loaded (image.hpp:39-52) in place: byte swap when
 *   big_endian, then ECC_ENAN "NaN value at linear index <base + i>" for the
 *   first NaN. */
ECC_API int ecc_uniform_noise_host(ecc_ctx* ctx, float* out, uint64_t n, uint64_t seed);
ECC_API int ecc_gaussian_smooth_host(ecc_ctx* ctx, const float* in, float* out, ecc_dims dims,
                                     double sigma, int width);
ECC_API int ecc_fixup_f32_host(ecc_ctx* ctx, float* data, uint64_t n, uint64_t base,
                               int big_endian);

/* ------------------------------------------------------------ one curve's text on the device
 * write_curve (curve.hpp:87-121; mode 0 CSV, 1 JSON) or write_vcec
 * (curve.hpp:154-169; mode 2) of ONE curve / VCEC, formatted on the GPU and
 * byte-identical to the reference writers: thresholds / values of dtype
 * (u8 / u16 integers; f32 as the shortest round-trip text std::to_chars
 * prints, format_value curve.hpp:56-66) and int64 chi / changes, n points,
 * host (where = 0) or device (where = 1) arrays.  `out` (host) receives the
 * bytes; *size_out = their count (also when it exceeds cap, with ECC_EINVAL). */
ECC_API int ecc_format_curve(ecc_ctx* ctx, ecc_dtype dtype, const void* thresholds,
                             const int64_t* chi, uint64_t n, int where, int mode, char* out,
                             uint64_t cap, uint64_t* size_out);

#ifdef __cplusplus
}
#endif

#endif /* ECC_B200_H_ */
