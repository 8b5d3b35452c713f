/*
 * mdrq_b200.h -- C ABI of the B200-native MDRQ scan engine (libmdrq_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as opaque `void*` = cudaStream_t, NULL = the store's
 * own stream).  Every call returns MDRQ_OK (0) or a negative status; the
 * message of the last failure on the calling thread is mdrq_last_error().
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/mdrq/):
 *
 *   Kernel-backend level (kernels.py:34-46, the MDRQ_BACKEND plugin slot):
 *     mdrq_match_rows   <- _kernels_cy.pyx:49-55  match_row (batched)
 *     mdrq_scan_rows    <- _kernels_cy.pyx:58-86  scan_rows
 *     mdrq_scan_column  <- _kernels_cy.pyx:89-120 scan_column
 *     mdrq_and_masks    <- scan.py:55-78          and_masks_chunked
 *     mdrq_mask_popcount<- scan.py:81-82          mask_popcount
 *     mdrq_mask_to_ids  <- scan.py:85-88          mask_to_ids
 *
 *   Access-method level (methods.py:20-47 build_method + the AccessMethod
 *   protocol .search / .search_with_stats of scan.py:91-214, vafile.py:88-219):
 *     mdrq_store_create   <- SequentialScan/VerticalScan.__init__ (scan.py:94,
 *                            174-181), ColumnSet.from_dataset (scan.py:35-37),
 *                            VaFile.build (vafile.py:106-147)
 *     mdrq_query_count    <- len(method.search(q))  (bench.py:176)
 *     mdrq_query_ids      <- method.search(q).ids   (scan.py:103-111, 187-211,
 *                            vafile.py:201-219)
 *     mdrq_query_ids64    <- the same as int64, ResultSet's dtype (core.py:185)
 *     mdrq_query_stats    <- SearchStats counters of search_with_stats
 *                            (core.py:218-237)
 *     mdrq_store_va_boundaries <- VaGrid (vafile.py:25-64) -- here a quantile
 *                            grid, see DESIGN.md
 */
#ifndef MDRQ_B200_H
#define MDRQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDRQ_ABI_VERSION 1

/* status codes */
#define MDRQ_OK          0
#define MDRQ_EINVAL     -1   /* bad argument (maps to ValueError)            */
#define MDRQ_ECUDA      -2   /* CUDA runtime failure (RuntimeError)          */
#define MDRQ_ENOMEM     -3   /* device/host allocation failed (MemoryError)  */
#define MDRQ_ETRUNC     -4   /* output buffer too small; *total holds need   */
#define MDRQ_ENODEV     -5   /* no CUDA device / bad ordinal                 */

/* store layouts (bit set) */
#define MDRQ_LAYOUT_COLUMNAR 1u   /* m contiguous float32 columns            */
#define MDRQ_LAYOUT_ROWWISE  2u   /* row-major float32 n x m                 */
#define MDRQ_LAYOUT_VAFILE   4u   /* per-dim quantile-grid codes (+columns)  */

/* query paths */
#define MDRQ_PATH_AUTO           0u
#define MDRQ_PATH_COLUMNAR       1u  /* one query per pass, dim-at-a-time, skip */
#define MDRQ_PATH_ROWWISE        2u  /* bulk-copy staged row tiles            */
#define MDRQ_PATH_VAFILE         3u  /* quantile-code filter + exact refine   */
#define MDRQ_PATH_COLUMNAR_BATCH 4u  /* many queries per pass over the columns */
#define MDRQ_PATH_VAFILE_BATCH   5u  /* bit-sliced: <= 1024 queries per pass over
                                        the VA code planes + exact refine    */

/* kernel modes (core.py:29-44 KernelMode; affect only early-break stats) */
#define MDRQ_MODE_SCALAR  0
#define MDRQ_MODE_BLOCKED 1

typedef struct mdrq_store mdrq_store;

typedef struct mdrq_store_info {
    uint64_t n;            /* tuples in this store (shard)                  */
    uint32_t m;            /* dimensions                                    */
    uint32_t layouts;      /* MDRQ_LAYOUT_* bits present                    */
    uint32_t va_bits;      /* bits per dimension of the VA-file codes (0 = none) */
    int32_t  device;       /* CUDA ordinal                                  */
    uint64_t n_pad;        /* padded tuple count of the device arrays       */
    uint64_t device_bytes; /* HBM held by the store (data + scratch)        */
} mdrq_store_info;

/* per-query counters, mirroring SearchStats (core.py:218-237) */
typedef struct mdrq_search_stats {
    uint64_t objects_compared;
    uint64_t nodes_visited;    /* VA-file: tuples refined (exact compares)  */
    uint64_t columns_scanned;
    uint64_t early_breaks;     /* row-wise path only                        */
    uint64_t and_chunks;       /* tiles the fused AND ran over              */
    uint64_t bytes_loaded;     /* HBM bytes the scan kernel requested: loads
                                  not skipped (single-query paths) or the
                                  union's planes / rows (multi-query passes,
                                  shared equally by the pass's queries)     */
} mdrq_search_stats;

/* -- library ------------------------------------------------------------ */
const char* mdrq_last_error(void);
/* Debug / test entry point: the failed device-side bounds checks since the
 * last call (bits per check kind, common.cuh), OR-ed over the library's units
 * and cleared; bit 31 is set when the library was built with the checks
 * (libmdrq_b200_checked.so, MDRQ_CHECKS).  Synchronises the device. */
int mdrq_check_flags(uint32_t* flags);

int mdrq_abi_version(void);
int mdrq_device_count(int* count);
/* Read-stream bandwidth probe (GB/s, best of iters) over a `bytes` buffer:
 * the roofline denominator beside MEASURED_PEAKS' copy figure (SURVEY.md
 * 8(d)).  Measurement utility, not part of the reference interface.       */
int mdrq_measure_read_bw(int device, uint64_t bytes, int iters, double* gbs);
/* Device-side segmented copy on `stream` (device pointers): segment i moves
 * len[i] uint32 from src + src_off[i] to dst + dst_off[i].  The multi-GPU
 * id merge places every rank's slice of every query with it (the
 * reference's concat + sort of per-partition results, parallel.py:156-157,
 * scan.py:160, without the sort).                                          */
int mdrq_copy_segments(const uint32_t* src, uint32_t* dst, const int64_t* src_off,
                       const int64_t* dst_off, const int64_t* len, uint64_t nseg,
                       void* stream);

/* The same segment placement with the copy engines, for a destination in
 * pinned (or registered) host memory: one asynchronous device-to-host copy
 * per segment (host arrays src_off / dst_off / len, in elements), enqueued on
 * `stream` (not the legacy default stream).  The multi-GPU host gather
 * (parallel.gather_ids_to_host) uses it: each rank's ids go to their
 * rank-ordered places over its own PCIe link at DMA speed. */
int mdrq_copy_segments_dma(const uint32_t* src, uint32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                           const int64_t* len, uint64_t nseg, void* stream);

/* -- kernel-backend level: host buffers in and out (parity / tests) ------ */
/* match_row for `nrows` rows against one query: out[r] = 1 match / 0 not.  */
int mdrq_match_rows(const float* rows, uint64_t nrows, uint32_t m,
                    const float* lower, const float* upper, int device,
                    uint8_t* out);
/* scan_rows: ascending local ids (int64, capacity n), match count, early
 * breaks under `mode` exactly as _kernels_cy.pyx:23-46 counts them.        */
int mdrq_scan_rows(const float* values, uint64_t n, uint32_t m,
                   const float* lower, const float* upper, int mode, int device,
                   int64_t* ids_out, uint64_t* count_out, uint64_t* early_out);
/* scan_column: little-endian packed bitmask of lo <= v <= hi, ceil(n/8) B. */
int mdrq_scan_column(const float* col, uint64_t n, float lo, float hi,
                     int device, uint8_t* mask_out);
/* AND of k masks of nbytes each (masks[j] are host pointers).              */
int mdrq_and_masks(const uint8_t* const* masks, uint32_t k, uint64_t nbytes,
                   int device, uint8_t* out);
int mdrq_mask_popcount(const uint8_t* mask, uint64_t nbytes, int device,
                       uint64_t* count_out);
/* positions of the set bits among the first n, ascending, int64.          */
int mdrq_mask_to_ids(const uint8_t* mask, uint64_t n, int device,
                     int64_t* ids_out, uint64_t* count_out);

/* -- device-resident store ------------------------------------------------ */
/* rows: host, row-major float32 n x m (NaN-free; checked by the caller's
 * DataSet).  id_base is added to every emitted id (row-sharded stores).    */
int mdrq_store_create(const float* rows, uint64_t n, uint32_t m, int device,
                      uint32_t layouts, uint32_t va_bits, uint64_t id_base,
                      mdrq_store** out);
int mdrq_store_destroy(mdrq_store* s);
int mdrq_store_get_info(const mdrq_store* s, mdrq_store_info* info);
/* VA-file boundaries, m x (2^va_bits - 1) float32, sorted per dimension.  */
int mdrq_store_va_boundaries(const mdrq_store* s, float* out);
/* observed per-dimension [min, max] (core.py:99-105), m x 2 float32.       */
int mdrq_store_bounds(const mdrq_store* s, float* out);

/* One batch of nq queries, lower/upper host float32 [nq][m] with the
 * reference's +-inf sentinels for unqueried dimensions (core.py:25-26,125). */
int mdrq_query_count(mdrq_store* s, const float* lower, const float* upper,
                     uint32_t nq, uint32_t path, uint64_t* counts);
/* ids mode: offsets[nq+1] (exclusive prefix), ids ascending per query.
 * When *total > ids_cap the call returns MDRQ_ETRUNC after filling offsets
 * and *total; the results stay cached and mdrq_fetch_ids() copies them.    */
int mdrq_query_ids(mdrq_store* s, const float* lower, const float* upper,
                   uint32_t nq, uint32_t path, uint64_t* offsets,
                   uint32_t* ids, uint64_t ids_cap, uint64_t* total);
int mdrq_fetch_ids(mdrq_store* s, uint32_t* ids, uint64_t ids_cap);
/* The same with the ids widened to int64 on the host, the dtype of the
 * reference's ResultSet (core.py:185, ResultSet.from_ids): the Python
 * search() builds its ResultSet straight from this buffer.  A call with
 * ids_cap == 0 returns MDRQ_ETRUNC with *total (the result stays cached,
 * small results in a pinned host buffer), so the caller can allocate exactly
 * *total ids and collect them with mdrq_fetch_ids64.                        */
int mdrq_query_ids64(mdrq_store* s, const float* lower, const float* upper,
                     uint32_t nq, uint32_t path, uint64_t* offsets,
                     int64_t* ids, uint64_t ids_cap, uint64_t* total);
int mdrq_fetch_ids64(mdrq_store* s, int64_t* ids, uint64_t ids_cap);
/* A stream of nbatches ids batches (replaces the reference's loop of
 * search_batch / search calls over successive query batches, bench.py:178-186,
 * methods.py search_batch): batch k holds nqs[k] queries, its bounds follow
 * batch k-1's in lower/upper.  Results go to offsets_out[k] (nqs[k]+1) and
 * ids_out[k] (capacity ids_caps[k]); totals[k] = its id count.  Batches are
 * pipelined: batch k's device->host copies overlap batch k+1's scan (three
 * slots with their own result pools, a copy stream).  Returns MDRQ_ETRUNC
 * when some totals[k] > ids_caps[k] (that batch's ids are not copied; the
 * rest are).  *h2d_bytes (optional) = query descriptor bytes uploaded.     */
int mdrq_query_ids_stream(mdrq_store* s, const float* lower, const float* upper,
                          const uint32_t* nqs, uint32_t nbatches, uint32_t path,
                          uint64_t* const* offsets_out, uint32_t* const* ids_out,
                          const uint64_t* ids_caps, uint64_t* totals,
                          uint64_t* h2d_bytes);

/* The stream's device->host copies are PCIe-bound on large results (C5:
 * 20 GB of ids per 10 000-query batch), so batches whose id lists are long
 * enough leave the device packed: the low 16 bits of every id (same order)
 * plus, per query, the end position of every 65 536-id bucket in its list;
 * the host rebuilds the uint32 ids on all its threads while the next batch
 * scans and the one after copies (MDRQ_STREAM_PACK=0 / 1 forces it off / on,
 * MDRQ_UNPACK_THREADS sets the thread count).  mdrq_unpack_ids16 is that
 * host step: out[offsets[q] + i] = (hb0 + b) << 16 | lo16[offsets[q] + i] for
 * ends[q][b-1] <= i < ends[q][b] (ends: nq x nbuckets, positions relative to
 * the query's list; offsets: nq + 1).  It needs no device.
 * A packed batch sends only a share of its queries packed and the rest raw;
 * the share follows the stream's measured step period (hill climbing: the
 * copy and the unpack share the host's memory bandwidth;
 * MDRQ_STREAM_PACK_SHARE fixes it, 0..1).
 * mdrq_stream_info: out[0] = device->host bytes of the store's last stream
 * call, out[1] = batches of it that were packed, out[2] = its batches,
 * out[3] = the current packed share of a batch's queries, in 1/1000.        */
int mdrq_unpack_ids16(const uint16_t* lo16, const uint32_t* ends, const uint64_t* offsets,
                      uint32_t nq, uint32_t hb0, uint32_t nbuckets, uint32_t* out, int threads);
int mdrq_stream_info(mdrq_store* s, uint64_t out[4]);
/* SearchStats of the last count/ids call, one entry per query.            */
int mdrq_query_stats(mdrq_store* s, int mode, mdrq_search_stats* stats,
                     uint32_t nq);

/* -- prepared (device-resident) batches: the timed path of bench.py ------ */
typedef struct mdrq_batch mdrq_batch;
int mdrq_batch_prepare(mdrq_store* s, const float* lower, const float* upper,
                       uint32_t nq, uint32_t path, mdrq_batch** out);
int mdrq_batch_destroy(mdrq_batch* b);
/* enqueue a count pass on `stream`; counts are device u64[nq] (no sync).   */
int mdrq_batch_count_async(mdrq_store* s, mdrq_batch* b, uint64_t* d_counts,
                           void* stream);
/* enqueue an ids pass on `stream` into the store's result buffers; no sync.
 * The output capacity is grown by mdrq_batch_reserve (a synchronising call). */
int mdrq_batch_ids_async(mdrq_store* s, mdrq_batch* b, void* stream);
/* run once synchronously, size the result buffers for this batch, and
 * report the total ids it produces.                                        */
int mdrq_batch_reserve(mdrq_store* s, mdrq_batch* b, uint64_t* total);
/* device pointers to the last ids pass: ids u32[total], offsets u64[nq+1]. */
int mdrq_result_device(mdrq_store* s, uint64_t* d_ids, uint64_t* d_offsets,
                       uint64_t* total);
/* number of kernels one count / ids pass of this batch launches.          */
int mdrq_batch_launches(mdrq_batch* b, int ids_mode, uint32_t* launches);
/* info[0] resolved path, [1] queries, [2] multi-query passes, [3] widest
 * union of dimensions over the passes (0 for single-query paths).         */
int mdrq_batch_info(mdrq_batch* b, uint32_t* info /*[4]*/);
/* run one pass with CUDA events between launch groups (synchronising) and
 * report per-class device time / kernel launches; classes: 0 scan / filter,
 * 1 ordered compaction, 2 id write (bit-sliced VA batch), 3 setup.          */
int mdrq_batch_profile(mdrq_store* s, mdrq_batch* b, int ids_mode, void* stream,
                       double* class_ms /*[4]*/, uint32_t* class_launches /*[4]*/);

#ifdef __cplusplus
}
#endif

#endif /* MDRQ_B200_H */
