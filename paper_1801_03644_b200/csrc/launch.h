// launch.h -- host-side launch wrappers shared between the kernel TUs and
// the C-ABI layer (store.cu).  Internal; not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace mdrq {

// Padding of the device arrays: every column / code plane holds n_pad
// entries, n_pad a multiple of kPadTuples; pad values are NaN (columns and
// rows) so they never satisfy lo <= v <= hi, codes are 0 (they are also
// masked by n).
constexpr uint64_t kPadTuples = 8192;
constexpr uint64_t kChunkTuples = 65536;  // compaction chunk (2048 mask words)

struct ScanArgs {
    const float* cols;       // columnar store [m][stride]
    const float* rows;       // row store [n_pad_rows][m]
    const uint8_t* codes;    // VA codes [m][stride]
    uint64_t stride;         // n_pad
    uint64_t n;              // live tuples
    uint32_t m;
    uint32_t rows_per_tile;  // row-wise tile height
    const QueryDesc* descs;  // device descriptors [nq]
    const DimPred* preds;    // device predicates, descs[q].off .. +k
    uint32_t q;              // query index of this launch
    uint32_t num_tiles;
    uint32_t* tile_counters; // [nq] zeroed per batch
    uint64_t* status;        // look-back status [num_tiles]
    uint32_t epoch;
    unsigned long long* counts;   // [nq]
    unsigned long long* offsets;  // [nq+1] ids mode (chained bases)
    uint32_t* ids;
    uint64_t ids_cap;
    uint32_t id_base;
    unsigned long long* stats;    // [nq][4]: early_scalar, early_blocked, refined, tiles
    // ids mode: the scan writes its verdicts as a bitmask + per-chunk counts,
    // launch_expand turns them into ordered ids (expand.cu)
    uint32_t* mask;               // [n_pad / 32] words
    uint32_t* chunk_counts;       // [n_pad / kChunkTuples], zeroed per query
    uint32_t* chunk_offs;         // [n_pad / kChunkTuples]
    // per-query accumulators spread over 32 slots (one CTA per tile would
    // otherwise serialise thousands of atomics on one address):
    // [nq][32][4] = count, bytes loaded, tuples refined, spare
    unsigned long long* partials;
    // single-query VA scan: track sure (strictly inside) tuples and refine
    // only edge cells -- set when the query is expected to return many tuples
    uint32_t va_sure;
};

constexpr int kPartialSlots = 32;

// add v to accumulator `field` of the launch's query (slot by CTA index)
__device__ __forceinline__ void partial_add(const ScanArgs& a, int field, unsigned long long v) {
    atomicAdd(a.partials + (uint64_t(a.q) * kPartialSlots + (blockIdx.x & (kPartialSlots - 1))) * 4 + field, v);
}

// fold the partial slots into counts (count mode) and stats[q][2..3]
void launch_reduce_partials(const unsigned long long* partials, uint32_t nq, bool add_counts,
                            unsigned long long* counts, unsigned long long* stats, cudaStream_t st);

// multi-query pass over the columnar store (union dims, <= 32 queries)
struct BatchArgs {
    const float* cols;
    uint64_t stride;
    uint64_t n;
    uint32_t kb;                 // union dims of this pass
    uint32_t nqp;                // queries in this pass (<= 32)
    const uint16_t* udims;       // [kb]
    const float2* bounds;        // [nqp][kb] (lo, hi), +-inf where unconstrained
    const unsigned long long* cmask;  // [nqp] constrained union dims (bit per union dim)
    unsigned long long* counts;  // [nqp] (already offset to the pass)
};

// bit-sliced multi-query VA pass (vabatch.cu), <= 1024 queries per pass
constexpr int kVaBatchMaxDims = 24;
// table cells per dimension for a pass with kb union dims (fits 227 KB smem)
// (11..16-dim unions use 32 cells so their on-chip bounds fit; 9 / 10 dims
// have room for 64 since their bounds are 15-bit codes)
#ifndef MDRQ_VB_Q15
#define MDRQ_VB_Q15 1
#endif
#ifndef MDRQ_VB_CELLS_WIDE
#define MDRQ_VB_CELLS_WIDE (MDRQ_VB_Q15 ? 64 : 32)
#endif
__host__ __device__ constexpr uint32_t va_batch_cells(uint32_t kb) {
    return kb <= 8 ? 64u : kb <= 10 ? uint32_t(MDRQ_VB_CELLS_WIDE) : 32u;
}
// Unions of kb <= kVbPvDims keep the exact query bounds in shared memory (and,
// up to 10 dims, the block's exact values) and refine every overlap candidate
// exactly, so their table is overlap-only: rows of dims (2p, 2p+1) at cell c
// are adjacent,
// word (u, c, w) at ((u/2 * cells + c) * 2 + u%2) * 32 + w.  Their exact
// bounds are [vdims/2][1024][2] float2 -- float4 (lo, hi of dims 2p, 2p+1)
// per dim pair p and query -- padded with (-inf, +inf).
// Wider unions use (overlap, containment) pairs [kb][cells][32][2] and refine
// only the edge-cell candidates from global memory.
constexpr uint32_t kVbPvDims = 16;   // values staged on chip up to 10 dims
__host__ __device__ constexpr bool va_batch_pv(uint32_t kb) { return kb <= kVbPvDims; }
__host__ __device__ constexpr uint32_t va_batch_vdims(uint32_t kb) {
    return kb <= 4 ? 4u : kb <= 8 ? 8u : (kb + 1) / 2 * 2;
}
__host__ __device__ constexpr uint32_t va_batch_table_words(uint32_t kb, uint32_t cells) {
    return va_batch_pv(kb) ? (kb + 1) / 2 * cells * 64 : kb * cells * 64;
}
// Staged unions (<= kVbStageDims dims: float32 values on chip up to 10 dims,
// their 15-bit codes above) refine on 15-bit
// monotone codes first (MDRQ_VB_Q15): value code c(v) = bits 8..22 of
// clamp(fma(v - vmin[u], vscale[u], 2)) in [1, 32766]; a query bound is the
// code of its lo / hi (0 / 32767 when it lies below / above every value), two
// dims per word with a guard bit per half.  c > L and c < H in every dim
// decides a candidate exactly (matches), c < L or c > H in some dim rejects
// it; only a code equal to a bound's falls back to the float32 compare
// against the exact bounds in global memory.  Per query the codes take
// vdims(kb) words (LN = 0x8000 - L per half for the vdims/2 dim pairs, then
// HG = 0x8000 + H): 40 bytes for 10 dims against 80 bytes of float bounds.
constexpr uint32_t kVbStageDims = 16;   // = kVbPvDims
__host__ __device__ constexpr bool va_batch_q15(uint32_t kb) { return MDRQ_VB_Q15 && kb <= kVbStageDims; }
constexpr float kVbQ15Min = 2.00006103515625f;    // 2 + 2^-14: code 1
constexpr float kVbQ15Max = 3.9998779296875f;     // 2 + 32766 * 2^-14: code 32766
// the code function, identical on host and device (monotone non-decreasing
// in v for scale > 0; NaN from inf - inf clamps to code 1 on both sides)
__host__ __device__ __forceinline__ float va_batch_q15_t(float v, float vmin, float scale) {
    return fminf(fmaxf(fmaf(v - vmin, scale, 2.0f), kVbQ15Min), kVbQ15Max);
}
struct VaBatchArgs {
    const uint8_t* codes;        // VA code planes [m][stride]
    const float* cols;           // exact columns [m][stride] (refinement)
    uint64_t stride;
    uint64_t n;
    uint32_t kb;                 // union dims of this pass (<= kVaBatchMaxDims)
    uint32_t cells;              // table cells per dim (2^tb: 32 or 64)
    uint32_t shift;              // stored code >> shift = table cell
    uint32_t nqp;                // queries in this pass (<= 1024)
    uint32_t lw;                 // lanes per tuple (32, or 16 / 8 for passes of <= 512 / 256 queries)
    const uint16_t* udims;       // [kb]
    const uint32_t* tables;      // query-mask words, layout per va_batch_pv(kb) (above)
    const float2* qbounds;       // exact (lo, hi), +-inf where unconstrained; layout per va_batch_pv(kb)
    const uint32_t* qcmask;      // [1024] constrained union dims per query (bit u)
    // Q15 refinement (staged unions): per query vdims words (LN pairs, HG
    // pairs) in 16-byte chunks [chunk][1024 slots] + an 8-byte tail
    // [1024 slots]; the code function's per-dim origin and scale
    const uint32_t* qb16;
    float vmin[kVbStageDims], vscale[kVbStageDims];
    uint32_t grid;               // CTAs (chunks = grid * warps)
    uint64_t chunk_tuples;       // tuples per chunk (multiple of 128, < 65536: u16 counters)
    uint32_t nchunks;            // subchunks: ceil(n / chunk_tuples), one warp each
    uint32_t ngroups;            // groups of kVbWarps consecutive subchunks, one CTA each
    unsigned long long* counts;  // [nqp] count mode (offset to the pass)
    uint32_t* chunk_counts;      // [groups][1024] (mode 2: [subchunks][1024] prefix scratch)
    unsigned long long* base;    // [groups][1024]
    unsigned long long* total;   // [1024]
    unsigned long long* qoff;    // [1024]
    unsigned long long* offsets;     // batch offsets [nq+1]
    unsigned long long* counts_all;  // batch counts [nq]
    uint32_t* ids;
    uint64_t ids_cap;
    uint32_t id_base;
    // single-pass ids (mode 3): (tuple offset << 10 | query) records staged in
    // 1024-record blocks allocated from a pool; each block is tagged with its
    // chunk and its ordinal in the chunk, and a block-list kernel puts the
    // pool in chunk order before the scatter
    uint32_t* rec;               // [max_blocks][kRecBlock]
    uint32_t* blk_count;         // [max_blocks] records in the block
    uint32_t* blk_chunk;         // [max_blocks] chunk of the block
    uint32_t* blk_seq;           // [max_blocks] ordinal of the block within its chunk
    uint32_t* chunk_nblk;        // [chunks] staged blocks of the chunk
    uint32_t* chunk_first;       // [chunks] exclusive scan of chunk_nblk
    uint32_t* blk_list;          // [max_blocks] block ids in (chunk, ordinal) order
    uint32_t* cursor;            // block allocator
    uint32_t* overflow;          // set when the staging pool ran out (mode 2 then runs)
    uint32_t max_blocks;
    // tuple pruning (multi-word passes): bit c of cellmask[u] = some query of
    // the pass overlaps table cell c of union dim u; a tuple whose cell is
    // clear in any dim of prune_dims cannot match and is skipped before its
    // table rows are read (the host sorts a batch's queries into passes so
    // these masks are sparse, store.cu build_vb_passes)
    uint32_t prune_dims;         // bit u: cellmask[u] is not all ones
    unsigned long long cellmask[kVaBatchMaxDims];
};
constexpr uint32_t kRecBlock = 1024;
constexpr uint32_t kNoBlock = 0xFFFFFFFFu;
size_t va_batch_smem(uint32_t kb, uint32_t cells, int mode);
int va_batch_max_dims();
int va_batch_words(uint32_t kb);   // query words per lane of a full pass (4 / 2: the multi-word layouts)
uint32_t va_batch_warps();
// mode 0 count, 2 ids (recount pass after a staging overflow), 3 group counts + staged records
void launch_va_batch(const VaBatchArgs& a, int mode, cudaStream_t st);
void launch_va_batch_scatter(const VaBatchArgs& a, cudaStream_t st);
void launch_va_batch_scans(const VaBatchArgs& a, uint32_t q0, cudaStream_t st);
void launch_va_batch_block_list(const VaBatchArgs& a, cudaStream_t st);
// sorted batches: slot-order counts / offsets / ids back to query order (the
// ids of queries >= q_from only); returns the number of kernels launched
uint32_t launch_va_batch_unpermute(const uint32_t* perm, const unsigned long long* counts_p,
                                   const unsigned long long* offsets_p, unsigned long long* counts,
                                   unsigned long long* offsets, const uint32_t* ids_p, uint64_t src_cap,
                                   uint32_t* ids, uint64_t cap, uint32_t nq, bool with_ids, uint32_t q_from,
                                   cudaStream_t st);

constexpr int kColTile = 4096;     // tuples per CTA tile, single-query columnar
constexpr int kVaTile = 8192;      // tuples per CTA tile, VA-file filter

void launch_col_scan(const ScanArgs& a, bool ids, cudaStream_t st);
void launch_row_scan(const ScanArgs& a, bool ids, cudaStream_t st);
void launch_va_scan(const ScanArgs& a, bool ids, cudaStream_t st);
void launch_expand(const ScanArgs& a, cudaStream_t st);
void launch_col_batch_count(const BatchArgs& a, int num_sms, cudaStream_t st);
// ids mode of the multi-query columnar pass: masks [nqp][mask_words] (one bit
// per tuple, query-major) + chunk_counts [nqp][n / kChunkTuples rounded up]
void launch_col_batch_ids(const BatchArgs& a, uint32_t* masks, uint64_t mask_words, uint32_t* chunk_counts,
                          int num_sms, cudaStream_t st);
// expansion of a multi-query pass's masks into ascending ids at the batch
// offsets (a.offsets[q0] must hold the pass's base): chunk scans per query,
// the pass's offsets, one expand grid (chunks x queries)
void launch_expand_pass(const ScanArgs& a, uint32_t q0, uint32_t nqp, const uint32_t* masks, uint64_t mask_words,
                        const uint32_t* chunk_counts, uint32_t* chunk_offs, cudaStream_t st);
int col_batch_max_dims();
uint32_t col_batch_padded_dims(uint32_t kb);   // union dims the kernel evaluates
uint32_t row_tile_rows(uint32_t m);
size_t row_scan_smem(uint32_t m);

// checked builds (MDRQ_CHECKS): every unit's failed-check bits, cleared on read
uint32_t vabatch_check_flags();
uint32_t columnar_check_flags();
uint32_t expand_check_flags();

// store construction
void launch_transpose_rows_to_cols(const float* rows, uint64_t n, uint32_t m, float* cols,
                                   uint64_t stride, cudaStream_t st);
void launch_fill_f32(float* p, uint64_t count, float v, cudaStream_t st);
void launch_va_sample(const float* col, uint64_t n, uint64_t step, uint64_t count, float* out,
                      cudaStream_t st);
void launch_va_pick_boundaries(const float* sorted, uint64_t count, uint32_t nbins, float* out,
                               cudaStream_t st);
void launch_va_encode(const float* col, uint64_t n_pad, const float* bounds, uint32_t nb,
                      uint8_t* codes, cudaStream_t st);
// sort `count` floats (ascending), temp storage sized by the helper
size_t va_sort_temp_bytes(uint64_t count);
void va_sort(const float* in, float* out, uint64_t count, void* temp, size_t temp_bytes,
             cudaStream_t st);
void launch_min_max(const float* col, uint64_t n, float* out2, cudaStream_t st);

// kernel-backend helpers (scan_column & mask algebra)
void launch_scan_column_mask(const float* col, uint64_t n, float lo, float hi, uint32_t* mask_words,
                             cudaStream_t st);
void launch_and_masks(const uint32_t* const* masks, uint32_t k, uint64_t nwords, uint32_t* out,
                      cudaStream_t st);
void launch_popcount(const uint32_t* words, uint64_t nwords, unsigned long long* out,
                     cudaStream_t st);
void launch_mask_to_ids(const uint32_t* words, uint64_t n, uint32_t* status_scratch,
                        uint64_t* status, uint32_t epoch, uint32_t* tile_counter,
                        unsigned long long* count, int64_t* ids, cudaStream_t st);
void launch_read_stream(const void* p, uint64_t bytes, uint32_t* sink, int num_sms, cudaStream_t st);
void launch_copy_segments(const uint32_t* src, uint32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                          const int64_t* len, uint64_t nseg, cudaStream_t st);
// 16-bit packing of a batch's id lists for the device->host copy (pack.cu):
// lo16[i] = ids[i] & 0xFFFF, ends[q][b] = ids of query q in buckets <= hb0 + b
// (perm / src_off / src_cap: the lists still in the slot order of a sorted
// bit-sliced batch -- list i at ids + src_off[i] is query perm[i]'s; else null)
// queries < q_to are packed (ends holds q_to rows); nq = lists to walk
void launch_pack_ids16(const uint32_t* ids, const unsigned long long* offsets, uint32_t nq, uint32_t q_to,
                       uint64_t cap, uint32_t hb0, uint32_t nbuckets, uint16_t* lo16, uint32_t* ends,
                       const uint32_t* perm, const unsigned long long* src_off, uint64_t src_cap, int num_sms,
                       cudaStream_t st);
void launch_match_rows(const float* rows, uint64_t nrows, uint32_t m, const float* lo,
                       const float* hi, uint8_t* out, cudaStream_t st);

}  // namespace mdrq
