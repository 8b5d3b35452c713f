// scan_columnar.cu -- columnar MDRQ scan kernels for sm_100a.
//
// Replaces VerticalScan.search_with_stats (reference scan.py:190-211): the
// reference runs one scan_column per queried dimension into a packed bitmask
// (_kernels_cy.pyx:89-120), ANDs the masks in chunks (scan.py:55-78) and
// unpacks the ids (scan.py:85-88).  Here the three steps are fused into one
// pass: the candidate mask of a tile lives in registers across dimensions,
// a lane skips its 128-bit load of the next column once its four tuples are
// all rejected, and in ids mode the verdicts leave as a bitmask + per-chunk
// counts that expand.cu turns into ascending ids.
//
// col_scan_kernel        one query per launch, dimension-at-a-time (HBM bound)
// col_batch_count_kernel up to 32 queries per pass over the union of their
//                        dimensions, every column byte read once per pass
// col_batch_ids_kernel   the same pass in ids mode: one verdict bitmask per
//                        query + per-chunk counts, expanded by expand.cu
#include <utility>

#include "launch.h"

namespace mdrq {

namespace {

constexpr int CS_THREADS = 256;
constexpr int CS_LANE_TUPLES = 16;                 // 64 contiguous bytes per lane and column
constexpr int CS_WARP_TUPLES = 32 * CS_LANE_TUPLES;  // 512
static_assert(CS_THREADS / 32 * CS_WARP_TUPLES == kColTile, "tile size");

// Lane l of a warp owns tuples wbase + 16l .. +15: one 64-byte block per
// column -- the HBM access granularity -- read as 4 x 16 B when any of its
// 16 tuples is still alive and skipped otherwise, so the bytes requested
// are exactly the blocks the dimension-at-a-time algorithm must touch.
template <bool IDS>
__global__ void __launch_bounds__(CS_THREADS) col_scan_kernel(const ScanArgs a) {
    __shared__ uint32_t s_cnt[CS_THREADS / 32];
    __shared__ uint32_t s_ld[CS_THREADS / 32];

    const QueryDesc qd = a.descs[a.q];
    const DimPred* __restrict__ P = a.preds + qd.off;
    const uint32_t k = qd.k;
    const uint32_t tile = blockIdx.x;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t wbase = uint64_t(tile) * kColTile + warp * CS_WARP_TUPLES;
    const uint64_t base = wbase + lane * CS_LANE_TUPLES;

    uint32_t alive = 0xFFFFu;   // bit j: tuple base + j
    if (base + CS_LANE_TUPLES > a.n) alive = base >= a.n ? 0u : (1u << (a.n - base)) - 1u;

    uint32_t nload = 0;  // 64-byte blocks read (skipped blocks are not)
    for (uint32_t i = 0; i < k; ++i) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;  // whole warp rejected: skip the rest
        const DimPred p = P[i];
        const float lo = p.lo, hi = p.hi;
        if (alive) {
            const float4* c = reinterpret_cast<const float4*>(a.cols + uint64_t(p.dim) * a.stride + base);
            float4 v[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) v[g] = ld_stream_f4(c + g);
            uint32_t in = 0;
#pragma unroll
            for (int g = 0; g < 4; ++g) in |= in_range4(v[g], lo, hi) << (4 * g);
            alive &= in;
            ++nload;
        }
    }

    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, __popc(alive));
    nload = __reduce_add_sync(0xFFFFFFFFu, nload);
    if (lane == 0) {
        s_cnt[warp] = wc;
        s_ld[warp] = nload;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0, ld = 0;
#pragma unroll
        for (int w = 0; w < CS_THREADS / 32; ++w) {
            t += s_cnt[w];
            ld += s_ld[w];
        }
        if (!IDS && t) partial_add(a, 0, t);
        if (ld) partial_add(a, 1, 64ull * ld);
    }
    if (!IDS) return;
    // ids mode: verdict bitmask (bit i of word w = tuple 32w+i) + chunk
    // count; lanes 2s, 2s+1 hold the two halves of one mask word
    uint32_t v = alive << (16 * (lane & 1u));
    v |= __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    if ((lane & 1u) == 0) a.mask[base / 32] = v;
    if (lane == 0 && wc) atomicAdd(a.chunk_counts + wbase / kChunkTuples, wc);
}

// ---------------------------------------------------------------------------
// Multi-query count pass.  Each thread holds TPT consecutive tuples of every
// union dimension in registers (one 16/8/4-byte load per column), then walks
// the pass's queries with their bounds broadcast from shared memory.  The
// dimension loop is fully unrolled over exactly KB dimensions (the host pads
// the union to KB with (-inf, +inf) bounds), so the per-tuple verdicts stay
// in predicate registers: two chained FSETP per (tuple, query, dimension).
template <int KB, int TPT>
__global__ void __launch_bounds__(256) col_batch_count_kernel(const BatchArgs a) {
    __shared__ float2 s_b[32][KB];
    __shared__ uint32_t s_cnt[32];
    __shared__ uint16_t s_ud[KB];

    const uint32_t nqp = a.nqp;
    for (uint32_t i = threadIdx.x; i < nqp * KB; i += blockDim.x) s_b[i / KB][i % KB] = a.bounds[i];
    for (uint32_t i = threadIdx.x; i < 32; i += blockDim.x) s_cnt[i] = 0;
    for (uint32_t i = threadIdx.x; i < KB; i += blockDim.x) s_ud[i] = a.udims[i];
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31u;
    constexpr uint32_t TILE = 256 * TPT;
    const uint64_t ntiles = (a.n + TILE - 1) / TILE;
    uint32_t acc = 0;  // lane q accumulates query q of this pass

    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t base = tile * TILE + uint64_t(threadIdx.x) * TPT;
        float v[KB][TPT];
#pragma unroll
        for (int d = 0; d < KB; ++d) {
            const float* col = a.cols + uint64_t(s_ud[d]) * a.stride + base;
            if constexpr (TPT == 4) {
                const float4 t = ld_stream_f4(reinterpret_cast<const float4*>(col));
                v[d][0] = t.x; v[d][1] = t.y; v[d][2] = t.z; v[d][3] = t.w;
            } else if constexpr (TPT == 2) {
                const float2 t = __ldcs(reinterpret_cast<const float2*>(col));
                v[d][0] = t.x; v[d][1] = t.y;
            } else {
                v[d][0] = __ldcs(col);
            }
        }
        bool valid[TPT];
#pragma unroll
        for (int t = 0; t < TPT; ++t) valid[t] = base + t < a.n;
        for (uint32_t q = 0; q < nqp; ++q) {
            bool ok[TPT];
#pragma unroll
            for (int t = 0; t < TPT; ++t) ok[t] = valid[t];
#pragma unroll
            for (int d = 0; d < KB; ++d) {
                const float2 b = s_b[q][d];
#pragma unroll
                for (int t = 0; t < TPT; ++t) ok[t] = ok[t] && (b.x <= v[d][t]) && (v[d][t] <= b.y);
            }
            uint32_t c = 0;
#pragma unroll
            for (int t = 0; t < TPT; ++t) c += ok[t] ? 1u : 0u;
            c = __reduce_add_sync(0xFFFFFFFFu, c);
            if (lane == q) acc += c;
        }
    }
    if (acc) atomicAdd(&s_cnt[lane], acc);
    __syncthreads();
    if (threadIdx.x < nqp && s_cnt[threadIdx.x])
        atomicAdd(a.counts + threadIdx.x, (unsigned long long)s_cnt[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Multi-query ids pass (VerticalScan.search over a batch, scan.py:190-211,
// with the column bytes read once per <= 32 queries).  A CTA owns whole
// 65536-tuple compaction chunks (grid-stride); each of its 8 warps takes 128
// consecutive tuples per step, lane l the tuples l, l+32, l+64, l+96 (four
// 128-byte coalesced loads per union column; the NaN padding up to n_pad
// never matches), so a query's bounds -- broadcast from shared memory -- are
// read once per 4 tuples, and ballot t of a query IS its mask word for
// tuples 32t..32t+31.  Lane q keeps query q's four words, stores them to
// query q's mask (query-major, the layout the expansion reads) and adds their
// popcounts to q's chunk count.  No atomics leave the CTA: every chunk count
// is written once.
template <int KB, int TPT>
__global__ void __launch_bounds__(256) col_batch_ids_kernel(const BatchArgs a, uint32_t* __restrict__ masks,
                                                            uint64_t mask_words, uint32_t* __restrict__ chunk_counts,
                                                            uint32_t nchunks) {
    __shared__ float2 s_b[32][KB];
    __shared__ uint32_t s_cnt[32];
    __shared__ uint16_t s_ud[KB];
    const uint32_t nqp = a.nqp;
    for (uint32_t i = threadIdx.x; i < nqp * KB; i += blockDim.x) s_b[i / KB][i % KB] = a.bounds[i];
    for (uint32_t i = threadIdx.x; i < KB; i += blockDim.x) s_ud[i] = a.udims[i];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
        if (threadIdx.x < 32) s_cnt[threadIdx.x] = 0;
        __syncthreads();
        uint32_t acc = 0;
        const uint64_t c0 = uint64_t(chunk) * kChunkTuples;
        const uint64_t c1 = c0 + kChunkTuples < a.n ? c0 + kChunkTuples : a.n;
        for (uint64_t t0 = c0 + warp * (32 * TPT); t0 < c1; t0 += 8 * 32 * TPT) {
            // words t0/32 .. +3; a word starting at or past n is not stored
            // (tuples past n inside a word read the NaN padding)
            float v[KB][TPT];
#pragma unroll
            for (int d = 0; d < KB; ++d) {
                const float* col = a.cols + uint64_t(s_ud[d]) * a.stride + t0 + lane;
#pragma unroll
                for (int t = 0; t < TPT; ++t)
                    v[d][t] = t0 + 32 * t < a.n ? __ldcs(col + 32 * t) : __int_as_float(0x7fc00000);
            }
            uint32_t mine[TPT];
#pragma unroll
            for (int t = 0; t < TPT; ++t) mine[t] = 0u;
            for (uint32_t q = 0; q < nqp; ++q) {
                bool ok[TPT];
#pragma unroll
                for (int t = 0; t < TPT; ++t) ok[t] = true;
#pragma unroll
                for (int d = 0; d < KB; ++d) {
                    const float2 b = s_b[q][d];
#pragma unroll
                    for (int t = 0; t < TPT; ++t) ok[t] = ok[t] && (b.x <= v[d][t]) && (v[d][t] <= b.y);
                }
#pragma unroll
                for (int t = 0; t < TPT; ++t) {
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, ok[t]);
                    if (lane == q) mine[t] = bal;
                }
            }
            if (lane < nqp) {
#pragma unroll
                for (int t = 0; t < TPT; ++t)
                    if (t0 + 32 * t < a.n) {
                        MDRQ_CHECK(t0 / 32 + t < mask_words, kChkMask);
                        masks[uint64_t(lane) * mask_words + t0 / 32 + t] = mine[t];
                        acc += __popc(mine[t]);
                    }
            }
        }
        if (acc) atomicAdd(&s_cnt[lane], acc);
        __syncthreads();
        if (threadIdx.x < nqp) chunk_counts[uint64_t(threadIdx.x) * nchunks + chunk] = s_cnt[threadIdx.x];
        __syncthreads();   // s_cnt is reset for the next chunk
    }
}

template <int KB, int TPT>
void run_batch(const BatchArgs& a, int num_sms, cudaStream_t st) {
    static int blocks_per_sm = -1;
    if (blocks_per_sm < 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, col_batch_count_kernel<KB, TPT>,
                                                      256, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    const uint64_t tile = 256 * TPT;
    const uint64_t ntiles = (a.n + tile - 1) / tile;
    uint64_t grid = uint64_t(num_sms) * blocks_per_sm;
    if (grid > ntiles) grid = ntiles;
    if (grid == 0) return;
    col_batch_count_kernel<KB, TPT><<<unsigned(grid), 256, 0, st>>>(a);
}

template <int... Ks>
void dispatch_exact(const BatchArgs& a, int num_sms, cudaStream_t st, std::integer_sequence<int, Ks...>) {
    ((a.kb == uint32_t(Ks + 1) ? run_batch<Ks + 1, 4>(a, num_sms, st) : void()), ...);
}

template <int KB>
void run_batch_ids(const BatchArgs& a, uint32_t* masks, uint64_t mask_words, uint32_t* chunk_counts, int num_sms,
                   cudaStream_t st) {
    // tuples per lane: as many as the registers allow (the count pass's choice)
    constexpr int TPT = KB <= 16 ? 4 : KB <= 32 ? 2 : 1;
    static int blocks_per_sm = -1;
    if (blocks_per_sm < 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, col_batch_ids_kernel<KB, TPT>, 256, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    const uint32_t nchunks = uint32_t((a.n + kChunkTuples - 1) / kChunkTuples);
    uint64_t grid = uint64_t(num_sms) * blocks_per_sm;
    if (grid > nchunks) grid = nchunks;
    if (grid == 0) return;
    col_batch_ids_kernel<KB, TPT><<<unsigned(grid), 256, 0, st>>>(a, masks, mask_words, chunk_counts, nchunks);
}

template <int... Ks>
void dispatch_ids(const BatchArgs& a, uint32_t* masks, uint64_t mask_words, uint32_t* chunk_counts, int num_sms,
                  cudaStream_t st, std::integer_sequence<int, Ks...>) {
    ((a.kb == uint32_t(Ks + 1) ? run_batch_ids<Ks + 1>(a, masks, mask_words, chunk_counts, num_sms, st) : void()),
     ...);
}

}  // namespace

void launch_col_batch_ids(const BatchArgs& a, uint32_t* masks, uint64_t mask_words, uint32_t* chunk_counts,
                          int num_sms, cudaStream_t st) {
    if (a.kb <= 16)
        dispatch_ids(a, masks, mask_words, chunk_counts, num_sms, st, std::make_integer_sequence<int, 16>{});
    else if (a.kb == 32)
        run_batch_ids<32>(a, masks, mask_words, chunk_counts, num_sms, st);
    else
        run_batch_ids<64>(a, masks, mask_words, chunk_counts, num_sms, st);
}

MDRQ_CHECK_FLAGS_FN(columnar_check_flags)

void launch_col_scan(const ScanArgs& a, bool ids, cudaStream_t st) {
    if (a.num_tiles == 0) return;
    if (ids)
        col_scan_kernel<true><<<a.num_tiles, CS_THREADS, 0, st>>>(a);
    else
        col_scan_kernel<false><<<a.num_tiles, CS_THREADS, 0, st>>>(a);
}

int col_batch_max_dims() { return 64; }

uint32_t col_batch_padded_dims(uint32_t kb) {
    if (kb <= 16) return kb;
    if (kb <= 32) return 32;
    return 64;
}

void launch_col_batch_count(const BatchArgs& a, int num_sms, cudaStream_t st) {
    if (a.kb <= 16)
        dispatch_exact(a, num_sms, st, std::make_integer_sequence<int, 16>{});
    else if (a.kb == 32)
        run_batch<32, 2>(a, num_sms, st);
    else
        run_batch<64, 1>(a, num_sms, st);
}

}  // namespace mdrq
