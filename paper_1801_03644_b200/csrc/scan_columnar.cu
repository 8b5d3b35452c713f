// scan_columnar.cu -- columnar MDRQ scan kernels for sm_100a.
//
// Replaces VerticalScan.search_with_stats (reference scan.py:190-211): the
// reference runs one scan_column per queried dimension into a packed bitmask
// (_kernels_cy.pyx:89-120), ANDs the masks in chunks (scan.py:55-78) and
// unpacks the ids (scan.py:85-88).  Here the three steps are fused into one
// pass: the candidate mask of a tile lives in registers across dimensions,
// a lane skips its 128-bit load of the next column once its four tuples are
// all rejected, and surviving tuples are compacted into ascending ids with a
// warp ballot + block scan + decoupled look-back (single pass, ordered).
//
// col_scan_kernel        one query per launch, dimension-at-a-time (HBM bound)
// col_batch_count_kernel up to 32 queries per pass over the union of their
//                        dimensions, every column byte read once per pass
#include "launch.h"

namespace mdrq {

namespace {

constexpr int CS_THREADS = 256;
constexpr int CS_G = 4;                            // float4 groups per thread
constexpr int CS_WARP_TUPLES = 32 * 4 * CS_G;      // 512
static_assert(CS_THREADS / 32 * CS_WARP_TUPLES == kColTile, "tile size");

template <bool IDS>
__global__ void __launch_bounds__(CS_THREADS) col_scan_kernel(const ScanArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_seg[32];
    __shared__ uint32_t s_excl;

    const QueryDesc qd = a.descs[a.q];
    const DimPred* __restrict__ P = a.preds + qd.off;
    const uint32_t k = qd.k;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counters + a.q, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t base = uint64_t(tile) * kColTile + warp * CS_WARP_TUPLES + lane * 4;

    uint32_t alive = 0xFFFFu;
    if (uint64_t(tile + 1) * kColTile > a.n) {  // tail tile: mask tuples >= n
        alive = 0;
#pragma unroll
        for (int g = 0; g < CS_G; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (base + g * 128 + j < a.n) alive |= 1u << (4 * g + j);
    }

    for (uint32_t i = 0; i < k; ++i) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;  // whole warp rejected: skip the rest
        const DimPred p = P[i];
        const uint32_t d = p.dim;
        const float lo = p.lo, hi = p.hi;
        const float4* c = reinterpret_cast<const float4*>(a.cols + uint64_t(d) * a.stride + base);
        float4 v[CS_G];
#pragma unroll
        for (int g = 0; g < CS_G; ++g)
            if ((alive >> (4 * g)) & 0xFu) v[g] = ld_stream_f4(c + g * 32);
#pragma unroll
        for (int g = 0; g < CS_G; ++g)
            if ((alive >> (4 * g)) & 0xFu)
                alive &= (in_range4(v[g], lo, hi) << (4 * g)) | ~(0xFu << (4 * g));
    }

    if (!IDS) {
        uint32_t c = __reduce_add_sync(0xFFFFFFFFu, __popc(alive));
        if (lane == 0) s_seg[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < CS_THREADS / 32; ++w) t += s_seg[w];
            if (t) atomicAdd(a.counts + a.q, (unsigned long long)t);
        }
        return;
    }

    // ---- ordered compaction: tuple order within the tile is (warp, g, lane, j)
    const uint32_t lt = lanemask_lt();
    uint32_t pre[CS_G];
#pragma unroll
    for (int g = 0; g < CS_G; ++g) {
        const uint32_t nib = (alive >> (4 * g)) & 0xFu;
        const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, nib & 1u);
        const uint32_t b1 = __ballot_sync(0xFFFFFFFFu, nib & 2u);
        const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, nib & 4u);
        const uint32_t b3 = __ballot_sync(0xFFFFFFFFu, nib & 8u);
        pre[g] = __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
        if (lane == 0) s_seg[warp * CS_G + g] = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = s_seg[lane];
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= uint32_t(o)) incl += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t excl = lookback_exclusive(a.status, tile, a.epoch, total);
        s_seg[lane] = incl - v;
        if (lane == 0) {
            s_excl = excl;
            if (tile == a.num_tiles - 1) {
                const unsigned long long qbase = a.offsets[a.q];
                a.offsets[a.q + 1] = qbase + excl + total;
                a.counts[a.q] = excl + total;
            }
        }
    }
    __syncthreads();
    if (alive) {
        const unsigned long long obase = a.offsets[a.q] + s_excl;
#pragma unroll
        for (int g = 0; g < CS_G; ++g) {
            uint32_t nib = (alive >> (4 * g)) & 0xFu;
            unsigned long long pos = obase + s_seg[warp * CS_G + g] + pre[g];
            while (nib) {
                const int j = __ffs(nib) - 1;
                nib &= nib - 1;
                if (pos < a.ids_cap) a.ids[pos] = a.id_base + uint32_t(base + g * 128 + j);
                ++pos;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Multi-query count pass.  Each thread holds TPT consecutive tuples of every
// union dimension in registers (one 16/8/4-byte load per column), then walks
// the pass's queries with their bounds broadcast from shared memory.
template <int KB, int TPT>
__global__ void __launch_bounds__(256) col_batch_count_kernel(const BatchArgs a) {
    __shared__ float2 s_b[32][KB];
    __shared__ unsigned long long s_cm[32];
    __shared__ uint32_t s_cnt[32];
    __shared__ uint16_t s_ud[KB];

    const uint32_t kb = a.kb, nqp = a.nqp;
    for (uint32_t i = threadIdx.x; i < nqp * kb; i += blockDim.x) s_b[i / kb][i % kb] = a.bounds[i];
    for (uint32_t i = threadIdx.x; i < 32; i += blockDim.x) {
        s_cm[i] = i < nqp ? a.cmask[i] : 0ull;
        s_cnt[i] = 0;
    }
    for (uint32_t i = threadIdx.x; i < kb; i += blockDim.x) s_ud[i] = a.udims[i];
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
            if (d < int(kb)) {
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
        }
        uint32_t valid = (1u << TPT) - 1u;
        if (base + TPT > a.n) {
            valid = 0;
#pragma unroll
            for (int t = 0; t < TPT; ++t)
                if (base + t < a.n) valid |= 1u << t;
        }
        for (uint32_t q = 0; q < nqp; ++q) {
            const unsigned long long cm = s_cm[q];
            bool ok[TPT];
#pragma unroll
            for (int t = 0; t < TPT; ++t) ok[t] = (valid >> t) & 1u;
#pragma unroll
            for (int d = 0; d < KB; ++d) {
                if (d < int(kb) && ((cm >> d) & 1ull)) {
                    const float2 b = s_b[q][d];
#pragma unroll
                    for (int t = 0; t < TPT; ++t) ok[t] = ok[t] & (b.x <= v[d][t]) & (v[d][t] <= b.y);
                }
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

}  // namespace

void launch_col_scan(const ScanArgs& a, bool ids, cudaStream_t st) {
    if (a.num_tiles == 0) return;
    if (ids)
        col_scan_kernel<true><<<a.num_tiles, CS_THREADS, 0, st>>>(a);
    else
        col_scan_kernel<false><<<a.num_tiles, CS_THREADS, 0, st>>>(a);
}

int col_batch_max_dims() { return 64; }

void launch_col_batch_count(const BatchArgs& a, int num_sms, cudaStream_t st) {
    if (a.kb <= 4)
        run_batch<4, 4>(a, num_sms, st);
    else if (a.kb <= 8)
        run_batch<8, 4>(a, num_sms, st);
    else if (a.kb <= 16)
        run_batch<16, 4>(a, num_sms, st);
    else if (a.kb <= 32)
        run_batch<32, 2>(a, num_sms, st);
    else
        run_batch<64, 1>(a, num_sms, st);
}

}  // namespace mdrq
