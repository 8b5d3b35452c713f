// scan_rowwise.cu -- row-wise MDRQ scan for sm_100a.
//
// Replaces SequentialScan / HorizontalScan (reference scan.py:91-164), whose
// hot loop is scan_rows (_kernels_cy.pyx:58-86) calling _match_code
// (_kernels_cy.pyx:23-46) once per row.  Each CTA claims row tiles in order
// (atomic tile counter), stages them into shared memory with the TMA bulk
// engine (cp.async.bulk + mbarrier, kRowStages stages of 32 KB: the next
// tiles stream in while the current one is evaluated), evaluates one row per
// thread, and in ids mode writes the verdicts as a bitmask + per-chunk counts
// that expand.cu turns into ascending ids (the same two light kernels as the
// columnar path; no look-back inside the bandwidth-bound scan).
//
// The early-break counter of the reference (`early`, pyx:84-85) is
// reproduced exactly for both kernel modes from the first failing
// dimension f of each row:
//   scalar  : early iff f < m - 1                             (pyx:31-32)
//   blocked : f inside the 8-lane blocks -> early iff block end < m
//             f in the scalar tail      -> early iff f < m - 1 (pyx:34-45)
// Reading dimension (i + rot) mod k in lane group `rot` keeps the 32 lanes
// of a warp on 32 distinct shared-memory banks for every m.
#include <utility>

#include "launch.h"

namespace mdrq {

namespace {

constexpr int RW_THREADS = 512;
constexpr int kRowStages = 3;                    // bulk-copy pipeline depth per CTA (2 CTAs / SM)
constexpr uint32_t kRowStageBytes = 32 * 1024;   // one row tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// M > 0: fixed dimensionality (m == M <= 16): the bounds of all M dims live
// in registers (+-inf for unqueried ones, which never fail a stored value),
// the row is read with immediate offsets (float4 when M % 4 == 0) and the
// failing dims collect in a bit mask whose lowest bit is the reference's
// first failing dimension.  M == 0: any m, predicate list in smem, bank-
// rotated dimension order.
template <bool IDS, int M>
__global__ void __launch_bounds__(RW_THREADS, 2) row_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[kRowStages];
    __shared__ uint32_t s_tiles[kRowStages];
    __shared__ uint16_t s_dims[kMaxDims];
    __shared__ float s_lo[kMaxDims], s_hi[kMaxDims];
    __shared__ unsigned long long s_early[3];
    __shared__ uint32_t s_cc[2];   // ids mode: matches of the current tile per chunk

    const QueryDesc qd = a.descs[a.q];
    const DimPred* __restrict__ P = a.preds + qd.off;
    const uint32_t k = qd.k, m = a.m, R = a.rows_per_tile;
    const uint32_t tile_bytes = R * m * 4u;

    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        s_dims[i] = P[i].dim;
        s_lo[i] = P[i].lo;
        s_hi[i] = P[i].hi;
    }
    // prologue: claim kRowStages tiles in order and start their bulk copies
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRowStages; ++s) mbar_init(&s_bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_early[0] = s_early[1] = s_early[2] = 0;
        s_cc[0] = s_cc[1] = 0;
        for (int s = 0; s < kRowStages; ++s) {
            const uint32_t t = atomicAdd(a.tile_counters + a.q, 1u);
            s_tiles[s] = t;
            if (t < a.num_tiles) {
                mbar_expect_tx(&s_bar[s], tile_bytes);
                bulk_g2s(smem + s * kRowStageBytes, a.rows + uint64_t(t) * R * m, tile_bytes, &s_bar[s]);
            }
        }
    }
    __syncthreads();

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    // bank rotation: lanes sharing (row*m mod 32) read different dims
    const uint32_t g = min(m & (~m + 1u), 32u);  // gcd(m, 32)
    const uint32_t rot = k ? ((lane * g) >> 5) % k : 0;
    // fixed-m path: bounds of every dimension in registers
    constexpr int MR = M > 0 ? M : 1;
    float flo[MR], fhi[MR];
    if constexpr (M > 0) {
#pragma unroll
        for (int d = 0; d < MR; ++d) {
            flo[d] = -INFINITY;
            fhi[d] = INFINITY;
        }
        for (uint32_t i = 0; i < k; ++i) {
            const uint32_t d = s_dims[i];
#pragma unroll
            for (int dd = 0; dd < MR; ++dd)
                if (uint32_t(dd) == d) {
                    flo[dd] = s_lo[i];
                    fhi[dd] = s_hi[i];
                }
        }
    }
    const uint32_t rows_per_thread = (R + RW_THREADS - 1) / RW_THREADS;
    const uint32_t blocks8 = m / 8;
    uint32_t early_s = 0, early_b = 0, matched = 0, tiles_done = 0;
    uint32_t phases = 0;   // bit s: parity of stage s
    int stage = 0;

    while (true) {
        const uint32_t tile = s_tiles[stage];
        if (tile >= a.num_tiles) break;
        mbar_wait(&s_bar[stage], (phases >> stage) & 1u);
        phases ^= 1u << stage;
        ++tiles_done;

        const float* tb = reinterpret_cast<const float*>(smem + stage * kRowStageBytes);
        const uint64_t tile_row0 = uint64_t(tile) * R;
        uint32_t hits = 0;  // bit r: row (r*RW_THREADS + tid) matches
        for (uint32_t r = 0; r < rows_per_thread; ++r) {
            const uint32_t row = r * RW_THREADS + threadIdx.x;
            if (row >= R || tile_row0 + row >= a.n) continue;
            const float* rv = tb + row * m;
            uint32_t first = 0xFFFFFFFFu;
            if constexpr (M > 0) {
                float v[MR];
                if constexpr (M % 4 == 0) {
#pragma unroll
                    for (int j = 0; j < M / 4; ++j) {
                        const float4 t4 = reinterpret_cast<const float4*>(rv)[j];
                        v[4 * j] = t4.x; v[4 * j + 1] = t4.y; v[4 * j + 2] = t4.z; v[4 * j + 3] = t4.w;
                    }
                } else {
#pragma unroll
                    for (int d = 0; d < MR; ++d) v[d] = rv[d];
                }
                uint32_t fail = 0;
#pragma unroll
                for (int d = 0; d < MR; ++d) fail |= uint32_t(!((flo[d] <= v[d]) & (v[d] <= fhi[d]))) << d;
                if (fail) first = __ffs(fail) - 1;
            } else {
                uint32_t ii = rot;
                for (uint32_t i = 0; i < k; ++i) {
                    const uint32_t d = s_dims[ii];
                    const float v = rv[d];
                    if (!((s_lo[ii] <= v) & (v <= s_hi[ii]))) first = min(first, d);
                    if (++ii == k) ii = 0;
                }
            }
            if (first == 0xFFFFFFFFu) {
                hits |= 1u << r;
            } else {
                early_s += first < m - 1;
                if (first < blocks8 * 8)
                    early_b += (first / 8) * 8 + 8 < m;
                else
                    early_b += first < m - 1;
            }
        }

        matched += __popc(hits);
        if (IDS) {
            // verdict bitmask: (r, warp) covers 32 consecutive rows = one word
            for (uint32_t r = 0; r < rows_per_thread; ++r) {
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, (hits >> r) & 1u);
                const uint32_t row0 = r * RW_THREADS + warp * 32;
                if (lane == 0 && row0 < R) {
                    const uint64_t g0 = tile_row0 + row0;
                    a.mask[g0 / 32] = b;
                    // a tile spans at most two compaction chunks
                    if (b) atomicAdd(&s_cc[g0 / kChunkTuples - tile_row0 / kChunkTuples], uint32_t(__popc(b)));
                }
            }
        }
        __syncthreads();  // every thread is done with this stage's buffer
        if (IDS && threadIdx.x == 0) {
            const uint64_t c0 = tile_row0 / kChunkTuples;
            if (s_cc[0]) atomicAdd(a.chunk_counts + c0, s_cc[0]);
            if (s_cc[1]) atomicAdd(a.chunk_counts + c0 + 1, s_cc[1]);
            s_cc[0] = s_cc[1] = 0;
        }
        if (threadIdx.x == 0) {
            // refill the stage with the next tile in claim order
            const uint32_t tn = atomicAdd(a.tile_counters + a.q, 1u);
            s_tiles[stage] = tn;
            if (tn < a.num_tiles) {
                fence_proxy_async();
                mbar_expect_tx(&s_bar[stage], tile_bytes);
                bulk_g2s(smem + stage * kRowStageBytes, a.rows + uint64_t(tn) * R * m, tile_bytes, &s_bar[stage]);
            }
        }
        stage = stage + 1 == kRowStages ? 0 : stage + 1;
        __syncthreads();  // s_tiles[] of the next stages are visible
    }

    // early-break counters (and, count mode, matches) of this CTA
    early_s = __reduce_add_sync(0xFFFFFFFFu, early_s);
    early_b = __reduce_add_sync(0xFFFFFFFFu, early_b);
    matched = __reduce_add_sync(0xFFFFFFFFu, matched);
    if (lane == 0) {
        if (early_s) atomicAdd(&s_early[0], (unsigned long long)early_s);
        if (early_b) atomicAdd(&s_early[1], (unsigned long long)early_b);
        if (matched) atomicAdd(&s_early[2], (unsigned long long)matched);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.stats && s_early[0]) atomicAdd(a.stats + 4 * a.q + 0, s_early[0]);
        if (a.stats && s_early[1]) atomicAdd(a.stats + 4 * a.q + 1, s_early[1]);
        if (a.stats && tiles_done) atomicAdd(a.stats + 4 * a.q + 3, (unsigned long long)tiles_done * tile_bytes);
        if (!IDS && s_early[2]) atomicAdd(a.counts + a.q, s_early[2]);
    }
}

}  // namespace

uint32_t row_tile_rows(uint32_t m) {
    uint32_t r = kRowStageBytes / (4u * m);
    r = (r / 32u) * 32u;
    if (r > 1024u) r = 1024u;
    if (r < 32u) r = 32u;
    return r;
}

size_t row_scan_smem(uint32_t /*m*/) { return size_t(kRowStages) * kRowStageBytes; }

template <bool IDS, int M>
void run_row(const ScanArgs& a, cudaStream_t st) {
    static int per_sm = 0;
    const size_t smem = row_scan_smem(a.m);
    if (!per_sm) {
        cudaFuncSetAttribute(row_scan_kernel<IDS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, row_scan_kernel<IDS, M>, RW_THREADS, smem);
        if (per_sm < 1) per_sm = 1;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t grid = uint64_t(sms) * per_sm;
    if (grid > a.num_tiles) grid = a.num_tiles;
    row_scan_kernel<IDS, M><<<unsigned(grid), RW_THREADS, smem, st>>>(a);
}

template <bool IDS, int... Ms>
void dispatch_m(const ScanArgs& a, cudaStream_t st, std::integer_sequence<int, Ms...>) {
    bool done = false;
    ((a.m == uint32_t(Ms + 1) ? (run_row<IDS, Ms + 1>(a, st), done = true) : false), ...);
    if (!done) run_row<IDS, 0>(a, st);
}

void launch_row_scan(const ScanArgs& a, bool ids, cudaStream_t st) {
    if (a.num_tiles == 0) return;
    using Seq = std::make_integer_sequence<int, 16>;
    if (ids)
        dispatch_m<true>(a, st, Seq{});
    else
        dispatch_m<false>(a, st, Seq{});
}

}  // namespace mdrq
