// scan_rowwise.cu -- row-wise MDRQ scan for sm_100a.
//
// Replaces SequentialScan / HorizontalScan (reference scan.py:91-164), whose
// hot loop is scan_rows (_kernels_cy.pyx:58-86) calling _match_code
// (_kernels_cy.pyx:23-46) once per row.  Each CTA claims row tiles in order
// (atomic tile counter), stages them into shared memory with the TMA bulk
// engine (cp.async.bulk + mbarrier, two stages: the next tile streams in
// while the current one is evaluated), evaluates one row per thread, and
// emits ascending ids through the same ballot / block-scan / decoupled
// look-back compaction as the columnar path.
//
// The early-break counter of the reference (`early`, pyx:84-85) is
// reproduced exactly for both kernel modes from the first failing
// dimension f of each row:
//   scalar  : early iff f < m - 1                             (pyx:31-32)
//   blocked : f inside the 8-lane blocks -> early iff block end < m
//             f in the scalar tail      -> early iff f < m - 1 (pyx:34-45)
// Reading dimension (i + rot) mod k in lane group `rot` keeps the 32 lanes
// of a warp on 32 distinct shared-memory banks for every m.
#include "launch.h"

namespace mdrq {

namespace {

constexpr int RW_THREADS = 256;
constexpr uint32_t kRowStageBytes = 48 * 1024;

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

template <bool IDS>
__global__ void __launch_bounds__(RW_THREADS) row_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_tiles[2];
    __shared__ uint16_t s_dims[kMaxDims];
    __shared__ float s_lo[kMaxDims], s_hi[kMaxDims];
    __shared__ unsigned long long s_early[3];

    const QueryDesc qd = a.descs[a.q];
    const DimPred* __restrict__ P = a.preds + qd.off;
    const uint32_t k = qd.k, m = a.m, R = a.rows_per_tile;
    const uint32_t tile_bytes = R * m * 4u;
    float* buf[2] = {reinterpret_cast<float*>(smem), reinterpret_cast<float*>(smem + kRowStageBytes)};

    // dims ascending (reference order) for the first-fail computation
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        s_dims[i] = P[i].dim;
        s_lo[i] = P[i].lo;
        s_hi[i] = P[i].hi;
    }
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_early[0] = s_early[1] = s_early[2] = 0;
        const uint32_t t0 = atomicAdd(a.tile_counters + a.q, 1u);
        s_tiles[0] = t0;
        if (t0 < a.num_tiles) {
            mbar_expect_tx(&s_bar[0], tile_bytes);
            bulk_g2s(buf[0], a.rows + uint64_t(t0) * R * m, tile_bytes, &s_bar[0]);
        }
    }
    __syncthreads();

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    // bank rotation: lanes sharing (row*m mod 32) read different dims
    const uint32_t g = min(m & (~m + 1u), 32u);  // gcd(m, 32)
    const uint32_t rot = k ? ((lane * g) >> 5) % k : 0;
    const uint32_t rows_per_thread = (R + RW_THREADS - 1) / RW_THREADS;
    const uint32_t blocks8 = m / 8;
    uint32_t early_s = 0, early_b = 0, matched = 0, tiles_done = 0;
    uint32_t phase[2] = {0, 0};
    int stage = 0;

    while (true) {
        const uint32_t tile = s_tiles[stage];
        if (tile >= a.num_tiles) break;
        if (threadIdx.x == 0) {
            const uint32_t tn = atomicAdd(a.tile_counters + a.q, 1u);
            s_tiles[stage ^ 1] = tn;
            if (tn < a.num_tiles) {
                fence_proxy_async();
                mbar_expect_tx(&s_bar[stage ^ 1], tile_bytes);
                bulk_g2s(buf[stage ^ 1], a.rows + uint64_t(tn) * R * m, tile_bytes, &s_bar[stage ^ 1]);
            }
        }
        mbar_wait(&s_bar[stage], phase[stage]);
        ++tiles_done;
        phase[stage] ^= 1u;

        const float* tb = buf[stage];
        const uint64_t tile_row0 = uint64_t(tile) * R;
        uint32_t hits = 0;  // bit r: row (r*256 + tid) matches
        for (uint32_t r = 0; r < rows_per_thread; ++r) {
            const uint32_t row = r * RW_THREADS + threadIdx.x;
            if (row >= R || tile_row0 + row >= a.n) continue;
            const float* rv = tb + row * m;
            uint32_t first = 0xFFFFFFFFu;
            uint32_t ii = rot;
            for (uint32_t i = 0; i < k; ++i) {
                const uint32_t d = s_dims[ii];
                const float v = rv[d];
                if (!((s_lo[ii] <= v) & (v <= s_hi[ii]))) first = min(first, d);
                if (++ii == k) ii = 0;
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
                    if (b) atomicAdd(a.chunk_counts + g0 / kChunkTuples, uint32_t(__popc(b)));
                }
            }
        }
        __syncthreads();  // buf[stage] free for reuse
        stage ^= 1;
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

size_t row_scan_smem(uint32_t /*m*/) { return 2 * size_t(kRowStageBytes); }

void launch_row_scan(const ScanArgs& a, bool ids, cudaStream_t st) {
    if (a.num_tiles == 0) return;
    static int configured = 0;
    const size_t smem = row_scan_smem(a.m);
    if (!configured) {
        cudaFuncSetAttribute(row_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(row_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        configured = 1;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (ids)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, row_scan_kernel<true>, RW_THREADS, smem);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, row_scan_kernel<false>, RW_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = uint64_t(sms) * per_sm;
    if (grid > a.num_tiles) grid = a.num_tiles;
    if (ids)
        row_scan_kernel<true><<<unsigned(grid), RW_THREADS, smem, st>>>(a);
    else
        row_scan_kernel<false><<<unsigned(grid), RW_THREADS, smem, st>>>(a);
}

}  // namespace mdrq
