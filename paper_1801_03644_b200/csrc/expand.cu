// expand.cu -- ordered result compaction (ids mode) shared by every scan path.
//
// The scan kernels of ids mode write the verdicts of a query as a packed
// bitmask over the store's tuples (bit i of 32-bit word w = tuple 32w+i, the
// reference's little-endian mask layout, scan.py:85-88) plus one count per
// 8192-tuple chunk.  Two light kernels then turn the mask into ascending ids:
//
//   chunk_scan_kernel  exclusive prefix of the chunk counts (one CTA), chains
//                      the query's output base: offsets[q+1] = offsets[q] + total
//   expand_kernel      one CTA per chunk, one mask word per thread: block scan
//                      of popcounts, then every set bit is written as
//                      id_base + tuple at offsets[q] + chunk_offset + rank
//
// The mask of a query is 1/32 of one column (6.25 MB at n = 5e7) and is read
// back from L2, so compaction costs a few microseconds instead of a
// decoupled look-back inside the bandwidth-bound scan.
#include "launch.h"

namespace mdrq {

namespace {

constexpr int SCAN_THREADS = 1024;

__global__ void __launch_bounds__(SCAN_THREADS) chunk_scan_kernel(const uint32_t* __restrict__ chunk_counts,
                                                                  uint32_t nchunks, uint32_t* __restrict__ chunk_offs,
                                                                  unsigned long long* offsets,
                                                                  unsigned long long* counts, uint32_t q) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < nchunks; base += SCAN_THREADS) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < nchunks ? chunk_counts[i] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= uint32_t(o)) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = s_warp[lane];
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
                if (lane >= uint32_t(o)) wi += t;
            }
            s_warp[lane] = wi - w;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (i < nchunks) chunk_offs[i] = carry + s_warp[warp] + incl - v;
        __syncthreads();
        if (threadIdx.x == SCAN_THREADS - 1) s_carry = carry + s_warp[warp] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const unsigned long long total = s_carry;
        offsets[q + 1] = offsets[q] + total;
        counts[q] = total;
    }
}

__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ mask, uint64_t n,
                                                     const uint32_t* __restrict__ chunk_offs,
                                                     const unsigned long long* __restrict__ offsets, uint32_t q,
                                                     uint32_t* __restrict__ ids, uint64_t cap, uint32_t id_base) {
    __shared__ uint32_t s_warp[8];
    const uint32_t chunk = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t w = uint64_t(chunk) * 256 + threadIdx.x;
    uint32_t bits = (w * 32 < n) ? mask[w] : 0u;
    if ((w + 1) * 32 > n && w * 32 < n) bits &= (n % 32) ? ((1u << (n % 32)) - 1u) : 0xFFFFFFFFu;
    const uint32_t c = __popc(bits);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = lane < 8 ? s_warp[lane] : 0u;
        uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= uint32_t(o)) wi += t;
        }
        if (lane < 8) s_warp[lane] = wi - v;
    }
    __syncthreads();
    if (!bits) return;
    unsigned long long pos = offsets[q] + chunk_offs[chunk] + s_warp[warp] + (incl - c);
    const uint32_t t0 = id_base + uint32_t(w * 32);
    while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1;
        if (pos < cap) ids[pos] = t0 + uint32_t(j);
        ++pos;
    }
}

}  // namespace

void launch_expand(const ScanArgs& a, cudaStream_t st) {
    const uint32_t nchunks = uint32_t((a.n + kChunkTuples - 1) / kChunkTuples);
    if (!nchunks) return;
    chunk_scan_kernel<<<1, SCAN_THREADS, 0, st>>>(a.chunk_counts, nchunks, a.chunk_offs, a.offsets, a.counts, a.q);
    expand_kernel<<<nchunks, 256, 0, st>>>(a.mask, a.n, a.chunk_offs, a.offsets, a.q, a.ids, a.ids_cap, a.id_base);
}

}  // namespace mdrq
