// expand.cu -- ordered result compaction (ids mode) shared by every scan path.
//
// The scan kernels of ids mode write the verdicts of a query as a packed
// bitmask over the store's tuples (bit i of 32-bit word w = tuple 32w+i, the
// reference's little-endian mask layout, scan.py:85-88) plus one count per
// 65536-tuple chunk.  Two light kernels then turn the mask into ascending ids:
//
//   chunk_scan_kernel  exclusive prefix of the chunk counts (one CTA), chains
//                      the query's output base: offsets[q+1] = offsets[q] + total
//   expand_kernel      one CTA per chunk, 8 mask words per thread: block scan
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

// CHAIN: one query, its output base chained from the previous query's.
// Otherwise CTA y scans query q + y's counts (at chunk_counts + y * nchunks)
// and only reports its total (pass_offsets_kernel chains the bases).
template <bool CHAIN>
__global__ void __launch_bounds__(SCAN_THREADS) chunk_scan_kernel(const uint32_t* __restrict__ chunk_counts,
                                                                  uint32_t nchunks, uint32_t* __restrict__ chunk_offs,
                                                                  unsigned long long* offsets,
                                                                  unsigned long long* counts, uint32_t q) {
    chunk_counts += uint64_t(blockIdx.x) * nchunks;
    chunk_offs += uint64_t(blockIdx.x) * nchunks;
    q += blockIdx.x;
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
        if (CHAIN) offsets[q + 1] = offsets[q] + total;
        counts[q] = total;
    }
}

// offsets[q0 + 1 + i] = offsets[q0] + counts[q0] + ... + counts[q0 + i], i < nqp <= 32
__global__ void pass_offsets_kernel(const unsigned long long* __restrict__ counts, uint32_t nqp,
                                    unsigned long long* offsets, uint32_t q0) {
    const uint32_t lane = threadIdx.x;
    unsigned long long incl = lane < nqp ? counts[q0 + lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
    }
    const unsigned long long base = offsets[q0];
    if (lane < nqp) offsets[q0 + 1 + lane] = base + incl;
}

// one CTA per 65536-tuple chunk: 256 threads x 8 consecutive mask words
// blockIdx.y selects query q + y of a multi-query pass (mask and chunk
// offsets at y * mask_stride / y * coff_stride)
__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ mask, uint64_t n,
                                                     const uint32_t* __restrict__ chunk_offs,
                                                     const unsigned long long* __restrict__ offsets, uint32_t q,
                                                     uint32_t* __restrict__ ids, uint64_t cap, uint32_t id_base,
                                                     uint64_t mask_stride, uint32_t coff_stride) {
    constexpr int WPT = kChunkTuples / 32 / 256;   // words per thread
    __shared__ uint32_t s_warp[8];
    const uint32_t chunk = blockIdx.x;
    mask += blockIdx.y * mask_stride;
    chunk_offs += uint64_t(blockIdx.y) * coff_stride;
    q += blockIdx.y;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t w0 = uint64_t(chunk) * (kChunkTuples / 32) + uint64_t(threadIdx.x) * WPT;
    const uint64_t nwords = (n + 31) / 32;
    uint32_t bits[WPT];
    if (w0 + WPT <= nwords) {
        const uint4* p = reinterpret_cast<const uint4*>(mask + w0);
#pragma unroll
        for (int i = 0; i < WPT / 4; ++i) {
            const uint4 v = p[i];
            bits[4 * i] = v.x; bits[4 * i + 1] = v.y; bits[4 * i + 2] = v.z; bits[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < WPT; ++i) bits[i] = w0 + i < nwords ? mask[w0 + i] : 0u;
    }
    if ((n % 32) && w0 <= nwords - 1 && nwords - 1 < w0 + WPT)
        bits[nwords - 1 - w0] &= (1u << (n % 32)) - 1u;
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < WPT; ++i) c += __popc(bits[i]);
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
    if (!c) return;
    unsigned long long pos = offsets[q] + chunk_offs[chunk] + s_warp[warp] + (incl - c);
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        uint32_t b = bits[i];
        const uint32_t t0 = id_base + uint32_t((w0 + i) * 32);
        while (b) {
            const int j = __ffs(b) - 1;
            b &= b - 1;
            if (pos < cap) ids[pos] = t0 + uint32_t(j);
            ++pos;
        }
    }
}

__global__ void reduce_partials_kernel(const unsigned long long* __restrict__ partials, uint32_t nq, bool add_counts,
                                       unsigned long long* counts, unsigned long long* stats) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long c = 0, bytes = 0, refined = 0;
    const unsigned long long* p = partials + uint64_t(q) * kPartialSlots * 4;
    for (int s = 0; s < kPartialSlots; ++s) {
        c += p[4 * s + 0];
        bytes += p[4 * s + 1];
        refined += p[4 * s + 2];
    }
    if (add_counts) counts[q] += c;
    stats[4 * q + 2] += refined;
    stats[4 * q + 3] += bytes;
}

}  // namespace

MDRQ_CHECK_FLAGS_FN(expand_check_flags)

void launch_reduce_partials(const unsigned long long* partials, uint32_t nq, bool add_counts,
                            unsigned long long* counts, unsigned long long* stats, cudaStream_t st) {
    if (!nq) return;
    reduce_partials_kernel<<<(nq + 255) / 256, 256, 0, st>>>(partials, nq, add_counts, counts, stats);
}

void launch_expand(const ScanArgs& a, cudaStream_t st) {
    const uint32_t nchunks = uint32_t((a.n + kChunkTuples - 1) / kChunkTuples);
    if (!nchunks) return;
    chunk_scan_kernel<true><<<1, SCAN_THREADS, 0, st>>>(a.chunk_counts, nchunks, a.chunk_offs, a.offsets, a.counts,
                                                        a.q);
    expand_kernel<<<nchunks, 256, 0, st>>>(a.mask, a.n, a.chunk_offs, a.offsets, a.q, a.ids, a.ids_cap, a.id_base, 0,
                                           0);
}

void launch_expand_pass(const ScanArgs& a, uint32_t q0, uint32_t nqp, const uint32_t* masks, uint64_t mask_words,
                        const uint32_t* chunk_counts, uint32_t* chunk_offs, cudaStream_t st) {
    const uint32_t nchunks = uint32_t((a.n + kChunkTuples - 1) / kChunkTuples);
    if (!nchunks || !nqp) return;
    chunk_scan_kernel<false><<<nqp, SCAN_THREADS, 0, st>>>(chunk_counts, nchunks, chunk_offs, a.offsets, a.counts,
                                                           q0);
    pass_offsets_kernel<<<1, 32, 0, st>>>(a.counts, nqp, a.offsets, q0);
    expand_kernel<<<dim3(nchunks, nqp), 256, 0, st>>>(masks, a.n, chunk_offs, a.offsets, q0, a.ids, a.ids_cap,
                                                      a.id_base, mask_words, nchunks);
}

}  // namespace mdrq
