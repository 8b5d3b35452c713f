// pack.cu -- 16-bit packing of a batch's id lists for the device->host copy.
//
// The reference returns every query's ids as a host array (scan.py:85-88,
// ResultSet core.py:185); on C5 that is 20 GB per 10 000-query batch, and the
// pipelined stream (mdrq_query_ids_stream) is bound by the PCIe copy, not by
// the scan.  A query's ids ascend, so within one 65 536-id bucket they share
// their high half: the device writes the low halves (2 bytes per id, same
// order) and, per query, the end position of every bucket in its run; the
// host rebuilds id = bucket << 16 | low (unpack_host.cpp, multi-threaded).
// The copy shrinks to half plus nq x nbuckets words.  The stream packs the
// first q_to queries of a batch and sends the rest raw, q_to chosen so the
// copy and the host unpack take about as long (store.cu).
#include <algorithm>

#include "launch.h"

namespace mdrq {

namespace {

constexpr uint64_t kPackSeg = 16384;   // ids per CTA step within one list

// One CTA per query run (grid-strided).  ends[q][b] = number of ids of query
// q in buckets <= b (positions relative to the run), b relative to hb0.
// Sorted bit-sliced batches (vabatch.cu) hold their lists in slot order: list
// i (at src_off[i]) is query perm[i]'s; packing straight from there saves the
// move of the uint32 ids to query order.
__global__ void __launch_bounds__(256) pack_ids16_kernel(const uint32_t* __restrict__ ids,
                                                         const unsigned long long* __restrict__ offsets, uint32_t nq,
                                                         uint32_t q_to, uint64_t cap, uint32_t hb0, uint32_t nbuckets,
                                                         uint16_t* __restrict__ lo16, uint32_t* __restrict__ ends,
                                                         const uint32_t* __restrict__ perm,
                                                         const unsigned long long* __restrict__ src_off,
                                                         uint64_t src_cap) {
    // blockIdx.y strides over the lists, blockIdx.x over kPackSeg-id segments
    // of one list (a batch of few long lists still fills the device)
    for (uint32_t i0 = blockIdx.y; i0 < nq; i0 += gridDim.y) {
        const uint32_t q = perm ? perm[i0] : i0;
        if (q >= q_to) continue;   // this query's ids travel raw
        const uint64_t o0 = offsets[q], o1 = offsets[q + 1];
        if (o1 > cap) continue;   // truncated result: the caller grows the pool and reruns
        const uint64_t cnt = o1 - o0;
        if (perm && src_off[i0] + cnt > src_cap) continue;
        uint32_t* e = ends + uint64_t(q) * nbuckets;
        if (cnt == 0) {
            if (blockIdx.x == 0)
                for (uint32_t b = threadIdx.x; b < nbuckets; b += blockDim.x) e[b] = 0;
            continue;
        }
        const uint32_t* s = ids + (perm ? src_off[i0] : o0);
        uint16_t* d = lo16 + o0;
        for (uint64_t seg = uint64_t(blockIdx.x) * kPackSeg; seg < cnt; seg += uint64_t(gridDim.x) * kPackSeg)
        for (uint64_t i = seg + threadIdx.x, i1 = seg + kPackSeg < cnt ? seg + kPackSeg : cnt; i < i1;
             i += blockDim.x) {
            const uint32_t id = __ldcs(s + i);
            d[i] = uint16_t(id);
            const uint32_t hb = (id >> 16) - hb0;
            // buckets [hb, next id's bucket) end after this id; the first id
            // also closes the empty buckets before it, the last id the rest
            const uint32_t hn = i + 1 < cnt ? (__ldg(s + i + 1) >> 16) - hb0 : nbuckets;
            if (i == 0)
                for (uint32_t b = 0; b < hb; ++b) e[b] = 0;
            for (uint32_t b = hb; b < hn; ++b) e[b] = uint32_t(i + 1);
        }
    }
}

}  // namespace

void launch_pack_ids16(const uint32_t* ids, const unsigned long long* offsets, uint32_t nq, uint32_t q_to,
                       uint64_t cap, uint32_t hb0, uint32_t nbuckets, uint16_t* lo16, uint32_t* ends,
                       const uint32_t* perm, const unsigned long long* src_off, uint64_t src_cap, int num_sms,
                       cudaStream_t st) {
    if (!nq || !q_to) return;
    if (!perm) nq = std::min(nq, q_to);   // lists in query order: only the packed ones
    const uint32_t want = uint32_t(num_sms) * 8;
    const uint32_t gy = std::min<uint32_t>(nq, want);
    const uint32_t gx = std::min<uint32_t>(64, std::max<uint32_t>(1, want / gy));
    pack_ids16_kernel<<<dim3(gx, gy), 256, 0, st>>>(ids, offsets, nq, q_to, cap, hb0, nbuckets, lo16, ends, perm,
                                                    src_off, src_cap);
}

}  // namespace mdrq
