// unpack_host.cpp -- host side of the 16-bit id packing (pack.cu): rebuild
// the uint32 ids of a batch from their low halves and the per-query bucket
// ends, on `threads` host threads (equal shares of the ids).  Plain
// C++ (g++), AVX2 where the CPU has it; exported as mdrq_unpack_ids16.
//
// A thread's queries are one contiguous range of the output, walked 16 ids
// at a time with streaming stores; the high half changes at bucket ends
// (every ~65 ids on C5), so a group with one bucket end inside blends the
// two high halves by lane, and only a group with several ends goes id by id.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace {

// position p of the output belongs to bucket `b` of query `q`: its ids end
// (exclusive, absolute position) at `end`
struct Cursor {
    const uint32_t* ends;
    const uint64_t* offsets;
    uint32_t nbuckets, hb0, q, q1, b;
    uint64_t end;
    uint32_t hi;
    void load() {
        end = offsets[q] + ends[uint64_t(q) * nbuckets + b];
        hi = (hb0 + b) << 16;
    }
    // the bucket holding position p (p < offsets[q1])
    void seek(uint64_t p) {
        while (p >= end) {
            if (++b == nbuckets) {
                b = 0;
                ++q;
            }
            load();
        }
    }
};

void unpack_scalar(const uint16_t* lo16, uint32_t* out, uint64_t p, uint64_t p1, Cursor& c) {
    for (; p < p1; ++p) {
        c.seek(p);
        out[p] = c.hi | lo16[p];
    }
}

#if defined(__x86_64__)
template <bool NT>
__attribute__((target("avx2"))) inline void store8(uint32_t* at, __m256i v) {
    if (NT)
        _mm256_stream_si256(reinterpret_cast<__m256i*>(at), v);
    else
        _mm256_store_si256(reinterpret_cast<__m256i*>(at), v);
}

// NT: streaming stores (no read-for-ownership of the output lines)
template <bool NT>
__attribute__((target("avx2"))) void unpack_avx2(const uint16_t* lo16, uint32_t* out, uint64_t p, uint64_t p1,
                                                 Cursor& c) {
    // head up to a 64-byte aligned output position
    uint64_t a = p;
    while (a < p1 && (reinterpret_cast<uintptr_t>(out + a) & 63u)) ++a;
    unpack_scalar(lo16, out, p, a, c);
    p = a;
    const __m256i lane_lo = _mm256_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7);
    const __m256i lane_hi = _mm256_setr_epi32(8, 9, 10, 11, 12, 13, 14, 15);
    for (; p + 16 <= p1; p += 16) {
        c.seek(p);
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(lo16 + p));
        const __m256i x0 = _mm256_cvtepu16_epi32(_mm256_castsi256_si128(v));
        const __m256i x1 = _mm256_cvtepu16_epi32(_mm256_extracti128_si256(v, 1));
        __m256i h0, h1;
        if (c.end >= p + 16) {
            h0 = h1 = _mm256_set1_epi32(int(c.hi));
        } else {
            // lanes below k keep this bucket's high half, the rest take the
            // next non-empty bucket's -- if that one covers the group
            const uint32_t k = uint32_t(c.end - p);
            const uint32_t hi_a = c.hi;
            c.seek(c.end);
            if (c.end >= p + 16) {
                const __m256i kk = _mm256_set1_epi32(int(k));
                const __m256i ha = _mm256_set1_epi32(int(hi_a)), hb = _mm256_set1_epi32(int(c.hi));
                h0 = _mm256_blendv_epi8(hb, ha, _mm256_cmpgt_epi32(kk, lane_lo));
                h1 = _mm256_blendv_epi8(hb, ha, _mm256_cmpgt_epi32(kk, lane_hi));
            } else {
                alignas(32) uint32_t tmp[16];
                for (uint32_t j = 0; j < 16; ++j) {
                    if (j < k) {
                        tmp[j] = hi_a;
                    } else {
                        c.seek(p + j);
                        tmp[j] = c.hi;
                    }
                }
                h0 = _mm256_load_si256(reinterpret_cast<const __m256i*>(tmp));
                h1 = _mm256_load_si256(reinterpret_cast<const __m256i*>(tmp + 8));
            }
        }
        store8<NT>(out + p, _mm256_or_si256(x0, h0));
        store8<NT>(out + p + 8, _mm256_or_si256(x1, h1));
    }
    unpack_scalar(lo16, out, p, p1, c);
    _mm_sfence();
}
#endif

// output positions [p0, p1) of the queries [0, nq): the cursor starts in the
// query and bucket that hold p0 (binary searches), so a thread's share is a
// range of ids, not of queries -- a batch of few long lists still uses every
// thread
void unpack_range(const uint16_t* lo16, const uint32_t* ends, const uint64_t* offsets, uint32_t nq, uint64_t p0,
                  uint64_t p1, uint32_t hb0, uint32_t nbuckets, uint32_t* out) {
    if (p0 >= p1) return;
    // last query whose list starts at or before p0 and is not empty up to p0
    const uint32_t q = uint32_t(std::upper_bound(offsets, offsets + nq + 1, p0) - offsets) - 1;
    const uint32_t* e = ends + uint64_t(q) * nbuckets;
    const uint32_t rel = uint32_t(p0 - offsets[q]);
    const uint32_t b = uint32_t(std::upper_bound(e, e + nbuckets, rel) - e);   // first bucket ending after rel
    Cursor c{ends, offsets, nbuckets, hb0, q, nq, b < nbuckets ? b : nbuckets - 1, 0, 0};
    c.load();
#if defined(__x86_64__)
    if (__builtin_cpu_supports("avx2")) {
        // MDRQ_UNPACK_NT=0: regular stores (measurement switch)
        static const bool nt = [] {
            const char* env = getenv("MDRQ_UNPACK_NT");
            return !(env && env[0] == '0');
        }();
        if (nt)
            unpack_avx2<true>(lo16, out, p0, p1, c);
        else
            unpack_avx2<false>(lo16, out, p0, p1, c);
        return;
    }
#endif
    unpack_scalar(lo16, out, p0, p1, c);
}

}  // namespace

extern "C" int mdrq_unpack_ids16(const uint16_t* lo16, const uint32_t* ends, const uint64_t* offsets, uint32_t nq,
                                 uint32_t hb0, uint32_t nbuckets, uint32_t* out, int threads) {
    if (nq && (!lo16 || !ends || !offsets || !out || !nbuckets)) return -1;
    if (!nq) return 0;
    int T = std::max(1, threads > 0 ? threads : int(std::thread::hardware_concurrency()));
    const uint64_t first = offsets[0], total = offsets[nq] - offsets[0];
    T = int(std::min<uint64_t>(uint64_t(T), std::max<uint64_t>(1, total >> 20)));   // >= 1 Mi ids per thread
    if (T == 1) {
        unpack_range(lo16, ends, offsets, nq, first, first + total, hb0, nbuckets, out);
        return 0;
    }
    // equal shares of the ids, cut at multiples of 16 positions
    std::vector<std::thread> th;
    th.reserve(size_t(T));
    for (int t = 0; t < T; ++t) {
        const uint64_t a = first + (total * uint64_t(t) / uint64_t(T) & ~uint64_t(15));
        const uint64_t b = t + 1 == T ? first + total : first + (total * uint64_t(t + 1) / uint64_t(T) & ~uint64_t(15));
        if (a < b) th.emplace_back(unpack_range, lo16, ends, offsets, nq, a, b, hb0, nbuckets, out);
    }
    for (auto& x : th) x.join();
    return 0;
}
