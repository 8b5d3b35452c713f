// unpack_host.cpp -- host side of the 16-bit id packing (pack.cu): rebuild
// the uint32 ids of a batch from their low halves and the per-query bucket
// ends, on `threads` host threads (the queries split by id count).  Plain
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

// queries [q0, q1): output positions offsets[q0] .. offsets[q1]
void unpack_range(const uint16_t* lo16, const uint32_t* ends, const uint64_t* offsets, uint32_t q0, uint32_t q1,
                  uint32_t hb0, uint32_t nbuckets, uint32_t* out) {
    const uint64_t p0 = offsets[q0], p1 = offsets[q1];
    if (p0 >= p1) return;
    Cursor c{ends, offsets, nbuckets, hb0, q0, q1, 0, 0, 0};
    c.load();
#if defined(__x86_64__)
    if (__builtin_cpu_supports("avx2")) {
        // MDRQ_UNPACK_NT=0: regular stores (measurement switch)
        static const bool nt = [] {
            const char* e = getenv("MDRQ_UNPACK_NT");
            return !(e && e[0] == '0');
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
    int T = threads > 0 ? threads : int(std::thread::hardware_concurrency());
    T = std::max(1, std::min<int>(T, int(nq)));
    const uint64_t total = offsets[nq] - offsets[0];
    if (T == 1 || total < (1u << 20)) {
        unpack_range(lo16, ends, offsets, 0, nq, hb0, nbuckets, out);
        return 0;
    }
    // query ranges of about equal id counts
    std::vector<uint32_t> cut(size_t(T) + 1, nq);
    cut[0] = 0;
    uint32_t q = 0;
    for (int t = 1; t < T; ++t) {
        const uint64_t want = offsets[0] + total * uint64_t(t) / uint64_t(T);
        while (q < nq && offsets[q] < want) ++q;
        cut[t] = q;
    }
    std::vector<std::thread> th;
    th.reserve(size_t(T));
    for (int t = 0; t < T; ++t)
        if (cut[t] < cut[t + 1])
            th.emplace_back(unpack_range, lo16, ends, offsets, cut[t], cut[t + 1], hb0, nbuckets, out);
    for (auto& x : th) x.join();
    return 0;
}
