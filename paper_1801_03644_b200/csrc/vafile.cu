// vafile.cu -- quantile-grid VA-file for sm_100a: builder, encoder and the
// filter-and-refine scan.
//
// Replaces the reference VA-file (reference vafile.py:88-219).  The reference
// approximates every object by a 2-bit equal-width cell per dimension
// (VaGrid.cell_index, vafile.py:38-45), files objects into a sparse
// code -> bucket directory (vafile.py:106-147), enumerates candidate cells
// (vafile.py:166-199) and refines every candidate bucket exactly with
// scan_rows (vafile.py:204-219).  On the GPU the approximation is a
// per-dimension QUANTILE grid of 2^bits cells stored as one byte plane per
// dimension (columnar, 1 B per tuple per dimension instead of 4 B), the
// filter streams those planes dimension-at-a-time, and only tuples that sit
// in an edge cell of the query box are refined against the exact float32
// columns.  Soundness (no false negatives, no false positives):
//   code(v) = #{ boundaries b_i : b_i <= v }            (monotone in v)
//   code(v) <  code(lo)  =>  v < lo      code(v) > code(hi) => v > hi
//   code(lo) < code(v) < code(hi)  =>  lo < v < hi      (no refine)
// so only code(v) == code(lo) (finite lo) or == code(hi) (finite hi) needs an
// exact compare.  Parity with the reference is therefore on id sets.
#include <cub/device/device_radix_sort.cuh>

#include "launch.h"

namespace mdrq {

namespace {

constexpr int VA_THREADS = 256;
constexpr int VA_G = 2;                         // uint4 (16 codes) groups per thread
constexpr int VA_WARP_TUPLES = 32 * 16 * VA_G;  // 1024
static_assert(VA_THREADS / 32 * VA_WARP_TUPLES == kVaTile, "tile size");

__global__ void sample_kernel(const float* __restrict__ col, uint64_t step, uint64_t count,
                              float* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = col[i * step];
}

// boundary i (1 <= i < nbins) = sorted[floor(i * count / nbins)]
__global__ void pick_kernel(const float* __restrict__ sorted, uint64_t count, uint32_t nbins,
                            float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (i < nbins) out[i - 1] = sorted[(uint64_t(i) * count) / nbins];
}

// code(v) = #{b <= v}, branchless binary search over nb = 2^bits - 1 sorted
// boundaries held in shared memory; 16 codes per thread, one uint4 store.
__global__ void __launch_bounds__(256) encode_kernel(const float* __restrict__ col, uint64_t n_pad,
                                                     const float* __restrict__ bounds, uint32_t nb,
                                                     uint8_t* __restrict__ codes) {
    __shared__ float s_b[256];
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) s_b[i] = i < nb ? bounds[i] : 0.f;
    __syncthreads();
    const uint32_t K = nb + 1;  // power of two
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) * 16; i < n_pad;
         i += uint64_t(gridDim.x) * blockDim.x * 16) {
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float v = col[i + j];
            uint32_t pos = 0;
            for (uint32_t step = K >> 1; step >= 1; step >>= 1)
                if (s_b[pos + step - 1] <= v) pos += step;
            w[j >> 2] |= pos << (8 * (j & 3));
        }
        *reinterpret_cast<uint4*>(codes + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void minmax_kernel(const float* __restrict__ col, uint64_t n, float* __restrict__ out2) {
    float lo = INFINITY, hi = -INFINITY;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float v = col[i];
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // float atomics via ordered-int trick
        auto key = [](float f) {
            int i = __float_as_int(f);
            return i >= 0 ? i : (i ^ 0x7FFFFFFF);
        };
        atomicMin(reinterpret_cast<int*>(out2), key(lo));
        atomicMax(reinterpret_cast<int*>(out2) + 1, key(hi));
    }
}

__global__ void minmax_finish(float* out2) {
    int* p = reinterpret_cast<int*>(out2);
    for (int j = 0; j < 2; ++j) {
        const int k = p[j];
        p[j] = k >= 0 ? k : (k ^ 0x7FFFFFFF);
    }
}

// SWAR range test of 4 byte-codes packed in one word against a code range
// [lo, hi] (0 <= lo <= hi <= 255): v is in range iff (v - lo) mod 256 <=
// hi - lo.  Per byte, B = (v | 0x80) - (lo & 0x7f) never borrows across
// bytes; its low 7 bits are those of v - lo and bit 7 of v - lo is
// B7 ^ v7 ^ ~lo7 (all folded into one LOP3 with the per-range mask km); the
// compare d <= w takes the low-7-bit borrow t7 of (w | 0x80) - (d & 0x7f)
// and the two top bits.  Seven ALU ops per word (the v | 0x80 shared by the
// two tests of the SURE path); the verdict is bit 7 of every byte, the
// other bits are don't-care (the alive flags keep only bits 7, 15, 23, 31).
// The formula is checked exhaustively over (v, lo, hi) by a numpy
// restatement in tests/test_host.py; the kernel by the -m gpu parity tests.
constexpr uint32_t kSwarHi = 0x80808080u;

struct SwarRange {
    uint32_t c1;    // lo replicated, bit 7 of every byte cleared
    uint32_t km;    // ~0 if lo7 == 0 (bit 7 of v - lo = B7 ^ v7 ^ 1), else 0
    uint32_t wH;    // (hi - lo) replicated with bit 7 set
    uint32_t wm;    // ~0 if bit 7 of hi - lo is set
    uint32_t live;  // 0 for an empty range (every code rejected)
};

__device__ __forceinline__ SwarRange swar_range(int lo, int hi) {
    SwarRange r;
    const bool empty = lo > hi || lo > 255 || hi < 0;
    const uint32_t l = empty ? 0u : uint32_t(lo), w = empty ? 0u : uint32_t(hi - lo);
    r.c1 = (l * 0x01010101u) & ~kSwarHi;
    r.km = (l & 0x80u) ? 0u : ~0u;
    r.wH = (w * 0x01010101u) | kSwarHi;
    r.wm = (w & 0x80u) ? ~0u : 0u;
    r.live = empty ? 0u : ~0u;
    return r;
}

template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3t(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return r;
}

// flags &= in-range verdicts of the 4 codes of x (xh = x | 0x80808080).  The
// boolean stages are explicit LOP3s: left to itself the compiler turns the
// 0 / ~0 range masks into predicates and spends a SEL per word on each.
__device__ __forceinline__ uint32_t swar_and(uint32_t flags, uint32_t x, uint32_t xh, const SwarRange& r) {
    const uint32_t b = xh - r.c1;
    const uint32_t t = r.wH - (b & ~kSwarHi);
    const uint32_t d = lop3t<0x96>(b, x, r.km);            // b ^ x ^ km
    const uint32_t le = lop3t<0x8E>(d, r.wm, t);           // (wm & ~d) | (~(d ^ wm) & t)
    return lop3t<0x80>(flags, le, r.live);                 // flags & le & live
}

// flags (bits 7, 15, 23, 31) of word w -> 4-bit tuple mask
__device__ __forceinline__ uint32_t flags_to_nib(uint32_t f) {
    return ((((f >> 7) & 0x01010101u) * 0x00204081u) >> 21) & 15u;
}

// SURE: also track "strictly inside the code range" per tuple and refine
// only the edge-cell tuples (queries expected to return many tuples);
// otherwise one range test per code and every alive tuple is refined.
//
// Occupancy decides this latency-bound loop: 8 CTAs per SM (32 registers, a
// few bytes of L1 spill) measured fastest for the plain test, 6 (40
// registers) with the second (SURE) test -- C2 single queries, 1e-3: 95 us
// vs 136 us at 61 registers; tools/probe_va_single.py.
template <bool IDS, bool SURE>
__global__ void __launch_bounds__(VA_THREADS, SURE ? 6 : 8) va_scan_kernel(const ScanArgs a) {
    __shared__ uint32_t s_cnt[VA_THREADS / 32];
    __shared__ uint32_t s_ld[VA_THREADS / 32];
    __shared__ uint32_t s_rf[VA_THREADS / 32];

    const QueryDesc qd = a.descs[a.q];
    const DimPred* __restrict__ P = a.preds + qd.off;
    const uint32_t k = qd.k;
    const uint32_t tile = blockIdx.x;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    // tuple of (group g, word w, byte b) = base + g*512 + w*4 + b
    const uint64_t wbase = uint64_t(tile) * kVaTile + warp * VA_WARP_TUPLES;
    const uint64_t base = wbase + lane * 16;

    // alive (and SURE: strictly inside) flags in SWAR layout, one word per
    // 4 tuples
    uint32_t al[VA_G][4], su[VA_G][4];
#pragma unroll
    for (int g = 0; g < VA_G; ++g)
#pragma unroll
        for (int w = 0; w < 4; ++w) al[g][w] = su[g][w] = kSwarHi;
    if (uint64_t(tile + 1) * kVaTile > a.n) {
#pragma unroll
        for (int g = 0; g < VA_G; ++g)
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                uint32_t f = 0;
                const uint64_t t0 = base + g * 512 + w * 4;
                if (t0 + 0 < a.n) f |= 1u << 7;
                if (t0 + 1 < a.n) f |= 1u << 15;
                if (t0 + 2 < a.n) f |= 1u << 23;
                if (t0 + 3 < a.n) f |= 1u << 31;
                al[g][w] = f;
            }
    }

    uint32_t nload = 0;  // 16-byte code loads issued
    // two dimensions per step: both planes' loads are issued together (the
    // second one's skip decided by the alive flags before the first), so a
    // lane has 4 independent 16-byte loads in flight instead of 2
    for (uint32_t i = 0; i < k; i += 2) {
        uint32_t any = 0;
#pragma unroll
        for (int g = 0; g < VA_G; ++g) any |= al[g][0] | al[g][1] | al[g][2] | al[g][3];
        if (!__any_sync(0xFFFFFFFFu, any)) break;
        const bool two = i + 1 < k;
        const DimPred p0 = P[i];
        const DimPred p1 = P[two ? i + 1 : i];
        const SwarRange r0 = swar_range(p0.cl, p0.ch), r1 = swar_range(p1.cl, p1.ch);
        // strict interior (SURE): the edge cells excluded
        const SwarRange s0 = swar_range(int(p0.cl) + p0.edge_lo, int(p0.ch) - p0.edge_hi);
        const SwarRange s1 = swar_range(int(p1.cl) + p1.edge_lo, int(p1.ch) - p1.edge_hi);
        const uint4* c0 = reinterpret_cast<const uint4*>(a.codes + uint64_t(p0.dim) * a.stride + base);
        const uint4* c1 = reinterpret_cast<const uint4*>(a.codes + uint64_t(p1.dim) * a.stride + base);
        uint4 x0[VA_G], x1[VA_G];
#pragma unroll
        for (int g = 0; g < VA_G; ++g) {
            const uint32_t ga = al[g][0] | al[g][1] | al[g][2] | al[g][3];
            nload += ga ? (two ? 2u : 1u) : 0u;
            if (ga) {
                x0[g] = ld_stream_u4(c0 + g * 32);
                if (two) x1[g] = ld_stream_u4(c1 + g * 32);
            }
        }
#pragma unroll
        for (int g = 0; g < VA_G; ++g) {
            const uint32_t ga = al[g][0] | al[g][1] | al[g][2] | al[g][3];
            if (ga) {
                const uint32_t xw[4] = {x0[g].x, x0[g].y, x0[g].z, x0[g].w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const uint32_t xh = xw[w] | kSwarHi;
                    al[g][w] = swar_and(al[g][w], xw[w], xh, r0);
                    if constexpr (SURE) su[g][w] = swar_and(su[g][w], xw[w], xh, s0);
                }
                if (two) {
                    const uint32_t yw[4] = {x1[g].x, x1[g].y, x1[g].z, x1[g].w};
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const uint32_t yh = yw[w] | kSwarHi;
                        al[g][w] = swar_and(al[g][w], yw[w], yh, r1);
                        if constexpr (SURE) su[g][w] = swar_and(su[g][w], yw[w], yh, s1);
                    }
                }
            }
        }
    }

    // exact refinement of the alive tuples (SURE: only those in an edge cell)
    uint32_t hit[VA_G];
    uint32_t refined = 0;
#pragma unroll
    for (int g = 0; g < VA_G; ++g) {
        uint32_t h = 0, r = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            if constexpr (SURE) {
                h |= flags_to_nib(al[g][w] & su[g][w]) << (4 * w);
                r |= flags_to_nib(al[g][w] & ~su[g][w]) << (4 * w);
            } else {
                r |= flags_to_nib(al[g][w]) << (4 * w);
            }
        }
        while (r) {
            const int j = __ffs(r) - 1;
            r &= r - 1;
            ++refined;
            const uint64_t t = base + g * 512 + j;
            bool ok = true;
            for (uint32_t i = 0; i < k && ok; ++i) {
                const DimPred p = P[i];
                const float v = __ldg(a.cols + uint64_t(p.dim) * a.stride + t);
                ok = (p.lo <= v) & (v <= p.hi);
            }
            if (ok) h |= 1u << j;
        }
        hit[g] = h;
    }
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, __popc(hit[0]) + __popc(hit[1]));
    nload = __reduce_add_sync(0xFFFFFFFFu, nload);
    refined = __reduce_add_sync(0xFFFFFFFFu, refined);
    if (lane == 0) {
        s_cnt[warp] = wc;
        s_ld[warp] = nload;
        s_rf[warp] = refined;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0, ld = 0, rf = 0;
#pragma unroll
        for (int w = 0; w < VA_THREADS / 32; ++w) {
            t += s_cnt[w];
            ld += s_ld[w];
            rf += s_rf[w];
        }
        if (!IDS && t) partial_add(a, 0, t);
        // code bytes + one 4-byte column value per queried dim per refined tuple
        const unsigned long long bytes = 16ull * ld + 4ull * k * rf;
        if (bytes) partial_add(a, 1, bytes);
        if (rf) partial_add(a, 2, rf);
    }
    if (!IDS) return;
    // ids mode: two lanes share one mask word per group
#pragma unroll
    for (int g = 0; g < VA_G; ++g) {
        uint32_t v = hit[g] << (16 * (lane & 1u));
        v |= __shfl_xor_sync(0xFFFFFFFFu, v, 1);
        if ((lane & 1u) == 0) a.mask[(base + g * 512) / 32] = v;
    }
    if (lane == 0 && wc) atomicAdd(a.chunk_counts + wbase / kChunkTuples, wc);
}

}  // namespace

void launch_va_scan(const ScanArgs& a, bool ids, cudaStream_t st) {
    if (a.num_tiles == 0) return;
    if (ids) {
        if (a.va_sure)
            va_scan_kernel<true, true><<<a.num_tiles, VA_THREADS, 0, st>>>(a);
        else
            va_scan_kernel<true, false><<<a.num_tiles, VA_THREADS, 0, st>>>(a);
    } else {
        if (a.va_sure)
            va_scan_kernel<false, true><<<a.num_tiles, VA_THREADS, 0, st>>>(a);
        else
            va_scan_kernel<false, false><<<a.num_tiles, VA_THREADS, 0, st>>>(a);
    }
}

void launch_va_sample(const float* col, uint64_t n, uint64_t step, uint64_t count, float* out,
                      cudaStream_t st) {
    (void)n;
    if (!count) return;
    const uint64_t blocks = (count + 255) / 256;
    sample_kernel<<<unsigned(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(col, step, count, out);
}

void launch_va_pick_boundaries(const float* sorted, uint64_t count, uint32_t nbins, float* out,
                               cudaStream_t st) {
    pick_kernel<<<(nbins + 255) / 256, 256, 0, st>>>(sorted, count, nbins, out);
}

void launch_va_encode(const float* col, uint64_t n_pad, const float* bounds, uint32_t nb,
                      uint8_t* codes, cudaStream_t st) {
    const uint64_t threads = n_pad / 16;
    uint64_t blocks = (threads + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (!blocks) return;
    encode_kernel<<<unsigned(blocks), 256, 0, st>>>(col, n_pad, bounds, nb, codes);
}

size_t va_sort_temp_bytes(uint64_t count) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, static_cast<const float*>(nullptr),
                                   static_cast<float*>(nullptr), int(count));
    return bytes;
}

void va_sort(const float* in, float* out, uint64_t count, void* temp, size_t temp_bytes,
             cudaStream_t st) {
    cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, int(count), 0, 32, st);
}

void launch_min_max(const float* col, uint64_t n, float* out2, cudaStream_t st) {
    static const float init[2] = {INFINITY, -INFINITY};
    // encode the identities as ordered ints on the host
    int key[2];
    for (int j = 0; j < 2; ++j) {
        int i;
        memcpy(&i, &init[j], 4);
        key[j] = i >= 0 ? i : (i ^ 0x7FFFFFFF);
    }
    cudaMemcpyAsync(out2, key, sizeof(key), cudaMemcpyHostToDevice, st);
    if (n) {
        uint64_t blocks = (n + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        minmax_kernel<<<unsigned(blocks), 256, 0, st>>>(col, n, out2);
    }
    minmax_finish<<<1, 1, 0, st>>>(out2);
}

}  // namespace mdrq
