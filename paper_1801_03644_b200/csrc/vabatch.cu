// vabatch.cu -- bit-sliced multi-query VA-file pass (up to 1024 queries per
// pass over the code planes), SURVEY.md 8(f) item 1.
//
// The reference answers a batch one query at a time (bench.py:178-186), each
// query a full scan (scan.py:103-111) or a VA-file bucket walk
// (vafile.py:204-219).  Here one pass over the quantile-code byte planes
// evaluates a whole batch:
//
//   * per union dimension u and coarse cell c the host builds a 1024-bit
//     query mask OV[u][c] (queries whose box overlaps cell c in dimension u)
//     and, for unions wider than 16 dims, SU[u][c] (queries that contain
//     cell c entirely).  Word w of a mask covers queries 32w .. 32w+31 and
//     lives in shared memory; a full pass reads a 1024-bit row with 8 lanes
//     x LDS.128 (4 words each), so one instruction serves 4 tuples (LW ==
//     128; 1 / 2 words per lane remain selectable), narrow passes replicate
//     their words across the row;
//   * the warp walks its chunk of tuples in order; per tuple it ANDs the rows
//     of the tuple's cells: maybe = AND_u OV.  The cells come from a
//     tuple-major staged copy of the block's codes (<= 8 dims) or from
//     shuffles of the loaded code words.  Unions of <= 16 dims queue every
//     nonzero (tuple, word) and refine the queue lane-parallel against the
//     query bounds in shared memory and the tuple's float32 values (staged
//     tuple-major for <= 10 dims, else from global); wider unions AND the
//     SU rows as well and refine only maybe & ~sure (edge cells) from global;
//   * matches are counted per query (mode 0), per (chunk, query) (mode 1),
//     or, in ids mode, counted per (chunk, query) while (tuple, query)
//     records are staged in tuple order (mode 3); a scan over the chunk
//     counts then places every record at qoff[q] + base[chunk][q] + rank
//     (vb_scatter_kernel) -- ascending per query because every warp owns one
//     contiguous tuple range.  If the staging pool overflows, mode 2
//     recomputes the pass writing the ids directly.
//
// The coarse cell of a tuple is its stored 8-bit quantile code shifted right
// (the 2^tb-cell grid's boundaries are every 2^(8-tb)-th boundary of the
// 256-cell grid, so code_tb = code_8 >> (8 - tb) exactly).  Soundness is the
// single-query VA-file's (vafile.cu): a tuple outside a query's box in some
// dimension has a cell outside [code(lo), code(hi)] there, so OV never drops
// a match; cells strictly inside need no refinement, edge cells are refined.
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "launch.h"

namespace mdrq {

namespace {

#ifndef MDRQ_VB_THREADS
#define MDRQ_VB_THREADS 512
#endif
#ifndef MDRQ_VB_ACODE
#define MDRQ_VB_ACODE 1
#endif
constexpr int VB_THREADS = MDRQ_VB_THREADS;
constexpr int VB_WARPS = VB_THREADS / 32;
// candidate queue per warp: < 32 left over + 2 ballots x 32 lanes (a step
// drains the queue after its second and its last ballot)
constexpr uint32_t VB_QCAP = 96;

__device__ __forceinline__ float f4_get(const float4& w, uint32_t i) {
    return i == 0 ? w.x : i == 1 ? w.y : i == 2 ? w.z : w.w;
}

// staged-value slot of tuple t (in the block) and pair h in a warp's buffer:
// h * 128 + (t & 3) * 32 + ((t >> 2) ^ ((t & 3) << SW)).  Lane l stages its
// tuples 4l .. 4l+3, so every store instruction hits 32 consecutive slots in a
// permuted order (conflict-free; the earlier tuple-major layout took 4
// wavefronts per ideal one on C5).  The XOR spreads the four tuples of a lane
// over the bank groups: a refinement round reads a handful of neighbouring
// tuples (queue order is tuple order), and without it tuples 4k .. 4k+3 shared
// one bank group (2-3 wavefronts per ideal one on C5's value reads).  SW = 2
// for 8-byte slots (16 bank pairs per half warp: tuples 4k .. 4k+15 distinct
// for k % 4 == 0), 1 for 16-byte slots (8 bank groups per quarter warp)
template <int VS>
__device__ __forceinline__ uint32_t val_slot(uint32_t t, uint32_t h) {
    constexpr uint32_t SW = VS == 4 ? 1u : 2u;
    return h * 128u + ((t & 3u) << 5) + ((t >> 2) ^ ((t & 3u) << SW));
}

// LW = lanes per tuple: 32 (a pass of up to 1 024 queries, lane w = query
// word w), or 16 / 8 for passes of <= 512 / <= 256 queries, whose 16 / 8
// query words leave room for 2 / 4 tuples per warp instruction.  LW == 64 /
// 128 mark the multi-word layouts of a full pass: 16 / 8 lanes per tuple,
// lane l reads query words NW*l .. NW*l+NW-1 (NW = 2 / 4) with one LDS.64 /
// LDS.128, so one instruction covers 2 / 4 tuples x 1 024 queries (a half /
// a quarter of the table loads and address builds of LW == 32, the same
// shared-memory wavefronts).
template <int MODE, int KB, int LW>
__global__ void __launch_bounds__(VB_THREADS, 1) va_batch_kernel(const VaBatchArgs a) {
    static_assert(LW == 128 || LW == 64 || LW == 32 || LW == 16 || LW == 8, "lanes per tuple");
    constexpr int NW = LW == 128 ? 4 : LW == 64 ? 2 : 1;   // query words per lane
    constexpr bool W2 = NW > 1;                    // multi-word layout
    constexpr int LPT = W2 ? 32 / NW : LW;         // lanes per tuple
    constexpr int TPI = 32 / LPT;                  // tuples per warp instruction
    constexpr int CWS = (LW == 32 || LW == 64) ? 1 : 2;   // code words (4 tuples each) per step
    constexpr int NS = 4 * CWS / TPI;              // sub-steps per step (<= 4)
    constexpr int NOV = NS * NW > 4 ? NS * NW : 4; // overlap words per lane and step
    static_assert(NS * NW <= 8, "at most eight overlap words per lane and step");
    static_assert(!W2 || (va_batch_pv(KB) && MODE != 2), "multi-word layout: narrow unions, dense modes");
    // passes with several tuples per instruction (multi-word, or narrow) of
    // <= 8 union dims stage every block's table cells tuple-major in shared
    // memory (8 bytes per tuple): one LDS.64 hands the TPI lane groups of an
    // instruction their tuples' cells of all dims, instead of one SHFL per
    // dimension and code word (the SHFLs cost data-pipe wavefronts too)
    constexpr bool SCODE = TPI > 1 && KB <= 8 && MODE != 2;
    // multi-word passes of 9 / 10 union dims have no room for staged cells;
    // their compacted tuple list carries, per unpruned tuple, the tuple index
    // (7 bits) and the table cells of the first AND dims (CB bits each) in one
    // word, so the sub-step's one list load replaces AND of its KB shuffles
    constexpr bool ACODE = MDRQ_VB_ACODE && W2 && !SCODE && MODE != 2;
    constexpr uint32_t CB = va_batch_cells(KB) == 64 ? 6u : 5u;   // bits per cell
    constexpr int AND = ACODE ? (int(25u / CB) < KB ? int(25u / CB) : KB) : 0;
    extern __shared__ __align__(16) uint32_t sm[];
    constexpr uint32_t K = va_batch_cells(KB);     // cells per dimension (64 / 32)
    constexpr bool PV = va_batch_pv(KB);           // values + bounds in smem, overlap-only table
    constexpr int KBV = PV ? int(va_batch_vdims(KB)) : KB;
    constexpr int VS = KBV % 4 == 0 ? 4 : 2;       // floats per staging slot (float4 / float2)
    constexpr int H = PV ? KBV / VS : 1;           // staging slots per tuple
    constexpr bool DENSE = MODE != 2;              // candidates refined lane-parallel from a queue
    // values staged on chip; the recount fallback of 9/10-dim unions reads
    // them from global memory instead (its per-warp counters need the room)
    constexpr bool STAGE = PV && KB <= 10 && !(MODE == 2 && KB > 8);
    // staged unions refine on 15-bit codes (launch.h): KBV words per query in
    // shared memory instead of KBV float2 bounds
    // 11..16-dim unions stage the block's 15-bit value codes instead (two
    // dims per word, PP words per tuple in 8-byte slots): their refinement
    // runs on chip too, only a code on a bound's reads float32 from global
    constexpr bool STAGEC = MDRQ_VB_Q15 && PV && KB > 10 && MODE != 2;
    constexpr int PP = (KBV / 2 + 1) / 2 * 2;       // STAGEC: code words per tuple (even)
    constexpr bool Q15 = (STAGE || STAGEC) && va_batch_q15(KB);
    constexpr int QC4 = KBV / 4;                   // Q15: 16-byte chunks per query (+ an 8-byte tail)
    constexpr bool QT2 = KBV % 4 == 2;
    __shared__ uint32_t s_dim[KB];
    uint32_t* s_end = sm + va_batch_table_words(KB, K);
    // PV: exact query bounds [KBV/2][1024] float4 (lo_u, hi_u, lo_u+1, hi_u+1
    // of dim pair u/2) and every warp's staged block values [128 * H] slots of
    // VS floats
    float4* s_qb = reinterpret_cast<float4*>(s_end);
    // (Q15: the code words instead, [QC4][1024] uint4 then [1024] uint2)
    const uint4* s_q16 = reinterpret_cast<const uint4*>(s_end);
    const uint2* s_q16t = reinterpret_cast<const uint2*>(s_q16 + QC4 * 1024);
    float* s_val = reinterpret_cast<float*>(s_qb + (PV ? (Q15 ? 1024 * KBV / 4 : 1024 * KBV / 2) : 0));
    constexpr int WV = STAGE ? 128 * KBV : STAGEC ? 128 * PP : 0;   // staged words per warp
    uint32_t* s_rest = reinterpret_cast<uint32_t*>(s_val + VB_WARPS * WV);
    // DENSE (modes 0, 3): CTA counters u32 [1024], then every warp's candidate
    // queue: entries uint2 [QCAP] = (overlap word, tuple-in-block << 5 | query
    // word), (wide unions) containment words u32 [QCAP].
    // MODE 2: per-warp counters u16 [warps][1024].
    uint32_t* s_cnt32 = s_rest;
    uint2* s_qe = reinterpret_cast<uint2*>(s_rest + 1024);
    uint32_t* s_qs = reinterpret_cast<uint32_t*>(s_qe + VB_WARPS * VB_QCAP);
    // SCODE (PV, so no containment words): every warp's staged cells [128] uint2
    uint2* s_code = reinterpret_cast<uint2*>(s_qe + VB_WARPS * VB_QCAP);
    uint16_t* s_cnt16 = reinterpret_cast<uint16_t*>(s_rest);
    // W2 (multi-word) dense passes: every warp's compacted list of the block's
    // unpruned tuples [128] u8, after the queues and staged cells
    // (ACODE: a word per tuple, see above)
    uint8_t* s_alive = reinterpret_cast<uint8_t*>(s_qe + VB_WARPS * VB_QCAP) + (SCODE ? VB_WARPS * 128 * 8 : 0);

    // the recount pass only runs when the single-pass staging overflowed
    if (MODE == 2 && *reinterpret_cast<volatile const uint32_t*>(a.overflow) == 0) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        const uint32_t n4 = va_batch_table_words(KB, K) / 4;
        for (uint32_t i = tid; i < n4; i += VB_THREADS) dst[i] = src[i];
        if constexpr (Q15) {
            const uint4* qsrc = reinterpret_cast<const uint4*>(a.qb16);
            uint4* qdst = reinterpret_cast<uint4*>(s_qb);
            for (uint32_t i = tid; i < 1024 * KBV / 4; i += VB_THREADS) qdst[i] = qsrc[i];
        } else if constexpr (PV) {
            const uint4* qsrc = reinterpret_cast<const uint4*>(a.qbounds);
            uint4* qdst = reinterpret_cast<uint4*>(s_qb);
            for (uint32_t i = tid; i < 1024 * KBV / 2; i += VB_THREADS) qdst[i] = qsrc[i];
        }
        if (MODE == 0)
            for (uint32_t i = tid; i < 1024; i += VB_THREADS) s_cnt32[i] = 0;
        if (tid < KB) s_dim[tid] = a.udims[tid];
    }
    __syncthreads();

    const uint32_t shift = a.shift;
    // byte offset of the lane's word in a table row:
    //   PV: overlap word (u, c, w) at byte (u/2*K + c)*256 + (u%2)*128 + w*4
    //   else (overlap, containment) uint2 (u, c, w) at byte (u*K + c)*256 + w*8
    // One PRMT builds (cell << 8) | lane offset from the code word; the rest
    // is an immediate.
    // (rows of LW < 32 passes hold their LW words replicated 32 / LW times:
    // lane l reads word l, i.e. query word l % LW, conflict-free)
    const uint32_t lane_off = W2 ? (lane % LPT) * (4u * NW) : lane * (PV ? 4 : 8);
    const uint32_t lane_tup = lane / LPT;          // this lane's tuple within a sub-step
    const char* s_tab = reinterpret_cast<const char*>(sm);
    float* wval = s_val + warp * WV;               // STAGE / STAGEC: this warp's staged values / codes
    uint2* qe = s_qe + warp * VB_QCAP;
    uint2* wcode = s_code + warp * 128;            // SCODE: this warp's staged cells
    uint32_t* qs = s_qs + warp * VB_QCAP;
    uint16_t* wcnt = s_cnt16 + warp * 1024;        // MODE 2
    uint8_t* walive = s_alive + warp * 128;        // W2: compacted tuple list of the block
    uint32_t* walive32 = reinterpret_cast<uint32_t*>(s_alive) + warp * 128;   // ACODE
    const uint32_t lt = lanemask_lt();

    // Exact refinement of one query word for one tuple: bit b of the result
    // is set iff query wq + b (a candidate in `word`) contains the tuple.
    // tl = tuple within the staged block (PV), t = tuple index (wide unions).
    auto refine_word = [&](uint32_t word, uint32_t su, uint32_t tl, uint64_t t, uint32_t wq) -> uint32_t {
        uint32_t hits = PV ? 0u : su;
        uint32_t r = PV ? word : (word & ~su);
        if (r) {
            float v[PV ? KBV : KB];
            if constexpr (STAGE && VS == 4) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float4 w4 = reinterpret_cast<const float4*>(wval)[val_slot<VS>(tl, h)];
                    v[4 * h] = w4.x;
                    v[4 * h + 1] = w4.y;
                    v[4 * h + 2] = w4.z;
                    v[4 * h + 3] = w4.w;
                }
            } else if constexpr (STAGE) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float2 w2 = reinterpret_cast<const float2*>(wval)[val_slot<VS>(tl, h)];
                    v[2 * h] = w2.x;
                    v[2 * h + 1] = w2.y;
                }
            } else if constexpr (STAGEC) {
                // codes only (below); float32 values are read when needed
            } else if constexpr (PV) {
                // unions too wide to stage: the values of the dims some
                // candidate of the word constrains, from global memory
                uint32_t need = 0;
                for (uint32_t rr = r; rr; rr &= rr - 1) need |= __ldg(a.qcmask + wq + __ffs(rr) - 1);
#pragma unroll
                for (int u = 0; u < KBV; ++u)
                    v[u] = (u < KB && (need >> u & 1u)) ? __ldg(a.cols + uint64_t(s_dim[u < KB ? u : 0]) * a.stride + t)
                                                        : 0.0f;
            } else {
                // the values of the dims some candidate of the word constrains
                // (partial-match queries leave most of a wide union free)
                uint32_t need = 0;
                for (uint32_t rr = r; rr; rr &= rr - 1) need |= __ldg(a.qcmask + wq + __ffs(rr) - 1);
#pragma unroll
                for (int u = 0; u < KB; ++u)
                    v[u] = (need >> u & 1u) ? __ldg(a.cols + uint64_t(s_dim[u]) * a.stride + t) : 0.0f;
            }
            if constexpr (Q15) {
                // the tuple's codes, two dims per word (bytes 1-2 of the
                // clamped transform: 15 code bits under a clear bit 15)
                constexpr int P = KBV / 2;
                uint32_t c[STAGEC ? PP : P];
                if constexpr (STAGEC) {
#pragma unroll
                    for (int h = 0; h < PP / 2; ++h) {
                        const uint2 w2 = reinterpret_cast<const uint2*>(wval)[val_slot<2>(tl, h)];
                        c[2 * h] = w2.x;
                        c[2 * h + 1] = w2.y;
                    }
                } else {
#pragma unroll
                    for (int p2 = 0; p2 < P; ++p2) {
                        const float ta = va_batch_q15_t(v[2 * p2], a.vmin[2 * p2], a.vscale[2 * p2]);
                        const float tb = va_batch_q15_t(v[2 * p2 + 1], a.vmin[2 * p2 + 1], a.vscale[2 * p2 + 1]);
                        c[p2] = __byte_perm(__float_as_uint(ta), __float_as_uint(tb), 0x6521);
                    }
                }
                constexpr uint32_t G2 = 0x80008000u, ONE2 = 0x00010001u;
                uint32_t amb = 0;
                while (r) {
                    const int b = __ffs(r) - 1;
                    r &= r - 1;
                    const uint32_t slot = wq + (uint32_t(b) ^ ((wq >> 5) & 7u));
                    uint32_t w[KBV];   // LN[0..P-1], HG[0..P-1]
#pragma unroll
                    for (int k4 = 0; k4 < QC4; ++k4) {
                        const uint4 x = s_q16[k4 * 1024 + slot];
                        w[4 * k4] = x.x, w[4 * k4 + 1] = x.y, w[4 * k4 + 2] = x.z, w[4 * k4 + 3] = x.w;
                    }
                    if constexpr (QT2) {
                        const uint2 y = s_q16t[slot];
                        w[4 * QC4] = y.x, w[4 * QC4 + 1] = y.y;
                    }
                    uint32_t nf = G2, sr = G2;
#pragma unroll
                    for (int p2 = 0; p2 < P; ++p2) {
                        const uint32_t d1 = c[p2] + w[p2];        // bit 15 per half: c >= L
                        const uint32_t d2 = w[P + p2] - c[p2];    //                  c <= H
                        nf &= d1 & d2;
                        sr &= (d1 - ONE2) & (d2 - ONE2);          // c > L, c < H
                    }
                    const bool sure = (sr & G2) == G2;
                    hits |= uint32_t(sure) << b;
                    amb |= uint32_t(!sure && (nf & G2) == G2) << b;
                }
                // a code on a bound's: the exact float32 compare against the
                // bounds in global memory (rare)
                if constexpr (STAGEC) {
                    if (amb) {
#pragma unroll
                        for (int u = 0; u < KBV; ++u)
                            v[u] = u < KB ? __ldg(a.cols + uint64_t(s_dim[u < KB ? u : 0]) * a.stride + t) : 0.0f;
                    }
                }
                while (amb) {
                    const int b = __ffs(amb) - 1;
                    amb &= amb - 1;
                    const float4* qq = reinterpret_cast<const float4*>(a.qbounds) + (wq + (uint32_t(b) ^ ((wq >> 5) & 7u)));
                    bool ok = true;
#pragma unroll
                    for (int u2 = 0; u2 < KBV / 2; ++u2) {
                        const float4 bb = __ldg(qq + u2 * 1024);
                        ok = ok & (bb.x <= v[2 * u2]) & (v[2 * u2] <= bb.y) & (bb.z <= v[2 * u2 + 1]) &
                             (v[2 * u2 + 1] <= bb.w);
                    }
                    hits |= uint32_t(ok) << b;
                }
                return hits;
            }
            while (r) {
                const int b = __ffs(r) - 1;
                r &= r - 1;
                bool ok = true;
                if constexpr (PV) {
                    // query q's bounds sit at q ^ (word & 7): the lowest set
                    // bits the lanes pop are mostly small, the XOR spreads
                    // them over the bank groups by query word
                    const float4* qq = s_qb + (wq + (uint32_t(b) ^ ((wq >> 5) & 7u)));
                    // unstaged (wide) unions skip the dim pairs the query leaves
                    // free (their values were not loaded)
                    const uint32_t cm = STAGE ? 0xFFFFFFFFu : __ldg(a.qcmask + wq + b);
#pragma unroll
                    for (int u2 = 0; u2 < KBV / 2; ++u2)
                        if (cm >> (2 * u2) & 3u) {
                            const float4 bb = qq[u2 * 1024];
                            ok = ok & (bb.x <= v[2 * u2]) & (v[2 * u2] <= bb.y) & (bb.z <= v[2 * u2 + 1]) &
                                 (v[2 * u2 + 1] <= bb.w);
                        }
                } else {
                    // only the query's constrained dims
                    const uint32_t q = wq + b;
                    const float2* qq = a.qbounds + q * KB;
                    const uint32_t cm = __ldg(a.qcmask + q);
#pragma unroll
                    for (int u = 0; u < KB; ++u)
                        if (cm >> u & 1u) {
                            const float2 bb = __ldg(qq + u);
                            ok = ok & (bb.x <= v[u]) & (v[u] <= bb.y);
                        }
                }
                hits |= uint32_t(ok) << b;
            }
        }
        return hits;
    };

    // Walk the tuples [start, end) of a subchunk in 128-tuple blocks (lane l
    // holds tuples t0+4l .. t0+4l+3 of every union dim; the next block's codes
    // and values are loaded while this one is evaluated).  Per block:
    // before_block(t0), the block's values staged (PV), then per 4-tuple step
    // the overlap (and containment) words of the lane's query word for the 4
    // tuples: step(t0, j4, jmax, ov4, su4).
    auto for_each_step = [&](uint64_t start, uint64_t end, auto&& before_block, auto&& step) {
        uint32_t cw_n[KB];
        float4 vv_n[STAGE ? KB : 1];
        auto load_block = [&](uint64_t tb) {
#pragma unroll
            for (int u = 0; u < KB; ++u) {
                const uint64_t off = uint64_t(s_dim[u]) * a.stride + tb;
                cw_n[u] = __ldcs(reinterpret_cast<const unsigned int*>(a.codes + off) + lane);
                if constexpr (STAGE) vv_n[u] = __ldcs(reinterpret_cast<const float4*>(a.cols + off) + lane);
            }
        };
        if (start < end) load_block(start);
        for (uint64_t t0 = start; t0 < end; t0 += 128) {
            uint32_t cw[KB];
#pragma unroll
            for (int u = 0; u < KB; ++u)
                // table cells of the 4 tuples of every word: (code >> shift) per byte
                cw[u] = (cw_n[u] >> shift) & (0x01010101u * (K - 1));
            before_block(t0);
            if constexpr (STAGE) {
                // stage the block's exact values (tuple t, dims VS*h ..
                // VS*h+VS-1 in slot val_slot(t, h), zero-padded dims) so a
                // refinement reads a tuple with H LDS.128 / LDS.64
                __syncwarp();
#pragma unroll
                for (uint32_t jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        float c[4];
#pragma unroll
                        for (int e = 0; e < VS; ++e) {
                            const int u = VS * h + e;
                            c[e] = u < KB ? f4_get(vv_n[u < KB ? u : 0], jj) : 0.0f;
                        }
                        if constexpr (VS == 4)
                            reinterpret_cast<float4*>(wval)[val_slot<VS>(4 * lane + jj, h)] =
                                make_float4(c[0], c[1], c[2], c[3]);
                        else
                            reinterpret_cast<float2*>(wval)[val_slot<VS>(4 * lane + jj, h)] = make_float2(c[0], c[1]);
                    }
                if constexpr (SCODE) {
                    // cells of tuples 4*lane + b (b = 0..3), dims 0..3 / 4..7
                    // byte-transposed into (lo, hi) words
                    uint32_t c8[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) c8[u] = u < KB ? cw[u < KB ? u : 0] : 0u;
                    uint32_t lo[4], hi[4];
#pragma unroll
                    for (uint32_t b = 0; b < 4; ++b) {
                        const uint32_t sb = b | ((4u + b) << 4);   // byte b of x, byte b of y
                        lo[b] = __byte_perm(__byte_perm(c8[0], c8[1], sb), __byte_perm(c8[2], c8[3], sb), 0x5410);
                        hi[b] = __byte_perm(__byte_perm(c8[4], c8[5], sb), __byte_perm(c8[6], c8[7], sb), 0x5410);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(wcode) + 2 * lane;
                    dst[0] = make_uint4(lo[0], hi[0], lo[1], hi[1]);
                    dst[1] = make_uint4(lo[2], hi[2], lo[3], hi[3]);
                }
                __syncwarp();
            }
            if constexpr (STAGEC) {
                // the block's value codes, four dims (one 8-byte slot per
                // tuple) at a time: lane l converts its tuples 4l .. 4l+3
                __syncwarp();
#pragma unroll
                for (int h = 0; h < PP / 2; ++h) {
                    float4 x[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int u = 4 * h + e;
                        x[e] = u < KB ? __ldcs(reinterpret_cast<const float4*>(
                                                   a.cols + uint64_t(s_dim[u < KB ? u : 0]) * a.stride + t0) + lane)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (uint32_t jj = 0; jj < 4; ++jj) {
                        uint32_t tb[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int u = 4 * h + e < int(kVbStageDims) ? 4 * h + e : 0;
                            tb[e] = __float_as_uint(va_batch_q15_t(f4_get(x[e], jj), a.vmin[u], a.vscale[u]));
                        }
                        reinterpret_cast<uint2*>(wval)[val_slot<2>(4 * lane + jj, h)] =
                            make_uint2(__byte_perm(tb[0], tb[1], 0x6521), __byte_perm(tb[2], tb[3], 0x6521));
                    }
                }
                __syncwarp();
            }
            if (t0 + 128 < end) load_block(t0 + 128);
            const uint32_t jmax = uint32_t(end - t0 < 128 ? end - t0 : 128);
            // W2: the block's tuples whose cell lies outside every query of
            // the pass in some pruned dim are dropped here; the sub-steps walk
            // the compacted list (tuple index, ascending) of the rest
            uint32_t nalive = jmax;
            bool compact = false;
            if constexpr (W2 && MODE != 2) {
                if (ACODE || a.prune_dims) {
                    uint32_t nib = 0xFu;
#pragma unroll
                    for (int u = 0; u < KB; ++u)
                        if (a.prune_dims >> u & 1u) {
                            const unsigned long long cm = a.cellmask[u];
#pragma unroll
                            for (uint32_t bb = 0; bb < 4; ++bb)
                                if (!((cm >> ((cw[u] >> (8 * bb)) & 0xFFu)) & 1ull)) nib &= ~(1u << bb);
                        }
                    if (4 * lane + 4 > jmax) nib &= 4 * lane >= jmax ? 0u : (1u << (jmax - 4 * lane)) - 1u;
                    const uint32_t c = __popc(nib);
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t x2 = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (lane >= uint32_t(o)) incl += x2;
                    }
                    nalive = __shfl_sync(0xFFFFFFFFu, incl, 31);
                    compact = ACODE || nalive < jmax;
                    if (compact) {
                        uint32_t pos = incl - c;
#pragma unroll
                        for (uint32_t bb = 0; bb < 4; ++bb)
                            if (nib >> bb & 1u) {
                                MDRQ_CHECK(pos < 128u, kChkAlive);
                                if constexpr (ACODE) {
                                    // tuple index << 25 | cells of dims 0 .. AND-1
                                    uint32_t e = (4 * lane + bb) << 25;
#pragma unroll
                                    for (int u = 0; u < AND; ++u) e |= ((cw[u] >> (8 * bb)) & 0xFFu) << (CB * u);
                                    walive32[pos++] = e;
                                } else {
                                    walive[pos++] = uint8_t(4 * lane + bb);
                                }
                            }
                        __syncwarp();
                    }
                }
            }
            for (uint32_t j4 = 0; j4 < nalive; j4 += 4 * CWS) {
                // this lane's tuple (index in the block) of every sub-step and
                // whether it exists: tix / tvm
                uint32_t tix[NS];
                uint32_t pk[ACODE ? NS : 1];   // ACODE: the list word (tuple index, packed cells)
                uint32_t tvm = 0;
#pragma unroll
                for (int ss = 0; ss < NS; ++ss) {
                    const uint32_t pos = j4 + ss * TPI + (LW == 32 ? 0u : lane_tup);
                    const bool ok = pos < nalive;
                    tvm |= uint32_t(ok) << ss;
                    if constexpr (ACODE) {
                        pk[ss] = ok ? walive32[pos] : 0u;
                        tix[ss] = pk[ss] >> 25;
                    } else {
                        tix[ss] = (W2 && compact) ? (ok ? uint32_t(walive[pos]) : 0u) : pos;
                    }
                }
                // the step's CWS code words of every union dim (narrow passes
                // take 8 tuples per step for more independent work)
                // (W2: one word per sub-step, fetched for the lane's own tuple)
                constexpr int NXW = W2 ? NS : CWS;
                uint32_t xw[NXW][KB];
                uint2 sc[SCODE ? NS : 1];   // SCODE: sub-step ss's tuple cells (dims 0-3, 4-7)
                if constexpr (SCODE) {
#pragma unroll
                    for (int ss = 0; ss < NS; ++ss) sc[ss] = wcode[tix[ss]];
                } else if constexpr (W2) {
                    // sub-step ss = code word ss: each lane group fetches the
                    // word holding its own (compacted) tuple
#pragma unroll
                    for (int c = 0; c < NS; ++c)
#pragma unroll
                        for (int u = AND; u < KB; ++u) xw[c][u] = __shfl_sync(0xFFFFFFFFu, cw[u], tix[c] >> 2);
                } else {
#pragma unroll
                    for (int c = 0; c < CWS; ++c)
#pragma unroll
                        for (int u = 0; u < KB; ++u) xw[c][u] = __shfl_sync(0xFFFFFFFFu, cw[u], (j4 >> 2) + c);
                }
                // sub-step s: this lane's tuple j4 + s*TPI + lane_tup, query
                // word lane % LW (LW == 32: tuple j4 + s, word lane)
                uint32_t ov4[NOV], su4[NOV];
#pragma unroll
                for (uint32_t jj = 0; jj < NOV; ++jj) ov4[jj] = su4[jj] = 0xFFFFFFFFu;
#pragma unroll
                for (int u = 0; u < KB; u += 2)
#pragma unroll
                    for (uint32_t ss = 0; ss < NS; ++ss) {
                        // byte 0 = lane offset, byte 1 = cell of the tuple (cells
                        // are pre-masked to < K); two dims per 3-input AND
                        const uint32_t jj = ss * TPI + (LW == 32 ? 0u : lane_tup);   // tuple in the step
                        const uint32_t* x = xw[W2 ? ss : (ss * TPI) / 4];   // its code word (compile-time)
                        // W2: byte (tuple % 4) of the word fetched for this lane's tuple
                        const uint32_t sel = 0x5504u | (((W2 ? tix[ss] : jj) & 3u) << 4);
                        // row address of dim uu (SCODE: byte uu % 4 of the
                        // staged word, a compile-time selector)
                        auto addr = [&](int uu) -> uint32_t {
                            if constexpr (SCODE) {
                                return __byte_perm(uu < 4 ? sc[ss].x : sc[ss].y, lane_off, 0x5504u | ((uint32_t(uu) & 3u) << 4));
                            } else if constexpr (ACODE) {
                                if (uu < AND) {
                                    // (cell << 8) | lane offset from the packed list word
                                    const int sh = int(CB) * uu - 8;
                                    const uint32_t c8 = sh < 0 ? pk[ss] << (sh < 0 ? -sh : 0) : pk[ss] >> (sh < 0 ? 0 : sh);
                                    return (c8 & ((K - 1u) << 8)) | lane_off;
                                }
                                return __byte_perm(x[uu], lane_off, sel);
                            } else {
                                return __byte_perm(x[uu], lane_off, sel);
                            }
                        };
                        const uint32_t ca = addr(u);
                        if constexpr (W2) {
                            // words NW*l .. NW*l+NW-1 of the rows: sub-step ss
                            // keeps word h in ov4[ss + NS*h]
                            uint32_t ea[NW], eb[NW];
                            const char* ra = s_tab + ca + (u / 2) * K * 256;
                            if constexpr (NW == 4) {
                                const uint4 t4 = *reinterpret_cast<const uint4*>(ra);
                                ea[0] = t4.x, ea[1] = t4.y, ea[2] = t4.z, ea[3] = t4.w;
                            } else {
                                const uint2 t2 = *reinterpret_cast<const uint2*>(ra);
                                ea[0] = t2.x, ea[1] = t2.y;
                            }
                            if (u + 1 < KB) {
                                const uint32_t cb = addr(u + 1);
                                const char* rb = s_tab + cb + (u / 2) * K * 256 + 128;
                                if constexpr (NW == 4) {
                                    const uint4 t4 = *reinterpret_cast<const uint4*>(rb);
                                    eb[0] = t4.x, eb[1] = t4.y, eb[2] = t4.z, eb[3] = t4.w;
                                } else {
                                    const uint2 t2 = *reinterpret_cast<const uint2*>(rb);
                                    eb[0] = t2.x, eb[1] = t2.y;
                                }
#pragma unroll
                                for (int h = 0; h < NW; ++h) ov4[ss + NS * h] = ov4[ss + NS * h] & ea[h] & eb[h];
                            } else {
#pragma unroll
                                for (int h = 0; h < NW; ++h) ov4[ss + NS * h] &= ea[h];
                            }
                        } else if constexpr (PV) {
                            const uint32_t ea = *reinterpret_cast<const uint32_t*>(s_tab + ca + (u / 2) * K * 256);
                            if (u + 1 < KB) {
                                const uint32_t cb = addr(u + 1);
                                const uint32_t eb =
                                    *reinterpret_cast<const uint32_t*>(s_tab + cb + (u / 2) * K * 256 + 128);
                                ov4[ss] = ov4[ss] & ea & eb;
                            } else {
                                ov4[ss] &= ea;
                            }
                        } else {
                            const uint2 ea = *reinterpret_cast<const uint2*>(s_tab + ca + u * K * 256);
                            if (u + 1 < KB) {
                                const uint32_t cb = addr(u + 1);
                                const uint2 eb = *reinterpret_cast<const uint2*>(s_tab + cb + (u + 1) * K * 256);
                                ov4[ss] = ov4[ss] & ea.x & eb.x;
                                su4[ss] = su4[ss] & ea.y & eb.y;
                            } else {
                                ov4[ss] &= ea.x;
                                su4[ss] &= ea.y;
                            }
                        }
                    }
                step(t0, j4, jmax, ov4, su4, tix, tvm);
            }
        }
    };

    for (uint32_t g = blockIdx.x; uint64_t(g) * VB_WARPS < a.nchunks; g += gridDim.x) {
        // group g = subchunks 16g .. 16g+15 (one per warp, consecutive tuple
        // ranges); counts / bases are per group, staged blocks per subchunk
        const uint32_t chunk = g * VB_WARPS + warp;
        const bool has_chunk = chunk < a.nchunks;
        const uint64_t gstart = uint64_t(g) * VB_WARPS * a.chunk_tuples;
        const uint64_t start = uint64_t(chunk) * a.chunk_tuples;
        const uint64_t end = has_chunk ? (start + a.chunk_tuples < a.n ? start + a.chunk_tuples : a.n) : start;
        if constexpr (MODE == 3) {
            for (uint32_t q = tid; q < 1024; q += VB_THREADS) s_cnt32[q] = 0;
            __syncthreads();
        }
        if constexpr (DENSE) {
            // Candidate words (tuple, query word, overlap bits) go to the
            // warp's queue in tuple order; every 32 entries are refined with
            // one entry per lane, so the refinement and the emission run on
            // full warps instead of the one or two lanes a tuple's candidates
            // touch.
            uint32_t qn = 0;
            uint64_t blk_t0 = start;
            uint32_t blk = kNoBlock, fill = 0, nblk = 0;   // MODE 3 staging state of the subchunk
            auto process = [&](uint32_t e0, uint32_t cnt) {
                const bool act = lane < cnt;
                const uint2 ent = act ? qe[e0 + lane] : make_uint2(0u, 0u);
                const uint32_t word = ent.x, meta = ent.y;
                const uint32_t su = (!PV && act) ? qs[e0 + lane] : 0u;
                const uint32_t tl = meta >> 5, wq = (meta & 31u) * 32;
                const uint64_t t = blk_t0 + tl;
                uint32_t hits = refine_word(word, su, tl, t, wq);
                if constexpr (MODE == 0) {
                    while (hits) {
                        const int b = __ffs(hits) - 1;
                        hits &= hits - 1;
                        MDRQ_CHECK(wq + b < 1024u, kChkCounter);
                        atomicAdd(&s_cnt32[wq + b], 1u);
                    }
                } else {
                    // stage (tuple offset in the group, query) records in
                    // entry order = tuple order: warp prefix of the per-lane
                    // hit counts (a ballot when no lane has two hits)
                    const uint32_t cnt_h = __popc(hits);
                    const uint32_t anyb = __ballot_sync(0xFFFFFFFFu, cnt_h != 0);
                    if (anyb) {
                        uint32_t excl, tot;
                        // hit counts below 4 (nearly always): prefix from two
                        // bit-plane ballots instead of a shuffle scan
                        if (__ballot_sync(0xFFFFFFFFu, cnt_h > 3) == 0) {
                            const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, cnt_h & 1u);
                            const uint32_t b1 = __ballot_sync(0xFFFFFFFFu, cnt_h & 2u);
                            excl = __popc(b0 & lt) + 2u * __popc(b1 & lt);
                            tot = __popc(b0) + 2u * __popc(b1);
                        } else {
                            uint32_t incl = cnt_h;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const uint32_t x2 = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                                if (lane >= uint32_t(o)) incl += x2;
                            }
                            excl = incl - cnt_h;
                            tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
                        }
                        if (blk != kNoBlock - 1 && (blk == kNoBlock || fill + tot > kRecBlock)) {
                            uint32_t nb = 0;
                            if (lane == 0) {
                                nb = atomicAdd(a.cursor, 1u);
                                if (nb >= a.max_blocks) {
                                    atomicExch(a.overflow, 1u);
                                    atomicExch(a.overflow + 1, 1u);   // sticky: some pass of the batch overflowed
                                    nb = kNoBlock - 1;   // stop staging this subchunk
                                } else {
                                    a.blk_chunk[nb] = chunk;
                                    a.blk_seq[nb] = nblk;
                                }
                                if (blk != kNoBlock) a.blk_count[blk] = fill;
                            }
                            blk = __shfl_sync(0xFFFFFFFFu, nb, 0);
                            nblk += blk != kNoBlock - 1;
                            fill = 0;
                        }
                        const bool stage_on = blk != kNoBlock - 1;
                        uint32_t* dst = a.rec + uint64_t(stage_on ? blk : 0) * kRecBlock + fill + excl;
                        const uint32_t trel = uint32_t(t - gstart) << 10;
                        while (hits) {
                            const int b = __ffs(hits) - 1;
                            hits &= hits - 1;
                            const uint32_t q = wq + b;
                            MDRQ_CHECK(!stage_on || dst < a.rec + (uint64_t(blk) + 1) * kRecBlock, kChkRecBlock);
                            MDRQ_CHECK(q < 1024u && t - gstart < (1ull << 22), kChkCounter);
                            if (stage_on) *dst++ = trel | q;
                            atomicAdd(&s_cnt32[q], 1u);
                        }
                        fill += tot;
                    }
                }
            };
            auto flush = [&]() {
                if (qn) {
                    __syncwarp();
                    process(0, qn);
                    qn = 0;
                }
            };
            // refine every full 32 entries, keep the rest at the front
            auto drain = [&]() {
                if (qn >= 32) {
                    __syncwarp();
                    uint32_t e0 = 0;
                    for (; e0 + 32 <= qn; e0 += 32) process(e0, 32);
                    // move the < 32 remaining entries to the front
                    const uint32_t rem = qn - e0;
                    uint2 me = make_uint2(0u, 0u);
                    uint32_t ms = 0;
                    if (lane < rem) {
                        me = qe[e0 + lane];
                        if constexpr (!PV) ms = qs[e0 + lane];
                    }
                    __syncwarp();
                    if (lane < rem) {
                        qe[lane] = me;
                        if constexpr (!PV) qs[lane] = ms;
                    }
                    __syncwarp();
                    qn = rem;
                }
            };
            for_each_step(
                start, end,
                [&](uint64_t t0) {
                    flush();   // the queued entries need the previous block's staged values
                    blk_t0 = t0;
                },
                [&](uint64_t, uint32_t j4, uint32_t jmax, const uint32_t(&ov4)[NOV], const uint32_t(&su4)[NOV],
                    const uint32_t(&tix)[NS], uint32_t tvm) {
                    if constexpr (W2) {
                        // multi-word layouts queue tuple-major -- tuple, then
                        // query word ascending (lane order is (tuple, l), a
                        // lane's words 4l..4l+3 are consecutive) -- so a
                        // refinement round covers few tuples and consecutive
                        // words (the bound slots' swizzle keys on the word) and
                        // the records of a query stay far apart for the scatter.
                        // A lane's rank = the prefix of its nonzero-word count
                        // over the lanes below, from the count's bit planes.
                        uint32_t pl[NS][3], nzm[NS], nb = 0;
#pragma unroll
                        for (uint32_t ss = 0; ss < NS; ++ss) {
                            uint32_t m = 0;
#pragma unroll
                            for (int h = 0; h < NW; ++h) m |= uint32_t(ov4[ss + NS * h] != 0u) << h;
                            if (!(tvm >> ss & 1u)) m = 0;
                            nzm[ss] = m;
                            const uint32_t c = __popc(m);
                            pl[ss][0] = __ballot_sync(0xFFFFFFFFu, c & 1u);
                            pl[ss][1] = __ballot_sync(0xFFFFFFFFu, c & 2u);
                            pl[ss][2] = NW == 4 ? __ballot_sync(0xFFFFFFFFu, c & 4u) : 0u;
                            nb += __popc(pl[ss][0]) + 2u * __popc(pl[ss][1]) + 4u * __popc(pl[ss][2]);
                        }
                        // queue the entries of sub-step ss's lanes in `lanes`
                        auto put = [&](uint32_t ss, uint32_t lanes) {
                            const uint32_t below = lt & lanes;
                            uint32_t slot = qn + __popc(pl[ss][0] & below) + 2u * __popc(pl[ss][1] & below) +
                                            4u * __popc(pl[ss][2] & below);
                            if (lanes >> lane & 1u) {
                                const uint32_t mb = ((tix[ss] << 5) | (NW * (lane % LPT)));
#pragma unroll
                                for (int h = 0; h < NW; ++h)
                                    if (nzm[ss] >> h & 1u) {
                                        MDRQ_CHECK(slot < VB_QCAP, kChkQueue);
                                        qe[slot++] = make_uint2(ov4[ss + NS * h], mb + h);
                                    }
                            }
                            qn += __popc(pl[ss][0] & lanes) + 2u * __popc(pl[ss][1] & lanes) +
                                  4u * __popc(pl[ss][2] & lanes);
                        };
                        if (qn + nb <= VB_QCAP) {
                            // the whole step fits the queue: one drain
#pragma unroll
                            for (uint32_t ss = 0; ss < NS; ++ss) put(ss, 0xFFFFFFFFu);
                            drain();
                        } else {
                            // dense step: half a sub-step (<= 64 entries) between drains
#pragma unroll
                            for (uint32_t ss = 0; ss < NS; ++ss) {
                                put(ss, 0x0000FFFFu);
                                drain();
                                put(ss, 0xFFFF0000u);
                                drain();
                            }
                        }
                    } else {
                    // lanes ascending = tuples ascending, then words
                    constexpr uint32_t NB = NS * NW;   // ballots per step
                    uint32_t bal[NB], meta[NB], nb = 0;
#pragma unroll
                    for (uint32_t s2 = 0; s2 < NB; ++s2) {
                        const uint32_t ss = s2 % NS;
                        const uint32_t jj = ss * TPI + (LW == 32 ? 0u : lane_tup);
                        meta[s2] = ((j4 + jj) << 5) | (lane % LW);
                        bal[s2] = __ballot_sync(0xFFFFFFFFu, ov4[s2] != 0u && j4 + jj < jmax);
                        nb += __popc(bal[s2]);
                    }
                    if (qn + nb <= VB_QCAP) {
                        // the whole step fits the queue: all entries at once
                        // (independent ballots, no drain between them)
#pragma unroll
                        for (uint32_t s2 = 0; s2 < NB; ++s2) {
                            if (bal[s2] >> lane & 1u) {
                                const uint32_t slot = qn + __popc(bal[s2] & lt);
                                MDRQ_CHECK(slot < VB_QCAP, kChkQueue);
                                qe[slot] = make_uint2(ov4[s2], meta[s2]);
                                if constexpr (!PV) qs[slot] = su4[s2];
                            }
                            qn += __popc(bal[s2]);
                        }
                        drain();
                    } else {
                        // dense step: < 32 + 2 ballots between drains
#pragma unroll
                        for (uint32_t s2 = 0; s2 < NB; ++s2) {
                            if (bal[s2] >> lane & 1u) {
                                const uint32_t slot = qn + __popc(bal[s2] & lt);
                                MDRQ_CHECK(slot < VB_QCAP, kChkQueue);
                                qe[slot] = make_uint2(ov4[s2], meta[s2]);
                                if constexpr (!PV) qs[slot] = su4[s2];
                            }
                            qn += __popc(bal[s2]);
                            if (s2 % 2 == 1 || s2 + 1 == NB) drain();
                        }
                    }
                    }
                });
            flush();
            if (MODE == 3 && has_chunk && lane == 0) {
                if (blk < kNoBlock - 1) a.blk_count[blk] = fill;
                a.chunk_nblk[chunk] = nblk;
            }
        } else {
            // MODE 2, the fallback when the staging pool overflowed: count the
            // subchunk per query, prefix the warps' counts within the group,
            // then walk the subchunk again writing ids in place (chunk_counts
            // is sized for subchunks, so its rows hold the prefixes)
            const unsigned long long* __restrict__ base = a.base + uint64_t(g) * 1024;
            uint32_t* pre = a.chunk_counts;
            const uint32_t* wpre = pre + uint64_t(chunk) * 1024;
            bool write_ids = false;
            // rows of narrow passes replicate their words: only lanes that own
            // a query word of the pass count
            const uint32_t own = lane * 32 < a.nqp ? 0xFFFFFFFFu : 0u;
            auto per_tuple = [&](uint64_t t0, uint32_t j4, uint32_t jmax, const uint32_t(&ov4_in)[4],
                                 const uint32_t(&su4)[4], const uint32_t(&)[NS], uint32_t) {
                uint32_t ov4[4];
#pragma unroll
                for (uint32_t jj = 0; jj < 4; ++jj) ov4[jj] = ov4_in[jj] & own;
                uint32_t nib = 0;
#pragma unroll
                for (uint32_t jj = 0; jj < 4; ++jj) nib |= uint32_t(ov4[jj] != 0u) << jj;
                uint32_t tm = __reduce_or_sync(0xFFFFFFFFu, nib);
                if (j4 + 4 > jmax) tm &= (1u << (jmax - j4)) - 1u;
                while (tm) {
                    const uint32_t jj = __ffs(tm) - 1;
                    tm &= tm - 1;
                    const uint32_t ovw = jj == 0 ? ov4[0] : jj == 1 ? ov4[1] : jj == 2 ? ov4[2] : ov4[3];
                    const uint32_t suw = jj == 0 ? su4[0] : jj == 1 ? su4[1] : jj == 2 ? su4[2] : su4[3];
                    const uint64_t t = t0 + j4 + jj;
                    uint32_t hits = refine_word(ovw, suw, j4 + jj, t, lane * 32);
                    while (hits) {
                        const int b = __ffs(hits) - 1;
                        hits &= hits - 1;
                        const uint32_t q = lane * 32 + b;
                        if (write_ids) {
                            const unsigned long long pos = a.qoff[q] + base[q] + wpre[q] + wcnt[q];
                            if (pos < a.ids_cap) a.ids[pos] = a.id_base + uint32_t(t);
                        }
                        wcnt[q] += 1;
                    }
                }
            };
            auto nothing = [](uint64_t) {};
#pragma unroll
            for (int i = 0; i < 32; ++i) wcnt[lane * 32 + i] = 0;
            __syncwarp();
            for_each_step(start, end, nothing, per_tuple);
            __syncthreads();
            // exclusive prefix over the group's warps per query (u32, kept in
            // the per-subchunk scratch rows of chunk_counts, free after the
            // scans), the u16 counters restart as running counts
            for (uint32_t q = tid; q < 1024; q += VB_THREADS) {
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < VB_WARPS; ++w) {
                    if (g * VB_WARPS + w < a.nchunks) pre[uint64_t(g * VB_WARPS + w) * 1024 + q] = run;
                    run += s_cnt16[w * 1024 + q];
                    s_cnt16[w * 1024 + q] = 0;
                }
            }
            __threadfence_block();
            __syncthreads();
            write_ids = true;
            for_each_step(start, end, nothing, per_tuple);
            __syncthreads();
        }
        if constexpr (MODE == 3) {
            __syncthreads();
            uint32_t* out = a.chunk_counts + uint64_t(g) * 1024;
            for (uint32_t q = tid; q < 1024; q += VB_THREADS) out[q] = s_cnt32[q];
            __syncthreads();
        }
    }

    if (MODE == 0) {
        __syncthreads();
        for (uint32_t q = tid; q < a.nqp; q += VB_THREADS)
            if (s_cnt32[q]) atomicAdd(a.counts + q, (unsigned long long)s_cnt32[q]);
    }
}

// per-query exclusive scan over chunks: base[c][q], total[q].  One CTA per
// 32 queries: thread (s, ql) sums slice s of the chunks for query ql, a scan
// over the 32 slice sums in smem, then every thread writes its slice's bases.
__global__ void __launch_bounds__(1024) vb_chunk_scan_kernel(const uint32_t* __restrict__ cc, uint32_t nchunks,
                                                             uint32_t nqp, unsigned long long* __restrict__ base,
                                                             unsigned long long* __restrict__ total) {
    __shared__ unsigned long long s_sum[32][33];
    const uint32_t ql = threadIdx.x & 31u, sl = threadIdx.x >> 5;
    const uint32_t q = blockIdx.x * 32 + ql;
    const uint32_t per = (nchunks + 31) / 32;
    const uint32_t c0 = min(nchunks, sl * per), c1 = min(nchunks, c0 + per);
    unsigned long long run = 0;
    if (q < nqp)
        for (uint32_t c = c0; c < c1; ++c) run += cc[uint64_t(c) * 1024 + q];
    s_sum[sl][ql] = run;
    __syncthreads();
    if (sl == 0) {
        unsigned long long acc = 0;
        for (uint32_t i = 0; i < 32; ++i) {
            const unsigned long long v = s_sum[i][ql];
            s_sum[i][ql] = acc;
            acc += v;
        }
        if (q < nqp) total[q] = acc;
    }
    __syncthreads();
    if (q >= nqp) return;
    run = s_sum[sl][ql];
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t v = cc[uint64_t(c) * 1024 + q];
        base[uint64_t(c) * 1024 + q] = run;
        run += v;
    }
}

// exclusive prefix of v over a 1024-thread CTA (s_w: 32 scratch words)
__device__ __forceinline__ unsigned long long cta_scan_excl(unsigned long long v, unsigned long long* s_w) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
    }
    __syncthreads();
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w = s_w[lane];
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= uint32_t(o)) wi += t;
        }
        s_w[lane] = wi - w;
    }
    __syncthreads();
    return s_w[warp] + incl - v;
}

// exclusive scan of the pass's query totals, chained on offsets[q0]; in ids
// mode also the exclusive scan of the chunks' staged block counts (the
// chunk offsets of the block list)
__global__ void __launch_bounds__(1024) vb_query_scan_kernel(const unsigned long long* __restrict__ total, uint32_t nqp,
                                                             unsigned long long* offsets, unsigned long long* counts,
                                                             unsigned long long* qoff, uint32_t q0,
                                                             const uint32_t* __restrict__ chunk_nblk,
                                                             uint32_t* chunk_first, uint32_t nchunks) {
    __shared__ unsigned long long s_w[32];
    const uint32_t q = threadIdx.x;
    const unsigned long long v = q < nqp ? total[q] : 0ull;
    const unsigned long long excl = cta_scan_excl(v, s_w);
    const unsigned long long b0 = offsets[q0];
    if (q < nqp) {
        qoff[q] = b0 + excl;
        offsets[q0 + q + 1] = b0 + excl + v;
        counts[q0 + q] = v;
    }
    if (!chunk_nblk) return;
    const uint32_t per = (nchunks + 1023) / 1024;
    const uint32_t c0 = min(nchunks, q * per), c1 = min(nchunks, c0 + per);
    unsigned long long sum = 0;
    for (uint32_t c = c0; c < c1; ++c) sum += chunk_nblk[c];
    unsigned long long ex = cta_scan_excl(sum, s_w);
    for (uint32_t c = c0; c < c1; ++c) {
        chunk_first[c] = uint32_t(ex);
        ex += chunk_nblk[c];
    }
}

// Put the staged blocks in (chunk, ordinal) order: blk_list[first[chunk] +
// seq] = block.  Skipped when the pool overflowed (the scatter is too).
__global__ void __launch_bounds__(256) vb_block_list_kernel(const VaBatchArgs a) {
    if (*reinterpret_cast<volatile const uint32_t*>(a.overflow)) return;
    const uint32_t used = min(*reinterpret_cast<volatile const uint32_t*>(a.cursor), a.max_blocks);
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < used; b += gridDim.x * blockDim.x)
        a.blk_list[a.chunk_first[a.blk_chunk[b]] + a.blk_seq[b]] = b;
}

// lanes of the warp whose (active) 10-bit query equals this lane's: ten
// ballots, cheaper than MATCH.ANY on this part
__device__ __forceinline__ uint32_t match_q10(uint32_t q, bool act) {
    uint32_t m = __ballot_sync(0xFFFFFFFFu, act);
#pragma unroll
    for (int b = 0; b < 10; ++b) {
        const uint32_t bit = (q >> b) & 1u;
        const uint32_t bb = __ballot_sync(0xFFFFFFFFu, bit);
        m &= bit ? bb : ~bb;
    }
    return m;
}

// 32-bit shared-window accesses for the scatter's placement loop: the
// addresses are formed once per kernel (kept opaque, so the compiler holds
// them in registers instead of re-deriving the window base with an
// S2R SR_CgaCtaId in every iteration, which it did under the register
// pressure of the prefetched records)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("" : "+r"(a));
    return a;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" : : "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" : : "r"(a), "h"(uint16_t(v)) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" : : "r"(a), "r"(v) : "memory");
}

// Scatter the staged records of mode 3 into place.  One CTA per group (grid-
// strided) takes the group's records in windows of up to 20 blocks, sorts a
// window by query in shared memory (stable counting sort: per-warp segment
// counts, a prefix over warps and queries, then ballot-match ranking inside
// each 32-record group) and writes every query's run of ids contiguously at
// pos[q] = qoff[q] + base[group][q] + ids of earlier windows.  Runs of
// adjacent groups abut in the output, so the L2 assembles full sectors
// instead of read-modify-writing scattered 4-byte stores.
#ifndef MDRQ_SC_THREADS
#define MDRQ_SC_THREADS 512
#endif
#ifndef MDRQ_SC_PTX
#define MDRQ_SC_PTX 1
#endif
#ifndef MDRQ_SC_WIN_BLOCKS
#define MDRQ_SC_WIN_BLOCKS 20
#endif
constexpr int SC_THREADS = MDRQ_SC_THREADS;
constexpr int SC_WARPS = SC_THREADS / 32;
constexpr uint32_t SC_WIN_BLOCKS = MDRQ_SC_WIN_BLOCKS;
constexpr uint32_t SC_PER = kRecBlock / SC_THREADS;      // records per thread per block
constexpr uint32_t SC_QPT = 1024 / SC_THREADS;           // queries per thread in the prefix
constexpr uint32_t SC_WIN = SC_WIN_BLOCKS * kRecBlock;   // records per window
constexpr size_t SC_SMEM = size_t(SC_WIN) * (4 + 4) + size_t(SC_WARPS) * 1024 * (2 + 1) + 1025 * 4 + 1024 * 8;

__global__ void __launch_bounds__(SC_THREADS, 1) vb_scatter_kernel(const VaBatchArgs a) {
    extern __shared__ __align__(16) uint32_t ss[];
    unsigned long long* s_pos = reinterpret_cast<unsigned long long*>(ss);   // [1024] next output position
    uint32_t* s_rec = ss + 2 * 1024;                   // [SC_WIN] the window's records, in order
    uint32_t* s_out = s_rec + SC_WIN;                  // [SC_WIN] the records, sorted by query (stable)
    uint32_t* s_off = s_out + SC_WIN;                  // [1025] window offsets by query
    uint16_t* s_wc = reinterpret_cast<uint16_t*>(s_off + 1025);   // [warps][1024] segment counts -> offsets
    uint8_t* s_tag = reinterpret_cast<uint8_t*>(s_wc + SC_WARPS * 1024);   // [warps][1024] duplicate probe
    // the block list of the current and the next window (double-buffered)
    __shared__ uint32_t s_blk[2][SC_WIN_BLOCKS], s_bcnt[2][SC_WIN_BLOCKS], s_boff[2][SC_WIN_BLOCKS + 1];
    __shared__ uint32_t s_wsum[SC_WARPS];
    if (*reinterpret_cast<volatile const uint32_t*>(a.overflow)) return;   // mode 2 recounts instead
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
#if MDRQ_SC_PTX
    const uint32_t a_rec = smem_addr(s_rec), a_out = smem_addr(s_out), a_off = smem_addr(s_off);
    const uint32_t a_wc = smem_addr(s_wc + warp * 1024), a_tag = smem_addr(s_tag + warp * 1024);
    const uint32_t a_pos = smem_addr(s_pos);
#endif
    // window w = blocks w*20 .. w*20+19 of the group's list: ids, counts and
    // offsets into buffer p (warp 0; the caller synchronises)
    auto load_list = [&](uint32_t first, uint32_t nblk, uint32_t k0, uint32_t p) {
        if (warp != 0) return;
        const uint32_t k = k0 + lane;
        const bool in = lane < SC_WIN_BLOCKS && k < nblk;
        const uint32_t blk = in ? a.blk_list[first + k] : 0u;
        const uint32_t c = in ? a.blk_count[blk] : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= uint32_t(o)) incl += x;
        }
        if (lane < SC_WIN_BLOCKS) {
            s_blk[p][lane] = blk;
            s_bcnt[p][lane] = c;
            s_boff[p][lane] = incl - c;
        }
        if (lane == SC_WIN_BLOCKS - 1) s_boff[p][SC_WIN_BLOCKS] = incl;
    };
    // every record load of a window in flight at once: 2 per thread per block
    uint32_t v[SC_WIN_BLOCKS][SC_PER];
    auto load_records = [&](uint32_t p) {
#pragma unroll
        for (uint32_t k = 0; k < SC_WIN_BLOCKS; ++k)
#pragma unroll
            for (uint32_t h = 0; h < SC_PER; ++h) {
                const uint32_t i = tid + h * SC_THREADS;
                v[k][h] = i < s_bcnt[p][k] ? __ldcs(a.rec + uint64_t(s_blk[p][k]) * kRecBlock + i) : 0u;
            }
    };
    for (uint32_t g = blockIdx.x; g < a.ngroups; g += gridDim.x) {
        // group g: the blocks of subchunks 16g .. 16g+15, consecutive in the
        // block list; record tuple offsets are relative to the group start
        const unsigned long long* base = a.base + uint64_t(g) * 1024;
        for (uint32_t q = tid; q < 1024; q += SC_THREADS) s_pos[q] = a.qoff[q] + base[q];
        for (uint32_t i = tid; i < SC_WARPS * 1024 / 2; i += SC_THREADS) reinterpret_cast<uint32_t*>(s_wc)[i] = 0;
        const uint64_t start = uint64_t(g) * VB_WARPS * a.chunk_tuples;
        const uint32_t c0 = g * VB_WARPS, c1 = min(a.nchunks, c0 + VB_WARPS) - 1;
        const uint32_t first = a.chunk_first[c0];
        const uint32_t nblk = a.chunk_first[c1] + a.chunk_nblk[c1] - first;
        if (nblk == 0) continue;
        load_list(first, nblk, 0, 0);
        __syncthreads();
        load_records(0);
        uint32_t p = 0;
        for (uint32_t k0 = 0; k0 < nblk; k0 += SC_WIN_BLOCKS, p ^= 1u) {
            // software pipeline: this window's records arrived in v during the
            // previous window; the next window's list and records are fetched
            // while this one is sorted and written
            const uint32_t n = s_boff[p][SC_WIN_BLOCKS];
#pragma unroll
            for (uint32_t k = 0; k < SC_WIN_BLOCKS; ++k)
#pragma unroll
                for (uint32_t h = 0; h < SC_PER; ++h) {
                    const uint32_t i = tid + h * SC_THREADS;
                    if (i < s_bcnt[p][k]) s_rec[s_boff[p][k] + i] = v[k][h];
                }
            const bool more = k0 + SC_WIN_BLOCKS < nblk;
            if (more) load_list(first, nblk, k0 + SC_WIN_BLOCKS, p ^ 1u);
            __syncthreads();
            // warp w owns the contiguous segment [s0, s1) of the window
            const uint32_t seg = (n + SC_WARPS * 32 - 1) / (SC_WARPS * 32) * 32;
            const uint32_t s0 = min(n, warp * seg), s1 = min(n, s0 + seg);
            uint16_t* wc = s_wc + warp * 1024;
            {
                // segment counts: two 16-bit counters per word (a segment
                // holds <= SC_WIN / SC_WARPS records, no carry between halves)
                uint32_t* wc32 = reinterpret_cast<uint32_t*>(wc);
#if MDRQ_SC_PTX
#pragma unroll 4
                for (uint32_t j = s0 + lane; j < s1; j += 32) {
                    const uint32_t q = lds_u32(a_rec + 4u * j) & 1023u;
                    asm volatile("red.shared.add.u32 [%0], %1;" : : "r"(a_wc + 4u * (q >> 1)),
                                 "r"(1u << ((q & 1u) * 16)) : "memory");
                }
#else
#pragma unroll 4
                for (uint32_t j = s0 + lane; j < s1; j += 32) {
                    const uint32_t q = s_rec[j] & 1023u;
                    atomicAdd(wc32 + (q >> 1), 1u << ((q & 1u) * 16));
                }
#endif
            }
            __syncthreads();
            if (more) load_records(p ^ 1u);   // the next list is visible now
            // per query: exclusive prefix over the warps' segments, window total
            uint32_t tot[SC_QPT];
#pragma unroll
            for (uint32_t h = 0; h < SC_QPT; ++h) {
                const uint32_t q = tid * SC_QPT + h;
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < SC_WARPS; ++w) {
                    const uint32_t c = s_wc[w * 1024 + q];
                    s_wc[w * 1024 + q] = uint16_t(run);
                    run += c;
                }
                tot[h] = run;
            }
            // exclusive scan of the totals over the 1024 queries
            uint32_t pair = 0;
#pragma unroll
            for (uint32_t h = 0; h < SC_QPT; ++h) pair += tot[h];
            uint32_t incl = pair;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= uint32_t(o)) incl += x;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            uint32_t wbase = 0;
            for (uint32_t w = 0; w < warp; ++w) wbase += s_wsum[w];
            uint32_t ex = wbase + incl - pair;
#pragma unroll
            for (uint32_t h = 0; h < SC_QPT; ++h) {
                s_off[tid * SC_QPT + h] = ex;
                ex += tot[h];
            }
            if (tid == 0) s_off[1024] = n;
            __syncthreads();
            // stable placement: rank = earlier warps' segments + earlier
            // groups of this segment + lanes below with the same query
            uint8_t* tag = s_tag + warp * 1024;
            uint32_t j = s0;
#if MDRQ_SC_PTX
            // full 32-record groups: no tail predicates, explicit addressing;
            // the next group's record and this group's window offset are
            // loaded ahead of the dependent tag / count round trips
            if (j + 32 <= s1) {
                uint32_t r = lds_u32(a_rec + 4u * (j + lane));
                for (; j + 32 <= s1; j += 32) {
                    const uint32_t q = r & 1023u;
                    sts_u8(a_tag + q, lane);
                    const uint32_t off = lds_u32(a_off + 4u * q);
                    __syncwarp();
                    // a lane whose tag was overwritten shares its query with
                    // the lane that wrote it: only those lanes (usually one
                    // pair) need the group mask, one ballot per duplicated query
                    const uint32_t w = lds_u8(a_tag + q);
                    const uint32_t c = lds_u16(a_wc + 2u * q);
                    const uint32_t rn = j + 64 <= s1 ? lds_u32(a_rec + 4u * (j + 32 + lane)) : 0u;
                    const bool dup = w != lane;
                    uint32_t same = 1u << lane;
                    const uint32_t losers = __ballot_sync(0xFFFFFFFFu, dup);
                    if (losers) {
                        uint32_t rem = losers | __reduce_or_sync(0xFFFFFFFFu, dup ? 1u << w : 0u);
                        while (rem) {
                            const uint32_t qi = __shfl_sync(0xFFFFFFFFu, q, __ffs(rem) - 1);
                            const uint32_t grp = __ballot_sync(0xFFFFFFFFu, q == qi);
                            if (q == qi) same = grp;
                            rem &= ~grp;
                        }
                    }
                    MDRQ_CHECK(off + c + __popc(same & lt) < SC_WIN, kChkWindow);
                    sts_u32(a_out + 4u * (off + c + __popc(same & lt)), r);
                    __syncwarp();   // every lane has read wc[q] before its leader bumps it
                    if ((same & lt) == 0) sts_u16(a_wc + 2u * q, c + __popc(same));
                    // (the next group's first __syncwarp orders this update
                    // before its count reads and these tag reads before its
                    // tag writes)
                    r = rn;
                }
            }
#endif
            for (; j < s1; j += 32) {
                const bool act = j + lane < s1;
                const uint32_t r = act ? s_rec[j + lane] : 0u;
                const uint32_t q = act ? (r & 1023u) : 0xFFFFFFFFu;
                // duplicate queries inside a group are rare: probe with a
                // last-writer tag, rank with the ballot match only if needed
                if (act) tag[q] = uint8_t(lane);
                __syncwarp();
                const bool dup = act && tag[q] != lane;
                const uint32_t same = __any_sync(0xFFFFFFFFu, dup) ? match_q10(q, act) : (1u << lane);
                if (act) {
                    const uint32_t pp = s_off[q] + wc[q] + __popc(same & lt);
                    MDRQ_CHECK(pp < SC_WIN, kChkWindow);
                    s_out[pp] = r;
                }
                __syncwarp();
                if (act && (same & lt) == 0) wc[q] += __popc(same);
                __syncwarp();
            }
            __syncthreads();
            // write the runs: consecutive slots of one query are consecutive ids
#if MDRQ_SC_PTX
#pragma unroll 4
            for (uint32_t j = tid; j < n; j += SC_THREADS) {
                const uint32_t r = lds_u32(a_out + 4u * j);
                const uint32_t q = r & 1023u;
                const unsigned long long at = lds_u64(a_pos + 8u * q) + (j - lds_u32(a_off + 4u * q));
                if (at < a.ids_cap) __stcs(a.ids + at, a.id_base + uint32_t(start + (r >> 10)));
            }
#else
#pragma unroll 4
            for (uint32_t j = tid; j < n; j += SC_THREADS) {
                const uint32_t r = s_out[j];
                const uint32_t q = r & 1023u;
                const unsigned long long at = s_pos[q] + (j - s_off[q]);
                if (at < a.ids_cap) __stcs(a.ids + at, a.id_base + uint32_t(start + (r >> 10)));
            }
#endif
            __syncthreads();
            for (uint32_t q = tid; q < 1024; q += SC_THREADS) s_pos[q] += s_off[q + 1] - s_off[q];
            for (uint32_t i = tid; i < SC_WARPS * 1024 / 2; i += SC_THREADS) reinterpret_cast<uint32_t*>(s_wc)[i] = 0;
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Sorted batches (store.cu build_vb_passes): the passes ran over the batch's
// queries in slot order perm (slot i = query perm[i]), their counts, offsets
// and ids landed in slot order.  Back to query order: counts, then the
// offsets (exclusive scan), then every slot's id run moved to its query's
// place -- one CTA per run, 16-byte copies when both ends are aligned.
__global__ void vb_unpermute_counts_kernel(const uint32_t* __restrict__ perm, const unsigned long long* __restrict__ cp,
                                           unsigned long long* __restrict__ counts, uint32_t nq) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x)
        counts[perm[i]] = cp[i];
}

__global__ void __launch_bounds__(1024) vb_offsets_scan_kernel(const unsigned long long* __restrict__ counts,
                                                               uint32_t nq, unsigned long long* __restrict__ offsets) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_tot;
    unsigned long long carry = 0;
    for (uint32_t base = 0; base < nq; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const unsigned long long v = i < nq ? counts[i] : 0ull;
        const unsigned long long ex = cta_scan_excl(v, s_w);
        if (i < nq) offsets[i] = carry + ex;
        // the block total: the last thread's exclusive + value
        if (threadIdx.x == 1023) s_tot = ex + v;
        __syncthreads();
        carry += s_tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[nq] = carry;
}

// The run of slot i (n ids at src + op[i]) to its query's place: the
// destination is 16-byte aligned after a head of <= 3 words, the source is
// read as aligned 16-byte words and realigned in registers (k = source word
// offset mod 4), so every load and store is a full 16-byte access.  The
// source buffer has >= 4 words of slack past its capacity (the realigning
// read of a run's last vector may touch up to 3 words beyond it).
__global__ void __launch_bounds__(256) vb_unpermute_ids_kernel(const uint32_t* __restrict__ perm,
                                                               const unsigned long long* __restrict__ op,
                                                               const unsigned long long* __restrict__ cp,
                                                               const unsigned long long* __restrict__ offsets,
                                                               const uint32_t* __restrict__ src, uint64_t src_cap,
                                                               uint32_t* __restrict__ dst, uint64_t cap, uint32_t nq,
                                                               uint32_t q_from) {
    for (uint32_t i = blockIdx.x; i < nq; i += gridDim.x) {
        uint64_t n = cp[i];
        if (perm[i] < q_from) continue;   // packed from slot order instead (pack.cu)
        const uint64_t d0 = offsets[perm[i]];
        // truncated result (either buffer too small): the caller grows the
        // pool and reruns
        if (!n || d0 + n > cap || op[i] + n > src_cap) continue;
        const uint32_t* s = src + op[i];
        uint32_t* d = dst + d0;
        uint64_t head = ((16u - (reinterpret_cast<uintptr_t>(d) & 15u)) & 15u) / 4;
        if (head > n) head = n;
        if (threadIdx.x < head) d[threadIdx.x] = __ldcs(s + threadIdx.x);
        s += head;
        d += head;
        n -= head;
        const uint32_t k = uint32_t(reinterpret_cast<uintptr_t>(s) & 15u) / 4;
        const uint4* sa = reinterpret_cast<const uint4*>(s - k);
        uint4* d4 = reinterpret_cast<uint4*>(d);
        const uint64_t n4 = n / 4;
        if (k == 0) {
#pragma unroll 4
            for (uint64_t j = threadIdx.x; j < n4; j += blockDim.x) __stcs(d4 + j, __ldcs(sa + j));
        } else {
#pragma unroll 2
            for (uint64_t j = threadIdx.x; j < n4; j += blockDim.x) {
                const uint4 x = __ldcs(sa + j), y = __ldcs(sa + j + 1);
                uint4 o;
                if (k == 1)
                    o = make_uint4(x.y, x.z, x.w, y.x);
                else if (k == 2)
                    o = make_uint4(x.z, x.w, y.x, y.y);
                else
                    o = make_uint4(x.w, y.x, y.y, y.z);
                __stcs(d4 + j, o);
            }
        }
        for (uint64_t t = n4 * 4 + threadIdx.x; t < n; t += blockDim.x) d[t] = __ldcs(s + t);
    }
}

template <int MODE, int KB, int LW>
void run_kb_lw(const VaBatchArgs& a, cudaStream_t st) {
    const size_t smem = va_batch_smem(KB, va_batch_cells(KB), MODE);
    static size_t configured = 0;   // dynamic smem limit set so far (static smem comes on top)
    if (smem > configured) {
        cudaFuncSetAttribute(va_batch_kernel<MODE, KB, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        configured = smem;
    }
    va_batch_kernel<MODE, KB, LW><<<a.grid, VB_THREADS, smem, st>>>(a);
}

// query words per lane of a full pass over a union of kb dims: 4 up to 10
// dims, 1 above (11..16 dims, C3: the one-word order measured 27.9 / 40.6 us
// per query count / ids against 29.6 / 50.8 for four words -- its passes are
// dense, ~25 candidates per tuple, and the refinement dominates);
// MDRQ_VB_WORDS (1, 2 or 4) overrides it for every union, for comparison and
// tests
int vb_words(uint32_t kb) {
    static const int v = [] {
        const char* e = std::getenv("MDRQ_VB_WORDS");
        const int w = e ? std::atoi(e) : 0;
        return (w == 1 || w == 2 || w == 4) ? w : 0;
    }();
    return v ? v : kb <= 10 ? 4 : 1;
}

template <int MODE, int KB>
void run_kb(const VaBatchArgs& a, cudaStream_t st) {
    // narrow passes of narrow unions pack 2 / 4 tuples per instruction (the
    // recount fallback keeps one tuple per instruction)
    if constexpr (MODE != 2 && va_batch_pv(KB)) {
        if (a.lw == 8) return run_kb_lw<MODE, KB, 8>(a, st);
        if (a.lw == 16) return run_kb_lw<MODE, KB, 16>(a, st);
        // full passes: NW query words per lane, NW tuples per instruction
        if (vb_words(KB) == 4) return run_kb_lw<MODE, KB, 128>(a, st);
        if (vb_words(KB) == 2) return run_kb_lw<MODE, KB, 64>(a, st);
    }
    run_kb_lw<MODE, KB, 32>(a, st);
}

template <int MODE, int... Ks>
void dispatch(const VaBatchArgs& a, cudaStream_t st, std::integer_sequence<int, Ks...>) {
    ((a.kb == uint32_t(Ks + 1) ? run_kb<MODE, Ks + 1>(a, st) : void()), ...);
}

}  // namespace

size_t va_batch_smem(uint32_t kb, uint32_t cells, int mode) {
    // mirrors the layout at the top of va_batch_kernel
    const bool pv = va_batch_pv(kb);
    const size_t vd = va_batch_vdims(kb);
    size_t bytes = size_t(va_batch_table_words(kb, cells)) * 4;
    const bool stage = pv && kb <= 10 && !(mode == 2 && kb > 8);
    const bool stagec = MDRQ_VB_Q15 && pv && kb > 10 && mode != 2;       // staged 15-bit value codes
    if (pv) bytes += vd * 1024 * (((stage || stagec) && va_batch_q15(kb)) ? 4 : 8);  // bounds (15-bit codes / float32)
    if (stage) bytes += size_t(VB_WARPS) * 128 * vd * 4;                 // staged values
    if (stagec) bytes += size_t(VB_WARPS) * 128 * ((vd / 2 + 1) / 2 * 2) * 4;
    if (mode == 2)
        bytes += size_t(VB_WARPS) * 1024 * 2;
    else
        bytes += 1024 * 4 + size_t(VB_WARPS) * VB_QCAP * (8 + (pv ? 0 : 4));
    if (mode != 2 && pv && kb <= 8) bytes += size_t(VB_WARPS) * 128 * 8;   // staged cells (multi-word passes)
    // compacted tuple lists (a word per tuple where they carry packed cells)
    if (mode != 2 && pv) bytes += size_t(VB_WARPS) * 128 * ((MDRQ_VB_ACODE && kb > 8 && pv && vb_words(kb) > 1) ? 4 : 1);
    return bytes;
}

int va_batch_max_dims() { return kVaBatchMaxDims; }

int va_batch_words(uint32_t kb) { return vb_words(kb); }

uint32_t va_batch_warps() { return VB_WARPS; }

void launch_va_batch(const VaBatchArgs& a, int mode, cudaStream_t st) {
    if (a.n == 0 || a.grid == 0) return;
    using Seq = std::make_integer_sequence<int, kVaBatchMaxDims>;
    if (mode == 0)
        dispatch<0>(a, st, Seq{});
    else if (mode == 2)
        dispatch<2>(a, st, Seq{});
    else
        dispatch<3>(a, st, Seq{});
}

void launch_va_batch_scatter(const VaBatchArgs& a, cudaStream_t st) {
    if (a.n == 0 || a.nchunks == 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(vb_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SC_SMEM));
        configured = true;
    }
    const uint32_t blocks = std::min<uint32_t>(a.ngroups, a.grid);   // one CTA per SM
    vb_scatter_kernel<<<blocks, SC_THREADS, SC_SMEM, st>>>(a);
}

void launch_va_batch_scans(const VaBatchArgs& a, uint32_t q0, cudaStream_t st) {
    vb_chunk_scan_kernel<<<(a.nqp + 31) / 32, 1024, 0, st>>>(a.chunk_counts, a.ngroups, a.nqp, a.base, a.total);
    vb_query_scan_kernel<<<1, 1024, 0, st>>>(a.total, a.nqp, a.offsets, a.counts_all, a.qoff, q0, a.chunk_nblk,
                                             a.chunk_first, a.nchunks);
}

uint32_t launch_va_batch_unpermute(const uint32_t* perm, const unsigned long long* counts_p,
                                   const unsigned long long* offsets_p, unsigned long long* counts,
                                   unsigned long long* offsets, const uint32_t* ids_p, uint64_t src_cap,
                                   uint32_t* ids, uint64_t cap, uint32_t nq, bool with_ids, uint32_t q_from,
                                   cudaStream_t st) {
    if (!nq) return 0;
    vb_unpermute_counts_kernel<<<(nq + 255) / 256, 256, 0, st>>>(perm, counts_p, counts, nq);
    vb_offsets_scan_kernel<<<1, 1024, 0, st>>>(counts, nq, offsets);
    if (!with_ids) return 2;
    // one CTA per id run (a run is a query's ids: ~5e5 on C5)
    vb_unpermute_ids_kernel<<<std::min<uint32_t>(nq, 65535), 256, 0, st>>>(perm, offsets_p, counts_p, offsets, ids_p,
                                                                         src_cap, ids, cap, nq, q_from);
    return 3;
}

MDRQ_CHECK_FLAGS_FN(vabatch_check_flags)

void launch_va_batch_block_list(const VaBatchArgs& a, cudaStream_t st) {
    vb_block_list_kernel<<<a.grid * 4, 256, 0, st>>>(a);
}

}  // namespace mdrq
