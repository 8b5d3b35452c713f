// common.cuh -- shared device structures and helpers of the MDRQ scan engine.
//
// Comparison semantics (bit-exact with the reference): a tuple matches a
// query iff for every queried dimension d  lo_d <= v_d && v_d <= hi_d in
// IEEE float32 (_kernels_cy.pyx:31,40,104,113).  No fast-math: the library is
// compiled with -fmad=false -ftz=false -prec-div=true; only compares happen.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace mdrq {

// ---------------------------------------------------------------------------
// Checked build (MDRQ_CHECKS, `build.py --checked` -> libmdrq_b200_checked.so):
// device-side bounds checks on the shared-memory queues, staging blocks,
// scatter windows, masks and result writes.  A failed check sets bit `bit`
// of this translation unit's flag word (the first failure of a bit prints
// its line) and the kernel carries on; the host reads every unit's flags
// with mdrq_check_flags().  This stands in for compute-sanitizer, which is
// not available on the GPU pool.  Release builds compile the checks away.
#ifdef MDRQ_CHECKS
static __device__ unsigned int g_check_flags;
static __device__ __noinline__ void check_fail(unsigned bit, int line) {
    if (!(atomicOr(&g_check_flags, 1u << bit) & (1u << bit))) printf("MDRQ_CHECK failed: bit %u line %d\n", bit, line);
}
#define MDRQ_CHECK(cond, bit)                              \
    do {                                                   \
        if (!(cond)) ::mdrq::check_fail((bit), __LINE__);  \
    } while (0)
#define MDRQ_CHECK_FLAGS_FN(name)                                            \
    uint32_t name() {                                                        \
        uint32_t v = 0;                                                      \
        cudaMemcpyFromSymbol(&v, g_check_flags, sizeof(v));                  \
        const uint32_t z = 0;                                                \
        cudaMemcpyToSymbol(g_check_flags, &z, sizeof(z));                    \
        return v;                                                            \
    }
#else
#define MDRQ_CHECK(cond, bit) \
    do {                      \
    } while (0)
#define MDRQ_CHECK_FLAGS_FN(name) \
    uint32_t name() { return 0; }
#endif
// check bits
enum : unsigned {
    kChkQueue = 0,      // candidate queue slot beyond VB_QCAP
    kChkRecBlock = 1,   // staged record beyond its 1 024-record block
    kChkAlive = 2,      // compacted tuple list beyond 128
    kChkCounter = 3,    // per-query counter index beyond 1 024
    kChkWindow = 4,     // scatter window slot beyond its capacity
    kChkMask = 5,       // mask word beyond the mask
    kChkIds = 6,        // id write beyond the result pool
    kChkTuple = 7,      // tuple index beyond the block / store
};

constexpr int kMaxDims = 256;      // dimensions a store may have
constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Query descriptor (device-resident, one per query of a prepared batch).
// Only queried dimensions are listed (core.py:125 `queried`); they are
// ordered by estimated selectivity (narrowest first) so the dimension-at-a-
// time kernels retire tuples -- and skip their loads -- as early as possible.
// The verdict does not depend on the order (AND is commutative).
struct DimPred {
    float lo, hi;       // float32 bounds (RangeQuery.lower/upper, core.py:119-120)
    uint16_t dim;       // dimension id
    uint16_t cl, ch;    // VA-file code range [code(lo), code(hi)]
    uint8_t edge_lo;    // lower edge cell needs exact refinement (lo > -inf)
    uint8_t edge_hi;    // upper edge cell needs exact refinement (hi < +inf)
};
static_assert(sizeof(DimPred) == 16, "DimPred layout");

struct QueryDesc {
    uint32_t k;         // queried dimensions
    uint32_t off;       // first DimPred of this query
};

// ---------------------------------------------------------------------------
// Decoupled look-back status word (single-pass ordered compaction).
//   bits 63..34 epoch (30 bits) | bits 33..32 flag | bits 31..0 value
// A word whose epoch differs from the current launch's reads as "not yet
// published", so the status array never needs clearing between launches.
constexpr uint64_t kFlagAgg = 1ull;
constexpr uint64_t kFlagIncl = 2ull;

__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag, uint32_t v) {
    return (uint64_t(epoch & 0x3FFFFFFFu) << 34) | (flag << 32) | uint64_t(v);
}

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-cooperative look-back (warp-uniform call, all 32 lanes).  Publishes
// the tile aggregate, walks predecessors 32 at a time, publishes the
// inclusive prefix and returns the exclusive prefix of `tile`.
__device__ __forceinline__ uint32_t lookback_exclusive(uint64_t* status, uint32_t tile,
                                                       uint32_t epoch, uint32_t aggregate) {
    const uint32_t lane = lane_id();
    if (tile == 0) {
        if (lane == 0) st_status(status, pack_status(epoch, kFlagIncl, aggregate));
        return 0;
    }
    if (lane == 0) st_status(status + tile, pack_status(epoch, kFlagAgg, aggregate));
    const uint32_t ep = epoch & 0x3FFFFFFFu;
    uint32_t excl = 0;
    int64_t window = int64_t(tile) - 1;
    while (true) {
        const int64_t idx = window - int64_t(lane);
        uint64_t flag = kFlagIncl, val = 0;
        if (idx >= 0) {
            uint64_t s;
            do {
                s = ld_status(status + idx);
                flag = (uint32_t(s >> 34) == ep) ? ((s >> 32) & 3ull) : 0ull;
            } while (flag == 0);
            val = s & 0xFFFFFFFFull;
        }
        const uint32_t incl_mask = __ballot_sync(0xFFFFFFFFu, flag == kFlagIncl);
        const int stop = incl_mask ? (__ffs(incl_mask) - 1) : 31;
        uint32_t contrib = (int(lane) <= stop) ? uint32_t(val) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
        excl += contrib;
        if (incl_mask) break;
        window -= 32;
    }
    if (lane == 0) st_status(status + tile, pack_status(epoch, kFlagIncl, excl + aggregate));
    return excl;
}

// Streaming 128-bit / 32-bit loads of the column store (read once per pass).
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
    float4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t in_range4(float4 v, float lo, float hi) {
    return uint32_t((lo <= v.x) & (v.x <= hi)) | (uint32_t((lo <= v.y) & (v.y <= hi)) << 1) |
           (uint32_t((lo <= v.z) & (v.z <= hi)) << 2) | (uint32_t((lo <= v.w) & (v.w <= hi)) << 3);
}

}  // namespace mdrq
