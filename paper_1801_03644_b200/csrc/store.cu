// store.cu -- the C ABI (include/mdrq_b200.h) of the B200 MDRQ scan engine:
// device-resident stores, query preparation, launch orchestration and the
// kernel-backend entry points.
//
// Reference anchors (relative to /root/reference/pkg/src/mdrq/):
//   DataSet / RangeQuery validation         core.py:56-174
//   queried dims = not (lo == -inf and hi == +inf)          core.py:125
//   lo > hi on a queried dim raises                        core.py:126-132
//   SequentialScan / HorizontalScan / VerticalScan         scan.py:91-214
//   VaFile filter + refine                                 vafile.py:88-219
//   SearchStats counters                                   core.py:218-237
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <new>
#include <stdexcept>
#include <atomic>
#include <exception>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "launch.h"
#include "mdrq_b200.h"

namespace mdrq {

namespace {

thread_local std::string g_err;

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg) { throw Error{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation) raise(MDRQ_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
        if (e == cudaErrorNoDevice || e == cudaErrorInvalidDevice || e == cudaErrorInsufficientDriver)
            raise(MDRQ_ENODEV, std::string(what) + ": " + cudaGetErrorString(e));
        raise(MDRQ_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

#define CK(expr) ck((expr), #expr)

template <class F>
int guard(F&& f) {
    try {
        f();
        return MDRQ_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return MDRQ_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MDRQ_ECUDA;
    }
}

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void reserve(size_t count) {
        if (count <= cap && p) return;
        release();
        size_t c = count ? count : 1;
        CK(cudaMalloc(reinterpret_cast<void**>(&p), c * sizeof(T)));
        cap = c;
    }
    size_t bytes() const { return cap * sizeof(T); }
};

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// a view into a DBuf (same `.p` spelling as DBuf)
template <class T>
struct Span {
    T* p = nullptr;
};

// u64 words of a batch's accumulator block: counts, offsets, stats,
// partials, tile counters (u32, rounded up)
size_t scratch_words_base(size_t nq) { return nq + (nq + 1) + 4 * nq + nq * kPartialSlots * 4 + (nq + 1) / 2 + 1; }
// + slot-order counts / offsets of a sorted VA batch
size_t scratch_words(size_t nq) { return scratch_words_base(nq) + nq + (nq + 1); }

}  // namespace

// ----------------------------------------------------------------- kernels --
namespace {

__global__ void fill_f32_kernel(float* p, uint64_t count, float v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

// rows [*, m] -> cols [m][stride]; one 32-row x 32-dim tile per block
__global__ void transpose_kernel(const float* __restrict__ rows, uint64_t n, uint32_t m,
                                 float* __restrict__ cols, uint64_t stride) {
    __shared__ float tile[32][33];
    const uint64_t r0 = uint64_t(blockIdx.x) * 32;
    const uint32_t d0 = blockIdx.y * 32;
    for (uint32_t r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t row = r0 + r;
        const uint32_t d = d0 + threadIdx.x;
        if (row < n && d < m) tile[r][threadIdx.x] = rows[row * m + d];
    }
    __syncthreads();
    for (uint32_t dd = threadIdx.y; dd < 32; dd += blockDim.y) {
        const uint32_t d = d0 + dd;
        const uint64_t row = r0 + threadIdx.x;
        if (row < n && d < m) cols[uint64_t(d) * stride + row] = tile[threadIdx.x][dd];
    }
}

}  // namespace

void launch_fill_f32(float* p, uint64_t count, float v, cudaStream_t st) {
    if (!count) return;
    uint64_t b = (count + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    fill_f32_kernel<<<unsigned(b), 256, 0, st>>>(p, count, v);
}

void launch_transpose_rows_to_cols(const float* rows, uint64_t n, uint32_t m, float* cols, uint64_t stride,
                                   cudaStream_t st) {
    if (!n) return;
    dim3 grid(unsigned((n + 31) / 32), (m + 31) / 32);
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, n, m, cols, stride);
}

}  // namespace mdrq

using namespace mdrq;

// ------------------------------------------------------------------ batches --
namespace {

struct Pass {
    uint32_t q0 = 0, nqp = 0, kb = 0;
    bool fallback = false;   // union too wide for the batch kernel
    size_t udim_off = 0, bound_off = 0, cmask_off = 0;
};

// one pass of the bit-sliced VA batch (<= 1024 queries)
struct VbPass {
    uint32_t q0 = 0, nqp = 0, kb = 0, cells = 0, shift = 0;
    bool fallback = false;   // union wider than kVaBatchMaxDims: per-query VA
    size_t udim_off = 0, table_off = 0, qb_off = 0, cm_off = 0, q16_off = 0;
    // staged unions (va_batch_q15): the 15-bit code function of every union dim
    float vmin[kVbStageDims] = {}, vscale[kVbStageDims] = {};
    uint32_t prune = 0;                  // union dims whose cell mask is not full
    unsigned long long cellmask[kVaBatchMaxDims] = {};
};

}  // namespace

struct mdrq_batch {
    mdrq_store* owner = nullptr;
    uint32_t nq = 0;
    uint32_t path = 0;
    std::vector<QueryDesc> descs;
    std::vector<DimPred> preds;
    std::vector<Pass> passes;
    std::vector<uint16_t> udims;
    std::vector<float2> bounds;
    std::vector<unsigned long long> cmask;
    // device copies + per-batch scratch
    DBuf<QueryDesc> d_descs;
    DBuf<DimPred> d_preds;
    DBuf<uint16_t> d_udims;
    DBuf<float2> d_bounds;
    DBuf<unsigned long long> d_cmask;
    std::vector<VbPass> vb_passes;
    std::vector<uint16_t> vb_udims;
    std::vector<uint32_t> vb_tables;
    std::vector<float2> vb_qb;
    std::vector<uint32_t> vb_cm;   // per query of a pass: constrained union dims
    std::vector<uint32_t> vb_q16;  // staged unions: the queries' 15-bit bound codes (launch.h)
    DBuf<uint32_t> d_vb_q16;
    // sorted batch: slot i of the passes holds query vb_perm[i] (empty: slot = query)
    std::vector<uint32_t> vb_perm;
    DBuf<uint32_t> d_vb_perm;
    DBuf<uint16_t> d_vb_udims;
    DBuf<uint32_t> d_vb_tables;
    DBuf<float2> d_vb_qb;
    DBuf<uint32_t> d_vb_cm;
    // per-batch accumulators, carved from one allocation so one memset
    // zeroes them all per pass (enqueue)
    DBuf<unsigned long long> d_scratch;
    Span<unsigned long long> d_counts;     // [nq]
    Span<unsigned long long> d_offsets;    // [nq+1]
    Span<unsigned long long> d_stats;      // [nq][4]
    Span<unsigned long long> d_partials;   // [nq][kPartialSlots][4]
    Span<uint32_t> d_tile_counters;        // [nq]
    Span<unsigned long long> d_counts_p;   // [nq]   sorted VA batch: slot order
    Span<unsigned long long> d_offsets_p;  // [nq+1]
    // result pool of its own (stream slots); otherwise the store's pool
    bool own_pool = false;
    DBuf<uint32_t> own_ids;
    // mdrq_batch_reserve: the ids total of this batch and the pool capacity
    // that held it (mdrq_batch_ids_async refuses to run unreserved batches or
    // into a pool that has since been replaced by a smaller one)
    bool reserved = false;
    uint64_t reserved_total = 0;
    // packed stream batches (pack.cu): the ids of queries < packed_to are
    // packed straight from the slot-order lists of a sorted bit-sliced batch
    // (counts and offsets still move to query order), only the ids of the
    // queries from packed_to on are moved to query order
    uint32_t packed_to = 0;
    // which of the store's two shared result pools a packed stream batch
    // writes (its raw tail is copied out of it while the next batch runs
    // into the other one)
    uint8_t shared_pool = 0;
    // device buffers freed (the owning store was destroyed first)
    void release_device() {
        d_descs.release(); d_preds.release(); d_udims.release(); d_bounds.release(); d_cmask.release();
        d_vb_udims.release(); d_vb_tables.release(); d_vb_qb.release(); d_vb_cm.release(); d_vb_q16.release();
        d_scratch.release(); own_ids.release();
    }
};

// One slot of the pipelined ids stream (mdrq_query_ids_stream): a batch with
// its own result pool, the events that order it, and a pinned mirror of its
// total / staging-overflow flag.
// pinned host buffer, grown on demand
template <class T>
struct HBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        CK(cudaMallocHost(reinterpret_cast<void**>(&p), n * sizeof(T)));
        cap = n;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct StreamSlot {
    mdrq_batch b;
    cudaEvent_t comp = nullptr, copy = nullptr;
    unsigned long long* h_flags = nullptr;   // pinned [3]: total, overflow, ids of the packed queries
    bool busy = false;                       // a D2H of this slot is in flight
    // packed copies (pack.cu): the batch's low id halves and bucket ends on
    // the device, their pinned staging on the host, and the thread that
    // rebuilds the caller's uint32 ids from the staging
    bool packed = false;
    uint32_t q_split = 0;                    // packed batches: queries below travel packed, the rest raw
    cudaEvent_t cp0 = nullptr, cp1 = nullptr;   // around the batch's copies (timed)
    double unpack_ms = 0;                    // host unpack of the slot's last packed batch
    bool measured = false;                   // cp0 / cp1 / unpack_ms belong to a finished packed batch
    uint64_t pool_cap = 0;                   // capacity of the result pool the batch ran into
    DBuf<uint16_t> d_lo16;
    DBuf<uint32_t> d_ends;
    HBuf<uint16_t> h_lo16;
    HBuf<uint32_t> h_ends;
    std::thread unpack;
    void join() {
        if (unpack.joinable()) unpack.join();
    }
};
constexpr int kStreamSlots = 3;

struct mdrq_store {
    int device = 0;
    int num_sms = 148;
    uint64_t n = 0, n_pad = 0, n_pad_rows = 0;
    uint32_t m = 0, layouts = 0, va_bits = 0, R = 0;
    uint32_t id_base = 0;
    cudaStream_t stream = nullptr;
    DBuf<float> cols, rows;
    DBuf<uint8_t> codes;
    DBuf<float> va_bounds;
    std::vector<float> h_va_bounds;  // [m][nb]
    std::vector<float> h_minmax;     // [m][2]
    DBuf<uint64_t> status;
    uint32_t epoch = 0;
    DBuf<uint32_t> mask;             // ids mode: verdict bitmask of one query
    // multi-query columnar ids pass: [32][mask words] masks, [32][chunks]
    // chunk counts / offsets (allocated on first use)
    DBuf<uint32_t> bmask, bchunk_counts, bchunk_offs;
    // sorted VA batches: ids in slot order before they move to query order
    DBuf<uint32_t> vb_ids_slot;
    // second shared result pool of the packed stream (pool_of)
    DBuf<uint32_t> ids_alt;
    DBuf<uint32_t> chunk_counts, chunk_offs;
    uint32_t nchunks = 0;
    // bit-sliced VA batch scratch ([chunks][1024] per pass)
    DBuf<uint32_t> vb_chunk_counts;
    DBuf<unsigned long long> vb_base, vb_total, vb_qoff;
    // single-pass ids staging (linked record blocks), grown when a pass overflows
    DBuf<uint32_t> vb_rec, vb_blk_count, vb_blk_chunk, vb_blk_seq, vb_blk_list;
    // flags: cursor, overflow of the current pass, overflow of any pass of the
    // batch (sticky: read after the batch to size the staging pool)
    DBuf<uint32_t> vb_chunk_nblk, vb_chunk_first, vb_flags;
    uint32_t vb_max_blocks = 1u << 16;   // 64K blocks x 1024 records x 4 B = 256 MB
    bool vb_sized = false;               // the staging pool was sized from a counted batch
    DBuf<uint32_t> ids;              // result pool
    uint64_t last_total = 0;
    uint32_t last_nq = 0;
    uint32_t last_path = 0;
    mdrq_batch* last_batch = nullptr;
    mdrq_batch scratch;
    std::mutex mu;
    // prepared batches still alive (detached when the store goes first)
    std::unordered_set<mdrq_batch*> batches;
    // cross-stream order of the shared scratch (verdict mask, chunk counts,
    // VA staging, result pool): every enqueue records `done` on its stream,
    // an enqueue on another stream waits for it first
    cudaEvent_t done = nullptr;
    cudaStream_t done_stream = nullptr;
    // pipelined ids stream: a copy stream + slots, created on first use
    cudaStream_t copy_stream = nullptr;
    StreamSlot* slots = nullptr;
    uint64_t stream_d2h = 0, stream_packed = 0, stream_batches = 0;   // the last stream call (mdrq_stream_info)
    uint64_t stream_hint = 0;        // largest batch total seen by the stream (pre-sizes fresh slot pools)
    uint64_t stream_per_query = 0;   // largest ids-per-query average of a stream batch (packed copies or not)
    // share of a packed batch's queries that travel packed (the rest raw):
    // steered to the shortest step period of the stream
    double stream_pack_share = 1.0;
    double stream_hc_last = 0;       // hill climbing on the step period: the last window's mean
    int stream_hc_dir = -1;          // and the direction of the last move
    bool stream_no_pack = false;     // the host could not pin the packed copies' staging
    // pinned bounce buffer of the synchronous ids calls: the offsets, the VA
    // overflow flag and a speculative prefix of the ids come back in one
    // copy + one synchronisation; bounce_ids = ids of the last call held in
    // it (0 = none; mdrq_fetch_ids copies from here when they cover the result)
    uint8_t* h_bounce = nullptr;
    size_t h_bounce_cap = 0;
    uint64_t bounce_ids = 0;
    size_t bounce_head = 0;          // byte offset of those ids in the buffer
    ~mdrq_store() {
        if (done) cudaEventDestroy(done);
        if (h_bounce) cudaFreeHost(h_bounce);
        if (slots) {
            for (int i = 0; i < kStreamSlots; ++i) {
                if (slots[i].comp) cudaEventDestroy(slots[i].comp);
                if (slots[i].copy) cudaEventDestroy(slots[i].copy);
                if (slots[i].h_flags) cudaFreeHost(slots[i].h_flags);
                if (slots[i].cp0) cudaEventDestroy(slots[i].cp0);
                if (slots[i].cp1) cudaEventDestroy(slots[i].cp1);
                slots[i].join();
                slots[i].h_lo16.release();
                slots[i].h_ends.release();
            }
            delete[] slots;
        }
        if (copy_stream) {
            cudaStreamSynchronize(copy_stream);
            cudaStreamDestroy(copy_stream);
        }
    }

    uint32_t nb() const { return va_bits ? ((1u << va_bits) - 1u) : 0u; }
    uint32_t tiles_for(uint32_t path) const {
        switch (path) {
            case MDRQ_PATH_ROWWISE: return uint32_t((n + R - 1) / R);
            case MDRQ_PATH_VAFILE: return uint32_t((n + kVaTile - 1) / kVaTile);
            default: return uint32_t((n + kColTile - 1) / kColTile);
        }
    }
    uint32_t next_epoch() {
        ++epoch;
        if (epoch >= (1u << 30)) {
            CK(cudaMemsetAsync(status.p, 0, status.bytes(), stream));
            epoch = 1;
        }
        return epoch;
    }
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool is_neg_inf(float v) { return std::isinf(v) && v < 0; }
bool is_pos_inf(float v) { return std::isinf(v) && v > 0; }

uint16_t host_code(const float* b, uint32_t nb, float v) {
    // #{b <= v}; b sorted ascending under float compare.  Branch-free binary
    // search (the prefix b[0..pos) is <= v; grow it by halving steps).
    uint32_t step = 1;
    while (step * 2 <= nb) step *= 2;
    uint32_t pos = 0;
    for (; step; step >>= 1) {
        const uint32_t cand = pos + step;
        pos = (cand <= nb && b[cand - 1] <= v) ? cand : pos;
    }
    return uint16_t(pos);
}

// Host-side fan-out for a batch's descriptor work (candidate pass orders, the
// passes' tables): fn(i) for i in [0, n) on up to 8 threads, fewer when the
// node's ranks share the host (LOCAL_WORLD_SIZE).  Exceptions are rethrown.
template <class F>
void host_parallel_for(size_t n, F&& fn) {
    static const size_t max_threads = [] {
        const char* lw = getenv("LOCAL_WORLD_SIZE");
        const size_t ranks = lw ? size_t(std::max(1, std::atoi(lw))) : 1;
        return std::max<size_t>(1, std::min<size_t>(8, std::thread::hardware_concurrency() / ranks));
    }();
    const size_t T = std::min(n, max_threads);
    if (T <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::exception_ptr err;
    std::mutex emu;
    auto work = [&] {
        try {
            for (size_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i);
        } catch (...) {
            std::lock_guard<std::mutex> lk(emu);
            if (!err) err = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (size_t t = 1; t < T; ++t) th.emplace_back(work);
    work();
    for (auto& x : th) x.join();
    if (err) std::rethrow_exception(err);
}

// Passes of the bit-sliced VA batch: <= 1024 queries each; per union
// dimension u and table cell c the overlap / containment masks of the pass's
// queries (vabatch.cu).  Table cells are the stored 8-bit codes >> shift.
// A batch of more than one pass is split into passes of queries that are
// close in one or two dimensions: sorted by their low cell there, a pass's
// queries overlap only a band of those dimensions' cells, so the pass's cell
// masks are sparse and the kernel drops every tuple outside the band before
// reading its table rows (vabatch.cu, W2 passes).  Orders tried: every
// constrained dimension alone, and pairs of the four best ones (groups of
// g_a x 1024 queries sorted by dimension a, each group's passes sorted by b);
// the score of an order is the mean over its passes of the product of the
// sorted dimensions' covered-cell fractions -- the surviving tuples, since
// quantile cells hold ~equal tuple counts.  No reordering when even the best
// keeps > 85 % of the tuples, or for a single pass.  Returns slot -> query,
// empty for the identity.
std::vector<uint32_t> choose_vb_order(const mdrq_store* s, const mdrq_batch* b) {
    const uint32_t nq = b->nq, m = s->m, bits = s->va_bits;
    if (nq <= 1024 || !bits) return {};
    const uint32_t cb = std::min<uint32_t>(bits, 6), cells = 1u << cb, sh = bits - cb;
    const unsigned long long full = cells == 64 ? ~0ull : ((1ull << cells) - 1);
    // per (query, dim): cell range in `cells` units; lo > hi = empty; kFree = unconstrained
    constexpr int16_t kFree = -1;
    std::vector<int16_t> clo(size_t(nq) * m, kFree), chi(size_t(nq) * m, kFree);
    std::vector<uint8_t> used(m, 0);
    for (uint32_t q = 0; q < nq; ++q)
        for (uint32_t i = 0; i < b->descs[q].k; ++i) {
            const DimPred& p = b->preds[b->descs[q].off + i];
            used[p.dim] = 1;
            const bool empty = p.lo > p.hi;
            clo[size_t(q) * m + p.dim] = int16_t(empty ? 1 : (p.cl >> sh));
            chi[size_t(q) * m + p.dim] = int16_t(empty ? 0 : (p.ch >> sh));
        }
    // covered-cell fraction of dimension d over slots [q0, q1) of `order`
    auto coverage = [&](const std::vector<uint32_t>& order, uint32_t d, uint32_t q0, uint32_t q1) {
        unsigned long long mk = 0;
        for (uint32_t i = q0; i < q1 && mk != full; ++i) {
            const int lo = clo[size_t(order[i]) * m + d], hi = chi[size_t(order[i]) * m + d];
            if (lo == kFree) {
                mk = full;
            } else if (lo <= hi) {
                const int l = std::max(lo, 0), h = std::min(hi, int(cells) - 1);
                if (l <= h) mk |= (h - l == 63 ? ~0ull : ((1ull << (h - l + 1)) - 1)) << l;
            }
        }
        return double(__builtin_popcountll(mk & full)) / cells;
    };
    auto by_dim = [&](std::vector<uint32_t>& order, uint32_t d, size_t from, size_t to) {
        std::stable_sort(order.begin() + from, order.begin() + to, [&](uint32_t x, uint32_t y) {
            return clo[size_t(x) * m + d] < clo[size_t(y) * m + d];
        });
    };
    // mean surviving fraction of an order whose passes are sorted on dims ds
    auto score = [&](const std::vector<uint32_t>& order, std::initializer_list<uint32_t> ds) {
        double sum = 0;
        for (uint32_t q0 = 0; q0 < nq; q0 += 1024) {
            const uint32_t q1 = std::min<uint32_t>(nq, q0 + 1024);
            double f = 1.0;
            for (uint32_t d : ds) f *= coverage(order, d, q0, q1);
            sum += f * (q1 - q0);
        }
        return sum / nq;
    };
    // every candidate order is scored on its own thread
    struct Cand {
        uint32_t da, db, ga;   // ga == 0: dimension da alone
        double sc = 2.0;
        std::vector<uint32_t> order;
    };
    auto eval = [&](Cand& c) {
        c.order.resize(nq);
        for (uint32_t q = 0; q < nq; ++q) c.order[q] = q;
        by_dim(c.order, c.da, 0, nq);
        if (c.ga == 0) {
            c.sc = score(c.order, {c.da});
        } else {
            const uint32_t gb = (((nq + 1023) / 1024) + c.ga - 1) / c.ga;   // passes per group
            for (size_t g0 = 0; g0 < nq; g0 += size_t(gb) * 1024)
                by_dim(c.order, c.db, g0, std::min<size_t>(nq, g0 + size_t(gb) * 1024));
            c.sc = score(c.order, {c.da, c.db});
        }
        if (c.sc >= 0.85) std::vector<uint32_t>().swap(c.order);   // never chosen
    };
    std::vector<Cand> singles;
    for (uint32_t d = 0; d < m; ++d)
        if (used[d]) singles.push_back(Cand{d, d, 0});
    host_parallel_for(singles.size(), [&](size_t i) { eval(singles[i]); });
    std::vector<std::pair<double, uint32_t>> one;
    for (const Cand& c : singles) one.push_back({c.sc, c.da});
    std::sort(one.begin(), one.end());
    const uint32_t passes = (nq + 1023) / 1024;
    const size_t top = std::min<size_t>(one.size(), 4);
    std::vector<Cand> pairs;
    for (size_t ia = 0; ia < top; ++ia)
        for (size_t ib = 0; ib < top; ++ib) {
            if (ia == ib) continue;
            for (uint32_t ga = 2; ga <= passes / 2; ++ga) pairs.push_back(Cand{one[ia].second, one[ib].second, ga});
        }
    host_parallel_for(pairs.size(), [&](size_t i) { eval(pairs[i]); });
    // the first best in the sequential order of the candidates (singles by
    // dimension, then the pairs), as the one-thread version chose
    double best = 0.85;
    std::vector<uint32_t> best_order;
    for (std::vector<Cand>* v : {&singles, &pairs})
        for (Cand& c : *v)
            if (c.sc < best) {
                best = c.sc;
                best_order = std::move(c.order);
            }
    return best_order;
}

void build_vb_passes_ordered(const mdrq_store* s, mdrq_batch* b);

// word j (of vd) of query slot qs in a pass's 15-bit bound codes: 16-byte
// chunks [vd / 4][1024 slots], then the 8-byte tail [1024 slots] (vabatch.cu)
inline size_t vb_q16_index(uint32_t vd, uint32_t j, uint32_t qs) {
    const uint32_t c4 = vd / 4;
    return j < 4 * c4 ? (size_t(j / 4) * 1024 + qs) * 4 + j % 4 : size_t(c4) * 4096 + size_t(qs) * 2 + (j - 4 * c4);
}

void build_vb_passes(const mdrq_store* s, mdrq_batch* b) {
    static const bool no_sort = getenv("MDRQ_VB_NO_SORT") != nullptr;   // measurement / test switch
    b->vb_perm = no_sort ? std::vector<uint32_t>() : choose_vb_order(s, b);
    build_vb_passes_ordered(s, b);
    bool fb = false, prunes = false;
    for (const VbPass& ps : b->vb_passes) {
        fb |= ps.fallback;
        // only the multi-word layout (full passes of <= 10 union dims,
        // vabatch.cu) drops pruned tuples
        prunes |= !ps.fallback && ps.prune && ps.nqp > 512 && va_batch_pv(ps.kb) && va_batch_words(ps.kb) > 1;
    }
    if (!b->vb_perm.empty() && (fb || !prunes)) {
        // a pass fell back to per-query scans, which write in query order, or
        // no pass can use its cell masks: keep the batch order (the sorted
        // order would only add the move back to query order)
        b->vb_perm.clear();
        build_vb_passes_ordered(s, b);
    }
}

void build_vb_passes_ordered(const mdrq_store* s, mdrq_batch* b) {
    b->vb_passes.clear();
    b->vb_udims.clear();
    b->vb_tables.clear();
    b->vb_qb.clear();
    b->vb_cm.clear();
    b->vb_q16.clear();
    const uint32_t m = s->m, bits = s->va_bits;
    const bool sorted = !b->vb_perm.empty();
    auto query_of = [&](uint32_t slot) { return sorted ? b->vb_perm[slot] : slot; };
    // every pass's tables on its own thread, appended in pass order afterwards
    struct PassOut {
        VbPass ps;
        std::vector<uint16_t> ud;
        std::vector<uint32_t> tab, cmv, q16;
        std::vector<float2> qbv;
    };
    const uint32_t npasses = (b->nq + 1023) / 1024;
    std::vector<PassOut> outs(npasses);
    host_parallel_for(npasses, [&](size_t pi) {
        PassOut& po = outs[pi];
        VbPass& ps = po.ps;
        const uint32_t q0 = uint32_t(pi) * 1024;
        ps.q0 = q0;
        ps.nqp = std::min<uint32_t>(1024, b->nq - q0);
        std::vector<int> uidx(m, -1);
        std::vector<uint16_t>& ud = po.ud;
        for (uint32_t sl = q0; sl < q0 + ps.nqp; ++sl)
            for (uint32_t i = 0; i < b->descs[query_of(sl)].k; ++i) {
                const uint32_t d = b->preds[b->descs[query_of(sl)].off + i].dim;
                if (uidx[d] < 0) {
                    uidx[d] = 0;
                    ud.push_back(uint16_t(d));
                }
            }
        std::sort(ud.begin(), ud.end());
        if (ud.empty()) ud.push_back(0);
        for (size_t i = 0; i < ud.size(); ++i) uidx[ud[i]] = int(i);
        ps.kb = uint32_t(ud.size());
        if (int(ps.kb) > va_batch_max_dims()) {
            ps.fallback = true;
            return;
        }
        // table cells: va_batch_cells(kb) (the kernel's constant); a store
        // with fewer code bits uses only the first 2^bits cells
        ps.cells = va_batch_cells(ps.kb);
        uint32_t tb = 0;
        while ((1u << (tb + 1)) <= ps.cells) ++tb;
        tb = std::min(bits, tb);
        ps.shift = bits - tb;
        const bool pv = va_batch_pv(ps.kb);
        const uint32_t qstride = pv ? va_batch_vdims(ps.kb) : ps.kb;
        const uint32_t cells = ps.cells;
        std::vector<uint32_t>& tab = po.tab;
        tab.assign(va_batch_table_words(ps.kb, cells), 0u);
        std::vector<float2>& qbv = po.qbv;
        qbv.assign(size_t(1024) * qstride, make_float2(-INFINITY, INFINITY));
        // staged unions: the 15-bit code function per union dim (monotone; any
        // positive scale is sound, a degenerate range only sends more
        // candidates to the exact compare) and the queries' bound codes, two
        // dims per word: LN = 0x8000 - L, HG = 0x8000 + H per half; a free dim
        // is (L, H) = (0, 32767), strictly outside every value code
        const bool q15 = va_batch_q15(ps.kb);
        const uint32_t vd = va_batch_vdims(ps.kb);
        std::vector<uint32_t>& q16 = po.q16;
        if (q15) {
            for (uint32_t u = 0; u < kVbStageDims; ++u) {
                ps.vmin[u] = 0.f;
                ps.vscale[u] = FLT_MIN;
                if (u >= ps.kb || s->h_minmax.size() < size_t(2) * m) continue;
                const float mn = s->h_minmax[2 * ud[u]], mx = s->h_minmax[2 * ud[u] + 1];
                const float range = mx - mn;
                if (std::isfinite(mn)) ps.vmin[u] = mn;
                if (range > 0.f && std::isfinite(range)) {
                    const float sc = float(2.0 * (1.0 - 1.0 / 4096) / double(range));
                    if (sc > 0.f && std::isfinite(sc)) ps.vscale[u] = sc;
                }
            }
            q16.assign(size_t(1024) * vd, 0u);
            for (uint32_t j = 0; j < vd; ++j)
                for (uint32_t qs = 0; qs < 1024; ++qs)
                    q16[vb_q16_index(vd, j, qs)] = j < vd / 2 ? 0x80008000u : 0xFFFFFFFFu;
        }
        auto q15_code = [&](float x, uint32_t u) -> uint32_t {
            const float t = va_batch_q15_t(x, ps.vmin[u], ps.vscale[u]);
            uint32_t bits32;
            std::memcpy(&bits32, &t, 4);
            return (bits32 >> 8) & 0x7FFFu;
        };
        // word index of (u, c, w): overlap word, and (wide unions) the
        // containment word right after it
        auto ov_idx = [&](uint32_t u, uint32_t c, uint32_t w) -> size_t {
            return pv ? ((size_t(u / 2) * cells + c) * 2 + u % 2) * 32 + w : ((size_t(u) * cells + c) * 32 + w) * 2;
        };
        // queries unconstrained in dimension u: every cell, set once per word below
        std::vector<uint32_t> free_mask(size_t(ps.kb) * 32, 0u);
        std::vector<uint32_t>& cmv = po.cmv;
        cmv.assign(1024, 0u);
        std::vector<unsigned long long> cmask(ps.kb, 0ull);
        const unsigned long long cfull = cells == 64 ? ~0ull : ((1ull << cells) - 1);
        for (uint32_t qi = 0; qi < ps.nqp; ++qi) {
            const QueryDesc& qd = b->descs[query_of(q0 + qi)];
            const uint32_t w = qi >> 5, bit = 1u << (qi & 31);
            uint32_t constrained = 0;   // bit per union dim (kb <= 24)
            for (uint32_t i = 0; i < qd.k; ++i) {
                const DimPred& p = b->preds[qd.off + i];
                const uint32_t u = uint32_t(uidx[p.dim]);
                constrained |= 1u << u;
                // narrow unions: dim-pair-major [u/2][1024 queries][2] (lanes
                // refining different queries hit different banks); wide
                // unions: query-major [1024][kb]
                // (narrow: query qi at slot qi ^ ((qi >> 5) & 7), vabatch.cu)
                const size_t qs = qi ^ ((qi >> 5) & 7u);
                qbv[pv ? (size_t(u / 2) * 1024 + qs) * 2 + u % 2 : size_t(qi) * qstride + u] = make_float2(p.lo, p.hi);
                if (q15) {
                    // a bound outside the observed [min, max] of the dimension
                    // decides every tuple: code 0 / 32767
                    const bool have = s->h_minmax.size() >= size_t(2) * m;
                    const uint32_t L = (have && p.lo < s->h_minmax[2 * p.dim]) ? 0u : q15_code(p.lo, u);
                    const uint32_t H = (have && p.hi > s->h_minmax[2 * p.dim + 1]) ? 32767u : q15_code(p.hi, u);
                    const uint32_t sh = 16 * (u % 2), keep = ~(0xFFFFu << sh);
                    uint32_t& ln = q16[vb_q16_index(vd, u / 2, uint32_t(qs))];
                    uint32_t& hg = q16[vb_q16_index(vd, vd / 2 + u / 2, uint32_t(qs))];
                    ln = (ln & keep) | ((0x8000u - L) << sh);
                    hg = (hg & keep) | ((0x8000u + H) << sh);
                }
                if (p.lo > p.hi) continue;   // empty interval (kernel level only): no cell overlaps
                // overlap cells [lo_c, hi_c]; containment drops the edge cells
                const int lo_c = int(p.cl) >> ps.shift, hi_c = int(p.ch) >> ps.shift, top = int(cells) - 1;
                for (int c = std::max(lo_c, 0); c <= std::min(hi_c, top); ++c) {
                    tab[ov_idx(u, uint32_t(c), w)] |= bit;
                    cmask[u] |= 1ull << c;
                }
                if (!pv) {
                    const int s_lo = lo_c + (p.edge_lo ? 1 : 0), s_hi = hi_c - (p.edge_hi ? 1 : 0);
                    for (int c = std::max(s_lo, 0); c <= std::min(s_hi, top); ++c)
                        tab[ov_idx(u, uint32_t(c), w) + 1] |= bit;
                }
            }
            for (uint32_t u = 0; u < ps.kb; ++u)
                if (!(constrained >> u & 1u)) {
                    free_mask[size_t(u) * 32 + w] |= bit;
                    cmask[u] = cfull;
                }
            cmv[qi] = constrained;
        }
        for (uint32_t u = 0; u < ps.kb; ++u) {
            ps.cellmask[u] = cmask[u] & cfull;
            if (ps.cellmask[u] != cfull) ps.prune |= 1u << u;
        }
        for (uint32_t u = 0; u < ps.kb; ++u)
            for (uint32_t w = 0; w < 32; ++w) {
                const uint32_t f = free_mask[size_t(u) * 32 + w];
                if (!f) continue;
                for (uint32_t c = 0; c < cells; ++c) {
                    tab[ov_idx(u, c, w)] |= f;
                    if (!pv) tab[ov_idx(u, c, w) + 1] |= f;
                }
            }
        // narrow passes of narrow unions run LW = 8 / 16 lanes per tuple
        // (vb_args): the first W words of every row are replicated across
        // the row, so the 4 / 2 tuples of one instruction read disjoint banks
        const uint32_t lw = pv ? (ps.nqp <= 256 ? 8u : ps.nqp <= 512 ? 16u : 32u) : 32u;
        if (lw < 32)
            for (size_t row = 0; row < tab.size() / 32; ++row)
                for (uint32_t w = lw; w < 32; ++w) tab[row * 32 + w] = tab[row * 32 + w % lw];
    });
    for (PassOut& po : outs) {
        VbPass& ps = po.ps;
        if (!ps.fallback) {
            ps.udim_off = b->vb_udims.size();
            ps.table_off = b->vb_tables.size();
            ps.qb_off = b->vb_qb.size();
            ps.cm_off = b->vb_cm.size();
            ps.q16_off = b->vb_q16.size();
            b->vb_udims.insert(b->vb_udims.end(), po.ud.begin(), po.ud.end());
            b->vb_tables.insert(b->vb_tables.end(), po.tab.begin(), po.tab.end());
            b->vb_qb.insert(b->vb_qb.end(), po.qbv.begin(), po.qbv.end());
            b->vb_cm.insert(b->vb_cm.end(), po.cmv.begin(), po.cmv.end());
            b->vb_q16.insert(b->vb_q16.end(), po.q16.begin(), po.q16.end());
        }
        b->vb_passes.push_back(ps);
    }
}

// Build the host descriptors of a batch.  strict = reference RangeQuery
// semantics (lo > hi on a queried dimension raises); the kernel-level entry
// points pass strict = false (scan_rows accepts any bounds).
void build_descs(const mdrq_store* s, const float* lo, const float* hi, uint32_t nq, uint32_t path, bool strict,
                 mdrq_batch* b) {
    const uint32_t m = s->m;
    b->nq = nq;
    b->path = path;
    b->descs.assign(nq, QueryDesc{0, 0});
    b->preds.clear();
    b->passes.clear();
    b->udims.clear();
    b->bounds.clear();
    b->cmask.clear();
    const uint32_t nb = s->nb();
    std::vector<std::pair<float, uint32_t>> order;
    std::vector<uint32_t> codes(m, 0);   // per dim of the query: code(lo) | code(hi) << 16
    for (uint32_t q = 0; q < nq; ++q) {
        const float* ql = lo + uint64_t(q) * m;
        const float* qh = hi + uint64_t(q) * m;
        order.clear();
        for (uint32_t j = 0; j < m; ++j) {
            const float l = ql[j], h = qh[j];
            if (std::isnan(l) || std::isnan(h)) raise(MDRQ_EINVAL, "NaN query bounds are not allowed");
            const bool queried = !(is_neg_inf(l) && is_pos_inf(h));
            if (!queried) continue;
            if (strict && l > h) {
                char buf[160];
                snprintf(buf, sizeof buf, "lower bound exceeds upper bound in dimension %u: %g > %g", j, double(l),
                         double(h));
                raise(MDRQ_EINVAL, buf);
            }
            // estimated pass fraction, used only to order the evaluation
            float est = 1.0f;
            if (nb && !s->h_va_bounds.empty()) {
                const float* bd = s->h_va_bounds.data() + size_t(j) * nb;
                const uint16_t cl = host_code(bd, nb, l), ch = host_code(bd, nb, h);
                codes[j] = uint32_t(cl) | uint32_t(ch) << 16;
                est = float(int(ch) - int(cl) + 1) / float(nb + 1);
            } else if (!s->h_minmax.empty()) {
                const float mn = s->h_minmax[2 * j], mx = s->h_minmax[2 * j + 1];
                const double w = double(mx) - double(mn);
                if (w > 0 && std::isfinite(w)) {
                    const double a = std::max(double(l), double(mn)), c = std::min(double(h), double(mx));
                    est = float(std::max(0.0, c - a) / w);
                }
            }
            order.emplace_back(path == MDRQ_PATH_ROWWISE ? float(j) : est, j);
        }
        // stable insertion sort by estimate (a handful of dims; no allocation)
        for (size_t i = 1; i < order.size(); ++i) {
            const auto e = order[i];
            size_t k = i;
            for (; k > 0 && e.first < order[k - 1].first; --k) order[k] = order[k - 1];
            order[k] = e;
        }
        b->descs[q].k = uint32_t(order.size());
        b->descs[q].off = uint32_t(b->preds.size());
        for (auto& e : order) {
            const uint32_t j = e.second;
            DimPred p{};
            p.lo = ql[j];
            p.hi = qh[j];
            p.dim = uint16_t(j);
            if (nb) {
                p.cl = uint16_t(codes[j] & 0xFFFFu);
                p.ch = uint16_t(codes[j] >> 16);
                p.edge_lo = is_neg_inf(p.lo) ? 0 : 1;
                p.edge_hi = is_pos_inf(p.hi) ? 0 : 1;
                if (p.lo > p.hi) {  // kernel-level only: empty interval, reject every code
                    p.cl = uint16_t(nb + 1);
                    p.ch = 0;
                }
            }
            b->preds.push_back(p);
        }
    }
    if (path == MDRQ_PATH_COLUMNAR_BATCH) {
        const int maxkb = col_batch_max_dims();
        for (uint32_t q0 = 0; q0 < nq; q0 += 32) {
            Pass ps;
            ps.q0 = q0;
            ps.nqp = std::min<uint32_t>(32, nq - q0);
            std::vector<uint8_t> used(m, 0);
            for (uint32_t q = q0; q < q0 + ps.nqp; ++q)
                for (uint32_t i = 0; i < b->descs[q].k; ++i) used[b->preds[b->descs[q].off + i].dim] = 1;
            std::vector<int> uidx(m, -1);
            std::vector<uint16_t> ud;
            for (uint32_t j = 0; j < m; ++j)
                if (used[j]) {
                    uidx[j] = int(ud.size());
                    ud.push_back(uint16_t(j));
                }
            ps.kb = uint32_t(ud.size());
            if (int(ps.kb) > maxkb) {
                ps.fallback = true;
                b->passes.push_back(ps);
                continue;
            }
            // pad the union to the kernel's dimension count: repeat the last
            // dimension with (-inf, +inf) bounds (never rejects a stored tuple)
            const uint32_t kbp = col_batch_padded_dims(std::max<uint32_t>(ps.kb, 1));
            if (ud.empty()) ud.push_back(0);
            while (ud.size() < kbp) ud.push_back(ud.back());
            ps.kb = kbp;
            ps.udim_off = b->udims.size();
            ps.bound_off = b->bounds.size();
            ps.cmask_off = b->cmask.size();
            b->udims.insert(b->udims.end(), ud.begin(), ud.end());
            for (uint32_t q = q0; q < q0 + ps.nqp; ++q) {
                std::vector<float2> row(ps.kb, make_float2(-INFINITY, INFINITY));
                unsigned long long cm = 0;
                for (uint32_t i = 0; i < b->descs[q].k; ++i) {
                    const DimPred& p = b->preds[b->descs[q].off + i];
                    const int u = uidx[p.dim];
                    row[u] = make_float2(p.lo, p.hi);
                    cm |= 1ull << u;
                }
                b->bounds.insert(b->bounds.end(), row.begin(), row.end());
                b->cmask.push_back(cm);
            }
            b->passes.push_back(ps);
        }
    }
    if (path == MDRQ_PATH_VAFILE_BATCH) build_vb_passes(s, b);
}

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
    d.reserve(h.size());
    if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

void upload_batch(mdrq_store* s, mdrq_batch* b, bool sync = true) {
    upload(b->d_descs, b->descs, s->stream);
    upload(b->d_preds, b->preds, s->stream);
    upload(b->d_udims, b->udims, s->stream);
    upload(b->d_bounds, b->bounds, s->stream);
    upload(b->d_cmask, b->cmask, s->stream);
    upload(b->d_vb_udims, b->vb_udims, s->stream);
    upload(b->d_vb_tables, b->vb_tables, s->stream);
    upload(b->d_vb_qb, b->vb_qb, s->stream);
    upload(b->d_vb_cm, b->vb_cm, s->stream);
    upload(b->d_vb_q16, b->vb_q16, s->stream);
    upload(b->d_vb_perm, b->vb_perm, s->stream);
    const size_t nq = b->nq;
    b->d_scratch.reserve(scratch_words(b->nq));
    unsigned long long* p = b->d_scratch.p;
    b->d_counts.p = p;
    b->d_offsets.p = p + nq;
    b->d_stats.p = p + 2 * nq + 1;
    b->d_partials.p = p + 6 * nq + 1;
    b->d_tile_counters.p = reinterpret_cast<uint32_t*>(p + 6 * nq + 1 + nq * kPartialSlots * 4);
    b->d_counts_p.p = p + scratch_words_base(nq);
    b->d_offsets_p.p = p + scratch_words_base(nq) + nq;
    // H2D copies above may read pageable host vectors that a later rebuild
    // mutates: make them complete before returning (the ids stream rebuilds
    // a slot only after its previous pass and copies completed).
    if (sync) CK(cudaStreamSynchronize(s->stream));
}

uint64_t upload_bytes(const mdrq_batch* b) {
    return b->descs.size() * sizeof(QueryDesc) + b->preds.size() * sizeof(DimPred) +
           b->udims.size() * sizeof(uint16_t) + b->bounds.size() * sizeof(float2) +
           b->cmask.size() * sizeof(unsigned long long) + b->vb_udims.size() * sizeof(uint16_t) +
           b->vb_tables.size() * sizeof(uint32_t) + b->vb_qb.size() * sizeof(float2) +
           b->vb_cm.size() * sizeof(uint32_t) + b->vb_perm.size() * sizeof(uint32_t) +
           b->vb_q16.size() * sizeof(uint32_t);
}

uint32_t resolve_path(const mdrq_store* s, uint32_t path, uint32_t nq, bool ids, const float* lower = nullptr,
                      const float* upper = nullptr) {
    if (path == MDRQ_PATH_AUTO) {
        // planner.  A bit-sliced VA pass reads a table
        // row per tuple and UNION dimension whatever the number of queries,
        // a single-query VA scan a code per tuple and dimension of ITS query:
        // on the B200 (tools/probe_planner.py, C2-C5) a row costs ~10x a
        // code for unions of <= 16 dims (8.3 on C2 / C3 / C4, 12.4 on C5)
        // and ~30x for the wider unions' (overlap, containment) rows, so the
        // pass wins once  sum of the queries' dims >= 10 (30) x union dims:
        // 10 full-match queries, ~25 of C3's (5 of 16 dims), ~130 of C4's
        // when their union reaches 19 dims.
        const bool va = (s->layouts & MDRQ_LAYOUT_VAFILE) != 0;
        if (!(s->layouts & MDRQ_LAYOUT_COLUMNAR)) return MDRQ_PATH_ROWWISE;
        if (va && nq >= 10) {
            if (!lower || !upper || nq >= 1024) return MDRQ_PATH_VAFILE_BATCH;
            uint64_t sum_k = 0;
            std::vector<uint8_t> used(s->m, 0);
            for (uint32_t q = 0; q < nq; ++q)
                for (uint32_t j = 0; j < s->m; ++j) {
                    const float l = lower[uint64_t(q) * s->m + j], h = upper[uint64_t(q) * s->m + j];
                    if (!(is_neg_inf(l) && is_pos_inf(h))) {
                        ++sum_k;
                        used[j] = 1;
                    }
                }
            uint64_t kb = 0;
            for (uint32_t j = 0; j < s->m; ++j) kb += used[j];
            const uint64_t row_cost = kb <= kVbPvDims ? 10 : 30;
            if (sum_k >= row_cost * kb) return MDRQ_PATH_VAFILE_BATCH;
            return MDRQ_PATH_VAFILE;
        }
        if (va) return MDRQ_PATH_VAFILE;
        // multi-query columnar pass (<= 32 queries per read of the union's
        // columns): counts from 2 queries, ids from 4 (its masks + expansion
        // cost about one single-query scan)
        if (nq >= (ids ? 4u : 2u)) return MDRQ_PATH_COLUMNAR_BATCH;
        return MDRQ_PATH_COLUMNAR;
    }
    switch (path) {
        case MDRQ_PATH_COLUMNAR:
        case MDRQ_PATH_COLUMNAR_BATCH:
            if (!(s->layouts & MDRQ_LAYOUT_COLUMNAR)) raise(MDRQ_EINVAL, "store has no columnar layout");
            return path;
        case MDRQ_PATH_ROWWISE:
            if (!(s->layouts & MDRQ_LAYOUT_ROWWISE)) raise(MDRQ_EINVAL, "store has no row-wise layout");
            return path;
        case MDRQ_PATH_VAFILE:
        case MDRQ_PATH_VAFILE_BATCH:
            if (!(s->layouts & MDRQ_LAYOUT_VAFILE)) raise(MDRQ_EINVAL, "store has no VA-file layout");
            return path;
        default: raise(MDRQ_EINVAL, "unknown query path " + std::to_string(path));
    }
}

// the result pool a batch writes: its own (stream slots) or the store's
DBuf<uint32_t>& pool_of(mdrq_store* s, mdrq_batch* b) {
    return b->own_pool ? b->own_ids : b->shared_pool ? s->ids_alt : s->ids;
}

ScanArgs base_args(mdrq_store* s, mdrq_batch* b, uint32_t path) {
    ScanArgs a{};
    a.cols = s->cols.p;
    a.rows = s->rows.p;
    a.codes = s->codes.p;
    a.stride = s->n_pad;
    a.n = s->n;
    a.m = s->m;
    a.rows_per_tile = s->R;
    a.descs = b->d_descs.p;
    a.preds = b->d_preds.p;
    a.num_tiles = s->tiles_for(path);
    a.tile_counters = b->d_tile_counters.p;
    a.status = s->status.p;
    a.counts = b->d_counts.p;
    a.offsets = b->d_offsets.p;
    a.ids = pool_of(s, b).p;
    a.ids_cap = pool_of(s, b).p ? pool_of(s, b).cap : 0;
    a.id_base = s->id_base;
    a.stats = b->d_stats.p;
    a.mask = s->mask.p;
    a.chunk_counts = s->chunk_counts.p;
    a.chunk_offs = s->chunk_offs.p;
    a.partials = b->d_partials.p;
    return a;
}

VaBatchArgs vb_args(mdrq_store* s, mdrq_batch* b, const VbPass& ps) {
    VaBatchArgs a{};
    a.codes = s->codes.p;
    a.cols = s->cols.p;
    a.stride = s->n_pad;
    a.n = s->n;
    a.kb = ps.kb;
    a.cells = ps.cells;
    a.shift = ps.shift;
    a.nqp = ps.nqp;
    // lanes per tuple (vabatch.cu); build_vb_passes replicates the words
    a.lw = va_batch_pv(ps.kb) ? (ps.nqp <= 256 ? 8u : ps.nqp <= 512 ? 16u : 32u) : 32u;
    a.udims = b->d_vb_udims.p + ps.udim_off;
    a.tables = b->d_vb_tables.p + ps.table_off;
    a.qbounds = b->d_vb_qb.p + ps.qb_off;
    a.qcmask = b->d_vb_cm.p + ps.cm_off;
    a.qb16 = b->d_vb_q16.p ? b->d_vb_q16.p + ps.q16_off : nullptr;
    for (uint32_t u = 0; u < kVbStageDims; ++u) {
        a.vmin[u] = ps.vmin[u];
        a.vscale[u] = ps.vscale[u];
    }
    // one CTA per SM (the tables take most of the shared memory); chunks of
    // < 65536 tuples (16-bit per-warp counters), identical in every mode
    a.grid = uint32_t(s->num_sms);
    const uint64_t warps = uint64_t(a.grid) * va_batch_warps();
    // k groups per CTA with k the smallest that keeps a subchunk under the
    // 16-bit counter limit: the groups divide evenly over the CTAs (C5 on
    // one GPU: 4 groups of 52 864-tuple subchunks per CTA; capping the
    // subchunk at 65 408 tuples instead gave 478 groups over 148 CTAs, i.e.
    // 4 rounds for some SMs and 3 for others, ~20 % of the SMs idle)
    const uint64_t per_warp = (s->n + warps - 1) / warps;
    const uint64_t k = std::max<uint64_t>(1, (per_warp + 65407) / 65408);
    a.chunk_tuples = std::min<uint64_t>(65408, round_up((s->n + warps * k - 1) / (warps * k), 128));
    a.nchunks = uint32_t((s->n + a.chunk_tuples - 1) / a.chunk_tuples);
    a.ngroups = (a.nchunks + va_batch_warps() - 1) / va_batch_warps();
    const uint64_t chunks = a.nchunks;
    s->vb_chunk_counts.reserve(chunks * 1024);
    s->vb_base.reserve(chunks * 1024);
    s->vb_total.reserve(1024);
    s->vb_qoff.reserve(1024);
    // sorted batch: the passes write in slot order (unpermuted by enqueue)
    const bool sorted = !b->vb_perm.empty();
    a.counts = (sorted ? b->d_counts_p.p : b->d_counts.p) + ps.q0;
    a.chunk_counts = s->vb_chunk_counts.p;
    a.base = s->vb_base.p;
    a.total = s->vb_total.p;
    a.qoff = s->vb_qoff.p;
    a.offsets = sorted ? b->d_offsets_p.p : b->d_offsets.p;
    a.counts_all = sorted ? b->d_counts_p.p : b->d_counts.p;
    DBuf<uint32_t>& dst = sorted ? s->vb_ids_slot : pool_of(s, b);
    a.ids = dst.p;
    a.ids_cap = dst.p ? dst.cap - (sorted ? std::min<size_t>(dst.cap, 4) : 0) : 0;
    a.id_base = s->id_base;
    a.prune_dims = ps.prune;
    for (uint32_t u = 0; u < ps.kb && u < uint32_t(kVaBatchMaxDims); ++u) a.cellmask[u] = ps.cellmask[u];
    s->vb_rec.reserve(size_t(s->vb_max_blocks) * kRecBlock);
    s->vb_blk_count.reserve(s->vb_max_blocks);
    s->vb_blk_chunk.reserve(s->vb_max_blocks);
    s->vb_blk_seq.reserve(s->vb_max_blocks);
    s->vb_blk_list.reserve(s->vb_max_blocks);
    s->vb_chunk_nblk.reserve(chunks);
    s->vb_chunk_first.reserve(chunks);
    s->vb_flags.reserve(3);
    a.rec = s->vb_rec.p;
    a.blk_count = s->vb_blk_count.p;
    a.blk_chunk = s->vb_blk_chunk.p;
    a.blk_seq = s->vb_blk_seq.p;
    a.blk_list = s->vb_blk_list.p;
    a.chunk_nblk = s->vb_chunk_nblk.p;
    a.chunk_first = s->vb_chunk_first.p;
    a.cursor = s->vb_flags.p;
    a.overflow = s->vb_flags.p + 1;
    a.max_blocks = s->vb_max_blocks;
    // test hook: cap the staging pool so small batches take the recount path
    static const char* cap = getenv("MDRQ_VB_STAGING_BLOCKS");
    if (cap) a.max_blocks = std::min<uint32_t>(a.max_blocks, uint32_t(strtoul(cap, nullptr, 10)));
    return a;
}

// Enqueue one count / ids pass of a prepared batch.  Returns kernel launches.
// Optional per-stage timing of one pass (mdrq_batch_profile): an event is
// recorded before every launch group; the time to the next mark is charged
// to the group's class (0 scan / filter, 1 compaction, 2 id write, 3 setup).
struct Profiler {
    cudaStream_t st = nullptr;
    bool counting = true;            // first run only counts the marks
    size_t used = 0;
    std::vector<cudaEvent_t> ev;     // created up front: no API cost between launches
    std::vector<int> cls;
    uint32_t launches[4] = {0, 0, 0, 0};
    void mark(int c, uint32_t nlaunch) {
        if (counting) {
            ++used;
            return;
        }
        if (used >= ev.size()) raise(MDRQ_ECUDA, "profiler event pool exhausted");
        CK(cudaEventRecord(ev[used], st));
        cls.push_back(c);
        ++used;
        if (c >= 0 && c < 4) launches[c] += nlaunch;
    }
    void arm() {
        ev.resize(used + 1);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        counting = false;
        used = 0;
    }
    ~Profiler() {
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
    }
};

uint32_t enqueue_impl(mdrq_store* s, mdrq_batch* b, bool ids, cudaStream_t st, Profiler* prof);

// order work on `st` after the store's last pass (which may have run on a
// caller's stream)
void join(mdrq_store* s, cudaStream_t st) {
    if (s->done && s->done_stream && s->done_stream != st) CK(cudaStreamWaitEvent(st, s->done, 0));
}

// Every pass goes through here: it orders the pass after the last pass the
// store ran on another stream (shared scratch and result pool), and marks
// its own end for the next one.
uint32_t enqueue(mdrq_store* s, mdrq_batch* b, bool ids, cudaStream_t st, Profiler* prof = nullptr) {
    if (!s->done) CK(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
    if (s->done_stream && s->done_stream != st) CK(cudaStreamWaitEvent(st, s->done, 0));
    const uint32_t nl = enqueue_impl(s, b, ids, st, prof);
    CK(cudaEventRecord(s->done, st));
    s->done_stream = st;
    return nl;
}

uint32_t enqueue_impl(mdrq_store* s, mdrq_batch* b, bool ids, cudaStream_t st, Profiler* prof) {
    const uint32_t nq = b->nq;
    if (!nq) return 0;
    auto mark = [&](int c, uint32_t nl) {
        if (prof) prof->mark(c, nl);
    };
    mark(3, 0);
    CK(cudaMemsetAsync(b->d_scratch.p, 0, sizeof(unsigned long long) * scratch_words(nq), st));
    if (s->n == 0) return 0;
    uint32_t launches = 0;
    bool used_partials = false;   // single-query column / VA kernels accumulate into partials
    const uint32_t path = b->path;
    auto single = [&](uint32_t sp, uint32_t q) {
        ScanArgs a = base_args(s, b, sp);
        a.q = q;
        if (sp == MDRQ_PATH_VAFILE) {
            // expected fraction of tuples alive after the code test (cells
            // independent): above ~3e-3 the refinement of every alive tuple
            // costs more than a second range test per code
            double sel = 1.0;
            const double cells = double(s->nb() + 1);
            for (uint32_t i = 0; i < b->descs[q].k; ++i) {
                const DimPred& p = b->preds[b->descs[q].off + i];
                sel *= p.ch >= p.cl ? double(p.ch - p.cl + 1) / cells : 0.0;
            }
            a.va_sure = sel > 3e-3 ? 1u : 0u;
        }
        a.epoch = s->next_epoch();
        if (ids) {
            mark(1, 0);
            CK(cudaMemsetAsync(s->chunk_counts.p, 0, sizeof(uint32_t) * s->nchunks, st));
        }
        mark(0, 1);
        if (sp == MDRQ_PATH_ROWWISE) {
            launch_row_scan(a, ids, st);
        } else if (sp == MDRQ_PATH_VAFILE) {
            launch_va_scan(a, ids, st);
            used_partials = true;
        } else {
            launch_col_scan(a, ids, st);
            used_partials = true;
        }
        ++launches;
        if (ids) {
            mark(1, 2);
            launch_expand(a, st);
            launches += 2;
        }
    };
    if (path == MDRQ_PATH_VAFILE_BATCH) {
        if (ids) {
            s->vb_flags.reserve(3);
            CK(cudaMemsetAsync(s->vb_flags.p + 2, 0, sizeof(uint32_t), st));
        }
        const bool sorted = !b->vb_perm.empty();
        DBuf<uint32_t>& pool = pool_of(s, b);
        // slot-order ids, as large as the result pool (+ 4 words of slack
        // for the realigning copy's reads)
        if (sorted && ids && pool.p) s->vb_ids_slot.reserve(pool.cap + 4);
        for (const VbPass& ps : b->vb_passes) {
            if (ps.fallback) {
                for (uint32_t q = ps.q0; q < ps.q0 + ps.nqp; ++q) single(MDRQ_PATH_VAFILE, q);
                continue;
            }
            VaBatchArgs va = vb_args(s, b, ps);
            if (!ids) {
                mark(0, 1);
                launch_va_batch(va, 0, st);
                launches += 1;
            } else {
                // single pass: filter + per-chunk counts + staged records,
                // scans, block list, scatter; the recount pass (mode 2) only
                // works when the staging pool overflowed (it checks the flag
                // on device)
                mark(3, 0);
                CK(cudaMemsetAsync(va.cursor, 0, 2 * sizeof(uint32_t), st));
                static const bool dbg = getenv("MDRQ_DEBUG_SYNC") != nullptr;
                auto dsync = [&](const char* what) {
                    if (dbg) ck(cudaStreamSynchronize(st), what);
                };
                mark(0, 1);
                launch_va_batch(va, 3, st);
                dsync("mode3");
                static const bool vdbg = getenv("MDRQ_DEBUG_VB") != nullptr;
                if (vdbg) {
                    uint32_t fl[2] = {0, 0};
                    CK(cudaMemcpyAsync(fl, va.cursor, sizeof(fl), cudaMemcpyDeviceToHost, st));
                    CK(cudaStreamSynchronize(st));
                    fprintf(stderr, "vb pass q0=%u nqp=%u kb=%u: staged blocks %u of %u, overflow %u\n", ps.q0, ps.nqp,
                            ps.kb, fl[0], va.max_blocks, fl[1]);
                }
                mark(1, 3);
                launch_va_batch_scans(va, ps.q0, st);
                dsync("scans");
                launch_va_batch_block_list(va, st);
                dsync("list");
                mark(2, 2);
                launch_va_batch_scatter(va, st);
                dsync("scatter");
                launch_va_batch(va, 2, st);
                dsync("mode2");
                launches += 6;
            }
        }
        if (sorted) {
            mark(ids ? 2 : 1, ids ? 3 : 2);
            launches += launch_va_batch_unpermute(b->d_vb_perm.p, b->d_counts_p.p, b->d_offsets_p.p, b->d_counts.p,
                                                  b->d_offsets.p, s->vb_ids_slot.p,
                                                  s->vb_ids_slot.cap > 4 ? s->vb_ids_slot.cap - 4 : 0, pool.p,
                                                  pool.p ? pool.cap : 0, nq,
                                                  ids && pool.p && s->vb_ids_slot.p && b->packed_to < nq, b->packed_to,
                                                  st);
        }
    } else if (path == MDRQ_PATH_COLUMNAR_BATCH) {
        // ids: query-major masks (word count a multiple of 4: 16-byte rows)
        const uint64_t mask_words = round_up(s->n_pad / 32, 4);
        const uint32_t nch = uint32_t((s->n + kChunkTuples - 1) / kChunkTuples);
        if (ids) {
            s->bmask.reserve(32 * mask_words);
            s->bchunk_counts.reserve(size_t(32) * nch);
            s->bchunk_offs.reserve(size_t(32) * nch);
        }
        for (const Pass& ps : b->passes) {
            if (ps.fallback) {
                for (uint32_t q = ps.q0; q < ps.q0 + ps.nqp; ++q) single(MDRQ_PATH_COLUMNAR, q);
                continue;
            }
            BatchArgs ba{};
            ba.cols = s->cols.p;
            ba.stride = s->n_pad;
            ba.n = s->n;
            ba.kb = ps.kb;
            ba.nqp = ps.nqp;
            ba.udims = b->d_udims.p + ps.udim_off;
            ba.bounds = b->d_bounds.p + ps.bound_off;
            ba.cmask = b->d_cmask.p + ps.cmask_off;
            ba.counts = b->d_counts.p + ps.q0;
            mark(0, 1);
            if (!ids) {
                launch_col_batch_count(ba, s->num_sms, st);
                ++launches;
                continue;
            }
            launch_col_batch_ids(ba, s->bmask.p, mask_words, s->bchunk_counts.p, s->num_sms, st);
            mark(1, 3);
            launch_expand_pass(base_args(s, b, MDRQ_PATH_COLUMNAR), ps.q0, ps.nqp, s->bmask.p, mask_words,
                               s->bchunk_counts.p, s->bchunk_offs.p, st);
            launches += 4;
        }
    } else {
        const uint32_t sp = path == MDRQ_PATH_COLUMNAR_BATCH ? MDRQ_PATH_COLUMNAR : path;
        for (uint32_t q = 0; q < nq; ++q) single(sp, q);
    }
    if (used_partials) {
        mark(3, 1);
        launch_reduce_partials(b->d_partials.p, nq, !ids, b->d_counts.p, b->d_stats.p, st);
        ++launches;
    }
    CK(cudaGetLastError());
    return launches;
}

uint32_t count_launches(const mdrq_store* s, const mdrq_batch* b, bool ids) {
    if (!b->nq || s->n == 0) return 0;
    // mirrors enqueue(): + 1 partial-reduction launch whenever a single-query
    // column / VA scan ran (it is not launched for row-wise scans)
    if (b->path == MDRQ_PATH_VAFILE_BATCH) {
        uint32_t l = 0;
        bool single = false;
        for (const VbPass& ps : b->vb_passes) {
            l += ps.fallback ? ps.nqp * (ids ? 3 : 1) : (ids ? 6 : 1);
            single |= ps.fallback;
        }
        if (!b->vb_perm.empty()) l += ids ? 3 : 2;
        return l + (single ? 1 : 0);
    }
    if (b->path == MDRQ_PATH_COLUMNAR_BATCH) {
        uint32_t l = 0;
        bool single = false;
        for (const Pass& ps : b->passes) {
            l += ps.fallback ? ps.nqp * (ids ? 3 : 1) : (ids ? 4 : 1);
            single |= ps.fallback;
        }
        return l + (single ? 1 : 0);
    }
    const uint32_t per_query = ids ? 3 : 1;   // ids: scan + chunk scan + expand
    return per_query * b->nq + (b->path == MDRQ_PATH_ROWWISE ? 0 : 1);
}

// Run an ids pass synchronously, growing the result pool until it fits.
// The single-pass VA staging ran out (the recount pass kept the result
// correct): size the pool for the pass's `total` records (one per match,
// + ~10 % for partly filled blocks, + one partial block per subchunk), at
// least twice the current pool, within 2^24 blocks (64 GB) and what the
// device has free beyond a 2 GB reserve.
void grow_vb_staging(mdrq_store* s, uint64_t total) {
    constexpr uint64_t kMaxBlocks = 1ull << 24;
    const uint64_t per_block = uint64_t(kRecBlock) * 4 + 4 * sizeof(uint32_t);
    // blocks close when a refinement round's records do not fit: dense passes
    // fill them to ~85-90 % (C2 1e-1: 5e9 records took 5.38 M blocks)
    uint64_t want = std::max<uint64_t>(2ull * s->vb_max_blocks,
                                       total / kRecBlock + total / (4 * kRecBlock) + 2ull * 16 * s->num_sms + 64);
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        // the current pool is released first, so its bytes count as free
        const uint64_t avail = free_b + uint64_t(s->vb_max_blocks) * per_block;
        const uint64_t reserve = 2ull << 30;
        want = std::min<uint64_t>(want, avail > reserve ? (avail - reserve) / per_block : 0);
    }
    want = std::min<uint64_t>(want, kMaxBlocks);
    if (want <= s->vb_max_blocks) return;
    s->vb_max_blocks = uint32_t(want);
    s->vb_rec.release();
    s->vb_blk_count.release();
    s->vb_blk_chunk.release();
    s->vb_blk_seq.release();
    s->vb_blk_list.release();
}

// The first bit-sliced ids batch of a store: count it first and size the
// staging pool from its total, so the batch does not overflow the default pool
// and take the recount pass (~6x a filter pass) on every overflowing pass.
void presize_vb_staging(mdrq_store* s, mdrq_batch* b) {
    if (s->vb_sized || b->path != MDRQ_PATH_VAFILE_BATCH || !b->nq || !s->n) return;
    enqueue(s, b, false, s->stream);
    std::vector<unsigned long long> c(b->nq);
    CK(cudaMemcpyAsync(c.data(), b->d_counts.p, sizeof(unsigned long long) * b->nq, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    uint64_t total = 0;
    for (unsigned long long v : c) total += v;
    if (total > uint64_t(s->vb_max_blocks) * kRecBlock / 2) grow_vb_staging(s, total);
    s->vb_sized = true;
}

uint64_t run_ids_sync(mdrq_store* s, mdrq_batch* b) {
    s->bounce_ids = 0;
    presize_vb_staging(s, b);
    // until the result pool holds the batch AND no pass overflowed the
    // staging pool (a reserved batch then never runs the recount pass)
    for (int attempt = 0; attempt < 4; ++attempt) {
        enqueue(s, b, true, s->stream);
        unsigned long long total = 0;
        if (b->nq && s->n)
            CK(cudaMemcpyAsync(&total, b->d_offsets.p + b->nq, sizeof(total), cudaMemcpyDeviceToHost, s->stream));
        uint32_t overflowed = 0;
        if (b->path == MDRQ_PATH_VAFILE_BATCH && s->vb_flags.p)
            CK(cudaMemcpyAsync(&overflowed, s->vb_flags.p + 2, sizeof(overflowed), cudaMemcpyDeviceToHost,
                               s->stream));
        CK(cudaStreamSynchronize(s->stream));
        if (overflowed) grow_vb_staging(s, total);
        DBuf<uint32_t>& pool = pool_of(s, b);
        if (total <= (pool.p ? pool.cap : 0) && (!overflowed || attempt == 3)) {
            s->last_total = total;
            s->last_nq = b->nq;
            s->last_path = b->path;
            s->last_batch = b;
            return total;
        }
        if (total > (pool.p ? pool.cap : 0)) pool.reserve(size_t(total + total / 8 + 4096));
    }
    raise(MDRQ_ECUDA, "result pool did not converge");
}

void check_store(const mdrq_store* s);

constexpr size_t kBounceMaxBytes = size_t(64) << 20;

uint8_t* bounce(mdrq_store* s, size_t bytes) {
    if (bytes > s->h_bounce_cap) {
        if (s->h_bounce) {
            cudaFreeHost(s->h_bounce);
            s->h_bounce = nullptr;
            s->h_bounce_cap = 0;
        }
        const size_t cap = (std::max<size_t>(bytes, size_t(1) << 20) + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
        CK(cudaMallocHost(reinterpret_cast<void**>(&s->h_bounce), cap));
        s->h_bounce_cap = cap;
    }
    return s->h_bounce;
}

// total ids from src (host) to the caller's buffer: as uint32, or widened to
// int64 (src may be the upper half of that int64 buffer: front-to-back
// widening never overwrites a source word before it is read)
void deliver_ids(const uint32_t* src, void* ids, uint64_t total, bool wide) {
    if (wide) {
        int64_t* o = static_cast<int64_t*>(ids);
        for (uint64_t i = 0; i < total; ++i) o[i] = int64_t(src[i]);
    } else if (src != ids) {
        std::memcpy(ids, src, sizeof(uint32_t) * total);
    }
}

// the cached result of the last ids call into the caller's buffer
void fetch_ids_impl(mdrq_store* s, void* ids, uint64_t ids_cap, bool wide) {
    if (s->last_total > ids_cap) raise(MDRQ_ETRUNC, "ids buffer too small");
    const uint64_t total = s->last_total;
    if (!total) return;
    if (!ids) raise(MDRQ_EINVAL, "null ids");
    if (s->bounce_ids >= total) {
        deliver_ids(reinterpret_cast<const uint32_t*>(s->h_bounce + s->bounce_head), ids, total, wide);
        return;
    }
    uint32_t* dst = wide ? static_cast<uint32_t*>(ids) + total : static_cast<uint32_t*>(ids);
    join(s, s->stream);
    CK(cudaMemcpyAsync(dst, s->ids.p, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    deliver_ids(dst, ids, total, wide);
}

// Synchronous ids call (mdrq_query_ids / mdrq_query_ids64): one pass, then
// offsets + overflow flag + a speculative prefix of the ids (the previous
// call's total + 25 %, >= 64 K ids) in one pinned copy and one
// synchronisation; the remainder, if any, in a second copy.
int query_ids_impl(mdrq_store* s, const float* lower, const float* upper, uint32_t nq, uint32_t path,
                   uint64_t* offsets, void* ids, bool wide, uint64_t ids_cap, uint64_t* total_out) {
    int trunc = 0;
    int rc = guard([&] {
        check_store(s);
        if (!offsets || !total_out) raise(MDRQ_EINVAL, "null argument");
        if (nq && (!lower || !upper)) raise(MDRQ_EINVAL, "null bounds");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        mdrq_batch* b = &s->scratch;
        b->owner = s;
        static const bool tdbg = getenv("MDRQ_DEBUG_TIMING") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        const auto t0 = now();
        build_descs(s, lower, upper, nq, resolve_path(s, path, nq, true, lower, upper), true, b);
        const auto t1 = now();
        // no synchronisation here: this call synchronises before it returns,
        // so the host descriptors stay untouched until their copies are done
        upload_batch(s, b, false);
        const auto t2 = now();
        s->bounce_ids = 0;
        const bool have = nq && s->n;
        const size_t head = (size_t(nq) + 1) * 8 + 8;
        if (head > kBounceMaxBytes) raise(MDRQ_EINVAL, "too many queries in one call");
        uint64_t total = 0, spec = 0;
        uint8_t* hb = nullptr;
        presize_vb_staging(s, b);
        for (int attempt = 0;; ++attempt) {
            if (attempt == 2) raise(MDRQ_ECUDA, "result pool did not converge");
            enqueue(s, b, true, s->stream);
            DBuf<uint32_t>& pool = pool_of(s, b);
            const uint64_t pcap = pool.p ? pool.cap : 0;
            // a speculative prefix only when the expected result fits the
            // bounce buffer: a larger one goes to the caller in ONE copy
            // (a prefix would be copied twice)
            const uint64_t want = std::max<uint64_t>(uint64_t(1) << 16, s->last_total + s->last_total / 4);
            spec = have && want <= (kBounceMaxBytes - head) / 4 ? std::min<uint64_t>(pcap, want) : 0;
            hb = bounce(s, head + spec * 4);
            uint64_t* h_off = reinterpret_cast<uint64_t*>(hb);
            uint32_t* h_flag = reinterpret_cast<uint32_t*>(hb + (size_t(nq) + 1) * 8);
            *h_flag = 0;
            const bool vb = b->path == MDRQ_PATH_VAFILE_BATCH && s->vb_flags.p;
            if (have)
                CK(cudaMemcpyAsync(h_off, b->d_offsets.p, sizeof(uint64_t) * (nq + 1), cudaMemcpyDeviceToHost,
                                   s->stream));
            if (vb) CK(cudaMemcpyAsync(h_flag, s->vb_flags.p + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream));
            if (spec) CK(cudaMemcpyAsync(hb + head, pool.p, sizeof(uint32_t) * spec, cudaMemcpyDeviceToHost, s->stream));
            CK(cudaStreamSynchronize(s->stream));
            total = have ? h_off[nq] : 0;
            if (vb && *h_flag) grow_vb_staging(s, total);   // the recount pass kept this result correct
            if (total <= pcap) break;
            pool.reserve(size_t(total + total / 8 + 4096));
        }
        const auto t3 = now();
        s->last_total = total;
        s->last_nq = nq;
        s->last_path = b->path;
        s->last_batch = b;
        s->bounce_ids = spec >= total ? spec : 0;
        s->bounce_head = head;
        *total_out = total;
        if (have)
            std::memcpy(offsets, hb, sizeof(uint64_t) * (size_t(nq) + 1));
        else
            std::memset(offsets, 0, sizeof(uint64_t) * (size_t(nq) + 1));
        if (total > ids_cap) {
            trunc = 1;
        } else {
            fetch_ids_impl(s, ids, ids_cap, wide);
        }
        if (tdbg) {
            const auto t4 = now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            fprintf(stderr, "query_ids: prepare %.3f upload %.3f run %.3f copy %.3f ms\n", ms(t0, t1), ms(t1, t2),
                    ms(t2, t3), ms(t3, t4));
        }
    });
    if (rc == MDRQ_OK && trunc) {
        g_err = "ids buffer too small";
        return MDRQ_ETRUNC;
    }
    return rc;
}

void check_store(const mdrq_store* s) {
    if (!s) raise(MDRQ_EINVAL, "null store");
}

}  // namespace

// ==================================================================== C ABI ==
extern "C" {

const char* mdrq_last_error(void) { return g_err.c_str(); }

int mdrq_abi_version(void) { return MDRQ_ABI_VERSION; }

int mdrq_check_flags(uint32_t* flags) {
    return guard([&] {
        if (!flags) raise(MDRQ_EINVAL, "null flags");
        CK(cudaDeviceSynchronize());
        *flags = vabatch_check_flags() | columnar_check_flags() | expand_check_flags();
#ifdef MDRQ_CHECKS
        *flags |= 0x80000000u;   // this library was built with the checks
#endif
    });
}

int mdrq_copy_segments(const uint32_t* src, uint32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                       const int64_t* len, uint64_t nseg, void* stream) {
    return guard([&] {
        if (nseg && (!src || !dst || !src_off || !dst_off || !len)) raise(MDRQ_EINVAL, "null argument");
        launch_copy_segments(src, dst, src_off, dst_off, len, nseg, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrq_copy_segments_dma(const uint32_t* src, uint32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                           const int64_t* len, uint64_t nseg, void* stream) {
    return guard([&] {
        if (nseg && (!src || !dst || !src_off || !dst_off || !len)) raise(MDRQ_EINVAL, "null argument");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!st) raise(MDRQ_EINVAL, "a non-default stream is required");
        // one asynchronous copy per segment (the copy engines; a segment is a
        // query's run of this rank's ids, ~1e4 per batch, ~2 us each to issue)
        for (uint64_t i = 0; i < nseg; ++i) {
            if (len[i] <= 0) continue;
            CK(cudaMemcpyAsync(dst + dst_off[i], src + src_off[i], size_t(len[i]) * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, st));
        }
    });
}

int mdrq_measure_read_bw(int device, uint64_t bytes, int iters, double* gbs) {
    return guard([&] {
        if (!gbs || bytes < 16 || iters < 1) raise(MDRQ_EINVAL, "bad argument");
        DeviceGuard dg(device);
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        bytes &= ~uint64_t(15);
        DBuf<uint8_t> buf;
        DBuf<uint32_t> sink;
        buf.reserve(bytes);
        sink.reserve(1);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CK(cudaMemsetAsync(buf.p, 1, bytes, st));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int i = 0; i < iters + 1; ++i) {   // first launch warms up
            CK(cudaEventRecord(e0, st));
            launch_read_stream(buf.p, bytes, sink.p, sms, st);
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (i) best = std::min(best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        *gbs = double(bytes) / (double(best) * 1e-3) / 1e9;
    });
}

int mdrq_device_count(int* count) {
    return guard([&] {
        if (!count) raise(MDRQ_EINVAL, "null count");
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

int mdrq_store_create(const float* rows, uint64_t n, uint32_t m, int device, uint32_t layouts, uint32_t va_bits,
                      uint64_t id_base, mdrq_store** out) {
    return guard([&] {
        if (!out) raise(MDRQ_EINVAL, "null out");
        *out = nullptr;
        if (m < 1) raise(MDRQ_EINVAL, "dimensionality must be at least 1");
        if (m > uint32_t(kMaxDims)) raise(MDRQ_EINVAL, "at most 256 dimensions are supported on the GPU");
        if (n && !rows) raise(MDRQ_EINVAL, "null rows");
        if (n + id_base > 0xFFFFFFFFull) raise(MDRQ_EINVAL, "store ids must fit in uint32");
        if (layouts == 0) layouts = MDRQ_LAYOUT_COLUMNAR;
        if (layouts & ~7u) raise(MDRQ_EINVAL, "unknown layout bits");
        if (layouts & MDRQ_LAYOUT_VAFILE) {
            if (va_bits < 1 || va_bits > 8) raise(MDRQ_EINVAL, "va_bits must be in 1..8");
            layouts |= MDRQ_LAYOUT_COLUMNAR;  // exact refine reads the columns
        } else {
            va_bits = 0;
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            raise(MDRQ_ENODEV, "no CUDA device available");
        }
        if (device < 0 || device >= ndev) raise(MDRQ_ENODEV, "bad device ordinal " + std::to_string(device));
        DeviceGuard dg(device);
        auto* s = new mdrq_store();
        try {
            s->device = device;
            s->n = n;
            s->m = m;
            s->layouts = layouts;
            s->va_bits = va_bits;
            s->id_base = uint32_t(id_base);
            CK(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device));
            CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
            s->n_pad = round_up(std::max<uint64_t>(n, 1), kPadTuples);
            s->R = row_tile_rows(m);
            s->n_pad_rows = round_up(std::max<uint64_t>(n, 1), s->R);
            cudaStream_t st = s->stream;
            // stage rows on the device (kept as the row-wise layout if asked)
            s->rows.reserve(s->n_pad_rows * m);
            if (n) CK(cudaMemcpyAsync(s->rows.p, rows, n * m * sizeof(float), cudaMemcpyHostToDevice, st));
            launch_fill_f32(s->rows.p + n * m, (s->n_pad_rows - n) * m, NAN, st);
            if (layouts & MDRQ_LAYOUT_COLUMNAR) {
                s->cols.reserve(s->n_pad * m);
                for (uint32_t d = 0; d < m; ++d)
                    launch_fill_f32(s->cols.p + uint64_t(d) * s->n_pad + n, s->n_pad - n, NAN, st);
                launch_transpose_rows_to_cols(s->rows.p, n, m, s->cols.p, s->n_pad, st);
            }
            // observed bounds (core.py:99-105), used to order predicates
            {
                DBuf<float> mm;
                mm.reserve(size_t(2) * m);
                s->h_minmax.assign(size_t(2) * m, 0.f);
                if (n) {
                    // a row-wise-only store: one column at a time through a
                    // temporary transpose of the staged rows
                    DBuf<float> tmp;
                    if (!(layouts & MDRQ_LAYOUT_COLUMNAR)) {
                        tmp.reserve(s->n_pad * m);
                        launch_transpose_rows_to_cols(s->rows.p, n, m, tmp.p, s->n_pad, st);
                    }
                    const float* cols = (layouts & MDRQ_LAYOUT_COLUMNAR) ? s->cols.p : tmp.p;
                    for (uint32_t d = 0; d < m; ++d)
                        launch_min_max(cols + uint64_t(d) * s->n_pad, n, mm.p + 2 * d, st);
                    CK(cudaMemcpyAsync(s->h_minmax.data(), mm.p, sizeof(float) * 2 * m, cudaMemcpyDeviceToHost, st));
                    CK(cudaStreamSynchronize(st));
                }
                CK(cudaStreamSynchronize(st));
            }
            if (layouts & MDRQ_LAYOUT_VAFILE) {
                const uint32_t nb = s->nb();
                s->va_bounds.reserve(size_t(nb) * m);
                s->h_va_bounds.assign(size_t(nb) * m, 0.f);
                s->codes.reserve(s->n_pad * m);
                if (n) {
                    const uint64_t cnt = std::min<uint64_t>(n, 1ull << 20);
                    const uint64_t step = n / cnt;
                    DBuf<float> samp, sorted;
                    DBuf<unsigned char> temp;
                    samp.reserve(cnt);
                    sorted.reserve(cnt);
                    const size_t tb = va_sort_temp_bytes(cnt);
                    temp.reserve(tb);
                    for (uint32_t d = 0; d < m; ++d) {
                        const float* col = s->cols.p + uint64_t(d) * s->n_pad;
                        launch_va_sample(col, n, step, cnt, samp.p, st);
                        va_sort(samp.p, sorted.p, cnt, temp.p, tb, st);
                        launch_va_pick_boundaries(sorted.p, cnt, nb + 1, s->va_bounds.p + size_t(d) * nb, st);
                        launch_va_encode(col, s->n_pad, s->va_bounds.p + size_t(d) * nb, nb,
                                         s->codes.p + uint64_t(d) * s->n_pad, st);
                    }
                    CK(cudaMemcpyAsync(s->h_va_bounds.data(), s->va_bounds.p, sizeof(float) * nb * m,
                                       cudaMemcpyDeviceToHost, st));
                } else {
                    CK(cudaMemsetAsync(s->va_bounds.p, 0, sizeof(float) * nb * m, st));
                    CK(cudaMemsetAsync(s->codes.p, 0, s->n_pad * m, st));
                }
                CK(cudaStreamSynchronize(st));
            }
            if (!(layouts & MDRQ_LAYOUT_ROWWISE)) s->rows.release();
            {
                const uint64_t span = round_up(std::max(s->n_pad, s->n_pad_rows), kChunkTuples);
                s->nchunks = uint32_t(span / kChunkTuples);
                s->mask.reserve(span / 32);
                s->chunk_counts.reserve(s->nchunks);
                s->chunk_offs.reserve(s->nchunks);
            }
            uint64_t tiles = std::max<uint64_t>((n + kColTile - 1) / kColTile, (n + s->R - 1) / s->R);
            s->status.reserve(std::max<uint64_t>(tiles, 1));
            CK(cudaMemsetAsync(s->status.p, 0, s->status.bytes(), st));
            CK(cudaStreamSynchronize(st));
            CK(cudaGetLastError());
        } catch (...) {
            if (s->stream) cudaStreamDestroy(s->stream);
            delete s;
            throw;
        }
        *out = s;
    });
}

int mdrq_store_destroy(mdrq_store* s) {
    return guard([&] {
        if (!s) return;
        DeviceGuard dg(s->device);
        cudaStreamSynchronize(s->stream);
        if (s->done_stream) cudaStreamSynchronize(s->done_stream);
        {
            std::lock_guard<std::mutex> lk(s->mu);
            for (mdrq_batch* b : s->batches) {   // the caller still holds these handles
                b->release_device();
                b->owner = nullptr;
            }
            s->batches.clear();
        }
        cudaStream_t st = s->stream;
        delete s;
        cudaStreamDestroy(st);
    });
}

int mdrq_store_get_info(const mdrq_store* s, mdrq_store_info* info) {
    return guard([&] {
        check_store(s);
        if (!info) raise(MDRQ_EINVAL, "null info");
        info->n = s->n;
        info->m = s->m;
        info->layouts = s->layouts;
        info->va_bits = s->va_bits;
        info->device = s->device;
        info->n_pad = s->n_pad;
        info->device_bytes = s->cols.bytes() + s->rows.bytes() + s->codes.bytes() + s->va_bounds.bytes() +
                             s->status.bytes() + s->ids.bytes();
    });
}

int mdrq_store_va_boundaries(const mdrq_store* s, float* out) {
    return guard([&] {
        check_store(s);
        if (!s->va_bits) raise(MDRQ_EINVAL, "store has no VA-file layout");
        if (!out) raise(MDRQ_EINVAL, "null out");
        std::memcpy(out, s->h_va_bounds.data(), s->h_va_bounds.size() * sizeof(float));
    });
}

int mdrq_store_bounds(const mdrq_store* s, float* out) {
    return guard([&] {
        check_store(s);
        if (!out) raise(MDRQ_EINVAL, "null out");
        std::memcpy(out, s->h_minmax.data(), s->h_minmax.size() * sizeof(float));
    });
}

int mdrq_query_count(mdrq_store* s, const float* lower, const float* upper, uint32_t nq, uint32_t path,
                     uint64_t* counts) {
    return guard([&] {
        check_store(s);
        if (nq && (!lower || !upper || !counts)) raise(MDRQ_EINVAL, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        mdrq_batch* b = &s->scratch;
        b->owner = s;
        build_descs(s, lower, upper, nq, resolve_path(s, path, nq, false, lower, upper), true, b);
        upload_batch(s, b, false);   // synchronised below, before the descriptors change
        enqueue(s, b, false, s->stream);
        // counts through the pinned bounce buffer (the cached ids, if any,
        // stay on the device: mdrq_fetch_ids copies them from the pool)
        s->bounce_ids = 0;
        const size_t cb = sizeof(uint64_t) * nq;
        uint8_t* hb = nq && cb <= kBounceMaxBytes ? bounce(s, cb) : nullptr;
        if (nq) CK(cudaMemcpyAsync(hb ? static_cast<void*>(hb) : static_cast<void*>(counts), b->d_counts.p, cb,
                                   cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        if (hb) std::memcpy(counts, hb, cb);
        s->last_batch = b;
        s->last_nq = nq;
        s->last_path = b->path;
    });
}

int mdrq_query_ids(mdrq_store* s, const float* lower, const float* upper, uint32_t nq, uint32_t path,
                   uint64_t* offsets, uint32_t* ids, uint64_t ids_cap, uint64_t* total) {
    return query_ids_impl(s, lower, upper, nq, path, offsets, ids, false, ids_cap, total);
}

int mdrq_query_ids64(mdrq_store* s, const float* lower, const float* upper, uint32_t nq, uint32_t path,
                     uint64_t* offsets, int64_t* ids, uint64_t ids_cap, uint64_t* total) {
    return query_ids_impl(s, lower, upper, nq, path, offsets, ids, true, ids_cap, total);
}

int mdrq_query_ids_stream(mdrq_store* s, const float* lower, const float* upper, const uint32_t* nqs,
                          uint32_t nbatches, uint32_t path, uint64_t* const* offsets_out, uint32_t* const* ids_out,
                          const uint64_t* ids_caps, uint64_t* totals, uint64_t* h2d_bytes) {
    int trunc = 0;
    int rc = guard([&] {
        check_store(s);
        if (nbatches && (!nqs || !offsets_out || !ids_out || !ids_caps || !totals)) raise(MDRQ_EINVAL, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        s->bounce_ids = 0;
        DeviceGuard dg(s->device);
        std::vector<uint64_t> q0(size_t(nbatches) + 1, 0);
        for (uint32_t k = 0; k < nbatches; ++k) {
            q0[k + 1] = q0[k] + nqs[k];
            if (nqs[k] && (!lower || !upper)) raise(MDRQ_EINVAL, "null bounds");
        }
        if (!s->slots) {
            CK(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
            s->slots = new StreamSlot[kStreamSlots];
            for (int i = 0; i < kStreamSlots; ++i) {
                CK(cudaEventCreateWithFlags(&s->slots[i].comp, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&s->slots[i].copy, cudaEventDisableTiming));
                CK(cudaMallocHost(reinterpret_cast<void**>(&s->slots[i].h_flags), 3 * sizeof(unsigned long long)));
                CK(cudaEventCreate(&s->slots[i].cp0));
                CK(cudaEventCreate(&s->slots[i].cp1));
                s->slots[i].b.owner = s;
                s->slots[i].b.own_pool = true;
            }
        }
        uint64_t up = 0;
        // packed copies (pack.cu): MDRQ_STREAM_PACK=0 never, =1 always,
        // otherwise when the lists are long enough for the bucket ends to be
        // small beside them (>= 32 ids per query and bucket, judged on the
        // longest lists a batch of this store's streams has produced)
        const bool sdbg = getenv("MDRQ_DEBUG_STREAM") != nullptr;   // per-stage host timings on stderr
        const auto t_call = std::chrono::steady_clock::now();
        auto since = [&] {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
        };
        const char* pk_env = getenv("MDRQ_STREAM_PACK");
        const int pk_mode = pk_env ? std::atoi(pk_env) : -1;
        const char* th_env = getenv("MDRQ_UNPACK_THREADS");
        int pk_threads = th_env ? std::atoi(th_env) : 0;
        if (pk_threads <= 0) {
            // one process per GPU: the node's ranks share the host threads
            const char* lw = getenv("LOCAL_WORLD_SIZE");
            const int ranks = lw ? std::max(1, std::atoi(lw)) : 1;
            // three quarters of the rank's share: the unpack is memory-bound
            // well before that (25 G ids/s alone on 16 threads, 23 on 12) and
            // the stream's own thread keeps building the next batches
            // (C5 stream on a slow-host box: 349 / 337 / 336 ms per step on
            // 16 / 12 / 8 threads)
            const int hc = std::max(1, int(std::thread::hardware_concurrency()) / ranks);
            pk_threads = std::max(1, hc - hc / 4);
        }
        const uint32_t hb0 = s->id_base >> 16;
        const uint32_t nbuckets = s->n ? uint32_t(((uint64_t(s->id_base) + s->n - 1) >> 16) - hb0 + 1) : 1;
        auto want_pack = [&](uint32_t nq) {
            if (!nq || !s->n || pk_mode == 0 || s->stream_no_pack) return false;
            if (pk_mode > 0) return true;
            return s->stream_per_query >= uint64_t(32) * nbuckets;
        };
        // A packed batch's ids only live in the result pool until the pack
        // kernel behind its pass has run, so packed batches share the store's
        // pool (one pass at a time on the store stream) and a slot holds the
        // low halves instead of a pool of its own; a raw batch's ids stay in
        // its slot's pool until they are copied.
        auto pack = [&](StreamSlot& sl, uint32_t nq) {
            mdrq_batch* b = &sl.b;
            DBuf<uint32_t>& pool = pool_of(s, b);
            sl.packed = !b->own_pool && pool.p;
            if (!sl.packed) return;
            sl.d_lo16.reserve(pool.cap);
            sl.d_ends.reserve(size_t(nq) * nbuckets);   // (not q_split rows: the share moves, a regrowth synchronises)
            if (b->path == MDRQ_PATH_VAFILE_BATCH && !b->vb_perm.empty() && s->vb_ids_slot.p)
                launch_pack_ids16(s->vb_ids_slot.p, b->d_offsets.p, nq, sl.q_split, pool.cap, hb0, nbuckets,
                                  sl.d_lo16.p, sl.d_ends.p, b->d_vb_perm.p, b->d_offsets_p.p,
                                  s->vb_ids_slot.cap > 4 ? s->vb_ids_slot.cap - 4 : 0, s->num_sms, s->stream);
            else
                launch_pack_ids16(pool.p, b->d_offsets.p, nq, sl.q_split, pool.cap, hb0, nbuckets, sl.d_lo16.p,
                                  sl.d_ends.p, nullptr, nullptr, 0, s->num_sms, s->stream);
        };
        // MDRQ_STREAM_PACK_SHARE fixes the packed share of a batch's queries
        // (0..1); otherwise it follows the stream's step period (climb, below)
        const char* sh_env = getenv("MDRQ_STREAM_PACK_SHARE");
        if (sh_env) s->stream_pack_share = std::min(1.0, std::max(0.0, std::atof(sh_env)));
        // MDRQ_DEBUG_STREAM: the copy and unpack times of a slot's last batch
        auto report_times = [&](StreamSlot& sl) {
            if (!sl.measured) return;
            sl.measured = false;
            if (!sdbg) return;
            float copy_ms = 0;
            if (cudaEventElapsedTime(&copy_ms, sl.cp0, sl.cp1) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
            fprintf(stderr, "[stream] copy %.1f ms, unpack %.1f ms at packed share %.2f\n", copy_ms, sl.unpack_ms,
                    s->stream_pack_share);
        };
        // The share follows the stream's step period (the interval between two
        // batches' copies being enqueued), not the two times above: copy and
        // unpack share the host's memory bandwidth, so a longer copy can call
        // for FEWER packed queries.  Hill climbing: every three packed
        // batches the mean of the last two periods is compared with the
        // previous window's; worse -> turn around; then one 0.04 step.
        double hc_prev_t = -1, hc_acc = 0;
        int hc_n = 0;
        auto climb = [&](bool packed_batch) {
            const double t = since();
            const double period = hc_prev_t >= 0 ? t - hc_prev_t : -1;
            hc_prev_t = t;
            if (sh_env || !packed_batch || period <= 0) return;
            if (++hc_n == 1) return;   // the first period after a move still mixes both shares
            hc_acc += period;
            if (hc_n < 3) return;
            const double avg = hc_acc / 2;
            hc_n = 0;
            hc_acc = 0;
            if (s->stream_hc_last > 0 && avg > 0.995 * s->stream_hc_last) s->stream_hc_dir = -s->stream_hc_dir;
            s->stream_hc_last = avg;
            s->stream_pack_share = std::min(1.0, std::max(0.4, s->stream_pack_share + 0.04 * s->stream_hc_dir));
            if (sdbg) fprintf(stderr, "[stream] period %.1f ms -> packed share %.2f\n", avg, s->stream_pack_share);
        };
        s->stream_d2h = s->stream_packed = 0;
        s->stream_batches = nbatches;
        // batch k: host build + H2D + filter/scatter on the store stream,
        // total and overflow flag mirrored to pinned memory
        auto launch = [&](uint32_t k) {
            StreamSlot& sl = s->slots[k % kStreamSlots];
            if (sl.busy) {
                CK(cudaEventSynchronize(sl.copy));   // batch k-3's results have left the slot
                sl.busy = false;
            }
            mdrq_batch* b = &sl.b;
            const uint32_t nq = nqs[k];
            build_descs(s, lower + q0[k] * s->m, upper + q0[k] * s->m, nq,
                        resolve_path(s, path, nq, true, lower + q0[k] * s->m, upper + q0[k] * s->m), true, b);
            upload_batch(s, b, false);
            b->own_pool = !want_pack(nq);
            if (!b->own_pool) {
                // the packed copy lands in pinned staging: if the host cannot
                // pin it, this store's streams stay raw
                try {
                    const size_t need_lo = size_t(s->stream_hint + s->stream_hint / 8 + 4096);
                    const size_t need_en = size_t(nq) * nbuckets;
                    if (need_lo > sl.h_lo16.cap || need_en > sl.h_ends.cap) {
                        sl.join();   // the slot's last unpack still reads the staging
                        sl.h_lo16.reserve(need_lo);
                        sl.h_ends.reserve(need_en);
                    }
                } catch (const Error&) {
                    cudaGetLastError();
                    s->stream_no_pack = true;
                    b->own_pool = true;
                }
            }
            sl.q_split = b->own_pool ? 0u
                                     : std::min<uint32_t>(nq, std::max<uint32_t>(1, uint32_t(s->stream_pack_share * nq + 0.5)));
            b->packed_to = sl.q_split;
            b->shared_pool = b->own_pool ? 0 : uint8_t(k & 1u);
            if (b->own_pool) {
                sl.d_lo16.release();
                sl.d_ends.release();
                s->ids_alt.release();
            } else {
                b->own_ids.release();
                // batch k-2 ran into the same shared pool: its raw tail must
                // have left it (its copies were enqueued an iteration ago)
                if (k >= 2) {
                    StreamSlot& prev = s->slots[(k - 2) % kStreamSlots];
                    if (prev.busy) CK(cudaStreamWaitEvent(s->stream, prev.copy, 0));
                }
            }
            // a pool starts at the size of the largest batch seen so far: a
            // fresh slot must not run its first batch twice
            DBuf<uint32_t>& pool = pool_of(s, b);
            if (s->stream_hint && (!pool.p || pool.cap < s->stream_hint))
                pool.reserve(size_t(s->stream_hint + s->stream_hint / 8 + 4096));
            sl.pool_cap = pool.p ? pool.cap : 0;
            presize_vb_staging(s, b);   // a store's first bit-sliced batch (synchronous, once)
            up += upload_bytes(b);
            enqueue(s, b, true, s->stream);
            pack(sl, nq);
            sl.h_flags[0] = sl.h_flags[1] = sl.h_flags[2] = 0;
            if (nq && s->n) {
                CK(cudaMemcpyAsync(sl.h_flags, b->d_offsets.p + nq, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   s->stream));
                CK(cudaMemcpyAsync(sl.h_flags + 2, b->d_offsets.p + sl.q_split, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s->stream));
                if (b->path == MDRQ_PATH_VAFILE_BATCH && s->vb_flags.p)
                    CK(cudaMemcpyAsync(sl.h_flags + 1, s->vb_flags.p + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                       s->stream));
            }
            CK(cudaEventRecord(sl.comp, s->stream));
            if (sdbg) fprintf(stderr, "[stream] %8.1f launch %u done (packed=%d)\n", since(), k, int(sl.packed));
        };
        // batch k's results to the caller on the copy stream, while batch
        // k+1 runs on the store stream
        auto finish = [&](uint32_t k) {
            StreamSlot& sl = s->slots[k % kStreamSlots];
            mdrq_batch* b = &sl.b;
            const uint32_t nq = nqs[k];
            CK(cudaEventSynchronize(sl.comp));
            if (sdbg) fprintf(stderr, "[stream] %8.1f finish %u: device pass done\n", since(), k);
            const uint64_t total = sl.h_flags[0];
            if (sl.h_flags[1]) grow_vb_staging(s, total);
            DBuf<uint32_t>& pool = pool_of(s, b);
            if (total > sl.pool_cap) {
                // the pool the batch ran into was too small: grow it and run
                // the batch again (behind the next batch's pass and pack)
                if (total > (pool.p ? pool.cap : 0)) pool.reserve(size_t(total + total / 8 + 4096));
                sl.pool_cap = pool.cap;
                enqueue(s, b, true, s->stream);
                pack(sl, nq);
                CK(cudaEventRecord(sl.comp, s->stream));
            }
            totals[k] = total;
            s->stream_hint = std::max<uint64_t>(s->stream_hint, total);
            if (nq) s->stream_per_query = std::max<uint64_t>(s->stream_per_query, total / nq);
            CK(cudaStreamWaitEvent(s->copy_stream, sl.comp, 0));
            if (nq && s->n) {
                CK(cudaMemcpyAsync(offsets_out[k], b->d_offsets.p, sizeof(uint64_t) * (nq + 1), cudaMemcpyDeviceToHost,
                                   s->copy_stream));
                s->stream_d2h += sizeof(uint64_t) * (nq + 1);
            } else {
                std::memset(offsets_out[k], 0, sizeof(uint64_t) * (size_t(nq) + 1));
            }
            if (total > ids_caps[k]) {
                trunc = 1;
                sl.packed = false;
            } else if (total && sl.packed) {
                // the staging still feeds the unpack of the slot's previous batch
                sl.join();
                report_times(sl);
                // ids [0, split) belong to the packed queries, [split, total) travel raw
                const uint64_t split = std::min<uint64_t>(sl.h_flags[2], total);
                sl.h_lo16.reserve(size_t(total + total / 8 + 4096));
                sl.h_ends.reserve(size_t(nq) * nbuckets);
                CK(cudaEventRecord(sl.cp0, s->copy_stream));
                if (split)
                    CK(cudaMemcpyAsync(sl.h_lo16.p, sl.d_lo16.p, sizeof(uint16_t) * split, cudaMemcpyDeviceToHost,
                                       s->copy_stream));
                CK(cudaMemcpyAsync(sl.h_ends.p, sl.d_ends.p, sizeof(uint32_t) * size_t(sl.q_split) * nbuckets,
                                   cudaMemcpyDeviceToHost, s->copy_stream));
                if (total > split)
                    CK(cudaMemcpyAsync(ids_out[k] + split, pool.p + split, sizeof(uint32_t) * (total - split),
                                       cudaMemcpyDeviceToHost, s->copy_stream));
                CK(cudaEventRecord(sl.cp1, s->copy_stream));
                s->stream_d2h += sizeof(uint16_t) * split + sizeof(uint32_t) * size_t(sl.q_split) * nbuckets +
                                 sizeof(uint32_t) * (total - split);
                s->stream_packed += 1;
            } else if (total) {
                sl.packed = false;
                CK(cudaMemcpyAsync(ids_out[k], pool.p, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost,
                                   s->copy_stream));
                s->stream_d2h += sizeof(uint32_t) * total;
            } else {
                sl.packed = false;
            }
            CK(cudaEventRecord(sl.copy, s->copy_stream));
            sl.busy = true;
            climb(sl.packed && k >= 2);
            if (sdbg) fprintf(stderr, "[stream] %8.1f finish %u: copies enqueued\n", since(), k);
        };
        // batch k's ids rebuilt from its packed copy, on host threads, while
        // batch k+1 copies and batch k+2 scans
        auto unpack = [&](uint32_t k) {
            StreamSlot& sl = s->slots[k % kStreamSlots];
            if (!sl.packed) return;
            CK(cudaEventSynchronize(sl.copy));
            if (sdbg) fprintf(stderr, "[stream] %8.1f unpack %u: copy done\n", since(), k);
            const uint16_t* lo = sl.h_lo16.p;
            const uint32_t* en = sl.h_ends.p;
            const uint64_t* of = offsets_out[k];
            uint32_t* out = ids_out[k];
            const uint32_t nq = sl.q_split;
            StreamSlot* slp = &sl;
            sl.join();
            sl.unpack = std::thread([=] {
                const auto t0 = std::chrono::steady_clock::now();
                mdrq_unpack_ids16(lo, en, of, nq, hb0, nbuckets, out, pk_threads);
                slp->unpack_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                slp->measured = true;
                if (sdbg)
                    fprintf(stderr, "[stream] unpack %u: %.1f ms (%llu ids of %u queries)\n", k, slp->unpack_ms,
                            (unsigned long long)(of[nq] - of[0]), nq);
            });
        };
        struct Joiner {   // no unpack thread outlives the call, also when it throws
            mdrq_store* s;
            ~Joiner() {
                if (s->slots)
                    for (int i = 0; i < kStreamSlots; ++i) s->slots[i].join();
            }
        } joiner{s};
        for (uint32_t k = 0; k < nbatches; ++k) {
            launch(k);
            if (k) finish(k - 1);
            if (k >= 2) unpack(k - 2);
        }
        if (nbatches) finish(nbatches - 1);
        if (nbatches >= 2) unpack(nbatches - 2);
        if (nbatches) unpack(nbatches - 1);
        CK(cudaStreamSynchronize(s->copy_stream));
        for (int i = 0; i < kStreamSlots; ++i) {
            s->slots[i].join();
            s->slots[i].busy = false;
        }
        if (h2d_bytes) *h2d_bytes = up;
    });
    if (rc == MDRQ_OK && trunc) {
        g_err = "ids buffer too small for at least one batch (see totals)";
        return MDRQ_ETRUNC;
    }
    return rc;
}

int mdrq_stream_info(mdrq_store* s, uint64_t out[4]) {
    return guard([&] {
        check_store(s);
        if (!out) raise(MDRQ_EINVAL, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        out[0] = s->stream_d2h;
        out[1] = s->stream_packed;
        out[2] = s->stream_batches;
        out[3] = uint64_t(s->stream_pack_share * 1000.0 + 0.5);
    });
}

int mdrq_fetch_ids(mdrq_store* s, uint32_t* ids, uint64_t ids_cap) {
    return guard([&] {
        check_store(s);
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        fetch_ids_impl(s, ids, ids_cap, false);
    });
}

int mdrq_fetch_ids64(mdrq_store* s, int64_t* ids, uint64_t ids_cap) {
    return guard([&] {
        check_store(s);
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        fetch_ids_impl(s, ids, ids_cap, true);
    });
}

int mdrq_query_stats(mdrq_store* s, int mode, mdrq_search_stats* stats, uint32_t nq) {
    return guard([&] {
        check_store(s);
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        mdrq_batch* b = s->last_batch;
        if (!b || b->nq != nq) raise(MDRQ_EINVAL, "no query batch of that size to report");
        if (nq && !stats) raise(MDRQ_EINVAL, "null stats");
        std::vector<unsigned long long> dev(size_t(nq) * 4, 0);
        join(s, s->stream);
        if (nq && s->n)
            CK(cudaMemcpyAsync(dev.data(), b->d_stats.p, sizeof(unsigned long long) * 4 * nq, cudaMemcpyDeviceToHost,
                               s->stream));
        CK(cudaStreamSynchronize(s->stream));
        const uint32_t path = b->path;
        // multi-query passes: the union's planes / columns, shared by the pass
        // (narrow VA unions also stream the union's exact columns for the
        // on-chip refinement: 1 + 4 bytes per tuple and dimension)
        std::vector<uint64_t> pass_bytes(nq, 0);
        if (path == MDRQ_PATH_VAFILE_BATCH) {
            for (const VbPass& p : b->vb_passes)
                for (uint32_t q = p.q0; q < p.q0 + p.nqp; ++q)
                    pass_bytes[b->vb_perm.empty() ? q : b->vb_perm[q]] =
                        p.fallback ? 0 : (s->n * p.kb * (p.kb <= 10 ? 5 : 1)) / p.nqp;
        } else if (path == MDRQ_PATH_COLUMNAR_BATCH) {
            for (const Pass& p : b->passes)
                for (uint32_t q = p.q0; q < p.q0 + p.nqp; ++q)
                    pass_bytes[q] = p.fallback ? 0 : (4 * s->n * p.kb) / p.nqp;
        }
        for (uint32_t q = 0; q < nq; ++q) {
            mdrq_search_stats& o = stats[q];
            const uint64_t k = b->descs[q].k;
            o = mdrq_search_stats{};
            o.bytes_loaded = dev[4 * q + 3] + pass_bytes[q];
            if (path == MDRQ_PATH_ROWWISE) {
                o.objects_compared = s->n;
                o.early_breaks = dev[4 * q + (mode == MDRQ_MODE_BLOCKED ? 1 : 0)];
            } else if (path == MDRQ_PATH_VAFILE) {
                o.objects_compared = dev[4 * q + 2];
                o.nodes_visited = dev[4 * q + 2];
                o.columns_scanned = k;
                o.and_chunks = s->tiles_for(path);
            } else {
                o.objects_compared = k ? k * s->n : 0;
                o.columns_scanned = k;
                o.and_chunks = k ? s->tiles_for(MDRQ_PATH_COLUMNAR) : 0;
            }
        }
    });
}

// ------------------------------------------------------- prepared batches --
int mdrq_batch_prepare(mdrq_store* s, const float* lower, const float* upper, uint32_t nq, uint32_t path,
                       mdrq_batch** out) {
    return guard([&] {
        check_store(s);
        if (!out) raise(MDRQ_EINVAL, "null out");
        if (nq && (!lower || !upper)) raise(MDRQ_EINVAL, "null bounds");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        auto* b = new mdrq_batch();
        try {
            b->owner = s;
            // the ids flavour of AUTO is resolved at run time
            build_descs(s, lower, upper, nq, resolve_path(s, path, nq, false, lower, upper), true, b);
            upload_batch(s, b);
            s->batches.insert(b);
        } catch (...) {
            delete b;
            throw;
        }
        *out = b;
    });
}

int mdrq_batch_destroy(mdrq_batch* b) {
    return guard([&] {
        if (!b) return;
        mdrq_store* s = b->owner;
        if (s) {
            std::lock_guard<std::mutex> lk(s->mu);
            DeviceGuard dg(s->device);
            cudaStreamSynchronize(s->stream);
            if (s->done_stream) cudaStreamSynchronize(s->done_stream);
            if (s->last_batch == b) s->last_batch = nullptr;
            s->batches.erase(b);
            delete b;
        } else {
            delete b;
        }
    });
}

int mdrq_batch_count_async(mdrq_store* s, mdrq_batch* b, uint64_t* d_counts, void* stream) {
    return guard([&] {
        check_store(s);
        if (!b || b->owner != s) raise(MDRQ_EINVAL, "batch does not belong to store");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
        enqueue(s, b, false, st);
        if (d_counts && b->nq)
            CK(cudaMemcpyAsync(d_counts, b->d_counts.p, sizeof(uint64_t) * b->nq, cudaMemcpyDeviceToDevice, st));
        s->last_batch = b;
    });
}

int mdrq_batch_ids_async(mdrq_store* s, mdrq_batch* b, void* stream) {
    return guard([&] {
        check_store(s);
        if (!b || b->owner != s) raise(MDRQ_EINVAL, "batch does not belong to store");
        std::lock_guard<std::mutex> lk(s->mu);
        s->bounce_ids = 0;
        DeviceGuard dg(s->device);
        if (!b->reserved) raise(MDRQ_EINVAL, "ids_async needs mdrq_batch_reserve on this batch first");
        if (b->reserved_total > (pool_of(s, b).p ? pool_of(s, b).cap : 0))
            raise(MDRQ_ETRUNC, "the result pool no longer holds this batch's ids (reserve it again)");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
        enqueue(s, b, true, st);
        s->last_batch = b;
        s->last_nq = b->nq;
        s->last_path = b->path;
        s->last_total = b->reserved_total;
    });
}

int mdrq_batch_reserve(mdrq_store* s, mdrq_batch* b, uint64_t* total) {
    return guard([&] {
        check_store(s);
        if (!b || b->owner != s) raise(MDRQ_EINVAL, "batch does not belong to store");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        const uint64_t t = run_ids_sync(s, b);
        b->reserved = true;
        b->reserved_total = t;
        if (total) *total = t;
    });
}

int mdrq_result_device(mdrq_store* s, uint64_t* d_ids, uint64_t* d_offsets, uint64_t* total) {
    return guard([&] {
        check_store(s);
        std::lock_guard<std::mutex> lk(s->mu);
        mdrq_batch* b = s->last_batch;
        if (!b) raise(MDRQ_EINVAL, "no ids pass has run");
        if (d_ids) *d_ids = reinterpret_cast<uint64_t>(s->ids.p);
        if (d_offsets) *d_offsets = reinterpret_cast<uint64_t>(b->d_offsets.p);
        if (total) *total = s->last_total;
    });
}

int mdrq_batch_info(mdrq_batch* b, uint32_t* info) {
    return guard([&] {
        if (!b || !info) raise(MDRQ_EINVAL, "null argument");
        info[0] = b->path;
        info[1] = b->nq;
        uint32_t passes = 0, kb = 0;
        if (b->path == MDRQ_PATH_VAFILE_BATCH)
            for (const VbPass& p : b->vb_passes) {
                ++passes;
                kb = std::max(kb, p.kb);
            }
        else if (b->path == MDRQ_PATH_COLUMNAR_BATCH)
            for (const Pass& p : b->passes) {
                ++passes;
                kb = std::max(kb, p.kb);
            }
        info[2] = passes;
        info[3] = kb;
    });
}

int mdrq_batch_profile(mdrq_store* s, mdrq_batch* b, int ids_mode, void* stream, double* class_ms,
                       uint32_t* class_launches) {
    return guard([&] {
        check_store(s);
        if (!b || b->owner != s) raise(MDRQ_EINVAL, "batch does not belong to store");
        if (!class_ms || !class_launches) raise(MDRQ_EINVAL, "null output");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
        Profiler prof;
        prof.st = st;
        enqueue(s, b, ids_mode != 0, st, &prof);   // counting run (also a warm-up pass)
        CK(cudaStreamSynchronize(st));
        prof.arm();
        enqueue(s, b, ids_mode != 0, st, &prof);
        prof.mark(-1, 0);
        CK(cudaStreamSynchronize(st));
        for (int c = 0; c < 4; ++c) {
            class_ms[c] = 0.0;
            class_launches[c] = prof.launches[c];
        }
        for (size_t i = 0; i + 1 < prof.ev.size(); ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, prof.ev[i], prof.ev[i + 1]));
            if (prof.cls[i] >= 0) class_ms[prof.cls[i]] += ms;
        }
        if (ids_mode) {
            s->last_batch = b;
            s->last_nq = b->nq;
            s->last_path = b->path;
        }
    });
}

int mdrq_batch_launches(mdrq_batch* b, int ids_mode, uint32_t* launches) {
    return guard([&] {
        if (!b || !b->owner || !launches) raise(MDRQ_EINVAL, "null argument");
        *launches = count_launches(b->owner, b, ids_mode != 0);
    });
}

// --------------------------------------------------- kernel-backend level --
namespace {

bool has_nan(const float* p, uint64_t count) {
    for (uint64_t i = 0; i < count; ++i)
        if (std::isnan(p[i])) return true;
    return false;
}

struct TmpStream {
    cudaStream_t st = nullptr;
    TmpStream() { CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
    ~TmpStream() {
        if (st) cudaStreamDestroy(st);
    }
};

void select_device(int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        raise(MDRQ_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) raise(MDRQ_ENODEV, "bad device ordinal " + std::to_string(device));
}

}  // namespace

int mdrq_match_rows(const float* rows, uint64_t nrows, uint32_t m, const float* lower, const float* upper,
                    int device, uint8_t* out) {
    return guard([&] {
        if (nrows && (!rows || !out)) raise(MDRQ_EINVAL, "null argument");
        if (m && (!lower || !upper)) raise(MDRQ_EINVAL, "null bounds");
        if (!nrows) return;
        if (m == 0) {  // _kernels_cy.pyx:53-54
            std::memset(out, 1, nrows);
            return;
        }
        if (has_nan(rows, nrows * m)) raise(MDRQ_EINVAL, "NaN values are rejected at ingestion");
        select_device(device);
        DeviceGuard dg(device);
        TmpStream ts;
        DBuf<float> d_rows, d_b;
        DBuf<uint8_t> d_out;
        d_rows.reserve(nrows * m);
        d_b.reserve(size_t(2) * m);
        d_out.reserve(nrows);
        CK(cudaMemcpyAsync(d_rows.p, rows, sizeof(float) * nrows * m, cudaMemcpyHostToDevice, ts.st));
        CK(cudaMemcpyAsync(d_b.p, lower, sizeof(float) * m, cudaMemcpyHostToDevice, ts.st));
        CK(cudaMemcpyAsync(d_b.p + m, upper, sizeof(float) * m, cudaMemcpyHostToDevice, ts.st));
        launch_match_rows(d_rows.p, nrows, m, d_b.p, d_b.p + m, d_out.p, ts.st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, d_out.p, nrows, cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
    });
}

int mdrq_scan_rows(const float* values, uint64_t n, uint32_t m, const float* lower, const float* upper, int mode,
                   int device, int64_t* ids_out, uint64_t* count_out, uint64_t* early_out) {
    return guard([&] {
        if (!count_out) raise(MDRQ_EINVAL, "null count");
        if (m < 1) raise(MDRQ_EINVAL, "dimensionality must be at least 1");
        if (!lower || !upper) raise(MDRQ_EINVAL, "null bounds");
        *count_out = 0;
        if (early_out) *early_out = 0;
        if (!n) return;
        if (!values || !ids_out) raise(MDRQ_EINVAL, "null argument");
        if (has_nan(values, n * m)) raise(MDRQ_EINVAL, "NaN values are rejected at ingestion");
        mdrq_store* s = nullptr;
        int rc = mdrq_store_create(values, n, m, device, MDRQ_LAYOUT_ROWWISE, 0, 0, &s);
        if (rc != MDRQ_OK) raise(rc, g_err);
        struct Holder {
            mdrq_store* s;
            ~Holder() { mdrq_store_destroy(s); }
        } holder{s};
        DeviceGuard dg(s->device);
        mdrq_batch* b = &s->scratch;
        b->owner = s;
        build_descs(s, lower, upper, 1, MDRQ_PATH_ROWWISE, false, b);
        upload_batch(s, b);
        const uint64_t tot = run_ids_sync(s, b);
        std::vector<uint32_t> tmp(tot);
        unsigned long long st4[4] = {0, 0, 0, 0};
        if (tot) CK(cudaMemcpyAsync(tmp.data(), s->ids.p, sizeof(uint32_t) * tot, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaMemcpyAsync(st4, b->d_stats.p, sizeof(st4), cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        for (uint64_t i = 0; i < tot; ++i) ids_out[i] = int64_t(tmp[i]);
        *count_out = tot;
        if (early_out) *early_out = st4[mode == MDRQ_MODE_BLOCKED ? 1 : 0];
    });
}

int mdrq_scan_column(const float* col, uint64_t n, float lo, float hi, int device, uint8_t* mask_out) {
    return guard([&] {
        if (!n) return;
        if (!col || !mask_out) raise(MDRQ_EINVAL, "null argument");
        select_device(device);
        DeviceGuard dg(device);
        TmpStream ts;
        const uint64_t nwords = (n + 31) / 32;
        DBuf<float> d_col;
        DBuf<uint32_t> d_mask;
        d_col.reserve(n);
        d_mask.reserve(nwords);
        CK(cudaMemcpyAsync(d_col.p, col, sizeof(float) * n, cudaMemcpyHostToDevice, ts.st));
        launch_scan_column_mask(d_col.p, n, lo, hi, d_mask.p, ts.st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(mask_out, d_mask.p, (n + 7) / 8, cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
    });
}

int mdrq_and_masks(const uint8_t* const* masks, uint32_t k, uint64_t nbytes, int device, uint8_t* out) {
    return guard([&] {
        if (k == 0) raise(MDRQ_EINVAL, "no masks to merge");
        if (!nbytes) return;
        if (!masks || !out) raise(MDRQ_EINVAL, "null argument");
        select_device(device);
        DeviceGuard dg(device);
        TmpStream ts;
        const uint64_t nwords = (nbytes + 3) / 4;
        DBuf<uint32_t> d_in, d_out;
        d_in.reserve(nwords * k);
        d_out.reserve(nwords);
        CK(cudaMemsetAsync(d_in.p, 0, d_in.bytes(), ts.st));
        std::vector<const uint32_t*> ptrs(k);
        for (uint32_t j = 0; j < k; ++j) {
            if (!masks[j]) raise(MDRQ_EINVAL, "null mask");
            CK(cudaMemcpyAsync(d_in.p + j * nwords, masks[j], nbytes, cudaMemcpyHostToDevice, ts.st));
            ptrs[j] = d_in.p + j * nwords;
        }
        launch_and_masks(ptrs.data(), k, nwords, d_out.p, ts.st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, d_out.p, nbytes, cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
    });
}

int mdrq_mask_popcount(const uint8_t* mask, uint64_t nbytes, int device, uint64_t* count_out) {
    return guard([&] {
        if (!count_out) raise(MDRQ_EINVAL, "null count");
        *count_out = 0;
        if (!nbytes) return;
        if (!mask) raise(MDRQ_EINVAL, "null mask");
        select_device(device);
        DeviceGuard dg(device);
        TmpStream ts;
        const uint64_t nwords = (nbytes + 3) / 4;
        DBuf<uint32_t> d_in;
        DBuf<unsigned long long> d_c;
        d_in.reserve(nwords);
        d_c.reserve(1);
        CK(cudaMemsetAsync(d_in.p, 0, d_in.bytes(), ts.st));
        CK(cudaMemcpyAsync(d_in.p, mask, nbytes, cudaMemcpyHostToDevice, ts.st));
        launch_popcount(d_in.p, nwords, d_c.p, ts.st);
        CK(cudaGetLastError());
        unsigned long long c = 0;
        CK(cudaMemcpyAsync(&c, d_c.p, sizeof(c), cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
        *count_out = c;
    });
}

int mdrq_mask_to_ids(const uint8_t* mask, uint64_t n, int device, int64_t* ids_out, uint64_t* count_out) {
    return guard([&] {
        if (!count_out) raise(MDRQ_EINVAL, "null count");
        *count_out = 0;
        if (!n) return;
        if (!mask || !ids_out) raise(MDRQ_EINVAL, "null argument");
        select_device(device);
        DeviceGuard dg(device);
        TmpStream ts;
        const uint64_t nbytes = (n + 7) / 8, nwords = (n + 31) / 32;
        const uint64_t tiles = (nwords + 255) / 256;
        DBuf<uint32_t> d_in, d_ctr;
        DBuf<uint64_t> d_status;
        DBuf<unsigned long long> d_c;
        DBuf<int64_t> d_ids;
        d_in.reserve(nwords);
        d_ctr.reserve(1);
        d_status.reserve(tiles);
        d_c.reserve(1);
        d_ids.reserve(n);
        CK(cudaMemsetAsync(d_in.p, 0, d_in.bytes(), ts.st));
        CK(cudaMemsetAsync(d_status.p, 0, d_status.bytes(), ts.st));
        CK(cudaMemcpyAsync(d_in.p, mask, nbytes, cudaMemcpyHostToDevice, ts.st));
        launch_mask_to_ids(d_in.p, n, nullptr, d_status.p, 1, d_ctr.p, d_c.p, d_ids.p, ts.st);
        CK(cudaGetLastError());
        unsigned long long c = 0;
        CK(cudaMemcpyAsync(&c, d_c.p, sizeof(c), cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
        if (c) CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(int64_t) * c, cudaMemcpyDeviceToHost, ts.st));
        CK(cudaStreamSynchronize(ts.st));
        *count_out = c;
    });
}

}  // extern "C"
