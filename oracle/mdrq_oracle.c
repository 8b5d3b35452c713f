/*
 * mdrq_oracle.c -- CPU restatement of the reference's MDRQ scan kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_1801_03644_b200) never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/mdrq/):
 *
 *   oracle_match_code   <- _kernels_cy.pyx:23-46   (_match_code: scalar early
 *                          break / 8-lane blocked verdict, codes 1 / 0 / -1)
 *   oracle_match_row    <- _kernels_cy.pyx:49-55   (match_row)
 *   oracle_scan_rows    <- _kernels_cy.pyx:58-86   (scan_rows: ascending local
 *                          ids, objects compared, early-break count)
 *   oracle_scan_column  <- _kernels_cy.pyx:89-120  (scan_column: packed
 *                          little-endian bitmask)
 *   oracle_and_masks    <- scan.py:55-78           (and_masks_chunked result)
 *   oracle_mask_popcount<- scan.py:81-82
 *   oracle_mask_to_ids  <- scan.py:85-88
 *   oracle_count_batch / oracle_ids_batch
 *                       <- SequentialScan.search (scan.py:103-111) applied to a
 *                          batch of queries; OpenMP over queries/rows so the
 *                          full-size configs can be checked in minutes
 *                          (SURVEY.md 8d parity budget).
 *   oracle_va_code      <- the quantile-grid cell function the GPU VA-file
 *                          uses: code(v) = #{boundaries <= v} (SURVEY.md 7,
 *                          "VA-file soundness"); the reference's equal-width
 *                          2-bit grid is vafile.py:38-45 and is not restated,
 *                          parity for the VA-file is on id sets only.
 *
 * Comparison semantics are exactly the reference's: float32 inclusive
 * lo <= v <= hi, evaluated as the reference writes it, no fast-math.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define LANE_C 8

/* _kernels_cy.pyx:23-46 */
int oracle_match_code(const float* v, const float* lo, const float* hi,
                      int64_t m, int mode) {
    if (mode == 0) {
        for (int64_t j = 0; j < m; ++j) {
            if ((v[j] < lo[j]) | (v[j] > hi[j]))
                return j < m - 1 ? -1 : 0;
        }
        return 1;
    }
    int64_t blocks = m / LANE_C;
    for (int64_t b = 0; b < blocks; ++b) {
        int64_t base = b * LANE_C;
        int ok = 1;
        for (int k = 0; k < LANE_C; ++k)
            ok = ok & (lo[base + k] <= v[base + k]) & (v[base + k] <= hi[base + k]);
        if (!ok)
            return base + LANE_C < m ? -1 : 0;
    }
    for (int64_t j = blocks * LANE_C; j < m; ++j) {
        if ((v[j] < lo[j]) | (v[j] > hi[j]))
            return j < m - 1 ? -1 : 0;
    }
    return 1;
}

/* _kernels_cy.pyx:49-55 (m == 0 matches) */
int oracle_match_row(const float* row, const float* lo, const float* hi,
                     int64_t m, int mode) {
    if (m == 0) return 1;
    return oracle_match_code(row, lo, hi, m, mode) == 1;
}

/* _kernels_cy.pyx:58-86.  ids_out must hold n entries. */
int64_t oracle_scan_rows(const float* values, int64_t n, int64_t m,
                         const float* lo, const float* hi, int mode,
                         int64_t* ids_out, int64_t* early_out) {
    int64_t cnt = 0, early = 0;
    for (int64_t i = 0; i < n; ++i) {
        int code = oracle_match_code(values + i * m, lo, hi, m, mode);
        if (code == 1)
            ids_out[cnt++] = i;
        else if (code < 0)
            ++early;
    }
    if (early_out) *early_out = early;
    return cnt;
}

/* _kernels_cy.pyx:89-120 (both modes produce the same mask). */
void oracle_scan_column(const float* col, int64_t n, float lo, float hi,
                        uint8_t* mask_out) {
    memset(mask_out, 0, (size_t)((n + 7) / 8));
    for (int64_t i = 0; i < n; ++i) {
        float v = col[i];
        if (lo <= v && v <= hi)
            mask_out[i >> 3] |= (uint8_t)(1u << (i & 7));
    }
}

/* scan.py:55-78 -- the chunking only changes who computes which byte. */
void oracle_and_masks(const uint8_t* const* masks, int64_t k, int64_t nbytes,
                      uint8_t* out) {
    for (int64_t b = 0; b < nbytes; ++b) {
        uint8_t acc = masks[0][b];
        for (int64_t j = 1; j < k; ++j) acc &= masks[j][b];
        out[b] = acc;
    }
}

/* scan.py:81-82 */
int64_t oracle_mask_popcount(const uint8_t* mask, int64_t nbytes) {
    int64_t c = 0;
    for (int64_t b = 0; b < nbytes; ++b) c += __builtin_popcount(mask[b]);
    return c;
}

/* scan.py:85-88 (only the first n bits count). */
int64_t oracle_mask_to_ids(const uint8_t* mask, int64_t n, int64_t* ids_out) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        if (mask[i >> 3] >> (i & 7) & 1) ids_out[c++] = i;
    return c;
}

/* Row match without the early-break bookkeeping; same verdict as
 * oracle_match_code(...) == 1 for either mode. */
static inline int row_matches(const float* v, const float* lo, const float* hi,
                              int64_t m) {
    for (int64_t j = 0; j < m; ++j)
        if ((v[j] < lo[j]) | (v[j] > hi[j])) return 0;
    return 1;
}

/* SequentialScan over a batch: counts[q] = |ids(q)|.  lo/hi are [nq][m]. */
void oracle_count_batch(const float* values, int64_t n, int64_t m,
                        const float* lo, const float* hi, int64_t nq,
                        int64_t* counts, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    for (int64_t q = 0; q < nq; ++q) counts[q] = 0;
    const int64_t CH = 1 << 14;
    int64_t nchunks = (n + CH - 1) / CH;
    /* rows outer (one pass over the data), queries inner, chunked so each
     * chunk stays cache resident while every query visits it */
#pragma omp parallel
    {
        int64_t* local = (int64_t*)calloc((size_t)(nq > 0 ? nq : 1), sizeof(int64_t));
#pragma omp for schedule(dynamic, 4)
        for (int64_t c = 0; c < nchunks; ++c) {
            int64_t r0 = c * CH, r1 = r0 + CH < n ? r0 + CH : n;
            for (int64_t q = 0; q < nq; ++q) {
                const float* ql = lo + q * m;
                const float* qh = hi + q * m;
                int64_t cnt = 0;
                for (int64_t i = r0; i < r1; ++i)
                    cnt += row_matches(values + i * m, ql, qh, m);
                local[q] += cnt;
            }
        }
#pragma omp critical
        for (int64_t q = 0; q < nq; ++q) counts[q] += local[q];
        free(local);
    }
}

/* SequentialScan over a batch, ids mode.  offsets[nq+1] must come from a
 * prior oracle_count_batch (exclusive prefix); ids_out holds offsets[nq]. */
void oracle_ids_batch(const float* values, int64_t n, int64_t m,
                      const float* lo, const float* hi, int64_t nq,
                      const int64_t* offsets, int64_t* ids_out, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nq; ++q) {
        const float* ql = lo + q * m;
        const float* qh = hi + q * m;
        int64_t w = offsets[q];
        for (int64_t i = 0; i < n; ++i)
            if (row_matches(values + i * m, ql, qh, m)) ids_out[w++] = i;
    }
}

/* Quantile-grid cell: number of boundaries b[0..nb-1] (sorted) that are <= v. */
int32_t oracle_va_code(const float* b, int32_t nb, float v) {
    int32_t c = 0;
    for (int32_t i = 0; i < nb; ++i) c += (b[i] <= v);
    return c;
}

void oracle_va_encode(const float* col, int64_t n, const float* b, int32_t nb,
                      uint8_t* codes_out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        codes_out[i] = (uint8_t)oracle_va_code(b, nb, col[i]);
}

int oracle_has_openmp(void) {
#ifdef _OPENMP
    return 1;
#else
    return 0;
#endif
}

/* ------------------------------------------------------------------------
 * oracle_hash_batch -- SequentialScan (scan.py:103-111) over a query batch,
 * reduced to (count, set hash) per query so the full-size configurations
 * (C2-C5: up to 5e8 rows x 1e4 queries, 5e9 ids) can be checked for EVERY
 * query without materialising the id lists.
 *
 * The verdict per (row, query) is the reference's _match_code predicate
 * (_kernels_cy.pyx:23-46): AND over the dims of lo_j <= v_j <= hi_j in
 * float32 (ordered compares, no fast-math).  A dim with lo = -inf and
 * hi = +inf (the reference's unconstrained sentinel, core.py:123-132) is true
 * for every non-NaN value and is skipped; NaN values are reported (return
 * value -1) because the reference rejects them at ingestion (core.py:65-66).
 *
 * The rows [0, n) of `values` (row-major [n][m]) carry the global ids
 * id0 .. id0+n-1.  Results are ACCUMULATED into counts[q] and
 * hashes[q] += sum over matching ids of mix64(id) (mod 2^64), so a table can
 * be streamed through in row chunks in any order.  A sorted, duplicate-free
 * id list (which the GPU tests check separately) is fixed by its set, and the
 * set by (count, hash) up to a 2^-64 collision.
 *
 * Work split: OpenMP over 8 192-row blocks; a block is transposed into
 * per-dim columns (L2-resident), then every query walks it in 16-row groups
 * with AVX2 compares, leaving a group at the first dim that rejects all 16.
 * ---------------------------------------------------------------------- */
static inline uint64_t oracle_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t oracle_id_hash(uint64_t id) { return oracle_mix64(id); }

#define HB_ROWS 8192
#define HB_GROUP 16

#if defined(__x86_64__)
#include <immintrin.h>
__attribute__((target("avx2")))
static void hb_block_avx2(const float* cols, int64_t rows, int64_t id0,
                          const int32_t* qdims, const int32_t* qnd, int64_t maxd,
                          const float* lo, const float* hi, int64_t m, int64_t nq,
                          int64_t* cnt, uint64_t* hsh) {
    int64_t groups = rows / HB_GROUP;
    for (int64_t q = 0; q < nq; ++q) {
        const int32_t* dims = qdims + q * maxd;
        int32_t nd = qnd[q];
        int64_t c = 0;
        uint64_t h = 0;
        if (nd == 0) {
            for (int64_t r = 0; r < rows; ++r) { ++c; h += oracle_mix64((uint64_t)(id0 + r)); }
        } else {
            const float* ql = lo + q * m;
            const float* qh = hi + q * m;
            for (int64_t g = 0; g < groups; ++g) {
                uint32_t alive = 0xFFFFu;
                /* two dims per test of `alive`: half the data-dependent branches */
                for (int32_t k = 0; k < nd && alive; k += 2) {
                    int32_t d0 = dims[k], d1 = dims[k + 1 < nd ? k + 1 : k];
                    const float* c0 = cols + (int64_t)d0 * HB_ROWS + g * HB_GROUP;
                    const float* c1 = cols + (int64_t)d1 * HB_ROWS + g * HB_GROUP;
                    __m256 l0 = _mm256_set1_ps(ql[d0]), u0 = _mm256_set1_ps(qh[d0]);
                    __m256 l1 = _mm256_set1_ps(ql[d1]), u1 = _mm256_set1_ps(qh[d1]);
                    __m256 a0 = _mm256_loadu_ps(c0), b0 = _mm256_loadu_ps(c0 + 8);
                    __m256 a1 = _mm256_loadu_ps(c1), b1 = _mm256_loadu_ps(c1 + 8);
                    __m256 ma = _mm256_and_ps(_mm256_and_ps(_mm256_cmp_ps(a0, l0, _CMP_GE_OQ), _mm256_cmp_ps(a0, u0, _CMP_LE_OQ)),
                                              _mm256_and_ps(_mm256_cmp_ps(a1, l1, _CMP_GE_OQ), _mm256_cmp_ps(a1, u1, _CMP_LE_OQ)));
                    __m256 mb = _mm256_and_ps(_mm256_and_ps(_mm256_cmp_ps(b0, l0, _CMP_GE_OQ), _mm256_cmp_ps(b0, u0, _CMP_LE_OQ)),
                                              _mm256_and_ps(_mm256_cmp_ps(b1, l1, _CMP_GE_OQ), _mm256_cmp_ps(b1, u1, _CMP_LE_OQ)));
                    alive &= (uint32_t)_mm256_movemask_ps(ma) | ((uint32_t)_mm256_movemask_ps(mb) << 8);
                }
                while (alive) {
                    int b = __builtin_ctz(alive);
                    alive &= alive - 1;
                    ++c;
                    h += oracle_mix64((uint64_t)(id0 + g * HB_GROUP + b));
                }
            }
            for (int64_t r = groups * HB_GROUP; r < rows; ++r) {
                int ok = 1;
                for (int32_t k = 0; k < nd && ok; ++k) {
                    float v = cols[(int64_t)dims[k] * HB_ROWS + r];
                    ok = lo[q * m + dims[k]] <= v && v <= hi[q * m + dims[k]];
                }
                if (ok) { ++c; h += oracle_mix64((uint64_t)(id0 + r)); }
            }
        }
        cnt[q] += c;
        hsh[q] += h;
    }
}
#endif

static void hb_block_scalar(const float* cols, int64_t rows, int64_t id0,
                            const int32_t* qdims, const int32_t* qnd, int64_t maxd,
                            const float* lo, const float* hi, int64_t m, int64_t nq,
                            int64_t* cnt, uint64_t* hsh) {
    for (int64_t q = 0; q < nq; ++q) {
        const int32_t* dims = qdims + q * maxd;
        for (int64_t r = 0; r < rows; ++r) {
            int ok = 1;
            for (int32_t k = 0; k < qnd[q] && ok; ++k) {
                float v = cols[(int64_t)dims[k] * HB_ROWS + r];
                ok = lo[q * m + dims[k]] <= v && v <= hi[q * m + dims[k]];
            }
            if (ok) { ++cnt[q]; hsh[q] += oracle_mix64((uint64_t)(id0 + r)); }
        }
    }
}

int oracle_hash_batch(const float* values, int64_t n, int64_t m, int64_t id0,
                      const float* lo, const float* hi, int64_t nq,
                      int64_t* counts, uint64_t* hashes, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    if (nq <= 0 || n <= 0) return 0;
    /* constrained dims per query (the +-inf sentinel pair is skipped) */
    int32_t* qdims = (int32_t*)malloc((size_t)(nq * (m > 0 ? m : 1)) * sizeof(int32_t));
    int32_t* qnd = (int32_t*)calloc((size_t)nq, sizeof(int32_t));
    for (int64_t q = 0; q < nq; ++q)
        for (int64_t j = 0; j < m; ++j) {
            float l = lo[q * m + j], u = hi[q * m + j];
            if (!(l == -__builtin_inff() && u == __builtin_inff())) qdims[q * m + qnd[q]++] = (int32_t)j;
        }
    int use_avx2 = 0;
#if defined(__x86_64__)
    use_avx2 = __builtin_cpu_supports("avx2");
#endif
    int64_t nblocks = (n + HB_ROWS - 1) / HB_ROWS;
    int bad = 0;
#pragma omp parallel
    {
        float* cols = (float*)malloc((size_t)(HB_ROWS * (m > 0 ? m : 1)) * sizeof(float));
        int64_t* cnt = (int64_t*)calloc((size_t)nq, sizeof(int64_t));
        uint64_t* hsh = (uint64_t*)calloc((size_t)nq, sizeof(uint64_t));
        int mybad = 0;
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < nblocks; ++b) {
            int64_t r0 = b * HB_ROWS, rows = n - r0 < HB_ROWS ? n - r0 : HB_ROWS;
            for (int64_t r = 0; r < rows; ++r)
                for (int64_t j = 0; j < m; ++j) {
                    float v = values[(r0 + r) * m + j];
                    mybad |= v != v;
                    cols[j * HB_ROWS + r] = v;
                }
#if defined(__x86_64__)
            if (use_avx2)
                hb_block_avx2(cols, rows, id0 + r0, qdims, qnd, m, lo, hi, m, nq, cnt, hsh);
            else
#endif
                hb_block_scalar(cols, rows, id0 + r0, qdims, qnd, m, lo, hi, m, nq, cnt, hsh);
        }
#pragma omp critical
        {
            for (int64_t q = 0; q < nq; ++q) { counts[q] += cnt[q]; hashes[q] += hsh[q]; }
            bad |= mybad;
        }
        free(cols); free(cnt); free(hsh);
    }
    free(qdims); free(qnd);
    return bad ? -1 : 0;
}
