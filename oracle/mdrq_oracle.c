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
