/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, or called by,
 * the product library (paper_2603_21444_b200/). Only tests/, smoke() and
 * bench.py's cpu_baseline leg load it, and only as the checker.
 *
 * Plain-C restatement of the reference simulator's hot-path arithmetic
 * (/root/reference/proj). Each function cites the reference lines it restates.
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   1. against the golden vectors in tests/golden/ (produced by the reference
 *      itself, oracle/_ref/libspgref.so, via tests/golden/make_golden.py), and
 *   2. against the reference library directly when oracle/_ref is present.
 * Build-side generators with no reference counterpart (rectangular ER, R-MAT)
 * live here too so the CPU checker and the GPU path consume identical inputs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t nrows, ncols;
    int64_t *rowptr; /* nrows+1 */
    int64_t *colind; /* nnz */
    double *values;  /* nnz */
} ocsr;

void oracle_free(ocsr *m) {
    free(m->rowptr);
    free(m->colind);
    free(m->values);
    m->rowptr = NULL;
    m->colind = NULL;
    m->values = NULL;
}

static int ocsr_alloc(ocsr *m, int64_t nrows, int64_t ncols, int64_t cap) {
    m->nrows = nrows;
    m->ncols = ncols;
    m->rowptr = (int64_t *)calloc((size_t)nrows + 1, sizeof(int64_t));
    m->colind = (int64_t *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int64_t));
    m->values = (double *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(double));
    return (m->rowptr && m->colind && m->values) ? 0 : -1;
}

/* ---- SplitMix64: rng.hpp:10-34 ------------------------------------------ */
typedef struct { uint64_t s; } sm64;
static uint64_t sm64_next(sm64 *r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double sm64_u01(sm64 *r) { return (double)(sm64_next(r) >> 11) * 0x1.0p-53; }
static double sm64_pos(sm64 *r) { return (double)((sm64_next(r) >> 11) + 1) * 0x1.0p-53; }

/* ---- products per row: Σ_{k∈A_i} nnz(B_k) (SURVEY §8(d) unit of work) --- */
int64_t oracle_products(const ocsr *a, const ocsr *b, int64_t *per_row) {
    int64_t total = 0;
    for (int64_t i = 0; i < a->nrows; ++i) {
        int64_t p = 0;
        for (int64_t t = a->rowptr[i]; t < a->rowptr[i + 1]; ++t) {
            const int64_t k = a->colind[t];
            p += b->rowptr[k + 1] - b->rowptr[k];
        }
        if (per_row) per_row[i] = p;
        total += p;
    }
    return total;
}

/*
 * spgemm_local: csr.cpp:132-165. Gustavson row merge with a dense accumulator
 * over B's columns; per output entry the contributions are summed in ascending
 * order of A's column index as acc = 0.0; acc += av*bv (separate multiply and
 * add, no FMA: this file is compiled with -ffp-contract=off). The touched list
 * is sorted per row, explicit zeros are kept. Returns -2 on a.ncols != b.nrows
 * (the reference's DimensionError, csr.cpp:133-135).
 */
static int cmp_i64(const void *x, const void *y) {
    const int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return a < b ? -1 : a > b;
}
int oracle_spgemm(const ocsr *a, const ocsr *b, ocsr *c) {
    if (a->ncols != b->nrows) return -2;
    const int64_t cap = oracle_products(a, b, NULL);
    if (ocsr_alloc(c, a->nrows, b->ncols, cap)) return -1;
    double *acc = (double *)calloc((size_t)(b->ncols > 0 ? b->ncols : 1), sizeof(double));
    int64_t *mark = (int64_t *)malloc((size_t)(b->ncols > 0 ? b->ncols : 1) * sizeof(int64_t));
    int64_t *touched = (int64_t *)malloc((size_t)(b->ncols > 0 ? b->ncols : 1) * sizeof(int64_t));
    for (int64_t j = 0; j < b->ncols; ++j) mark[j] = -1;
    int64_t out = 0;
    for (int64_t i = 0; i < a->nrows; ++i) {
        int64_t nt = 0;
        for (int64_t t = a->rowptr[i]; t < a->rowptr[i + 1]; ++t) {
            const int64_t k = a->colind[t];
            const double av = a->values[t];
            for (int64_t u = b->rowptr[k]; u < b->rowptr[k + 1]; ++u) {
                const int64_t j = b->colind[u];
                if (mark[j] != i) {
                    mark[j] = i;
                    acc[j] = 0.0;
                    touched[nt++] = j;
                }
                const double p = av * b->values[u];
                acc[j] = acc[j] + p;
            }
        }
        qsort(touched, (size_t)nt, sizeof(int64_t), cmp_i64);
        for (int64_t s = 0; s < nt; ++s) {
            c->colind[out] = touched[s];
            c->values[out] = acc[touched[s]];
            ++out;
        }
        c->rowptr[i + 1] = out;
    }
    free(acc);
    free(mark);
    free(touched);
    return 0;
}

/* spgeam: csr.cpp:167-196. Row-wise two-pointer merge, union pattern,
 * equal columns summed a+b, cancellation zeros kept. -2 on shape mismatch. */
int oracle_spgeam(const ocsr *a, const ocsr *b, ocsr *c) {
    if (a->nrows != b->nrows || a->ncols != b->ncols) return -2;
    const int64_t cap = a->rowptr[a->nrows] + b->rowptr[b->nrows];
    if (ocsr_alloc(c, a->nrows, a->ncols, cap)) return -1;
    int64_t out = 0;
    for (int64_t i = 0; i < a->nrows; ++i) {
        int64_t ta = a->rowptr[i], tb = b->rowptr[i];
        const int64_t ea = a->rowptr[i + 1], eb = b->rowptr[i + 1];
        while (ta < ea || tb < eb) {
            const int64_t ja = ta < ea ? a->colind[ta] : a->ncols;
            const int64_t jb = tb < eb ? b->colind[tb] : a->ncols;
            if (ja < jb) {
                c->colind[out] = ja;
                c->values[out++] = a->values[ta++];
            } else if (jb < ja) {
                c->colind[out] = jb;
                c->values[out++] = b->values[tb++];
            } else {
                c->colind[out] = ja;
                c->values[out++] = a->values[ta++] + b->values[tb++];
            }
        }
        c->rowptr[i + 1] = out;
    }
    return 0;
}

/* vconcat: csr.cpp:348-363. -2 on column-count mismatch. */
int oracle_vconcat(const ocsr *const *slices, int n, ocsr *out) {
    int64_t rows = 0, nnz = 0;
    if (n == 0) return ocsr_alloc(out, 0, 0, 0);
    for (int s = 0; s < n; ++s) {
        if (slices[s]->ncols != slices[0]->ncols) return -2;
        rows += slices[s]->nrows;
        nnz += slices[s]->rowptr[slices[s]->nrows];
    }
    if (ocsr_alloc(out, rows, slices[0]->ncols, nnz)) return -1;
    int64_t r = 0, base = 0;
    for (int s = 0; s < n; ++s) {
        const ocsr *m = slices[s];
        for (int64_t i = 0; i < m->nrows; ++i) out->rowptr[++r] = base + m->rowptr[i + 1];
        const int64_t k = m->rowptr[m->nrows];
        memcpy(out->colind + base, m->colind, (size_t)k * sizeof(int64_t));
        memcpy(out->values + base, m->values, (size_t)k * sizeof(double));
        base += k;
    }
    return 0;
}

/* gen_erdos_renyi: csr.cpp:257-279. Geometric skip over the n*n cells with
 * SplitMix64; values uniform_pos. Returns -3 on bad parameters. */
int oracle_gen_erdos_renyi(int64_t n, double density, uint64_t seed, ocsr *m) {
    if (n < 0 || !(density > 0.0) || density > 1.0) return -3;
    const double expect = (double)n * (double)n * density;
    int64_t cap = (int64_t)(expect + 10.0 * sqrt(expect + 1.0) + 16.0);
    if (ocsr_alloc(m, n, n, cap)) return -1;
    sm64 rng = {seed};
    const double logq = log1p(-density);
    const int64_t ncells = n * n;
    int64_t cell = -1, nnz = 0;
    for (;;) {
        const double u = sm64_u01(&rng);
        const int64_t skip = density == 1.0 ? 0 : (int64_t)floor(log1p(-u) / logq);
        cell += 1 + skip;
        if (cell >= ncells) break;
        if (nnz == cap) {
            cap *= 2;
            m->colind = (int64_t *)realloc(m->colind, (size_t)cap * sizeof(int64_t));
            m->values = (double *)realloc(m->values, (size_t)cap * sizeof(double));
        }
        m->colind[nnz] = cell % n;
        m->values[nnz] = sm64_pos(&rng);
        m->rowptr[cell / n + 1]++;
        ++nnz;
    }
    for (int64_t r = 0; r < n; ++r) m->rowptr[r + 1] += m->rowptr[r];
    return 0;
}

/* Rectangular ER (build-side addition): the same
 * geometric skip over nrows*ncols cells. No reference counterpart. */
int oracle_gen_erdos_renyi_rect(int64_t nrows, int64_t ncols, double density, uint64_t seed, ocsr *m) {
    if (nrows < 0 || ncols < 0 || !(density > 0.0) || density > 1.0) return -3;
    const double expect = (double)nrows * (double)ncols * density;
    int64_t cap = (int64_t)(expect + 10.0 * sqrt(expect + 1.0) + 16.0);
    if (ocsr_alloc(m, nrows, ncols, cap)) return -1;
    sm64 rng = {seed};
    const double logq = log1p(-density);
    const int64_t ncells = nrows * ncols;
    int64_t cell = -1, nnz = 0;
    for (;;) {
        const double u = sm64_u01(&rng);
        const int64_t skip = density == 1.0 ? 0 : (int64_t)floor(log1p(-u) / logq);
        cell += 1 + skip;
        if (cell >= ncells) break;
        if (nnz == cap) {
            cap *= 2;
            m->colind = (int64_t *)realloc(m->colind, (size_t)cap * sizeof(int64_t));
            m->values = (double *)realloc(m->values, (size_t)cap * sizeof(double));
        }
        m->colind[nnz] = cell % ncols;
        m->values[nnz] = sm64_pos(&rng);
        m->rowptr[cell / ncols + 1]++;
        ++nnz;
    }
    for (int64_t r = 0; r < nrows; ++r) m->rowptr[r + 1] += m->rowptr[r];
    return 0;
}

/* ---- partition (trident scheme) : partition.cpp:74-81, 104-127, 161-222 --- */
static void block_bounds(int64_t dim, int64_t nb, int64_t *out) {
    out[0] = 0;
    for (int64_t b = 0; b < nb; ++b) out[b + 1] = out[b] + dim / nb + (b < dim % nb ? 1 : 0);
}

/* Tile rectangle of `rank` under the trident scheme (rank = (i*q+j)*lam+k). */
void oracle_trident_rect(int64_t nrows, int64_t ncols, int q, int lam, int rank, int64_t rect[4]) {
    int64_t coarse[65], cols[65], fine[65];
    block_bounds(nrows, q, coarse);
    block_bounds(ncols, q, cols);
    const int node = rank / lam, i = node / q, j = node % q, k = rank % lam;
    block_bounds(coarse[i + 1] - coarse[i], lam, fine);
    rect[0] = coarse[i] + fine[k];
    rect[1] = coarse[i] + fine[k + 1];
    rect[2] = cols[j];
    rect[3] = cols[j + 1];
}

/* Extracts the sub-block [r0,r1)x[c0,c1) with local indices. */
int oracle_extract(const ocsr *m, const int64_t rect[4], ocsr *t) {
    int64_t cnt = 0;
    for (int64_t i = rect[0]; i < rect[1]; ++i)
        for (int64_t u = m->rowptr[i]; u < m->rowptr[i + 1]; ++u)
            cnt += (m->colind[u] >= rect[2] && m->colind[u] < rect[3]);
    if (ocsr_alloc(t, rect[1] - rect[0], rect[3] - rect[2], cnt)) return -1;
    int64_t o = 0;
    for (int64_t i = rect[0]; i < rect[1]; ++i) {
        for (int64_t u = m->rowptr[i]; u < m->rowptr[i + 1]; ++u)
            if (m->colind[u] >= rect[2] && m->colind[u] < rect[3]) {
                t->colind[o] = m->colind[u] - rect[2];
                t->values[o++] = m->values[u];
            }
        t->rowptr[i - rect[0] + 1] = o;
    }
    return 0;
}

/* column_normalize: csr.cpp:224-234 (column sums in storage order; divide
 * when the sum is nonzero). prune: csr.cpp:236-249 (drop v < theta). In place
 * for normalize; prune allocates. */
int oracle_column_normalize(ocsr *m) {
    double *s = (double *)calloc((size_t)(m->ncols > 0 ? m->ncols : 1), sizeof(double));
    const int64_t nnz = m->rowptr[m->nrows];
    for (int64_t t = 0; t < nnz; ++t) s[m->colind[t]] += m->values[t];
    for (int64_t t = 0; t < nnz; ++t)
        if (s[m->colind[t]] != 0.0) m->values[t] /= s[m->colind[t]];
    free(s);
    return 0;
}

int oracle_prune(const ocsr *a, double theta, ocsr *r) {
    if (theta < 0.0) return -3;
    if (ocsr_alloc(r, a->nrows, a->ncols, a->rowptr[a->nrows])) return -1;
    int64_t o = 0;
    for (int64_t i = 0; i < a->nrows; ++i) {
        for (int64_t t = a->rowptr[i]; t < a->rowptr[i + 1]; ++t) {
            if (a->values[t] < theta) continue;
            r->colind[o] = a->colind[t];
            r->values[o++] = a->values[t];
        }
        r->rowptr[i + 1] = o;
    }
    return 0;
}
