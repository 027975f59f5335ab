// spgsim:: CSR API of the drop-in library. Kernels run on the B200 through the
// C ABI; the small host helpers (canonical check, triplets, permutations,
// comparisons, vconcat of host slices) are plain C++.
#include "spgsim/csr.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "device.hpp"
#include "spgsim/rng.hpp"

namespace spgsim {

using detail::check;
using detail::context;
using detail::DevCsr;

CsrMatrix CsrMatrix::zeros(index_t nrows, index_t ncols) {
    CsrMatrix m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.rowptr.assign(static_cast<std::size_t>(nrows) + 1, 0);
    return m;
}

CsrMatrix CsrMatrix::identity(index_t n) {
    CsrMatrix m = zeros(n, n);
    m.colind.resize(static_cast<std::size_t>(n));
    m.values.assign(static_cast<std::size_t>(n), 1.0);
    std::iota(m.colind.begin(), m.colind.end(), index_t{0});
    std::iota(m.rowptr.begin(), m.rowptr.end(), index_t{0});
    return m;
}

void CsrMatrix::check_canonical() const {
    if (nrows < 0 || ncols < 0) throw Error("negative dimension");
    if (rowptr.size() != static_cast<std::size_t>(nrows) + 1) throw Error("rowptr length != nrows+1");
    if (rowptr.front() != 0) throw Error("rowptr[0] != 0");
    if (colind.size() != values.size()) throw Error("colind/values length mismatch");
    if (rowptr.back() != static_cast<index_t>(colind.size())) throw Error("rowptr[nrows] != nnz");
    for (index_t i = 0; i < nrows; ++i) {
        const index_t lo = rowptr[static_cast<std::size_t>(i)], hi = rowptr[static_cast<std::size_t>(i) + 1];
        if (lo > hi) throw Error("rowptr not non-decreasing at row " + std::to_string(i));
        index_t prev = -1;
        for (index_t t = lo; t < hi; ++t) {
            const index_t j = colind[static_cast<std::size_t>(t)];
            if (j < 0 || j >= ncols) throw Error("column index out of range in row " + std::to_string(i));
            if (j <= prev) throw Error("columns not strictly increasing in row " + std::to_string(i));
            prev = j;
        }
    }
}

bool CsrMatrix::is_canonical() const {
    try {
        check_canonical();
    } catch (const Error&) {
        return false;
    }
    return true;
}

CsrMatrix from_triplets(index_t nrows, index_t ncols, std::vector<Triplet> entries) {
    for (const Triplet& e : entries)
        if (e.row < 0 || e.row >= nrows || e.col < 0 || e.col >= ncols)
            throw ParameterError("triplet coordinate out of range");
    // Stable order by (row, col): duplicates are summed in input order.
    std::stable_sort(entries.begin(), entries.end(),
                     [](const Triplet& x, const Triplet& y) { return x.row != y.row ? x.row < y.row : x.col < y.col; });
    CsrMatrix m = CsrMatrix::zeros(nrows, ncols);
    m.colind.reserve(entries.size());
    m.values.reserve(entries.size());
    for (std::size_t i = 0; i < entries.size();) {
        const index_t r = entries[i].row, c = entries[i].col;
        double s = 0.0;
        for (; i < entries.size() && entries[i].row == r && entries[i].col == c; ++i) s += entries[i].value;
        m.colind.push_back(c);
        m.values.push_back(s);
        ++m.rowptr[static_cast<std::size_t>(r) + 1];
    }
    std::partial_sum(m.rowptr.begin(), m.rowptr.end(), m.rowptr.begin());
    return m;
}

Permutation Permutation::identity(index_t n) {
    Permutation p;
    p.n = n;
    p.map.resize(static_cast<std::size_t>(n));
    std::iota(p.map.begin(), p.map.end(), index_t{0});
    return p;
}

Permutation Permutation::reversal(index_t n) {
    Permutation p = identity(n);
    std::reverse(p.map.begin(), p.map.end());
    return p;
}

Permutation Permutation::random(index_t n, std::uint64_t seed) {
    // Fisher-Yates from the top with the SplitMix64 stream (same draws as the reference).
    Permutation p = identity(n);
    SplitMix64 rng(seed);
    for (index_t i = n - 1; i > 0; --i) {
        const auto j = static_cast<index_t>(rng.below(static_cast<std::uint64_t>(i) + 1));
        std::swap(p.map[static_cast<std::size_t>(i)], p.map[static_cast<std::size_t>(j)]);
    }
    return p;
}

Permutation Permutation::inverse() const {
    Permutation q;
    q.n = n;
    q.map.assign(static_cast<std::size_t>(n), 0);
    for (index_t i = 0; i < n; ++i) q.map[static_cast<std::size_t>(map[static_cast<std::size_t>(i)])] = i;
    return q;
}

void Permutation::check_valid() const {
    if (static_cast<index_t>(map.size()) != n) throw ParameterError("permutation length != n");
    std::vector<char> seen(static_cast<std::size_t>(n), 0);
    for (const index_t v : map) {
        if (v < 0 || v >= n || seen[static_cast<std::size_t>(v)]) throw ParameterError("permutation is not a bijection on [0,n)");
        seen[static_cast<std::size_t>(v)] = 1;
    }
}

// ------------------------------------------------------------ device kernels
CsrMatrix spgemm_local(const CsrMatrix& a, const CsrMatrix& b) {
    if (a.ncols != b.nrows)
        throw DimensionError("spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    spg_ctx* ctx = context(0);
    DevCsr da = detail::upload(ctx, a), db = detail::upload(ctx, b);
    spg_csr* c = nullptr;
    check(spg_spgemm(ctx, da.p, db.p, &c));
    DevCsr dc(c);
    return detail::download(ctx, dc.p);
}

CsrMatrix spgeam(const CsrMatrix& a, const CsrMatrix& b) {
    if (a.nrows != b.nrows || a.ncols != b.ncols) throw DimensionError("spgeam: shape mismatch");
    spg_ctx* ctx = context(0);
    DevCsr da = detail::upload(ctx, a), db = detail::upload(ctx, b);
    spg_csr* c = nullptr;
    check(spg_spgeam(ctx, da.p, db.p, &c));
    DevCsr dc(c);
    return detail::download(ctx, dc.p);
}

CsrMatrix column_normalize(const CsrMatrix& a) {
    spg_ctx* ctx = context(0);
    DevCsr da = detail::upload(ctx, a);
    check(spg_column_normalize(ctx, da.p));
    return detail::download(ctx, da.p);
}

CsrMatrix prune(const CsrMatrix& a, double threshold) {
    if (threshold < 0.0) throw ParameterError("prune: negative threshold");
    spg_ctx* ctx = context(0);
    DevCsr da = detail::upload(ctx, a);
    spg_csr* r = nullptr;
    check(spg_prune(ctx, da.p, threshold, &r));
    DevCsr dr(r);
    return detail::download(ctx, dr.p);
}

// csr.cpp:251-255 on the device (values within 1e-12 of glibc's pow)
CsrMatrix elementwise_power(const CsrMatrix& a, double exponent) {
    spg_ctx* ctx = context(0);
    DevCsr da = detail::upload(ctx, a);
    check(spg_elementwise_power(ctx, da.p, exponent));
    return detail::download(ctx, da.p);
}

// -------------------------------------------------------------- host helpers
CsrMatrix permute_symmetric(const CsrMatrix& a, const Permutation& p) {
    if (a.nrows != a.ncols) throw DimensionError("permute_symmetric: matrix not square");
    if (p.n != a.nrows) throw DimensionError("permute_symmetric: permutation size mismatch");
    const Permutation inv = p.inverse();
    CsrMatrix r = CsrMatrix::zeros(a.nrows, a.ncols);
    r.colind.resize(a.colind.size());
    r.values.resize(a.values.size());
    for (index_t out = 0; out < a.nrows; ++out) {
        const index_t src = inv.map[static_cast<std::size_t>(out)];
        r.rowptr[static_cast<std::size_t>(out) + 1] = r.rowptr[static_cast<std::size_t>(out)] +
                                                      a.rowptr[static_cast<std::size_t>(src) + 1] -
                                                      a.rowptr[static_cast<std::size_t>(src)];
    }
    std::vector<std::pair<index_t, double>> row;
    for (index_t out = 0; out < a.nrows; ++out) {
        const index_t src = inv.map[static_cast<std::size_t>(out)];
        row.clear();
        for (index_t t = a.rowptr[static_cast<std::size_t>(src)]; t < a.rowptr[static_cast<std::size_t>(src) + 1]; ++t)
            row.emplace_back(p.map[static_cast<std::size_t>(a.colind[static_cast<std::size_t>(t)])],
                             a.values[static_cast<std::size_t>(t)]);
        std::sort(row.begin(), row.end());
        index_t o = r.rowptr[static_cast<std::size_t>(out)];
        for (const auto& [j, v] : row) {
            r.colind[static_cast<std::size_t>(o)] = j;
            r.values[static_cast<std::size_t>(o++)] = v;
        }
    }
    return r;
}


CsrMatrix vconcat(const std::vector<const CsrMatrix*>& slices) {
    if (slices.empty()) return {};
    CsrMatrix out;
    out.ncols = slices.front()->ncols;
    std::size_t nnz = 0, rows = 0;
    for (const CsrMatrix* s : slices) {
        if (s->ncols != out.ncols) throw DimensionError("vconcat: column count mismatch");
        nnz += s->colind.size();
        rows += static_cast<std::size_t>(s->nrows);
    }
    out.rowptr.reserve(rows + 1);
    out.colind.reserve(nnz);
    out.values.reserve(nnz);
    for (const CsrMatrix* s : slices) {
        const index_t base = out.nnz();
        for (index_t i = 1; i <= s->nrows; ++i) out.rowptr.push_back(base + s->rowptr[static_cast<std::size_t>(i)]);
        out.colind.insert(out.colind.end(), s->colind.begin(), s->colind.end());
        out.values.insert(out.values.end(), s->values.begin(), s->values.end());
        out.nrows += s->nrows;
    }
    return out;
}

bool pattern_equal(const CsrMatrix& a, const CsrMatrix& b) {
    return a.nrows == b.nrows && a.ncols == b.ncols && a.rowptr == b.rowptr && a.colind == b.colind;
}

bool allclose(const CsrMatrix& a, const CsrMatrix& b, double rel_tol) {
    if (!pattern_equal(a, b)) return false;
    for (std::size_t t = 0; t < a.values.size(); ++t) {
        const double x = a.values[t], y = b.values[t];
        if (x != y && std::abs(x - y) > rel_tol * std::max(std::abs(x), std::abs(y))) return false;
    }
    return true;
}

}  // namespace spgsim
