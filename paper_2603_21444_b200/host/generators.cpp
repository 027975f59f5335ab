// Deterministic synthetic inputs. gen_erdos_renyi reproduces the reference's
// stream (csr.cpp:257-279) bit for bit, but runs on all host cores: SplitMix64
// is counter-based, so entry e's skip draw is call 2e+1 and its value draw is
// call 2e+2 of the stream, independent of every other entry. Cell positions are
// then a prefix sum of (1 + skip). R-MAT and the rectangular ER are build-side
// additions for configs 3 and 5; they have no reference
// counterpart.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>

#include "spgsim/csr.hpp"
#include "spgsim/rng.hpp"

namespace spgsim {
namespace {

int nthreads() {
    const unsigned h = std::thread::hardware_concurrency();
    return static_cast<int>(h == 0 ? 4 : std::min(h, 64u));
}

template <class F>
void parallel_for(std::int64_t n, F&& f) {
    const int T = nthreads();
    std::vector<std::thread> th;
    const std::int64_t chunk = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const std::int64_t lo = t * chunk, hi = std::min<std::int64_t>(n, lo + chunk);
        if (lo >= hi) break;
        th.emplace_back([=, &f] { f(t, lo, hi); });
    }
    for (auto& x : th) x.join();
}

// ER over nrows x ncols cells with the reference's geometric skip.
CsrMatrix er_cells(index_t nrows, index_t ncols, double density, std::uint64_t seed) {
    if (nrows < 0 || ncols < 0) throw ParameterError("gen_erdos_renyi: negative n");
    if (!(density > 0.0) || density > 1.0) throw ParameterError("gen_erdos_renyi: density must be in (0, 1]");
    const double logq = std::log1p(-density);
    const index_t ncells = nrows * ncols;
    CsrMatrix m = CsrMatrix::zeros(nrows, ncols);
    std::vector<index_t> cells;
    const double expect = static_cast<double>(ncells) * density;
    index_t batch = static_cast<index_t>(expect + 8.0 * std::sqrt(expect + 1.0) + 1024.0);
    index_t cell = -1, e0 = 0;
    bool done = false;
    while (!done) {
        std::vector<index_t> step(static_cast<std::size_t>(batch));
        const int T = nthreads();
        std::vector<index_t> part(static_cast<std::size_t>(T) + 1, 0);
        parallel_for(batch, [&](int t, std::int64_t lo, std::int64_t hi) {
            index_t s = 0;
            for (std::int64_t e = lo; e < hi; ++e) {
                const std::uint64_t t_call = 2 * static_cast<std::uint64_t>(e0 + e) + 1;
                const double u = static_cast<double>(SplitMix64::at(seed, t_call) >> 11) * 0x1.0p-53;
                const index_t skip = density == 1.0 ? 0 : static_cast<index_t>(std::floor(std::log1p(-u) / logq));
                step[static_cast<std::size_t>(e)] = 1 + skip;
                s += 1 + skip;
            }
            part[static_cast<std::size_t>(t) + 1] = s;
        });
        // exclusive offsets per chunk, then local prefix
        const std::int64_t chunk = (batch + T - 1) / T;
        std::vector<index_t> base(static_cast<std::size_t>(T) + 1, cell);
        for (int t = 0; t < T; ++t) base[static_cast<std::size_t>(t) + 1] = base[static_cast<std::size_t>(t)] + part[static_cast<std::size_t>(t) + 1];
        parallel_for(batch, [&](int t, std::int64_t lo, std::int64_t hi) {
            index_t c = base[static_cast<std::size_t>(lo / chunk)];
            (void)t;
            for (std::int64_t e = lo; e < hi; ++e) {
                c += step[static_cast<std::size_t>(e)];
                step[static_cast<std::size_t>(e)] = c;
            }
        });
        const auto end = std::lower_bound(step.begin(), step.end(), ncells);
        cells.insert(cells.end(), step.begin(), end);
        if (end != step.end()) done = true;
        else {
            cell = step.back();
            e0 += batch;
            batch = std::max<index_t>(batch / 4, 1 << 16);
        }
    }
    const std::int64_t E = static_cast<std::int64_t>(cells.size());
    m.colind.resize(static_cast<std::size_t>(E));
    m.values.resize(static_cast<std::size_t>(E));
    parallel_for(E, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t e = lo; e < hi; ++e) {
            const index_t c = cells[static_cast<std::size_t>(e)];
            m.colind[static_cast<std::size_t>(e)] = c % ncols;
            const std::uint64_t t_call = 2 * static_cast<std::uint64_t>(e) + 2;
            m.values[static_cast<std::size_t>(e)] = static_cast<double>((SplitMix64::at(seed, t_call) >> 11) + 1) * 0x1.0p-53;
        }
    });
    for (std::int64_t e = 0; e < E; ++e) ++m.rowptr[static_cast<std::size_t>(cells[static_cast<std::size_t>(e)] / ncols) + 1];
    std::partial_sum(m.rowptr.begin(), m.rowptr.end(), m.rowptr.begin());
    return m;
}

}  // namespace

CsrMatrix gen_erdos_renyi(index_t n, double density, std::uint64_t seed) {
    if (n < 0) throw ParameterError("gen_erdos_renyi: negative n");
    return er_cells(n, n, density, seed);
}

CsrMatrix gen_erdos_renyi_rect(index_t nrows, index_t ncols, double density, std::uint64_t seed) {
    return er_cells(nrows, ncols, density, seed);
}

CsrMatrix gen_uniform_stride(index_t n, index_t row_nnz) {
    if (row_nnz <= 0 || n % row_nnz != 0) throw ParameterError("gen_uniform_stride: row_nnz must divide n");
    const index_t stride = n / row_nnz;
    CsrMatrix m = CsrMatrix::zeros(n, n);
    std::vector<index_t> cols(static_cast<std::size_t>(row_nnz));
    for (index_t i = 0; i < n; ++i) {
        for (index_t t = 0; t < row_nnz; ++t) cols[static_cast<std::size_t>(t)] = (i + t * stride) % n;
        std::sort(cols.begin(), cols.end());
        for (const index_t j : cols) {
            m.colind.push_back(j);
            m.values.push_back(1.0 + static_cast<double>((i + j) % 7) * 0.125);
        }
        m.rowptr[static_cast<std::size_t>(i) + 1] = static_cast<index_t>(m.colind.size());
    }
    return m;
}

// Sorted-by-(row, col) canonical CSR from coordinate arrays; duplicates summed
// in input order. Counting sort by row, then a stable per-row sort by column.
static CsrMatrix from_coo(index_t nrows, index_t ncols, const std::vector<index_t>& r, const std::vector<index_t>& c,
                          const std::vector<double>& v) {
    const std::size_t E = r.size();
    std::vector<index_t> cnt(static_cast<std::size_t>(nrows) + 1, 0);
    for (std::size_t e = 0; e < E; ++e) ++cnt[static_cast<std::size_t>(r[e]) + 1];
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    std::vector<index_t> pos(cnt.begin(), cnt.end() - 1);
    std::vector<std::pair<index_t, double>> byrow(E);
    for (std::size_t e = 0; e < E; ++e) byrow[static_cast<std::size_t>(pos[static_cast<std::size_t>(r[e])]++)] = {c[e], v[e]};
    CsrMatrix m = CsrMatrix::zeros(nrows, ncols);
    std::vector<index_t> rowlen(static_cast<std::size_t>(nrows), 0);
    std::vector<std::vector<std::pair<index_t, double>>> dedup(static_cast<std::size_t>(nthreads()));
    // per-row stable sort + dedup (in parallel over rows), then compact
    std::vector<index_t> newlen(static_cast<std::size_t>(nrows), 0);
    parallel_for(nrows, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t i = lo; i < hi; ++i) {
            auto b = byrow.begin() + cnt[static_cast<std::size_t>(i)], e = byrow.begin() + cnt[static_cast<std::size_t>(i) + 1];
            std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
            index_t w = 0;
            for (auto it = b; it != e;) {
                const index_t col = it->first;
                double s = 0.0;
                for (; it != e && it->first == col; ++it) s += it->second;
                *(b + w) = {col, s};
                ++w;
            }
            newlen[static_cast<std::size_t>(i)] = w;
        }
    });
    for (index_t i = 0; i < nrows; ++i) m.rowptr[static_cast<std::size_t>(i) + 1] = m.rowptr[static_cast<std::size_t>(i)] + newlen[static_cast<std::size_t>(i)];
    m.colind.resize(static_cast<std::size_t>(m.nnz()));
    m.values.resize(static_cast<std::size_t>(m.nnz()));
    parallel_for(nrows, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t i = lo; i < hi; ++i) {
            index_t o = m.rowptr[static_cast<std::size_t>(i)];
            const index_t b = cnt[static_cast<std::size_t>(i)];
            for (index_t t = 0; t < newlen[static_cast<std::size_t>(i)]; ++t, ++o) {
                m.colind[static_cast<std::size_t>(o)] = byrow[static_cast<std::size_t>(b + t)].first;
                m.values[static_cast<std::size_t>(o)] = byrow[static_cast<std::size_t>(b + t)].second;
            }
        }
    });
    return m;
}

CsrMatrix gen_rmat(int scale, int edge_factor, std::uint64_t seed, std::uint64_t perm_seed) {
    if (scale < 1 || scale > 30 || edge_factor < 1) throw ParameterError("gen_rmat: bad scale/edge factor");
    const double a = 0.57, b = 0.19, c = 0.19;
    const index_t n = index_t{1} << scale;
    const std::int64_t E = static_cast<std::int64_t>(edge_factor) * n;
    std::vector<index_t> rr(static_cast<std::size_t>(E)), cc(static_cast<std::size_t>(E));
    std::vector<double> vv(static_cast<std::size_t>(E));
    const std::uint64_t per = static_cast<std::uint64_t>(scale) + 1;
    parallel_for(E, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t e = lo; e < hi; ++e) {
            std::uint64_t t = static_cast<std::uint64_t>(e) * per;
            index_t r = 0, col = 0;
            for (int l = 0; l < scale; ++l) {
                const double u = static_cast<double>(SplitMix64::at(seed, ++t) >> 11) * 0x1.0p-53;
                const index_t rb = u >= a + b;
                const index_t cb = (u >= a && u < a + b) || u >= a + b + c;
                r = (r << 1) | rb;
                col = (col << 1) | cb;
            }
            rr[static_cast<std::size_t>(e)] = r;
            cc[static_cast<std::size_t>(e)] = col;
            vv[static_cast<std::size_t>(e)] = static_cast<double>((SplitMix64::at(seed, ++t) >> 11) + 1) * 0x1.0p-53;
        }
    });
    CsrMatrix m = from_coo(n, n, rr, cc, vv);
    return permute_symmetric(m, Permutation::random(n, perm_seed));
}

CsrMatrix transpose(const CsrMatrix& a) {
    CsrMatrix t = CsrMatrix::zeros(a.ncols, a.nrows);
    for (const index_t j : a.colind) ++t.rowptr[static_cast<std::size_t>(j) + 1];
    std::partial_sum(t.rowptr.begin(), t.rowptr.end(), t.rowptr.begin());
    t.colind.resize(a.colind.size());
    t.values.resize(a.values.size());
    std::vector<index_t> pos(t.rowptr.begin(), t.rowptr.end() - 1);
    for (index_t i = 0; i < a.nrows; ++i)
        for (index_t u = a.rowptr[static_cast<std::size_t>(i)]; u < a.rowptr[static_cast<std::size_t>(i) + 1]; ++u) {
            const index_t o = pos[static_cast<std::size_t>(a.colind[static_cast<std::size_t>(u)])]++;
            t.colind[static_cast<std::size_t>(o)] = i;
            t.values[static_cast<std::size_t>(o)] = a.values[static_cast<std::size_t>(u)];
        }
    return t;
}

}  // namespace spgsim
