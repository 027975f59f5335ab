// spgsim::CsrMatrix and the sparse kernels of the drop-in library.
//
// Same types, names and semantics as the reference header
// (proj/include/spgsim/csr.hpp): a caller of the reference compiles against this
// header unchanged. The multiply, add, normalize and prune kernels execute on a
// B200 through the C ABI (include/spg/capi.h); there is no CPU fallback — with
// no usable sm_100 device they throw spgsim::DeviceError.
#pragma once

#include <cstdint>
#include <vector>

#include "spgsim/errors.hpp"

namespace spgsim {

using index_t = std::int64_t;

// Canonical CSR (csr.hpp:12-17 of the reference): rowptr[0]==0, non-decreasing,
// rowptr[nrows]==nnz; per row strictly increasing columns in [0,ncols);
// explicit zeros are stored entries and are never dropped.
struct CsrMatrix {
    index_t nrows = 0;
    index_t ncols = 0;
    std::vector<index_t> rowptr{0};
    std::vector<index_t> colind;
    std::vector<double> values;

    index_t nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
    static CsrMatrix zeros(index_t nrows, index_t ncols);
    static CsrMatrix identity(index_t n);
    void check_canonical() const;  // throws Error naming the violated invariant
    bool is_canonical() const;
    bool operator==(const CsrMatrix&) const = default;
};

struct Triplet {
    index_t row;
    index_t col;
    double value;
};

// Canonical matrix from coordinates; duplicates are summed (a zero sum stays stored).
CsrMatrix from_triplets(index_t nrows, index_t ncols, std::vector<Triplet> entries);

struct Permutation {
    index_t n = 0;
    std::vector<index_t> map;
    static Permutation identity(index_t n);
    static Permutation reversal(index_t n);
    static Permutation random(index_t n, std::uint64_t seed);
    Permutation inverse() const;
    void check_valid() const;
};

// --- device kernels (B200) ----------------------------------------------------
// C = A*B; per output entry the contributions are summed in ascending inner
// index with separate multiply/add, so C equals the reference bit for bit.
CsrMatrix spgemm_local(const CsrMatrix& a, const CsrMatrix& b);
// C = A + B over the union pattern.
CsrMatrix spgeam(const CsrMatrix& a, const CsrMatrix& b);
CsrMatrix column_normalize(const CsrMatrix& a);
CsrMatrix prune(const CsrMatrix& a, double threshold);

// --- host helpers -------------------------------------------------------------
CsrMatrix permute_symmetric(const CsrMatrix& a, const Permutation& p);
CsrMatrix elementwise_power(const CsrMatrix& a, double exponent);
CsrMatrix vconcat(const std::vector<const CsrMatrix*>& slices);
bool pattern_equal(const CsrMatrix& a, const CsrMatrix& b);
bool allclose(const CsrMatrix& a, const CsrMatrix& b, double rel_tol);

// --- synthetic generators (deterministic per seed) ------------------------------
// Reference generator (same stream, same matrix).
CsrMatrix gen_erdos_renyi(index_t n, double density, std::uint64_t seed);
CsrMatrix gen_uniform_stride(index_t n, index_t row_nnz);
// Build-side additions for the benchmark configs (no reference counterpart):
// rectangular ER over nrows*ncols cells (config 5) and Graph500 R-MAT (config 3,
// SURVEY §8(d) draw order, duplicates summed, then a random symmetric permutation).
CsrMatrix gen_erdos_renyi_rect(index_t nrows, index_t ncols, double density, std::uint64_t seed);
CsrMatrix gen_rmat(int scale, int edge_factor, std::uint64_t seed, std::uint64_t perm_seed);
CsrMatrix transpose(const CsrMatrix& a);

}  // namespace spgsim
