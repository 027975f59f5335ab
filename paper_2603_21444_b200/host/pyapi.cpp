// extern "C" helpers of libspgsim_b200.so for the Python mirror: the host-side
// generators (parallel, bit-identical to the reference stream where one
// exists). Results are malloc'd; free with spgx_free.
#include <cstdlib>
#include <cstring>
#include <string>

#include "spgsim/csr.hpp"

extern "C" {

struct spgx_csr {
    std::int64_t nrows, ncols, nnz;
    std::int64_t* rowptr;
    std::int64_t* colind;
    double* values;
};

static thread_local std::string g_err;
const char* spgx_last_error() { return g_err.c_str(); }

static int fill(const spgsim::CsrMatrix& m, spgx_csr* out) {
    out->nrows = m.nrows;
    out->ncols = m.ncols;
    out->nnz = m.nnz();
    out->rowptr = static_cast<std::int64_t*>(std::malloc(sizeof(std::int64_t) * (m.rowptr.size())));
    out->colind = static_cast<std::int64_t*>(std::malloc(sizeof(std::int64_t) * (m.colind.size() + 1)));
    out->values = static_cast<double*>(std::malloc(sizeof(double) * (m.values.size() + 1)));
    if (!out->rowptr || !out->colind || !out->values) return -1;
    std::memcpy(out->rowptr, m.rowptr.data(), sizeof(std::int64_t) * m.rowptr.size());
    std::memcpy(out->colind, m.colind.data(), sizeof(std::int64_t) * m.colind.size());
    std::memcpy(out->values, m.values.data(), sizeof(double) * m.values.size());
    return 0;
}

}  // extern "C"

template <class F>
static int wrap(F&& f, spgx_csr* out) {
    try {
        return fill(f(), out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

extern "C" {

void spgx_free(spgx_csr* m) {
    std::free(m->rowptr);
    std::free(m->colind);
    std::free(m->values);
    m->rowptr = m->colind = nullptr;
    m->values = nullptr;
}

int spgx_gen_erdos_renyi(std::int64_t n, double density, std::uint64_t seed, spgx_csr* out) {
    return wrap([&] { return spgsim::gen_erdos_renyi(n, density, seed); }, out);
}

int spgx_gen_erdos_renyi_rect(std::int64_t nr, std::int64_t nc, double density, std::uint64_t seed, spgx_csr* out) {
    return wrap([&] { return spgsim::gen_erdos_renyi_rect(nr, nc, density, seed); }, out);
}

int spgx_gen_rmat(int scale, int edge_factor, std::uint64_t seed, std::uint64_t perm_seed, spgx_csr* out) {
    return wrap([&] { return spgsim::gen_rmat(scale, edge_factor, seed, perm_seed); }, out);
}

int spgx_transpose(const spgx_csr* in, spgx_csr* out) {
    return wrap(
        [&] {
            spgsim::CsrMatrix m;
            m.nrows = in->nrows;
            m.ncols = in->ncols;
            m.rowptr.assign(in->rowptr, in->rowptr + in->nrows + 1);
            m.colind.assign(in->colind, in->colind + in->nnz);
            m.values.assign(in->values, in->values + in->nnz);
            return spgsim::transpose(m);
        },
        out);
}

}  // extern "C"
