// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the reference simulator's own C++ code (compiled from the
// sources under /root/reference/proj with -Dspgsim=spgref, see oracle/Makefile)
// so that pytest, smoke() and bench.py's cpu_baseline / --impl reference arm
// can call the reference's spgemm_local / spgeam / vconcat / partition /
// trident_spgemm / summa_spgemm directly through ctypes.
//
// Every function below forwards to exactly one reference entry point:
//   ref_spgemm_local     -> csr.cpp:132-165       (spgemm_local)
//   ref_spgeam           -> csr.cpp:167-196       (spgeam)
//   ref_vconcat          -> csr.cpp:348-363       (vconcat)
//   ref_gen_erdos_renyi  -> csr.cpp:257-279       (gen_erdos_renyi)
//   ref_from_triplets    -> csr.cpp:61-88         (from_triplets)
//   ref_permute_random   -> csr.cpp:104-112, 198-222
//   ref_column_normalize -> csr.cpp:224-234 ; ref_prune -> csr.cpp:236-249
//   ref_elementwise_power -> csr.cpp:251-255 ; ref_result_checksum -> report.cpp:11-26
//   ref_partition        -> partition.cpp:161-222 ; ref_reassemble -> :224-261
//   ref_trident          -> algorithms.cpp:24-101 (trident_spgemm)
//   ref_summa            -> algorithms.cpp:103-174 (summa_spgemm)
//   ref_oned             -> algorithms.cpp:176-269 (oned_spgemm)
//   ref_predict_volume   -> netmodel.cpp:210-224
// The namespace is renamed by the preprocessor, so nothing here collides with
// the product library's own `spgsim` symbols if both end up in one process.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "spgsim/algorithms.hpp"
#include "spgsim/report.hpp"
#include "spgsim/csr.hpp"
#include "spgsim/netmodel.hpp"
#include "spgsim/partition.hpp"

using namespace spgsim;  // == spgref after -Dspgsim=spgref

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const DimensionError*>(&e)) return 2;
    if (dynamic_cast<const ParameterError*>(&e)) return 3;
    if (dynamic_cast<const GridError*>(&e)) return 4;
    if (dynamic_cast<const IncompleteTileSet*>(&e)) return 5;
    if (dynamic_cast<const RoutingError*>(&e)) return 6;
    if (dynamic_cast<const ScheduleError*>(&e)) return 7;
    if (dynamic_cast<const DeadlockError*>(&e)) return 8;
    return 1;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

CsrMatrix* box(CsrMatrix&& m) { return new CsrMatrix(std::move(m)); }

// ledger layout: [rank][dir: 0 sent, 1 received][class: 0 LI, 1 GI][messages, nnz, bytes]
void dump_ledger(const CommLedger& l, int procs, std::uint64_t* out) {
    if (!out) return;
    for (int r = 0; r < procs; ++r)
        for (int d = 0; d < 2; ++d)
            for (int c = 0; c < 2; ++c) {
                const LinkClass lc = c == 0 ? LinkClass::LI : LinkClass::GI;
                const LedgerCell& cell = d == 0 ? l.sent(r, lc) : l.received(r, lc);
                std::uint64_t* o = out + ((static_cast<std::size_t>(r) * 2 + d) * 2 + c) * 3;
                o[0] = cell.messages;
                o[1] = cell.nnz;
                o[2] = cell.bytes;
            }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_csr_new(std::int64_t nrows, std::int64_t ncols, const std::int64_t* rowptr,
                  const std::int64_t* colind, const double* values) {
    auto* m = new CsrMatrix;
    m->nrows = nrows;
    m->ncols = ncols;
    m->rowptr.assign(rowptr, rowptr + nrows + 1);
    const std::int64_t nnz = rowptr[nrows];
    m->colind.assign(colind, colind + nnz);
    m->values.assign(values, values + nnz);
    return m;
}

void ref_csr_free(void* h) { delete static_cast<CsrMatrix*>(h); }

void ref_csr_info(const void* h, std::int64_t* nrows, std::int64_t* ncols, std::int64_t* nnz) {
    const auto* m = static_cast<const CsrMatrix*>(h);
    *nrows = m->nrows;
    *ncols = m->ncols;
    *nnz = m->nnz();
}

const std::int64_t* ref_csr_rowptr(const void* h) { return static_cast<const CsrMatrix*>(h)->rowptr.data(); }
const std::int64_t* ref_csr_colind(const void* h) { return static_cast<const CsrMatrix*>(h)->colind.data(); }
const double* ref_csr_values(const void* h) { return static_cast<const CsrMatrix*>(h)->values.data(); }

int ref_csr_is_canonical(const void* h) { return static_cast<const CsrMatrix*>(h)->is_canonical() ? 1 : 0; }

int ref_gen_erdos_renyi(std::int64_t n, double density, std::uint64_t seed, void** out) {
    return guarded([&] { *out = box(gen_erdos_renyi(n, density, seed)); });
}

int ref_identity(std::int64_t n, void** out) {
    return guarded([&] { *out = box(CsrMatrix::identity(n)); });
}

int ref_from_triplets(std::int64_t nrows, std::int64_t ncols, std::int64_t n, const std::int64_t* rows,
                      const std::int64_t* cols, const double* vals, void** out) {
    return guarded([&] {
        std::vector<Triplet> t(static_cast<std::size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) t[static_cast<std::size_t>(i)] = {rows[i], cols[i], vals[i]};
        *out = box(from_triplets(nrows, ncols, std::move(t)));
    });
}

int ref_permute_random(const void* a, std::uint64_t seed, void** out) {
    return guarded([&] {
        const auto* m = static_cast<const CsrMatrix*>(a);
        *out = box(permute_symmetric(*m, Permutation::random(m->nrows, seed)));
    });
}

int ref_column_normalize(const void* a, void** out) {
    return guarded([&] { *out = box(column_normalize(*static_cast<const CsrMatrix*>(a))); });
}

int ref_result_checksum(const void* a, std::int64_t* nnz, std::uint64_t* hash) {
    return guarded([&] {
        const auto cs = result_checksum(*static_cast<const CsrMatrix*>(a));
        *nnz = cs.nnz;
        *hash = cs.hash;
    });
}

int ref_elementwise_power(const void* a, double r, void** out) {
    return guarded([&] { *out = box(elementwise_power(*static_cast<const CsrMatrix*>(a), r)); });
}

int ref_prune(const void* a, double theta, void** out) {
    return guarded([&] { *out = box(prune(*static_cast<const CsrMatrix*>(a), theta)); });
}

int ref_spgemm_local(const void* a, const void* b, void** out) {
    return guarded([&] {
        *out = box(spgemm_local(*static_cast<const CsrMatrix*>(a), *static_cast<const CsrMatrix*>(b)));
    });
}

// Times one spgemm_local call with std::chrono (the CPU baseline); the
// product is freed unless `out` is non-null.
int ref_spgemm_local_timed(const void* a, const void* b, double* seconds, std::int64_t* nnz_c, void** out) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        CsrMatrix c = spgemm_local(*static_cast<const CsrMatrix*>(a), *static_cast<const CsrMatrix*>(b));
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        *nnz_c = c.nnz();
        if (out) *out = box(std::move(c));
    });
}

int ref_spgeam(const void* a, const void* b, void** out) {
    return guarded([&] {
        *out = box(spgeam(*static_cast<const CsrMatrix*>(a), *static_cast<const CsrMatrix*>(b)));
    });
}

int ref_vconcat(const void* const* slices, int n, void** out) {
    return guarded([&] {
        std::vector<const CsrMatrix*> v;
        for (int i = 0; i < n; ++i) v.push_back(static_cast<const CsrMatrix*>(slices[i]));
        *out = box(vconcat(v));
    });
}

// scheme: 0 trident, 1 grid2d, 2 rows1d. tiles_out must hold `procs` handles;
// rects_out (optional) holds procs*4 int64 (row_begin,row_end,col_begin,col_end).
int ref_partition(const void* a, int scheme, int procs, int gpus_per_node, void** tiles_out,
                  std::int64_t* rects_out) {
    return guarded([&] {
        const Scheme s = scheme == 0 ? Scheme::trident : scheme == 1 ? Scheme::grid2d : Scheme::rows1d;
        PartitionResult pr = partition(*static_cast<const CsrMatrix*>(a), s, procs, gpus_per_node);
        for (int r = 0; r < procs; ++r) {
            tiles_out[r] = box(std::move(pr.tiles[static_cast<std::size_t>(r)]));
            if (rects_out) {
                const TileRect& t = pr.map.tiles[static_cast<std::size_t>(r)];
                rects_out[4 * r + 0] = t.row_begin;
                rects_out[4 * r + 1] = t.row_end;
                rects_out[4 * r + 2] = t.col_begin;
                rects_out[4 * r + 3] = t.col_end;
            }
        }
    });
}

int ref_reassemble(const void* const* tiles, int procs, std::int64_t nrows, std::int64_t ncols, int scheme,
                   int gpus_per_node, void** out) {
    return guarded([&] {
        const Scheme s = scheme == 0 ? Scheme::trident : scheme == 1 ? Scheme::grid2d : Scheme::rows1d;
        std::vector<CsrMatrix> t;
        for (int r = 0; r < procs; ++r) t.push_back(*static_cast<const CsrMatrix*>(tiles[r]));
        *out = box(reassemble(t, make_tile_map(nrows, ncols, s, procs, gpus_per_node)));
    });
}

// algo: 0 trident, 1 summa, 2 oned. ledger_out: procs*2*2*3 uint64 (see dump_ledger).
// events_out (optional): counts per EventType (5 entries).
int ref_run_algo(int algo, const void* a, const void* b, int procs, int gpus_per_node, void** c_out,
                 std::uint64_t* ledger_out, double* makespan, std::int64_t* events_out) {
    return guarded([&] {
        const TopologySpec topo = TopologySpec::preset(0, gpus_per_node);
        const Algo al = algo == 0 ? Algo::trident : algo == 1 ? Algo::summa : Algo::oned;
        DriverResult dr = run_algo(al, *static_cast<const CsrMatrix*>(a), *static_cast<const CsrMatrix*>(b),
                                   procs, gpus_per_node, topo);
        dump_ledger(dr.ledger, procs, ledger_out);
        if (makespan) *makespan = dr.makespan;
        if (events_out) {
            for (int k = 0; k < 5; ++k) events_out[k] = 0;
            for (const auto& e : dr.timeline.events) events_out[static_cast<int>(e.type)]++;
        }
        if (c_out) *c_out = box(std::move(dr.c));
    });
}

// The reference's own dr.timeline.to_jsonl() (engine.cpp:25-41) of run_algo
// (node_start_delay optional, trident only: n_delays entries) into buf (cap
// bytes, NUL-terminated when it fits); *len receives the full length.
int ref_timeline_jsonl(int algo, const void* a, const void* b, int procs, int gpus_per_node, const double* delays,
                       int n_delays, char* buf, std::size_t cap, std::size_t* len) {
    return guarded([&] {
        const TopologySpec topo = TopologySpec::preset(0, gpus_per_node);
        const CsrMatrix& A = *static_cast<const CsrMatrix*>(a);
        const CsrMatrix& B = *static_cast<const CsrMatrix*>(b);
        DriverResult dr;
        if (algo == 0 && n_delays > 0)
            dr = trident_spgemm(A, B, TridentGrid::create(procs, gpus_per_node), topo,
                                std::vector<double>(delays, delays + n_delays));
        else
            dr = run_algo(algo == 0 ? Algo::trident : algo == 1 ? Algo::summa : Algo::oned, A, B, procs,
                          gpus_per_node, topo);
        const std::string j = dr.timeline.to_jsonl();
        *len = j.size();
        if (buf && cap > j.size()) {
            std::memcpy(buf, j.data(), j.size());
            buf[j.size()] = 0;
        }
    });
}

int ref_grid(int procs, int gpus_per_node, int* q) {
    return guarded([&] { *q = TridentGrid::create(procs, gpus_per_node).q; });
}

int ref_predict_volume(std::int64_t nnz, int procs, int gpus_per_node, double* out6) {
    return guarded([&] {
        const VolumePrediction v = predict_trident_volume(nnz, procs, gpus_per_node);
        out6[0] = v.gi_nnz_per_process_per_iter;
        out6[1] = v.li_nnz_per_process_per_iter;
        out6[2] = v.gi_nnz_per_node_total;
        out6[3] = v.summa_gi_nnz_per_process;
        out6[4] = v.gi_nnz_per_process_total_exact;
        out6[5] = v.li_nnz_per_process_total_exact;
    });
}

}  // extern "C"
