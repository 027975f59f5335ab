// Distributed drivers of the drop-in library (reference algorithms.cpp:24-174):
// partition on the host, tiles uploaded to the GPUs of this box (rank r ->
// device r % ndev), the exchange + multiply + merge run by the C ABI
// (spg_trident_spgemm / spg_summa_spgemm), C tiles downloaded and reassembled.
#include "spgsim/algorithms.hpp"

#include <algorithm>

#include "device.hpp"

namespace spgsim {

using detail::check;
using detail::DevCsr;

const char* algo_name(Algo a) { return a == Algo::trident ? "trident" : a == Algo::summa ? "summa" : "oned"; }

Algo algo_from_name(const std::string& name) {
    if (name == "trident") return Algo::trident;
    if (name == "summa") return Algo::summa;
    if (name == "oned") return Algo::oned;
    throw ParameterError("unknown algorithm '" + name + "'");
}

namespace {

using Driver = spg_status (*)(spg_ctx* const*, int, const spg_csr* const*, const spg_csr* const*, int, int, int, int,
                              spg_csr**, spg_ledger_cell*, double*);

DriverResult run_device(Driver drv, const PartitionResult& pa, const PartitionResult& pb, const TileMap& cmap,
                        int procs, int gpus_per_node, const TopologySpec& topo, int rounds) {
    const int ndev = detail::device_count();
    const int nctx = std::min(ndev, procs);
    std::vector<spg_ctx*> ctxs(static_cast<std::size_t>(nctx));
    for (int d = 0; d < nctx; ++d) ctxs[static_cast<std::size_t>(d)] = detail::context(d);
    std::vector<DevCsr> da, db;
    std::vector<const spg_csr*> ha, hb;
    for (int r = 0; r < procs; ++r) {
        spg_ctx* c = ctxs[static_cast<std::size_t>(r % nctx)];
        da.push_back(detail::upload(c, pa.tiles[static_cast<std::size_t>(r)]));
        db.push_back(detail::upload(c, pb.tiles[static_cast<std::size_t>(r)]));
        ha.push_back(da.back().p);
        hb.push_back(db.back().p);
    }
    std::vector<spg_csr*> hc(static_cast<std::size_t>(procs), nullptr);
    std::vector<spg_ledger_cell> cells(static_cast<std::size_t>(procs) * 4);
    std::vector<double> tl(static_cast<std::size_t>(procs) * rounds * 4, 0.0);
    check(drv(ctxs.data(), nctx, ha.data(), hb.data(), procs, gpus_per_node, topo.index_width, topo.value_width,
              hc.data(), cells.data(), tl.data()));
    std::vector<DevCsr> dc;
    for (auto* h : hc) dc.emplace_back(h);

    DriverResult out;
    out.rounds = rounds;
    std::vector<CsrMatrix> ctiles;
    for (int r = 0; r < procs; ++r) ctiles.push_back(detail::download(ctxs[static_cast<std::size_t>(r % nctx)], dc[static_cast<std::size_t>(r)].p));
    out.c = reassemble(ctiles, cmap);
    std::vector<int> nodes(static_cast<std::size_t>(procs));
    for (int r = 0; r < procs; ++r) nodes[static_cast<std::size_t>(r)] = r / gpus_per_node;
    out.ledger = CommLedger(procs, nodes);
    for (int r = 0; r < procs; ++r)
        for (int d = 0; d < 2; ++d)
            for (int c = 0; c < 2; ++c) {
                const spg_ledger_cell& x = cells[(static_cast<std::size_t>(r) * 2 + d) * 2 + c];
                const LinkClass lc = c == 0 ? LinkClass::LI : LinkClass::GI;
                LedgerCell& y = d == 0 ? out.ledger.sent_cell(r, lc) : out.ledger.received_cell(r, lc);
                y.messages = x.messages;
                y.nnz = x.nnz;
                y.bytes = x.bytes;
            }
    // Measured timeline: per rank and round, exchange then compute (seconds).
    for (int r = 0; r < procs; ++r) {
        double t = 0.0;
        for (int k = 0; k < rounds; ++k) {
            const double* x = &tl[(static_cast<std::size_t>(r) * rounds + k) * 4];
            const double wait = x[1] * 1e-3, mul = x[2] * 1e-3, merge = x[3] * 1e-3;
            out.timeline.events.push_back({EventType::transfer_complete, r, r, k, Operand::B, LinkClass::SELF, t,
                                           t + x[0] * 1e-3, 0, 0});
            t += wait;
            out.timeline.events.push_back({EventType::compute_complete, r, r, k, Operand::A, LinkClass::SELF, t,
                                           t + mul + merge, 0, 0});
            t += mul + merge;
        }
        out.ledger.set_completion(r, t);
    }
    out.makespan = out.ledger.makespan();
    return out;
}

}  // namespace

DriverResult trident_spgemm(const CsrMatrix& a, const CsrMatrix& b, const TridentGrid& grid, const TopologySpec& topo,
                            const std::vector<double>& node_start_delay) {
    (void)node_start_delay;  // skew knob of the modeled clock; real devices start together
    if (a.ncols != b.nrows)
        throw DimensionError("trident_spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    topo.validate();
    const int P = grid.procs, lam = grid.gpus_per_node;
    const PartitionResult pa = partition(a, Scheme::trident, P, lam);
    const PartitionResult pb = partition(b, Scheme::trident, P, lam);
    const TileMap cmap = make_tile_map(a.nrows, b.ncols, Scheme::trident, P, lam);
    return run_device(spg_trident_spgemm, pa, pb, cmap, P, lam, topo, grid.q);
}

DriverResult summa_spgemm(const CsrMatrix& a, const CsrMatrix& b, int procs, int gpus_per_node, const TopologySpec& topo) {
    if (a.ncols != b.nrows)
        throw DimensionError("summa_spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    topo.validate();
    const PartitionResult pa = partition(a, Scheme::grid2d, procs, 1);  // GridError when P is not a square
    const PartitionResult pb = partition(b, Scheme::grid2d, procs, 1);
    const TileMap cmap = make_tile_map(a.nrows, b.ncols, Scheme::grid2d, procs, 1);
    int pr = 0;
    while ((pr + 1) * (pr + 1) <= procs) ++pr;
    return run_device(spg_summa_spgemm, pa, pb, cmap, procs, gpus_per_node, topo, pr);
}

DriverResult run_algo(Algo algo, const CsrMatrix& a, const CsrMatrix& b, int procs, int gpus_per_node,
                      const TopologySpec& topo) {
    switch (algo) {
        case Algo::trident: return trident_spgemm(a, b, TridentGrid::create(procs, gpus_per_node), topo);
        case Algo::summa: return summa_spgemm(a, b, procs, gpus_per_node, topo);
        case Algo::oned: break;
    }
    throw ParameterError("run_algo: the 1D driver is outside the B200 hot path");
}

}  // namespace spgsim
