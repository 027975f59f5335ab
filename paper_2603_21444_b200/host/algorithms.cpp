// Distributed drivers of the drop-in library (reference algorithms.cpp:24-174):
// each global operand uploaded once and split into tiles on the GPUs of this
// box (spg_partition; rank r -> device r % ndev), the exchange + multiply +
// merge run by the C ABI (spg_trident_spgemm / spg_summa_spgemm), C tiles
// merged on device 0 (spg_reassemble) and downloaded once.
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

enum class Drv { trident, summa, oned };

DriverResult run_device(Drv drv, const CsrMatrix& a, const CsrMatrix& b, Scheme scheme, const TileMap& cmap,
                        int procs, int gpus_per_node, const TopologySpec& topo, int rounds,
                        const std::vector<double>& node_start_delay = {}) {
    const int ndev = detail::device_count();
    const int nctx = std::min(ndev, procs);
    std::vector<spg_ctx*> ctxs(static_cast<std::size_t>(nctx));
    for (int d = 0; d < nctx; ++d) ctxs[static_cast<std::size_t>(d)] = detail::context(d);
    // Device tile store: one upload per global operand, tiles split on the GPUs
    // (spg_partition, rank r on device r % ndev).
    const int plam = scheme == Scheme::trident ? gpus_per_node : 1;
    std::vector<DevCsr> da, db;
    std::vector<const spg_csr*> ha, hb;
    auto split = [&](const CsrMatrix& g, std::vector<DevCsr>& own, std::vector<const spg_csr*>& view) {
        DevCsr dg = detail::upload(ctxs[0], g);
        std::vector<spg_csr*> t(static_cast<std::size_t>(procs), nullptr);
        check(spg_partition(ctxs.data(), nctx, dg.p, static_cast<int>(scheme), procs, plam, t.data()));
        for (auto* h : t) {
            own.emplace_back(h);
            view.push_back(h);
        }
    };
    split(a, da, ha);
    if (&a == &b) {
        hb = ha;
    } else {
        split(b, db, hb);
    }
    std::vector<spg_csr*> hc(static_cast<std::size_t>(procs), nullptr);
    std::vector<spg_ledger_cell> cells(static_cast<std::size_t>(procs) * 4);
    std::vector<double> tl(static_cast<std::size_t>(procs) * rounds * 4, 0.0);
    // events: at most 3 per fetch (2 per rank and round) + allgather + compute
    std::vector<spg_event> ev(static_cast<std::size_t>(procs) * rounds * 8 + 16);
    int nev = 0;
    switch (drv) {
        case Drv::trident:
            check(spg_trident_spgemm_ex(ctxs.data(), nctx, ha.data(), hb.data(), procs, gpus_per_node,
                                        topo.index_width, topo.value_width, node_start_delay.data(),
                                        static_cast<int>(node_start_delay.size()), hc.data(), cells.data(), tl.data(),
                                        ev.data(), static_cast<int>(ev.size()), &nev, nullptr));
            break;
        case Drv::summa:
            check(spg_summa_spgemm_ex(ctxs.data(), nctx, ha.data(), hb.data(), procs, gpus_per_node, topo.index_width,
                                      topo.value_width, hc.data(), cells.data(), tl.data(), ev.data(),
                                      static_cast<int>(ev.size()), &nev, nullptr));
            break;
        case Drv::oned:
            check(spg_oned_spgemm(ctxs.data(), nctx, ha.data(), hb.data(), procs, gpus_per_node, topo.index_width,
                                  topo.value_width, hc.data(), cells.data(), tl.data()));
            nev = -1;
            break;
    }
    std::vector<DevCsr> dc;
    for (auto* h : hc) dc.emplace_back(h);

    DriverResult out;
    out.rounds = rounds;
    {  // C tiles merged on device 0 (spg_reassemble), one download
        std::vector<const spg_csr*> hv;
        for (auto& d : dc) hv.push_back(d.p);
        spg_csr* g = nullptr;
        check(spg_reassemble(ctxs[0], hv.data(), procs, cmap.nrows, cmap.ncols, static_cast<int>(cmap.scheme), procs,
                             plam, &g));
        DevCsr dg(g);
        out.c = detail::download(ctxs[0], dg.p);
    }
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
    // Measured timeline: the device run's events (engine.hpp schema); the
    // 1D driver reports per-rank phase times only.
    if (nev >= 0) {
        std::vector<double> done(static_cast<std::size_t>(procs), 0.0);
        for (int e = 0; e < nev; ++e) {
            const spg_event& x = ev[static_cast<std::size_t>(e)];
            TimelineEvent t{static_cast<EventType>(x.type), x.src, x.dst, x.round,
                            x.operand ? Operand::B : Operand::A, static_cast<LinkClass>(x.link), x.t_start, x.t_end,
                            x.nnz, x.bytes};
            out.timeline.events.push_back(t);
            if (t.type == EventType::compute_complete)
                done[static_cast<std::size_t>(x.src)] = std::max(done[static_cast<std::size_t>(x.src)], x.t_end);
        }
        for (int r = 0; r < procs; ++r) out.ledger.set_completion(r, done[static_cast<std::size_t>(r)]);
    } else {
        for (int r = 0; r < procs; ++r) {
            const double* x = &tl[static_cast<std::size_t>(r) * 4];
            const double t = (x[1] + x[2]) * 1e-3;
            out.timeline.events.push_back({EventType::compute_complete, r, r, 0, Operand::A, LinkClass::SELF, t, t, 0, 0});
            out.ledger.set_completion(r, t);
        }
    }
    out.makespan = out.ledger.makespan();
    return out;
}

}  // namespace

DriverResult trident_spgemm(const CsrMatrix& a, const CsrMatrix& b, const TridentGrid& grid, const TopologySpec& topo,
                            const std::vector<double>& node_start_delay) {
    if (a.ncols != b.nrows)
        throw DimensionError("trident_spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    topo.validate();
    const int P = grid.procs, lam = grid.gpus_per_node;
    const TileMap cmap = make_tile_map(a.nrows, b.ncols, Scheme::trident, P, lam);
    // node_start_delay: virtual node n's ranks start their pulls that many
    // seconds late on the device (engine.cpp:217-221)
    for (double d : node_start_delay)
        if (!(d >= 0.0)) throw ParameterError("trident_spgemm: node_start_delay must be >= 0");
    return run_device(Drv::trident, a, b, Scheme::trident, cmap, P, lam, topo, grid.q, node_start_delay);
}

DriverResult summa_spgemm(const CsrMatrix& a, const CsrMatrix& b, int procs, int gpus_per_node, const TopologySpec& topo) {
    if (a.ncols != b.nrows)
        throw DimensionError("summa_spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    topo.validate();
    const TileMap cmap = make_tile_map(a.nrows, b.ncols, Scheme::grid2d, procs, 1);  // GridError when P is not a square
    int pr = 0;
    while ((pr + 1) * (pr + 1) <= procs) ++pr;
    return run_device(Drv::summa, a, b, Scheme::grid2d, cmap, procs, gpus_per_node, topo, pr);
}

DriverResult oned_spgemm(const CsrMatrix& a, const CsrMatrix& b, int procs, int gpus_per_node, const TopologySpec& topo) {
    if (a.ncols != b.nrows)
        throw DimensionError("oned_spgemm: a.ncols=" + std::to_string(a.ncols) + " != b.nrows=" + std::to_string(b.nrows));
    if (procs <= 0) throw GridError("oned: P must be positive");
    topo.validate();
    const TileMap cmap = make_tile_map(a.nrows, b.ncols, Scheme::rows1d, procs, 1);
    return run_device(Drv::oned, a, b, Scheme::rows1d, cmap, procs, gpus_per_node, topo, 1);
}

DriverResult run_algo(Algo algo, const CsrMatrix& a, const CsrMatrix& b, int procs, int gpus_per_node,
                      const TopologySpec& topo) {
    switch (algo) {
        case Algo::trident: return trident_spgemm(a, b, TridentGrid::create(procs, gpus_per_node), topo);
        case Algo::summa: return summa_spgemm(a, b, procs, gpus_per_node, topo);
        case Algo::oned: return oned_spgemm(a, b, procs, gpus_per_node, topo);
    }
    throw ParameterError("run_algo: bad algorithm");
}

}  // namespace spgsim
