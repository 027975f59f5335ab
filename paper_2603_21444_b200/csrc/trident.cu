// Distributed drivers on one NVSwitch box: trident (reference
// algorithms.cpp:24-101) and Sparse SUMMA (algorithms.cpp:103-174).
//
// Each rank owns its tiles of A and B in its GPU's HBM (read-only for the
// whole run) and its C tile (never moves, the reference's C-stationarity).
// Round r of rank (i,j,k) under the Cannon stagger s = (r+i+j) mod q
// (algorithms.hpp:19-30):
//   * pull A_{i,s,k} from its owner (GI class when remote, free when self),
//   * assemble B_{s,j} = vconcat of the lambda slices B_{s,j,k'}. The
//     reference moves slice k' owner->(i,j,k') over GI and then (i,j,k')->(i,j,k)
//     over LI; on one NVSwitch box every GPU is one hop from every other, so the
//     slice is pulled straight from its owner into its place in B_{s,j}: the
//     bytes each rank receives are identical (1 A tile + lambda B slices), there
//     is no intra-node dependency and no request queue. The ledger still books
//     the reference's GI/LI classes exactly (CommLedger semantics, netmodel.cpp).
//   * C_r = A_{i,s,k} * B_{s,j} (local SpGEMM), acc = spgeam(acc, C_r).
// Round r+1's pulls are issued on a copy stream before round r's multiply, so
// the NVLink transfer overlaps the multiply (double buffering).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "spg_internal.cuh"

using namespace spgb;

namespace spgb {

struct GridInfo {
    int P, lam, q;
    int rank_of(int i, int j, int k) const { return (i * q + j) * lam + k; }
    void coords(int r, int& i, int& j, int& k) const {
        const int node = r / lam;
        i = node / q;
        j = node % q;
        k = r % lam;
    }
};

struct Ledger {
    // [rank][dir][class] ; dir 0 sent 1 received ; class 0 LI 1 GI
    std::vector<spg_ledger_cell> cells;
    std::vector<int> node_of;
    int iw, vw;
    Ledger(int P, std::vector<int> nodes, int iw_, int vw_) : cells(size_t(P) * 4), node_of(std::move(nodes)), iw(iw_), vw(vw_) {}
    int cls(int s, int r) const { return node_of[s] == node_of[r] ? 0 : 1; }
    spg_ledger_cell& at(int rank, int dir, int c) { return cells[(size_t(rank) * 2 + dir) * 2 + c]; }
    uint64_t payload(int64_t rows, int64_t nnz) const { return uint64_t(nnz) * (iw + vw) + uint64_t(rows + 1) * iw; }
    // netmodel.cpp:143-157
    void transfer(int sender, int receiver, int64_t rows, int64_t nnz) {
        if (sender == receiver) return;
        const int c = cls(sender, receiver);
        for (int d = 0; d < 2; ++d) {
            spg_ledger_cell& x = at(d == 0 ? sender : receiver, d, c);
            x.messages += 1;
            x.nnz += uint64_t(nnz);
            x.bytes += payload(rows, nnz);
        }
    }
    // netmodel.cpp:159-163
    void control(int sender, int receiver) {
        if (sender == receiver) return;
        const int c = cls(sender, receiver);
        at(sender, 0, c).messages += 1;
        at(receiver, 1, c).messages += 1;
    }
};

// Reference ledger of trident_spgemm: the engine's request/serve/allgather
// bookkeeping (engine.cpp:228-302) for the plan of algorithms.cpp:53-74.
void trident_ledger(const GridInfo& g, const std::vector<std::pair<int64_t, int64_t>>& a_shape,
                    const std::vector<std::pair<int64_t, int64_t>>& b_shape, Ledger& L) {
    for (int r = 0; r < g.q; ++r) {
        for (int rank = 0; rank < g.P; ++rank) {
            int i, j, k;
            g.coords(rank, i, j, k);
            const int s = (r + i + j) % g.q;
            const int oa = g.rank_of(i, s, k), ob = g.rank_of(s, j, k);
            if (oa != rank) {
                L.control(rank, oa);
                L.transfer(oa, rank, a_shape[oa].first, a_shape[oa].second);
            }
            if (ob != rank) {
                L.control(rank, ob);
                L.transfer(ob, rank, b_shape[ob].first, b_shape[ob].second);
            }
        }
        // allgather inside each node: member k2 contributes the B slice it fetched
        for (int node = 0; node < g.q * g.q; ++node) {
            for (int k = 0; k < g.lam; ++k)
                for (int k2 = 0; k2 < g.lam; ++k2) {
                    if (k == k2) continue;
                    const int recv = node * g.lam + k, send = node * g.lam + k2;
                    int i, j, kk;
                    g.coords(send, i, j, kk);
                    const int s = (r + i + j) % g.q;
                    const int ob = g.rank_of(s, j, kk);
                    L.transfer(send, recv, b_shape[ob].first, b_shape[ob].second);
                }
        }
    }
}

// Reference ledger of summa_spgemm (algorithms.cpp:133-160).
void summa_ledger(int P, int pr, const std::vector<std::pair<int64_t, int64_t>>& a_shape,
                  const std::vector<std::pair<int64_t, int64_t>>& b_shape, Ledger& L) {
    for (int r = 0; r < pr; ++r)
        for (int rank = 0; rank < P; ++rank) {
            const int i = rank / pr, j = rank % pr;
            const int oa = i * pr + r, ob = r * pr + j;
            if (oa != rank) L.transfer(oa, rank, a_shape[oa].first, a_shape[oa].second);
            if (ob != rank) L.transfer(ob, rank, b_shape[ob].first, b_shape[ob].second);
        }
}

namespace {

struct RoundPlan {
    int a_owner;
    std::vector<int> b_owners;  // slices of the B block, in row order
    int s = 0;                  // the k block of the round (A column block, B row block)
};

struct EvPair {
    cudaEvent_t a = nullptr, b = nullptr;
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (a && b) cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// Runs all rounds of one rank on its context. `views[t]` are handles to every
// owner's tile readable from this device (local, peer or IPC-mapped).
// q >= 2 rounds as ONE multiply: the rounds' A tiles side by side in k order,
// [A_{i,0,k} | A_{i,1,k} | ...], times their B blocks stacked in the same
// order. Every C entry is then summed over ascending global k in one pass —
// bit-identical to the serial reference spgemm_local — and the partial-C
// merges (the reference's spgeam per round, algorithms.cpp:82-90) disappear.
// Every tile still moves exactly as the reference schedule moves it (same
// ledger); the pulls of all rounds are issued together on the copy stream.
spg_csr* run_rank_concat(spg_ctx* ctx, const std::vector<RoundPlan>& plan, const spg_csr* const* a_views,
                         const spg_csr* const* b_views, double* tl) {
    const int R = static_cast<int>(plan.size());
    cudaStream_t cs = ctx->xfer;
    spg_ctx cctx = *ctx;
    cctx.stream = cs;
    cctx.big_cache.clear();
    cctx.timer = Timer{};
    std::vector<int> ord(R);
    for (int r = 0; r < R; ++r) ord[r] = r;
    std::sort(ord.begin(), ord.end(), [&](int x, int y) { return plan[x].s < plan[y].s; });
    cudaEvent_t f0 = ctx->timer.ev(), ready = ctx->timer.ev(), e0 = ctx->timer.ev(), e1 = ctx->timer.ev(),
                e2 = ctx->timer.ev(), rp_ready = ctx->timer.ev();
    std::vector<spg_csr*> a_parts;
    std::vector<bool> a_owned;
    spg_csr *a_all = nullptr, *b_all = nullptr, *c = nullptr;
    try {
        SPG_CUDA(cudaEventRecord(f0, cs));
        std::vector<const spg_csr*> bsl;
        for (int r : ord) {
            const spg_csr* av = a_views[plan[r].a_owner];
            const bool local = av->ctx == ctx && av->storage != 2;
            a_parts.push_back(local ? const_cast<spg_csr*>(av) : copy_csr(&cctx, av));
            a_owned.push_back(!local);
            for (int o : plan[r].b_owners) bsl.push_back(b_views[o]);
        }
        b_all = vconcat(&cctx, bsl.data(), static_cast<int>(bsl.size()), rp_ready);
        SPG_CUDA(cudaEventRecord(ready, cs));
        SPG_CUDA(cudaEventRecord(e0, ctx->stream));
        // A tiles and B's row pointers are in place: hconcat and the multiply's
        // row preparation overlap the column/value pulls
        SPG_CUDA(cudaStreamWaitEvent(ctx->stream, rp_ready, 0));
        SPG_CUDA(cudaEventRecord(e1, ctx->stream));
        for (size_t p = 0; p < a_parts.size(); ++p)
            if (a_owned[p]) a_parts[p]->ctx = ctx;  // freed on the compute stream below
        b_all->ctx = ctx;
        a_all = hconcat(ctx, a_parts.data(), R);
        c = spgemm(ctx, a_all, b_all, ready);
        SPG_CUDA(cudaEventRecord(e2, ctx->stream));
        free_csr(a_all);
        free_csr(b_all);
        for (size_t p = 0; p < a_parts.size(); ++p)
            if (a_owned[p]) free_csr(a_parts[p]);
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(cs));
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(cs);
        throw;
    }
    if (tl) {
        for (int r = 0; r < R * 4; ++r) tl[r] = 0.0;
        tl[0] = elapsed(f0, ready);  // pull every round's A tile + assemble B (copy stream)
        tl[1] = elapsed(e0, e1);     // exposed wait (A tiles + B row pointers)
        tl[2] = elapsed(e1, e2);     // hconcat of the A tiles + local multiply (overlaps the B data pulls)
    }
    for (auto e : {f0, ready, e0, e1, e2, rp_ready}) ctx->timer.pool.push_back(e);
    big_cache_release(&cctx);
    return c;
}

spg_csr* run_rank(spg_ctx* ctx, const std::vector<RoundPlan>& plan, const spg_csr* const* a_views,
                  const spg_csr* const* b_views, int64_t c_rows, int64_t c_cols, double* tl /* rounds*4 */) {
    DeviceScope ds(ctx->device);
    // SPG_ROUND_MERGE=1: the reference's structure (multiply per round, merge
    // the partial C tiles), kept for comparison
    const char* me = std::getenv("SPG_ROUND_MERGE");
    const bool merge_rounds = me && me[0] == '1';
    if (plan.size() > 1 && plan.size() <= 16 && !merge_rounds) return run_rank_concat(ctx, plan, a_views, b_views, tl);
    cudaStream_t cs = ctx->xfer;  // persistent transfer stream of the context
    spg_ctx cctx = *ctx;  // same device and pool, copy stream
    cctx.stream = cs;
    cctx.big_cache.clear();  // the block cache belongs to ctx (its stream orders reuse)
    cctx.timer = Timer{};
    const int R = static_cast<int>(plan.size());
    std::vector<spg_csr*> a_in(R, nullptr), b_in(R, nullptr);
    std::vector<bool> a_owned(R, false), b_owned(R, false);
    std::vector<cudaEvent_t> ready(R), e0(R), e1(R), e2(R), e3(R), f0(R), rp(R);
    for (int r = 0; r < R; ++r) {  // events from the context's pool (returned below)
        for (auto* e : {&ready[r], &e0[r], &e1[r], &e2[r], &e3[r], &f0[r], &rp[r]}) *e = ctx->timer.ev();
    }
    auto issue_fetch = [&](int r) {
        SPG_CUDA(cudaEventRecord(f0[r], cs));
        const RoundPlan& p = plan[r];
        const spg_csr* av = a_views[p.a_owner];
        if (av->ctx == ctx && av->storage != 2) a_in[r] = const_cast<spg_csr*>(av);
        else {
            a_in[r] = copy_csr(&cctx, av);
            a_owned[r] = true;
        }
        if (p.b_owners.size() == 1 && b_views[p.b_owners[0]]->ctx == ctx && b_views[p.b_owners[0]]->storage != 2) {
            b_in[r] = const_cast<spg_csr*>(b_views[p.b_owners[0]]);
        } else {
            std::vector<const spg_csr*> sl;
            for (int o : p.b_owners) sl.push_back(b_views[o]);
            b_in[r] = vconcat(&cctx, sl.data(), static_cast<int>(sl.size()), rp[r]);
            b_owned[r] = true;
        }
        if (!b_owned[r]) SPG_CUDA(cudaEventRecord(rp[r], cs));
        // Free on the compute stream once the multiply has consumed them.
        a_in[r]->ctx = a_owned[r] ? ctx : a_in[r]->ctx;
        b_in[r]->ctx = b_owned[r] ? ctx : b_in[r]->ctx;
        SPG_CUDA(cudaEventRecord(ready[r], cs));
    };
    spg_csr* acc = nullptr;
    try {
        issue_fetch(0);
        for (int r = 0; r < R; ++r) {
            if (r + 1 < R) issue_fetch(r + 1);  // overlaps this round's multiply
            SPG_CUDA(cudaEventRecord(e0[r], ctx->stream));
            SPG_CUDA(cudaStreamWaitEvent(ctx->stream, rp[r], 0));  // A + B row pointers
            SPG_CUDA(cudaEventRecord(e1[r], ctx->stream));
            spg_csr* cr = spgemm(ctx, a_in[r], b_in[r], ready[r]);  // waits for B's data after its row prep
            SPG_CUDA(cudaEventRecord(e2[r], ctx->stream));
            if (!acc) acc = cr;
            else {
                spg_csr* z = spgeam(ctx, acc, cr);
                free_csr(acc);
                free_csr(cr);
                acc = z;
            }
            SPG_CUDA(cudaEventRecord(e3[r], ctx->stream));
            if (a_owned[r]) free_csr(a_in[r]);
            if (b_owned[r]) free_csr(b_in[r]);
            a_in[r] = b_in[r] = nullptr;
        }
        if (!acc) acc = new_csr(ctx, c_rows, c_cols, 0);
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(cs));
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(cs);
        throw;
    }
    for (int r = 0; r < R; ++r) {
        if (tl) {
            tl[r * 4 + 0] = elapsed(f0[r], ready[r]);  // pull A + assemble B (copy stream)
            tl[r * 4 + 1] = elapsed(e0[r], e1[r]);     // exposed wait (A + B row pointers)
            tl[r * 4 + 2] = elapsed(e1[r], e2[r]);     // local multiply (overlaps the B data pulls)
            tl[r * 4 + 3] = elapsed(e2[r], e3[r]);     // partial-C merge
        }
        for (auto e : {ready[r], e0[r], e1[r], e2[r], e3[r], f0[r], rp[r]}) ctx->timer.pool.push_back(e);
    }
    big_cache_release(&cctx);
    cudaStreamSynchronize(cs);
    return acc;
}

std::vector<std::pair<int64_t, int64_t>> shapes(const spg_csr* const* t, int P) {
    std::vector<std::pair<int64_t, int64_t>> v(P);
    for (int r = 0; r < P; ++r) v[r] = {t[r]->nrows, t[r]->nnz};
    return v;
}

// Runs `body(rank)` for every rank, one host thread per context (ranks mapped
// rank -> ctxs[rank % nctx], sequential within a context).
void for_ranks(int P, int nctx, const std::function<void(int)>& body) {
    std::vector<std::thread> th;
    std::mutex mu;
    std::exception_ptr err;
    for (int c = 0; c < nctx; ++c)
        th.emplace_back([&, c] {
            try {
                for (int r = c; r < P; r += nctx) body(r);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) err = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    if (err) std::rethrow_exception(err);
}

}  // namespace

std::vector<RoundPlan> trident_plan(const GridInfo& g, int rank) {
    int i, j, k;
    g.coords(rank, i, j, k);
    std::vector<RoundPlan> plan(g.q);
    for (int r = 0; r < g.q; ++r) {
        const int s = (r + i + j) % g.q;
        plan[r].a_owner = g.rank_of(i, s, k);
        plan[r].s = s;
        for (int k2 = 0; k2 < g.lam; ++k2) plan[r].b_owners.push_back(g.rank_of(s, j, k2));
    }
    return plan;
}

}  // namespace spgb

extern "C" spg_status spgb_set_error(spg_status st, const char* msg);

namespace {
template <class F>
spg_status guard2(F&& f) {
    try {
        f();
        return SPG_OK;
    } catch (const StatusError& e) {
        return spgb_set_error(e.code, e.what());
    } catch (const std::exception& e) {
        return spgb_set_error(SPG_ERROR, e.what());
    }
}

void check_tiles(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a, const spg_csr* const* b, int P) {
    if (!ctxs || nctx <= 0) fail(SPG_PARAMETER_ERROR, "no contexts");
    if (!a || !b) fail(SPG_PARAMETER_ERROR, "null tile array");
    for (int r = 0; r < P; ++r) {
        if (!a[r] || !b[r]) fail(SPG_PARAMETER_ERROR, "null tile");
        if (a[r]->ctx != ctxs[r % nctx] || b[r]->ctx != ctxs[r % nctx])
            fail(SPG_PARAMETER_ERROR, "tile of rank " + std::to_string(r) + " does not live on ctxs[rank % nctx]");
    }
}
}  // namespace

extern "C" {

spg_status spg_trident_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                              const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                              int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                              double* timeline_out) {
    return guard2([&] {
        int q = 0;
        const spg_status st = spg_trident_grid(procs, gpus_per_node, &q);
        if (st != SPG_OK) fail(st, spg_last_error());
        check_tiles(ctxs, nctx, a_tiles, b_tiles, procs);
        if (!c_tiles_out) fail(SPG_PARAMETER_ERROR, "null c_tiles_out");
        const GridInfo g{procs, gpus_per_node, q};
        // dimension check: inner blocks must agree (a.ncols == b.nrows globally)
        int64_t a_cols = 0, b_rows = 0;
        for (int j = 0; j < q; ++j) a_cols += a_tiles[g.rank_of(0, j, 0)]->ncols;
        for (int r = 0; r < procs; ++r) {
            int i, j, k;
            g.coords(r, i, j, k);
            if (j == 0) b_rows += b_tiles[r]->nrows;
        }
        if (a_cols != b_rows)
            fail(SPG_DIMENSION_ERROR, "trident_spgemm: a.ncols=" + std::to_string(a_cols) +
                                          " != b.nrows=" + std::to_string(b_rows));
        std::vector<int> nodes(procs);
        for (int r = 0; r < procs; ++r) nodes[r] = r / gpus_per_node;
        Ledger L(procs, nodes, index_width, value_width);
        trident_ledger(g, shapes(a_tiles, procs), shapes(b_tiles, procs), L);
        std::vector<spg_csr*> out(procs, nullptr);
        try {
            for_ranks(procs, nctx, [&](int rank) {
                int i, j, k;
                g.coords(rank, i, j, k);
                const int64_t c_cols = b_tiles[g.rank_of(0, j, 0)]->ncols;
                out[rank] = run_rank(ctxs[rank % nctx], trident_plan(g, rank), a_tiles, b_tiles, a_tiles[rank]->nrows,
                                     c_cols, timeline_out ? timeline_out + size_t(rank) * q * 4 : nullptr);
            });
        } catch (...) {
            for (auto* c : out) free_csr(c);
            throw;
        }
        for (int r = 0; r < procs; ++r) c_tiles_out[r] = out[r];
        if (ledger_out) std::memcpy(ledger_out, L.cells.data(), L.cells.size() * sizeof(spg_ledger_cell));
    });
}

spg_status spg_trident_rank(spg_ctx* ctx, int rank, int procs, int gpus_per_node, const spg_csr* const* a_views,
                            const spg_csr* const* b_views, spg_csr** c_out, double* timeline_out) {
    return guard2([&] {
        int q = 0;
        const spg_status st = spg_trident_grid(procs, gpus_per_node, &q);
        if (st != SPG_OK) fail(st, spg_last_error());
        if (!ctx || !a_views || !b_views || !c_out) fail(SPG_PARAMETER_ERROR, "null argument");
        if (rank < 0 || rank >= procs) fail(SPG_ROUTING_ERROR, "rank outside the grid");
        for (int r = 0; r < procs; ++r)
            if (!a_views[r] || !b_views[r]) fail(SPG_PARAMETER_ERROR, "null tile view");
        const GridInfo g{procs, gpus_per_node, q};
        int i, j, k;
        g.coords(rank, i, j, k);
        *c_out = run_rank(ctx, trident_plan(g, rank), a_views, b_views, a_views[rank]->nrows,
                          b_views[g.rank_of(0, j, 0)]->ncols, timeline_out);
    });
}

spg_status spg_summa_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                            const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                            int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                            double* timeline_out) {
    return guard2([&] {
        if (procs <= 0) fail(SPG_GRID_ERROR, "summa: P must be positive");
        int pr = 0;
        while ((pr + 1) * (pr + 1) <= procs) ++pr;
        if (pr * pr != procs) fail(SPG_GRID_ERROR, "summa: P=" + std::to_string(procs) + " is not a perfect square");
        if (gpus_per_node <= 0) fail(SPG_GRID_ERROR, "gpus_per_node must be positive");
        check_tiles(ctxs, nctx, a_tiles, b_tiles, procs);
        if (!c_tiles_out) fail(SPG_PARAMETER_ERROR, "null c_tiles_out");
        int64_t a_cols = 0, b_rows = 0;
        for (int j = 0; j < pr; ++j) a_cols += a_tiles[j]->ncols;
        for (int i = 0; i < pr; ++i) b_rows += b_tiles[i * pr]->nrows;
        if (a_cols != b_rows)
            fail(SPG_DIMENSION_ERROR, "summa_spgemm: a.ncols=" + std::to_string(a_cols) +
                                          " != b.nrows=" + std::to_string(b_rows));
        std::vector<int> nodes(procs);
        for (int r = 0; r < procs; ++r) nodes[r] = r / gpus_per_node;
        Ledger L(procs, nodes, index_width, value_width);
        summa_ledger(procs, pr, shapes(a_tiles, procs), shapes(b_tiles, procs), L);
        std::vector<spg_csr*> out(procs, nullptr);
        try {
            for_ranks(procs, nctx, [&](int rank) {
                const int i = rank / pr, j = rank % pr;
                std::vector<RoundPlan> plan(pr);
                for (int r = 0; r < pr; ++r) {
                    plan[r].a_owner = i * pr + r;
                    plan[r].b_owners = {r * pr + j};
                    plan[r].s = r;
                }
                out[rank] = run_rank(ctxs[rank % nctx], plan, a_tiles, b_tiles, a_tiles[rank]->nrows,
                                     b_tiles[j]->ncols, timeline_out ? timeline_out + size_t(rank) * pr * 4 : nullptr);
            });
        } catch (...) {
            for (auto* c : out) free_csr(c);
            throw;
        }
        for (int r = 0; r < procs; ++r) c_tiles_out[r] = out[r];
        if (ledger_out) std::memcpy(ledger_out, L.cells.data(), L.cells.size() * sizeof(spg_ledger_cell));
    });
}

}  // extern "C"
