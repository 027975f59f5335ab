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
    int link(int s, int r) const { return s == r ? 0 : (node_of[s] == node_of[r] ? 1 : 2); }  // LinkClass
    spg_ledger_cell& at(int rank, int dir, int c) { return cells[(size_t(rank) * 2 + dir) * 2 + c]; }
    int64_t payload(int64_t rows, int64_t nnz) const { return nnz * (iw + vw) + (rows + 1) * iw; }
    // netmodel.cpp:143-157
    void transfer(int sender, int receiver, int64_t rows, int64_t nnz) {
        if (sender == receiver) return;
        const int c = cls(sender, receiver);
        for (int d = 0; d < 2; ++d) {
            spg_ledger_cell& x = at(d == 0 ? sender : receiver, d, c);
            x.messages += 1;
            x.nnz += uint64_t(nnz);
            x.bytes += uint64_t(payload(rows, nnz));
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

namespace {

struct RoundPlan {
    int a_owner;
    std::vector<int> b_owners;  // slices of the B block, in row order
    std::vector<int> b_slice;   // trident: slice index k' of each (the owner's k); summa: -1
    int s = 0;                  // the k block of the round (A column block, B row block)
};

// One tile a rank consumed: pulled (t0/t1 bracket the copy on its stream) or
// read in place (same device, no copy: t0 = t1 = null).
struct Pull {
    int round = 0, operand = 0, owner = -1, kslice = -1;  // operand 0 A, 1 B
    int64_t rows = 0, nnz = 0, dev_bytes = 0;
    bool copied = false;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    double s0 = 0.0, s1 = 0.0;  // seconds from the rank's start (resolved after the run)
};

// An in-place read is stamped with the time its rank reached it on the copy
// stream (after any start delay).
void stamp(spg_ctx* ctx, cudaStream_t st, Pull& p) {
    p.t0 = ctx->timer.ev();
    p.t1 = ctx->timer.ev();
    SPG_CUDA(cudaEventRecord(p.t0, st));
    SPG_CUDA(cudaEventRecord(p.t1, st));
}

struct RankLog {
    std::vector<Pull> pulls;
    std::vector<double> compute_s;  // per round: end of its multiply (+ merge), seconds from the start
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (a && b) cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// Virtual-node start delay (the reference's node_start_delay skew knob):
// spins on the global timer, so the rank's pulls start that much later.
__global__ void k_spin_delay(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

// Pulls A tile `av` for round r (copy when it lives elsewhere, in place
// otherwise) and logs it. SPG_DEBUG_DOUBLE_PULL=1 (fault injection for the
// ledger tests) makes the first A tile owned by another rank cost one extra,
// redundant device copy that is logged like any pull.
spg_csr* pull_a(spg_ctx* ctx, spg_ctx* cctx, const spg_csr* av, int r, int owner, int rank, bool& owned,
                RankLog* L, bool& injected) {
    const bool local = av->ctx == ctx && av->storage != 2;
    owned = !local;
    Pull p;
    p.round = r;
    p.operand = 0;
    p.owner = owner;
    p.rows = av->nrows;
    p.nnz = av->nnz;
    auto copy = [&]() {
        Pull q = p;
        q.copied = true;
        if (L) {
            q.t0 = ctx->timer.ev();
            q.t1 = ctx->timer.ev();
            q.dev_bytes = (av->nrows + 1) * int64_t(sizeof(int64_t)) + av->nnz * int64_t(sizeof(int32_t) + sizeof(double));
            SPG_CUDA(cudaEventRecord(q.t0, cctx->stream));
        }
        spg_csr* c = copy_csr(cctx, av);
        if (L) {
            SPG_CUDA(cudaEventRecord(q.t1, cctx->stream));
            L->pulls.push_back(q);
        }
        return c;
    };
    static const char* dbg = std::getenv("SPG_DEBUG_DOUBLE_PULL");
    if (dbg && dbg[0] == '1' && !injected && owner != rank) {
        injected = true;
        spg_csr* extra = copy();
        extra->ctx = cctx;
        free_csr(extra);  // stream-ordered on the copy stream
    }
    if (local) {
        if (L) {
            stamp(ctx, cctx->stream, p);
            L->pulls.push_back(p);
        }
        return const_cast<spg_csr*>(av);
    }
    return copy();
}

void log_b(RankLog* L, const RoundPlan& p, int r, const std::vector<SlicePull>& sl, size_t first) {
    if (!L) return;
    for (size_t q = 0; q < p.b_owners.size(); ++q) {
        const SlicePull& x = sl[first + q];
        Pull u;
        u.round = r;
        u.operand = 1;
        u.owner = p.b_owners[q];
        u.kslice = p.b_slice[q];
        u.rows = x.rows;
        u.nnz = x.nnz;
        u.dev_bytes = x.dev_bytes;
        u.copied = true;
        u.t0 = x.t0;
        u.t1 = x.t1;
        L->pulls.push_back(u);
    }
}

// Resolves the logged events into seconds from `base` and returns them to the pool.
void resolve(spg_ctx* ctx, RankLog* L, cudaEvent_t base) {
    if (!L) return;
    for (auto& p : L->pulls) {
        if (p.t0) {
            p.s0 = elapsed(base, p.t0) * 1e-3;
            p.s1 = elapsed(base, p.t1) * 1e-3;
            ctx->timer.pool.push_back(p.t0);
            ctx->timer.pool.push_back(p.t1);
            p.t0 = p.t1 = nullptr;
        }
    }
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
                         const spg_csr* const* b_views, double* tl, int rank, double delay_s, RankLog* L) {
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
    bool injected = false;
    try {
        SPG_CUDA(cudaEventRecord(f0, cs));
        if (delay_s > 0) {
            k_spin_delay<<<1, 1, 0, cs>>>(static_cast<unsigned long long>(delay_s * 1e9));
            SPG_LAUNCH_CHECK();
        }
        std::vector<const spg_csr*> bsl;
        for (int r : ord) {
            bool owned = false;
            a_parts.push_back(pull_a(ctx, &cctx, a_views[plan[r].a_owner], r, plan[r].a_owner, rank, owned, L,
                                     injected));
            a_owned.push_back(owned);
            for (int o : plan[r].b_owners) bsl.push_back(b_views[o]);
        }
        std::vector<SlicePull> slog;
        b_all = vconcat(&cctx, bsl.data(), static_cast<int>(bsl.size()), rp_ready, L ? &slog : nullptr);
        {
            size_t first = 0;
            for (int r : ord) {
                log_b(L, plan[r], r, slog, first);
                first += plan[r].b_owners.size();
            }
        }
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
    if (L) {
        resolve(ctx, L, f0);
        L->compute_s.assign(R, elapsed(f0, e2) * 1e-3);  // one multiply for all rounds
    }
    for (auto e : {f0, ready, e0, e1, e2, rp_ready}) ctx->timer.pool.push_back(e);
    big_cache_release(&cctx);
    return c;
}

spg_csr* run_rank(spg_ctx* ctx, const std::vector<RoundPlan>& plan, const spg_csr* const* a_views,
                  const spg_csr* const* b_views, int64_t c_rows, int64_t c_cols, double* tl /* rounds*4 */,
                  int rank = -1, double delay_s = 0.0, RankLog* L = nullptr) {
    DeviceScope ds(ctx->device);
    // SPG_ROUND_MERGE=1: the reference's structure (multiply per round, merge
    // the partial C tiles), kept for comparison
    const char* me = std::getenv("SPG_ROUND_MERGE");
    const bool merge_rounds = me && me[0] == '1';
    if (plan.size() > 1 && plan.size() <= 16 && !merge_rounds)
        return run_rank_concat(ctx, plan, a_views, b_views, tl, rank, delay_s, L);
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
    cudaEvent_t base = ctx->timer.ev();
    bool injected = false;
    auto issue_fetch = [&](int r) {
        SPG_CUDA(cudaEventRecord(f0[r], cs));
        const RoundPlan& p = plan[r];
        bool owned = false;
        a_in[r] = pull_a(ctx, &cctx, a_views[p.a_owner], r, p.a_owner, rank, owned, L, injected);
        a_owned[r] = owned;
        const spg_csr* b0 = b_views[p.b_owners[0]];
        if (p.b_owners.size() == 1 && b0->ctx == ctx && b0->storage != 2) {
            b_in[r] = const_cast<spg_csr*>(b0);  // read in place
            if (L) {
                Pull u;
                u.round = r;
                u.operand = 1;
                u.owner = p.b_owners[0];
                u.kslice = p.b_slice[0];
                u.rows = b0->nrows;
                u.nnz = b0->nnz;
                stamp(ctx, cs, u);
                L->pulls.push_back(u);
            }
        } else {
            std::vector<const spg_csr*> sl;
            for (int o : p.b_owners) sl.push_back(b_views[o]);
            std::vector<SlicePull> slog;
            b_in[r] = vconcat(&cctx, sl.data(), static_cast<int>(sl.size()), rp[r], L ? &slog : nullptr);
            log_b(L, p, r, slog, 0);
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
        SPG_CUDA(cudaEventRecord(base, cs));
        if (delay_s > 0) {
            k_spin_delay<<<1, 1, 0, cs>>>(static_cast<unsigned long long>(delay_s * 1e9));
            SPG_LAUNCH_CHECK();
        }
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
    if (L) {
        resolve(ctx, L, base);
        L->compute_s.resize(R);
        for (int r = 0; r < R; ++r) L->compute_s[r] = elapsed(base, e3[r]) * 1e-3;
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
    ctx->timer.pool.push_back(base);
    big_cache_release(&cctx);
    cudaStreamSynchronize(cs);
    return acc;
}

// Ledger and events of a driver run from the ranks' logs. Trident routes
// (engine.cpp:228-302 for the plan of algorithms.cpp:53-74): an A tile and
// the rank's own B slice index come from their owners (a control message and
// a transfer each when remote); the other slices of B_{s,j} arrive through the
// node's LI allgather from the node-mate that fetched them. Summa
// (algorithms.cpp:133-160): every remote tile is one transfer, no control.
struct Record {
    std::vector<spg_event> ev;
    void add(int type, int src, int dst, int round, int operand, int link, double t0, double t1, int64_t nnz,
             int64_t bytes) {
        ev.push_back(spg_event{type, src, dst, round, operand, link, t0, t1, nnz, bytes});
    }
};

void book_trident(const GridInfo& g, const std::vector<RankLog>& logs, Ledger& L, Record& E) {
    for (int r = 0; r < g.q; ++r) {
        for (int rank = 0; rank < g.P; ++rank) {
            int i, j, k;
            g.coords(rank, i, j, k);
            for (const Pull& p : logs[rank].pulls) {
                if (p.round != r) continue;
                const bool direct = p.operand == 0 || p.kslice == k;
                if (direct) {
                    if (p.owner == rank) continue;
                    const int64_t by = L.payload(p.rows, p.nnz);
                    L.control(rank, p.owner);
                    L.transfer(p.owner, rank, p.rows, p.nnz);
                    E.add(0, rank, p.owner, r, p.operand, L.link(rank, p.owner), p.s0, p.s0, 0, 0);
                    E.add(1, p.owner, rank, r, p.operand, L.link(p.owner, rank), p.s0, p.s0, 0, 0);
                    E.add(2, p.owner, rank, r, p.operand, L.link(p.owner, rank), p.s0, p.s1, p.nnz, by);
                } else {
                    L.transfer(g.rank_of(i, j, p.kslice), rank, p.rows, p.nnz);  // the node's allgather (LI)
                }
            }
        }
        // one allgather per node and round (every trident round has one)
        for (int node = 0; node < g.q * g.q; ++node) {
            double t0 = 0.0, t1 = 0.0;
            bool any = false;
            int64_t nnz = 0, by = 0;
            for (int k = 0; k < g.lam; ++k) {
                const int rank = node * g.lam + k;
                for (const Pull& p : logs[rank].pulls) {
                    if (p.round != r || p.operand != 1 || p.kslice == k) continue;
                    nnz += p.nnz;
                    by += L.payload(p.rows, p.nnz);
                    t0 = any ? std::min(t0, p.s0) : p.s0;
                    t1 = any ? std::max(t1, p.s1) : p.s1;
                    any = true;
                }
            }
            E.add(3, node, -1, r, 1, 1, t0, t1, nnz, by);
        }
        for (int rank = 0; rank < g.P; ++rank) {
            const double t = r < static_cast<int>(logs[rank].compute_s.size()) ? logs[rank].compute_s[r] : 0.0;
            E.add(4, rank, rank, r, 0, 0, t, t, 0, 0);
        }
    }
}

void book_summa(int P, int pr, const std::vector<RankLog>& logs, Ledger& L, Record& E) {
    for (int r = 0; r < pr; ++r)
        for (int rank = 0; rank < P; ++rank) {
            for (const Pull& p : logs[rank].pulls) {
                if (p.round != r || p.owner == rank) continue;
                L.transfer(p.owner, rank, p.rows, p.nnz);
                E.add(2, p.owner, rank, r, p.operand, L.link(p.owner, rank), p.s0, p.s1, p.nnz,
                      L.payload(p.rows, p.nnz));
            }
            const double t = r < static_cast<int>(logs[rank].compute_s.size()) ? logs[rank].compute_s[r] : 0.0;
            E.add(4, rank, rank, r, 0, 0, t, t, 0, 0);
        }
}

// Per-rank transfer statistics: device bytes pulled, pull span, tiles pulled,
// tiles of other ranks read in place.
void xfer_stats(const std::vector<RankLog>& logs, int rank, double* out) {
    double bytes = 0, n_pull = 0, n_inplace = 0, t0 = 0, t1 = 0;
    bool any = false;
    for (const Pull& p : logs[rank].pulls) {
        if (p.owner == rank) continue;
        if (!p.copied) {
            n_inplace += 1;
            continue;
        }
        bytes += static_cast<double>(p.dev_bytes);
        n_pull += 1;
        t0 = any ? std::min(t0, p.s0) : p.s0;
        t1 = any ? std::max(t1, p.s1) : p.s1;
        any = true;
    }
    out[0] = bytes;
    out[1] = (t1 - t0) * 1e3;
    out[2] = n_pull;
    out[3] = n_inplace;
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
        for (int k2 = 0; k2 < g.lam; ++k2) {
            plan[r].b_owners.push_back(g.rank_of(s, j, k2));
            plan[r].b_slice.push_back(k2);
        }
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

// The tiles may still be in flight on their contexts' streams (partition,
// uploads): every context is drained before the ranks' copy streams read them.
void sync_ctxs(spg_ctx* const* ctxs, int nctx) {
    for (int c = 0; c < nctx; ++c) {
        DeviceScope ds(ctxs[c]->device);
        SPG_CUDA(cudaStreamSynchronize(ctxs[c]->stream));
    }
}

void emit(const Record& E, const Ledger& L, spg_ledger_cell* ledger_out, spg_event* events_out, int events_cap,
          int* n_events) {
    if (ledger_out) std::memcpy(ledger_out, L.cells.data(), L.cells.size() * sizeof(spg_ledger_cell));
    if (n_events) *n_events = static_cast<int>(E.ev.size());
    if (events_out) {
        const size_t n = std::min(E.ev.size(), static_cast<size_t>(std::max(events_cap, 0)));
        std::memcpy(events_out, E.ev.data(), n * sizeof(spg_event));
        if (E.ev.size() > n)
            fail(SPG_PARAMETER_ERROR, "events_out holds " + std::to_string(events_cap) + " events, the run produced " +
                                          std::to_string(E.ev.size()));
    }
}

extern "C" {

spg_status spg_trident_spgemm_ex(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                                 const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                                 int value_width, const double* node_start_delay, int n_delays,
                                 spg_csr** c_tiles_out, spg_ledger_cell* ledger_out, double* timeline_out,
                                 spg_event* events_out, int events_cap, int* n_events, double* xfer_out) {
    return guard2([&] {
        int q = 0;
        const spg_status st = spg_trident_grid(procs, gpus_per_node, &q);
        if (st != SPG_OK) fail(st, spg_last_error());
        check_tiles(ctxs, nctx, a_tiles, b_tiles, procs);
        if (!c_tiles_out) fail(SPG_PARAMETER_ERROR, "null c_tiles_out");
        if (n_delays < 0 || (n_delays > 0 && !node_start_delay)) fail(SPG_PARAMETER_ERROR, "bad node_start_delay");
        for (int d = 0; d < n_delays; ++d)
            if (!(node_start_delay[d] >= 0.0)) fail(SPG_PARAMETER_ERROR, "node_start_delay must be >= 0");
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
        sync_ctxs(ctxs, nctx);
        std::vector<RankLog> logs(procs);
        std::vector<spg_csr*> out(procs, nullptr);
        try {
            for_ranks(procs, nctx, [&](int rank) {
                int i, j, k;
                g.coords(rank, i, j, k);
                const int64_t c_cols = b_tiles[g.rank_of(0, j, 0)]->ncols;
                const int node = rank / gpus_per_node;
                const double delay = node < n_delays ? node_start_delay[node] : 0.0;
                out[rank] = run_rank(ctxs[rank % nctx], trident_plan(g, rank), a_tiles, b_tiles, a_tiles[rank]->nrows,
                                     c_cols, timeline_out ? timeline_out + size_t(rank) * q * 4 : nullptr, rank, delay,
                                     &logs[rank]);
            });
        } catch (...) {
            for (auto* c : out) free_csr(c);
            throw;
        }
        for (int r = 0; r < procs; ++r) c_tiles_out[r] = out[r];
        std::vector<int> nodes(procs);
        for (int r = 0; r < procs; ++r) nodes[r] = r / gpus_per_node;
        Ledger L(procs, nodes, index_width, value_width);
        Record E;
        book_trident(g, logs, L, E);
        if (xfer_out)
            for (int r = 0; r < procs; ++r) xfer_stats(logs, r, xfer_out + size_t(r) * 4);
        emit(E, L, ledger_out, events_out, events_cap, n_events);
    });
}

spg_status spg_trident_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                              const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                              int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                              double* timeline_out) {
    return spg_trident_spgemm_ex(ctxs, nctx, a_tiles, b_tiles, procs, gpus_per_node, index_width, value_width,
                                 nullptr, 0, c_tiles_out, ledger_out, timeline_out, nullptr, 0, nullptr, nullptr);
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

spg_status spg_summa_spgemm_ex(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                               const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                               int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                               double* timeline_out, spg_event* events_out, int events_cap, int* n_events,
                               double* xfer_out) {
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
        sync_ctxs(ctxs, nctx);
        std::vector<RankLog> logs(procs);
        std::vector<spg_csr*> out(procs, nullptr);
        try {
            for_ranks(procs, nctx, [&](int rank) {
                const int i = rank / pr, j = rank % pr;
                std::vector<RoundPlan> plan(pr);
                for (int r = 0; r < pr; ++r) {
                    plan[r].a_owner = i * pr + r;
                    plan[r].b_owners = {r * pr + j};
                    plan[r].b_slice = {-1};
                    plan[r].s = r;
                }
                out[rank] = run_rank(ctxs[rank % nctx], plan, a_tiles, b_tiles, a_tiles[rank]->nrows,
                                     b_tiles[j]->ncols, timeline_out ? timeline_out + size_t(rank) * pr * 4 : nullptr,
                                     rank, 0.0, &logs[rank]);
            });
        } catch (...) {
            for (auto* c : out) free_csr(c);
            throw;
        }
        for (int r = 0; r < procs; ++r) c_tiles_out[r] = out[r];
        std::vector<int> nodes(procs);
        for (int r = 0; r < procs; ++r) nodes[r] = r / gpus_per_node;
        Ledger L(procs, nodes, index_width, value_width);
        Record E;
        book_summa(procs, pr, logs, L, E);
        if (xfer_out)
            for (int r = 0; r < procs; ++r) xfer_stats(logs, r, xfer_out + size_t(r) * 4);
        emit(E, L, ledger_out, events_out, events_cap, n_events);
    });
}

spg_status spg_summa_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                            const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                            int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                            double* timeline_out) {
    return spg_summa_spgemm_ex(ctxs, nctx, a_tiles, b_tiles, procs, gpus_per_node, index_width, value_width,
                               c_tiles_out, ledger_out, timeline_out, nullptr, 0, nullptr, nullptr);
}

}  // extern "C"
