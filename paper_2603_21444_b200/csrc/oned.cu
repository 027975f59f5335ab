// Sparsity-aware 1D driver: the reference's oned_spgemm
// (algorithms.cpp:176-269) on the GPUs of this box. Ranks own rows1d blocks
// of A and B. Rank p needs the B rows named by the distinct columns of its A
// block; it pulls exactly those rows from their owners' HBM (read in place
// over NVLink by a gather kernel on p's device — the row-selective fetch the
// reference models), stacks them with its own block into the K x n "gathered"
// operand the reference builds (rows nobody asked for stay empty), and runs
// the same local multiply as the other drivers.
//
// Per rank, on its own device and stream:
//   k_oned_mark    flag[k] = 1 for every column k of A_p            (A_p read once)
//   k_oned_need    per row k of B: gathered length (own or flagged), and per
//                  owner the number of remote rows / nnz fetched (the ledger)
//   scan           gathered rowptr
//   k_oned_gather  copy of the kept rows from their owners' tiles (8 lanes/row)
//   spgemm         C_p = A_p * gathered
#include <algorithm>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "spg_internal.cuh"

using namespace spgb;

namespace {

struct BTile {
    const int64_t* rp;
    const int32_t* col;
    const double* val;
};

__device__ __forceinline__ int owner_of(const int64_t* __restrict__ bb, int P, int64_t k) {
    int lo = 0, hi = P;  // last o with bb[o] <= k
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bb[mid] <= k) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_oned_mark(const int32_t* __restrict__ col, int64_t nnz, uint8_t* __restrict__ flag) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nnz; t += int64_t(gridDim.x) * blockDim.x)
        flag[col[t]] = 1;
}

// stats[2*o] = remote rows fetched from owner o, stats[2*o+1] = their nnz
__global__ void k_oned_need(const BTile* __restrict__ T, const int64_t* __restrict__ bb, int P, int self, int64_t K,
                            const uint8_t* __restrict__ flag, int64_t* __restrict__ len,
                            unsigned long long* __restrict__ stats) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) & ~int64_t(31); base < K; base += stride) {
        const int64_t k = base + lane;
        int o = -1;
        int64_t n = 0;
        bool remote = false;
        if (k < K) {
            o = owner_of(bb, P, k);
            const bool want = flag[k] != 0;
            if (o == self || want) {
                const int64_t lr = k - bb[o];
                n = T[o].rp[lr + 1] - T[o].rp[lr];
            }
            remote = want && o != self;
            len[k] = o == self || want ? n : 0;
        }
        const int o0 = __shfl_sync(FULL, o, 0);
        if (__all_sync(FULL, o == o0 || k >= K)) {  // one owner for the warp: reduce, one atomic
            unsigned long long rows = remote ? 1ull : 0ull, nz = remote ? static_cast<unsigned long long>(n) : 0ull;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                rows += __shfl_xor_sync(FULL, rows, s);
                nz += __shfl_xor_sync(FULL, nz, s);
            }
            if (lane == 0 && rows) {
                atomicAdd(stats + 2 * o0, rows);
                atomicAdd(stats + 2 * o0 + 1, nz);
            }
        } else if (remote) {
            atomicAdd(stats + 2 * o, 1ull);
            atomicAdd(stats + 2 * o + 1, static_cast<unsigned long long>(n));
        }
    }
}

__global__ void __launch_bounds__(256) k_oned_gather(const BTile* __restrict__ T, const int64_t* __restrict__ bb,
                                                     int P, int64_t K, const int64_t* __restrict__ grp,
                                                     int32_t* __restrict__ gcol, double* __restrict__ gval) {
    constexpr int G = 8;
    const int lane = threadIdx.x & (G - 1);
    const int64_t g0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / G;
    const int64_t ng = (int64_t(gridDim.x) * blockDim.x) / G;
    for (int64_t k = g0; k < K; k += ng) {
        const int64_t o = grp[k], n = grp[k + 1] - o;
        if (n == 0) continue;
        const int w = owner_of(bb, P, k);
        const BTile t = T[w];
        const int64_t s = t.rp[k - bb[w]];
        for (int64_t u = lane; u < n; u += G) {
            gcol[o + u] = __ldg(t.col + s + u);
            gval[o + u] = __ldg(t.val + s + u);
        }
    }
}

int grid_n(spg_ctx* ctx, int64_t threads) {
    const int64_t want = (threads + 255) / 256, cap = int64_t(ctx->num_sms) * 16;
    return static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
}

// One rank: gathered operand + local multiply on ctx. stats_out: 2*P counts.
spg_csr* oned_rank(spg_ctx* ctx, int p, int P, const spg_csr* const* a, const spg_csr* const* b,
                   const std::vector<int64_t>& bb, unsigned long long* stats_out, double* tl) {
    DeviceScope ds(ctx->device);
    const spg_csr* ap = a[p];
    const int64_t K = bb[P], n = b[0]->ncols;
    std::vector<BTile> ht(P);
    for (int o = 0; o < P; ++o) ht[o] = {b[o]->rowptr, b[o]->colind, b[o]->values};
    cudaEvent_t e0 = ctx->timer.ev(), e1 = ctx->timer.ev(), e2 = ctx->timer.ev();
    SPG_CUDA(cudaEventRecord(e0, ctx->stream));
    spg_csr* g = new_csr(ctx, K, n, -1);
    try {
        DBuf<BTile> dT(ctx, P);
        DBuf<int64_t> dbb(ctx, P + 1), len(ctx, K + 1);
        DBuf<uint8_t> flag(ctx, K + 1);
        DBuf<unsigned long long> st(ctx, 2 * P);
        SPG_CUDA(cudaMemcpyAsync(dT.p, ht.data(), P * sizeof(BTile), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(dbb.p, bb.data(), (P + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemsetAsync(flag.p, 0, K + 1, ctx->stream));
        SPG_CUDA(cudaMemsetAsync(st.p, 0, 2 * P * sizeof(unsigned long long), ctx->stream));
        {
            KTime kt(ctx, "oned_gather");
            if (ap->nnz) k_oned_mark<<<grid_n(ctx, ap->nnz), 256, 0, ctx->stream>>>(ap->colind, ap->nnz, flag);
            if (K) k_oned_need<<<grid_n(ctx, K), 256, 0, ctx->stream>>>(dT, dbb, P, p, K, flag, len, st);
            SPG_LAUNCH_CHECK();
            exclusive_scan_i64(ctx, len, g->rowptr, K);
            SPG_CUDA(cudaMemcpyAsync(stats_out, st.p, 2 * P * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            g->nnz = read_scalar(ctx, g->rowptr + K);  // synchronizes: stats_out is ready too
            alloc_c_arrays(ctx, g, g->nnz);
            if (g->nnz)
                k_oned_gather<<<grid_n(ctx, K * 8), 256, 0, ctx->stream>>>(dT, dbb, P, K, g->rowptr, g->colind,
                                                                           g->values);
            SPG_LAUNCH_CHECK();
        }
        SPG_CUDA(cudaEventRecord(e1, ctx->stream));
        spg_csr* c = spgemm(ctx, ap, g);
        SPG_CUDA(cudaEventRecord(e2, ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tl) {
            float f = 0.f, m = 0.f;
            cudaEventElapsedTime(&f, e0, e1);
            cudaEventElapsedTime(&m, e1, e2);
            tl[0] = f;    // exchange: row-selective pull of the needed B rows
            tl[1] = f;    // exposed (nothing overlaps it in one round)
            tl[2] = m;    // local multiply
            tl[3] = 0.0;  // no merge
        }
        free_csr(g);
        ctx->timer.pool.push_back(e0);
        ctx->timer.pool.push_back(e1);
        ctx->timer.pool.push_back(e2);
        return c;
    } catch (...) {
        free_csr(g);
        throw;
    }
}

}  // namespace

extern "C" spg_status spgb_set_error(spg_status st, const char* msg);

extern "C" spg_status spg_oned_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                                      const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                                      int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                                      double* timeline_out) {
    try {
        if (procs <= 0) fail(SPG_GRID_ERROR, "oned: P must be positive");
        if (gpus_per_node <= 0) fail(SPG_GRID_ERROR, "gpus_per_node must be positive");
        if (!ctxs || nctx <= 0 || !a_tiles || !b_tiles || !c_tiles_out) fail(SPG_PARAMETER_ERROR, "null argument");
        for (int r = 0; r < procs; ++r) {
            if (!a_tiles[r] || !b_tiles[r]) fail(SPG_PARAMETER_ERROR, "null tile");
            if (a_tiles[r]->ctx != ctxs[r % nctx] || b_tiles[r]->ctx != ctxs[r % nctx])
                fail(SPG_PARAMETER_ERROR, "tile of rank " + std::to_string(r) + " does not live on ctxs[rank % nctx]");
        }
        // rows1d blocks: A tiles are full-width row blocks, B tiles the row
        // blocks of the inner dimension (partition.cpp:148-156)
        std::vector<int64_t> bb(procs + 1, 0);
        for (int r = 0; r < procs; ++r) bb[r + 1] = bb[r] + b_tiles[r]->nrows;
        const int64_t K = a_tiles[0]->ncols;
        if (K != bb[procs])
            fail(SPG_DIMENSION_ERROR,
                 "oned_spgemm: a.ncols=" + std::to_string(K) + " != b.nrows=" + std::to_string(bb[procs]));
        for (int r = 0; r < procs; ++r)
            if (a_tiles[r]->ncols != K || b_tiles[r]->ncols != b_tiles[0]->ncols)
                fail(SPG_DIMENSION_ERROR, "oned_spgemm: tiles are not rows1d blocks of one matrix");
        if (K >= (int64_t(1) << 31)) fail(SPG_PARAMETER_ERROR, "oned_spgemm: inner dimension exceeds 2^31");
        for (int c = 0; c < nctx; ++c) SPG_CUDA(cudaStreamSynchronize(ctxs[c]->stream));

        std::vector<unsigned long long> stats(size_t(procs) * 2 * procs, 0);
        std::vector<spg_csr*> out(procs, nullptr);
        std::vector<std::thread> th;
        std::mutex mu;
        std::exception_ptr err;
        for (int c = 0; c < nctx && c < procs; ++c)
            th.emplace_back([&, c] {
                try {
                    for (int r = c; r < procs; r += nctx)
                        out[r] = oned_rank(ctxs[c], r, procs, a_tiles, b_tiles, bb, &stats[size_t(r) * 2 * procs],
                                           timeline_out ? timeline_out + size_t(r) * 4 : nullptr);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err) err = std::current_exception();
                }
            });
        for (auto& t : th) t.join();
        if (err) {
            for (auto* x : out) free_csr(x);
            std::rethrow_exception(err);
        }
        // Reference ledger (engine.cpp:228-302 for the plan of
        // algorithms.cpp:211-227): one request + one transfer of
        // (rows, nnz) per (rank, owner) with a nonempty needed set.
        std::vector<spg_ledger_cell> cells(size_t(procs) * 4);
        auto at = [&](int rank, int dir, int cls) -> spg_ledger_cell& { return cells[(size_t(rank) * 2 + dir) * 2 + cls]; };
        const auto cls = [&](int s, int r) { return s / gpus_per_node == r / gpus_per_node ? 0 : 1; };
        for (int p = 0; p < procs; ++p)
            for (int o = 0; o < procs; ++o) {
                const unsigned long long rows = stats[(size_t(p) * procs + o) * 2];
                const unsigned long long nz = stats[(size_t(p) * procs + o) * 2 + 1];
                if (o == p || rows == 0) continue;
                const int c = cls(o, p);
                at(p, 0, c).messages += 1;  // request p -> o
                at(o, 1, c).messages += 1;
                const uint64_t bytes = nz * uint64_t(index_width + value_width) + (rows + 1) * uint64_t(index_width);
                for (int d = 0; d < 2; ++d) {  // payload o -> p
                    spg_ledger_cell& x = at(d == 0 ? o : p, d, c);
                    x.messages += 1;
                    x.nnz += nz;
                    x.bytes += bytes;
                }
            }
        for (int r = 0; r < procs; ++r) c_tiles_out[r] = out[r];
        if (ledger_out) std::memcpy(ledger_out, cells.data(), cells.size() * sizeof(spg_ledger_cell));
        return SPG_OK;
    } catch (const StatusError& e) {
        return spgb_set_error(e.code, e.what());
    } catch (const std::exception& e) {
        return spgb_set_error(SPG_ERROR, e.what());
    }
}
