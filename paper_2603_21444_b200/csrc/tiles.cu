// Device tile store: the reference's tile map, partition
// and reassemble (partition.cpp:74-261) on the GPUs, so a distributed multiply
// takes ONE host->device copy of each global operand and ONE device->host copy
// of the global C instead of a host-side split / merge (the reference spends
// 1.1 s in partition and 11.5 s in reassemble at n=2^20).
//
//   tile_rects       make_tile_map (partition.cpp:95-159) + block_bounds (:74-81)
//   partition_device partition     (partition.cpp:161-222): one extract per
//                    tile, run on the tile's own device and reading the global
//                    matrix in place (NVLink peer loads when it lives elsewhere)
//   reassemble_device reassemble   (partition.cpp:224-261): a count pass and a
//                    warp-per-row copy pass that walks the row's tiles in
//                    column order, tiles read in place on their devices
//
// Both are pure data movement (HBM-bound): partition reads A once and writes
// the tiles once; reassemble reads every tile once and writes C once.
#include <algorithm>
#include <cmath>

#include "spg_internal.cuh"

namespace spgb {
namespace {

int exact_sqrt(int v) {
    int r = static_cast<int>(std::lround(std::sqrt(static_cast<double>(v))));
    while (r > 0 && r * r > v) --r;
    while ((r + 1) * (r + 1) <= v) ++r;
    return r * r == v ? r : -1;
}

std::vector<int64_t> block_bounds(int64_t dim, int64_t g) {
    std::vector<int64_t> b(static_cast<size_t>(g) + 1, 0);
    const int64_t q = dim / g, extra = dim % g;
    for (int64_t k = 0; k < g; ++k) b[k + 1] = b[k] + q + (k < extra);
    return b;
}

struct TileRef {
    const int64_t* rp;
    const int32_t* col;
    const double* val;
    int64_t r0, c0;
};

__device__ __forceinline__ int slice_of(const int64_t* __restrict__ rb, int ns, int64_t i) {
    int lo = 0, hi = ns;  // last s with rb[s] <= i (empty slices repeat a bound)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rb[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_reasm_count(const TileRef* __restrict__ T, const int64_t* __restrict__ rb,
                              const int32_t* __restrict__ first, int ns, int64_t nrows, int64_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nrows; i += int64_t(gridDim.x) * blockDim.x) {
        const int s = slice_of(rb, ns, i);
        int64_t n = 0;
        for (int t = first[s]; t < first[s + 1]; ++t) {
            const int64_t li = i - T[t].r0;
            n += T[t].rp[li + 1] - T[t].rp[li];
        }
        cnt[i] = n;
    }
}

template <int G>  // G lanes per row
__global__ void __launch_bounds__(256) k_reasm_copy(const TileRef* __restrict__ T, const int64_t* __restrict__ rb,
                                                    const int32_t* __restrict__ first, int ns, int64_t nrows,
                                                    const int64_t* __restrict__ orp, int32_t* __restrict__ ocol,
                                                    double* __restrict__ oval) {
    const int lane = threadIdx.x & (G - 1);
    const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / G;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) / G;
    for (int64_t i = w0; i < nrows; i += nw) {
        const int s = slice_of(rb, ns, i);
        int64_t o = orp[i];
        for (int t = first[s]; t < first[s + 1]; ++t) {
            const TileRef tr = T[t];
            const int64_t li = i - tr.r0, b = tr.rp[li], n = tr.rp[li + 1] - b;
            const int32_t c0 = static_cast<int32_t>(tr.c0);
            for (int64_t u = lane; u < n; u += G) {
                ocol[o + u] = __ldg(tr.col + b + u) + c0;
                oval[o + u] = __ldg(tr.val + b + u);
            }
            o += n;
        }
    }
}

int grid_rows(spg_ctx* ctx, int64_t threads) {
    const int64_t want = (threads + 255) / 256, cap = int64_t(ctx->num_sms) * 16;
    return static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
}

}  // namespace

std::vector<TileRect> tile_rects(int64_t nrows, int64_t ncols, int scheme, int procs, int gpus_per_node) {
    if (procs <= 0) fail(SPG_GRID_ERROR, "partition: process count must be positive");
    if (nrows < 0 || ncols < 0) fail(SPG_DIMENSION_ERROR, "partition: negative matrix shape");
    std::vector<TileRect> t(static_cast<size_t>(procs));
    if (scheme == 0) {  // trident (partition.cpp:40-60, 115-135)
        if (gpus_per_node <= 0) fail(SPG_GRID_ERROR, "trident grid: process and GPU counts must be positive");
        if (procs % gpus_per_node)
            fail(SPG_GRID_ERROR, "trident grid: P=" + std::to_string(procs) + " not divisible by gpus_per_node=" +
                                     std::to_string(gpus_per_node));
        const int q = exact_sqrt(procs / gpus_per_node);
        if (q < 0)
            fail(SPG_GRID_ERROR, "trident grid: P/gpus_per_node=" + std::to_string(procs / gpus_per_node) +
                                     " is not a perfect square");
        const auto coarse = block_bounds(nrows, q), cb = block_bounds(ncols, q);
        std::vector<int64_t> rb{0};
        for (int i = 0; i < q; ++i) {
            const auto fine = block_bounds(coarse[i + 1] - coarse[i], gpus_per_node);
            for (int k = 1; k <= gpus_per_node; ++k) rb.push_back(coarse[i] + fine[k]);
        }
        for (int r = 0; r < procs; ++r) {
            const int node = r / gpus_per_node, i = node / q, j = node % q, k = r % gpus_per_node;
            const int f = i * gpus_per_node + k;
            t[r] = {rb[f], rb[f + 1], cb[j], cb[j + 1]};
        }
    } else if (scheme == 1) {  // grid2d (partition.cpp:136-147)
        const int pr = exact_sqrt(procs);
        if (pr < 0) fail(SPG_GRID_ERROR, "grid2d: P=" + std::to_string(procs) + " is not a perfect square");
        const auto rb = block_bounds(nrows, pr), cb = block_bounds(ncols, pr);
        for (int r = 0; r < procs; ++r) t[r] = {rb[r / pr], rb[r / pr + 1], cb[r % pr], cb[r % pr + 1]};
    } else if (scheme == 2) {  // rows1d (partition.cpp:148-156)
        const auto rb = block_bounds(nrows, procs);
        for (int r = 0; r < procs; ++r) t[r] = {rb[r], rb[r + 1], 0, ncols};
    } else {
        fail(SPG_PARAMETER_ERROR, "partition: unknown scheme " + std::to_string(scheme));
    }
    return t;
}

void partition_device(spg_ctx* const* ctxs, int nctx, const spg_csr* m, int scheme, int procs, int gpus_per_node,
                      spg_csr** out) {
    if (nctx <= 0) fail(SPG_PARAMETER_ERROR, "partition: no contexts");
    const auto rects = tile_rects(m->nrows, m->ncols, scheme, procs, gpus_per_node);
    // The global matrix was produced on its own context's stream.
    SPG_CUDA(cudaStreamSynchronize(m->ctx->stream));
    std::fill(out, out + procs, nullptr);
    try {
        for (int r = 0; r < procs; ++r) {
            spg_ctx* c = ctxs[r % nctx];
            DeviceScope ds(c->device);
            const TileRect& x = rects[r];
            out[r] = extract(c, m, x.r0, x.r1, x.c0, x.c1);  // kernels on c's device, m read in place
        }
        // The extract copies read m in place on every tile's own stream: they
        // must be done before the caller may free m (stream-ordered on m's
        // context, which knows nothing of the other streams) and before a
        // driver pulls the tiles on its transfer streams.
        for (int r = 0; r < std::min(procs, nctx); ++r) {
            DeviceScope ds(ctxs[r]->device);
            SPG_CUDA(cudaStreamSynchronize(ctxs[r]->stream));
        }
    } catch (...) {
        for (int r = 0; r < procs; ++r)
            if (out[r]) free_csr(out[r]), out[r] = nullptr;
        throw;
    }
}

spg_csr* reassemble_device(spg_ctx* ctx, const spg_csr* const* tiles, int ntiles, int64_t nrows, int64_t ncols,
                           int scheme, int procs, int gpus_per_node) {
    if (ntiles != procs)
        fail(SPG_INCOMPLETE_TILE_SET,
             "reassemble: expected " + std::to_string(procs) + " tiles, got " + std::to_string(ntiles));
    const auto rects = tile_rects(nrows, ncols, scheme, procs, gpus_per_node);
    for (int r = 0; r < procs; ++r) {
        if (!tiles[r]) fail(SPG_PARAMETER_ERROR, "null argument: tiles[" + std::to_string(r) + "]");
        if (tiles[r]->nrows != rects[r].r1 - rects[r].r0 || tiles[r]->ncols != rects[r].c1 - rects[r].c0)
            fail(SPG_INCOMPLETE_TILE_SET, "reassemble: tile " + std::to_string(r) + " does not match its map rectangle");
    }
    // Tiles in (row slice, column) order; a slice = the tiles sharing one row
    // range. Zero-row tiles hold nothing (and would share a row start with the
    // next slice), so they are left out.
    std::vector<int> ord;
    for (int r = 0; r < procs; ++r)
        if (rects[r].r1 > rects[r].r0) ord.push_back(r);
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
        return rects[a].r0 != rects[b].r0 ? rects[a].r0 < rects[b].r0 : rects[a].c0 < rects[b].c0;
    });
    std::vector<TileRef> refs;
    std::vector<int64_t> rb;
    std::vector<int32_t> first;
    const int nt = static_cast<int>(ord.size());
    for (int t = 0; t < nt; ++t) {
        const TileRect& x = rects[ord[t]];
        if (t == 0 || x.r0 != rects[ord[t - 1]].r0 || x.r1 != rects[ord[t - 1]].r1) {
            rb.push_back(x.r0);
            first.push_back(t);
        }
        const spg_csr* s = tiles[ord[t]];
        refs.push_back({s->rowptr, s->colind, s->values, x.r0, x.c0});
    }
    first.push_back(nt);
    rb.push_back(nrows);
    if (nt == 0) {  // no rows: a single empty slice
        rb.assign({0, nrows});
        first.assign({0, 0});
        refs.push_back({nullptr, nullptr, nullptr, 0, 0});
    }
    const int ns = static_cast<int>(rb.size()) - 1;
    for (int r = 0; r < procs; ++r)  // tiles were produced on their own streams
        if (tiles[r]->ctx != ctx) SPG_CUDA(cudaStreamSynchronize(tiles[r]->ctx->stream));

    spg_csr* c = new_csr(ctx, nrows, ncols, -1);
    try {
        DBuf<TileRef> dT(ctx, refs.size());
        DBuf<int64_t> drb(ctx, rb.size());
        DBuf<int32_t> dfirst(ctx, first.size());
        SPG_CUDA(cudaMemcpyAsync(dT.p, refs.data(), refs.size() * sizeof(TileRef), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(drb.p, rb.data(), rb.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(dfirst.p, first.data(), first.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        {
            DBuf<int64_t> cnt(ctx, static_cast<size_t>(nrows) + 1);
            KTime kt(ctx, "reassemble_count");
            if (nrows > 0) {
                k_reasm_count<<<grid_rows(ctx, nrows), 256, 0, ctx->stream>>>(dT, drb, dfirst, ns, nrows, cnt);
                SPG_LAUNCH_CHECK();
            }
            exclusive_scan_i64(ctx, cnt, c->rowptr, nrows);
        }
        c->nnz = read_scalar(ctx, c->rowptr + nrows);
        alloc_c_arrays(ctx, c, c->nnz);
        if (c->nnz > 0) {
            KTime kt(ctx, "reassemble_copy");
            if (c->nnz <= 24 * nrows)
                k_reasm_copy<8><<<grid_rows(ctx, nrows * 8), 256, 0, ctx->stream>>>(dT, drb, dfirst, ns, nrows,
                                                                                    c->rowptr, c->colind, c->values);
            else
                k_reasm_copy<32><<<grid_rows(ctx, nrows * 32), 256, 0, ctx->stream>>>(dT, drb, dfirst, ns, nrows,
                                                                                      c->rowptr, c->colind, c->values);
            SPG_LAUNCH_CHECK();
        }
        // the descriptors are freed stream-ordered; the tiles must outlive the copy
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        free_csr(c);
        throw;
    }
    return c;
}

}  // namespace spgb
