// C-ABI entry points of libspgb200.so (include/spg/capi.h). Every function
// catches, records the message in a thread-local buffer and returns a status.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "spg_internal.cuh"

namespace spgb {
void narrow_index(spg_ctx* ctx, const int64_t* d_in, int32_t* d_out, int64_t n);
void widen_index(spg_ctx* ctx, const int32_t* d_in, int64_t* d_out, int64_t n);
}  // namespace spgb

using namespace spgb;

namespace {
thread_local std::string g_last_error;

template <class F>
spg_status guard(F&& f) {
    try {
        f();
        return SPG_OK;
    } catch (const StatusError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SPG_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SPG_ERROR;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(SPG_PARAMETER_ERROR, std::string("null argument: ") + what);
}

void flush_timer(spg_ctx* ctx) {
    auto& t = ctx->timer;
    if (t.pending.empty()) return;
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& r : t.pending) {
        float ms = 0.f;
        SPG_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
        auto& tot = t.totals[r.name];
        tot.first += 1;
        tot.second += ms;
        t.pool.push_back(r.start);
        t.pool.push_back(r.stop);
    }
    t.pending.clear();
}
}  // namespace

// Host <-> device copy in 64 MB chunks spread over the context's copy streams
// (several DMA transfers in flight use the PCIe link better than one), forked
// from and joined back into the context stream.
void copy_chunked(spg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    constexpr size_t CH = size_t(64) << 20;
    if (bytes < 2 * CH || !ctx->aux[0]) {
        SPG_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream));
        return;
    }
    SPG_CUDA(cudaEventRecord(ctx->aux_ev[spg_ctx::NAUX], ctx->stream));
    for (int i = 0; i < spg_ctx::NAUX; ++i) SPG_CUDA(cudaStreamWaitEvent(ctx->aux[i], ctx->aux_ev[spg_ctx::NAUX], 0));
    int c = 0;
    for (size_t off = 0; off < bytes; off += CH, ++c)
        SPG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                                 std::min(CH, bytes - off), kind, ctx->aux[c % spg_ctx::NAUX]));
    for (int i = 0; i < spg_ctx::NAUX; ++i) {
        SPG_CUDA(cudaEventRecord(ctx->aux_ev[i], ctx->aux[i]));
        SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[i], 0));
    }
}

extern "C" {

const char* spg_last_error(void) { return g_last_error.c_str(); }

// Internal: lets other translation units report through the same buffer.
spg_status spgb_set_error(spg_status st, const char* msg) {
    g_last_error = msg ? msg : "";
    return st;
}
const char* spg_version(void) { return "spgb200 0.1 (sm_100a)"; }

spg_status spg_device_count(int* count) {
    return guard([&] {
        need(count, "count");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

spg_status spg_init(int device, spg_ctx** out) {
    return guard([&] {
        need(out, "out");
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            fail(SPG_NO_DEVICE, std::string("no CUDA device available: ") + cudaGetErrorString(e));
        if (device < 0 || device >= n) fail(SPG_PARAMETER_ERROR, "device index out of range");
        DeviceScope ds(device);
        cudaDeviceProp prop{};
        SPG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) fail(SPG_NO_DEVICE, std::string("device is not sm_100 (") + prop.name + ")");
        auto* ctx = new spg_ctx;
        ctx->device = device;
        ctx->num_sms = prop.multiProcessorCount;
        ctx->l2_bytes = prop.l2CacheSize;
        ctx->mem_total = prop.totalGlobalMem;
        ctx_live(device, 1);
        SPG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        for (int i = 0; i < spg_ctx::NAUX; ++i) SPG_CUDA(cudaStreamCreateWithFlags(&ctx->aux[i], cudaStreamNonBlocking));
        SPG_CUDA(cudaStreamCreateWithFlags(&ctx->xfer, cudaStreamNonBlocking));
        for (auto& e : ctx->aux_ev) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        SPG_CUDA(cudaDeviceGetDefaultMemPool(&ctx->pool, device));
        uint64_t keep = UINT64_MAX;  // keep freed blocks cached in the pool
        SPG_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep));
        SPG_CUDA(cudaMallocHost(&ctx->host_scalars, spg_ctx::HOST_SCALAR_BYTES));
        // Peer access to every other device (NVLink P2P for the exchange).
        for (int d = 0; d < n; ++d) {
            if (d == device) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, device, d);
            if (can) {
                const cudaError_t pe = cudaDeviceEnablePeerAccess(d, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) SPG_CUDA(pe);
                cudaGetLastError();
                // Let this device's kernels/copies read allocations of peer pools.
                cudaMemPool_t peer_pool;
                if (cudaDeviceGetDefaultMemPool(&peer_pool, d) == cudaSuccess) {
                    cudaMemAccessDesc desc{};
                    desc.location.type = cudaMemLocationTypeDevice;
                    desc.location.id = device;
                    desc.flags = cudaMemAccessFlagsProtReadWrite;
                    cudaMemPoolSetAccess(peer_pool, &desc, 1);
                    cudaGetLastError();
                }
            }
        }
        *out = ctx;
    });
}

spg_status spg_finalize(spg_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        DeviceScope ds(ctx->device);
        big_cache_release(ctx);
        ctx_live(ctx->device, -1);
        cudaStreamSynchronize(ctx->stream);
        for (auto& r : ctx->timer.pending) {
            cudaEventDestroy(r.start);
            cudaEventDestroy(r.stop);
        }
        for (auto e : ctx->timer.pool) cudaEventDestroy(e);
        cudaFreeHost(ctx->host_scalars);
        for (auto st : ctx->aux) cudaStreamDestroy(st);
        cudaStreamDestroy(ctx->xfer);
        for (auto e : ctx->aux_ev) cudaEventDestroy(e);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

void* spg_ctx_stream(spg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int spg_ctx_device(const spg_ctx* ctx) { return ctx ? ctx->device : -1; }

spg_status spg_ctx_synchronize(spg_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceScope ds(ctx->device);
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

spg_status spg_timing_enable(spg_ctx* ctx, int on) {
    return guard([&] {
        need(ctx, "ctx");
        ctx->timer.on = on != 0;
    });
}

spg_status spg_timing_reset(spg_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceScope ds(ctx->device);
        flush_timer(ctx);
        ctx->timer.totals.clear();
    });
}

int spg_timing_read(spg_ctx* ctx, char* names_out, size_t names_cap, int64_t* launches, double* ms, int cap) {
    int count = -1;
    const spg_status st = guard([&] {
        need(ctx, "ctx");
        DeviceScope ds(ctx->device);
        flush_timer(ctx);
        count = 0;
        size_t off = 0;
        for (auto& kv : ctx->timer.totals) {
            if (count >= cap) break;
            const size_t len = kv.first.size() + 1;
            if (names_out && off + len <= names_cap) {
                std::memcpy(names_out + off, kv.first.c_str(), len);
                off += len;
            }
            if (launches) launches[count] = kv.second.first;
            if (ms) ms[count] = kv.second.second;
            ++count;
        }
    });
    return st == SPG_OK ? count : -1;
}

spg_status spg_csr_upload(spg_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* rowptr, const void* colind,
                          int colind_width, const double* values, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        need(rowptr, "rowptr");
        if (nrows < 0 || ncols < 0) fail(SPG_PARAMETER_ERROR, "negative dimension");
        if (ncols > INT32_MAX) fail(SPG_PARAMETER_ERROR, "ncols exceeds the 32-bit device column index");
        if (colind_width != 4 && colind_width != 8) fail(SPG_PARAMETER_ERROR, "colind_width must be 4 or 8");
        DeviceScope ds(ctx->device);
        const int64_t nnz = rowptr[nrows];
        if (rowptr[0] != 0 || nnz < 0) fail(SPG_ERROR, "rowptr[0] != 0");
        if (nnz) {
            need(colind, "colind");
            need(values, "values");
        }
        spg_csr* m = new_csr(ctx, nrows, ncols, nnz);
        SPG_CUDA(cudaMemcpyAsync(m->rowptr, rowptr, (nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        if (nnz) {
            if (colind_width == 4) {
                copy_chunked(ctx, m->colind, colind, nnz * sizeof(int32_t), cudaMemcpyHostToDevice);
            } else {
                DBuf<int64_t> wide(ctx, nnz);
                SPG_CUDA(cudaMemcpyAsync(wide.get(), colind, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
                try {
                    narrow_index(ctx, wide, m->colind, nnz);
                } catch (...) {
                    free_csr(m);
                    throw;
                }
            }
            copy_chunked(ctx, m->values, values, nnz * sizeof(double), cudaMemcpyHostToDevice);
        }
        *out = m;
    });
}

spg_status spg_csr_zeros(spg_ctx* ctx, int64_t nrows, int64_t ncols, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (nrows < 0 || ncols < 0) fail(SPG_PARAMETER_ERROR, "negative dimension");
        DeviceScope ds(ctx->device);
        *out = new_csr(ctx, nrows, ncols, 0);
    });
}

spg_status spg_csr_shape(const spg_csr* m, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    return guard([&] {
        need(m, "m");
        if (nrows) *nrows = m->nrows;
        if (ncols) *ncols = m->ncols;
        if (nnz) *nnz = m->nnz;
    });
}

spg_status spg_csr_upload_into(spg_ctx* ctx, spg_csr* m, const int64_t* rowptr, const int32_t* colind,
                               const double* values) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        if (m->storage == 2) fail(SPG_PARAMETER_ERROR, "spg_csr_upload_into: read-only IPC view");
        DeviceScope ds(m->ctx->device);
        cudaStream_t st = m->ctx->stream;
        SPG_CUDA(cudaMemcpyAsync(m->rowptr, rowptr, (m->nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        if (m->nnz) {
            copy_chunked(m->ctx, m->colind, colind, m->nnz * sizeof(int32_t), cudaMemcpyHostToDevice);
            copy_chunked(m->ctx, m->values, values, m->nnz * sizeof(double), cudaMemcpyHostToDevice);
        }
        SPG_CUDA(cudaStreamSynchronize(st));
    });
}

spg_status spg_csr_download(spg_ctx* ctx, const spg_csr* m, int64_t* rowptr, void* colind, int colind_width,
                            double* values) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        if (colind_width != 4 && colind_width != 8) fail(SPG_PARAMETER_ERROR, "colind_width must be 4 or 8");
        DeviceScope ds(ctx->device);
        // The matrix may live on another device: stage through this context.
        const spg_csr* src = m;
        spg_csr* tmp = nullptr;
        if (m->ctx->device != ctx->device) src = tmp = copy_csr(ctx, m);
        if (rowptr)
            SPG_CUDA(cudaMemcpyAsync(rowptr, src->rowptr, (src->nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                     ctx->stream));
        if (colind && src->nnz) {
            if (colind_width == 4) {
                copy_chunked(ctx, colind, src->colind, src->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost);
            } else {
                DBuf<int64_t> wide(ctx, src->nnz);
                widen_index(ctx, src->colind, wide, src->nnz);
                SPG_CUDA(cudaMemcpyAsync(colind, wide.get(), src->nnz * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                         ctx->stream));
            }
        }
        if (values && src->nnz) copy_chunked(ctx, values, src->values, src->nnz * sizeof(double), cudaMemcpyDeviceToHost);
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tmp) free_csr(tmp);
    });
}

spg_status spg_csr_check(spg_ctx* ctx, const spg_csr* m) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        DeviceScope ds(ctx->device);
        check_canonical(ctx, m);
    });
}

spg_status spg_csr_free(spg_csr* m) {
    return guard([&] { free_csr(m); });
}

spg_status spg_csr_device_ptrs(const spg_csr* m, void** rowptr, void** colind, void** values) {
    return guard([&] {
        need(m, "m");
        if (rowptr) *rowptr = m->rowptr;
        if (colind) *colind = m->colind;
        if (values) *values = m->values;
    });
}

spg_status spg_spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, spg_csr** c) {
    return guard([&] {
        need(ctx, "ctx");
        need(a, "a");
        need(b, "b");
        need(c, "c");
        DeviceScope ds(ctx->device);
        *c = spgemm(ctx, a, b);
    });
}

spg_status spg_spgemm_products(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, int64_t* products) {
    return guard([&] {
        need(ctx, "ctx");
        need(products, "products");
        DeviceScope ds(ctx->device);
        *products = spgemm_products(ctx, a, b);
    });
}

spg_status spg_spgeam(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, spg_csr** c) {
    return guard([&] {
        need(ctx, "ctx");
        need(a, "a");
        need(b, "b");
        need(c, "c");
        DeviceScope ds(ctx->device);
        *c = spgeam(ctx, a, b);
    });
}

spg_status spg_spgeam_inplace(spg_ctx* ctx, spg_csr** acc, const spg_csr* x) {
    return guard([&] {
        need(ctx, "ctx");
        need(acc, "acc");
        need(*acc, "*acc");
        need(x, "x");
        DeviceScope ds(ctx->device);
        spg_csr* z = spgeam(ctx, *acc, x);
        free_csr(*acc);
        *acc = z;
    });
}

spg_status spg_vconcat(spg_ctx* ctx, const spg_csr* const* slices, int n, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (n > 0) need(slices, "slices");
        DeviceScope ds(ctx->device);
        *out = vconcat(ctx, slices, n);
    });
}

spg_status spg_csr_extract(spg_ctx* ctx, const spg_csr* m, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                           spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        need(out, "out");
        DeviceScope ds(ctx->device);
        *out = extract(ctx, m, r0, r1, c0, c1);
    });
}

spg_status spg_csr_copy(spg_ctx* ctx, const spg_csr* m, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        need(out, "out");
        DeviceScope ds(ctx->device);
        *out = copy_csr(ctx, m);
    });
}

spg_status spg_result_checksum(spg_ctx* ctx, const spg_csr* m, int64_t* nnz, uint64_t* hash) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        need(hash, "hash");
        DeviceScope ds(ctx->device);
        if (nnz) *nnz = m->nnz;
        *hash = result_checksum(ctx, m);
    });
}

spg_status spg_tile_rects(int64_t nrows, int64_t ncols, int scheme, int procs, int gpus_per_node,
                          int64_t* rects_out) {
    return guard([&] {
        need(rects_out, "rects_out");
        const auto r = tile_rects(nrows, ncols, scheme, procs, gpus_per_node);
        for (size_t t = 0; t < r.size(); ++t) {
            rects_out[4 * t + 0] = r[t].r0;
            rects_out[4 * t + 1] = r[t].r1;
            rects_out[4 * t + 2] = r[t].c0;
            rects_out[4 * t + 3] = r[t].c1;
        }
    });
}

spg_status spg_partition(spg_ctx* const* ctxs, int nctx, const spg_csr* m, int scheme, int procs, int gpus_per_node,
                         spg_csr** tiles_out) {
    return guard([&] {
        need(ctxs, "ctxs");
        need(m, "m");
        need(tiles_out, "tiles_out");
        for (int i = 0; i < nctx; ++i) need(ctxs[i], "ctxs[i]");
        partition_device(ctxs, nctx, m, scheme, procs, gpus_per_node, tiles_out);
    });
}

spg_status spg_reassemble(spg_ctx* ctx, const spg_csr* const* tiles, int ntiles, int64_t nrows, int64_t ncols,
                          int scheme, int procs, int gpus_per_node, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (ntiles > 0) need(tiles, "tiles");
        DeviceScope ds(ctx->device);
        *out = reassemble_device(ctx, tiles, ntiles, nrows, ncols, scheme, procs, gpus_per_node);
    });
}

spg_status spg_spgemm_host(spg_ctx* ctx, int64_t a_nrows, int64_t a_ncols, const int64_t* a_rowptr,
                           const void* a_colind, const double* a_values, int64_t b_nrows, int64_t b_ncols,
                           const int64_t* b_rowptr, const void* b_colind, const double* b_values, int colind_width,
                           spg_csr** c) {
    spg_csr *a = nullptr, *b = nullptr;
    // C = A*A (the same host matrix passed twice) uploads it once
    const bool same = a_nrows == b_nrows && a_ncols == b_ncols && a_rowptr == b_rowptr && a_colind == b_colind &&
                      a_values == b_values;
    spg_status st = spg_csr_upload(ctx, a_nrows, a_ncols, a_rowptr, a_colind, colind_width, a_values, &a);
    if (st == SPG_OK && !same)
        st = spg_csr_upload(ctx, b_nrows, b_ncols, b_rowptr, b_colind, colind_width, b_values, &b);
    if (st == SPG_OK) st = spg_spgemm(ctx, a, same ? a : b, c);
    if (a) spg_csr_free(a);
    if (b) spg_csr_free(b);
    return st;
}

spg_status spg_spgemm_host_to_host(spg_ctx* ctx, int64_t a_nrows, int64_t a_ncols, const int64_t* a_rowptr,
                                   const void* a_colind, const double* a_values, int64_t b_nrows, int64_t b_ncols,
                                   const int64_t* b_rowptr, const void* b_colind, const double* b_values,
                                   int colind_width, int batches, int64_t c_cap, int64_t* c_rowptr,
                                   void* c_colind, double* c_values, int64_t* c_nnz) {
    spg_csr *a = nullptr, *b = nullptr;
    const bool same = a_nrows == b_nrows && a_ncols == b_ncols && a_rowptr == b_rowptr && a_colind == b_colind &&
                      a_values == b_values;
    spg_status st = guard([&] {
        need(ctx, "ctx");
        need(c_rowptr, "c_rowptr");
        need(c_nnz, "c_nnz");
        need(a_rowptr, "a_rowptr");
        if (c_cap > 0) {
            need(c_colind, "c_colind");
            need(c_values, "c_values");
        }
        if (colind_width != 4 && colind_width != 8) fail(SPG_PARAMETER_ERROR, "colind_width must be 4 or 8");
        if (a_ncols != b_nrows) fail(SPG_DIMENSION_ERROR, "spgemm_local: inner dimensions differ");
    });
    if (st == SPG_OK) st = spg_csr_upload(ctx, a_nrows, a_ncols, a_rowptr, a_colind, colind_width, a_values, &a);
    if (st == SPG_OK && !same)
        st = spg_csr_upload(ctx, b_nrows, b_ncols, b_rowptr, b_colind, colind_width, b_values, &b);
    if (st == SPG_OK)
        st = guard([&] {
            DeviceScope ds(ctx->device);
            // batch cuts at equal shares of A's entries (host row pointers)
            const int nb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(batches > 0 ? batches : 8,
                                                                                   std::max<int64_t>(1, a_nrows))));
            std::vector<int64_t> cuts(nb + 1, 0);
            const int64_t nnz = a_rowptr[a_nrows];
            for (int i = 1; i < nb; ++i) {
                const int64_t target = nnz / nb * i + (nnz % nb) * i / nb;
                const int64_t r = std::lower_bound(a_rowptr, a_rowptr + a_nrows + 1, target) - a_rowptr;
                cuts[i] = std::max(cuts[i - 1], std::min<int64_t>(r, a_nrows));
            }
            cuts[nb] = a_nrows;
            *c_nnz = spgemm_to_host(ctx, a, same ? a : b, cuts.data(), nb, c_rowptr, c_colind, colind_width,
                                    c_values, c_cap);
            if (*c_nnz > c_cap)
                fail(SPG_PARAMETER_ERROR, "spgemm_host_to_host: nnz(C)=" + std::to_string(*c_nnz) +
                                              " exceeds c_cap=" + std::to_string(c_cap));
        });
    if (a) spg_csr_free(a);
    if (b) spg_csr_free(b);
    return st;
}

spg_status spg_column_normalize(spg_ctx* ctx, spg_csr* m) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        DeviceScope ds(ctx->device);
        column_normalize(ctx, m);
    });
}

spg_status spg_prune(spg_ctx* ctx, const spg_csr* m, double threshold, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        need(out, "out");
        DeviceScope ds(ctx->device);
        *out = prune(ctx, m, threshold);
    });
}

spg_status spg_elementwise_power(spg_ctx* ctx, spg_csr* m, double exponent) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "m");
        DeviceScope ds(ctx->device);
        elementwise_power(ctx, m, exponent);
    });
}

spg_status spg_mcl_poststep(spg_ctx* ctx, const spg_csr* c, double prune_threshold, double inflation, spg_csr** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(c, "c");
        need(out, "out");
        DeviceScope ds(ctx->device);
        *out = mcl_poststep(ctx, c, prune_threshold, inflation);
    });
}

spg_status spg_trident_grid(int procs, int gpus_per_node, int* q) {
    return guard([&] {
        need(q, "q");
        if (procs <= 0 || gpus_per_node <= 0)
            fail(SPG_GRID_ERROR, "trident grid: process and GPU counts must be positive");
        if (procs % gpus_per_node != 0)
            fail(SPG_GRID_ERROR, "trident grid: P=" + std::to_string(procs) + " not divisible by gpus_per_node=" +
                                     std::to_string(gpus_per_node));
        const int v = procs / gpus_per_node;
        int r = 0;
        while ((r + 1) * (r + 1) <= v) ++r;
        if (r * r != v)
            fail(SPG_GRID_ERROR, "trident grid: P/gpus_per_node=" + std::to_string(v) + " is not a perfect square");
        *q = r;
    });
}

}  // extern "C"
