// One-process-per-GPU support: host pinning and CUDA IPC views of peer tiles
// (the exchange then pulls peer HBM over NVLink with plain device copies).
#include <cstring>

#include "spg_internal.cuh"

using namespace spgb;

extern "C" spg_status spgb_set_error(spg_status st, const char* msg);

namespace {
template <class F>
spg_status guard3(F&& f) {
    try {
        f();
        return SPG_OK;
    } catch (const StatusError& e) {
        return spgb_set_error(e.code, e.what());
    } catch (const std::exception& e) {
        return spgb_set_error(SPG_ERROR, e.what());
    }
}

struct IpcBlob {
    cudaIpcMemHandle_t rowptr, colind, values;
    int64_t nrows, ncols, nnz;
    int32_t device;
};
static_assert(sizeof(IpcBlob) <= 256, "ipc blob");
}  // namespace

extern "C" {

spg_status spg_host_register(void* ptr, size_t bytes) {
    return guard3([&] {
        if (!ptr || !bytes) return;
        SPG_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
    });
}

spg_status spg_host_unregister(void* ptr) {
    return guard3([&] {
        if (!ptr) return;
        SPG_CUDA(cudaHostUnregister(ptr));
    });
}

spg_status spg_csr_make_shareable(spg_ctx* ctx, const spg_csr* m, spg_csr** out) {
    return guard3([&] {
        if (!ctx || !m || !out) fail(SPG_PARAMETER_ERROR, "null argument");
        DeviceScope ds(ctx->device);
        auto* s = new spg_csr;
        s->ctx = ctx;
        s->nrows = m->nrows;
        s->ncols = m->ncols;
        s->nnz = m->nnz;
        s->storage = 1;
        SPG_CUDA(cudaMalloc(&s->rowptr, (m->nrows + 1) * sizeof(int64_t)));
        SPG_CUDA(cudaMalloc(&s->colind, (m->nnz ? m->nnz : 1) * sizeof(int32_t)));
        SPG_CUDA(cudaMalloc(&s->values, (m->nnz ? m->nnz : 1) * sizeof(double)));
        SPG_CUDA(cudaMemcpyAsync(s->rowptr, m->rowptr, (m->nrows + 1) * sizeof(int64_t), cudaMemcpyDefault, ctx->stream));
        if (m->nnz) {
            SPG_CUDA(cudaMemcpyAsync(s->colind, m->colind, m->nnz * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
            SPG_CUDA(cudaMemcpyAsync(s->values, m->values, m->nnz * sizeof(double), cudaMemcpyDefault, ctx->stream));
        }
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = s;
    });
}

spg_status spg_csr_ipc_export(const spg_csr* m, char* out256) {
    return guard3([&] {
        if (!m || !out256) fail(SPG_PARAMETER_ERROR, "null argument");
        if (m->storage != 1) fail(SPG_PARAMETER_ERROR, "ipc export needs spg_csr_make_shareable memory");
        DeviceScope ds(m->ctx->device);
        IpcBlob b{};
        SPG_CUDA(cudaIpcGetMemHandle(&b.rowptr, m->rowptr));
        SPG_CUDA(cudaIpcGetMemHandle(&b.colind, m->colind));
        SPG_CUDA(cudaIpcGetMemHandle(&b.values, m->values));
        b.nrows = m->nrows;
        b.ncols = m->ncols;
        b.nnz = m->nnz;
        b.device = m->ctx->device;
        std::memset(out256, 0, 256);
        std::memcpy(out256, &b, sizeof(b));
    });
}

spg_status spg_csr_ipc_open(spg_ctx* ctx, const char* in256, spg_csr** out) {
    return guard3([&] {
        if (!ctx || !in256 || !out) fail(SPG_PARAMETER_ERROR, "null argument");
        DeviceScope ds(ctx->device);
        IpcBlob b;
        std::memcpy(&b, in256, sizeof(b));
        auto* v = new spg_csr;
        v->ctx = ctx;
        v->nrows = b.nrows;
        v->ncols = b.ncols;
        v->nnz = b.nnz;
        v->storage = 2;
        void* p = nullptr;
        SPG_CUDA(cudaIpcOpenMemHandle(&p, b.rowptr, cudaIpcMemLazyEnablePeerAccess));
        v->rowptr = static_cast<int64_t*>(p);
        SPG_CUDA(cudaIpcOpenMemHandle(&p, b.colind, cudaIpcMemLazyEnablePeerAccess));
        v->colind = static_cast<int32_t*>(p);
        SPG_CUDA(cudaIpcOpenMemHandle(&p, b.values, cudaIpcMemLazyEnablePeerAccess));
        v->values = static_cast<double*>(p);
        *out = v;
    });
}

}  // extern "C"
