#include "device.hpp"

#include <mutex>
#include <string>

namespace spgsim::detail {

void throw_status(spg_status st) {
    const std::string msg = spg_last_error();
    switch (st) {
        case SPG_DIMENSION_ERROR: throw DimensionError(msg);
        case SPG_PARAMETER_ERROR: throw ParameterError(msg);
        case SPG_GRID_ERROR: throw GridError(msg);
        case SPG_INCOMPLETE_TILE_SET: throw IncompleteTileSet(msg);
        case SPG_ROUTING_ERROR: throw RoutingError(msg);
        case SPG_SCHEDULE_ERROR: throw ScheduleError(msg);
        case SPG_DEADLOCK_ERROR: throw DeadlockError(msg);
        case SPG_CUDA_ERROR:
        case SPG_OOM:
        case SPG_NO_DEVICE: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

namespace {
std::mutex g_mu;
std::vector<spg_ctx*> g_ctx;
int g_count = -1;
}  // namespace

int device_count() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_count < 0) {
        int n = 0;
        check(spg_device_count(&n));
        g_count = n;
        g_ctx.assign(static_cast<std::size_t>(n), nullptr);
    }
    if (g_count == 0) throw DeviceError("no CUDA device: the spgsim B200 library has no CPU fallback");
    return g_count;
}

spg_ctx* context(int device) {
    const int n = device_count();
    if (device < 0 || device >= n) throw ParameterError("device index out of range");
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx[static_cast<std::size_t>(device)]) check(spg_init(device, &g_ctx[static_cast<std::size_t>(device)]));
    return g_ctx[static_cast<std::size_t>(device)];
}

DevCsr upload(spg_ctx* ctx, const CsrMatrix& m) {
    if (m.rowptr.size() != static_cast<std::size_t>(m.nrows) + 1) throw Error("rowptr length != nrows+1");
    spg_csr* h = nullptr;
    check(spg_csr_upload(ctx, m.nrows, m.ncols, m.rowptr.data(), m.colind.data(), 8, m.values.data(), &h));
    return DevCsr(h);
}

CsrMatrix download(spg_ctx* ctx, const spg_csr* h) {
    CsrMatrix m;
    index_t nnz = 0;
    check(spg_csr_shape(h, &m.nrows, &m.ncols, &nnz));
    m.rowptr.resize(static_cast<std::size_t>(m.nrows) + 1);
    m.colind.resize(static_cast<std::size_t>(nnz));
    m.values.resize(static_cast<std::size_t>(nnz));
    check(spg_csr_download(ctx, h, m.rowptr.data(), m.colind.data(), 8, m.values.data()));
    return m;
}

}  // namespace spgsim::detail
