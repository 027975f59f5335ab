// Internal definitions shared by the CUDA translation units of libspgb200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "spg/capi.h"

namespace spgb {

struct StatusError : std::runtime_error {
    spg_status code;
    StatusError(spg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(spg_status c, const std::string& m) { throw StatusError(c, m); }

#define SPG_CUDA(call)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            ::spgb::fail(e_ == cudaErrorMemoryAllocation ? SPG_OOM : SPG_CUDA_ERROR,                \
                         std::string(#call) + " failed: " + cudaGetErrorString(e_) + " (" __FILE__ \
                         ":" + std::to_string(__LINE__) + ")");                                     \
    } while (0)

#define SPG_LAUNCH_CHECK() SPG_CUDA(cudaGetLastError())

// Per-kernel CUDA-event timing on the context stream.
struct Timer {
    struct Rec {
        std::string name;
        cudaEvent_t start, stop;
    };
    bool on = false;
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<int64_t, double>> totals;

    cudaEvent_t ev() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        SPG_CUDA(cudaEventCreate(&e));
        return e;
    }
};

}  // namespace spgb

struct spg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool = nullptr;
    int num_sms = 148;
    size_t l2_bytes = 0;
    spgb::Timer timer;
    // Pinned host staging for small scalar read-backs.
    static constexpr int HOST_SCALAR_BYTES = 256;
    int64_t* host_scalars = nullptr;
    // fork/join streams for concurrent slice copies (vconcat pulls from several peers at once)
    static constexpr int NAUX = 4;
    cudaStream_t aux[NAUX] = {};
    cudaStream_t xfer = nullptr;  // trident rounds: tile pulls of the next round
    cudaEvent_t aux_ev[NAUX + 1] = {};
    // Large C arrays (>= 256 MB) come from this block cache instead of the pool:
    // the pool splits freed blocks for smaller requests, after which a
    // multi-GB request maps fresh memory on every call (see big_alloc).
    std::vector<std::pair<void*, size_t>> big_cache;
    size_t mem_total = 0;  // device memory (sizes the block cache)
};

struct spg_csr {
    spg_ctx* ctx = nullptr;  // owning context (device + pool)
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int64_t* rowptr = nullptr;  // nrows+1
    int32_t* colind = nullptr;  // nnz
    double* values = nullptr;   // nnz
    // Storage kind: 0 = stream-ordered pool (default), 1 = cudaMalloc (IPC
    // exportable), 2 = IPC view of a peer process's matrix (read-only).
    int storage = 0;
    size_t big_col = 0, big_val = 0;  // capacities (bytes) of colind/values taken from ctx->big_cache
};

namespace spgb {

// RAII scope that binds the context's device.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        SPG_CUDA(cudaGetDevice(&prev));
        if (prev != dev) SPG_CUDA(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Stream-ordered pool allocation; on OOM the context's block cache and the
// pool's cached memory are released and the allocation retried once.
void* pool_alloc(spg_ctx* ctx, size_t bytes);

template <class T>
T* dalloc(spg_ctx* ctx, size_t n) {
    if (n == 0) n = 1;
    return static_cast<T*>(pool_alloc(ctx, n * sizeof(T)));
}

inline void dfree(spg_ctx* ctx, void* p) {
    if (p) cudaFreeAsync(p, ctx->stream);
}

void* big_alloc(spg_ctx* ctx, size_t bytes, size_t* cap);
void big_free(spg_ctx* ctx, void* p, size_t cap);
constexpr size_t BIG_BYTES = size_t(256) << 20;

// Stream-ordered scratch buffer freed at scope exit (>= 256 MB: block cache).
template <class T>
struct DBuf {
    spg_ctx* ctx;
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DBuf(spg_ctx* c, size_t count) : ctx(c), n(count) {
        if (count * sizeof(T) >= BIG_BYTES) p = static_cast<T*>(big_alloc(c, count * sizeof(T), &cap));
        else p = dalloc<T>(c, count);
    }
    ~DBuf() {
        if (cap) big_free(ctx, p, cap);
        else dfree(ctx, p);
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    T* get() const { return p; }
    operator T*() const { return p; }
};

// Kernel timing bracket: records events around a launch when timing is enabled.
struct KTime {
    spg_ctx* ctx;
    const char* name;
    cudaEvent_t s = nullptr, e = nullptr;
    KTime(spg_ctx* c, const char* n) : ctx(c), name(n) {
        if (ctx->timer.on) {
            s = ctx->timer.ev();
            e = ctx->timer.ev();
            cudaEventRecord(s, ctx->stream);
        }
    }
    ~KTime() {
        if (s) {
            cudaEventRecord(e, ctx->stream);
            ctx->timer.pending.push_back({name, s, e});
        }
    }
};

spg_csr* new_csr(spg_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz);
void free_csr(spg_csr* m);
// colind/values of a new product with room for `cap` entries (big arrays via the block cache).
void alloc_c_arrays(spg_ctx* ctx, spg_csr* c, int64_t cap);
void big_cache_release(spg_ctx* ctx);
// live contexts per device (the block cache's byte budget is shared among them)
void ctx_live(int device, int delta);
int64_t read_scalar(spg_ctx* ctx, const int64_t* dptr);
// Enqueue a kernel copy of `bytes` device bytes into the context's pinned
// scalars at byte offset `off` (slot 0-7 belongs to read_scalar); returns the
// host address, valid after the next synchronisation of ctx->stream.
void* peek_async(spg_ctx* ctx, int off, const void* dsrc, int bytes);

// Kernels (spgemm.cu / spgeam.cu / misc.cu)
// b_data: when set, B's column/value arrays are complete only at this event
// (its row pointers and A are ready): the symbolic preparation overlaps the pull.
spg_csr* spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, cudaEvent_t b_data = nullptr);
int64_t spgemm_products(spg_ctx* ctx, const spg_csr* a, const spg_csr* b);
spg_csr* spgeam(spg_ctx* ctx, const spg_csr* a, const spg_csr* b);
// rp_ready (optional): recorded once the row pointers are assembled; the
// column/value pulls may still be running on the aux streams then.
// One slice pull of vconcat, for the exchange log: t0/t1 bracket its copies
// on the stream that ran them (pooled events of ctx->timer).
struct SlicePull {
    int64_t rows = 0, nnz = 0, dev_bytes = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
};
spg_csr* vconcat(spg_ctx* ctx, const spg_csr* const* slices, int n, cudaEvent_t rp_ready = nullptr,
                 std::vector<SlicePull>* log = nullptr);
// [A_0 | A_1 | ...] of row-aligned parts (at most 16)
spg_csr* hconcat(spg_ctx* ctx, const spg_csr* const* parts, int n);
spg_csr* extract(spg_ctx* ctx, const spg_csr* m, int64_t r0, int64_t r1, int64_t c0, int64_t c1);
spg_csr* copy_csr(spg_ctx* ctx, const spg_csr* m);
// C = A*B into host arrays, A in row batches cuts[0..nb] with each batch's
// download overlapping the next batch's multiply. Returns nnz(C); nothing but
// the count is written when it exceeds cap.
int64_t spgemm_to_host(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const int64_t* cuts, int nb,
                       int64_t* h_rowptr, void* h_colind, int colind_width, double* h_values, int64_t cap);

// Device tile store (tiles.cu): make_tile_map rectangles (partition.cpp:95-159),
// partition (:161-222) onto the tiles' devices, reassemble (:224-261).
// scheme: 0 trident, 1 grid2d, 2 rows1d (partition.hpp:10).
struct TileRect {
    int64_t r0, r1, c0, c1;
};
std::vector<TileRect> tile_rects(int64_t nrows, int64_t ncols, int scheme, int procs, int gpus_per_node);
void partition_device(spg_ctx* const* ctxs, int nctx, const spg_csr* m, int scheme, int procs, int gpus_per_node,
                      spg_csr** out);
spg_csr* reassemble_device(spg_ctx* ctx, const spg_csr* const* tiles, int ntiles, int64_t nrows, int64_t ncols,
                           int scheme, int procs, int gpus_per_node);
void column_normalize(spg_ctx* ctx, spg_csr* m);
spg_csr* prune(spg_ctx* ctx, const spg_csr* m, double threshold);
void elementwise_power(spg_ctx* ctx, spg_csr* m, double exponent);
// One MCL iteration's post-step (apps.cpp:79-82): column_normalize(power(prune(column_normalize(c))))
spg_csr* mcl_poststep(spg_ctx* ctx, const spg_csr* c, double prune_threshold, double inflation);
void check_canonical(spg_ctx* ctx, const spg_csr* m);
// report.cpp:11-26 result_checksum hash (order-independent, exact)
uint64_t result_checksum(spg_ctx* ctx, const spg_csr* m);

// Exclusive scan of n int64 counts into out[0..n] (out[n] = total). In-place allowed.
void exclusive_scan_i64(spg_ctx* ctx, const int64_t* in, int64_t* out, int64_t n);

inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace spgb
