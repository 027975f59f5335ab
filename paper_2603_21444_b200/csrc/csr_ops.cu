// Device CSR store and the non-multiply kernels of the hot path:
//   spgeam   (reference csr.cpp:167-196)  — partial-C merge
//   vconcat  (reference csr.cpp:348-363)  — data effect of the node allgather
//   extract  (reference partition.cpp:161-222, one tile)
//   column_normalize / prune (reference csr.cpp:224-249) — MCL post-step
//   check_canonical (reference csr.cpp:30-50)
#include <atomic>
#include <deque>
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <climits>
#include <cstdlib>

#include "block_scan.cuh"
#include "spg_internal.cuh"

namespace spgb {
namespace {

int grid_for(spg_ctx* ctx, int64_t n, int bs = 256) {
    const int64_t want = (n + bs - 1) / bs;
    const int64_t cap = int64_t(ctx->num_sms) * 16;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); i += int64_t(gridDim.x) * blockDim.x)

// ----------------------------------------------------------------- spgeam
// Warp per row: merge-path split of the two sorted rows among the 32 lanes,
// each lane merges its diagonal segment sequentially. Pass 1 counts the
// union size per row; pass 2 writes at the scanned offsets.
__device__ __forceinline__ int64_t merge_path(const int32_t* a, int64_t na, const int32_t* b, int64_t nb,
                                              int64_t diag) {
    // number of elements taken from `a` at diagonal `diag` (a wins ties: a[i] <= b[j] goes first)
    int64_t lo = diag > nb ? diag - nb : 0;
    int64_t hi = diag < na ? diag : na;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= b[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <bool WRITE>
__global__ void k_spgeam(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                         const double* __restrict__ aval, const int64_t* __restrict__ brp,
                         const int32_t* __restrict__ bcol, const double* __restrict__ bval, int64_t m,
                         int64_t* __restrict__ cnt, const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                         double* __restrict__ cval) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nwarps) {
        const int64_t a0 = arp[i], na = arp[i + 1] - a0;
        const int64_t b0 = brp[i], nb = brp[i + 1] - b0;
        const int32_t* ac = acol + a0;
        const int32_t* bc = bcol + b0;
        const int64_t tot = na + nb;
        const int64_t per = (tot + 31) / 32;
        const int64_t d0 = ::min(tot, per * lane), d1 = ::min(tot, per * (lane + 1));
        int64_t ia = merge_path(ac, na, bc, nb, d0);
        int64_t ib = d0 - ia;
        const int64_t ia_end = merge_path(ac, na, bc, nb, d1);
        const int64_t ib_end = d1 - ia_end;
        // An equal pair (a[ia]==b[ib]) is merged into one output by the lane that
        // consumes the `a` element; a lane whose first element is a `b` equal to
        // the preceding `a` skips it.
        int64_t out = 0;
        int64_t o = WRITE ? crp[i] : 0;
        int64_t wpos = 0;
        if (WRITE) {
            // exclusive prefix of per-lane counts computed in a first sweep
            int64_t c = 0;
            {
                int64_t xa = ia, xb = ib;
                while (xa < ia_end || xb < ib_end) {
                    const int32_t ja = xa < na ? ac[xa] : INT_MAX;
                    const int32_t jb = xb < nb ? bc[xb] : INT_MAX;
                    if (xa < ia_end && (xb >= ib_end || ja <= jb)) {
                        ++c;
                        if (xb < nb && ja == jb) ++xb;  // merged pair (may extend past ib_end)
                        ++xa;
                    } else {
                        // a `b` element: skip if it equals the previous `a` (consumed by earlier lane)
                        if (!(xa > 0 && ac[xa - 1] == jb)) ++c;
                        ++xb;
                    }
                }
            }
            int64_t inc = c;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, inc, s);
                if (lane >= s) inc += y;
            }
            wpos = o + inc - c;
        }
        int64_t xa = ia, xb = ib;
        while (xa < ia_end || xb < ib_end) {
            const int32_t ja = xa < na ? ac[xa] : INT_MAX;
            const int32_t jb = xb < nb ? bc[xb] : INT_MAX;
            if (xa < ia_end && (xb >= ib_end || ja <= jb)) {
                if (xb < nb && ja == jb) {
                    if (WRITE) {
                        ccol[wpos] = ja;
                        cval[wpos] = __dadd_rn(aval[a0 + xa], bval[b0 + xb]);
                    }
                    ++xb;
                } else if (WRITE) {
                    ccol[wpos] = ja;
                    cval[wpos] = aval[a0 + xa];
                }
                ++out;
                ++wpos;
                ++xa;
            } else {
                if (!(xa > 0 && ac[xa - 1] == jb)) {
                    if (WRITE) {
                        ccol[wpos] = jb;
                        cval[wpos] = bval[b0 + xb];
                    }
                    ++out;
                    ++wpos;
                }
                ++xb;
            }
        }
        if (!WRITE) {
            int64_t s = out;
#pragma unroll
            for (int k = 16; k > 0; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
            if (lane == 0) cnt[i] = s;
        }
    }
}

// ----------------------------------------------------------------- vconcat
__global__ void k_rebase_rowptr(const int64_t* __restrict__ src, int64_t rows, int64_t base,
                                int64_t* __restrict__ dst) {
    GRID_STRIDE(i, rows) dst[i] = base + src[i + 1];
}

// ----------------------------------------------------------------- hconcat
// [A_0 | A_1 | ...]: equal row counts, part p's columns shifted by the widths
// of the parts before it; a row's entries stay in column order.
constexpr int HCAT_MAX = 16;
struct HcatParts {
    const int64_t* rp[HCAT_MAX];
    const int32_t* ci[HCAT_MAX];
    const double* va[HCAT_MAX];
    int32_t coff[HCAT_MAX];
    int n;
};

// Block per 256-row chunk: every part's row bounds in smem and the output
// row starts (every part's rowptr starts at 0, so a row's output start is the
// sum of the parts' row starts: no scan); then each part's contiguous entry
// range is copied striped (coalesced reads), an entry's row found by a binary
// search over the chunk's bounds. 3 TB/s (scripts/hcat_bench.cu) against
// 1.9 for a thread per (part, row).
__global__ void __launch_bounds__(256) k_hcat(HcatParts P, int64_t rows, int64_t* __restrict__ orp,
                                              int32_t* __restrict__ oci, double* __restrict__ ova) {
    __shared__ int64_t sb[HCAT_MAX][257];
    __shared__ int64_t so[257];
    const int tid = threadIdx.x;
    for (int64_t r0 = blockIdx.x * int64_t(256); r0 < rows; r0 += int64_t(gridDim.x) * 256) {
        const int nr = static_cast<int>(min(int64_t(256), rows - r0));
        for (int q = 0; q < P.n; ++q)
            for (int i = tid; i <= nr; i += 256) sb[q][i] = P.rp[q][r0 + i];
        __syncthreads();
        for (int i = tid; i <= nr; i += 256) {
            int64_t o = 0;
            for (int q = 0; q < P.n; ++q) o += sb[q][i];
            so[i] = o;
            orp[r0 + i] = o;  // entry nr is also the next chunk's first: same value
        }
        __syncthreads();
        for (int q = 0; q < P.n; ++q) {
            const int64_t e0 = sb[q][0], e1 = sb[q][nr];
            const int32_t* __restrict__ ci = P.ci[q];
            const double* __restrict__ va = P.va[q];
            const int32_t off = P.coff[q];
            for (int64_t x = e0 + tid; x < e1; x += 256) {
                int lo = 0, hi = nr - 1;  // the last row starting at or before x
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sb[q][mid] <= x) lo = mid;
                    else hi = mid - 1;
                }
                int64_t d = so[lo] + (x - sb[q][lo]);
                for (int q2 = 0; q2 < q; ++q2) d += sb[q2][lo + 1] - sb[q2][lo];
                oci[d] = ci[x] + off;
                ova[d] = va[x];
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------- extract
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* p, int64_t lo, int64_t hi, int64_t v) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (p[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_extract_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t r0,
                                int64_t rows, int64_t c0, int64_t c1, int64_t* __restrict__ beg,
                                int64_t* __restrict__ cnt) {
    GRID_STRIDE(i, rows) {
        const int64_t lo = rp[r0 + i], hi = rp[r0 + i + 1];
        const int64_t a = lower_bound_i32(col, lo, hi, c0);
        const int64_t b = lower_bound_i32(col, a, hi, c1);
        beg[i] = a;
        cnt[i] = b - a;
    }
}

// G lanes per row (G = 8 for short rows: a 16-entry ER row split over q tiles
// would leave most of a warp idle)
template <int G>
__global__ void k_extract_copy(const int64_t* __restrict__ beg, const int64_t* __restrict__ orp, int64_t rows,
                               const int32_t* __restrict__ col, const double* __restrict__ val, int64_t c0,
                               int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int lane = threadIdx.x & (G - 1);
    const int64_t grp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / G;
    const int64_t ngrp = (int64_t(gridDim.x) * blockDim.x) / G;
    for (int64_t i = grp; i < rows; i += ngrp) {
        const int64_t s = beg[i], o = orp[i], n = orp[i + 1] - o;
        for (int64_t t = lane; t < n; t += G) {
            ocol[o + t] = static_cast<int32_t>(col[s + t] - c0);
            oval[o + t] = val[s + t];
        }
    }
}

// ------------------------------------------------------- column_normalize
// Column sums in CSR storage order (reference csr.cpp:225-227): entries are
// stably radix-sorted by column (value as payload), then each column is summed
// sequentially in storage order, so sums are bit-identical.

// Runs of the sorted keys (one run per column present), in two passes over
// blocks of CS_BLK keys (16 per thread, 16-byte loads): k_colsum_heads<false>
// counts each block's run heads, a scan gives each block its first slot,
// k_colsum_heads<true> writes the head positions in order (heads[nh] = nnz).
// k_colsum_fold then gives every run one thread that folds its values in
// storage order: the run [heads[h], heads[h+1]) is contiguous, so its loads
// are independent (unrolled 8 deep) while the dependent adds retire in order —
// bit-identical to the reference's loop.
constexpr int CS_IT = 16, CS_BLK = 256 * CS_IT;
template <bool WRITE>
__global__ void __launch_bounds__(256) k_colsum_heads(const int32_t* __restrict__ keys, int64_t nnz,
                                                      int64_t* __restrict__ bcount, int64_t* __restrict__ heads) {
    __shared__ int ws[9];
    const int64_t nblk = (nnz + CS_BLK - 1) / CS_BLK;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t i0 = blk * CS_BLK + int64_t(threadIdx.x) * CS_IT;
        int32_t k[CS_IT];
        uint32_t hm = 0;
        if (i0 < nnz) {
            if (i0 + CS_IT <= nnz) {
#pragma unroll
                for (int u = 0; u < CS_IT / 4; ++u) {
                    const int4 w = __ldg(reinterpret_cast<const int4*>(keys + i0) + u);
                    k[4 * u] = w.x;
                    k[4 * u + 1] = w.y;
                    k[4 * u + 2] = w.z;
                    k[4 * u + 3] = w.w;
                }
            } else {
#pragma unroll
                for (int u = 0; u < CS_IT; ++u) k[u] = i0 + u < nnz ? keys[i0 + u] : -1;
            }
            int32_t prev = i0 > 0 ? keys[i0 - 1] : -1;
#pragma unroll
            for (int u = 0; u < CS_IT; ++u) {
                if (i0 + u < nnz && k[u] != prev) hm |= 1u << u;
                prev = k[u];
            }
        }
        int total;
        const int pre = block_exclusive_scan<256>(__popc(hm), &total, ws);
        if (!WRITE) {
            if (threadIdx.x == 0) bcount[blk] = total;
        } else {
            int64_t o = bcount[blk] + pre;
            while (hm) {
                const int u = __ffs(hm) - 1;
                hm &= hm - 1;
                heads[o++] = i0 + u;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_colsum_fold(const int32_t* __restrict__ keys, const double* __restrict__ sval,
                                                     const int64_t* __restrict__ heads, int64_t nh,
                                                     double* __restrict__ colsum) {
    for (int64_t h = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = heads[h], e = heads[h + 1];
        double acc = 0.0;
        int64_t u = s;
        for (; u + 8 <= e; u += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(sval + u + q);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
        }
        for (; u < e; ++u) acc = __dadd_rn(acc, __ldg(sval + u));
        colsum[keys[s]] = acc;
    }
}

__global__ void k_scale_cols(const int32_t* __restrict__ col, double* __restrict__ val, int64_t nnz,
                             const double* __restrict__ colsum) {
    GRID_STRIDE(t, nnz) {
        const double s = colsum[col[t]];
        if (s != 0.0) val[t] = __ddiv_rn(val[t], s);
    }
}

// -------------------------------------------------------------------- prune
// MCL transform of a value before the prune test (apps.cpp:79-81): with
// colsum, v' = v / colsum[col] when the sum is nonzero (column_normalize,
// csr.cpp:228-232); the kept value is written as pow(v', r) (elementwise_power,
// csr.cpp:251-255; r = 2 is the correctly rounded square, r = 1 the identity).
__device__ __forceinline__ double mcl_scale(double v, int32_t c, const double* __restrict__ colsum) {
    if (colsum) {
        const double s = colsum[c];
        if (s != 0.0) v = __ddiv_rn(v, s);
    }
    return v;
}
__device__ __forceinline__ double mcl_power(double v, double r) {
    if (r == 1.0) return v;
    if (r == 2.0) return __dmul_rn(v, v);
    return pow(v, r);
}

__global__ void k_prune_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ val, int64_t m, double th, const double* __restrict__ colsum,
                              int64_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nwarps) {
        int64_t c = 0;
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32)
            c += !(mcl_scale(val[t], colsum ? col[t] : 0, colsum) < th);
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) c += __shfl_xor_sync(0xffffffffu, c, k);
        if (lane == 0) cnt[i] = c;
    }
}
__global__ void k_prune_copy(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const double* __restrict__ val, int64_t m, double th, const double* __restrict__ colsum,
                             double r, const int64_t* __restrict__ orp, int32_t* __restrict__ ocol,
                             double* __restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nwarps) {
        int64_t o = orp[i];
        for (int64_t base = rp[i]; base < rp[i + 1]; base += 32) {
            const int64_t t = base + lane;
            int32_t c = 0;
            double v = 0.0;
            if (t < rp[i + 1]) {
                c = col[t];
                v = mcl_scale(val[t], c, colsum);
            }
            const bool keep = t < rp[i + 1] && !(v < th);
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int64_t w = o + __popc(mask & ((1u << lane) - 1));
                ocol[w] = c;
                oval[w] = mcl_power(v, r);
            }
            o += __popc(mask);
        }
    }
}

__global__ void k_power(double* __restrict__ val, int64_t nnz, double r) {
    GRID_STRIDE(t, nnz) val[t] = mcl_power(val[t], r);
}

// ---------------------------------------------------------- result checksum
// report.cpp:11-26: Σ (mod 2^64) over entries of
// mix64(mix64(mix64(row + K) ^ col) ^ llround(v * 1e9)) — order-independent
// integer work, so the device sum equals the reference's exactly. 8 lanes per
// row, per-thread partial sums, one atomic per warp.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_checksum(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                           const double* __restrict__ val, int64_t m, unsigned long long* __restrict__ out) {
    constexpr int G = 8;
    const int lane = threadIdx.x & (G - 1);
    const int64_t g0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / G;
    const int64_t ng = (int64_t(gridDim.x) * blockDim.x) / G;
    uint64_t acc = 0;
    for (int64_t i = g0; i < m; i += ng) {
        const uint64_t hr = mix64(static_cast<uint64_t>(i) + 0x51ED270B9A3E51EBull);
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += G) {
            const long long q = llround(__dmul_rn(val[t], 1e9));
            uint64_t h = mix64(hr ^ static_cast<uint64_t>(static_cast<int64_t>(col[t])));
            acc += mix64(h ^ static_cast<uint64_t>(q));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, static_cast<unsigned long long>(acc));
}

// -------------------------------------------------------- canonical check
// err[0] = first offending row (or INT64_MAX), err[1] = violation code.
__global__ void k_check(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t m, int64_t ncols,
                        int64_t nnz, unsigned long long* __restrict__ err) {
    GRID_STRIDE(i, m) {
        const int64_t lo = rp[i], hi = rp[i + 1];
        int code = 0;
        if (lo > hi) code = 1;
        else if (hi > nnz || lo < 0) code = 2;
        else
            for (int64_t t = lo; t < hi; ++t) {
                if (col[t] < 0 || col[t] >= ncols) { code = 3; break; }
                if (t > lo && col[t - 1] >= col[t]) { code = 4; break; }
            }
        if (code) atomicMin(err, (static_cast<unsigned long long>(i) << 3) | code);
    }
}

// ---------------------------------------------------------- index widening
__global__ void k_narrow(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                         unsigned long long* __restrict__ bad) {
    GRID_STRIDE(i, n) {
        const int64_t v = in[i];
        if (v < INT_MIN || v > INT_MAX) atomicOr(bad, 1ull);
        out[i] = static_cast<int32_t>(v);
    }
}

__global__ void k_widen(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    GRID_STRIDE(i, n) out[i] = in[i];
}

}  // namespace

// ===================================================================== host
spg_csr* new_csr(spg_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz) {
    auto* m = new spg_csr;
    m->ctx = ctx;
    m->nrows = nrows;
    m->ncols = ncols;
    m->rowptr = dalloc<int64_t>(ctx, nrows + 1);
    if (nnz >= 0) {
        m->nnz = nnz;
        m->colind = dalloc<int32_t>(ctx, nnz);
        m->values = dalloc<double>(ctx, nnz);
        if (nnz == 0) SPG_CUDA(cudaMemsetAsync(m->rowptr, 0, (nrows + 1) * sizeof(int64_t), ctx->stream));
    }
    return m;
}

namespace {
constexpr size_t BIG_ROUND = size_t(64) << 20;
constexpr size_t BIG_KEEP = 48;  // cached blocks per context
std::atomic<int> g_live[64];     // live contexts per device
// at most this many bytes per context: 45% of device memory shared among the
// device's live contexts (at least 16 GB)
size_t big_keep_bytes(const spg_ctx* ctx) {
    const int live = std::max(1, g_live[ctx->device & 63].load());
    return std::max(size_t(16) << 30, static_cast<size_t>(0.45 * static_cast<double>(ctx->mem_total)) / live);
}
}  // namespace

void ctx_live(int device, int delta) { g_live[device & 63] += delta; }

void* pool_alloc(spg_ctx* ctx, size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        big_cache_release(ctx);
        cudaStreamSynchronize(ctx->stream);
        cudaMemPoolTrimTo(ctx->pool, 0);
        e = cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream);
    }
    if (e != cudaSuccess)
        fail(e == cudaErrorMemoryAllocation ? SPG_OOM : SPG_CUDA_ERROR,
             "device allocation of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    return p;
}

// Best-fit block of at least `bytes` (at most 2x larger) from the context's
// cache, else a fresh pool block rounded up to 64 MB. Stream order on the
// context stream makes reuse safe (the block was freed on the same stream).
void* big_alloc(spg_ctx* ctx, size_t bytes, size_t* cap) {
    int best = -1;
    for (size_t i = 0; i < ctx->big_cache.size(); ++i) {
        const size_t sz = ctx->big_cache[i].second;
        if (sz >= bytes && sz <= 2 * bytes + BIG_ROUND && (best < 0 || sz < ctx->big_cache[best].second))
            best = static_cast<int>(i);
    }
    if (best >= 0) {
        void* p = ctx->big_cache[best].first;
        *cap = ctx->big_cache[best].second;
        ctx->big_cache.erase(ctx->big_cache.begin() + best);
        return p;
    }
    // fresh block: round up to a size class (64 MB steps up to 1 GB, then
    // steps of 1/8 of the power of two) so later requests of similar size reuse it
    size_t sz = (bytes + BIG_ROUND - 1) / BIG_ROUND * BIG_ROUND;
    if (sz > (size_t(1) << 30)) {
        size_t p2 = size_t(1) << 30;
        while (p2 * 2 <= sz) p2 *= 2;
        const size_t step = p2 / 8;
        sz = (sz + step - 1) / step * step;
    }
    void* p = pool_alloc(ctx, sz);
    *cap = sz;
    return p;
}

void big_free(spg_ctx* ctx, void* p, size_t cap) {
    ctx->big_cache.emplace_back(p, cap);
    size_t held = 0;
    for (auto& b : ctx->big_cache) held += b.second;
    const size_t keep = big_keep_bytes(ctx);
    while (held > keep && ctx->big_cache.size() > 1) {  // drop the oldest
        held -= ctx->big_cache.front().second;
        cudaFreeAsync(ctx->big_cache.front().first, ctx->stream);
        ctx->big_cache.erase(ctx->big_cache.begin());
    }
    if (ctx->big_cache.size() > BIG_KEEP) {  // drop the smallest
        size_t k = 0;
        for (size_t i = 1; i < ctx->big_cache.size(); ++i)
            if (ctx->big_cache[i].second < ctx->big_cache[k].second) k = i;
        cudaFreeAsync(ctx->big_cache[k].first, ctx->stream);
        ctx->big_cache.erase(ctx->big_cache.begin() + k);
    }
}

void alloc_c_arrays(spg_ctx* ctx, spg_csr* c, int64_t cap) {
    const size_t n = static_cast<size_t>(cap > 0 ? cap : 1);
    if (n * sizeof(int32_t) >= BIG_BYTES) {
        c->colind = static_cast<int32_t*>(big_alloc(ctx, n * sizeof(int32_t), &c->big_col));
        c->values = static_cast<double*>(big_alloc(ctx, n * sizeof(double), &c->big_val));
    } else {
        c->colind = dalloc<int32_t>(ctx, n);
        c->values = dalloc<double>(ctx, n);
    }
}

void big_cache_release(spg_ctx* ctx) {
    for (auto& b : ctx->big_cache) cudaFreeAsync(b.first, ctx->stream);
    ctx->big_cache.clear();
}

void free_csr(spg_csr* m) {
    if (!m) return;
    DeviceScope ds(m->ctx->device);
    if (m->storage == 0) {
        dfree(m->ctx, m->rowptr);
        if (m->big_col) big_free(m->ctx, m->colind, m->big_col);
        else dfree(m->ctx, m->colind);
        if (m->big_val) big_free(m->ctx, m->values, m->big_val);
        else dfree(m->ctx, m->values);
    } else if (m->storage == 1) {
        cudaStreamSynchronize(m->ctx->stream);
        cudaFree(m->rowptr);
        cudaFree(m->colind);
        cudaFree(m->values);
    } else {
        cudaIpcCloseMemHandle(m->rowptr);
        if (m->colind) cudaIpcCloseMemHandle(m->colind);
        if (m->values) cudaIpcCloseMemHandle(m->values);
    }
    delete m;
}

// Small read-backs are written by a kernel straight into the context's
// mapped pinned scalars instead of a cudaMemcpy: a D2H copy would queue on the
// copy engine behind bulk downloads running on other streams (the
// host-to-host multiply downloads batch i while batch i+1 is multiplied).
__global__ void k_peek(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

void* peek_async(spg_ctx* ctx, int off, const void* dsrc, int bytes) {
    if (off < 0 || off + bytes > spg_ctx::HOST_SCALAR_BYTES) fail(SPG_ERROR, "peek_async: slot out of range");
    unsigned char* dst = reinterpret_cast<unsigned char*>(ctx->host_scalars) + off;
    KTime kt(ctx, "peek");
    k_peek<<<1, 32, 0, ctx->stream>>>(static_cast<const unsigned char*>(dsrc), dst, bytes);
    SPG_LAUNCH_CHECK();
    return dst;
}

int64_t read_scalar(spg_ctx* ctx, const int64_t* dptr) {
    peek_async(ctx, 0, dptr, sizeof(int64_t));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    return *reinterpret_cast<volatile int64_t*>(ctx->host_scalars);
}

spg_csr* spgeam(spg_ctx* ctx, const spg_csr* a, const spg_csr* b) {
    if (a->nrows != b->nrows || a->ncols != b->ncols) fail(SPG_DIMENSION_ERROR, "spgeam: shape mismatch");
    const int64_t m = a->nrows;
    if (a->nnz == 0) return copy_csr(ctx, b);
    if (b->nnz == 0) return copy_csr(ctx, a);
    DBuf<int64_t> cnt(ctx, m + 1);
    spg_csr* c = new_csr(ctx, m, a->ncols, -1);
    const int g = grid_for(ctx, m * 32);
    {
        KTime kt(ctx, "spgeam_count");
        k_spgeam<false><<<g, 256, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values,
                                                     m, cnt, nullptr, nullptr, nullptr);
        SPG_LAUNCH_CHECK();
    }
    exclusive_scan_i64(ctx, cnt, c->rowptr, m);
    c->nnz = read_scalar(ctx, c->rowptr + m);
    alloc_c_arrays(ctx, c, c->nnz);
    {
        KTime kt(ctx, "spgeam_write");
        k_spgeam<true><<<g, 256, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values,
                                                    m, nullptr, c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    return c;
}

spg_csr* copy_csr(spg_ctx* ctx, const spg_csr* s) {
    spg_csr* c = new_csr(ctx, s->nrows, s->ncols, s->nnz);
    const int sd = s->ctx->device, dd = ctx->device;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
        if (!bytes) return;
        if (sd == dd) SPG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
        else SPG_CUDA(cudaMemcpyPeerAsync(dst, dd, src, sd, bytes, ctx->stream));
    };
    cp(c->rowptr, s->rowptr, (s->nrows + 1) * sizeof(int64_t));
    cp(c->colind, s->colind, s->nnz * sizeof(int32_t));
    cp(c->values, s->values, s->nnz * sizeof(double));
    return c;
}

// A slice that lives in this device's own memory is copied by the SMs (HBM
// bound), so that the copy engines are left to the peer pulls: a local
// device-to-device copy on a copy engine competes with the NVLink pulls of the
// other slices.
template <typename T>
__global__ void k_copy_elems(const T* __restrict__ src, T* __restrict__ dst, int64_t n) {
    GRID_STRIDE(i, n) dst[i] = src[i];
}

// Contiguous copy by the TMA engine (cp.async.bulk): each CTA moves chunks of
// BULK_CH bytes global -> shared (completion on an mbarrier's transaction
// count) -> global (bulk group), double-buffered; src and dst 16-byte
// aligned, bytes a multiple of 16 (the caller copies the tail).
constexpr int BULK_CH = 16384;
__global__ void __launch_bounds__(32) k_bulk_copy(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                                  int64_t bytes) {
    __shared__ __align__(128) unsigned char buf[2][BULK_CH];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x != 0) return;
    const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[0]));
    const uint32_t b1 = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[1]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned ph[2] = {0u, 0u};
    int k = 0;
    for (int64_t off = int64_t(blockIdx.x) * BULK_CH; off < bytes; off += int64_t(gridDim.x) * BULK_CH, k ^= 1) {
        const uint32_t n = static_cast<uint32_t>(min(int64_t(BULK_CH), bytes - off));
        const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(buf[k]));
        const uint32_t bk = k ? b1 : b0;
        // the store that last read buf[k] (two chunks ago) must be done
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bk), "r"(n) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                     "l"(src + off), "r"(n), "r"(bk)
                     : "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                : "=r"(done)
                : "r"(bk), "r"(ph[k])
                : "memory");
        }
        ph[k] ^= 1u;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(sb), "r"(n)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// dst[0, n) = src[0, n) on stream st: by the TMA engine when src and dst are
// 16-byte co-aligned (the unaligned tail by a small element kernel), else by
// the SMs.
template <typename T>
void device_copy(spg_ctx* ctx, cudaStream_t st, T* dst, const T* src, int64_t n) {
    if (n <= 0) return;
    const uintptr_t a = reinterpret_cast<uintptr_t>(src), b = reinterpret_cast<uintptr_t>(dst);
    const int64_t bytes = n * static_cast<int64_t>(sizeof(T));
    if ((a % 16) == 0 && (b % 16) == 0 && bytes >= 16) {
        const int64_t body = bytes & ~int64_t(15);
        const int g = static_cast<int>(std::min<int64_t>((body + BULK_CH - 1) / BULK_CH, int64_t(ctx->num_sms) * 4));
        k_bulk_copy<<<g, 32, 0, st>>>(reinterpret_cast<const unsigned char*>(src), reinterpret_cast<unsigned char*>(dst),
                                      body);
        SPG_LAUNCH_CHECK();
        const int64_t done = body / static_cast<int64_t>(sizeof(T));
        if (done < n) {
            k_copy_elems<T><<<1, 32, 0, st>>>(src + done, dst + done, n - done);
            SPG_LAUNCH_CHECK();
        }
        return;
    }
    k_copy_elems<T><<<grid_for(ctx, n), 256, 0, st>>>(src, dst, n);
    SPG_LAUNCH_CHECK();
}

// Slices in peers' memory (peer access or IPC mappings): with three or more
// of them pulled at once (N=4 at q = 1: an all-to-all) the SMs pull them —
// each thread keeps 8 independent NVLink loads in flight, column indices
// first, then values; SM pulls reach 580-640 GB/s into each of 4 GPUs in an
// all-to-all against 402 for the copy engines, at any element width
// (`scripts/peer_bench.cu`, `profiles/r2r_*`). With one or two peers the copy
// engines are faster (one puller: 790 against 717 GB/s; N=2 step 12.84 ms
// against 13.23). The SM pulls of all slices together take SPG_PULL_BLOCKS
// (default 2) 512-thread CTAs per SM, so that the multiply's row preparation
// still finds room beside them. SPG_PULL_CE=1 / 0 forces copy engines / SMs.
template <typename T>
__device__ __forceinline__ void pull_elems(const T* __restrict__ src, T* __restrict__ dst, int64_t n) {
    constexpr int U = 8;
    const int64_t st = int64_t(gridDim.x) * blockDim.x;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * st < n; i += U * st) {
        T r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = src[i + u * st];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * st] = r[u];
    }
    for (; i < n; i += st) dst[i] = src[i];
}

__global__ void __launch_bounds__(512) k_pull_slice(const int32_t* __restrict__ sc, int32_t* __restrict__ dc,
                                                    const double* __restrict__ sv, double* __restrict__ dv,
                                                    int64_t nnz) {
    pull_elems(sc, dc, nnz);
    pull_elems(sv, dv, nnz);
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

spg_csr* vconcat(spg_ctx* ctx, const spg_csr* const* slices, int n, cudaEvent_t rp_ready,
                 std::vector<SlicePull>* log) {
    if (n == 0) {
        spg_csr* z = new_csr(ctx, 0, 0, 0);
        if (rp_ready) SPG_CUDA(cudaEventRecord(rp_ready, ctx->stream));
        return z;
    }
    int64_t rows = 0, nnz = 0;
    const int64_t ncols = slices[0]->ncols;
    for (int s = 0; s < n; ++s) {
        if (slices[s]->ncols != ncols) fail(SPG_DIMENSION_ERROR, "vconcat: column count mismatch");
        rows += slices[s]->nrows;
        nnz += slices[s]->nnz;
    }
    spg_csr* out = new_csr(ctx, rows, ncols, nnz);
    SPG_CUDA(cudaMemsetAsync(out->rowptr, 0, sizeof(int64_t), ctx->stream));
    const bool fork = n > 1 && ctx->aux[0];
    if (fork) SPG_CUDA(cudaEventRecord(ctx->aux_ev[spg_ctx::NAUX], ctx->stream));  // fork point
    const int dd = ctx->device;
    if (log) log->assign(n, SlicePull{});
    // 1: the row pointers, rebased by kernels reading every slice's row
    // pointers in place (peer access / IPC mapping: no staging copy); issued
    // first so that they are not queued behind the pulls
    int64_t r = 0, base = 0;
    for (int s = 0; s < n; ++s) {
        const spg_csr* sl = slices[s];
        if (sl->nrows) {
            KTime kt(ctx, "vconcat_rebase");
            k_rebase_rowptr<<<grid_for(ctx, sl->nrows), 256, 0, ctx->stream>>>(sl->rowptr, sl->nrows, base,
                                                                                 out->rowptr + r + 1);
            SPG_LAUNCH_CHECK();
        }
        r += sl->nrows;
        base += sl->nnz;
    }
    if (rp_ready) SPG_CUDA(cudaEventRecord(rp_ready, ctx->stream));
    // 2: the column/value pulls (one aux stream per slice, concurrently; local
    // slices by the SMs)
    int remote = 0;  // slices pulled from a peer: they share the pull CTAs
    for (int s = 0; s < n; ++s)
        remote += slices[s]->nnz && (slices[s]->ctx->device != dd || slices[s]->storage == 2);
    static const int pull_ce_env = env_int("SPG_PULL_CE", -1);
    const bool pull_ce = pull_ce_env == 1 || (pull_ce_env != 0 && remote < 3);
    static const int pull_per_sm = std::max(1, env_int("SPG_PULL_BLOCKS", 2));
    const int pull_grid = std::max(1, ctx->num_sms * pull_per_sm / std::max(remote, 1));
    base = 0;
    for (int s = 0; s < n; ++s) {
        const spg_csr* sl = slices[s];
        const int sd = sl->ctx->device;
        cudaStream_t st = ctx->stream;
        if (fork) {
            st = ctx->aux[s % spg_ctx::NAUX];
            if (s < spg_ctx::NAUX) SPG_CUDA(cudaStreamWaitEvent(st, ctx->aux_ev[spg_ctx::NAUX], 0));
        }
        if (log) {
            SlicePull& L = (*log)[s];
            L.rows = sl->nrows;
            L.nnz = sl->nnz;
            L.dev_bytes = (sl->nrows + 1) * int64_t(sizeof(int64_t)) + sl->nnz * int64_t(sizeof(int32_t) + sizeof(double));
            L.t0 = ctx->timer.ev();
            L.t1 = ctx->timer.ev();
            SPG_CUDA(cudaEventRecord(L.t0, st));
        }
        if (sl->nnz) {
            const bool own = sd == dd && sl->storage != 2;  // this device's memory (not an IPC view)
            if (own) {
                device_copy(ctx, st, out->colind + base, sl->colind, sl->nnz);
                device_copy(ctx, st, out->values + base, sl->values, sl->nnz);
            } else if (!pull_ce) {
                k_pull_slice<<<pull_grid, 512, 0, st>>>(sl->colind, out->colind + base, sl->values, out->values + base,
                                                        sl->nnz);
                SPG_LAUNCH_CHECK();
            } else if (sd == dd) {
                SPG_CUDA(cudaMemcpyAsync(out->colind + base, sl->colind, sl->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
                SPG_CUDA(cudaMemcpyAsync(out->values + base, sl->values, sl->nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
            } else {
                SPG_CUDA(cudaMemcpyPeerAsync(out->colind + base, dd, sl->colind, sd, sl->nnz * sizeof(int32_t), st));
                SPG_CUDA(cudaMemcpyPeerAsync(out->values + base, dd, sl->values, sd, sl->nnz * sizeof(double), st));
            }
        }
        if (log) SPG_CUDA(cudaEventRecord((*log)[s].t1, st));
        base += sl->nnz;
    }
    if (fork)
        for (int i = 0; i < std::min(n, spg_ctx::NAUX); ++i) {
            SPG_CUDA(cudaEventRecord(ctx->aux_ev[i], ctx->aux[i]));
            SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[i], 0));
        }
    return out;
}

spg_csr* hconcat(spg_ctx* ctx, const spg_csr* const* parts, int n) {
    if (n <= 0 || n > HCAT_MAX) fail(SPG_PARAMETER_ERROR, "hconcat: 1.." + std::to_string(HCAT_MAX) + " parts");
    const int64_t rows = parts[0]->nrows;
    HcatParts P{};
    int64_t cols = 0, nnz = 0;
    for (int p = 0; p < n; ++p) {
        if (parts[p]->nrows != rows) fail(SPG_DIMENSION_ERROR, "hconcat: row count mismatch");
        P.rp[p] = parts[p]->rowptr;
        P.ci[p] = parts[p]->colind;
        P.va[p] = parts[p]->values;
        P.coff[p] = static_cast<int32_t>(cols);
        cols += parts[p]->ncols;
        nnz += parts[p]->nnz;
    }
    P.n = n;
    if (cols > (int64_t(1) << 31)) fail(SPG_PARAMETER_ERROR, "hconcat: more than 2^31 columns");
    spg_csr* out = new_csr(ctx, rows, cols, -1);
    out->nnz = nnz;
    alloc_c_arrays(ctx, out, nnz);
    KTime kt(ctx, "hconcat");
    if (rows == 0) SPG_CUDA(cudaMemsetAsync(out->rowptr, 0, sizeof(int64_t), ctx->stream));
    else k_hcat<<<static_cast<int>(std::min<int64_t>((rows + 255) / 256, int64_t(ctx->num_sms) * 64)), 256, 0,
                  ctx->stream>>>(P, rows, out->rowptr, out->colind, out->values);
    SPG_LAUNCH_CHECK();
    return out;
}

spg_csr* extract(spg_ctx* ctx, const spg_csr* m, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
    if (r0 < 0 || r1 < r0 || r1 > m->nrows || c0 < 0 || c1 < c0 || c1 > m->ncols)
        fail(SPG_PARAMETER_ERROR, "extract: rectangle outside the matrix");
    const int64_t rows = r1 - r0;
    spg_csr* t = new_csr(ctx, rows, c1 - c0, -1);
    if (rows == 0 || m->nnz == 0) {
        t->nnz = 0;
        t->colind = dalloc<int32_t>(ctx, 0);
        t->values = dalloc<double>(ctx, 0);
        SPG_CUDA(cudaMemsetAsync(t->rowptr, 0, (rows + 1) * sizeof(int64_t), ctx->stream));
        return t;
    }
    DBuf<int64_t> beg(ctx, rows), cnt(ctx, rows);
    KTime kt(ctx, "extract");
    k_extract_count<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(m->rowptr, m->colind, r0, rows, c0, c1, beg, cnt);
    SPG_LAUNCH_CHECK();
    exclusive_scan_i64(ctx, cnt, t->rowptr, rows);
    t->nnz = read_scalar(ctx, t->rowptr + rows);
    alloc_c_arrays(ctx, t, t->nnz);
    if (t->nnz <= 24 * rows)
        k_extract_copy<8><<<grid_for(ctx, rows * 8), 256, 0, ctx->stream>>>(beg, t->rowptr, rows, m->colind, m->values,
                                                                            c0, t->colind, t->values);
    else
        k_extract_copy<32><<<grid_for(ctx, rows * 32), 256, 0, ctx->stream>>>(beg, t->rowptr, rows, m->colind,
                                                                              m->values, c0, t->colind, t->values);
    SPG_LAUNCH_CHECK();
    return t;
}

namespace {
// Column sums in CSR storage order (csr.cpp:225-227) into colsum[ncols]:
// stable radix sort of (column -> value) makes each column's values
// contiguous in storage (row) order, then one thread per column sums them
// sequentially like the reference loop.
void column_sums(spg_ctx* ctx, const spg_csr* m, double* colsum) {
    const int64_t nnz = m->nnz;
    SPG_CUDA(cudaMemsetAsync(colsum, 0, m->ncols * sizeof(double), ctx->stream));
    if (nnz == 0) return;
    if (nnz > INT32_MAX) fail(SPG_PARAMETER_ERROR, "column_normalize: nnz exceeds 2^31");
    DBuf<int32_t> keys(ctx, nnz);
    DBuf<double> vals(ctx, nnz);
    int bits = 1;
    while ((int64_t(1) << bits) < m->ncols) ++bits;
    size_t tmp = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, m->colind, keys.get(), m->values, vals.get(),
                                             static_cast<int>(nnz), 0, bits, ctx->stream));
    DBuf<unsigned char> t(ctx, tmp);
    {
        KTime kt(ctx, "colsum_sort");
        SPG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, m->colind, keys.get(), m->values, vals.get(),
                                                 static_cast<int>(nnz), 0, bits, ctx->stream));
    }
    KTime kt(ctx, "colsum_runs");
    const int64_t nblk = (nnz + CS_BLK - 1) / CS_BLK;
    const int hg = static_cast<int>(std::min<int64_t>(nblk, int64_t(ctx->num_sms) * 8));
    DBuf<int64_t> bcount(ctx, nblk), bbase(ctx, nblk + 1), heads(ctx, std::min<int64_t>(nnz, m->ncols) + 1);
    k_colsum_heads<false><<<hg, 256, 0, ctx->stream>>>(keys, nnz, bcount, nullptr);
    SPG_LAUNCH_CHECK();
    exclusive_scan_i64(ctx, bcount, bbase, nblk);
    k_colsum_heads<true><<<hg, 256, 0, ctx->stream>>>(keys, nnz, bbase, heads);
    SPG_LAUNCH_CHECK();
    const int64_t nh = read_scalar(ctx, bbase.get() + nblk);
    SPG_CUDA(cudaMemcpyAsync(heads.get() + nh, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    k_colsum_fold<<<grid_for(ctx, nh), 256, 0, ctx->stream>>>(keys, vals, heads, nh, colsum);
    SPG_LAUNCH_CHECK();
}

// Rows of a kept where !(v' < th), v' the MCL-scaled value; kept values raised to r.
spg_csr* prune_transform(spg_ctx* ctx, const spg_csr* a, double th, const double* colsum, double r) {
    const int64_t m = a->nrows;
    DBuf<int64_t> cnt(ctx, m + 1);
    spg_csr* out = new_csr(ctx, m, a->ncols, -1);
    if (m) {
        k_prune_count<<<grid_for(ctx, m * 32), 256, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, m, th, colsum,
                                                                      cnt);
        SPG_LAUNCH_CHECK();
    }
    exclusive_scan_i64(ctx, cnt, out->rowptr, m);
    out->nnz = read_scalar(ctx, out->rowptr + m);
    alloc_c_arrays(ctx, out, out->nnz);
    if (m && out->nnz) {
        k_prune_copy<<<grid_for(ctx, m * 32), 256, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, m, th, colsum, r,
                                                                     out->rowptr, out->colind, out->values);
        SPG_LAUNCH_CHECK();
    }
    return out;
}
}  // namespace

void column_normalize(spg_ctx* ctx, spg_csr* m) {
    if (m->nnz == 0) return;
    DBuf<double> colsum(ctx, m->ncols);
    KTime kt(ctx, "column_normalize");
    column_sums(ctx, m, colsum);
    k_scale_cols<<<grid_for(ctx, m->nnz), 256, 0, ctx->stream>>>(m->colind, m->values, m->nnz, colsum);
    SPG_LAUNCH_CHECK();
}

spg_csr* prune(spg_ctx* ctx, const spg_csr* a, double th) {
    if (th < 0.0) fail(SPG_PARAMETER_ERROR, "prune: negative threshold");
    KTime kt(ctx, "prune");
    return prune_transform(ctx, a, th, nullptr, 1.0);
}

void elementwise_power(spg_ctx* ctx, spg_csr* m, double r) {
    if (m->nnz == 0 || r == 1.0) return;
    KTime kt(ctx, "elementwise_power");
    k_power<<<grid_for(ctx, m->nnz), 256, 0, ctx->stream>>>(m->values, m->nnz, r);
    SPG_LAUNCH_CHECK();
}

spg_csr* mcl_poststep(spg_ctx* ctx, const spg_csr* c, double th, double r) {
    if (th < 0.0) fail(SPG_PARAMETER_ERROR, "mcl: negative prune threshold");
    spg_csr* out = nullptr;
    {
        // column_normalize + prune + elementwise_power in one pass over c
        DBuf<double> colsum(ctx, c->ncols);
        KTime kt(ctx, "mcl_normalize_prune_power");
        column_sums(ctx, c, colsum);
        out = prune_transform(ctx, c, th, colsum, r);
    }
    try {
        column_normalize(ctx, out);
    } catch (...) {
        free_csr(out);
        throw;
    }
    return out;
}

uint64_t result_checksum(spg_ctx* ctx, const spg_csr* m) {
    DBuf<unsigned long long> d(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), ctx->stream));
    if (m->nrows && m->nnz) {
        KTime kt(ctx, "result_checksum");
        k_checksum<<<grid_for(ctx, m->nrows * 8), 256, 0, ctx->stream>>>(m->rowptr, m->colind, m->values, m->nrows, d);
        SPG_LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    SPG_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
}

void check_canonical(spg_ctx* ctx, const spg_csr* m) {
    if (m->nrows < 0 || m->ncols < 0) fail(SPG_ERROR, "negative dimension");
    int64_t h[2];
    SPG_CUDA(cudaMemcpyAsync(&h[0], m->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(&h[1], m->rowptr + m->nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h[0] != 0) fail(SPG_ERROR, "rowptr[0] != 0");
    if (h[1] != m->nnz) fail(SPG_ERROR, "rowptr[nrows] != nnz");
    DBuf<unsigned long long> err(ctx, 1);
    const unsigned long long none = ~0ull;
    SPG_CUDA(cudaMemcpyAsync(err.get(), &none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream));
    if (m->nrows) {
        k_check<<<grid_for(ctx, m->nrows), 256, 0, ctx->stream>>>(m->rowptr, m->colind, m->nrows, m->ncols, m->nnz, err);
        SPG_LAUNCH_CHECK();
    }
    unsigned long long e = 0;
    SPG_CUDA(cudaMemcpyAsync(&e, err.get(), sizeof(e), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (e != none) {
        const int64_t row = static_cast<int64_t>(e >> 3);
        const int code = static_cast<int>(e & 7);
        const char* what = code == 1 ? "rowptr not non-decreasing at row "
                           : code == 2 ? "rowptr out of range at row "
                           : code == 3 ? "column index out of range in row "
                                       : "columns not strictly increasing in row ";
        fail(SPG_ERROR, what + std::to_string(row));
    }
}

void narrow_index(spg_ctx* ctx, const int64_t* d_in, int32_t* d_out, int64_t n) {
    if (n == 0) return;
    DBuf<unsigned long long> bad(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), ctx->stream));
    k_narrow<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(d_in, d_out, n, bad);
    SPG_LAUNCH_CHECK();
    unsigned long long h = 0;
    SPG_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) fail(SPG_PARAMETER_ERROR, "column index does not fit in 32 bits");
}

void widen_index(spg_ctx* ctx, const int32_t* d_in, int64_t* d_out, int64_t n) {
    if (n == 0) return;
    k_widen<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(d_in, d_out, n);
    SPG_LAUNCH_CHECK();
}

// C = A*B straight into host arrays (the reference's spgemm_local returns C
// by value, csr.cpp:132-165). A is multiplied in row batches (cuts[0..nb]);
// batch i's columns/values go down the host link on the aux streams while
// batch i+1 is multiplied on the context stream, so only the last batch's
// download is exposed. At most two batch products are alive on the device
// (batch i is freed once its download has finished, before batch i+2 is
// multiplied), so batches also bound the device memory C needs. Row pointers
// are rebased into one device array and fetched at the end.
int64_t spgemm_to_host(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const int64_t* cuts, int nb,
                       int64_t* h_rowptr, void* h_colind, int colind_width, double* h_values, int64_t cap) {
    if (a->ncols != b->nrows) fail(SPG_DIMENSION_ERROR, "spgemm: inner dimensions differ");
    constexpr size_t CH = size_t(64) << 20;
    const int64_t m = a->nrows;
    DBuf<int64_t> rp(ctx, m + 1);
    SPG_CUDA(cudaMemsetAsync(rp.get(), 0, sizeof(int64_t), ctx->stream));
    struct Part {
        spg_csr* c = nullptr;
        int64_t* wide = nullptr;
        cudaEvent_t ev[spg_ctx::NAUX + 1] = {};  // [0]: product ready; [1..]: downloads done per aux stream
    };
    std::deque<Part> live;
    auto retire = [&](Part& p) {  // wait for the part's downloads, then release it
        for (int s = 1; s <= spg_ctx::NAUX; ++s)
            if (p.ev[s]) cudaEventSynchronize(p.ev[s]);
        if (p.wide) dfree(ctx, p.wide);
        free_csr(p.c);
        for (auto e : p.ev)
            if (e) cudaEventDestroy(e);
    };
    auto cleanup = [&] {
        for (int i = 0; i < spg_ctx::NAUX; ++i) cudaStreamSynchronize(ctx->aux[i]);
        while (!live.empty()) {
            retire(live.front());
            live.pop_front();
        }
        cudaStreamSynchronize(ctx->stream);
    };
    int64_t off = 0;
    int chunk = 0;
    try {
        for (int i = 0; i < nb; ++i) {
            const int64_t r0 = cuts[i], r1 = cuts[i + 1];
            if (r1 <= r0) continue;
            if (live.size() >= 2) {
                retire(live.front());
                live.pop_front();
            }
            spg_csr* sub = extract(ctx, a, r0, r1, 0, a->ncols);
            live.emplace_back();
            Part& p = live.back();
            try {
                p.c = spgemm(ctx, sub, b);
            } catch (...) {
                free_csr(sub);
                live.pop_back();
                throw;
            }
            free_csr(sub);
            spg_csr* c = p.c;
            {
                KTime kt(ctx, "rebase_rowptr");
                k_rebase_rowptr<<<grid_for(ctx, r1 - r0), 256, 0, ctx->stream>>>(c->rowptr, r1 - r0, off,
                                                                                rp.get() + r0 + 1);
                SPG_LAUNCH_CHECK();
            }
            const int64_t n = c->nnz;
            if (off + n <= cap && n > 0) {
                const void* csrc = c->colind;
                size_t cw = sizeof(int32_t);
                if (colind_width == 8) {
                    p.wide = dalloc<int64_t>(ctx, n);
                    widen_index(ctx, c->colind, p.wide, n);
                    csrc = p.wide;
                    cw = sizeof(int64_t);
                }
                for (auto& e : p.ev) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                SPG_CUDA(cudaEventRecord(p.ev[0], ctx->stream));
                for (int s = 0; s < spg_ctx::NAUX; ++s) SPG_CUDA(cudaStreamWaitEvent(ctx->aux[s], p.ev[0], 0));
                auto down = [&](void* dst, const void* src, size_t bytes) {
                    for (size_t o = 0; o < bytes; o += CH, ++chunk)
                        SPG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                                                 std::min(CH, bytes - o), cudaMemcpyDeviceToHost,
                                                 ctx->aux[chunk % spg_ctx::NAUX]));
                };
                down(static_cast<char*>(h_colind) + off * cw, csrc, n * cw);
                down(h_values + off, c->values, n * sizeof(double));
                for (int s = 0; s < spg_ctx::NAUX; ++s) SPG_CUDA(cudaEventRecord(p.ev[s + 1], ctx->aux[s]));
            }
            off += n;
        }
        if (off <= cap) SPG_CUDA(cudaMemcpyAsync(h_rowptr, rp.get(), (m + 1) * sizeof(int64_t),
                                                 cudaMemcpyDeviceToHost, ctx->stream));
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    SPG_CUDA(cudaGetLastError());
    return off;
}

}  // namespace spgb
