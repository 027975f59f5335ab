// Local SpGEMM C = A*B on one B200 (sm_100a): the replacement of
// spgemm_local (reference csr.cpp:132-165).
//
// Algorithm: row-wise Gustavson, expressed as a per-row
// "bucketed ESC" (expand - sort - compress) in shared memory.
//
//   1. k_row_products  : products(i) = Σ_{k∈A_i} nnz(B_k)           (work per row)
//   2. scan            : exclusive prefix of products -> product offsets
//   3. k_tile_flags    : rows are cut into TILES of consecutive rows with
//                        ≤ 2*TILE_H products, ≤ TILE_RH rows and ≤ 2*TILE_EH A
//                        entries; rows over the caps are HEAVY (own path)
//   4. symbolic pass   : per tile/heavy row, exact nnz per row (columns only)
//   5. scan            : C rowptr
//   6. numeric pass    : same expansion with values; each output entry's
//                        contributions are summed in ascending inner index k
//                        with a separate multiply and add (no FMA), so values
//                        are bit-identical to the reference's serial kernel.
//
// Per tile (one CTA): products are expanded into smem (col, value) in
// A-entry order x (x increases with k inside a row), bucketed by a per-row
// monotone map of the column range into ~products/2 buckets (counting sort
// with smem atomics), each bucket is sorted by (col, x), duplicates are
// combined in x order, and the compacted row is written to C. Bucket order is
// row-major then column order, so the tile's output is one contiguous run of C.
#include <cub/device/device_scan.cuh>

#include <climits>

#include "block_scan.cuh"
#include "spg_internal.cuh"

namespace spgb {
namespace {

constexpr int NT = 256;              // threads per tile CTA
constexpr int TILE_H = 1024;         // product half-capacity (tile ≤ 2*TILE_H)
constexpr int TILE_P = 2 * TILE_H;   // product capacity
constexpr int TILE_RH = 128;         // rows per tile ≤ TILE_RH
constexpr int TILE_EH = 256;         // A entries per tile ≤ 2*TILE_EH
constexpr int TILE_E = 2 * TILE_EH;
constexpr int BUCKET_LOAD = 2;       // target products per bucket
constexpr int NB_MAX = TILE_P / BUCKET_LOAD + TILE_RH;

struct TileSmem {
    int32_t col[TILE_P];
    double val[TILE_P];
    uint16_t bkt[TILE_P];
    uint16_t perm[TILE_P];
    int64_t e_bst[TILE_E];
    double e_av[TILE_E];
    int32_t e_pre[TILE_E + 1];
    uint8_t e_row[TILE_E];
    int32_t r_pbase[TILE_RH + 1];
    int32_t r_bbase[TILE_RH + 1];
    int32_t r_minc[TILE_RH];
    int32_t r_maxc[TILE_RH];
    float r_scale[TILE_RH];
    int32_t b_off[NB_MAX + 1];
    int32_t b_cnt[NB_MAX + 1];
    int32_t ws[NT / 32 + 1];
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// ------------------------------------------------------------ row products
__global__ void k_row_products(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                               const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = 0;
        const int64_t e1 = arp[i + 1];
        for (int64_t e = arp[i]; e < e1; ++e) {
            const int32_t k = __ldg(acol + e);
            p += __ldg(brp + k + 1) - __ldg(brp + k);
        }
        prod[i] = p;
    }
}

__device__ __forceinline__ bool row_is_heavy(int64_t prod, int64_t nent) {
    return prod > TILE_H || nent > TILE_EH;
}

__device__ __forceinline__ int64_t tile_key(int64_t i, const int64_t* pex, const int64_t* arp) {
    return pex[i] / TILE_H + i / TILE_RH + arp[i] / TILE_EH;
}

// flags[i] = 1 when row i starts a tile; heavy rows appended to heavy_list.
__global__ void k_tile_flags(const int64_t* __restrict__ pex, const int64_t* __restrict__ arp, int64_t m,
                             int32_t* __restrict__ flags, int32_t* __restrict__ heavy_list,
                             int32_t* __restrict__ heavy_count) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        flags[i] = (i == 0 || tile_key(i, pex, arp) != tile_key(i - 1, pex, arp)) ? 1 : 0;
        if (row_is_heavy(pex[i + 1] - pex[i], arp[i + 1] - arp[i])) {
            const int slot = atomicAdd(heavy_count, 1);
            heavy_list[slot] = static_cast<int32_t>(i);
        }
    }
}

__global__ void k_tile_scatter(const int32_t* __restrict__ flags, const int64_t* __restrict__ pos, int64_t m,
                               int32_t* __restrict__ tile_start) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        if (flags[i]) tile_start[pos[i]] = static_cast<int32_t>(i);
        if (i == m - 1) tile_start[pos[m]] = static_cast<int32_t>(m);
    }
}

// Monotone map of a column into the row's bucket range.
__device__ __forceinline__ int bucket_of(int32_t col, int32_t minc, float scale, int nb) {
    int b = static_cast<int>(static_cast<float>(col - minc) * scale);
    return b < nb - 1 ? b : nb - 1;
}

// Sorts perm[lo,hi) by (col[x], x) with insertion sort; returns the number of
// distinct columns. Buckets hold ~BUCKET_LOAD entries on average.
template <typename PermT, typename ColP>
__device__ __forceinline__ int sort_bucket(PermT* perm, int64_t lo, int64_t hi, const ColP* col) {
    for (int64_t a = lo + 1; a < hi; ++a) {
        const PermT xa = perm[a];
        const int32_t ca = col[xa];
        int64_t b = a - 1;
        while (b >= lo) {
            const PermT xb = perm[b];
            const int32_t cb = col[xb];
            if (cb < ca || (cb == ca && xb < xa)) break;
            perm[b + 1] = xb;
            --b;
        }
        perm[b + 1] = xa;
    }
    int u = 0;
    int32_t last = INT_MIN;
    for (int64_t a = lo; a < hi; ++a) {
        const int32_t c = col[perm[a]];
        u += (a == lo || c != last);
        last = c;
    }
    return u;
}

// --------------------------------------------------------------- tile kernel
template <bool NUMERIC>
__global__ void __launch_bounds__(NT) k_tile(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                             const double* __restrict__ aval, const int64_t* __restrict__ brp,
                                             const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                             const int64_t* __restrict__ pex, const int32_t* __restrict__ tile_start,
                                             int ntiles, int64_t* __restrict__ row_nnz,
                                             const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                             double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem& s = *reinterpret_cast<TileSmem*>(smem_raw);
    const int tid = threadIdx.x;

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = tile_start[t];
        const int64_t r1 = tile_start[t + 1];
        int64_t rl1 = r1;  // end of light rows; a heavy row can only be last
        if (row_is_heavy(pex[r1] - pex[r1 - 1], arp[r1] - arp[r1 - 1])) rl1 = r1 - 1;
        const int nr = static_cast<int>(rl1 - r0);
        if (nr <= 0) continue;
        const int64_t e0 = arp[r0];
        const int ne = static_cast<int>(arp[rl1] - e0);
        const int64_t pbase0 = pex[r0];
        const int ptile = static_cast<int>(pex[rl1] - pbase0);

        // P0: row metadata, entry -> row map
        for (int r = tid; r < nr; r += NT) {
            s.r_pbase[r] = static_cast<int32_t>(pex[r0 + r] - pbase0);
            s.r_minc[r] = INT_MAX;
            s.r_maxc[r] = -1;
            const int ea = static_cast<int>(arp[r0 + r] - e0), eb = static_cast<int>(arp[r0 + r + 1] - e0);
            for (int e = ea; e < eb; ++e) s.e_row[e] = static_cast<uint8_t>(r);
        }
        if (tid == 0) s.r_pbase[nr] = ptile;
        __syncthreads();

        // P1: A entries -> B row spans, column range per row, product prefix
        {
            constexpr int EI = TILE_E / NT;
            int lens[EI];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < EI; ++q) {
                const int e = tid * EI + q;
                lens[q] = 0;
                if (e < ne) {
                    const int32_t k = acol[e0 + e];
                    const int64_t bs = brp[k], be = brp[k + 1];
                    s.e_bst[e] = bs;
                    s.e_av[e] = aval[e0 + e];
                    lens[q] = static_cast<int>(be - bs);
                    if (be > bs) {
                        const int r = s.e_row[e];
                        atomicMin(&s.r_minc[r], bcol[bs]);
                        atomicMax(&s.r_maxc[r], bcol[be - 1]);
                    }
                }
                sum += lens[q];
            }
            int total;
            int pre = block_exclusive_scan<NT>(sum, &total, s.ws);
#pragma unroll
            for (int q = 0; q < EI; ++q) {
                const int e = tid * EI + q;
                if (e < ne) s.e_pre[e] = pre;
                pre += lens[q];
            }
            if (tid == 0) s.e_pre[ne] = total;
        }
        __syncthreads();

        // P2: bucket ranges per row
        {
            int nb = 0;
            if (tid < nr) {
                const int pr = s.r_pbase[tid + 1] - s.r_pbase[tid];
                nb = (pr + BUCKET_LOAD - 1) / BUCKET_LOAD;
                if (pr > 0) {
                    const int64_t range = int64_t(s.r_maxc[tid]) - s.r_minc[tid] + 1;
                    s.r_scale[tid] = static_cast<float>(nb) / static_cast<float>(range);
                }
            }
            static_assert(TILE_RH <= NT, "one thread per row");
            int total;
            const int pre = block_exclusive_scan<NT>(nb, &total, s.ws);
            if (tid < nr) s.r_bbase[tid] = pre;
            if (tid == 0) s.r_bbase[nr] = total;
            for (int b = tid; b <= total; b += NT) s.b_cnt[b] = 0;
        }
        __syncthreads();
        const int nbt = s.r_bbase[nr];

        // P3: expand products into smem and count buckets
        for (int x = tid; x < ptile; x += NT) {
            int lo = 0, hi = ne;  // largest e with e_pre[e] <= x
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s.e_pre[mid] <= x) lo = mid; else hi = mid;
            }
            const int e = lo;
            const int64_t u = s.e_bst[e] + (x - s.e_pre[e]);
            const int32_t c = bcol[u];
            const int r = s.e_row[e];
            const int nb = s.r_bbase[r + 1] - s.r_bbase[r];
            const int b = s.r_bbase[r] + bucket_of(c, s.r_minc[r], s.r_scale[r], nb);
            s.col[x] = c;
            s.bkt[x] = static_cast<uint16_t>(b);
            if (NUMERIC) s.val[x] = dmul(s.e_av[e], bval[u]);
            atomicAdd(&s.b_cnt[b], 1);
        }
        __syncthreads();

        // P4: bucket offsets
        block_scan_array<NT, (NB_MAX + NT) / NT, int32_t>(s.b_cnt, nbt, s.ws);
        for (int b = tid; b <= nbt; b += NT) {
            s.b_off[b] = s.b_cnt[b];
            s.b_cnt[b] = 0;
        }
        __syncthreads();

        // P5: scatter product ids into buckets
        for (int x = tid; x < ptile; x += NT) {
            const int b = s.bkt[x];
            const int pos = s.b_off[b] + atomicAdd(&s.b_cnt[b], 1);
            s.perm[pos] = static_cast<uint16_t>(x);
        }
        __syncthreads();

        // P6: sort each bucket by (col, x); count distinct columns
        for (int b = tid; b < nbt; b += NT) s.b_cnt[b] = sort_bucket(s.perm, s.b_off[b], s.b_off[b + 1], s.col);
        __syncthreads();
        block_scan_array<NT, (NB_MAX + NT) / NT, int32_t>(s.b_cnt, nbt, s.ws);  // -> unique offsets

        if (!NUMERIC) {
            for (int r = tid; r < nr; r += NT) row_nnz[r0 + r] = s.b_cnt[s.r_bbase[r + 1]] - s.b_cnt[s.r_bbase[r]];
        } else {
            const int64_t obase = crp[r0];
            for (int b = tid; b < nbt; b += NT) {
                int64_t o = obase + s.b_cnt[b];
                const int lo = s.b_off[b], hi = s.b_off[b + 1];
                int a = lo;
                while (a < hi) {
                    const int x = s.perm[a];
                    const int32_t c = s.col[x];
                    double sum = dadd(0.0, s.val[x]);
                    ++a;
                    while (a < hi && s.col[s.perm[a]] == c) {
                        sum = dadd(sum, s.val[s.perm[a]]);
                        ++a;
                    }
                    ccol[o] = c;
                    cval[o] = sum;
                    ++o;
                }
            }
        }
        __syncthreads();
    }
}

// -------------------------------------------------------------- heavy rows
// One CTA per heavy row; the same bucketed ESC with the arrays in a global
// workspace slice of `cap` products (the row's products).
struct HeavyWs {
    int64_t* e_pre;   // per row: nent+1
    int32_t* col;     // per row: prod
    double* val;      // per row: prod
    int32_t* bkt;     // per row: prod
    int32_t* perm;    // per row: prod
    int64_t* b_off;   // per row: nb+1
    int64_t* b_cnt;   // per row: nb+1
};

template <bool NUMERIC>
__global__ void __launch_bounds__(NT) k_heavy(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                              const double* __restrict__ aval, const int64_t* __restrict__ brp,
                                              const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                              const int32_t* __restrict__ rows, const int64_t* __restrict__ p_off,
                                              const int64_t* __restrict__ e_off, const int64_t* __restrict__ b_offs,
                                              HeavyWs ws, int64_t* __restrict__ row_nnz,
                                              const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                              double* __restrict__ cval) {
    __shared__ int64_t wsc[NT / 32 + 1];
    __shared__ int32_t s_minc, s_maxc;
    __shared__ float s_scale;
    const int h = blockIdx.x;
    const int64_t i = rows[h];
    const int tid = threadIdx.x;
    const int64_t ea = arp[i], ne = arp[i + 1] - ea;
    int64_t* e_pre = ws.e_pre + e_off[h];
    const int64_t pofs = p_off[h];
    int32_t* col = ws.col + pofs;
    double* val = ws.val + pofs;
    int32_t* bkt = ws.bkt + pofs;
    int32_t* perm = ws.perm + pofs;
    int64_t* b_off = ws.b_off + b_offs[h];
    int64_t* b_cnt = ws.b_cnt + b_offs[h];
    const int64_t nb = b_offs[h + 1] - b_offs[h] - 1;

    if (tid == 0) {
        s_minc = INT_MAX;
        s_maxc = -1;
    }
    __syncthreads();
    for (int64_t e = tid; e < ne; e += NT) {
        const int32_t k = acol[ea + e];
        const int64_t bs = brp[k], be = brp[k + 1];
        e_pre[e] = be - bs;
        if (be > bs) {
            atomicMin(&s_minc, bcol[bs]);
            atomicMax(&s_maxc, bcol[be - 1]);
        }
    }
    for (int64_t b = tid; b <= nb; b += NT) b_cnt[b] = 0;
    __syncthreads();
    block_scan_array<NT, 4, int64_t>(e_pre, ne, wsc);
    const int64_t prod = e_pre[ne];
    if (tid == 0) s_scale = static_cast<float>(nb) / static_cast<float>(int64_t(s_maxc) - s_minc + 1);
    __syncthreads();
    const int32_t minc = s_minc;
    const float scale = s_scale;

    for (int64_t x = tid; x < prod; x += NT) {
        int64_t lo = 0, hi = ne;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (e_pre[mid] <= x) lo = mid; else hi = mid;
        }
        const int64_t u = brp[acol[ea + lo]] + (x - e_pre[lo]);
        const int32_t c = bcol[u];
        int64_t b = static_cast<int64_t>(static_cast<float>(c - minc) * scale);
        if (b > nb - 1) b = nb - 1;
        col[x] = c;
        bkt[x] = static_cast<int32_t>(b);
        if (NUMERIC) val[x] = dmul(aval[ea + lo], bval[u]);
        atomicAdd(reinterpret_cast<unsigned long long*>(b_cnt + b), 1ull);
    }
    __syncthreads();
    block_scan_array<NT, 4, int64_t>(b_cnt, nb, wsc);
    for (int64_t b = tid; b <= nb; b += NT) {
        b_off[b] = b_cnt[b];
        b_cnt[b] = 0;
    }
    __syncthreads();
    for (int64_t x = tid; x < prod; x += NT) {
        const int32_t b = bkt[x];
        const int64_t pos = b_off[b] + static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long*>(b_cnt + b), 1ull));
        perm[pos] = static_cast<int32_t>(x);
    }
    __syncthreads();
    for (int64_t b = tid; b < nb; b += NT) b_cnt[b] = sort_bucket(perm, b_off[b], b_off[b + 1], col);
    __syncthreads();
    block_scan_array<NT, 4, int64_t>(b_cnt, nb, wsc);
    if (!NUMERIC) {
        if (tid == 0) row_nnz[i] = b_cnt[nb];
    } else {
        const int64_t obase = crp[i];
        for (int64_t b = tid; b < nb; b += NT) {
            int64_t o = obase + b_cnt[b];
            const int64_t lo = b_off[b], hi = b_off[b + 1];
            int64_t a = lo;
            while (a < hi) {
                const int32_t x = perm[a];
                const int32_t c = col[x];
                double sum = dadd(0.0, val[x]);
                ++a;
                while (a < hi && col[perm[a]] == c) {
                    sum = dadd(sum, val[perm[a]]);
                    ++a;
                }
                ccol[o] = c;
                cval[o] = sum;
                ++o;
            }
        }
    }
}

__global__ void k_heavy_info(const int32_t* __restrict__ rows, int n, const int64_t* __restrict__ prod,
                             const int64_t* __restrict__ arp, int64_t* __restrict__ out) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x) {
        const int64_t i = rows[h];
        out[2 * h] = prod[i];
        out[2 * h + 1] = arp[i + 1] - arp[i];
    }
}


int grid_for(spg_ctx* ctx, int64_t n, int bs = 256) {
    const int64_t want = (n + bs - 1) / bs;
    const int64_t cap = int64_t(ctx->num_sms) * 16;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void exclusive_scan_i64(spg_ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
    // out[0] = 0, out[1..n] = inclusive prefix of in[0..n): out[n] is the total.
    SPG_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), ctx->stream));
    if (n == 0) return;
    size_t tmp = 0;
    SPG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, n, ctx->stream));
    DBuf<unsigned char> t(ctx, tmp);
    SPG_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, in, out + 1, n, ctx->stream));
}

int64_t spgemm_products(spg_ctx* ctx, const spg_csr* a, const spg_csr* b) {
    if (a->ncols != b->nrows) fail(SPG_DIMENSION_ERROR, "spgemm: a.ncols != b.nrows");
    const int64_t m = a->nrows;
    if (m == 0 || a->nnz == 0) return 0;
    DBuf<int64_t> prod(ctx, m), pex(ctx, m + 1);
    k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod);
    SPG_LAUNCH_CHECK();
    exclusive_scan_i64(ctx, prod, pex, m);
    return read_scalar(ctx, pex.get() + m);
}

spg_csr* spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b) {
    if (a->ncols != b->nrows)
        fail(SPG_DIMENSION_ERROR,
             "spgemm: a.ncols=" + std::to_string(a->ncols) + " != b.nrows=" + std::to_string(b->nrows));
    const int64_t m = a->nrows, n = b->ncols;
    if (m == 0 || a->nnz == 0 || b->nnz == 0) return new_csr(ctx, m, n, 0);

    // 1-2: products per row and their prefix
    DBuf<int64_t> prod(ctx, m), pex(ctx, m + 1);
    {
        KTime kt(ctx, "row_products");
        k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod);
        SPG_LAUNCH_CHECK();
    }
    exclusive_scan_i64(ctx, prod, pex, m);

    // 3: tiles + heavy rows
    DBuf<int32_t> flags(ctx, m), heavy(ctx, m), counters(ctx, 2);
    DBuf<int64_t> tpos(ctx, m + 1);
    SPG_CUDA(cudaMemsetAsync(counters.get(), 0, 2 * sizeof(int32_t), ctx->stream));
    {
        KTime kt(ctx, "tile_plan");
        k_tile_flags<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(pex, a->rowptr, m, flags, heavy, counters);
        SPG_LAUNCH_CHECK();
    }
    {
        size_t tmp = 0;
        SPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flags.get(), tpos.get(), m, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        SPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, flags.get(), tpos.get(), m, ctx->stream));
    }
    // tpos[m] = number of tiles = tpos[m-1] + flags[m-1]
    int64_t host[4];
    {
        int32_t hflag = 0, hheavy = 0;
        SPG_CUDA(cudaMemcpyAsync(&host[0], tpos.get() + m - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(&hflag, flags.get() + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(&hheavy, counters.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        host[1] = host[0] + hflag;
        host[2] = hheavy;
    }
    const int64_t ntiles = host[1];
    const int nheavy = static_cast<int>(host[2]);
    SPG_CUDA(cudaMemcpyAsync(tpos.get() + m, &host[1], sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    DBuf<int32_t> tile_start(ctx, ntiles + 1);
    k_tile_scatter<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(flags, tpos, m, tile_start);
    SPG_LAUNCH_CHECK();

    // heavy-row workspace plan (host side; heavy rows are few)
    std::vector<int32_t> hrows(nheavy);
    std::vector<int64_t> hp_off(nheavy + 1, 0), he_off(nheavy + 1, 0), hb_off(nheavy + 1, 0);
    if (nheavy) {
        SPG_CUDA(cudaMemcpyAsync(hrows.data(), heavy.get(), nheavy * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        DBuf<int64_t> info(ctx, 2 * int64_t(nheavy));
        k_heavy_info<<<grid_for(ctx, nheavy), 256, 0, ctx->stream>>>(heavy, nheavy, prod, a->rowptr, info);
        SPG_LAUNCH_CHECK();
        std::vector<int64_t> hinfo(2 * size_t(nheavy));
        SPG_CUDA(cudaMemcpyAsync(hinfo.data(), info.get(), hinfo.size() * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<int64_t> hprod(nheavy), hnent(nheavy);
        for (int h = 0; h < nheavy; ++h) {
            hprod[h] = hinfo[2 * h];
            hnent[h] = hinfo[2 * h + 1];
        }
        for (int h = 0; h < nheavy; ++h) {
            hp_off[h + 1] = hp_off[h] + hprod[h];
            he_off[h + 1] = he_off[h] + hnent[h] + 1;
            const int64_t nb = (hprod[h] + BUCKET_LOAD - 1) / BUCKET_LOAD;
            hb_off[h + 1] = hb_off[h] + nb + 1;
        }
    }
    DBuf<int32_t> d_hrows(ctx, nheavy);
    DBuf<int64_t> d_hp(ctx, nheavy + 1), d_he(ctx, nheavy + 1), d_hb(ctx, nheavy + 1);
    HeavyWs hws{};
    DBuf<int64_t> w_epre(ctx, he_off[nheavy]);
    DBuf<int32_t> w_col(ctx, hp_off[nheavy]), w_bkt(ctx, hp_off[nheavy]), w_perm(ctx, hp_off[nheavy]);
    DBuf<double> w_val(ctx, hp_off[nheavy]);
    DBuf<int64_t> w_boff(ctx, hb_off[nheavy]), w_bcnt(ctx, hb_off[nheavy]);
    if (nheavy) {
        SPG_CUDA(cudaMemcpyAsync(d_hrows.get(), hrows.data(), nheavy * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(d_hp.get(), hp_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(d_he.get(), he_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(d_hb.get(), hb_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        hws = HeavyWs{w_epre, w_col, w_val, w_bkt, w_perm, w_boff, w_bcnt};
    }

    const size_t smem = sizeof(TileSmem);
    if (!ctx->tile_attr_set) {
        SPG_CUDA(cudaFuncSetAttribute(k_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPG_CUDA(cudaFuncSetAttribute(k_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ctx->tile_attr_set = true;
    }
    int occ = 1;
    SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile<true>, NT, smem));
    const int tgrid = static_cast<int>(std::min<int64_t>(ntiles, int64_t(ctx->num_sms) * std::max(occ, 1) * 8));

    // 4: symbolic
    DBuf<int64_t> rnnz(ctx, m + 1);
    SPG_CUDA(cudaMemsetAsync(rnnz.get(), 0, (m + 1) * sizeof(int64_t), ctx->stream));
    {
        KTime kt(ctx, "spgemm_symbolic");
        if (ntiles > 0)
            k_tile<false><<<tgrid, NT, smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                             b->values, pex, tile_start, static_cast<int>(ntiles),
                                                             rnnz, nullptr, nullptr, nullptr);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<false><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                           b->values, d_hrows, d_hp, d_he, d_hb, hws, rnnz, nullptr,
                                                           nullptr, nullptr);
        SPG_LAUNCH_CHECK();
    }
    // 5: rowptr of C
    spg_csr* c = new_csr(ctx, m, n, -1);
    exclusive_scan_i64(ctx, rnnz, c->rowptr, m);
    c->nnz = read_scalar(ctx, c->rowptr + m);
    c->colind = dalloc<int32_t>(ctx, c->nnz);
    c->values = dalloc<double>(ctx, c->nnz);

    // 6: numeric
    {
        KTime kt(ctx, "spgemm_numeric");
        if (ntiles > 0)
            k_tile<true><<<tgrid, NT, smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                            b->values, pex, tile_start, static_cast<int>(ntiles),
                                                            nullptr, c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<true><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                          b->values, d_hrows, d_hp, d_he, d_hb, hws, nullptr,
                                                          c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    return c;
}

}  // namespace spgb
