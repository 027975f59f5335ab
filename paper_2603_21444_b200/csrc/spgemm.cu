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
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <climits>

#include "block_scan.cuh"
#include "spg_internal.cuh"

namespace spgb {
namespace {

// ----------------------------------------------------------- row classes
// WARP rows: ≤ 32 A entries and ≤ WARP_P products — one warp per row, the
// products live in registers, one bucket-sorted copy in the warp's smem slice.
// CTA rows: ≤ CTA_E entries and ≤ CTA_P products — one CTA per row in smem.
// HEAVY rows: the rest — one CTA per row with the arrays in global memory.
#ifndef SPG_WARP_MINB
#define SPG_WARP_MINB 2
#endif
constexpr int WARP_NJ = 16;                // products per lane
constexpr int WARP_P = 32 * WARP_NJ;       // 512
constexpr int NT = 256;                    // threads per CTA
constexpr int CTA_P = 4096;
constexpr int CTA_E = 1024;
constexpr int BUCKET_LOAD = 2;             // target products per bucket
constexpr int CTA_NB = CTA_P / BUCKET_LOAD + 1;

enum RowClass : int8_t { RC_EMPTY = 0, RC_WARP = 1, RC_CTA = 2, RC_HEAVY = 3 };

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// ------------------------------------------------------------ row products
// products(i) = Σ_{k∈A_i} nnz(B_k). Rows are appended (warp-aggregated, so runs
// of consecutive rows stay together) to the list of their class:
// 0: warp rows ≤ 256 products, 1: warp rows ≤ 512, 2: CTA rows, 3: heavy rows.
__global__ void k_row_products(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                               const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod,
                               int32_t* __restrict__ lists, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = (blockIdx.x * int64_t(blockDim.x)) & ~int64_t(31); base < m;
         base += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = base + (threadIdx.x & ~31) + lane;
        int cls = -1;
        if (i < m) {
            int64_t p = 0;
            const int64_t e0 = arp[i], e1 = arp[i + 1];
            for (int64_t e = e0; e < e1; ++e) {
                const int32_t k = __ldg(acol + e);
                p += __ldg(brp + k + 1) - __ldg(brp + k);
            }
            prod[i] = p;
            const int64_t ne = e1 - e0;
            if (p > 0) {
                if (ne <= 32 && p <= 256) cls = 0;
                else if (ne <= 32 && p <= WARP_P) cls = 1;
                else if (ne <= CTA_E && p <= CTA_P) cls = 2;
                else cls = 3;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned mk = __ballot_sync(0xffffffffu, cls == c);
            if (!mk) continue;
            const int leader = __ffs(mk) - 1;
            int b0 = 0;
            if (lane == leader) b0 = atomicAdd(counts + c, __popc(mk));
            b0 = __shfl_sync(0xffffffffu, b0, leader);
            if (cls == c) lists[c * m + b0 + __popc(mk & ((1u << lane) - 1))] = static_cast<int32_t>(i);
        }
    }
}

// Monotone map column -> [0, nb): high bits of the column scaled by nb.
__device__ __forceinline__ int bucket_of(uint32_t col, int cshift, int nb) {
    return static_cast<int>(__umulhi(col << cshift, static_cast<uint32_t>(nb)));
}

// Warp-cooperative A-row setup. The row's entries whose B row is nonempty are
// compacted onto lanes 0..mn-1 (ascending k); lane t holds base_t = (B row
// start) - (product prefix), so product x of entry t sits at B position base_t + x.
struct RowEntries {
    int64_t base;
    double av;
    int pre;  // exclusive product prefix; INT_MAX on lanes >= mn
    int p;    // products of the row
};

// Raw A-row fetch of one lane: its entry's B row span and A value.
struct RowFetch {
    int64_t bs;
    double av;
    int len;
};

__device__ __forceinline__ RowEntries make_row(const RowFetch& f, int lane) {
    const int len = f.len;
    const unsigned nz = __ballot_sync(0xffffffffu, len > 0);
    const int mn = __popc(nz);
    const int src = static_cast<int>(__fns(nz, 0, lane + 1)) & 31;
    int lc = __shfl_sync(0xffffffffu, len, src);
    const int64_t bc = __shfl_sync(0xffffffffu, f.bs, src);
    RowEntries r;
    r.av = __shfl_sync(0xffffffffu, f.av, src);
    if (lane >= mn) lc = 0;
    int inc = lc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    r.p = __shfl_sync(0xffffffffu, inc, 31);
    const int pre = inc - lc;
    r.base = bc - pre;
    r.pre = lane < mn ? pre : INT_MAX;
    return r;
}

template <bool VALS>
__device__ __forceinline__ RowEntries load_row(const int32_t* __restrict__ acol, const double* __restrict__ aval,
                                               const int64_t* __restrict__ brp, int64_t e0, int m, int lane) {
    RowFetch f{0, 0.0, 0};
    if (lane < m) {
        const int32_t k = __ldg(acol + e0 + lane);
        if (VALS) f.av = __ldg(aval + e0 + lane);
        f.bs = __ldg(brp + k);
        f.len = static_cast<int>(__ldg(brp + k + 1) - f.bs);
    }
    return make_row(f, lane);
}

// Software pipeline over a row list. While row t is processed: the list entry
// of row t+3, the A row pointers of row t+2 and the A entries of row t+1 are in
// flight, and the B row spans of row t+1 are requested after row t's gathers.
// No loaded value is consumed in the iteration that issued it.
template <bool VALS>
struct RowPipe {
    const int64_t* arp;
    const int32_t* acol;
    const double* aval;
    const int64_t* brp;
    const int32_t* list;
    int64_t n, nw;
    int32_t i1, i2, i3;  // row ids of t+1, t+2, t+3 (-1 past the end)
    int64_t e1, f1;      // arp[i1], arp[i1 + 1]
    int64_t e2, f2;      // arp[i2], arp[i2 + 1]
    int32_t k1;          // A column of this lane's entry in row t+1
    double av1;

    __device__ __forceinline__ int32_t row_at(int64_t t) const { return t < n ? list[t] : -1; }
    __device__ __forceinline__ void ptrs(int32_t i, int64_t& e, int64_t& f) const {
        e = 0;
        f = 0;
        if (i >= 0) {
            e = arp[i];
            f = arp[i + 1];
        }
    }
    __device__ __forceinline__ void entries(int lane) {
        k1 = 0;
        av1 = 0.0;
        if (i1 >= 0 && lane < f1 - e1) {
            k1 = __ldg(acol + e1 + lane);
            if (VALS) av1 = __ldg(aval + e1 + lane);
        }
    }
    // B row spans of row t+1 (consumes k1, issued one phase earlier)
    __device__ __forceinline__ RowFetch spans(int lane) const {
        RowFetch f{0, av1, 0};
        if (i1 >= 0 && lane < f1 - e1) {
            f.bs = __ldg(brp + k1);
            f.len = static_cast<int>(__ldg(brp + k1 + 1) - f.bs);
        }
        return f;
    }
    // prime: returns row t's fetch (blocking) and its id
    __device__ __forceinline__ RowFetch start(int64_t t, int lane, int32_t& i0) {
        i1 = row_at(t);
        ptrs(i1, e1, f1);
        entries(lane);
        const RowFetch f = spans(lane);
        i0 = i1;
        i1 = row_at(t + nw);
        i2 = row_at(t + 2 * nw);
        i3 = row_at(t + 3 * nw);
        ptrs(i1, e1, f1);
        ptrs(i2, e2, f2);
        entries(lane);
        return f;
    }
    // row t+1 becomes current: shift the stages and issue the next loads
    __device__ __forceinline__ void advance(int64_t t_next, int lane) {
        i1 = i2;
        e1 = e2;
        f1 = f2;
        i2 = i3;
        ptrs(i2, e2, f2);
        i3 = row_at(t_next + 3 * nw);
        entries(lane);
    }
};

// Entry of product x = 32*j + lane: t0 = entry covering 32*j (ballot), plus the
// entries that start inside the chunk before x (one OR-reduction of start bits).
__device__ __forceinline__ int chunk_entry(int pre, int j, int lane) {
    const int c0 = 32 * j;
    const int t0 = __popc(__ballot_sync(0xffffffffu, pre <= c0)) - 1;
    const int rel = pre - c0;
    const unsigned sm = __reduce_or_sync(0xffffffffu, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
    return t0 + __popc(sm & ((2u << lane) - 1u));
}

// Per-warp smem slice of the numeric kernel for rows of ≤ 32*NJ products:
// products in bucket order and the 2p bucket counters / offsets.
template <int NJ>
struct WarpSliceT {
    static constexpr int P = 32 * NJ;
    int32_t col[P];
    double val[P];
    int64_t e_base[32];  // per entry: B position of product x is e_base[t] + x
    double e_av[32];
    uint16_t x[P];
    uint8_t e_of[P];     // entry of product x
    int32_t off[2 * P + 1];
    int32_t big[P / 3 + 1];  // starts of buckets holding >= 3 products
    int32_t nbig;
};

// Entry tables of a row in the warp's smem: lane t < mn owns entry t and fills
// e_of over its product range. Replaces per-product warp collectives.
template <bool VALS>
__device__ __forceinline__ void fill_entries(const RowEntries& re, int64_t* e_base, double* e_av, uint8_t* e_of,
                                             int lane) {
    const int hi = __shfl_down_sync(0xffffffffu, re.pre, 1);
    if (re.pre != INT_MAX) {
        e_base[lane] = re.base;
        if (VALS) e_av[lane] = re.av;
        const int end = (lane == 31 || hi == INT_MAX) ? re.p : hi;
        for (int x = re.pre; x < end; ++x) e_of[x] = static_cast<uint8_t>(lane);
    }
    __syncwarp();
}
using WarpSlice = WarpSliceT<WARP_NJ>;

// Row classes of the warp kernels: NJ = 8 for products in [1, 256], NJ = 16
// for (256, 512] (separate kernels so the small class runs at higher occupancy).
template <int NJ>
__device__ __forceinline__ bool in_class(int64_t p, int ne) {
    return ne <= 32 && p > (NJ == 8 ? 0 : 256) && p <= 32 * NJ;
}

// --------------------------------------------------------- warp symbolic
// Distinct columns per row via an open-addressing set in the warp's smem.
template <int WPB, int NJ>
__global__ void __launch_bounds__(WPB * 32, 4) k_warp_symbolic(const int64_t* __restrict__ arp,
                                                            const int32_t* __restrict__ acol,
                                                            const int64_t* __restrict__ brp,
                                                            const int32_t* __restrict__ bcol,
                                                            const int32_t* __restrict__ list,
                                                            const int32_t* __restrict__ count,
                                                            int64_t* __restrict__ row_nnz) {
    constexpr int T = 2 * 32 * NJ;
    __shared__ int32_t table[WPB][T];
    __shared__ int64_t s_base[WPB][32];
    __shared__ uint8_t s_of[WPB][32 * NJ];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t* tab = table[w];
    const int64_t gw = blockIdx.x * int64_t(WPB) + w, nw = int64_t(gridDim.x) * WPB;
    RowPipe<false> pipe{arp, acol, nullptr, brp, list, *count, nw};
    int32_t i;
    RowFetch cur = pipe.start(gw, lane, i);
    for (int64_t t = gw; t < pipe.n; t += nw) {
        const RowEntries re = make_row(cur, lane);
        const int p = re.p;
        const int lg = max(6, 32 - __clz(2 * p - 1));  // 2^lg >= 2p
        const int TT = 1 << lg;
        for (int q = lane; q < TT; q += 32) tab[q] = -1;
        __syncwarp();
        fill_entries<false>(re, s_base[w], nullptr, s_of[w], lane);
        int32_t cols[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int x = 32 * j + lane;
            cols[j] = x < p ? __ldg(bcol + s_base[w][s_of[w][x]] + x) : -1;
        }
        const RowFetch nxt = pipe.spans(lane);
        int fresh = 0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            if (cols[j] < 0) continue;
            uint32_t h = (static_cast<uint32_t>(cols[j]) * 0x9E3779B1u) >> (32 - lg);
            while (true) {
                const int32_t old = atomicCAS(&tab[h], -1, cols[j]);
                if (old == -1) { ++fresh; break; }
                if (old == cols[j]) break;
                h = (h + 1) & (TT - 1);
            }
        }
        __syncwarp();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
        if (lane == 0) row_nnz[i] = fresh;
        const int32_t inext = pipe.i1;
        pipe.advance(t + nw, lane);
        cur = nxt;
        i = inext;
        __syncwarp();
    }
}

// ---------------------------------------------------------- warp numeric
// Products are gathered into registers (x = 32j + lane, ascending k within the
// row), counted into 2p column buckets, and scattered once into the warp's smem
// slice in bucket order. Singleton buckets are final, pairs are ordered by one
// compare in registers, and buckets of ≥ 3 are insertion-sorted by (col, x)
// from a short list: the slice then holds the row sorted by column. Runs of
// equal columns (duplicates; rare for ER) are summed in x order (= ascending
// k, separate mul and add) and compacted in place, so values are bit-identical
// to the reference. Returns nnz; the row is S.col[0..nnz), S.val[0..nnz).
// Warp-collective operations are never under a data-dependent branch.
template <int NJ>
__device__ __forceinline__ int warp_row_sorted(WarpSliceT<NJ>& S, const RowEntries& re,
                                               const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                               int cshift, int lane) {
    const int p = re.p;
    const int nb = 2 * p;  // ~0.5 products per bucket
    for (int q = lane; q <= nb; q += 32) S.off[q] = 0;

    fill_entries<true>(re, S.e_base, S.e_av, S.e_of, lane);
    // expand: every gather issued before any is consumed
    int32_t col[NJ];
    double val[NJ];
    int aux[NJ];  // entry index, then the bucket's first position, then the target
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int x = 32 * j + lane;
        col[j] = 0;
        val[j] = 0.0;
        aux[j] = 0;
        if (x < p) {
            const int t = S.e_of[x];
            const int64_t u = S.e_base[t] + x;
            aux[j] = t;
            col[j] = __ldg(bcol + u);
            val[j] = __ldg(bval + u);
        }
    }
    int slot[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        slot[j] = -1;
        if (32 * j + lane < p) {
            val[j] = dmul(S.e_av[aux[j]], val[j]);
            slot[j] = atomicAdd(&S.off[bucket_of(col[j], cshift, nb)], 1);
        }
    }
    __syncwarp();
    // exclusive scan of the nb counts (contiguous block per lane); off[nb] = p
    {
        const int per = (nb + 1 + 31) >> 5;
        const int b0 = lane * per;
        int s = 0;
        for (int q = 0; q < per; ++q) s += (b0 + q < nb) ? S.off[b0 + q] : 0;
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        int pre = inc - s;
        __syncwarp();
        for (int q = 0; q < per; ++q) {
            const int b = b0 + q;
            if (b <= nb) {
                const int c = b < nb ? S.off[b] : 0;
                S.off[b] = pre;
                pre += c;
            }
        }
        if (lane == 0) S.nbig = 0;
    }
    __syncwarp();
    // scatter into bucket order; remember each product's bucket start
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (slot[j] >= 0) {
            const int lo = S.off[bucket_of(col[j], cshift, nb)];
            aux[j] = lo;
            S.col[lo + slot[j]] = col[j];
            S.val[lo + slot[j]] = val[j];
            S.x[lo + slot[j]] = static_cast<uint16_t>(32 * j + lane);
        }
    }
    __syncwarp();
    bool dup = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        int dst = -1;
        if (slot[j] >= 0) {
            const int lo = aux[j];
            const int sz = S.off[bucket_of(col[j], cshift, nb) + 1] - lo;
            if (sz == 2) {
                const int other = lo + 1 - slot[j];
                const int32_t pc = S.col[other];
                const bool eq = pc == col[j];
                dup |= eq;
                const int r = (pc < col[j] || (eq && S.x[other] < 32 * j + lane)) ? 1 : 0;
                if (r != slot[j]) dst = lo + r;
            } else if (sz > 2 && slot[j] == 0) {
                S.big[atomicAdd(&S.nbig, 1)] = lo;
            }
        }
        aux[j] = dst;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NJ; ++j)
        if (aux[j] >= 0) {
            S.col[aux[j]] = col[j];
            S.val[aux[j]] = val[j];
        }
    const int nbig = S.nbig;
    for (int k = lane; k < nbig; k += 32) {
        const int lo = S.big[k];
        const int hi = S.off[bucket_of(S.col[lo], cshift, nb) + 1];
        for (int q = lo + 1; q < hi; ++q) {
            const int32_t cq = S.col[q];
            const double vq = S.val[q];
            const uint16_t xq = S.x[q];
            int r = q - 1;
            while (r >= lo && (S.col[r] > cq || (S.col[r] == cq && S.x[r] > xq))) {
                S.col[r + 1] = S.col[r];
                S.val[r + 1] = S.val[r];
                S.x[r + 1] = S.x[r];
                --r;
            }
            S.col[r + 1] = cq;
            S.val[r + 1] = vq;
            S.x[r + 1] = xq;
        }
        for (int q = lo + 1; q < hi; ++q) dup |= S.col[q] == S.col[q - 1];
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, dup)) return p;
    // combine runs of equal columns chunk by chunk, compacting in place: the
    // writes of a chunk land below the next chunk's first position
    int out = 0;
    for (int base = 0; base < p; base += 32) {
        const int q = base + lane;
        const bool head = q < p && (q == 0 || S.col[q] != S.col[q - 1]);
        const unsigned hm = __ballot_sync(0xffffffffu, head);
        int32_t c = 0;
        double sum = 0.0;
        if (head) {
            c = S.col[q];
            sum = dadd(0.0, S.val[q]);
            for (int u = q + 1; u < p && S.col[u] == c; ++u) sum = dadd(sum, S.val[u]);
        }
        __syncwarp();
        if (head) {
            const int o = out + __popc(hm & ((1u << lane) - 1));
            S.col[o] = c;
            S.val[o] = sum;
        }
        out += __popc(hm);
        __syncwarp();
    }
    return out;
}

template <int NJ>
__device__ __forceinline__ void warp_copy_out(const WarpSliceT<NJ>& S, int nnz, int64_t obase,
                                              int32_t* __restrict__ ccol, double* __restrict__ cval, int lane) {
    for (int q = lane; q < nnz; q += 32) {
        ccol[obase + q] = S.col[q];
        cval[obase + q] = dadd(0.0, S.val[q]);
    }
}

template <int WPB, int NJ, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB) k_warp_numeric(const int64_t* __restrict__ arp,
                                                                 const int32_t* __restrict__ acol,
                                                                 const double* __restrict__ aval,
                                                                 const int64_t* __restrict__ brp,
                                                                 const int32_t* __restrict__ bcol,
                                                                 const double* __restrict__ bval,
                                                                 const int32_t* __restrict__ list,
                                                                 const int32_t* __restrict__ count, int cshift,
                                                                 const int64_t* __restrict__ crp,
                                                                 int32_t* __restrict__ ccol,
                                                                 double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSliceT<NJ>& S = reinterpret_cast<WarpSliceT<NJ>*>(smem_raw)[w];
    const int64_t gw = blockIdx.x * int64_t(WPB) + w, nw = int64_t(gridDim.x) * WPB;
    RowPipe<true> pipe{arp, acol, aval, brp, list, *count, nw};
    int32_t i;
    RowFetch cur = pipe.start(gw, lane, i);
    for (int64_t t = gw; t < pipe.n; t += nw) {
        const RowEntries re = make_row(cur, lane);
        const int nnz = warp_row_sorted<NJ>(S, re, bcol, bval, cshift, lane);
        const RowFetch nxt = pipe.spans(lane);
        warp_copy_out<NJ>(S, nnz, crp[i], ccol, cval, lane);
        const int32_t inext = pipe.i1;
        pipe.advance(t + nw, lane);
        cur = nxt;
        i = inext;
        __syncwarp();
    }
}

// ------------------------------------------------------------- fused pass
// Single pass: warps take rows in order from a global ticket, compute the
// sorted row into their smem slice, publish its nnz, and find the row's offset
// in C with a decoupled look-back over the predecessors' status words (a warp
// only ever waits on rows with smaller tickets, which are already running, so
// progress is guaranteed). Rows of the CTA / heavy classes were computed
// beforehand into a side buffer; their warp just publishes and copies.
// status word: bits 62-63 flag (0 none, 1 aggregate, 2 inclusive), bits 0-61 value.
constexpr uint64_t ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive prefix of row i's nnz over rows [0, i) (all lanes return it).
__device__ __forceinline__ int64_t look_back(const uint64_t* status, int64_t i, int lane) {
    int64_t excl = 0;
    int64_t j = i - 1;
    while (j >= 0) {
        const int64_t idx = j - lane;
        uint64_t s = idx >= 0 ? ld_status(status + idx) : ST_INC;
        while (true) {
            const unsigned inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
            const unsigned none = __ballot_sync(0xffffffffu, (s >> 62) == 0);
            const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1u : 0xffffffffu;  // lanes <= first inclusive
            if (none & upto) {
                if ((s >> 62) == 0 && idx >= 0) s = ld_status(status + idx);
                continue;
            }
            int64_t v = ((1u << lane) & upto) ? static_cast<int64_t>(s & ST_VAL) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            excl += v;
            if (inc) return excl;
            break;
        }
        j -= 32;
    }
    return excl;
}

template <int WPB>
__global__ void __launch_bounds__(WPB * 32, SPG_WARP_MINB) k_warp_fused(
    const int64_t* __restrict__ arp, const int32_t* __restrict__ acol, const double* __restrict__ aval,
    const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol, const double* __restrict__ bval, int64_t m,
    int cshift, const int64_t* __restrict__ side_off, const int64_t* __restrict__ side_nnz,
    const int32_t* __restrict__ side_col, const double* __restrict__ side_val, unsigned long long* __restrict__ ticket,
    uint64_t* __restrict__ status, int64_t* __restrict__ crp, int32_t* __restrict__ ccol, double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSlice& S = reinterpret_cast<WarpSlice*>(smem_raw)[w];
    while (true) {
        int64_t i = 0;
        if (lane == 0) i = static_cast<int64_t>(atomicAdd(ticket, 1ull));
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= m) break;
        const int64_t e0 = arp[i];
        const int ne = static_cast<int>(arp[i + 1] - e0);
        const int64_t so = side_off[i];
        int64_t nnz = 0;
        if (so >= 0) {
            nnz = side_nnz[i];
        } else if (ne > 0 && ne <= 32) {
            const RowEntries re = load_row<true>(acol, aval, brp, e0, ne, lane);
            if (re.p > 0) nnz = warp_row_sorted<WARP_NJ>(S, re, bcol, bval, cshift, lane);
        }
        if (lane == 0) st_status(status + i, (i == 0 ? ST_INC : ST_AGG) | static_cast<uint64_t>(nnz));
        const int64_t excl = i == 0 ? 0 : look_back(status, i, lane);
        if (lane == 0) {
            if (i > 0) st_status(status + i, ST_INC | static_cast<uint64_t>(excl + nnz));
            crp[i + 1] = excl + nnz;
        }
        if (so >= 0) {
            for (int64_t q = lane; q < nnz; q += 32) {
                ccol[excl + q] = side_col[so + q];
                cval[excl + q] = side_val[so + q];
            }
        } else {
            warp_copy_out<WARP_NJ>(S, static_cast<int>(nnz), excl, ccol, cval, lane);
        }
        __syncwarp();
    }
}

// side_off[row] = offset of a CTA/heavy row in the side buffer (products-bounded).
__global__ void k_side_gather(const int32_t* __restrict__ rows, const int32_t* __restrict__ count,
                              const int64_t* __restrict__ prod, int64_t* __restrict__ out) {
    const int n = *count;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) out[t] = prod[rows[t]];
}

__global__ void k_side_scatter(const int32_t* __restrict__ rows, const int32_t* __restrict__ count,
                               const int64_t* __restrict__ off, int64_t* __restrict__ side_off) {
    const int n = *count;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) side_off[rows[t]] = off[t];
}

// ---------------------------------------------------------------- CTA rows
// One CTA per row (≤ CTA_P products, ≤ CTA_E entries): the same bucketed ESC
// with the product arrays in shared memory and block-wide phases.
struct CtaSmem {
    int32_t col[CTA_P];
    double val[CTA_P];
    uint16_t bkt[CTA_P];
    uint16_t perm[CTA_P];
    int64_t e_bst[CTA_E];
    double e_av[CTA_E];
    int32_t e_pre[CTA_E + 1];
    int32_t b_off[CTA_NB + 1];
    int32_t b_cnt[CTA_NB + 1];
    int32_t ws[NT / 32 + 1];
    int32_t minc, maxc;
    float scale;
};

// Monotone map of a column into [0, nb) over the row's [minc, maxc] range.
__device__ __forceinline__ int bucket_range(int32_t col, int32_t minc, float scale, int nb) {
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

template <bool NUMERIC>
__global__ void __launch_bounds__(NT) k_cta_rows(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                                 const double* __restrict__ aval, const int64_t* __restrict__ brp,
                                                 const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                                 const int64_t* __restrict__ prod, const int32_t* __restrict__ rows,
                                                 const int32_t* __restrict__ nrows_dev, int64_t* __restrict__ row_nnz,
                                                 const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                                 double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CtaSmem& s = *reinterpret_cast<CtaSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int nrows = *nrows_dev;
    for (int t = blockIdx.x; t < nrows; t += gridDim.x) {
        const int64_t i = rows[t];
        const int64_t e0 = arp[i];
        const int ne = static_cast<int>(arp[i + 1] - e0);
        const int ptile = static_cast<int>(prod[i]);
        if (tid == 0) {
            s.minc = INT_MAX;
            s.maxc = -1;
        }
        __syncthreads();
        // A entries -> B row spans, column range, product prefix
        {
            constexpr int EI = CTA_E / NT;
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
                        atomicMin(&s.minc, bcol[bs]);
                        atomicMax(&s.maxc, bcol[be - 1]);
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
        const int nb = (ptile + BUCKET_LOAD - 1) / BUCKET_LOAD;
        for (int b = tid; b <= nb; b += NT) s.b_cnt[b] = 0;
        __syncthreads();
        if (tid == 0) s.scale = static_cast<float>(nb) / static_cast<float>(int64_t(s.maxc) - s.minc + 1);
        __syncthreads();
        const int32_t minc = s.minc;
        const float scale = s.scale;

        for (int x = tid; x < ptile; x += NT) {
            int lo = 0, hi = ne;  // largest e with e_pre[e] <= x
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s.e_pre[mid] <= x) lo = mid; else hi = mid;
            }
            const int64_t u = s.e_bst[lo] + (x - s.e_pre[lo]);
            const int32_t c = bcol[u];
            const int b = bucket_range(c, minc, scale, nb);
            s.col[x] = c;
            s.bkt[x] = static_cast<uint16_t>(b);
            if (NUMERIC) s.val[x] = dmul(s.e_av[lo], bval[u]);
            atomicAdd(&s.b_cnt[b], 1);
        }
        __syncthreads();
        block_scan_array<NT, (CTA_NB + NT) / NT, int32_t>(s.b_cnt, nb, s.ws);
        for (int b = tid; b <= nb; b += NT) {
            s.b_off[b] = s.b_cnt[b];
            s.b_cnt[b] = 0;
        }
        __syncthreads();
        for (int x = tid; x < ptile; x += NT) {
            const int b = s.bkt[x];
            s.perm[s.b_off[b] + atomicAdd(&s.b_cnt[b], 1)] = static_cast<uint16_t>(x);
        }
        __syncthreads();
        for (int b = tid; b < nb; b += NT) s.b_cnt[b] = sort_bucket(s.perm, s.b_off[b], s.b_off[b + 1], s.col);
        __syncthreads();
        block_scan_array<NT, (CTA_NB + NT) / NT, int32_t>(s.b_cnt, nb, s.ws);
        if (!NUMERIC) {
            if (tid == 0) row_nnz[i] = s.b_cnt[nb];
        } else {
            const int64_t obase = crp[i];
            for (int b = tid; b < nb; b += NT) {
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
    DBuf<int32_t> lists(ctx, 4 * m), counts(ctx, 4);
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, 4 * sizeof(int32_t), ctx->stream));
    k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod, lists,
                                                              counts);
    SPG_LAUNCH_CHECK();
    exclusive_scan_i64(ctx, prod, pex, m);
    return read_scalar(ctx, pex.get() + m);
}

namespace {
constexpr int WPB = 8;  // warps per block of the warp kernels

int cshift_for(int64_t ncols) {
    int bits = 1;
    while ((int64_t(1) << bits) < ncols) ++bits;
    return 32 - bits;  // col << cshift puts the top column bit at bit 31
}
}  // namespace

spg_csr* spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b) {
    if (a->ncols != b->nrows)
        fail(SPG_DIMENSION_ERROR,
             "spgemm: a.ncols=" + std::to_string(a->ncols) + " != b.nrows=" + std::to_string(b->nrows));
    const int64_t m = a->nrows, n = b->ncols;
    if (m == 0 || a->nnz == 0 || b->nnz == 0) return new_csr(ctx, m, n, 0);
    const int cshift = cshift_for(n);

    // 1: products per row + CTA/heavy row lists + total products
    DBuf<int64_t> prod(ctx, m), total(ctx, 1);
    DBuf<int32_t> lists(ctx, 4 * m), counts(ctx, 4);
    int32_t* cta_list = lists.get() + 2 * m;
    int32_t* heavy_list = lists.get() + 3 * m;
    int32_t* cta_count = counts.get() + 2;
    int32_t* heavy_count = counts.get() + 3;
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, 4 * sizeof(int32_t), ctx->stream));
    {
        KTime kt(ctx, "row_products");
        k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod,
                                                                  lists, counts);
        SPG_LAUNCH_CHECK();
    }
    {
        size_t tmp = 0;
        SPG_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, prod.get(), total.get(), m, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        SPG_CUDA(cub::DeviceReduce::Sum(t.get(), tmp, prod.get(), total.get(), m, ctx->stream));
    }
    int32_t hc[4];
    int64_t products = 0;
    SPG_CUDA(cudaMemcpyAsync(hc, counts.get(), sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(&products, total.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    const int ncta = hc[2], nheavy = hc[3];

    // single pass needs C sized by the products (an upper bound of nnz(C))
    size_t free_b = 0, total_b = 0;
    SPG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const bool fused = ctx->force_two_pass == 0 &&
                       static_cast<double>(products) * 12.0 < 0.6 * static_cast<double>(free_b);

    // heavy-row workspace plan (host side; heavy rows are few)
    std::vector<int64_t> hp_off(nheavy + 1, 0), he_off(nheavy + 1, 0), hb_off(nheavy + 1, 0);
    if (nheavy) {
        DBuf<int64_t> info(ctx, 2 * int64_t(nheavy));
        k_heavy_info<<<grid_for(ctx, nheavy), 256, 0, ctx->stream>>>(heavy_list, nheavy, prod, a->rowptr, info);
        SPG_LAUNCH_CHECK();
        std::vector<int64_t> hinfo(2 * size_t(nheavy));
        SPG_CUDA(cudaMemcpyAsync(hinfo.data(), info.get(), hinfo.size() * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        SPG_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int h = 0; h < nheavy; ++h) {
            hp_off[h + 1] = hp_off[h] + hinfo[2 * h];
            he_off[h + 1] = he_off[h] + hinfo[2 * h + 1] + 1;
            hb_off[h + 1] = hb_off[h] + (hinfo[2 * h] + BUCKET_LOAD - 1) / BUCKET_LOAD + 1;
        }
    }
    DBuf<int64_t> d_hp(ctx, nheavy + 1), d_he(ctx, nheavy + 1), d_hb(ctx, nheavy + 1);
    HeavyWs hws{};
    DBuf<int64_t> w_epre(ctx, he_off[nheavy]);
    DBuf<int32_t> w_col(ctx, hp_off[nheavy]), w_bkt(ctx, hp_off[nheavy]), w_perm(ctx, hp_off[nheavy]);
    DBuf<double> w_val(ctx, hp_off[nheavy]);
    DBuf<int64_t> w_boff(ctx, hb_off[nheavy]), w_bcnt(ctx, hb_off[nheavy]);
    if (nheavy) {
        SPG_CUDA(cudaMemcpyAsync(d_hp.get(), hp_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(d_he.get(), he_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        SPG_CUDA(cudaMemcpyAsync(d_hb.get(), hb_off.data(), (nheavy + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        hws = HeavyWs{w_epre, w_col, w_val, w_bkt, w_perm, w_boff, w_bcnt};
    }

    const size_t cta_smem = sizeof(CtaSmem);
    const size_t warp_smem = sizeof(WarpSlice) * WPB;
    if (!ctx->tile_attr_set) {
        SPG_CUDA(cudaFuncSetAttribute(k_cta_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_smem));
        SPG_CUDA(cudaFuncSetAttribute(k_cta_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_smem));
        SPG_CUDA(cudaFuncSetAttribute(k_warp_numeric<WPB, 8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(WarpSliceT<8>) * WPB)));
        SPG_CUDA(cudaFuncSetAttribute(k_warp_numeric<WPB, 16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(WarpSliceT<16>) * WPB)));
        SPG_CUDA(cudaFuncSetAttribute(k_warp_fused<WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_smem));
        ctx->tile_attr_set = true;
    }
    const int gc = std::max(1, std::min(ncta, ctx->num_sms * 2));
    DBuf<int64_t> rnnz(ctx, m + 1);
    SPG_CUDA(cudaMemsetAsync(rnnz.get(), 0, (m + 1) * sizeof(int64_t), ctx->stream));

    auto side_symbolic = [&] {
        if (ncta)
            k_cta_rows<false><<<gc, NT, cta_smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                                 b->values, prod, cta_list, cta_count, rnnz, nullptr,
                                                                 nullptr, nullptr);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<false><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                           b->values, heavy_list, d_hp, d_he, d_hb, hws, rnnz, nullptr,
                                                           nullptr, nullptr);
        SPG_LAUNCH_CHECK();
    };
    auto side_numeric = [&](const int64_t* orp, int32_t* ocol, double* oval) {
        if (ncta)
            k_cta_rows<true><<<gc, NT, cta_smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                                b->values, prod, cta_list, cta_count, nullptr, orp, ocol,
                                                                oval);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<true><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                          b->values, heavy_list, d_hp, d_he, d_hb, hws, nullptr, orp,
                                                          ocol, oval);
        SPG_LAUNCH_CHECK();
    };

    if (fused) {
        // side rows (CTA + heavy classes) first, into a products-bounded buffer
        const int nside = ncta + nheavy;
        DBuf<int64_t> side_off(ctx, m), sprod(ctx, nside + 1), soff(ctx, nside + 1);
        SPG_CUDA(cudaMemsetAsync(side_off.get(), 0xff, m * sizeof(int64_t), ctx->stream));
        int64_t side_total = 0;
        if (nside) {
            k_side_gather<<<grid_for(ctx, ncta), 256, 0, ctx->stream>>>(cta_list, cta_count, prod, sprod);
            k_side_gather<<<grid_for(ctx, nheavy), 256, 0, ctx->stream>>>(heavy_list, heavy_count, prod,
                                                                          sprod.get() + ncta);
            SPG_LAUNCH_CHECK();
            exclusive_scan_i64(ctx, sprod, soff, nside);
            k_side_scatter<<<grid_for(ctx, ncta), 256, 0, ctx->stream>>>(cta_list, cta_count, soff, side_off);
            k_side_scatter<<<grid_for(ctx, nheavy), 256, 0, ctx->stream>>>(heavy_list, heavy_count,
                                                                           soff.get() + ncta, side_off);
            SPG_LAUNCH_CHECK();
            side_total = read_scalar(ctx, soff.get() + nside);
        }
        DBuf<int32_t> s_col(ctx, side_total);
        DBuf<double> s_val(ctx, side_total);
        if (nside) {
            KTime kt(ctx, "spgemm_side_rows");
            side_symbolic();
            side_numeric(side_off, s_col, s_val);
        }
        spg_csr* c = new_csr(ctx, m, n, -1);
        c->colind = dalloc<int32_t>(ctx, products);
        c->values = dalloc<double>(ctx, products);
        DBuf<uint64_t> status(ctx, m);
        DBuf<unsigned long long> ticket(ctx, 1);
        SPG_CUDA(cudaMemsetAsync(status.get(), 0, m * sizeof(uint64_t), ctx->stream));
        SPG_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned long long), ctx->stream));
        SPG_CUDA(cudaMemsetAsync(c->rowptr, 0, sizeof(int64_t), ctx->stream));
        int occ = 1;
        SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_warp_fused<WPB>, WPB * 32, warp_smem));
        const int64_t wblocks = (m + WPB - 1) / WPB;
        const int gf = static_cast<int>(std::min<int64_t>(wblocks, int64_t(ctx->num_sms) * std::max(occ, 1)));
        {
            KTime kt(ctx, "spgemm_numeric");
            k_warp_fused<WPB><<<gf, WPB * 32, warp_smem, ctx->stream>>>(
                a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values, m, cshift, side_off, rnnz, s_col,
                s_val, ticket, status, c->rowptr, c->colind, c->values);
            SPG_LAUNCH_CHECK();
        }
        c->nnz = read_scalar(ctx, c->rowptr + m);
        return c;
    }

    // two-pass: symbolic (exact nnz) then numeric at exact offsets
    const int64_t wblocks = (m + WPB - 1) / WPB;
    auto grid_of = [&](const void* fn, size_t smem) {
        int occ = 1;
        SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, WPB * 32, smem));
        return static_cast<int>(std::min<int64_t>(wblocks, int64_t(ctx->num_sms) * std::max(occ, 1)));
    };
    const int32_t* list8 = lists.get();
    const int32_t* list16 = lists.get() + m;
    {
        KTime kt(ctx, "spgemm_symbolic");
        {
        KTime kt8(ctx, "sym_w8");
        k_warp_symbolic<WPB, 8><<<grid_of((const void*)k_warp_symbolic<WPB, 8>, 0), WPB * 32, 0, ctx->stream>>>(
            a->rowptr, a->colind, b->rowptr, b->colind, list8, counts.get(), rnnz);
        }
        KTime kt16(ctx, "sym_w16");
        k_warp_symbolic<WPB, 16><<<grid_of((const void*)k_warp_symbolic<WPB, 16>, 0), WPB * 32, 0, ctx->stream>>>(
            a->rowptr, a->colind, b->rowptr, b->colind, list16, counts.get() + 1, rnnz);
        SPG_LAUNCH_CHECK();
        side_symbolic();
    }
    spg_csr* c = new_csr(ctx, m, n, -1);
    exclusive_scan_i64(ctx, rnnz, c->rowptr, m);
    c->nnz = read_scalar(ctx, c->rowptr + m);
    c->colind = dalloc<int32_t>(ctx, c->nnz);
    c->values = dalloc<double>(ctx, c->nnz);
    {
        KTime kt(ctx, "spgemm_numeric");
        const size_t s8 = sizeof(WarpSliceT<8>) * WPB, s16 = sizeof(WarpSliceT<16>) * WPB;
        {
        KTime k8(ctx, "num_w8");
        k_warp_numeric<WPB, 8, 3><<<grid_of((const void*)k_warp_numeric<WPB, 8, 3>, s8), WPB * 32, s8,
                                    ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values,
                                                   list8, counts.get(), cshift, c->rowptr, c->colind, c->values);
        }
        KTime k16(ctx, "num_w16");
        k_warp_numeric<WPB, 16, 2><<<grid_of((const void*)k_warp_numeric<WPB, 16, 2>, s16), WPB * 32, s16,
                                     ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values,
                                                    list16, counts.get() + 1, cshift, c->rowptr, c->colind,
                                                    c->values);
        SPG_LAUNCH_CHECK();
        side_numeric(c->rowptr, c->colind, c->values);
    }
    return c;
}

}  // namespace spgb
