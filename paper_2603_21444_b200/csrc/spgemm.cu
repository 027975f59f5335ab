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

// ----------------------------------------------------------- row classes
// WARP rows: ≤ 32 A entries and ≤ WARP_P products — one warp per row, the
// products live in registers, one bucket-sorted copy in the warp's smem slice.
// CTA rows: ≤ CTA_E entries and ≤ CTA_P products — one CTA per row in smem.
// HEAVY rows: the rest — one CTA per row with the arrays in global memory.
#ifndef SPG_WARP_MINB
#define SPG_WARP_MINB 3
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
// products(i) = Σ_{k∈A_i} nnz(B_k); rows outside the warp class are appended
// to the CTA / heavy lists.
__global__ void k_row_products(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                               const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod,
                               int32_t* __restrict__ cta_list, int32_t* __restrict__ heavy_list,
                               int32_t* __restrict__ counts) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = 0;
        const int64_t e0 = arp[i], e1 = arp[i + 1];
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t k = __ldg(acol + e);
            p += __ldg(brp + k + 1) - __ldg(brp + k);
        }
        prod[i] = p;
        const int64_t ne = e1 - e0;
        if (p == 0 || (ne <= 32 && p <= WARP_P)) continue;
        if (ne <= CTA_E && p <= CTA_P) cta_list[atomicAdd(counts + 0, 1)] = static_cast<int32_t>(i);
        else heavy_list[atomicAdd(counts + 1, 1)] = static_cast<int32_t>(i);
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

template <bool VALS>
__device__ __forceinline__ RowEntries load_row(const int32_t* __restrict__ acol, const double* __restrict__ aval,
                                               const int64_t* __restrict__ brp, int64_t e0, int m, int lane) {
    int len = 0;
    int64_t bs = 0;
    double av = 0.0;
    if (lane < m) {
        const int32_t k = __ldg(acol + e0 + lane);
        if (VALS) av = __ldg(aval + e0 + lane);
        bs = __ldg(brp + k);
        len = static_cast<int>(__ldg(brp + k + 1) - bs);
    }
    const unsigned nz = __ballot_sync(0xffffffffu, len > 0);
    const int mn = __popc(nz);
    const int src = static_cast<int>(__fns(nz, 0, lane + 1)) & 31;
    int lc = __shfl_sync(0xffffffffu, len, src);
    const int64_t bc = __shfl_sync(0xffffffffu, bs, src);
    RowEntries r;
    r.av = VALS ? __shfl_sync(0xffffffffu, av, src) : 0.0;
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

// Entry of product x = 32*j + lane: t0 = entry covering 32*j (ballot), plus the
// entries that start inside the chunk before x (one OR-reduction of start bits).
__device__ __forceinline__ int chunk_entry(int pre, int j, int lane) {
    const int c0 = 32 * j;
    const int t0 = __popc(__ballot_sync(0xffffffffu, pre <= c0)) - 1;
    const int rel = pre - c0;
    const unsigned sm = __reduce_or_sync(0xffffffffu, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
    return t0 + __popc(sm & ((2u << lane) - 1u));
}

// Per-warp smem slice of the numeric kernel: products in bucket order plus
// 16-bit bucket counters / offsets packed two per word (2p buckets, p ≤ 512).
constexpr int WARP_NB = 2 * WARP_P;
struct WarpSlice {
    int32_t col[WARP_P];
    double val[WARP_P];
    uint16_t x[WARP_P];
    uint32_t offw[WARP_NB / 2 + 1];
};

__device__ __forceinline__ int off16(const uint32_t* offw, int b) {
    return static_cast<int>((offw[b >> 1] >> ((b & 1) << 4)) & 0xffffu);
}

// --------------------------------------------------------- warp symbolic
// Distinct columns per row via an open-addressing set in the warp's smem.
constexpr int SYM_T = 2 * WARP_P;
template <int WPB>
__global__ void __launch_bounds__(WPB * 32) k_warp_symbolic(const int64_t* __restrict__ arp,
                                                            const int32_t* __restrict__ acol,
                                                            const int64_t* __restrict__ brp,
                                                            const int32_t* __restrict__ bcol, int64_t m,
                                                            int64_t* __restrict__ row_nnz) {
    __shared__ int32_t table[WPB][SYM_T];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t* tab = table[w];
    const int64_t gw = blockIdx.x * int64_t(WPB) + w, nw = int64_t(gridDim.x) * WPB;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t e0 = arp[i];
        const int ne = static_cast<int>(arp[i + 1] - e0);
        if (ne == 0 || ne > 32) continue;
        const RowEntries re = load_row<false>(acol, nullptr, brp, e0, ne, lane);
        const int p = re.p;
        if (p == 0 || p > WARP_P) continue;
        int lg = 6;
        while ((1 << lg) < 2 * p) ++lg;
        const int T = 1 << lg;
        for (int q = lane; q < T; q += 32) tab[q] = -1;
        __syncwarp();
        int32_t cols[WARP_NJ];
#pragma unroll
        for (int j = 0; j < WARP_NJ; ++j) {
            cols[j] = -1;
            if (j * 32 < p) {
                const int t = chunk_entry(re.pre, j, lane);
                const int64_t base = __shfl_sync(0xffffffffu, re.base, t);
                const int x = 32 * j + lane;
                if (x < p) cols[j] = __ldg(bcol + base + x);
            }
        }
        int fresh = 0;
#pragma unroll
        for (int j = 0; j < WARP_NJ; ++j) {
            if (cols[j] < 0) continue;
            uint32_t h = (static_cast<uint32_t>(cols[j]) * 0x9E3779B1u) >> (32 - lg);
            while (true) {
                const int32_t old = atomicCAS(&tab[h], -1, cols[j]);
                if (old == -1) { ++fresh; break; }
                if (old == cols[j]) break;
                h = (h + 1) & (T - 1);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
        if (lane == 0) row_nnz[i] = fresh;
        __syncwarp();
    }
}

// ---------------------------------------------------------- warp numeric
// Products are gathered into registers (x = 32j + lane, ascending k within the
// row), counted into ~p/2 column buckets, and scattered once into the warp's
// smem slice in bucket order. Each lane then sorts its buckets (≈2 entries) in
// place by (col, x): the slice holds the row sorted by column and is copied to
// C with coalesced stores. Rows with duplicate columns combine each run of
// equal columns in x order (= ascending k, separate mul and add), so values are
// bit-identical to the reference.
template <int WPB>
__global__ void __launch_bounds__(WPB * 32, SPG_WARP_MINB) k_warp_numeric(const int64_t* __restrict__ arp,
                                                           const int32_t* __restrict__ acol,
                                                           const double* __restrict__ aval,
                                                           const int64_t* __restrict__ brp,
                                                           const int32_t* __restrict__ bcol,
                                                           const double* __restrict__ bval, int64_t m, int cshift,
                                                           const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                                           double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSlice& S = reinterpret_cast<WarpSlice*>(smem_raw)[w];
    const int64_t gw = blockIdx.x * int64_t(WPB) + w, nw = int64_t(gridDim.x) * WPB;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t e0 = arp[i];
        const int ne = static_cast<int>(arp[i + 1] - e0);
        if (ne == 0 || ne > 32) continue;
        const RowEntries re = load_row<true>(acol, aval, brp, e0, ne, lane);
        const int p = re.p;
        if (p == 0 || p > WARP_P) continue;
        const int nb = 2 * p;          // ~0.5 products per bucket
        const int nw = (nb + 2) >> 1;  // packed words incl. the off[nb] slot
        for (int q = lane; q < nw; q += 32) S.offw[q] = 0u;

        // expand: every gather issued before any is consumed
        int32_t col[WARP_NJ];
        double val[WARP_NJ];
        int ent[WARP_NJ];
#pragma unroll
        for (int j = 0; j < WARP_NJ; ++j) {
            col[j] = 0;
            val[j] = 0.0;
            ent[j] = 0;
            if (j * 32 < p) {
                const int t = chunk_entry(re.pre, j, lane);
                const int64_t base = __shfl_sync(0xffffffffu, re.base, t);
                ent[j] = t;
                const int x = 32 * j + lane;
                if (x < p) {
                    col[j] = __ldg(bcol + base + x);
                    val[j] = __ldg(bval + base + x);
                }
            }
        }
        __syncwarp();
        int slot[WARP_NJ];
#pragma unroll
        for (int j = 0; j < WARP_NJ; ++j) {
            slot[j] = -1;
            if (j * 32 < p) {
                const double a = __shfl_sync(0xffffffffu, re.av, ent[j]);
                if (32 * j + lane < p) {
                    val[j] = dmul(a, val[j]);
                    const int b = bucket_of(col[j], cshift, nb);
                const int sh = (b & 1) << 4;
                    slot[j] = static_cast<int>((atomicAdd(&S.offw[b >> 1], 1u << sh) >> sh) & 0xffffu);
                }
            }
        }
        __syncwarp();
        // exclusive scan of the 16-bit counts (contiguous words per lane)
        {
            constexpr int PERW = (WARP_NB / 2 + 1 + 31) / 32;
            uint32_t wv[PERW];
            int s = 0;
#pragma unroll
            for (int q = 0; q < PERW; ++q) {
                const int wi = lane * PERW + q;
                wv[q] = wi < nw ? S.offw[wi] : 0u;
                s += static_cast<int>((wv[q] & 0xffffu) + (wv[q] >> 16));
            }
            int inc = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t pre = static_cast<uint32_t>(inc - s);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < PERW; ++q) {
                const int wi = lane * PERW + q;
                const uint32_t lo = pre, hi = pre + (wv[q] & 0xffffu);
                if (wi < nw) S.offw[wi] = lo | (hi << 16);
                pre = hi + (wv[q] >> 16);
            }
        }
        __syncwarp();
        // scatter into bucket order
#pragma unroll
        for (int j = 0; j < WARP_NJ; ++j) {
            if (slot[j] >= 0) {
                const int pos = off16(S.offw, bucket_of(col[j], cshift, nb)) + slot[j];
                S.col[pos] = col[j];
                S.val[pos] = val[j];
                S.x[pos] = static_cast<uint16_t>(32 * j + lane);
            }
        }
        __syncwarp();
        // order each bucket by (col, x): pairs in one uniform pass, larger
        // buckets (rare at 0.5 products/bucket) by their first lane
        bool dup = false;
        unsigned big = 0;  // bit i: position lane+32i starts a bucket of >= 3
        for (int q0 = 0; q0 < p; q0 += 32) {
            const int q = q0 + lane;
            if (q < p) {
                const int32_t c = S.col[q];
                const int bb = bucket_of(c, cshift, nb);
                const int lo = off16(S.offw, bb), hi = off16(S.offw, bb + 1);
                if (q == lo && hi - lo == 2) {
                    const int32_t c2 = S.col[q + 1];
                    const uint16_t x1 = S.x[q], x2 = S.x[q + 1];
                    dup |= c2 == c;
                    if (c2 < c || (c2 == c && x2 < x1)) {
                        const double v1 = S.val[q];
                        S.col[q] = c2;
                        S.col[q + 1] = c;
                        S.val[q] = S.val[q + 1];
                        S.val[q + 1] = v1;
                        S.x[q] = x2;
                        S.x[q + 1] = x1;
                    }
                } else if (q == lo && hi - lo > 2) {
                    big |= 1u << (q0 >> 5);
                }
            }
        }
        while (big) {
            const int q = lane + 32 * (__ffs(big) - 1);
            big &= big - 1;
            const int bb = bucket_of(S.col[q], cshift, nb);
            const int lo = q, hi = off16(S.offw, bb + 1);
            for (int a = lo + 1; a < hi; ++a) {
                const int32_t ca = S.col[a];
                const double va = S.val[a];
                const uint16_t xa = S.x[a];
                int r = a - 1;
                while (r >= lo && (S.col[r] > ca || (S.col[r] == ca && S.x[r] > xa))) {
                    S.col[r + 1] = S.col[r];
                    S.val[r + 1] = S.val[r];
                    S.x[r + 1] = S.x[r];
                    --r;
                }
                S.col[r + 1] = ca;
                S.val[r + 1] = va;
                S.x[r + 1] = xa;
            }
            for (int a = lo + 1; a < hi; ++a) dup |= S.col[a] == S.col[a - 1];
        }
        __syncwarp();
        const int64_t obase = crp[i];
        if (!__any_sync(0xffffffffu, dup)) {
            for (int q = lane; q < p; q += 32) {
                ccol[obase + q] = S.col[q];
                cval[obase + q] = dadd(0.0, S.val[q]);
            }
        } else {
            // runs of equal columns, already in ascending x (= ascending k)
            int out = 0;
            for (int base = 0; base < p; base += 32) {
                const int q = base + lane;
                const bool head = q < p && (q == 0 || S.col[q] != S.col[q - 1]);
                const unsigned hm = __ballot_sync(0xffffffffu, head);
                if (head) {
                    const int32_t c = S.col[q];
                    double sum = dadd(0.0, S.val[q]);
                    for (int u = q + 1; u < p && S.col[u] == c; ++u) sum = dadd(sum, S.val[u]);
                    const int o = out + __popc(hm & ((1u << lane) - 1));
                    ccol[obase + o] = c;
                    cval[obase + o] = sum;
                }
                out += __popc(hm);
            }
        }
        __syncwarp();
    }
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
    DBuf<int32_t> lists(ctx, 2 * m), counts(ctx, 2);
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, 2 * sizeof(int32_t), ctx->stream));
    k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod, lists,
                                                              lists.get() + m, counts);
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

    // 1: products per row + CTA/heavy row lists
    DBuf<int64_t> prod(ctx, m);
    DBuf<int32_t> lists(ctx, 2 * m), counts(ctx, 2);
    int32_t* cta_list = lists.get();
    int32_t* heavy_list = lists.get() + m;
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, 2 * sizeof(int32_t), ctx->stream));
    {
        KTime kt(ctx, "row_products");
        k_row_products<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod, cta_list,
                                                                  heavy_list, counts);
        SPG_LAUNCH_CHECK();
    }
    int32_t hc[2];
    SPG_CUDA(cudaMemcpyAsync(hc, counts.get(), sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    const int ncta = hc[0], nheavy = hc[1];

    // heavy-row workspace plan (host side; heavy rows are few)
    std::vector<int32_t> hrows(nheavy);
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
        SPG_CUDA(cudaFuncSetAttribute(k_warp_numeric<WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_smem));
        ctx->tile_attr_set = true;
    }
    int occ_w = 1, occ_s = 1;
    SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, k_warp_numeric<WPB>, WPB * 32, warp_smem));
    SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_warp_symbolic<WPB>, WPB * 32, 0));
    const int64_t wblocks = (m + WPB - 1) / WPB;
    const int gw = static_cast<int>(std::min<int64_t>(wblocks, int64_t(ctx->num_sms) * std::max(occ_w, 1)));
    const int gs = static_cast<int>(std::min<int64_t>(wblocks, int64_t(ctx->num_sms) * std::max(occ_s, 1)));
    const int gc = std::max(1, std::min(ncta, ctx->num_sms * 2));

    // 2: symbolic — exact nnz per row
    DBuf<int64_t> rnnz(ctx, m + 1);
    SPG_CUDA(cudaMemsetAsync(rnnz.get(), 0, (m + 1) * sizeof(int64_t), ctx->stream));
    {
        KTime kt(ctx, "spgemm_symbolic");
        k_warp_symbolic<WPB><<<gs, WPB * 32, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, b->colind, m, rnnz);
        SPG_LAUNCH_CHECK();
        if (ncta)
            k_cta_rows<false><<<gc, NT, cta_smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                                 b->values, prod, cta_list, counts, rnnz, nullptr,
                                                                 nullptr, nullptr);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<false><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                           b->values, heavy_list, d_hp, d_he, d_hb, hws, rnnz, nullptr,
                                                           nullptr, nullptr);
        SPG_LAUNCH_CHECK();
    }
    // 3: rowptr of C
    spg_csr* c = new_csr(ctx, m, n, -1);
    exclusive_scan_i64(ctx, rnnz, c->rowptr, m);
    c->nnz = read_scalar(ctx, c->rowptr + m);
    c->colind = dalloc<int32_t>(ctx, c->nnz);
    c->values = dalloc<double>(ctx, c->nnz);

    // 4: numeric
    {
        KTime kt(ctx, "spgemm_numeric");
        k_warp_numeric<WPB><<<gw, WPB * 32, warp_smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr,
                                                                       b->colind, b->values, m, cshift, c->rowptr,
                                                                       c->colind, c->values);
        SPG_LAUNCH_CHECK();
        if (ncta)
            k_cta_rows<true><<<gc, NT, cta_smem, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                                b->values, prod, cta_list, counts, nullptr, c->rowptr,
                                                                c->colind, c->values);
        SPG_LAUNCH_CHECK();
        if (nheavy)
            k_heavy<true><<<nheavy, NT, 0, ctx->stream>>>(a->rowptr, a->colind, a->values, b->rowptr, b->colind,
                                                          b->values, heavy_list, d_hp, d_he, d_hb, hws, nullptr,
                                                          c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    return c;
}

}  // namespace spgb
