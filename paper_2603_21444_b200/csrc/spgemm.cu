// Local SpGEMM C = A*B on one B200 (sm_100a): the replacement of
// spgemm_local (reference csr.cpp:132-165).
//
// Row-wise Gustavson in one pass over B:
//
//   k_row_prep   per row of A: products, kind (SMALL / MEDIUM / BIG), tile
//                weight; per A entry of a tile row its packed span (B row
//                start, length, product offset in the row, row products)
//   tiles        runs of consecutive SMALL rows within one TW-window of the
//                weight prefix (k_tile_flags + scan + k_tile_scatter); MEDIUM
//                and BIG rows are tiles of their own
//   side path    BIG rows (R-MAT hubs): sort-based ESC, computed before k_tile;
//                k_big_copy moves them into C after it
//   k_tile       persistent CTAs, tiles from a global ticket: gather the tile's
//                products into registers, multiply, bucket by (row, column),
//                scan, place, rank shared buckets, fold duplicates in
//                ascending k, decoupled look-back over the tiles' nnz, copy the
//                tile's C rows out as one contiguous run.
//
// Values are bit-identical to the reference: every C entry is
// 0 + a*b for its first product, then + a*b in ascending k, with separate
// multiply and add (no FMA).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "block_scan.cuh"
#include "spg_internal.cuh"

#ifndef SPG_K32_COLBITS
#define SPG_K32_COLBITS 24  // 32-bit sort keys for the BIG rows up to this many column bits
#endif

namespace spgb {
namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

constexpr unsigned FULL = 0xffffffffu;

// -DSPG_CHECKED: device-side invariant checks (shared-memory indices, bucket
// ranges, look-back values). A failed check traps, which fails the launch —
// the checked build is run over the GPU parity tests (compute-sanitizer is
// not available on the GPU pool).
#ifdef SPG_CHECKED
#define SPG_DCHECK(cond)                                                                             \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("SPG_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   blockIdx.x, threadIdx.x);                                                         \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define SPG_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// Monotone map column -> [0, nb): high bits of the column scaled by nb.
__device__ __forceinline__ int bucket_of(uint32_t col, int cshift, int nb) {
    return static_cast<int>(__umulhi(col << cshift, static_cast<uint32_t>(nb)));
}

namespace tile {
constexpr int NT = 256;                         // threads per CTA
constexpr int NW = NT / 32;
constexpr int SMALL_P = 512;                    // a tile row has <= SMALL_P products
constexpr int SMALL_E = 64;                     // ... and <= SMALL_E entries
constexpr int ROW_W_MAX = SMALL_P + 4 * SMALL_E + 4;
#ifndef SPG_TILE_BPP
#define SPG_TILE_BPP 2
#endif
constexpr int BPP = SPG_TILE_BPP;               // column buckets per product of a row (2 or 4)
constexpr int CW = BPP / 2;                     // counter words per product (2 x 16-bit counters a word)
// espan[e] of an entry of a tile row: B row start (30 bits) | B row length (10)
// | product offset of the entry in its row (12) | products of the row (12)
constexpr int SP_BS = 30, SP_LEN = 30, SP_IN = 40, SP_PR = 52;
constexpr int SP_LEN_MAX = 1023;
constexpr uint64_t SP_BS_MASK = (uint64_t(1) << SP_BS) - 1;
}  // namespace tile

// Tile geometry: the window TW of the row weight prefix bounds a tile's
// products, 4*entries and 4*rows by PMAX, which sizes the shared memory and
// the per-thread product slots; MINB = CTAs per SM the registers are capped
// for. Two are compiled (`profiles/r2o_*`, `r2u_*`): the wide one (84 KB, 2
// CTAs/SM) is best when B's rows are short (config 2: 23.7 ms against 26.1),
// the small one (3 CTAs/SM) when they are long (config 5, A*A^T with 64-entry
// B rows: 34.6 ms against 38.5; a random B of that shape 26.1 against 27.8).
#ifndef SPG_TILE_W
#define SPG_TILE_W 2048
#endif
#ifndef SPG_TILE_MINB
#define SPG_TILE_MINB 2
#endif
template <int TW_, int MINB_>
struct TileGeo {
    static constexpr int NT = tile::NT;
    static constexpr int TW = TW_;
    static constexpr int MINB = MINB_;
    static constexpr int PMAX = TW + tile::ROW_W_MAX;     // bound of products, 4*entries, 4*rows of a tile
    static constexpr int EMAX = PMAX / 4;
    static constexpr int RMAX = PMAX / 4;
    static constexpr int NJ = (PMAX + NT - 1) / NT;      // product slots per thread
    static constexpr int EPT = (EMAX + NT - 1) / NT;     // entry slots per thread
    static constexpr int HW = PMAX / 32 + 2;             // words of the head bitmap
    static constexpr int LMAX = PMAX / 3 + 1;            // shared buckets of >= 3 products
};
using GeoWide = TileGeo<SPG_TILE_W, SPG_TILE_MINB>;
using GeoSmall = TileGeo<1536, 3>;

// The geometry decision, made identically by the row pass, the tile flags
// (on the device, from the sampled sum, so no host round trip precedes the
// row pass) and the host (after its one read-back): force 1 = wide, 2 =
// small, else small iff the nsamp sampled entries of A reference B rows of
// mean length >= 32.
__host__ __device__ __forceinline__ bool geo_small(unsigned long long refsum, int64_t nsamp, int force) {
    if (force) return force == 2;
    return nsamp > 0 && refsum >= 32ull * static_cast<unsigned long long>(nsamp);
}

// Row kinds: SMALL rows share windowed tiles; a MEDIUM row (not small, but
// products + 4*entries + 4 <= PMAX and every B row it reads <= SP_LEN_MAX
// long) is a tile of its own; BIG rows go to the side path.
enum : int8_t { RK_SMALL = 0, RK_MEDIUM = 1, RK_BIG = 2 };

// Row weight: tiles are runs of small rows within one TW-window of the
// exclusive prefix of weights, so a tile has < PMAX products, < PMAX/4
// entries and < PMAX/4 rows.
__host__ __device__ __forceinline__ int64_t tile_weight(int64_t p, int64_t ne) { return p + 4 * ne + 4; }
__host__ __device__ __forceinline__ bool tile_small(int64_t p, int64_t ne) {
    return p <= tile::SMALL_P && ne <= tile::SMALL_E;
}

// Per row (warp per row, lanes over entries): products(i) = Σ nnz(B_k), the
// row kind, the packed entry spans of tile rows (so the tile kernel reads its
// entries with no dependent B.rowptr load and no row pass), the row weight,
// and the BIG-row lists: 0 = CTA rows (<= CTA_P products, <= CTA_E entries),
// 1 = heavy.
__global__ void k_row_prep(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                           const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod,
                           int64_t* __restrict__ wt, int8_t* __restrict__ kind, uint64_t* __restrict__ espan,
                           int32_t* __restrict__ big_rows, int32_t* __restrict__ nbig, bool medium_big,
                           const unsigned long long* __restrict__ refsum, int64_t nsamp, int force) {
    const int pmax = geo_small(*refsum, nsamp, force) ? GeoSmall::PMAX : GeoWide::PMAX;
    // half-warp per row (two rows in flight per warp: the row is a chain of
    // dependent loads arp -> acol -> brp); loops are warp-uniform
    const int lane = threadIdx.x & 31, sub = lane & 15, half = lane >> 4;
    const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i0 = 2 * gw; i0 < m; i0 += 2 * nw) {
        const int64_t i = i0 + half;
        const bool ok = i < m;
        int64_t e0 = 0, e1 = 0;
        if (ok) {
            e0 = arp[i];
            e1 = arp[i + 1];
        }
        const int64_t ne = e1 - e0;
        const int64_t ne_max = max(ne, static_cast<int64_t>(__shfl_xor_sync(FULL, ne, 16)));
        int64_t p = 0, maxlen = 0, bsr[2] = {0, 0}, lenr[2] = {0, 0};  // rows of <= 32 entries keep their spans
        for (int64_t t = 0; t < ne_max; t += 16) {
            int64_t bs = 0, len = 0;
            if (t + sub < ne) {
                const int32_t k = __ldg(acol + e0 + t + sub);
                bs = __ldg(brp + k);
                len = __ldg(brp + k + 1) - bs;
            }
            if (t == 0) {  // (the other half's row may take more iterations)
                bsr[0] = bs;
                lenr[0] = len;
            } else if (t == 16) {
                bsr[1] = bs;
                lenr[1] = len;
            }
            int64_t sum = len;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
            p += sum;
            maxlen = max(maxlen, len);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) maxlen = max(maxlen, static_cast<int64_t>(__shfl_xor_sync(FULL, maxlen, o)));
        int8_t rk = RK_BIG;
        if (tile_small(p, ne)) rk = RK_SMALL;
        else if (!medium_big && tile_weight(p, ne) <= pmax && maxlen <= tile::SP_LEN_MAX) rk = RK_MEDIUM;
        const uint64_t pr = static_cast<uint64_t>(p);
        const bool spans = ok && rk != RK_BIG;
        {  // rows of <= 32 entries: in-row product offsets from registers
            int64_t carry = 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                int64_t inc = lenr[c];
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    const int64_t y = __shfl_up_sync(FULL, inc, o, 16);
                    if (sub >= o) inc += y;
                }
                if (spans && ne <= 32 && 16 * c + sub < ne)
                    espan[e0 + 16 * c + sub] = (static_cast<uint64_t>(bsr[c]) & tile::SP_BS_MASK) |
                                               (static_cast<uint64_t>(lenr[c]) << tile::SP_LEN) |
                                               (static_cast<uint64_t>(carry + inc - lenr[c]) << tile::SP_IN) |
                                               (pr << tile::SP_PR);
                carry += __shfl_sync(FULL, inc, 15, 16);
            }
        }
        const bool slow = spans && ne > 32;
        if (__any_sync(FULL, slow)) {  // longer rows: a second pass
            int64_t carry = 0;
            for (int64_t t = 0; t < ne_max; t += 16) {
                int64_t bs = 0, len = 0;
                if (slow && t + sub < ne) {
                    const int32_t k = __ldg(acol + e0 + t + sub);
                    bs = __ldg(brp + k);
                    len = __ldg(brp + k + 1) - bs;
                }
                int64_t inc = len;
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    const int64_t y = __shfl_up_sync(FULL, inc, o, 16);
                    if (sub >= o) inc += y;
                }
                if (slow && t + sub < ne)
                    espan[e0 + t + sub] = (static_cast<uint64_t>(bs) & tile::SP_BS_MASK) |
                                          (static_cast<uint64_t>(len) << tile::SP_LEN) |
                                          (static_cast<uint64_t>(carry + inc - len) << tile::SP_IN) |
                                          (pr << tile::SP_PR);
                carry += __shfl_sync(FULL, inc, 15, 16);
            }
        }
        if (ok && sub == 0) {
            prod[i] = p;
            kind[i] = rk;
            wt[i] = rk == RK_SMALL ? tile_weight(p, ne) : 0;
            if (rk == RK_BIG) big_rows[atomicAdd(nbig, 1)] = static_cast<int32_t>(i);
        }
    }
}

// Tile starts: row i starts a tile if it is not SMALL, follows a row that is
// not SMALL, or its weight prefix enters a new TW-window.
__global__ void k_tile_flags(const int64_t* __restrict__ wpre, const int8_t* __restrict__ kind, int64_t m,
                             const unsigned long long* __restrict__ refsum, int64_t nsamp, int force,
                             int64_t* __restrict__ flag) {
    const int64_t tw = geo_small(*refsum, nsamp, force) ? GeoSmall::TW : GeoWide::TW;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        int f = 1;
        if (i > 0 && kind[i] == RK_SMALL)
            f = kind[i - 1] != RK_SMALL || (wpre[i] / tw != wpre[i - 1] / tw);
        flag[i] = f;
    }
}

// Compacts the tile starts: tr[t] = first row | BIG flag (bit 62), te[t] = its
// first entry; tr[ntiles] = m, te[ntiles] = nnz(A).
__global__ void k_tile_scatter(const int64_t* __restrict__ flag, const int64_t* __restrict__ fpos,
                               const int8_t* __restrict__ kind, const int64_t* __restrict__ arp, int64_t m,
                               int64_t* __restrict__ tr, int64_t* __restrict__ te) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= m; i += int64_t(gridDim.x) * blockDim.x) {
        if (i == m) {
            const int64_t nt = fpos[m];
            tr[nt] = m;
            te[nt] = arp[m];
        } else if (flag[i]) {
            tr[fpos[i]] = i | (kind[i] == RK_BIG ? (int64_t(1) << 62) : 0);
            te[fpos[i]] = arp[i];
        }
    }
}

// ================================================================ BIG rows (side path)
// entries of the listed rows of A
__global__ void k_row_nnz(const int32_t* __restrict__ rows, int n, const int64_t* __restrict__ arp,
                          int64_t* __restrict__ out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        out[t] = arp[rows[t] + 1] - arp[rows[t]];
}
// per-row values of the BIG rows in their list order.
__global__ void k_side_gather(const int32_t* __restrict__ rows, int n, const int64_t* __restrict__ rnnz,
                              int64_t* __restrict__ out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) out[t] = rnnz[rows[t]];
}

// ------------------------------------------------- BIG rows: sort-based ESC
// Rows too large for a tile (R-MAT hubs: up to millions of products, heavy
// duplication) are multiplied in memory-bounded batches: expand every product
// as (row-in-batch << colbits | column, av*bv) in product order, stable radix
// sort by that key (CUB), then sum each run of equal keys sequentially — the
// stable sort keeps a run in product order = ascending k, so the sums are
// bit-identical to the reference's acc[j] += av*bv.

// Expansion of a batch, balanced by products (one R-MAT row can hold 3.6e7
// of them): k_big_ent lists the batch's A entries (B row start, B row
// length, A value, row in batch) in row order; a scan of the lengths gives
// every entry its first product; k_big_fill then takes chunks of FILL_CH
// consecutive products, marks where each entry starts inside the chunk,
// propagates the entry id with a max-scan and writes every product as
// (row-in-batch << colbits | column, av*bv) — product order within a row is
// ascending k, which the stable sort keeps.
// K = uint32_t when row-in-batch and column bits fit 32 (a third less sort
// traffic), else uint64_t.
__global__ void __launch_bounds__(256) k_big_ent(const int32_t* __restrict__ rows, int nrows,
                                                 const int64_t* __restrict__ eoff, const int64_t* __restrict__ arp,
                                                 const int32_t* __restrict__ acol, const double* __restrict__ aval,
                                                 const int64_t* __restrict__ brp, int64_t* __restrict__ eb,
                                                 int64_t* __restrict__ elen, double* __restrict__ eav,
                                                 int32_t* __restrict__ erow) {
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int64_t i = rows[r], ea = arp[i], ne = arp[i + 1] - ea, g0 = eoff[r];
        for (int64_t t = threadIdx.x; t < ne; t += blockDim.x) {
            const int32_t k = acol[ea + t];
            const int64_t bs = brp[k];
            eb[g0 + t] = bs;
            elen[g0 + t] = brp[k + 1] - bs;
            eav[g0 + t] = aval[ea + t];
            erow[g0 + t] = r;
        }
    }
}

constexpr int FILL_CH = 4096, FILL_IT = FILL_CH / 256;

template <typename K>
__global__ void __launch_bounds__(256) k_big_fill(const int64_t* __restrict__ pst, int64_t E,
                                                  const int64_t* __restrict__ eb, const double* __restrict__ eav,
                                                  const int32_t* __restrict__ erow, const int32_t* __restrict__ bcol,
                                                  const double* __restrict__ bval, int colbits, int64_t P,
                                                  K* __restrict__ keys, double* __restrict__ vals) {
    __shared__ int32_t mark[FILL_CH];
    __shared__ int32_t ws[9];
    __shared__ int64_t s_lo;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t c = blockIdx.x; c * FILL_CH < P; c += gridDim.x) {
        const int64_t P0 = c * FILL_CH;
        const int n = static_cast<int>(min(int64_t(FILL_CH), P - P0));
        if (tid == 0) {  // the entry holding product P0: the last g with pst[g] <= P0
            int64_t lo = 0, hi = E - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (pst[mid] <= P0) lo = mid;
                else hi = mid - 1;
            }
            s_lo = lo;
        }
        for (int x = tid; x < FILL_CH; x += 256) mark[x] = -1;
        __syncthreads();
        const int64_t glo = s_lo;
        if (tid == 0) mark[0] = static_cast<int32_t>(glo);
        // entries starting inside the chunk; among entries sharing a start
        // only the last can have products, so the largest id wins
        for (int64_t g = glo + 1 + tid; g < E; g += 256) {
            const int64_t p = pst[g];
            if (p >= P0 + n) break;
            atomicMax(&mark[p - P0], static_cast<int32_t>(g));
        }
        __syncthreads();
        // inclusive max-scan of mark (thread t owns [t*FILL_IT, (t+1)*FILL_IT))
        int32_t m[FILL_IT], run = -1;
#pragma unroll
        for (int u = 0; u < FILL_IT; ++u) {
            m[u] = mark[tid * FILL_IT + u];
            run = max(run, m[u]);
        }
        int32_t inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc = max(inc, y);
        }
        if (lane == 31) ws[warp] = inc;
        __syncthreads();
        int32_t carry = -1;
        for (int w = 0; w < warp; ++w) carry = max(carry, ws[w]);
        int32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) ex = -1;
        carry = max(carry, ex);
#pragma unroll
        for (int u = 0; u < FILL_IT; ++u) {
            carry = max(carry, m[u]);
            mark[tid * FILL_IT + u] = carry;
        }
        __syncthreads();
        for (int x = tid; x < n; x += 256) {
            const int32_t g = mark[x];
            const int64_t u = eb[g] + (P0 + x - pst[g]);
            keys[P0 + x] = (static_cast<K>(erow[g]) << colbits) | static_cast<K>(static_cast<uint32_t>(bcol[u]));
            vals[P0 + x] = dmul(eav[g], bval[u]);
        }
        __syncthreads();
    }
}

// Runs of equal keys in the sorted batch, in chunks of RUN_CH elements (each
// thread owns RUN_IT consecutive ones): k_run_count counts the run heads per
// chunk; after a scan of the counts k_run_sum gives every head its output slot
// and sums its run sequentially (product order = ascending k, so the sum is
// bit-identical to the reference's acc[j] += av*bv), and records where each
// row of the batch starts in the output.
constexpr int RUN_IT = 16, RUN_CH = 256 * RUN_IT;

// Loads the RUN_IT keys owned by the thread at i0 (16-byte loads when the
// chunk is full: i0 is a multiple of RUN_IT and the buffer 256-byte aligned)
// and returns the mask of run heads among them.
template <typename K>
__device__ __forceinline__ uint32_t run_heads(const K* __restrict__ keys, int64_t n, int64_t i0, K (&k)[RUN_IT]) {
    if (i0 >= n) return 0;
    if (i0 + RUN_IT <= n) {
        constexpr int PER = 16 / sizeof(K);
#pragma unroll
        for (int u = 0; u < RUN_IT / PER; ++u) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(keys + i0) + u);
            memcpy(&k[u * PER], &w, 16);
        }
    } else {
#pragma unroll
        for (int u = 0; u < RUN_IT; ++u) k[u] = i0 + u < n ? keys[i0 + u] : K(0);
    }
    K prev = i0 > 0 ? keys[i0 - 1] : ~k[0];
    uint32_t hm = 0;
#pragma unroll
    for (int u = 0; u < RUN_IT; ++u) {
        if (i0 + u < n && k[u] != prev) hm |= 1u << u;
        prev = k[u];
    }
    return hm;
}

template <typename K>
__global__ void __launch_bounds__(256) k_run_count(const K* __restrict__ keys, int64_t n, int64_t* __restrict__ cnt) {
    __shared__ int ws[9];
    const int64_t nch = (n + RUN_CH - 1) / RUN_CH;
    for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        K k[RUN_IT];
        const int h = __popc(run_heads(keys, n, ch * RUN_CH + int64_t(threadIdx.x) * RUN_IT, k));
        int total;
        block_exclusive_scan<256>(h, &total, ws);
        if (threadIdx.x == 0) cnt[ch] = total;
    }
}

// Run heads in order: k_run_heads writes the position of every run head at
// its output slot (hpos[total] = n is set by the host), so run o is
// [hpos[o], hpos[o+1]).
template <typename K>
__global__ void __launch_bounds__(256) k_run_heads(const K* __restrict__ keys, int64_t n,
                                                   const int64_t* __restrict__ cbase, int64_t* __restrict__ hpos) {
    __shared__ int ws[9];
    const int64_t nch = (n + RUN_CH - 1) / RUN_CH;
    for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const int64_t i0 = ch * RUN_CH + int64_t(threadIdx.x) * RUN_IT;
        K k[RUN_IT];
        uint32_t hm = run_heads(keys, n, i0, k);
        int total;
        int64_t o = cbase[ch] + block_exclusive_scan<256>(__popc(hm), &total, ws);
        while (hm) {
            const int u = __ffs(hm) - 1;
            hm &= hm - 1;
            hpos[o++] = i0 + u;
        }
    }
}

// One thread per run folds its values in sorted order (stable sort: product
// order = ascending k, so the sum is bit-identical to the reference's
// acc[j] += av*bv); the run is contiguous, so its loads are independent and
// unrolled 8 deep (hub columns make runs of thousands). The first and last
// run of a row record where the row's output starts and ends (rows of the
// batch without products keep start = end = 0).
template <typename K>
__global__ void __launch_bounds__(256) k_run_fold(const K* __restrict__ keys, const double* __restrict__ vals,
                                                  const int64_t* __restrict__ hpos, int64_t total, int colbits,
                                                  int32_t* __restrict__ ocol, double* __restrict__ oval,
                                                  int64_t* __restrict__ rowstart, int64_t* __restrict__ rowend) {
    const K cmask = (K(1) << colbits) - 1;
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total; o += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = hpos[o], e = hpos[o + 1];
        const K key = keys[s];
        double sum = dadd(0.0, vals[s]);
        int64_t u = s + 1;
        for (; u + 8 <= e; u += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(vals + u + q);
#pragma unroll
            for (int q = 0; q < 8; ++q) sum = dadd(sum, v[q]);
        }
        for (; u < e; ++u) sum = dadd(sum, __ldg(vals + u));
        ocol[o] = static_cast<int32_t>(key & cmask);
        oval[o] = sum;
        const K row = key >> colbits;
        if (o == 0 || (keys[hpos[o - 1]] >> colbits) != row) rowstart[row] = o;
        if (o + 1 == total || (keys[e] >> colbits) != row) rowend[row] = o + 1;
    }
}

// Per big row of the batch: its output is [rowstart[r], rowend[r]) of the
// batch output (no rowstart: a batch without products, every row empty).
__global__ void k_big_finish(const int32_t* __restrict__ rows, int nrows, const int64_t* __restrict__ rowstart,
                             const int64_t* __restrict__ rowend, const int32_t* ocol, const double* oval,
                             uint64_t* __restrict__ side_cp, uint64_t* __restrict__ side_vp,
                             int64_t* __restrict__ side_nnz) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
        const int64_t i = rows[r];
        const int64_t f = rowstart ? rowstart[r] : 0, l = rowstart ? rowend[r] : 0;
        side_cp[i] = reinterpret_cast<uint64_t>(ocol + f);
        side_vp[i] = reinterpret_cast<uint64_t>(oval + f);
        side_nnz[i] = l - f;
    }
}

// ------------------------------------------- BIG rows: dense hub accumulator
// Rows too large for a tile (R-MAT hubs: up to 3.6e7 products) without a
// sort, for B with at most HUB_W columns. One CTA per row (rows from a
// ticket, heaviest first); warp w owns the column range [w*RANGE,
// (w+1)*RANGE) of the 2^18-column window with a shared-memory bitmap of its
// columns (RANGE = 16384 in the symbolic pass, 8192 in the numeric pass).
//  * symbolic (k_hub_sym): every warp walks the row's entries — 32 lanes
//    binary-search 32 entries' B rows for the warp's range at once, then set
//    the bits of the entries' columns — and stores its bitmap; the row's nnz
//    (side_nnz) sizes k_tile's row pointers.
//  * numeric (k_hub_num, after k_tile): the warp loads its bitmap and the
//    prefix of its words' popcounts, so column c of the row is C entry
//    crp[i] + (earlier warps' columns) + rank(c). The entries are applied in
//    ascending k, one after another (__syncwarp between them), the lanes over
//    the entry's columns in the range — distinct, so no two lanes share an
//    entry of C — and every C entry is 0 + a*b (first touch, a second bitmap),
//    then + a*b in ascending k, accumulated in place in C: bit-identical to the
//    reference's acc[j] += av*bv. The running sums live in the row's own C
//    range (compact, L2-resident), not in a dense scratch.
// Warps per CTA: the symbolic pass 16 (ranges of 16384 columns), the numeric
// pass 32 (8192): the numeric pass waits a DRAM round trip per entry and warp,
// and its shared memory allows one CTA per SM, so more warps over narrower
// ranges hide more latency (R-MAT 18: numeric 67.2 ms with 8 warps, 56.5 with
// 16, 51.8 with 32; symbolic 7.9 / 6.5 / 9.6; `profiles/r2y_hub_warps.txt`).
// Both address a row's bitmap in column order, so their splits are independent.
#ifndef SPG_HUB_SYM_NW
#define SPG_HUB_SYM_NW 16
#endif
#ifndef SPG_HUB_NUM_NW
#define SPG_HUB_NUM_NW 32
#endif
constexpr int HUB_W = 262144;  // columns of one hub window (2^18)
constexpr int SYM_NW = SPG_HUB_SYM_NW, SYM_RANGE = HUB_W / SYM_NW, SYM_WORDS = SYM_RANGE / 32;
constexpr int NUM_NW = SPG_HUB_NUM_NW, NUM_RANGE = HUB_W / NUM_NW, NUM_WORDS = NUM_RANGE / 32;
struct HubSymSmem {
    uint32_t bm[SYM_NW][SYM_WORDS];  // the row's columns
    int64_t cnt[SYM_NW];
    int row;
};
struct HubSmem {
    uint32_t sb[NUM_NW][NUM_WORDS];  // the row's columns (symbolic bitmap)
    uint32_t sp[NUM_NW][NUM_WORDS];  // exclusive prefix of the words' popcounts
    uint32_t bm[NUM_NW][NUM_WORDS];  // touched so far
    int64_t cnt[NUM_NW];
    int row;
};

// First position in bcol[lo, hi) with column >= c (the B row is sorted).
__device__ __forceinline__ int64_t lower_col(const int32_t* __restrict__ bcol, int64_t lo, int64_t hi, int64_t c) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(bcol + mid) < c) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// The part [s, f) of entry e's B row inside [lo_c, hi_c), with its A value.
__device__ __forceinline__ void hub_span(const int32_t* __restrict__ acol, const double* __restrict__ aval,
                                         const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol,
                                         int64_t e, int64_t e1, int64_t lo_c, int64_t hi_c, int64_t& s, int64_t& f,
                                         double& av, bool want_av) {
    s = f = 0;
    av = 0.0;
    if (e >= e1) return;
    const int32_t k = __ldg(acol + e);
    const int64_t bs = __ldg(brp + k), be = __ldg(brp + k + 1);
    if (bs < be && __ldg(bcol + bs) < hi_c && __ldg(bcol + be - 1) >= lo_c) {
        s = lower_col(bcol, bs, be, lo_c);
        f = lower_col(bcol, s, be, hi_c);
    }
    if (want_av) av = __ldg(aval + e);
}

__global__ void __launch_bounds__(32 * SYM_NW) k_hub_sym(const int32_t* __restrict__ rows, int nrows,
                                                         const int64_t* __restrict__ arp,
                                                         const int32_t* __restrict__ acol,
                                                         const int64_t* __restrict__ brp,
                                                         const int32_t* __restrict__ bcol, unsigned* __restrict__ ticket,
                                                         uint32_t* __restrict__ gbm, int64_t* __restrict__ side_nnz) {
    extern __shared__ __align__(16) unsigned char hub_raw[];
    HubSymSmem& S = *reinterpret_cast<HubSymSmem*>(hub_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* my = S.bm[warp];
    const int64_t lo_c = int64_t(warp) * SYM_RANGE, hi_c = lo_c + SYM_RANGE;
    while (true) {
        if (threadIdx.x == 0) S.row = static_cast<int>(atomicAdd(ticket, 1u));
        __syncthreads();
        const int t = S.row;
        __syncthreads();
        if (t >= nrows) break;
        const int64_t i = rows[t];
        const int64_t e0 = arp[i], e1 = arp[i + 1];
        for (int x = lane; x < SYM_WORDS; x += 32) my[x] = 0u;
        __syncwarp();
        for (int64_t c0 = e0; c0 < e1; c0 += 32) {
            int64_t s, f;
            double av;
            hub_span(acol, nullptr, brp, bcol, c0 + lane, e1, lo_c, hi_c, s, f, av, false);
            const int ne = static_cast<int>(min(int64_t(32), e1 - c0));
            for (int q = 0; q < ne; ++q) {  // order does not matter for the count
                const int64_t qs = __shfl_sync(FULL, s, q), qf = __shfl_sync(FULL, f, q);
                for (int64_t u = qs + lane; u < qf; u += 32) {
                    const int b = static_cast<int>(__ldg(bcol + u) - lo_c);
                    atomicOr(&my[b >> 5], 1u << (b & 31));
                }
            }
        }
        __syncwarp();
        int64_t cnt = 0;
        uint32_t* g = gbm + static_cast<size_t>(t) * (HUB_W / 32) + static_cast<size_t>(warp) * SYM_WORDS;
        for (int x = lane; x < SYM_WORDS; x += 32) {
            const uint32_t w = my[x];
            g[x] = w;
            cnt += __popc(w);
        }
        cnt = warp_reduce_sum(cnt);
        if (lane == 0) S.cnt[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t tot = 0;
            for (int w = 0; w < SYM_NW; ++w) tot += S.cnt[w];
            side_nnz[i] = tot;
        }
    }
}

__global__ void __launch_bounds__(32 * NUM_NW) k_hub_num(const int32_t* __restrict__ rows, int nrows,
                                                         const int64_t* __restrict__ arp,
                                                         const int32_t* __restrict__ acol,
                                                         const double* __restrict__ aval,
                                                         const int64_t* __restrict__ brp,
                                                         const int32_t* __restrict__ bcol,
                                                         const double* __restrict__ bval, unsigned* __restrict__ ticket,
                                                         const uint32_t* __restrict__ gbm,
                                                         const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                                         double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char hub_raw[];
    HubSmem& S = *reinterpret_cast<HubSmem*>(hub_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* sb = S.sb[warp];
    uint32_t* sp = S.sp[warp];
    uint32_t* bm = S.bm[warp];
    const int64_t lo_c = int64_t(warp) * NUM_RANGE, hi_c = lo_c + NUM_RANGE;
    constexpr int WPL = NUM_WORDS / 32;  // words per lane (contiguous)
    while (true) {
        if (threadIdx.x == 0) S.row = static_cast<int>(atomicAdd(ticket, 1u));
        __syncthreads();
        const int t = S.row;
        __syncthreads();
        if (t >= nrows) break;
        const int64_t i = rows[t];
        const int64_t e0 = arp[i], e1 = arp[i + 1];
        // this warp's bitmap, the prefix of its popcounts, and its first C entry
        const uint32_t* g = gbm + static_cast<size_t>(t) * (HUB_W / 32) + static_cast<size_t>(warp) * NUM_WORDS;
        uint32_t wsum = 0;
#pragma unroll 8
        for (int u = 0; u < WPL; ++u) {
            const uint32_t w = g[lane * WPL + u];
            sb[lane * WPL + u] = w;
            bm[lane * WPL + u] = 0u;
            wsum += __popc(w);
        }
        const uint32_t winc = warp_inclusive_scan(wsum);
        {
            uint32_t e = winc - wsum;
            for (int u = 0; u < WPL; ++u) {
                sp[lane * WPL + u] = e;
                e += __popc(sb[lane * WPL + u]);
            }
        }
        if (lane == 31) S.cnt[warp] = winc;
        __syncthreads();
        int64_t base = crp[i];
        for (int w = 0; w < warp; ++w) base += S.cnt[w];
        int32_t* oc = ccol + base;
        double* ov = cval + base;
        // the running sums live in place in C (the row's range, L2-resident);
        // a shared-memory copy for warps with few columns paid with 8 warps
        // but not with 32 (numeric 51.7 -> 48.8 ms without it, R-MAT 18)
        double* acc = ov;
        for (int64_t c0 = e0; c0 < e1; c0 += 32) {
            int64_t s, f;
            double av;
            hub_span(acol, aval, brp, bcol, c0 + lane, e1, lo_c, hi_c, s, f, av, true);
            const int ne = static_cast<int>(min(int64_t(32), e1 - c0));
            for (int q = 0; q < ne; ++q) {  // the entries in ascending k
                const int64_t qs = __shfl_sync(FULL, s, q), qf = __shfl_sync(FULL, f, q);
                const double qa = __shfl_sync(FULL, av, q);
                // 4 elements per lane in flight: the columns of one B row are
                // distinct, so their C entries never alias
                for (int64_t u0 = qs + lane; u0 < qf; u0 += 128) {
                    int r[4];
                    int32_t cc[4];
                    double p[4], cur[4];
                    uint32_t first = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t u = u0 + 32 * j;
                        cc[j] = u < qf ? __ldg(bcol + u) : -1;
                        p[j] = u < qf ? dmul(qa, __ldg(bval + u)) : 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        r[j] = -1;
                        if (cc[j] >= 0) {
                            const int b = static_cast<int>(cc[j] - lo_c), wd = b >> 5;
                            const uint32_t bit = 1u << (b & 31);
                            r[j] = static_cast<int>(sp[wd] + __popc(sb[wd] & (bit - 1u)));
                            if (!(atomicOr(&bm[wd], bit) & bit)) first |= 1u << j;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) cur[j] = (r[j] >= 0 && !((first >> j) & 1)) ? acc[r[j]] : 0.0;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (r[j] >= 0) {
                            if ((first >> j) & 1) {
                                oc[r[j]] = cc[j];
                                acc[r[j]] = dadd(0.0, p[j]);
                            } else {
                                acc[r[j]] = dadd(cur[j], p[j]);
                            }
                        }
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
}

// BIG rows' sorted products into C[crp[r], crp[r+1]) (after k_rows wrote the
// row pointers): one CTA-range per row chunk, 16 independent copies per thread
// in flight.
__global__ void __launch_bounds__(256) k_big_copy(const int32_t* __restrict__ rows, int nrows,
                                                  const uint64_t* __restrict__ side_cp,
                                                  const uint64_t* __restrict__ side_vp, const int64_t* __restrict__ crp,
                                                  int32_t* __restrict__ ccol, double* __restrict__ cval) {
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int64_t i = rows[r];
        const int64_t base = crp[i], n = crp[i + 1] - base;
        const int32_t* __restrict__ sc = reinterpret_cast<const int32_t*>(side_cp[i]);
        const double* __restrict__ sv = reinterpret_cast<const double*>(side_vp[i]);
        for (int64_t q0 = 0; q0 < n; q0 += 8 * 256) {
            int32_t c8[8];
            double v8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t q = q0 + u * 256 + threadIdx.x;
                if (q < n) {
                    c8[u] = sc[q];
                    v8[u] = sv[q];
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t q = q0 + u * 256 + threadIdx.x;
                if (q < n) {
                    ccol[base + q] = c8[u];
                    cval[base + q] = v8[u];
                }
            }
        }
    }
}

// Decoupled look-back status word: bits 62-63 flag (0 none, 1 aggregate,
// 2 inclusive prefix), bits 0-61 value.
constexpr uint64_t ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive block scan with one barrier: warp totals go to ws (NW slots); the
// caller guarantees a barrier between two uses of the same ws.
template <typename T>
__device__ __forceinline__ T tile_scan(T v, T* total, T* ws) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const T inc = warp_inclusive_scan(v);
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    T before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < tile::NW; ++w) {
        const T t = ws[w];
        before += w < wid ? t : T(0);
        tot += t;
    }
    *total = tot;
    return before + inc - v;
}

struct __align__(16) TileEnt {
    int64_t base;  // B position of tile product x is base + x
    double av;     // A value
};

template <class G>
struct __align__(16) TileSmem {
    double val[G::PMAX];        // staging: the tile's C entries (values)
    TileEnt ent[G::EMAX];
    int32_t col[G::PMAX];       // staging: columns
    uint32_t cnt[tile::CW * G::PMAX + 2];  // 2 x 16-bit bucket counters per word, then prefixes
    uint32_t ebin[G::EMAX];     // per entry: row bucket base (lo 16) | row bucket count (hi 16)
    int32_t epre[G::EMAX + 1];  // product prefix of the tile's entries
    int32_t re[G::RMAX + 1];    // first entry of each row (relative to the tile)
    int32_t rend[G::RMAX];      // end of each row in the (compacted) staging
    uint32_t list[G::LMAX];     // shared buckets of >= 3 products: start | end << 16
    uint32_t dbm[G::HW];        // duplicates: staged entries that repeat their predecessor's (row, column)
    int32_t dpre[G::HW];        //   and the word prefix of their count
    uint16_t xs[G::PMAX];       // product id of a staged entry of a shared bucket
    uint16_t eof[G::PMAX];      // entry of each product
    int32_t ws[4][tile::NW];       // scan workspaces (rotated)
    int64_t lbs[tile::NW];         // look-back: per-warp sums
    int32_t lbi[tile::NW];         //   and "found an inclusive prefix"
    int64_t ticket;                // next tile of this CTA
    int32_t nlist;
};

// Tile descriptor (uniform across the CTA).
struct TileDesc {
    int64_t k, r0, e0;
    int R, E, ptile;
    bool big;
};

// Number of duplicate entries before staging position q.
template <class G>
__device__ __forceinline__ int dups_before(const TileSmem<G>& S, int q) {
    return S.dpre[q >> 5] + __popc(S.dbm[q >> 5] & ((1u << (q & 31)) - 1u));
}

// Contiguous smem -> global copy of n staged entries to C[base, base+n) with
// 16-byte stores in the aligned middle.
template <class G>
__device__ __forceinline__ void tile_copy_out(const TileSmem<G>& S, int n, int64_t base, int32_t* __restrict__ ccol,
                                              double* __restrict__ cval, int tid) {
    {
        const int head = min(n, static_cast<int>((4 - (base & 3)) & 3));
        const int nv = (n - head) >> 2;
        if (tid < head) ccol[base + tid] = S.col[tid];
        int4* dst = reinterpret_cast<int4*>(ccol + base + head);
        for (int v = tid; v < nv; v += tile::NT) {
            const int q = head + 4 * v;
            dst[v] = make_int4(S.col[q], S.col[q + 1], S.col[q + 2], S.col[q + 3]);
        }
        for (int q = head + 4 * nv + tid; q < n; q += tile::NT) ccol[base + q] = S.col[q];
    }
    {
        const int head = min(n, static_cast<int>(base & 1));
        const int nv = (n - head) >> 1;
        if (tid < head) cval[base + tid] = S.val[tid];
        double2* dst = reinterpret_cast<double2*>(cval + base + head);
        for (int v = tid; v < nv; v += tile::NT) {
            const int q = head + 2 * v;
            dst[v] = make_double2(S.val[q], S.val[q + 1]);
        }
        for (int q = head + 2 * nv + tid; q < n; q += tile::NT) cval[base + q] = S.val[q];
    }
}

#ifdef SPG_TILE_PROF
// Dev instrumentation (-DSPG_TILE_PROF): per-phase clock64 totals of thread 0.
__device__ unsigned long long g_tile_prof[16];
__shared__ unsigned long long s_tp_last, s_tp_acc[16];
#define TPROF_DECL                                            \
    if (threadIdx.x == 0) {                                   \
        s_tp_last = clock64();                                \
        for (int i_ = 0; i_ < 16; ++i_) s_tp_acc[i_] = 0;     \
    }
#define TPROF(i)                                              \
    if (threadIdx.x == 0) {                                   \
        const unsigned long long t_ = clock64();              \
        s_tp_acc[i] += t_ - s_tp_last;                        \
        s_tp_last = t_;                                       \
    }
#define TPROF_FLUSH                                                              \
    if (threadIdx.x == 0)                                                        \
        for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_tile_prof[i_], s_tp_acc[i_]);
#else
#define TPROF_DECL
#define TPROF(i)
#define TPROF_FLUSH
#endif

// Prologue: the tile's rows and entries (contiguous in A and espan: one round
// trip), the entry product prefix, the product -> entry map and the per-entry
// row bucket ranges. Ends with the tables visible to the CTA.
template <class G>
__device__ __forceinline__ TileDesc tile_prologue(TileSmem<G>& S, int64_t k, const int64_t* __restrict__ arp,
                                                  const double* __restrict__ aval,
                                                  const uint64_t* __restrict__ espan,
                                                  const int64_t* __restrict__ tr, const int64_t* __restrict__ te) {
    constexpr int NT = tile::NT, EPT = G::EPT;
    const int tid = threadIdx.x;
    TileDesc T;
    T.k = k;
    const int64_t trk = tr[k];
    T.r0 = trk & ((int64_t(1) << 62) - 1);
    T.big = (trk >> 62) != 0;
    T.e0 = te[k];
    T.R = static_cast<int>((tr[k + 1] & ((int64_t(1) << 62) - 1)) - T.r0);
    T.E = static_cast<int>(te[k + 1] - T.e0);
    T.ptile = 0;
    if (T.big) return T;
    for (int t = tid; t <= T.R; t += NT) S.re[t] = static_cast<int32_t>(arp[T.r0 + t] - T.e0);
    const int per = (T.E + NT - 1) / NT;  // contiguous entries per thread (1 for typical tiles)
    uint64_t sp[EPT];
    double av[EPT];
    int sum = 0;
#pragma unroll
    for (int c = 0; c < EPT; ++c) {
        const int q = tid * per + c;
        sp[c] = 0;
        av[c] = 0.0;
        if (c < per && q < T.E) {
            sp[c] = espan[T.e0 + q];
            av[c] = aval[T.e0 + q];
        }
        sum += static_cast<int>((sp[c] >> tile::SP_LEN) & 1023u);  // 10-bit length
    }
    TPROF(15)
    int ptile;
    int pre = tile_scan(sum, &ptile, S.ws[0]);
    T.ptile = ptile;
#pragma unroll
    for (int c = 0; c < EPT; ++c) {
        const int q = tid * per + c;
        if (c < per && q < T.E) {
            const int len = static_cast<int>((sp[c] >> tile::SP_LEN) & 1023u);
            const int inrow = static_cast<int>((sp[c] >> tile::SP_IN) & 4095u);
            const int prow = pre - inrow, pr = static_cast<int>(sp[c] >> tile::SP_PR);
            S.ent[q] = TileEnt{static_cast<int64_t>(sp[c] & tile::SP_BS_MASK) - pre, av[c]};
            S.ebin[q] = static_cast<uint32_t>(tile::BPP * prow) | (static_cast<uint32_t>(tile::BPP * pr) << 16);
            S.epre[q] = pre;
            for (int x = pre; x < pre + len; ++x) S.eof[x] = static_cast<uint16_t>(q);
            pre += len;
        }
    }
    if (tid == 0) {
        S.epre[T.E] = ptile;
        S.nlist = 0;
    }
    for (int q = tid; q <= tile::CW * ptile; q += NT) S.cnt[q] = 0u;  // CW*ptile words = BPP*ptile buckets
    __syncthreads();
    return T;
}

// Gathers of the tile's products x = tid + NT*j (all issued, none consumed).
template <class G, int NJ>
__device__ __forceinline__ void tile_gather(const TileSmem<G>& S, int ptile, const int32_t* __restrict__ bcol,
                                            const double* __restrict__ bval, int32_t (&col)[NJ], double (&val)[NJ],
                                            int (&aux)[NJ]) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        aux[j] = -1;
        if (j * tile::NT >= ptile) break;  // uniform
        const int x = threadIdx.x + tile::NT * j;
        if (x < ptile) {
            const int q = S.eof[x];
            SPG_DCHECK(q >= 0 && q < G::EMAX);
            const int64_t u = S.ent[q].base + x;
            aux[j] = q;
            col[j] = __ldg(bcol + u);
            val[j] = __ldg(bval + u);
        }
    }
}

// The tile's rows of C into the staging (sorted by (row, column), duplicates
// combined in ascending k); S.rend[t] = end of row t. Returns the tile's nnz.
template <class G, int NJ>
__device__ __forceinline__ int tile_process(TileSmem<G>& S, const TileDesc& T, int cshift, int32_t (&col)[NJ],
                                            double (&val)[NJ], int (&aux)[NJ]) {
    constexpr int NT = tile::NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ptile = T.ptile;
    const int nj = (ptile + NT - 1) / NT;
    // multiply (0 + av*bv, the reference's first accumulation) and count
    int bk[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        bk[j] = -1;
        if (j >= nj) break;
        if (aux[j] >= 0) {
            const int q = aux[j];
            val[j] = dadd(0.0, dmul(S.ent[q].av, val[j]));
            const uint32_t bi = S.ebin[q];
            const int b = static_cast<int>(bi & 0xffffu) + bucket_of(col[j], cshift, static_cast<int>(bi >> 16));
            SPG_DCHECK(b >= 0 && b < 2 * tile::CW * ptile && col[j] >= 0);
            bk[j] = b;
            const int sh = (b & 1) << 4;
            aux[j] = static_cast<int>((atomicAdd(&S.cnt[b >> 1], 1u << sh) >> sh) & 0xffffu);
        }
    }
    // duplicate bitmap of this tile (the previous tile's was consumed by its copy-out)
    for (int q = tid; q < (ptile >> 5) + 2; q += NT) S.dbm[q] = 0u;
    TPROF(8)
    __syncthreads();
    TPROF(9)
    // exclusive scan of the packed counters (odd-strided blocks: conflict-free)
    {
        const int W = tile::CW * ptile;
        const int per = ((W + NT - 1) / NT) | 1;
        const int w0 = tid * per;
        constexpr int PERMAX = ((tile::CW * G::PMAX + NT - 1) / NT) | 1;
        uint32_t wd[PERMAX];
        uint32_t s = 0;
#pragma unroll
        for (int q = 0; q < PERMAX; ++q) {
            wd[q] = (q < per && w0 + q < W) ? S.cnt[w0 + q] : 0u;
            s += wd[q];
        }
        int tot;
        const int cnt_s = static_cast<int>((s & 0xffffu) + (s >> 16));
        uint32_t p2 = static_cast<uint32_t>(tile_scan(cnt_s, &tot, S.ws[1]));
#pragma unroll
        for (int q = 0; q < PERMAX; ++q) {
            if (q < per && w0 + q < W) S.cnt[w0 + q] = p2 * 0x10001u + (wd[q] << 16);
            p2 += (wd[q] + (wd[q] << 16)) >> 16;
        }
        if (tid == 0) S.cnt[W] = static_cast<uint32_t>(ptile);  // end of the last bucket
    }
    __syncthreads();
    TPROF(10)
    // place: alone in the bucket -> final; pairs ranked below; >= 3 -> list
    unsigned pair = 0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (j >= nj) break;
        uint32_t lreg = 0u;  // a >= 3 bucket whose first slot is this product
        if (bk[j] >= 0) {
            const int b = bk[j];
            const uint32_t r = __funnelshift_r(S.cnt[b >> 1], S.cnt[(b >> 1) + 1], (b & 1) << 4);
            const int st = static_cast<int>(r & 0xffffu), sz = static_cast<int>(r >> 16) - st;
            const int slot = aux[j];
            const int pos = st + slot;
            SPG_DCHECK(pos >= 0 && pos < ptile && sz >= 1 && slot < sz);
            S.col[pos] = col[j];
            if (sz == 1) {
                S.val[pos] = val[j];
            } else {
                S.xs[pos] = static_cast<uint16_t>(tid + NT * j);
                if (sz == 2) {
                    pair |= 1u << j;
                    aux[j] = pos | (slot << 16);
                } else {
                    S.val[pos] = val[j];
                    if (slot == 0) lreg = r;  // this thread sorts the bucket
                }
            }
        }
        // append >= 3 buckets to the list: one smem atomic per warp
        const unsigned has = __ballot_sync(0xffffffffu, lreg != 0u);
        if (has) {
            int b0 = 0;
            if (lane == 0) b0 = atomicAdd(&S.nlist, __popc(has));
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            SPG_DCHECK(!lreg || b0 + __popc(has & ((1u << lane) - 1u)) < G::LMAX);
            if (lreg) S.list[b0 + __popc(has & ((1u << lane) - 1u))] = lreg;
        }
    }
    TPROF(11)
    __syncthreads();
    TPROF(12)
    // order shared buckets by (column, product id), detect duplicates. A pair
    // reads only its partner's slot and, when swapped, writes only the
    // partner's slot: no barrier is needed between the compare and the write.
    bool dup = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (j >= nj) break;
        if ((pair >> j) & 1u) {
            const int pos = aux[j] & 0xffff, slot = aux[j] >> 16;
            const int other = pos + 1 - 2 * slot;
            SPG_DCHECK(other >= 0 && other < ptile);
            const int32_t oc = S.col[other];
            const int ox = S.xs[other];
            const int x = tid + NT * j;
            const int fpos = pos - slot + ((oc < col[j] || (oc == col[j] && ox < x)) ? 1 : 0);
            if (fpos != pos) S.col[fpos] = col[j];
            S.val[fpos] = val[j];
            if (oc == col[j]) {  // equal columns: the larger product id repeats the smaller
                dup = true;
                if (ox < x) atomicOr(&S.dbm[fpos >> 5], 1u << (fpos & 31));
            }
        }
    }
    const int nlist = S.nlist;
    for (int l = tid; l < nlist; l += NT) {
        const int lo = static_cast<int>(S.list[l] & 0xffffu), hi = static_cast<int>(S.list[l] >> 16);
        SPG_DCHECK(lo >= 0 && lo + 3 <= hi && hi <= ptile);
        for (int a = lo + 1; a < hi; ++a) {
            const int32_t ca = S.col[a];
            const uint16_t xa = S.xs[a];
            const double va = S.val[a];
            int c = a - 1;
            while (c >= lo && (S.col[c] > ca || (S.col[c] == ca && S.xs[c] > xa))) {
                S.col[c + 1] = S.col[c];
                S.xs[c + 1] = S.xs[c];
                S.val[c + 1] = S.val[c];
                --c;
            }
            S.col[c + 1] = ca;
            S.xs[c + 1] = xa;
            S.val[c + 1] = va;
        }
        for (int a = lo + 1; a < hi; ++a)
            if (S.col[a] == S.col[a - 1]) {
                dup = true;
                atomicOr(&S.dbm[a >> 5], 1u << (a & 31));
            }
    }
    TPROF(13)
    const int anydup = __syncthreads_or(dup);
    TPROF(14)
    if (!anydup) {
        for (int t = tid; t < T.R; t += NT) S.rend[t] = S.epre[S.re[t + 1]];
        return ptile;
    }
    // duplicates (equal (row, column); rare): the ranking marked every staged
    // entry that repeats its predecessor; their word prefix (one warp) gives
    // every head its compacted position. Runs are folded in product-id order
    // = ascending k.
    const int hw = (ptile >> 5) + 1;
    if (warp == 0) {
        constexpr int PW = (G::HW + 31) / 32;
        int c[PW], sum = 0;
#pragma unroll
        for (int u = 0; u < PW; ++u) {
            const int w = lane * PW + u;
            c[u] = w < hw ? __popc(S.dbm[w]) : 0;
            sum += c[u];
        }
        int pre = warp_inclusive_scan(sum) - sum;
#pragma unroll
        for (int u = 0; u < PW; ++u) {
            const int w = lane * PW + u;
            if (w < G::HW) S.dpre[w] = pre;
            pre += c[u];
        }
    }
    __syncthreads();
    // fold each run into its head and move the heads down (two phases: all
    // reads, a barrier, all writes), so the copy-out stays one contiguous run
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int x = tid + NT * j;
        aux[j] = -1;
        if (x < ptile && !((S.dbm[x >> 5] >> (x & 31)) & 1u)) {
            double v = S.val[x];
            for (int u = x + 1; u < ptile && ((S.dbm[u >> 5] >> (u & 31)) & 1u); ++u) v = dadd(v, S.val[u]);
            aux[j] = x - dups_before(S, x);
            SPG_DCHECK(aux[j] >= 0 && aux[j] <= x);
            col[j] = S.col[x];
            val[j] = v;
        }
    }
    for (int t = tid; t < T.R; t += NT) {
        const int pe = S.epre[S.re[t + 1]];
        S.rend[t] = pe - dups_before(S, pe);
    }
    const int nnz = ptile - dups_before(S, ptile);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NJ; ++j)
        if (aux[j] >= 0) {
            S.col[aux[j]] = col[j];
            S.val[aux[j]] = val[j];
        }
    return nnz;
}

// Exclusive prefix of tile k from the status words (all warps: 256
// predecessors per round trip). Tile k only waits on tiles with smaller
// tickets, whose CTAs publish their aggregates without waiting on anything,
// so the chain always makes progress.
template <class G>
__device__ __forceinline__ int64_t tile_look_back(TileSmem<G>& S, uint64_t* status, int64_t k, uint64_t s_first) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t excl = 0;
    for (int64_t j0 = k - 1; j0 >= 0; j0 -= tile::NT) {
        const int64_t idx = j0 - tid;
        uint64_t s = j0 == k - 1 ? s_first : (idx >= 0 ? ld_status(status + idx) : ST_INC);
        unsigned inc, upto;
        while (true) {
            inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
            const unsigned none = __ballot_sync(0xffffffffu, (s >> 62) == 0);
            upto = inc ? ((inc & (0u - inc)) << 1) - 1u : 0xffffffffu;  // lanes up to the first inclusive
            if (!(none & upto)) break;
            if ((s >> 62) == 0) s = ld_status(status + idx);
        }
        const int64_t v = warp_reduce_sum(((1u << lane) & upto) ? static_cast<int64_t>(s & ST_VAL) : int64_t(0));
        if (lane == 0) {
            S.lbs[warp] = v;
            S.lbi[warp] = inc != 0;
        }
        __syncthreads();
        bool found = false;
#pragma unroll
        for (int w = 0; w < tile::NW; ++w) {
            if (!found) {
                excl += S.lbs[w];
                found = S.lbi[w] != 0;
            }
        }
        __syncthreads();
        if (found) break;
    }
    return excl;
}

// Persistent tile kernel. Per CTA, tiles come from a global ticket; for tile F
// the order is: process F (its products already in registers) -> publish F's
// aggregate -> prologue + gathers of the next tile -> look-back, row pointers
// and copy-out of F (overlapping the next tile's gather latency).
template <class G>
__global__ void __launch_bounds__(G::NT, G::MINB) k_tile(
    const int64_t* __restrict__ arp, const double* __restrict__ aval, const uint64_t* __restrict__ espan,
    const int32_t* __restrict__ bcol, const double* __restrict__ bval, const int64_t* __restrict__ tr,
    const int64_t* __restrict__ te, int64_t ntiles, unsigned long long* __restrict__ ticket, int cshift,
    const uint64_t* __restrict__ side_cp, const uint64_t* __restrict__ side_vp, const int64_t* __restrict__ side_nnz,
    uint64_t* __restrict__ status,
    int64_t* __restrict__ crp, int32_t* __restrict__ ccol, double* __restrict__ cval) {
    constexpr int NT = tile::NT, NJ = G::NJ;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem<G>& S = *reinterpret_cast<TileSmem<G>*>(smem_raw);
    const int tid = threadIdx.x;
    TPROF_DECL

    if (tid == 0) S.ticket = static_cast<int64_t>(atomicAdd(ticket, 1ull));
    __syncthreads();
    const int64_t k0 = S.ticket;
    if (k0 >= ntiles) return;
    int32_t col[NJ];
    double val[NJ];
    int aux[NJ];
    TileDesc T = tile_prologue(S, k0, arp, aval, espan, tr, te);
    if (!T.big) tile_gather<G, NJ>(S, T.ptile, bcol, bval, col, val, aux);
    while (true) {
#ifdef SPG_TICKET_SMEM
        if (tid == 0) S.ticket = static_cast<int64_t>(atomicAdd(ticket, 1ull));
#else
        // the next ticket stays in thread 0's register while the tile is
        // processed: its round trip is only waited for at the publish barrier
        unsigned long long tk = 0;
        if (tid == 0) tk = atomicAdd(ticket, 1ull);
#endif
        TPROF(0)
        const int nnz = T.big ? 0 : tile_process<G, NJ>(S, T, cshift, col, val, aux);
        TPROF(1)
        const int64_t agg = T.big ? side_nnz[T.r0] : static_cast<int64_t>(nnz);
        if (tid == 0) st_status(status + T.k, (T.k == 0 ? ST_INC : ST_AGG) | static_cast<uint64_t>(agg));
#ifndef SPG_TICKET_SMEM
        if (tid == 0) S.ticket = static_cast<int64_t>(tk);
#endif
        __syncthreads();  // staging + rend complete, ticket visible
        TPROF(2)
        const TileDesc F = T;  // tile to finish
        const int64_t k2 = S.ticket;
        const bool more = k2 < ntiles;
        if (more) {
            T = tile_prologue(S, k2, arp, aval, espan, tr, te);
            TPROF(3)
            if (!T.big) tile_gather<G, NJ>(S, T.ptile, bcol, bval, col, val, aux);
            TPROF(4)
        }
        // finish F: offset, row pointers, copy-out
        const int64_t lbi = F.k - 1 - tid;
        const int64_t base = tile_look_back(S, status, F.k, lbi >= 0 ? ld_status(status + lbi) : ST_INC);
        TPROF(5)
        if (tid == 0 && F.k > 0) st_status(status + F.k, ST_INC | static_cast<uint64_t>(base + agg));
        if (F.big) {  // its entries are copied into C after this kernel (k_big_copy)
            if (tid == 0) crp[F.r0 + 1] = base + agg;
        } else {
            for (int t = tid; t < F.R; t += NT) crp[F.r0 + t + 1] = base + S.rend[t];
            tile_copy_out(S, nnz, base, ccol, cval, tid);
        }
        TPROF(6)
        __syncthreads();
        TPROF(7)
        if (!more) break;
    }
    TPROF_FLUSH
}

int grid_for(spg_ctx* ctx, int64_t n, int bs = 256) {
    const int64_t want = (n + bs - 1) / bs;
    const int64_t cap = int64_t(ctx->num_sms) * 16;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

// products(i) = Σ_{k∈A_i} nnz(B_k) (half a warp per row)
__global__ void k_row_products(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                               const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod) {
    const int lane = threadIdx.x & 31, sub = lane & 15, half = lane >> 4;
    const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i0 = 2 * gw; i0 < m; i0 += 2 * nw) {
        const int64_t i = i0 + half;
        int64_t e0 = 0, e1 = 0;
        if (i < m) {
            e0 = arp[i];
            e1 = arp[i + 1];
        }
        const int64_t ne = e1 - e0;
        const int64_t ne_max = max(ne, static_cast<int64_t>(__shfl_xor_sync(FULL, ne, 16)));
        int64_t p = 0;
        for (int64_t t = 0; t < ne_max; t += 16) {
            int64_t len = 0;
            if (t + sub < ne) {
                const int32_t k = __ldg(acol + e0 + t + sub);
                len = __ldg(brp + k + 1) - __ldg(brp + k);
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) len += __shfl_xor_sync(FULL, len, o);
            p += len;
        }
        if (i < m && sub == 0) prod[i] = p;
    }
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
    k_row_products<<<grid_for(ctx, 16 * m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod);
    SPG_LAUNCH_CHECK();
    exclusive_scan_i64(ctx, prod, pex, m);
    return read_scalar(ctx, pex.get() + m);
}

namespace {
// Host-side phase timer (SPG_HOST_PROF=1 prints one line per multiply).
struct HostProf {
    bool on = std::getenv("SPG_HOST_PROF") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    std::string out;
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        out += std::string(what) + "=" + std::to_string(std::chrono::duration<double, std::milli>(t - last).count()) + " ";
        last = t;
    }
    ~HostProf() {
        if (on) std::fprintf(stderr, "[spgemm host ms] %s\n", out.c_str());
    }
};

// BIG rows, dense hub path (k_hub) when the columns fit one window: the
// symbolic pass sizes the rows (side_nnz) for k_tile; the numeric pass runs
// after k_tile (hub_numeric). drows receives the BIG rows in ascending order.
constexpr int64_t HUB_MAX_COLS = HUB_W;
// CTAs per SM: the symbolic pass as many as fit (4 of 512 threads); the
// numeric pass one of 1024 threads (58 registers: a second does not fit)
int hub_grid(spg_ctx* ctx, bool numeric) {
    static const char* g = std::getenv("SPG_HUB_CTAS");
    return ctx->num_sms * (g ? std::atoi(g) : (numeric ? 1 : 2048 / (32 * SYM_NW)));
}
void hub_attr(spg_ctx* ctx) {
    static bool done[64] = {};
    if (ctx->device < 64 && done[ctx->device]) return;
    SPG_CUDA(cudaFuncSetAttribute(k_hub_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HubSymSmem)));
    SPG_CUDA(cudaFuncSetAttribute(k_hub_num, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HubSmem)));
    if (ctx->device < 64) done[ctx->device] = true;
}

int64_t hub_symbolic(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const int32_t* big_list, int nbig,
                     const int64_t* prod, int32_t* drows, int64_t* side_nnz, uint32_t* gbm, int64_t* big_products) {
    // the rows, heaviest first (each row is one CTA's job: the long ones
    // must not start last): a device sort of (products, row) pairs
    DBuf<int64_t> dprod(ctx, nbig), dnnz(ctx, nbig), sums(ctx, 2), pkeys(ctx, nbig);
    {
        k_side_gather<<<grid_for(ctx, nbig), 256, 0, ctx->stream>>>(big_list, nbig, prod, dprod);
        SPG_LAUNCH_CHECK();
        size_t tmp = 0;
        SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, dprod.get(), pkeys.get(), big_list, drows,
                                                           nbig, 0, 64, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.get(), tmp, dprod.get(), pkeys.get(), big_list, drows,
                                                           nbig, 0, 64, ctx->stream));
    }
    hub_attr(ctx);
    DBuf<unsigned> ticket(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), ctx->stream));
    {
        KTime kt(ctx, "hub_symbolic");
        k_hub_sym<<<hub_grid(ctx, false), 32 * SYM_NW, sizeof(HubSymSmem), ctx->stream>>>(drows, nbig, a->rowptr, a->colind,
                                                                               b->rowptr, b->colind, ticket, gbm,
                                                                               side_nnz);
        SPG_LAUNCH_CHECK();
    }
    k_side_gather<<<grid_for(ctx, nbig), 256, 0, ctx->stream>>>(drows, nbig, prod, dprod);
    SPG_LAUNCH_CHECK();
    k_side_gather<<<grid_for(ctx, nbig), 256, 0, ctx->stream>>>(drows, nbig, side_nnz, dnnz);
    SPG_LAUNCH_CHECK();
    size_t tmp = 0;
    SPG_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, dprod.get(), sums.get(), nbig, ctx->stream));
    DBuf<unsigned char> t(ctx, tmp);
    SPG_CUDA(cub::DeviceReduce::Sum(t.get(), tmp, dprod.get(), sums.get(), nbig, ctx->stream));
    SPG_CUDA(cub::DeviceReduce::Sum(t.get(), tmp, dnnz.get(), sums.get() + 1, nbig, ctx->stream));
    int64_t h[2];
    SPG_CUDA(cudaMemcpyAsync(h, sums.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    *big_products = h[0];
    return h[1];
}

void hub_numeric(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const int32_t* drows, int nbig,
                 const uint32_t* gbm, spg_csr* c) {
    DBuf<unsigned> ticket(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), ctx->stream));
    KTime kt(ctx, "hub_numeric");
    k_hub_num<<<hub_grid(ctx, true), 32 * NUM_NW, sizeof(HubSmem), ctx->stream>>>(
        drows, nbig, a->rowptr, a->colind, a->values, b->rowptr, b->colind, b->values, ticket, gbm, c->rowptr,
        c->colind, c->values);
    SPG_LAUNCH_CHECK();
}

// BIG rows: sort-based ESC in memory-bounded batches of consecutive big rows
// (matrices wider than one hub window).
// Fills side_cp/side_vp/side_nnz (per row of A) and keeps the batch outputs
// alive in outc/outv until k_big_copy has moved them into C.
int64_t big_rows_esc(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const int32_t* big_list, int nbig,
                     const int64_t* prod, int32_t* drows, uint64_t* side_cp, uint64_t* side_vp, int64_t* side_nnz,
                     std::vector<std::unique_ptr<DBuf<int32_t>>>& outc,
                     std::vector<std::unique_ptr<DBuf<double>>>& outv, HostProf& hprof, int64_t* big_products) {
    const int64_t n = b->ncols;
    std::vector<int32_t> hrows(nbig);
    SPG_CUDA(cudaMemcpyAsync(hrows.data(), big_list, nbig * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::sort(hrows.begin(), hrows.end());
    DBuf<int64_t> dprod(ctx, nbig);
    SPG_CUDA(cudaMemcpyAsync(drows, hrows.data(), nbig * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    DBuf<int64_t> dne(ctx, nbig);
    k_side_gather<<<grid_for(ctx, nbig), 256, 0, ctx->stream>>>(drows, nbig, prod, dprod);
    SPG_LAUNCH_CHECK();
    k_row_nnz<<<grid_for(ctx, nbig), 256, 0, ctx->stream>>>(drows, nbig, a->rowptr, dne);
    SPG_LAUNCH_CHECK();
    std::vector<int64_t> hp(nbig), hne(nbig);
    SPG_CUDA(cudaMemcpyAsync(hp.data(), dprod.get(), nbig * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(hne.data(), dne.get(), nbig * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    int colbits = 1;
    while ((int64_t(1) << colbits) < n) ++colbits;
    // 32-bit sort keys when the row-in-batch bits fit beside the column bits
    const bool k32 = colbits <= SPG_K32_COLBITS;
    const int64_t rows_cap = k32 ? (int64_t(1) << (32 - colbits)) : (int64_t(1) << 30);
    int64_t bmax = int64_t(400) << 20;  // products per batch (~24-32 B of workspace each)
    for (int64_t v : hp) bmax = std::max(bmax, v);
    *big_products = 0;
    for (int64_t v : hp) *big_products += v;
    int64_t big_nnz = 0;
    // rows without products never reach the ESC (nothing to expand): nnz 0
    std::vector<int> cut{0};  // batches of consecutive big rows
    for (int64_t r = 0, acc = 0, eacc = 0; r < nbig; ++r) {  // entry ids of a batch fit int32
        if (r > cut.back() &&
            (acc + hp[r] > bmax || r - cut.back() >= rows_cap || eacc + hne[r] > (int64_t(1) << 30))) {
            cut.push_back(static_cast<int>(r));
            acc = eacc = 0;
        }
        acc += hp[r];
        eacc += hne[r];
    }
    cut.push_back(nbig);
    int64_t pmax = 0, nbmax = 0, emax = 0;
    for (size_t t = 0; t + 1 < cut.size(); ++t) {
        int64_t P = 0, E = 0;
        for (int r = cut[t]; r < cut[t + 1]; ++r) P += hp[r], E += hne[r];
        pmax = std::max(pmax, P);
        emax = std::max(emax, E);
        nbmax = std::max<int64_t>(nbmax, cut[t + 1] - cut[t]);
    }
    DBuf<int64_t> eb(ctx, emax), elen(ctx, emax), pst(ctx, emax + 1), deoff(ctx, nbmax + 1);
    DBuf<double> eav(ctx, emax);
    DBuf<int32_t> erow(ctx, emax);
    std::vector<int64_t> heoff(nbmax + 1);
    const size_t kb = k32 ? 4 : 8;
    DBuf<unsigned char> keys(ctx, pmax * kb), keys2(ctx, pmax * kb);
    DBuf<double> vals(ctx, pmax), vals2(ctx, pmax);
    const int64_t nchmax = (pmax + RUN_CH - 1) / RUN_CH;
    DBuf<int64_t> ccnt(ctx, nchmax + 1), cbase(ctx, nchmax + 1), rstart(ctx, nbmax + 1), rend(ctx, nbmax + 1);
    size_t tmp_bytes = 0;
    if (k32)
        SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint32_t*)keys.get(), (uint32_t*)keys2.get(),
                                                 vals.get(), vals2.get(), std::max<int64_t>(pmax, 1), 0, 32,
                                                 ctx->stream));
    else
        SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint64_t*)keys.get(), (uint64_t*)keys2.get(),
                                                 vals.get(), vals2.get(), std::max<int64_t>(pmax, 1), 0, 64,
                                                 ctx->stream));
    DBuf<unsigned char> tmp(ctx, tmp_bytes);
    for (size_t t = 0; t + 1 < cut.size(); ++t) {
        const int r0 = cut[t], nb = cut[t + 1] - cut[t];
        int64_t P = 0;
        for (int r = 0; r < nb; ++r) P += hp[r0 + r];
        if (P == 0) {  // a batch of rows without products (entries over empty B rows)
            k_big_finish<<<grid_for(ctx, nb), 256, 0, ctx->stream>>>(drows + r0, nb, nullptr, nullptr, nullptr,
                                                                     nullptr, side_cp, side_vp, side_nnz);
            SPG_LAUNCH_CHECK();
            continue;
        }
        heoff[0] = 0;
        for (int r = 0; r < nb; ++r) heoff[r + 1] = heoff[r] + hne[r0 + r];
        const int64_t E = heoff[nb];
        SPG_CUDA(cudaMemcpyAsync(deoff.get(), heoff.data(), (nb + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        int rowbits = 1;
        while ((int64_t(1) << rowbits) < nb) ++rowbits;
        const int64_t nch = (P + RUN_CH - 1) / RUN_CH;
        const int rgrid = static_cast<int>(std::min<int64_t>(nch, int64_t(ctx->num_sms) * 8));
        {
            KTime kx(ctx, "big_expand");
            k_big_ent<<<std::min(nb, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
                drows + r0, nb, deoff, a->rowptr, a->colind, a->values, b->rowptr, eb, elen, eav, erow);
            SPG_LAUNCH_CHECK();
            exclusive_scan_i64(ctx, elen, pst, E);
            const int fgrid = static_cast<int>(std::min<int64_t>((P + FILL_CH - 1) / FILL_CH, ctx->num_sms * 8));
            if (k32)
                k_big_fill<uint32_t><<<fgrid, 256, 0, ctx->stream>>>(pst, E, eb, eav, erow, b->colind, b->values,
                                                                     colbits, P, (uint32_t*)keys.get(), vals);
            else
                k_big_fill<uint64_t><<<fgrid, 256, 0, ctx->stream>>>(pst, E, eb, eav, erow, b->colind, b->values,
                                                                     colbits, P, (uint64_t*)keys.get(), vals);
            SPG_LAUNCH_CHECK();
        }
        {
            KTime ks(ctx, "big_sort");
            if (k32)
                SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, (uint32_t*)keys.get(),
                                                         (uint32_t*)keys2.get(), vals.get(), vals2.get(), P, 0,
                                                         colbits + rowbits, ctx->stream));
            else
                SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, (uint64_t*)keys.get(),
                                                         (uint64_t*)keys2.get(), vals.get(), vals2.get(), P, 0,
                                                         colbits + rowbits, ctx->stream));
        }
        {
            KTime kc(ctx, "big_count");
            if (k32)
                k_run_count<uint32_t><<<rgrid, 256, 0, ctx->stream>>>((uint32_t*)keys2.get(), P, ccnt);
            else
                k_run_count<uint64_t><<<rgrid, 256, 0, ctx->stream>>>((uint64_t*)keys2.get(), P, ccnt);
            SPG_LAUNCH_CHECK();
            exclusive_scan_i64(ctx, ccnt, cbase, nch);
        }
        const int64_t total = read_scalar(ctx, cbase.get() + nch);
        big_nnz += total;
        outc.emplace_back(new DBuf<int32_t>(ctx, total));
        outv.emplace_back(new DBuf<double>(ctx, total));
        SPG_CUDA(cudaMemsetAsync(rstart.get(), 0, (nb + 1) * sizeof(int64_t), ctx->stream));
        SPG_CUDA(cudaMemsetAsync(rend.get(), 0, (nb + 1) * sizeof(int64_t), ctx->stream));
        {
            KTime kr(ctx, "big_runs");
            DBuf<int64_t> hpos(ctx, total + 1);
            SPG_CUDA(cudaMemcpyAsync(hpos.get() + total, &P, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
            const int fg = grid_for(ctx, total);
            if (k32) {
                k_run_heads<uint32_t><<<rgrid, 256, 0, ctx->stream>>>((uint32_t*)keys2.get(), P, cbase, hpos);
                SPG_LAUNCH_CHECK();
                k_run_fold<uint32_t><<<fg, 256, 0, ctx->stream>>>((uint32_t*)keys2.get(), vals2, hpos, total, colbits,
                                                                  outc.back()->get(), outv.back()->get(), rstart, rend);
            } else {
                k_run_heads<uint64_t><<<rgrid, 256, 0, ctx->stream>>>((uint64_t*)keys2.get(), P, cbase, hpos);
                SPG_LAUNCH_CHECK();
                k_run_fold<uint64_t><<<fg, 256, 0, ctx->stream>>>((uint64_t*)keys2.get(), vals2, hpos, total, colbits,
                                                                  outc.back()->get(), outv.back()->get(), rstart, rend);
            }
            SPG_LAUNCH_CHECK();
        }
        k_big_finish<<<grid_for(ctx, nb), 256, 0, ctx->stream>>>(drows + r0, nb, rstart, rend, outc.back()->get(),
                                                                 outv.back()->get(), side_cp, side_vp, side_nnz);
        SPG_LAUNCH_CHECK();
        hprof.mark("big_batch");
    }
    return big_nnz;
}
}  // namespace

namespace {
int cshift_for(int64_t ncols) {
    int bits = 1;
    while ((int64_t(1) << bits) < ncols) ++bits;
    return 32 - bits;  // col << cshift puts the top column bit at bit 31
}

// The tile kernel of geometry G over the tiles [0, ntiles).
template <class G>
void launch_tiles(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, const uint64_t* espan, const int64_t* tr,
                  const int64_t* te, int64_t ntiles, unsigned long long* ticket, int cshift, const uint64_t* side_cp,
                  const uint64_t* side_vp, const int64_t* side_nnz, uint64_t* status, spg_csr* c) {
    static bool attr_set[64] = {};
    if (ctx->device >= 64 || !attr_set[ctx->device]) {
        SPG_CUDA(cudaFuncSetAttribute(k_tile<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<G>)));
        if (ctx->device < 64) attr_set[ctx->device] = true;
    }
    int occ = 1;
    SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile<G>, G::NT, sizeof(TileSmem<G>)));
    const int grid = static_cast<int>(std::min<int64_t>(ntiles, int64_t(ctx->num_sms) * std::max(occ, 1)));
    KTime kt(ctx, "spgemm_tile");
    k_tile<G><<<grid, G::NT, sizeof(TileSmem<G>), ctx->stream>>>(a->rowptr, a->values, espan, b->colind, b->values, tr,
                                                                 te, ntiles, ticket, cshift, side_cp, side_vp,
                                                                 side_nnz, status, c->rowptr, c->colind, c->values);
    SPG_LAUNCH_CHECK();
}

// Sum of the lengths of the B rows referenced by n evenly spaced entries of A.
__global__ void k_ref_len(const int32_t* __restrict__ acol, int64_t stride, int64_t n,
                          const int64_t* __restrict__ brp, unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t k = __ldg(acol + i * stride);
        s += static_cast<unsigned long long>(__ldg(brp + k + 1) - __ldg(brp + k));
    }
    s = warp_reduce_sum(s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// Tile geometry by the mean length of the B rows that A's entries reference
// (= products / nnz(A)), estimated from up to 65536 evenly spaced entries of
// A (when A has >= 2^20 entries; smaller multiplies take the wide tiles):
// >= 32 takes the small tiles (config 5: 64, R-MAT: 744 — its tile rows
// gather from hub rows; configs 2 and 4: 16, config 1: 8). The sum stays on
// the device for the row pass and the tile flags; the host reads it with the
// row pass's totals. SPG_TILE_GEO=wide|small forces one.
int tile_geo_force() {
    static const char* g = std::getenv("SPG_TILE_GEO");
    return (g && g[0] == 'w') ? 1 : (g && g[0] == 's') ? 2 : 0;
}
int64_t sample_ref_len(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, unsigned long long* refsum) {
    SPG_CUDA(cudaMemsetAsync(refsum, 0, sizeof(unsigned long long), ctx->stream));
    if (tile_geo_force() || a->nnz < (int64_t(1) << 20) || b->nrows == 0) return 0;
    const int64_t n = std::min<int64_t>(a->nnz, 65536), stride = a->nnz / n;
    KTime kt(ctx, "tile_geometry");
    k_ref_len<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 256)), 256, 0, ctx->stream>>>(a->colind, stride, n,
                                                                                               b->rowptr, refsum);
    SPG_LAUNCH_CHECK();
    return n;
}

// Single-pass tiled multiply.
spg_csr* spgemm_tiled(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, cudaEvent_t b_data) {
    HostProf hprof;
    const int64_t m = a->nrows, n = b->ncols;
    const int cshift = cshift_for(n);
    const int force = tile_geo_force();
    DBuf<unsigned long long> refsum(ctx, 1);
    const int64_t nsamp = sample_ref_len(ctx, a, b, refsum);
    // BIG rows (and, with the hub path, MEDIUM rows too: single-row tiles whose
    // cost varies 10x stall k_tile's look-back chain) go to the side path
    static const char* esc_env = std::getenv("SPG_BIG_ESC");
    const bool hub = b->ncols <= HUB_MAX_COLS && !(esc_env && esc_env[0] == '1');
    // 1: products, entry spans, row weights, BIG-row list
    DBuf<int64_t> prod(ctx, m), wt(ctx, m), total(ctx, 1);
    DBuf<int8_t> kind(ctx, m);
    DBuf<uint64_t> espan(ctx, a->nnz);
    DBuf<int32_t> big_list(ctx, m), nbig_d(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(nbig_d.get(), 0, sizeof(int32_t), ctx->stream));
    {
        KTime kt(ctx, "row_prep");
        k_row_prep<<<grid_for(ctx, 32 * m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod, wt,
                                                                   kind, espan, big_list, nbig_d, hub, refsum,
                                                                   nsamp, force);
        SPG_LAUNCH_CHECK();
    }
    {
        size_t tmp = 0;
        SPG_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, prod.get(), total.get(), m, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        SPG_CUDA(cub::DeviceReduce::Sum(t.get(), tmp, prod.get(), total.get(), m, ctx->stream));
    }
    // 2: tile starts (weight windows; BIG rows alone)
    DBuf<int64_t> wpre(ctx, m + 1), flag(ctx, m), fpos(ctx, m + 1);
    exclusive_scan_i64(ctx, wt, wpre, m);
    {
        KTime kt(ctx, "tile_setup");
        k_tile_flags<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(wpre, kind, m, refsum, nsamp, force, flag);
        SPG_LAUNCH_CHECK();
    }
    exclusive_scan_i64(ctx, flag, fpos, m);
    const volatile int32_t* hnbig = static_cast<int32_t*>(peek_async(ctx, 64, nbig_d.get(), sizeof(int32_t)));
    const volatile int64_t* hprod = static_cast<int64_t*>(peek_async(ctx, 72, total.get(), sizeof(int64_t)));
    const volatile int64_t* hnt = static_cast<int64_t*>(peek_async(ctx, 80, fpos.get() + m, sizeof(int64_t)));
    const volatile unsigned long long* hrs =
        static_cast<unsigned long long*>(peek_async(ctx, 88, refsum.get(), sizeof(unsigned long long)));
    hprof.mark("launch1");
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    hprof.mark("sync1");
    const int nbig = *hnbig;
    const int64_t products = *hprod, ntiles = *hnt;
    const bool small = geo_small(*hrs, nsamp, force);  // the decision the row pass and the flags made
    // B's columns and values may still be arriving (trident pulls): everything
    // above read only B's row pointers
    if (b_data) SPG_CUDA(cudaStreamWaitEvent(ctx->stream, b_data, 0));
    // 3: BIG rows: sort-based ESC in batches bounded by products
    DBuf<uint64_t> side_cp(ctx, nbig ? m : 1), side_vp(ctx, nbig ? m : 1);
    DBuf<int64_t> side_nnz(ctx, nbig ? m : 1);
    DBuf<int32_t> drows(ctx, nbig ? nbig : 1);
    std::vector<std::unique_ptr<DBuf<int32_t>>> outc;
    std::vector<std::unique_ptr<DBuf<double>>> outv;
    int64_t big_products = 0, big_nnz = 0;  // C capacity = products of tile rows + exact nnz of big rows

    // hub path: one bitmap of HUB_W bits per BIG row (the symbolic pass's
    // columns, read back by the numeric pass)
    DBuf<uint32_t> gbm(ctx, (nbig && hub) ? static_cast<size_t>(nbig) * (HUB_W / 32) : 1);
    if (nbig) {
        KTime kt(ctx, "big_rows");
        if (hub)
            big_nnz = hub_symbolic(ctx, a, b, big_list, nbig, prod, drows, side_nnz, gbm, &big_products);
        else
            big_nnz = big_rows_esc(ctx, a, b, big_list, nbig, prod, drows, side_cp, side_vp, side_nnz, outc, outv,
                                   hprof, &big_products);
    }
    hprof.mark("side");
    // 4: tiles
    DBuf<int64_t> tr(ctx, ntiles + 1), te(ctx, ntiles + 1);
    DBuf<uint64_t> status(ctx, ntiles);
    {
        KTime kt(ctx, "tile_setup");
        k_tile_scatter<<<grid_for(ctx, m + 1), 256, 0, ctx->stream>>>(flag, fpos, kind, a->rowptr, m, tr, te);
        SPG_LAUNCH_CHECK();
    }
    SPG_CUDA(cudaMemsetAsync(status.get(), 0, ntiles * sizeof(uint64_t), ctx->stream));
    DBuf<unsigned long long> ticket(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned long long), ctx->stream));
    spg_csr* c = new_csr(ctx, m, n, -1);
    alloc_c_arrays(ctx, c, products - big_products + big_nnz);  // upper bound of nnz(C)
    SPG_CUDA(cudaMemsetAsync(c->rowptr, 0, sizeof(int64_t), ctx->stream));
    if (small)
        launch_tiles<GeoSmall>(ctx, a, b, espan, tr, te, ntiles, ticket, cshift, side_cp, side_vp, side_nnz, status, c);
    else
        launch_tiles<GeoWide>(ctx, a, b, espan, tr, te, ntiles, ticket, cshift, side_cp, side_vp, side_nnz, status, c);
    if (nbig && hub) {
        hub_numeric(ctx, a, b, drows, nbig, gbm, c);
    } else if (nbig) {
        KTime kt(ctx, "big_copy");
        k_big_copy<<<std::min(nbig, ctx->num_sms * 8), 256, 0, ctx->stream>>>(drows, nbig, side_cp, side_vp,
                                                                             c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    hprof.mark("launch_tile");
    c->nnz = read_scalar(ctx, c->rowptr + m);
    hprof.mark("tile");
    return c;
}
}  // namespace

#ifdef SPG_TILE_PROF
extern "C" int spg_dev_tile_prof(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_tile_prof, 16 * sizeof(unsigned long long));
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_tile_prof, z, sizeof(z));
    return 0;
}
#endif

// C = A*B (reference spgemm_local, csr.cpp:132-165).
spg_csr* spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, cudaEvent_t b_data) {
    if (a->ncols != b->nrows)
        fail(SPG_DIMENSION_ERROR,
             "spgemm: a.ncols=" + std::to_string(a->ncols) + " != b.nrows=" + std::to_string(b->nrows));
    const int64_t m = a->nrows, n = b->ncols;
    if (n > (int64_t(1) << 31)) fail(SPG_PARAMETER_ERROR, "spgemm: b.ncols must be <= 2^31 (int32 column indices)");
    if (b_data && (m == 0 || a->nnz == 0 || b->nnz == 0)) SPG_CUDA(cudaStreamWaitEvent(ctx->stream, b_data, 0));
    if (m == 0 || a->nnz == 0 || b->nnz == 0) return new_csr(ctx, m, n, 0);
    // the tile path packs B row starts in SP_BS = 30 bits: B up to 2^30 - 1
    // entries (12 GB); larger B is refused rather than multiplied slowly
    if (b->nnz >= (int64_t(1) << tile::SP_BS))
        fail(SPG_PARAMETER_ERROR, "spgemm: nnz(B) = " + std::to_string(b->nnz) +
                                      " exceeds the 2^30 - 1 entries the tile path addresses; split B by rows");
    return spgemm_tiled(ctx, a, b, b_data);
}

}  // namespace spgb
