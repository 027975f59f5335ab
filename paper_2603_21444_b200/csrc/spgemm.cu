// Local SpGEMM C = A*B on one B200 (sm_100a): the replacement of
// spgemm_local (reference csr.cpp:132-165).
//
// Row-wise Gustavson in one pass over B:
//
//   k_row_plan   per row of A: products, staged slots, tile weight, kind; per
//                A entry its B row block (espan = block << 32 | length)
//   tiles        runs of consecutive SMALL rows within one TW-window of the
//                weight prefix (k_tile_flags + scan + k_tile_scatter); every
//                BIG row is a tile of its own, multiplied by the side path
//   k_pack_rows  B re-laid as one 128-byte-aligned block per row:
//                [columns, padded to 4 with -1 | values, padded to 4]
//   side path    BIG rows (too many slots for a warp row: R-MAT hubs) — ESC
//   k_merge      persistent, warp-specialised, one CTA per SM:
//                 * setup warp: takes tile tickets and stages the tile's A
//                   side (entry spans, A values, row pointers) into shared
//                   memory with three cp.async.bulk (TMA) copies;
//                 * 12 row workers: claim rows of the staged tiles; each
//                   worker gathers its next row's B blocks with 16-byte
//                   cp.async (half a warp per entry, a B block is contiguous)
//                   while it sorts the previous one: count into per-row
//                   column buckets (smem atomics), scan, place, order each
//                   multi-product bucket by (column, slot), sum duplicate
//                   columns in slot order = ascending k — the row's C entries
//                   replace its staged products in place;
//                 * 2 epilogue warps: decoupled look-back over the tiles'
//                   nnz for the tile's offset in C, row pointers, copy-out.
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

// ------------------------------------------------------------------ geometry
namespace mg {
#ifndef SPG_MERGE_NWORK
#define SPG_MERGE_NWORK 12
#endif
#ifndef SPG_MERGE_NST
#define SPG_MERGE_NST 3
#endif
#ifndef SPG_MERGE_TS
#define SPG_MERGE_TS 2560
#endif
constexpr int NWORK = SPG_MERGE_NWORK; // row workers
constexpr int NEPI = 2;                // epilogue warps
constexpr int WSETUP = NWORK;          // warp id of the setup warp
constexpr int WEPI = NWORK + 1;        // first epilogue warp
constexpr int NWARP = NWORK + 1 + NEPI;
constexpr int NT = 32 * NWARP;
constexpr int NST = SPG_MERGE_NST;     // tile stages
constexpr int TS = SPG_MERGE_TS;       // tile weight capacity: slots <= TS, entries/rows <= TS/8
constexpr int TE = TS / 8, TR = TS / 8;
constexpr int RS = 512;                // slots of a worker row
constexpr int J = RS / 32;             // slots per lane
constexpr int RW = 640;                // weight of a SMALL row <= RW (so entries <= 79)
constexpr int TW = TS - RW;            // tiling window
#ifndef SPG_MERGE_BPS
#define SPG_MERGE_BPS 2
#endif
constexpr int BPS = SPG_MERGE_BPS;     // column buckets per staged slot of a row
constexpr int CW = BPS * RS + 8;       // bucket words per worker (claim tag << 16 | extra count)
constexpr int EMIN = 8;                // weight of an entry >= EMIN, of a row >= EMIN
}  // namespace mg

// B row block of row k in the packed copy: 128-byte units from the packed base.
// Disjoint for consecutive rows: start(k+1) - start(k) >= 12*len(k)/128 + 1 units
// and a block is 12*roundup4(len) <= 12*len + 36 bytes.
__host__ __device__ __forceinline__ uint64_t block_of(int64_t brow_start, int64_t k) {
    return static_cast<uint64_t>((12 * brow_start) / 128 + 2 * k);
}
__host__ __device__ __forceinline__ int64_t packed_units(int64_t nnz, int64_t nrows) {
    return (12 * nnz) / 128 + 2 * nrows + 2;
}

enum : int8_t { RK_SMALL = 0, RK_BIG = 1 };

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Non-blocking probe of a phase (try_wait may suspend the thread for a while).
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Waits for the phase of `parity` to complete, backing off with nanosleep so
// that waiting warps do not take issue slots from working ones. A wait longer
// than ~20 s of SM clock traps (a scheduling bug must fail the launch, not
// hang the device).
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    if (mbar_try(b, parity)) return;
    const long long t0 = clock64();
    unsigned ns = 32;
    while (!mbar_try(b, parity)) {
        __nanosleep(ns);
        ns = min(ns * 2, 256u);
        if (clock64() - t0 > 40000000000ll) __trap();
    }
}
// 16-byte global -> shared copy (LDGSTS), completion tracked by wait_group.
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Bulk (TMA) global -> shared copy completing on an mbarrier's transaction count.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
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

#ifdef SPG_MERGE_PROF
// Dev instrumentation (-DSPG_MERGE_PROF): clock64 totals per role phase, lane 0.
__device__ unsigned long long g_merge_prof[24];
#define MP_DECL long long mp_last_ = clock64(), mp_acc_[24] = {0};
#define MP(i)                                   \
    do {                                        \
        const long long t_ = clock64();         \
        mp_acc_[i] += t_ - mp_last_;            \
        mp_last_ = t_;                          \
    } while (0)
#define MP_CNT(i) mp_acc_[i] += 1
#define MP_FLUSH                                                                                  \
    if ((threadIdx.x & 31) == 0)                                                                  \
        for (int i_ = 0; i_ < 24; ++i_)                                                           \
            if (mp_acc_[i_]) atomicAdd(&g_merge_prof[i_], static_cast<unsigned long long>(mp_acc_[i_]));
#else
#define MP_DECL
#define MP(i)
#define MP_CNT(i)
#define MP_FLUSH
#endif

// ------------------------------------------------------------- row plan
// Half a warp per row of A (two rows in flight per warp: the row is a chain of
// dependent loads arp -> acol -> brp). Per row: products, kind and the tile
// weight of a SMALL row; per entry the packed B block and the B row length.
// A row is SMALL when its staged slots (sum of roundup4(len)) fit a worker
// row and its weight sum(max(roundup4(len), EMIN)) + EMIN fits RW.
__global__ void k_row_plan(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                           const int64_t* __restrict__ brp, int64_t m, int64_t* __restrict__ prod,
                           int64_t* __restrict__ wt, int8_t* __restrict__ kind, uint64_t* __restrict__ espan,
                           int32_t* __restrict__ big_rows, int32_t* __restrict__ nbig) {
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
        int64_t p = 0, slots = 0, w = 0;
        for (int64_t t = 0; t < ne_max; t += 16) {
            int64_t len = 0, l4 = 0, we = 0;
            if (t + sub < ne) {
                const int32_t k = __ldg(acol + e0 + t + sub);
                const int64_t bs = __ldg(brp + k);
                len = __ldg(brp + k + 1) - bs;
                l4 = (len + 3) & ~int64_t(3);
                we = max(l4, int64_t(mg::EMIN));
                espan[e0 + t + sub] = (block_of(bs, k) << 32) | static_cast<uint64_t>(min(len, int64_t(0xffffffff)));
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                len += __shfl_xor_sync(FULL, len, o);
                l4 += __shfl_xor_sync(FULL, l4, o);
                we += __shfl_xor_sync(FULL, we, o);
            }
            p += len;
            slots += l4;
            w += we;
        }
        w += mg::EMIN;
        if (ok && sub == 0) {
            const bool small = slots <= mg::RS && w <= mg::RW;
            prod[i] = p;
            kind[i] = small ? RK_SMALL : RK_BIG;
            wt[i] = small ? w : 0;
            if (!small) big_rows[atomicAdd(nbig, 1)] = static_cast<int32_t>(i);
        }
    }
}

// Tile starts: row i starts a tile if it is BIG, follows a BIG row, or its
// weight prefix enters a new TW-window (so a tile of SMALL rows has weight
// < TW + RW = TS).
__global__ void k_tile_flags(const int64_t* __restrict__ wpre, const int8_t* __restrict__ kind, int64_t m,
                             int64_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        int f = 1;
        if (i > 0 && kind[i] == RK_SMALL)
            f = kind[i - 1] != RK_SMALL || (wpre[i] / mg::TW != wpre[i - 1] / mg::TW);
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

// B -> packed row blocks (block_of): a warp per row, columns then values, each
// padded to a multiple of 4 (pad columns -1, pad values 0).
__global__ void k_pack_rows(const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol,
                            const double* __restrict__ bval, int64_t n, unsigned char* __restrict__ bp) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = gw; k < n; k += nw) {
        const int64_t b0 = brp[k], len = brp[k + 1] - b0, l4 = (len + 3) & ~int64_t(3);
        int32_t* dc = reinterpret_cast<int32_t*>(bp + block_of(b0, k) * 128);
        double* dv = reinterpret_cast<double*>(dc + l4);
        for (int64_t t = lane; t < l4; t += 32) {
            const bool in = t < len;
            dc[t] = in ? __ldg(bcol + b0 + t) : -1;
            dv[t] = in ? __ldg(bval + b0 + t) : 0.0;
        }
    }
}

// ------------------------------------------------------------- k_merge
namespace mg {
enum : int { F_BIG = 1, F_END = 2 };
struct Hdr {
    int64_t k, r0, e0;
    int R, E, flags;
    int claim, slots;       // row claims, slot allocation
    int rows_done, nnz;     // finished rows and their nnz (the tile's aggregate)
};
struct __align__(16) Stage {
    double val[TS];            // staged products' values, then the rows' C values
    int32_t col[TS];           // staged products' columns, then the rows' C columns
    uint64_t espan[TE + 2];    // tile entries' B blocks (element i - (e0 & ~1))
    double aval[TE + 2];       // tile entries' A values
    int64_t arp[TR + 4];       // tile row pointers (element i - (r0 & ~1))
    uint16_t q[TS / 4];        // tile entry of each staged slot quad
    uint16_t rs0[TR];          // first slot of each row
    uint16_t perm[TS];         // per row position: the slot holding its C entry (bit 15: hole)
    uint16_t rnnz[TR];         // nnz of each row's C
    uint16_t rsrc[TR];         // staged C entries of each row (bit 15: holes among them)
    Hdr hdr;
};
struct __align__(16) Worker {
    uint32_t cnt[CW];          // bucket counters (gather: entry slot offsets)
    uint16_t rk[RS];           // per slot: rank in its bucket
    uint16_t pa[RS];           // per bucket position: the slot placed there
};
struct __align__(16) Smem {
    Stage st[NST];
    Worker wk[NWORK];
    uint64_t ready[NST];       // setup -> workers/epilogue: the stage holds tile t
    uint64_t done[NST];        // workers -> epilogue: every worker is past tile t
    uint64_t freed[NST];       // epilogue -> setup: the stage is free
};
static_assert(sizeof(Smem) <= 227 * 1024, "k_merge shared memory exceeds 227 KB");
}  // namespace mg

// Copies elements [i0, i1) of an 8-byte array g into s so that element i lands
// at s[i - (i0 & ~1)]: the 16-byte-aligned middle by one bulk copy, an odd
// tail element by the calling lane. Returns the bulk bytes (for expect_tx).
__device__ __forceinline__ unsigned stage_slice8(void* s, const void* g, int64_t i0, int64_t i1, uint64_t* bar,
                                                 int lane, bool issue) {
    const int64_t ib = i0 & ~int64_t(1), ie = i1 & ~int64_t(1);
    const unsigned bytes = ie > ib ? static_cast<unsigned>(8 * (ie - ib)) : 0u;
    if (issue) {
        if (bytes) bulk_g2s(s, static_cast<const uint64_t*>(g) + ib, bytes, bar);
    } else if (lane == 0 && (i1 & 1) && i1 - 1 >= i0) {
        static_cast<uint64_t*>(s)[i1 - 1 - ib] = __ldg(static_cast<const unsigned long long*>(g) + (i1 - 1));
    }
    return bytes;
}

// Setup warp: tickets -> stages. Publishes END into NEPI consecutive stages so
// that every epilogue warp meets one.
__device__ void merge_setup(mg::Smem& S, const int64_t* __restrict__ arp, const double* __restrict__ aval,
                            const uint64_t* __restrict__ espan, const int64_t* __restrict__ tr,
                            const int64_t* __restrict__ te, int64_t ntiles, unsigned long long* ticket,
                            const int64_t* __restrict__ side_nnz, uint64_t* __restrict__ status) {
    using namespace mg;
    const int lane = threadIdx.x & 31;
    int nend = 0;
    MP_DECL
    for (int t = 0;; ++t) {
        const int s = t % NST;
        MP(6);
        mbar_wait(&S.freed[s], ((t / NST) & 1) ^ 1);
        MP(5);
        MP_CNT(7);
        Stage& G = S.st[s];
        // the ticket is taken only once the stage is free: a tile ticketed is a
        // tile staged, so look-backs never wait on a ticket parked in a setup warp
        int64_t tk = 0;
        if (lane == 0) tk = static_cast<int64_t>(atomicAdd(ticket, 1ull));
        tk = __shfl_sync(FULL, tk, 0);
        if (tk >= ntiles) {
            if (lane == 0) {
                G.hdr.flags = F_END;
                mbar_arrive(&S.ready[s]);
            }
            if (++nend == NEPI) break;
            continue;
        }
        const int64_t k = tk;
        int64_t v = 0;
        if (lane < 4) v = __ldg((lane & 1 ? te : tr) + k + (lane >> 1));
        const int64_t trk = __shfl_sync(FULL, v, 0), e0 = __shfl_sync(FULL, v, 1);
        const int64_t trk1 = __shfl_sync(FULL, v, 2), e1 = __shfl_sync(FULL, v, 3);
        const int64_t mask = (int64_t(1) << 62) - 1;
        const int64_t r0 = trk & mask, r1 = trk1 & mask;
        const bool big = (trk >> 62) != 0;
        if (lane == 0) {
            G.hdr.k = k;
            G.hdr.r0 = r0;
            G.hdr.e0 = e0;
            G.hdr.R = static_cast<int>(r1 - r0);
            G.hdr.E = static_cast<int>(e1 - e0);
            G.hdr.flags = big ? F_BIG : 0;
            G.hdr.claim = 0;
            G.hdr.slots = 0;
            G.hdr.rows_done = 0;
            G.hdr.nnz = 0;
        }
        if (big) {
            // the side path sized the row already: publish the aggregate now
            if (lane == 0) st_status(status + k, (k == 0 ? ST_INC : ST_AGG) | static_cast<uint64_t>(side_nnz[r0]));
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.ready[s]);
        } else {
            // odd tails by plain loads, then arm the barrier and issue the bulk copies
            unsigned bytes = stage_slice8(G.espan, espan, e0, e1, &S.ready[s], lane, false);
            bytes += stage_slice8(G.aval, aval, e0, e1, &S.ready[s], lane == 1 ? 0 : 1, false);
            bytes += stage_slice8(G.arp, arp, r0, r1 + 1, &S.ready[s], lane == 2 ? 0 : 1, false);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_tx(&S.ready[s], bytes);
                stage_slice8(G.espan, espan, e0, e1, &S.ready[s], 0, true);
                stage_slice8(G.aval, aval, e0, e1, &S.ready[s], 0, true);
                stage_slice8(G.arp, arp, r0, r1 + 1, &S.ready[s], 0, true);
            }
        }
    }
    MP_FLUSH
}

// Per-worker state of a claimed row.
struct RowJob {
    int s, j, t;
    int S0, ns;  // first slot, slots
};

// Issues the cp.async gathers of row j of stage s (one commit group) and
// allocates its slots. The B block of an entry is contiguous: chunk c of the
// block goes to the column region for c < len4/4, else to the value region.
__device__ __forceinline__ void merge_gather(mg::Smem& S, RowJob& R, uint32_t* scratch,
                                             const unsigned char* __restrict__ bp) {
    using namespace mg;
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    Stage& G = S.st[R.s];
    const int64_t r0 = G.hdr.r0, e0 = G.hdr.e0;
    const int ro = static_cast<int>(r0 & 1), eo = static_cast<int>(e0 & 1);
    const int eb = static_cast<int>(G.arp[R.j + ro] - e0), ee = static_cast<int>(G.arp[R.j + 1 + ro] - e0);
    const int ne = ee - eb;  // <= 79 for a SMALL row
    int tot = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (32 * c >= ne) break;
        const int q = 32 * c + lane;
        int l4 = 0;
        if (q < ne) l4 = (static_cast<int>(static_cast<uint32_t>(G.espan[eb + q + eo])) + 3) & ~3;
        const int inc = warp_inclusive_scan(l4);
        if (q < ne) scratch[q] = static_cast<uint32_t>(tot + inc - l4);
        tot += __shfl_sync(FULL, inc, 31);
    }
    int S0 = 0;
    if (lane == 0) {
        S0 = atomicAdd(&G.hdr.slots, tot);
        G.rs0[R.j] = static_cast<uint16_t>(S0);
    }
    S0 = __shfl_sync(FULL, S0, 0);
    R.S0 = S0;
    R.ns = tot;
    __syncwarp();
    // slot quad -> tile entry
    for (int q = lane; q < ne; q += 32) {
        const int l4 = (static_cast<int>(static_cast<uint32_t>(G.espan[eb + q + eo])) + 3) & ~3;
        const int qb = (S0 + static_cast<int>(scratch[q])) >> 2;
        for (int u = 0; u < (l4 >> 2); ++u) G.q[qb + u] = static_cast<uint16_t>(eb + q);
    }
    // gathers: half a warp per entry
    for (int q0 = 0; q0 < ne; q0 += 2) {
        const int q = q0 + half;
        if (q < ne) {
            const uint64_t sp = G.espan[eb + q + eo];
            const int l4 = (static_cast<int>(static_cast<uint32_t>(sp)) + 3) & ~3;
            const int nc4 = l4 >> 2, nc = 3 * nc4;
            const int sl = S0 + static_cast<int>(scratch[q]);
            const unsigned char* src = bp + (sp >> 32) * 128;
            unsigned char* dcol = reinterpret_cast<unsigned char*>(G.col + sl);
            unsigned char* dval = reinterpret_cast<unsigned char*>(G.val + sl) - 16 * nc4;
            for (int c = hl; c < nc; c += 16) cp16((c < nc4 ? dcol : dval) + 16 * c, src + 16 * c);
        }
    }
    cp_commit();
}

#ifdef SPG_MERGE_PROF
#define SP(i)                                  \
    do {                                       \
        const long long t_ = clock64();        \
        sp[i] += t_ - sp_last;                 \
        sp_last = t_;                          \
    } while (0)
#else
#define SP(i)
#endif
// Sorts a gathered row without moving its entries: every slot's value
// becomes 0 + a*b in place, and perm[q] (q in [0, p), p the row's products)
// names the slot of the q-th C entry in column order. Equal columns are
// summed into the first of their run in slot order (= ascending k); the
// others are marked as holes (bit 15) that the copy-out skips. Returns
// p | holes << 16.
__device__ __noinline__ uint32_t merge_sort_row(mg::Smem& S, const RowJob& R, mg::Worker& W
#ifdef SPG_MERGE_PROF
                                                , long long* sp
#endif
) {
    using namespace mg;
    const int lane = threadIdx.x & 31;
#ifdef SPG_MERGE_PROF
    long long sp_last = clock64();
#endif
    Stage& G = S.st[R.s];
    const int S0 = R.S0, ns = R.ns;
    const int eo = static_cast<int>(G.hdr.e0 & 1);
    const int32_t* col = G.col + S0;
    double* val = G.val + S0;
    uint16_t* pb = G.perm + S0;
    const int nw = (ns + 31) >> 5;
    // column range of the row (padding slots hold -1)
    uint32_t cmin = 0xffffffffu;
    int cmax = -1;
    for (int i = 0; i < nw; ++i) {
        const int sl = 32 * i + lane;
        const int c = sl < ns ? col[sl] : -1;
        cmin = min(cmin, static_cast<uint32_t>(c));
        cmax = max(cmax, c);
    }
    cmin = __reduce_min_sync(FULL, cmin);
    cmax = static_cast<int>(__reduce_max_sync(FULL, static_cast<unsigned>(max(cmax, 0))));
    SP(0);
    if (cmin == 0xffffffffu) return 0;  // no products (empty B rows only)
    // buckets: nb in [256, BPS * RS], monotone in the column over the row's range
    const int nb = max(256, (BPS * ns + 255) & ~255);
    const int K = nb >> 5;  // bucket words per lane
    const int sh = __clz(max(static_cast<uint32_t>(cmax) - cmin, 1u));
    uint32_t* cnt = W.cnt;
    for (int u = 0; u < (K >> 2); ++u) reinterpret_cast<uint4*>(cnt + lane * K)[u] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    // values (0 + a*b, in place), then each product's rank in its bucket:
    // every product writes its slot into the bucket's claim tag, the one that
    // reads its own slot back has rank 0, the others take 1 + an atomic count
    // (rank order within a bucket is arbitrary; the ordering below sorts a
    // bucket of several by (column, slot))
    uint16_t* tag = reinterpret_cast<uint16_t*>(cnt) + 1;  // high half of each bucket word
#pragma unroll 4
    for (int i = 0; i < nw; ++i) {
        const int sl = 32 * i + lane;
        if (sl < ns) {
            const int c = col[sl];
            const double bv = val[sl];
            const double av = G.aval[G.q[(S0 + sl) >> 2] + eo];
            val[sl] = dadd(0.0, dmul(av, bv));
            if (c >= 0) {
                const uint32_t b = __umulhi((static_cast<uint32_t>(c) - cmin) << sh, static_cast<uint32_t>(nb));
                tag[2 * b] = static_cast<uint16_t>(sl + 1);
            }
        }
    }
    __syncwarp();
#pragma unroll 4
    for (int i = 0; i < nw; ++i) {
        const int sl = 32 * i + lane;
        const int c = sl < ns ? col[sl] : -1;
        if (c >= 0) {
            const uint32_t b = __umulhi((static_cast<uint32_t>(c) - cmin) << sh, static_cast<uint32_t>(nb));
            uint32_t rank = 0;
            if (tag[2 * b] != sl + 1) rank = 1u + (atomicAdd(&cnt[b], 1u) & 0xffffu);
            W.rk[sl] = static_cast<uint16_t>(rank);
        }
    }
    __syncwarp();
    SP(1);
    // exclusive scan of the bucket sizes (claimed + extra): word b becomes E[b]
    uint32_t* wp = cnt + lane * K;
    constexpr int KMAX = BPS * RS / 32;
    uint32_t wv[KMAX];
    int sum = 0;
#pragma unroll
    for (int u = 0; u < KMAX; ++u) {
        wv[u] = 0;
        if (u < K) {
            const uint32_t x = wp[u];
            wv[u] = (x >> 16 ? 1u : 0u) + (x & 0xffffu);
        }
        sum += static_cast<int>(wv[u]);
    }
    const int inc = warp_inclusive_scan(sum);
    const int total = __shfl_sync(FULL, inc, 31);
    {
        uint32_t e = static_cast<uint32_t>(inc - sum);
#pragma unroll
        for (int u = 0; u < KMAX; ++u) {
            if (u < K) wp[u] = e;
            e += wv[u];
        }
    }
    if (lane == 31) cnt[nb] = static_cast<uint32_t>(total);
    __syncwarp();
    SP(2);
    // place: a product alone in its bucket is final; buckets of several are
    // listed by position (pa) and ordered below
    bool multi = false;
#pragma unroll 2
    for (int i = 0; i < nw; ++i) {
        const int sl = 32 * i + lane;
        const int c = sl < ns ? col[sl] : -1;
        if (c >= 0) {
            const uint32_t b = __umulhi((static_cast<uint32_t>(c) - cmin) << sh, static_cast<uint32_t>(nb));
            const uint32_t st = cnt[b], n = cnt[b + 1] - st;
            const int pos = static_cast<int>(st) + W.rk[sl];
            if (n == 1) {
                pb[pos] = static_cast<uint16_t>(sl);
            } else {
                W.pa[pos] = static_cast<uint16_t>(sl);
                multi = true;
            }
        }
    }
    SP(3);
    if (!__any_sync(FULL, multi)) return static_cast<uint32_t>(total);
    __syncwarp();
    // buckets of several: each product's place in (column, slot) order from
    // its mates; a product equal in column to a mate of smaller slot becomes
    // a hole, and the first of a run sums the run in slot order (= ascending k)
    int holes = 0;
    for (int i = 0; i < nw; ++i) {
        const int sl = 32 * i + lane;
        const int c = sl < ns ? col[sl] : -1;
        if (c < 0) continue;
        const uint32_t b = __umulhi((static_cast<uint32_t>(c) - cmin) << sh, static_cast<uint32_t>(nb));
        const int st = static_cast<int>(cnt[b]), n = static_cast<int>(cnt[b + 1]) - st;
        if (n < 2) continue;
        int lo = 0, eqb = 0, eqa = 0;
        for (int u = 0; u < n; ++u) {
            const int s2 = W.pa[st + u];
            const int mc = col[s2];
            lo += mc < c ? 1 : 0;
            eqb += (mc == c && s2 < sl) ? 1 : 0;
            eqa += (mc == c && s2 > sl) ? 1 : 0;
        }
        pb[st + lo + eqb] = static_cast<uint16_t>(sl | (eqb ? 0x8000 : 0));
        if (eqb) {
            ++holes;
        } else if (eqa) {
            // followers in slot order: repeatedly the smallest equal slot above the last
            double acc = val[sl];
            int last = sl;
            for (int f = 0; f < eqa; ++f) {
                int nxt = 0x7fffffff;
                for (int u = 0; u < n; ++u) {
                    const int s2 = W.pa[st + u];
                    if (s2 > last && s2 < nxt && col[s2] == c) nxt = s2;
                }
                acc = dadd(acc, val[nxt]);
                last = nxt;
            }
            val[sl] = acc;
        }
    }
    holes = __reduce_add_sync(FULL, holes);
    SP(4);
    return static_cast<uint32_t>(total) | (static_cast<uint32_t>(holes) << 16);
}

// Row worker: claim -> gather (one row ahead) -> sort. A worker arrives on a
// tile's `done` barrier once it has moved past the tile and finished its own
// rows of it (the pending row of the tile, if any, is finished first). The
// pending row is also finished before the worker blocks on a stage that is
// not staged yet.
__device__ void merge_worker(mg::Smem& S, int w, const unsigned char* __restrict__ bp, uint64_t* __restrict__ status) {
    using namespace mg;
    const int lane = threadIdx.x & 31;
    Worker& W = S.wk[w];
    int cur = 0;
    RowJob P{-1, 0, 0, 0, 0};
    bool owe = false;
    MP_DECL
#ifdef SPG_MERGE_PROF
    long long sp_acc[5] = {0, 0, 0, 0, 0};
#endif
    auto finish = [&](bool one_in_flight) {
        MP(1);
        if (one_in_flight) cp_wait<1>();
        else cp_wait<0>();
        __syncwarp();
        MP(2);
#ifdef SPG_MERGE_PROF
        const uint32_t res = merge_sort_row(S, P, W, sp_acc);
#else
        const uint32_t res = merge_sort_row(S, P, W);
#endif
        const int nnz = static_cast<int>((res & 0xffffu) - (res >> 16));
        MP(3);
        MP_CNT(4);
        if (lane == 0) {
            // the worker finishing a tile's last row publishes the tile's
            // aggregate at once (not behind the epilogue's look-backs)
            Hdr& H = S.st[P.s].hdr;
            S.st[P.s].rnnz[P.j] = static_cast<uint16_t>(nnz);
            S.st[P.s].rsrc[P.j] = static_cast<uint16_t>((res & 0xffffu) | (res >> 16 ? 0x8000u : 0u));
            atomicAdd(&H.nnz, nnz);
            __threadfence_block();
            if (atomicAdd(&H.rows_done, 1) == H.R - 1) {
                const int agg = atomicAdd(&H.nnz, 0);
                st_status(status + H.k, (H.k == 0 ? ST_INC : ST_AGG) | static_cast<uint64_t>(agg));
            }
        }
        if (owe) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.done[P.s]);
        }
        P.s = -1;
        owe = false;
        MP(14);
    };
    while (true) {
        RowJob N{-1, 0, 0, 0, 0};
        while (true) {
            const int s = cur % NST;
            // never block on a stage while a gathered row is pending: the
            // pending row may be the last of a tile whose aggregate the
            // look-backs (and so the refill of this stage) wait for
            if (P.s >= 0 && !mbar_test(&S.ready[s], (cur / NST) & 1)) finish(false);
            MP(1);
            mbar_wait(&S.ready[s], (cur / NST) & 1);
            MP(0);
            Hdr& H = S.st[s].hdr;
            const int flags = *reinterpret_cast<volatile int*>(&H.flags);
            if (flags & F_END) break;
            if (!(flags & F_BIG)) {
                int j = 0;
                if (lane == 0) j = atomicAdd(&H.claim, 1);
                j = __shfl_sync(FULL, j, 0);
                if (j < H.R) {
                    N.s = s;
                    N.j = j;
                    N.t = cur;
                    break;
                }
            }
            if (P.s >= 0 && P.t == cur) owe = true;
            else if (lane == 0) mbar_arrive(&S.done[s]);
            ++cur;
        }
        MP(1);
        if (N.s >= 0) merge_gather(S, N, W.cnt, bp);
        MP(13);
        if (P.s >= 0) finish(N.s >= 0);
        if (N.s < 0) break;
        P = N;
    }
#ifdef SPG_MERGE_PROF
    for (int i = 0; i < 5; ++i) mp_acc_[16 + i] += sp_acc[i];
#endif
    MP_FLUSH
}

// Exclusive prefix of tile k (one warp, 128 predecessors per round trip).
#ifdef SPG_MERGE_PROF
__device__ unsigned long long g_lb_prof[4];
#endif
__device__ __forceinline__ int64_t merge_look_back(const uint64_t* status, int64_t k) {
    const int lane = threadIdx.x & 31;
    int64_t excl = 0;
    for (int64_t j0 = k - 1;; j0 -= 128) {
#ifdef SPG_MERGE_PROF
        if (lane == 0) atomicAdd(&g_lb_prof[0], 1ull);
#endif
        uint64_t sv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t idx = j0 - (32 * u + lane);
            sv[u] = idx >= 0 ? ld_status(status + idx) : ST_INC;
        }
        int first = 128;
        const long long t0 = clock64();
        while (true) {
            first = 128;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned mk = __ballot_sync(FULL, (sv[u] >> 62) == 2);
                if (mk && first == 128) first = 32 * u + __ffs(mk) - 1;
            }
            bool wait = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) wait |= (32 * u + lane <= first) && (sv[u] >> 62) == 0;
            if (!__any_sync(FULL, wait)) break;
            if (clock64() - t0 > 40000000000ll) __trap();
#ifdef SPG_MERGE_PROF
            if (lane == 0) atomicAdd(&g_lb_prof[1], 1ull);
#endif
            __nanosleep(64);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t idx = j0 - (32 * u + lane);
                if ((32 * u + lane <= first) && (sv[u] >> 62) == 0) sv[u] = ld_status(status + idx);
            }
        }
        int64_t part = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (32 * u + lane <= first) part += static_cast<int64_t>(sv[u] & ST_VAL);
        excl += warp_reduce_sum(part);
        if (first < 128) break;
    }
    return excl;
}

// Epilogue warp e: tiles t = e, e + NEPI, ... of this CTA.
__device__ void merge_epilogue(mg::Smem& S, int e, uint64_t* __restrict__ status,
                               const int64_t* __restrict__ side_nnz, int64_t* __restrict__ crp,
                               int32_t* __restrict__ ccol, double* __restrict__ cval) {
    using namespace mg;
    const int lane = threadIdx.x & 31;
    MP_DECL
    for (int t = e;; t += NEPI) {
        const int s = t % NST;
        const unsigned par = (t / NST) & 1;
        MP(10);
        mbar_wait(&S.ready[s], par);
        Stage& G = S.st[s];
        if (*reinterpret_cast<volatile int*>(&G.hdr.flags) & F_END) break;
        mbar_wait(&S.done[s], par);
        MP(8);
        MP_CNT(11);
        const int64_t k = G.hdr.k, r0 = G.hdr.r0;
        const int R = G.hdr.R;
        const bool big = (G.hdr.flags & F_BIG) != 0;
        // the tile's aggregate is already published (setup for a BIG tile,
        // the worker of the last row otherwise)
        const int64_t agg = big ? side_nnz[r0] : static_cast<int64_t>(G.hdr.nnz);
        MP(10);
        const int64_t excl = k == 0 ? 0 : merge_look_back(status, k);
        MP(9);
        if (lane == 0 && k > 0) st_status(status + k, ST_INC | static_cast<uint64_t>(excl + agg));
        if (big) {
            if (lane == 0) crp[r0 + 1] = excl + agg;
        } else {
            int64_t carry = excl;
            for (int c0 = 0; c0 < R; c0 += 32) {
                const int j = c0 + lane;
                const int nj = j < R ? G.rnnz[j] : 0;
                const int inc = warp_inclusive_scan(nj);
                if (j < R) crp[r0 + j + 1] = carry + inc;
                const int nr = min(32, R - c0);
                for (int jj = 0; jj < nr; ++jj) {
                    const int n = __shfl_sync(FULL, nj, jj);
                    const int64_t o = carry + __shfl_sync(FULL, inc, jj) - n;
                    const int s0 = G.rs0[c0 + jj], src = G.rsrc[c0 + jj], p = src & 0x7fff;
                    const uint16_t* pm = G.perm + s0;
                    if (!(src & 0x8000)) {
                        for (int qq = lane; qq < p; qq += 32) {
                            const int sl = s0 + pm[qq];
                            ccol[o + qq] = G.col[sl];
                            cval[o + qq] = G.val[sl];
                        }
                    } else {  // duplicates left holes: compact while copying
                        int64_t d = o;
                        for (int q0 = 0; q0 < p; q0 += 32) {
                            const int qq = q0 + lane;
                            const int e = qq < p ? pm[qq] : 0x8000;
                            const bool keep = !(e & 0x8000);
                            const unsigned km = __ballot_sync(FULL, keep);
                            if (keep) {
                                const int64_t at = d + __popc(km & ((1u << lane) - 1u));
                                ccol[at] = G.col[s0 + e];
                                cval[at] = G.val[s0 + e];
                            }
                            d += __popc(km);
                        }
                    }
                }
                carry += __shfl_sync(FULL, inc, 31);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.freed[s]);
    }
    MP_FLUSH
}

__global__ void __launch_bounds__(mg::NT, 1)
    k_merge(const int64_t* __restrict__ arp, const double* __restrict__ aval, const uint64_t* __restrict__ espan,
            const unsigned char* __restrict__ bp, const int64_t* __restrict__ tr, const int64_t* __restrict__ te,
            int64_t ntiles, unsigned long long* __restrict__ ticket, const int64_t* __restrict__ side_nnz,
            uint64_t* __restrict__ status, int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
            double* __restrict__ cval) {
    using namespace mg;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&S.ready[s], 1);
            mbar_init(&S.done[s], NWORK);
            mbar_init(&S.freed[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < NWORK) merge_worker(S, warp, bp, status);
    else if (warp == WSETUP) merge_setup(S, arp, aval, espan, tr, te, ntiles, ticket, side_nnz, status);
    else merge_epilogue(S, warp - WEPI, status, side_nnz, crp, ccol, cval);
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

// Each head sums its run sequentially from memory (runs are short except
// for hub columns, where one thread walks the run and the others skip), and
// records where its row's output starts (first run of the row) and ends (last
// run): rows of the batch without products keep start = end = 0.
template <typename K>
__global__ void __launch_bounds__(256) k_run_sum(const K* __restrict__ keys, const double* __restrict__ vals, int64_t n,
                                                 const int64_t* __restrict__ cbase, int colbits,
                                                 int32_t* __restrict__ ocol, double* __restrict__ oval,
                                                 int64_t* __restrict__ rowstart, int64_t* __restrict__ rowend) {
    __shared__ int ws[9];
    const K cmask = (K(1) << colbits) - 1;
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
            const int64_t i = i0 + u;
            const K key = keys[i];
            double sum = dadd(0.0, vals[i]);
            int64_t v = i + 1;
            for (; v < n && keys[v] == key; ++v) sum = dadd(sum, vals[v]);
            ocol[o] = static_cast<int32_t>(key & cmask);
            oval[o] = sum;
            if (i == 0 || (keys[i - 1] >> colbits) != (key >> colbits)) rowstart[key >> colbits] = o;
            if (v == n || (keys[v] >> colbits) != (key >> colbits)) rowend[key >> colbits] = o + 1;
            ++o;
        }
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

// BIG rows' sorted products into C[crp[r], crp[r+1]) (after k_tile wrote the
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

#ifdef SPG_MERGE_PROF
}  // namespace
}  // namespace spgb
extern "C" int spg_dev_merge_prof(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, spgb::g_merge_prof, 24 * sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 24, spgb::g_lb_prof, 4 * sizeof(unsigned long long));
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(spgb::g_merge_prof, z, sizeof(z));
    cudaMemcpyToSymbol(spgb::g_lb_prof, z, 4 * sizeof(unsigned long long));
    return 0;
}
namespace spgb {
namespace {
#endif

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

// BIG rows: sort-based ESC in memory-bounded batches of consecutive big rows.
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
            if (k32)
                k_run_sum<uint32_t><<<rgrid, 256, 0, ctx->stream>>>((uint32_t*)keys2.get(), vals2, P, cbase, colbits,
                                                                    outc.back()->get(), outv.back()->get(), rstart, rend);
            else
                k_run_sum<uint64_t><<<rgrid, 256, 0, ctx->stream>>>((uint64_t*)keys2.get(), vals2, P, cbase, colbits,
                                                                    outc.back()->get(), outv.back()->get(), rstart, rend);
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

// C = A*B (reference spgemm_local, csr.cpp:132-165).
spg_csr* spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, cudaEvent_t b_data) {
    if (a->ncols != b->nrows)
        fail(SPG_DIMENSION_ERROR,
             "spgemm: a.ncols=" + std::to_string(a->ncols) + " != b.nrows=" + std::to_string(b->nrows));
    const int64_t m = a->nrows, n = b->ncols;
    if (n > (int64_t(1) << 31)) fail(SPG_PARAMETER_ERROR, "spgemm: b.ncols must be <= 2^31 (int32 column indices)");
    if (b_data && (m == 0 || a->nnz == 0 || b->nnz == 0)) SPG_CUDA(cudaStreamWaitEvent(ctx->stream, b_data, 0));
    if (m == 0 || a->nnz == 0 || b->nnz == 0) return new_csr(ctx, m, n, 0);
    if (packed_units(b->nnz, b->nrows) >= (int64_t(1) << 32))
        fail(SPG_PARAMETER_ERROR, "spgemm: B too large for 32-bit packed block offsets");
    HostProf hprof;
    // 1: row plan (products, kind, weight; entry spans), BIG-row list
    DBuf<int64_t> prod(ctx, m), wt(ctx, m), total(ctx, 1);
    DBuf<int8_t> kind(ctx, m);
    DBuf<uint64_t> espan(ctx, a->nnz + 2);
    DBuf<int32_t> big_list(ctx, m), nbig_d(ctx, 1);
    SPG_CUDA(cudaMemsetAsync(nbig_d.get(), 0, sizeof(int32_t), ctx->stream));
    {
        KTime kt(ctx, "row_plan");
        k_row_plan<<<grid_for(ctx, 16 * m), 256, 0, ctx->stream>>>(a->rowptr, a->colind, b->rowptr, m, prod, wt,
                                                                   kind, espan, big_list, nbig_d);
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
        k_tile_flags<<<grid_for(ctx, m), 256, 0, ctx->stream>>>(wpre, kind, m, flag);
        SPG_LAUNCH_CHECK();
    }
    exclusive_scan_i64(ctx, flag, fpos, m);
    const volatile int32_t* hnbig = static_cast<int32_t*>(peek_async(ctx, 64, nbig_d.get(), sizeof(int32_t)));
    const volatile int64_t* hprod = static_cast<int64_t*>(peek_async(ctx, 72, total.get(), sizeof(int64_t)));
    const volatile int64_t* hnt = static_cast<int64_t*>(peek_async(ctx, 80, fpos.get() + m, sizeof(int64_t)));
    hprof.mark("launch1");
    // B's columns and values may still be arriving (trident pulls): everything
    // above read only B's row pointers
    if (b_data) SPG_CUDA(cudaStreamWaitEvent(ctx->stream, b_data, 0));
    // 3: packed B (one 128-byte-aligned block per row)
    DBuf<unsigned char> bp(ctx, static_cast<size_t>(packed_units(b->nnz, b->nrows)) * 128);
    {
        KTime kt(ctx, "pack_b");
        k_pack_rows<<<grid_for(ctx, 32 * b->nrows), 256, 0, ctx->stream>>>(b->rowptr, b->colind, b->values,
                                                                          b->nrows, bp);
        SPG_LAUNCH_CHECK();
    }
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    hprof.mark("sync1");
    const int nbig = *hnbig;
    const int64_t products = *hprod, ntiles = *hnt;
    // 4: BIG rows
    DBuf<uint64_t> side_cp(ctx, nbig ? m : 1), side_vp(ctx, nbig ? m : 1);
    DBuf<int64_t> side_nnz(ctx, nbig ? m : 1);
    DBuf<int32_t> drows(ctx, nbig ? nbig : 1);
    std::vector<std::unique_ptr<DBuf<int32_t>>> outc;
    std::vector<std::unique_ptr<DBuf<double>>> outv;
    int64_t big_products = 0, big_nnz = 0;
    if (nbig) {
        KTime kt(ctx, "big_rows");
        big_nnz = big_rows_esc(ctx, a, b, big_list, nbig, prod, drows, side_cp, side_vp, side_nnz, outc, outv, hprof,
                               &big_products);
    }
    hprof.mark("side");
    // 5: tiles
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
    if (!ctx->tile_attr_set) {
        SPG_CUDA(cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(mg::Smem)));
        ctx->tile_attr_set = true;
    }
    {
        KTime kt(ctx, "spgemm_merge");
        k_merge<<<ctx->num_sms, mg::NT, sizeof(mg::Smem), ctx->stream>>>(a->rowptr, a->values, espan, bp, tr, te,
                                                                         ntiles, ticket, side_nnz, status, c->rowptr,
                                                                         c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    if (nbig) {
        KTime kt(ctx, "big_copy");
        k_big_copy<<<std::min(nbig, ctx->num_sms * 8), 256, 0, ctx->stream>>>(drows, nbig, side_cp, side_vp,
                                                                             c->rowptr, c->colind, c->values);
        SPG_LAUNCH_CHECK();
    }
    hprof.mark("launch_merge");
    c->nnz = read_scalar(ctx, c->rowptr + m);
    hprof.mark("merge");
    return c;
}

}  // namespace spgb
