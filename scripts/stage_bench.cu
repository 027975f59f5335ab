// Micro-benchmark (dev tool): the gather floor of the ER(2^22, ~16/row)
// row-wise C = A*A pattern on one B200, by B layout and gather mechanism.
//   ldg   : warp-per-row LDG gathers from split colind/values (round-1 layout)
//   tma/A : B repacked as one block per row [values (8L) | columns (4L)]
//           padded to 16 B, rows starting at A-byte boundaries; every A entry's
//           B row is staged into shared memory by ONE cp.async.bulk issued by
//           a producer warp; consumer warps read the staged products (and,
//           with write=1, store each product's (col, av*bv) contiguously).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stage_bench stage_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

static inline uint64_t hsh(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned par) {
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}

// ---------------------------------------------------------------- ldg baseline
template <int NJ>
__global__ void __launch_bounds__(256) k_ldg(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                             const double* __restrict__ val, int64_t n, double* out, int32_t* ocol,
                                             double* oval, const int64_t* __restrict__ pre, int write) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    double acc = 0.0;
    for (int64_t i = w; i < n; i += nw) {
        const int64_t e0 = rp[i];
        const int m = static_cast<int>(rp[i + 1] - e0);
        int64_t bs = 0;
        int len = 0;
        double av = 0;
        if (lane < m) {
            const int k = col[e0 + lane];
            av = val[e0 + lane];
            bs = rp[k];
            len = static_cast<int>(rp[k + 1] - bs);
        }
        int inc = len;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(~0u, inc, o);
            if (lane >= o) inc += y;
        }
        const int p = __shfl_sync(~0u, inc, 31);
        const int pr = lane < m ? inc - len : 0x7fffffff;
        const int64_t base = bs - pr;
        const int64_t o = pre[i];
        for (int c0 = 0; c0 < p; c0 += 32 * NJ) {
            int32_t c[NJ];
            double v[NJ];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int cc = c0 + 32 * j;
                c[j] = 0;
                v[j] = 0;
                if (cc < p) {
                    const int t0 = __popc(__ballot_sync(~0u, pr <= cc)) - 1;
                    const int rel = pr - cc;
                    const unsigned sm = __reduce_or_sync(~0u, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
                    const int t = t0 + __popc(sm & ((2u << lane) - 1u));
                    const int64_t b = __shfl_sync(~0u, base, t);
                    const double a = __shfl_sync(~0u, av, t);
                    const int x = cc + lane;
                    if (x < p) {
                        c[j] = col[b + x];
                        v[j] = a * val[b + x];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int x = c0 + 32 * j + lane;
                if (x < p) {
                    if (write) {
                        ocol[o + x] = c[j];
                        oval[o + x] = v[j];
                    } else {
                        acc += v[j] + c[j];
                    }
                }
            }
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

// warp-per-row LDG gathers from the packed row blocks [cols (4*L4) | vals (8*L4)]
template <int NJ>
__global__ void __launch_bounds__(256) k_ldgp(const int64_t* __restrict__ rp, const double* __restrict__ aval,
                                              const uint64_t* __restrict__ edesc, const unsigned char* __restrict__ bp,
                                              int64_t n, double* out, int32_t* ocol, double* oval,
                                              const int64_t* __restrict__ pre, int write) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    double acc = 0.0;
    for (int64_t i = w; i < n; i += nw) {
        const int64_t e0 = rp[i];
        const int m = static_cast<int>(rp[i + 1] - e0);
        uint64_t d = 0;
        int len = 0;
        double av = 0;
        if (lane < m) {
            d = edesc[e0 + lane];
            av = aval[e0 + lane];
            len = static_cast<int>(d & 0xffffff);
        }
        int inc = len;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(~0u, inc, o);
            if (lane >= o) inc += y;
        }
        const int p = __shfl_sync(~0u, inc, 31);
        const int pr = lane < m ? inc - len : 0x7fffffff;
        // per entry: col base (in 4-byte units, relative to bp) minus product offset; val base likewise in 8-byte units
        const int64_t st = static_cast<int64_t>(d >> 24) * 16;
        const int64_t cb = st / 4 - pr;
        const int64_t vb = (st + 4 * ((len + 3) & ~3)) / 8 - pr;
        const int64_t o = pre[i];
        const int32_t* bc = reinterpret_cast<const int32_t*>(bp);
        const double* bv = reinterpret_cast<const double*>(bp);
        for (int c0 = 0; c0 < p; c0 += 32 * NJ) {
            int32_t c[NJ];
            double v[NJ];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int cc = c0 + 32 * j;
                c[j] = 0;
                v[j] = 0;
                if (cc < p) {
                    const int t0 = __popc(__ballot_sync(~0u, pr <= cc)) - 1;
                    const int rel = pr - cc;
                    const unsigned sm = __reduce_or_sync(~0u, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
                    const int t = t0 + __popc(sm & ((2u << lane) - 1u));
                    const int64_t b1 = __shfl_sync(~0u, cb, t);
                    const int64_t b2 = __shfl_sync(~0u, vb, t);
                    const double a = __shfl_sync(~0u, av, t);
                    const int x = cc + lane;
                    if (x < p) {
                        c[j] = bc[b1 + x];
                        v[j] = a * bv[b2 + x];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int x = c0 + 32 * j + lane;
                if (x < p) {
                    if (write) {
                        ocol[o + x] = c[j];
                        oval[o + x] = v[j];
                    } else {
                        acc += v[j] + c[j];
                    }
                }
            }
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

// ---------------------------------------------------------------- tma staging
constexpr int EMAX = 384;  // entries per tile (bench: tiles cut on the host)
struct StageMeta {
    uint32_t soff[EMAX];  // smem byte offset of the entry's block within the stage
    int32_t len[EMAX];
    int32_t pofs[EMAX];   // product offset of the entry within the tile
    double av[EMAX];
    int ne;
    int64_t obase;
};

template <int NST, int SB, int NCW, int MODE>  // MODE 1: one copy per entry; 2: cols and vals copied apart (slots)
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    k_tma(const int64_t* __restrict__ arp, const double* __restrict__ aval, const uint64_t* __restrict__ edesc,
          const unsigned char* __restrict__ bp, const int64_t* __restrict__ tiles, int ntiles,
          const int64_t* __restrict__ ppre, double* out, int32_t* __restrict__ ocol, double* __restrict__ oval,
          int write) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* stage = sm;  // NST * SB
    StageMeta* meta = reinterpret_cast<StageMeta*>(sm + NST * SB);
    uint64_t* full = reinterpret_cast<uint64_t*>(meta + NST);
    uint64_t* empty = full + NST;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int PER = EMAX / 32;
    if (warp == NCW) {  // producer
        int s = 0;
        unsigned ph = 0;
        int t = blockIdx.x;
        int64_t r0 = t < ntiles ? tiles[t] : 0, r1 = t < ntiles ? tiles[t + 1] : 0;
        for (; t < ntiles; t += gridDim.x) {
            const int64_t e0 = arp[r0], e1 = arp[r1];
            const int ne = static_cast<int>(e1 - e0);
            uint64_t d[PER];
            double av[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int q = u * 32 + lane;
                d[u] = 0;
                av[u] = 0;
                if (q < ne) {
                    d[u] = __ldg(edesc + e0 + q);
                    av[u] = __ldg(aval + e0 + q);
                }
            }
            const int64_t ob = ppre[r0];
            // next tile's bounds
            const int tn = t + gridDim.x;
            if (tn < ntiles) {
                r0 = tiles[tn];
                r1 = tiles[tn + 1];
            }
            mbar_wait(&empty[s], ph ^ 1);
            StageMeta& M = meta[s];
            unsigned char* dst = stage + size_t(s) * SB;
            uint32_t soff = 0;
            int pofs = 0;
            uint32_t sreg[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                sreg[u] = 0;
                if (u * 32 >= ne) break;
                const int q = u * 32 + lane;
                const int len = static_cast<int>(d[u] & 0xffffff);
                const int bytes = MODE == 1 ? ((12 * len + 15) & ~15) : 12 * ((len + 3) & ~3);
                sreg[u] = soff;
                int ib = bytes, il = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(~0u, ib, o), z = __shfl_up_sync(~0u, il, o);
                    if (lane >= o) ib += y, il += z;
                }
                sreg[u] += ib - bytes;
                if (q < ne) {
                    M.soff[q] = soff + ib - bytes;
                    M.len[q] = len;
                    M.pofs[q] = pofs + il - len;
                    M.av[q] = av[u];
                }
                soff += __shfl_sync(~0u, ib, 31);
                pofs += __shfl_sync(~0u, il, 31);
            }
            if (lane == 0) {
                M.ne = ne;
                M.obase = ob;
            }
            __syncwarp();
            if (MODE == 3) {
                const int half = lane >> 4, hl = lane & 15;
#pragma unroll
                for (int u = 0; u < PER; ++u) {
                    if (u * 32 >= ne) break;
                    for (int pi = 0; pi < 16; ++pi) {
                        const int sl = 2 * pi + half;
                        const uint64_t dd = __shfl_sync(~0u, d[u], sl);
                        const uint32_t so = __shfl_sync(~0u, sreg[u], sl);
                        if (u * 32 + sl < ne) {
                            const int len = static_cast<int>(dd & 0xffffff);
                            const int nch = 3 * ((len + 3) & ~3) / 4;
                            const unsigned char* src = bp + (dd >> 24) * 16;
                            for (int c = hl; c < nch; c += 16) cp16(dst + so + 16 * c, src + 16 * c);
                        }
                    }
                }
                cp_arrive(&full[s]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (++s == NST) s = 0, ph ^= 1;
                continue;
            }
            if (lane == 0) mbar_arrive_tx(&full[s], soff);
            __syncwarp();
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                if (u * 32 >= ne) break;
                const int q = u * 32 + lane;
                if (q < ne) {
                    const int len = static_cast<int>(d[u] & 0xffffff);
                    const unsigned char* src = bp + (d[u] >> 24) * 16;
                    if (MODE == 1) {
                        const int bytes = (12 * len + 15) & ~15;
                        if (bytes) bulk_g2s(dst + M.soff[q], src, bytes, &full[s]);
                    } else if (len) {
                        // slots: [cols of all entries | vals of all entries] would need the
                        // tile's slot total; the bench keeps the per-entry block and issues
                        // the two halves as two copies
                        const int l4 = (len + 3) & ~3;
                        bulk_g2s(dst + M.soff[q], src, 4 * l4, &full[s]);
                        bulk_g2s(dst + M.soff[q] + 4 * l4, src + 4 * l4, 8 * l4, &full[s]);
                    }
                }
            }
            if (++s == NST) s = 0, ph ^= 1;
        }
    } else {  // consumers
        int s = 0;
        unsigned ph = 0;
        double acc = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            mbar_wait(&full[s], ph);
            const StageMeta& M = meta[s];
            const unsigned char* src = stage + size_t(s) * SB;
            const int ne = M.ne;
            const int64_t ob = M.obase;
            // half-warp per entry
            const int hw = lane >> 4, hl = lane & 15;
            for (int q = warp * 2 + hw; q < ne; q += NCW * 2) {
                const int len = M.len[q];
                const double av = M.av[q];
                const int l4 = MODE == 1 ? len : ((len + 3) & ~3);
                const int32_t* cc = reinterpret_cast<const int32_t*>(src + M.soff[q] + (MODE == 1 ? 8 * len : 0));
                const double* v = reinterpret_cast<const double*>(src + M.soff[q] + (MODE == 1 ? 0 : 4 * l4));
                const int64_t o = ob + M.pofs[q];
                for (int j = hl; j < len; j += 16) {
                    const double x = av * v[j];
                    const int32_t c = cc[j];
                    if (write) {
                        ocol[o + j] = c;
                        oval[o + j] = x;
                    } else {
                        acc += x + c;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == NST) s = 0, ph ^= 1;
        }
        if (acc == 12345.678) out[0] = acc;
    }
}

__global__ void k_sum(const int32_t* c, const double* v, int64_t n, unsigned long long* out) {
    unsigned long long h = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        h += (unsigned long long)(uint32_t)c[i] * 0x9e3779b97f4a7c15ull ^ (unsigned long long)__double_as_longlong(v[i]) * (i | 1);
    atomicAdd(out, h);
}
static unsigned long long checksum(const int32_t* c, const double* v, int64_t n) {
    unsigned long long* d;
    CK(cudaMalloc(&d, 8));
    CK(cudaMemset(d, 0, 8));
    k_sum<<<1184, 256>>>(c, v, n, d);
    unsigned long long h;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return h;
}

int main() {
    const int64_t n = int64_t(1) << 22;
    // host: row lengths 8..24 (mean 16), stratified increasing columns
    std::vector<int64_t> rp(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + 8 + int64_t(hsh(i * 31 + 7) % 17);
    const int64_t nnz = rp[n];
    std::vector<int32_t> col(nnz);
    std::vector<double> val(nnz);
    for (int64_t i = 0; i < n; ++i) {
        const int L = static_cast<int>(rp[i + 1] - rp[i]);
        const int64_t stride = n / L;
        for (int t = 0; t < L; ++t) {
            col[rp[i] + t] = static_cast<int32_t>(t * stride + hsh(i * 64 + t) % stride);
            val[rp[i] + t] = double(hsh(i * 77 + t) >> 11) * (1.0 / 9007199254740992.0) + 1e-300;
        }
    }
    // products per row and their prefix
    std::vector<int64_t> ppre(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        int64_t p = 0;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) p += rp[col[e] + 1] - rp[col[e]];
        ppre[i + 1] = ppre[i] + p;
    }
    const int64_t prods = ppre[n];
    printf("n=%lld nnz=%lld products=%lld\n", (long long)n, (long long)nnz, (long long)prods);

    int64_t *d_rp, *d_ppre;
    int32_t* d_col;
    double* d_val;
    CK(cudaMalloc(&d_rp, (n + 1) * 8));
    CK(cudaMalloc(&d_ppre, (n + 1) * 8));
    CK(cudaMalloc(&d_col, nnz * 4));
    CK(cudaMalloc(&d_val, nnz * 8));
    CK(cudaMemcpy(d_rp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ppre, ppre.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_col, col.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_val, val.data(), nnz * 8, cudaMemcpyHostToDevice));
    double* out;
    CK(cudaMalloc(&out, 8));
    int32_t* ocol;
    double* oval;
    CK(cudaMalloc(&ocol, prods * 4));
    CK(cudaMalloc(&oval, prods * 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto&& fn) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        return best;
    };
    const double alg_r = nnz * 12.0 + prods * 12.0, alg_w = prods * 12.0;
    for (int write = 0; write < 2; ++write)
        for (int bpsm : {4, 8}) {
            const float ms = timeit([&] {
                k_ldg<4><<<148 * bpsm, 256>>>(d_rp, d_col, d_val, n, out, ocol, oval, d_ppre, write);
            });
            const double alg = alg_r + (write ? alg_w : 0);
            printf("ldg   write=%d blocks/SM=%d          %7.3f ms  alg %.2f GB -> %6.0f GB/s\n", write, bpsm, ms,
                   alg / 1e9, alg / ms / 1e6);
            if (write) printf("      checksum %016llx\n", checksum(ocol, oval, prods));
        }

    constexpr int NST = 4, SB = 40 * 1024, NCW = 8;
    const size_t smem = NST * SB + NST * sizeof(StageMeta) + 2 * NST * 8;
    CK(cudaFuncSetAttribute(k_tma<NST, SB, NCW, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tma<NST, SB, NCW, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tma<NST, SB, NCW, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    uint64_t* d_edesc;
    CK(cudaMalloc(&d_edesc, nnz * 8));
    for (int mode = 3; mode >= 1; --mode)
        for (int align : {16, 32, 64, 128}) {
            if (mode != 3 && align != 16) continue;
            // pack
            std::vector<uint64_t> boff16(n);
            int64_t pos = 0;
            auto blk = [&](int L) { return mode == 1 ? int64_t((12 * L + 15) & ~15) : int64_t(12 * ((L + 3) & ~3)); };
            for (int64_t k = 0; k < n; ++k) {
                pos = (pos + align - 1) / align * align;
                boff16[k] = static_cast<uint64_t>(pos / 16);
                pos += blk(static_cast<int>(rp[k + 1] - rp[k]));
            }
            std::vector<unsigned char> bp(pos, 0);
            for (int64_t k = 0; k < n; ++k) {
                const int L = static_cast<int>(rp[k + 1] - rp[k]);
                unsigned char* d = bp.data() + size_t(boff16[k]) * 16;
                if (mode == 1) {
                    memcpy(d, val.data() + rp[k], 8 * L);
                    memcpy(d + 8 * L, col.data() + rp[k], 4 * L);
                } else {
                    const int l4 = (L + 3) & ~3;
                    memcpy(d, col.data() + rp[k], 4 * L);
                    memset(d + 4 * L, 0xff, 4 * (l4 - L));
                    memcpy(d + 4 * l4, val.data() + rp[k], 8 * L);
                }
            }
            std::vector<uint64_t> ed(nnz);
            for (int64_t e = 0; e < nnz; ++e) {
                const int64_t k = col[e];
                ed[e] = (boff16[k] << 24) | uint64_t(rp[k + 1] - rp[k]);
            }
            // tiles: consecutive rows while the staged bytes fit SB and entries fit EMAX
            std::vector<int64_t> tiles{0};
            int64_t tb = 0, te = 0;
            for (int64_t i = 0; i < n; ++i) {
                int64_t rb = 0;
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) rb += blk(static_cast<int>(rp[col[e] + 1] - rp[col[e]]));
                const int64_t re = rp[i + 1] - rp[i];
                if (tb + rb > SB || te + re > EMAX) {
                    tiles.push_back(i);
                    tb = te = 0;
                }
                tb += rb;
                te += re;
            }
            tiles.push_back(n);
            const int ntiles = static_cast<int>(tiles.size() - 1);
            unsigned char* d_bp;
            int64_t* d_tiles;
            CK(cudaMalloc(&d_bp, pos));
            CK(cudaMalloc(&d_tiles, tiles.size() * 8));
            CK(cudaMemcpy(d_bp, bp.data(), pos, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d_edesc, ed.data(), nnz * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d_tiles, tiles.data(), tiles.size() * 8, cudaMemcpyHostToDevice));
            if (mode == 3)
                for (int write = 0; write < 2; ++write) {
                    const float ms = timeit([&] {
                        k_ldgp<4><<<148 * 8, 256>>>(d_rp, d_val, d_edesc, d_bp, n, out, ocol, oval, d_ppre, write);
                    });
                    const float ms8 = timeit([&] {
                        k_ldgp<8><<<148 * 8, 256>>>(d_rp, d_val, d_edesc, d_bp, n, out, ocol, oval, d_ppre, write);
                    });
                    const float ms16 = timeit([&] {
                        k_ldgp<16><<<148 * 4, 256>>>(d_rp, d_val, d_edesc, d_bp, n, out, ocol, oval, d_ppre, write);
                    });
                    const float ms16b = timeit([&] {
                        k_ldgp<16><<<148 * 8, 256>>>(d_rp, d_val, d_edesc, d_bp, n, out, ocol, oval, d_ppre, write);
                    });
                    printf("ldgp  NJ=8: %.3f ms  NJ=16 4/SM: %.3f ms  NJ=16 8/SM: %.3f\n", ms8, ms16, ms16b);
                    const double alg = alg_r + (write ? alg_w : 0);
                    printf("ldgp  write=%d align=%3d blocks/SM=8 %7.3f ms  alg %.2f GB -> %6.0f GB/s\n", write, align, ms,
                           alg / 1e9, alg / ms / 1e6);
                    if (write) printf("      checksum %016llx\n", checksum(ocol, oval, prods));
                }
            if (getenv("SKIP_TMA")) {
                CK(cudaFree(d_bp));
                CK(cudaFree(d_tiles));
                continue;
            }
            for (int write = 0; write < 2; ++write) {
                const float ms = timeit([&] {
                    if (mode == 3)
                        k_tma<NST, SB, NCW, 3><<<148, (NCW + 1) * 32, smem>>>(d_rp, d_val, d_edesc, d_bp, d_tiles,
                                                                              ntiles, d_ppre, out, ocol, oval, write);
                    else if (mode == 1)
                        k_tma<NST, SB, NCW, 1><<<148, (NCW + 1) * 32, smem>>>(d_rp, d_val, d_edesc, d_bp, d_tiles,
                                                                              ntiles, d_ppre, out, ocol, oval, write);
                    else
                        k_tma<NST, SB, NCW, 2><<<148, (NCW + 1) * 32, smem>>>(d_rp, d_val, d_edesc, d_bp, d_tiles,
                                                                              ntiles, d_ppre, out, ocol, oval, write);
                });
                const double alg = alg_r + (write ? alg_w : 0);
                printf("tma%d  write=%d align=%3d tiles=%d Bp=%.0f MB  %7.3f ms  alg %.2f GB -> %6.0f GB/s\n", mode,
                       write, align, ntiles, pos / 1e6, ms, alg / 1e9, alg / ms / 1e6);
            }
            printf("      checksum %016llx\n", (unsigned long long)checksum(ocol, oval, prods));
            CK(cudaFree(d_bp));
            CK(cudaFree(d_tiles));
        }
    return 0;
}
