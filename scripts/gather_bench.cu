// Micro-benchmark (dev tool): how fast can a B200 do the ER(2^22, 16/row)
// row-wise gather pattern of C = A*A, independent of the sort/compress work?
//   K1: warp-per-row, products gathered into registers, summed (read only)
//   K2: K1 + write every product (col,val) to a contiguous output (upper bound
//       layout) -> read+write traffic of the numeric pass
//   K3: warp-per-row with cp.async into a per-warp smem double buffer
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bench gather_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
            return 1;                                                              \
        }                                                                          \
    } while (0)

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return static_cast<uint32_t>(x);
}

// 16 entries per row with strictly increasing random columns (stratified).
__global__ void k_make(int64_t n, int64_t* rp, int32_t* col, double* val) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        rp[i + 1] = (i + 1) * 16;
        if (i == 0) rp[0] = 0;
        const int64_t stride = n / 16;
        for (int t = 0; t < 16; ++t) {
            col[i * 16 + t] = static_cast<int32_t>(t * stride + hsh(i * 16 + t) % stride);
            val[i * 16 + t] = 1.0 + (hsh(i * 77 + t) & 1023) * 1e-3;
        }
    }
}

template <int NJ>
__global__ void __launch_bounds__(256) k_gather(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, int64_t n, double* out,
                                                int32_t* ocol, double* oval, int write) {
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
        const int pre = lane < m ? inc - len : 0x7fffffff;
        const int64_t base = bs - pre;
        int32_t c[NJ];
        double v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            c[j] = 0;
            v[j] = 0;
            if (32 * j < p) {
                const int c0 = 32 * j;
                const int t0 = __popc(__ballot_sync(~0u, pre <= c0)) - 1;
                const int rel = pre - c0;
                const unsigned sm = __reduce_or_sync(~0u, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
                const int t = t0 + __popc(sm & ((2u << lane) - 1u));
                const int64_t b = __shfl_sync(~0u, base, t);
                const double a = __shfl_sync(~0u, av, t);
                const int x = c0 + lane;
                if (x < p) {
                    c[j] = col[b + x];
                    v[j] = a * val[b + x];
                }
            }
        }
        if (write) {
            const int64_t o = i * 256;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
                if (32 * j + lane < p) {
                    ocol[o + 32 * j + lane] = c[j];
                    oval[o + 32 * j + lane] = v[j];
                }
        } else {
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc += v[j] + c[j];
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

struct __align__(16) Rec {
    int32_t col;
    int32_t pad;
    double val;
};

__global__ void k_pack(const int32_t* col, const double* val, int64_t nnz, Rec* r) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz; i += int64_t(gridDim.x) * blockDim.x)
        r[i] = Rec{col[i], 0, val[i]};
}

template <int NJ>
__global__ void __launch_bounds__(256) k_gather_aos(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const double* __restrict__ val, const Rec* __restrict__ rec,
                                                    int64_t n, double* out, int32_t* ocol, double* oval, int write) {
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
        const int pre = lane < m ? inc - len : 0x7fffffff;
        const int64_t base = bs - pre;
        int32_t c[NJ];
        double v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            c[j] = 0;
            v[j] = 0;
            if (32 * j < p) {
                const int c0 = 32 * j;
                const int t0 = __popc(__ballot_sync(~0u, pre <= c0)) - 1;
                const int rel = pre - c0;
                const unsigned sm = __reduce_or_sync(~0u, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
                const int t = t0 + __popc(sm & ((2u << lane) - 1u));
                const int64_t b = __shfl_sync(~0u, base, t);
                const double a = __shfl_sync(~0u, av, t);
                const int x = c0 + lane;
                if (x < p) {
                    const Rec r = rec[b + x];
                    c[j] = r.col;
                    v[j] = a * r.val;
                }
            }
        }
        if (write) {
            const int64_t o = i * 256;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
                if (32 * j + lane < p) {
                    ocol[o + 32 * j + lane] = c[j];
                    oval[o + 32 * j + lane] = v[j];
                }
        } else {
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc += v[j] + c[j];
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

int main() {
    const int64_t n = 1 << 22;
    int64_t* rp;
    int32_t* col;
    double* val;
    CK(cudaMalloc(&rp, (n + 1) * 8));
    CK(cudaMalloc(&col, n * 16 * 4));
    CK(cudaMalloc(&val, n * 16 * 8));
    double* out;
    CK(cudaMalloc(&out, 8));
    int32_t* ocol;
    double* oval;
    CK(cudaMalloc(&ocol, n * 256 * 4));
    CK(cudaMalloc(&oval, n * 256 * 8));
    k_make<<<1184, 256>>>(n, rp, col, val);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double prods = double(n) * 256;
    for (int write = 0; write < 2; ++write)
        for (int bpsm : {2, 4, 8}) {
            const int grid = 148 * bpsm;
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(a);
                k_gather<8><<<grid, 256>>>(rp, col, val, n, out, ocol, oval, write);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const double alg = n * 16 * 12.0 + prods * 12 + (write ? prods * 12 : 0);
            printf("write=%d blocks/SM=%d  %.3f ms  %.0f Mprod/s  alg %.2f GB -> %.0f GB/s\n", write, bpsm, best,
                   prods / best / 1e3, alg / 1e9, alg / best / 1e6);
        }
    Rec* rec;
    CK(cudaMalloc(&rec, n * 16 * sizeof(Rec)));
    {
        cudaEventRecord(a);
        k_pack<<<1184, 256>>>(col, val, n * 16, rec);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("pack AoS: %.3f ms\n", ms);
    }
    for (int write = 0; write < 2; ++write)
        for (int bpsm : {4, 8}) {
            const int grid = 148 * bpsm;
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(a);
                k_gather_aos<8><<<grid, 256>>>(rp, col, val, rec, n, out, ocol, oval, write);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const double alg = n * 16 * 12.0 + prods * 12 + (write ? prods * 12 : 0);
            printf("AoS write=%d blocks/SM=%d  %.3f ms  %.0f Mprod/s  alg %.2f GB -> %.0f GB/s\n", write, bpsm, best,
                   prods / best / 1e3, alg / 1e9, alg / best / 1e6);
        }
    return 0;
}
