// Micro-benchmark of hconcat variants (dev tool): 2 parts, R rows, L entries per row per part.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hcat_bench scripts/hcat_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); i += int64_t(gridDim.x) * blockDim.x)
constexpr int HCAT_MAX = 16;
struct HcatParts { const int64_t* rp[HCAT_MAX]; const int32_t* ci[HCAT_MAX]; const double* va[HCAT_MAX]; int32_t coff[HCAT_MAX]; int n; };

__global__ void v1(HcatParts P, int64_t rows, int64_t* __restrict__ orp, int32_t* __restrict__ oci, double* __restrict__ ova) {
    GRID_STRIDE(t, rows * P.n) {
        const int p = static_cast<int>(t / rows);
        const int64_t r = t - int64_t(p) * rows;
        int64_t o = 0;
        for (int q = 0; q < P.n; ++q) o += q < p ? P.rp[q][r + 1] : P.rp[q][r];
        const int64_t b = P.rp[p][r], e = P.rp[p][r + 1];
        if (p == 0) orp[r] = o;
        const int32_t* __restrict__ ci = P.ci[p];
        const double* __restrict__ va = P.va[p];
        const int32_t off = P.coff[p];
        int64_t x = b;
        for (; x + 4 <= e; x += 4, o += 4) {
            int32_t c4[4]; double v4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { c4[u] = ci[x + u]; v4[u] = va[x + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u) { oci[o + u] = c4[u] + off; ova[o + u] = v4[u]; }
        }
        for (; x < e; ++x, ++o) { oci[o] = ci[x] + off; ova[o] = va[x]; }
    }
}

// G lanes per row (32/G rows per warp pass), lanes over the row's flattened entries
template <int G>
__global__ void v2(HcatParts P, int64_t rows, int64_t* __restrict__ orp, int32_t* __restrict__ oci, double* __restrict__ ova) {
    const int lane = threadIdx.x & 31, sub = lane % G, grp = lane / G;
    const unsigned gmask = (G == 32) ? ~0u : (((1u << G) - 1u) << (grp * G));
    const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t npass = (rows + 32 / G - 1) / (32 / G);
    for (int64_t w = w0; w < npass; w += nw) {
        const int64_t r = w * (32 / G) + grp;
        const bool ok = r < rows;
        int64_t b = 0, l = 0;
        if (ok && sub < P.n) { b = P.rp[sub][r]; l = P.rp[sub][r + 1] - b; }
        int64_t pre = l;
        for (int o = 1; o < G; o <<= 1) { int64_t y = __shfl_up_sync(gmask, pre, o, G); if (sub >= o) pre += y; }
        const int64_t tot = __shfl_sync(gmask, pre, G - 1, G);
        pre -= l;
        int64_t bsum = b;
        for (int o = G / 2; o > 0; o >>= 1) bsum += __shfl_xor_sync(gmask, bsum, o, G);
        if (ok && sub == 0) orp[r] = bsum;
        int64_t pq[HCAT_MAX], bq[HCAT_MAX];
#pragma unroll
        for (int q = 0; q < HCAT_MAX; ++q) if (q < P.n) { pq[q] = __shfl_sync(gmask, pre, q, G); bq[q] = __shfl_sync(gmask, b, q, G); }
        if (!ok) continue;
        for (int64_t x = sub; x < tot; x += G) {
            int p = 0;
#pragma unroll
            for (int q = 1; q < HCAT_MAX; ++q) if (q < P.n && x >= pq[q]) p = q;
            int64_t src = 0, pp = 0;
#pragma unroll
            for (int q = 0; q < HCAT_MAX; ++q) if (q == p) { src = bq[q]; pp = pq[q]; }
            src += x - pp;
            oci[bsum + x] = P.ci[p][src] + P.coff[p];
            ova[bsum + x] = P.va[p][src];
        }
    }
}

// block per 256-row chunk: row bounds of every part in smem, then each
// part's contiguous entry range copied striped (coalesced reads), the row of
// an entry found by a binary search over the chunk's bounds in smem
__global__ void __launch_bounds__(256) v5(HcatParts P, int64_t rows, int64_t* __restrict__ orp, int32_t* __restrict__ oci, double* __restrict__ ova) {
    __shared__ int64_t sb[HCAT_MAX][257];
    __shared__ int64_t so[257];  // output start of each row of the chunk
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
            orp[r0 + i] = o;  // row nr's entry is rewritten by the next chunk with the same value
        }
        __syncthreads();
        for (int q = 0; q < P.n; ++q) {
            const int64_t e0 = sb[q][0], e1 = sb[q][nr];
            const int32_t* __restrict__ ci = P.ci[q];
            const double* __restrict__ va = P.va[q];
            for (int64_t x = e0 + tid; x < e1; x += 256) {
                int lo = 0, hi = nr - 1;  // last row with sb[q][row] <= x
                while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (sb[q][mid] <= x) lo = mid; else hi = mid - 1; }
                int64_t d = so[lo] + (x - sb[q][lo]);
                for (int q2 = 0; q2 < q; ++q2) d += sb[q2][lo + 1] - sb[q2][lo];
                oci[d] = ci[x] + P.coff[q];
                ova[d] = va[x];
            }
        }
        __syncthreads();
    }
}

int main() {
    const int64_t R = 2 << 20; const int L = 8; const int n = 2;
    HcatParts P{}; P.n = n;
    std::vector<int64_t> hrp(R + 1);
    for (int64_t r = 0; r <= R; ++r) hrp[r] = r * L;
    for (int p = 0; p < n; ++p) {
        int64_t* rp; int32_t* ci; double* va;
        cudaMalloc(&rp, (R + 1) * 8); cudaMalloc(&ci, R * L * 4); cudaMalloc(&va, R * L * 8);
        cudaMemcpy(rp, hrp.data(), (R + 1) * 8, cudaMemcpyHostToDevice);
        cudaMemset(ci, 0, R * L * 4); cudaMemset(va, 0, R * L * 8);
        P.rp[p] = rp; P.ci[p] = ci; P.va[p] = va; P.coff[p] = p * 1000;
    }
    int64_t* orp; int32_t* oci; double* ova;
    cudaMalloc(&orp, (R + 1) * 8); cudaMalloc(&oci, R * L * n * 4); cudaMalloc(&ova, R * L * n * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double bytes = 2.0 * R * L * n * 12;
    for (int v : {1, 4, 5})
        for (int g : {148 * 16, 148 * 64, 148 * 256}) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (v == 1) v1<<<g, 256>>>(P, R, orp, oci, ova);
                else if (v == 2) v2<32><<<g, 256>>>(P, R, orp, oci, ova);
                else if (v == 3) v2<16><<<g, 256>>>(P, R, orp, oci, ova);
                else if (v == 4) v2<8><<<g, 256>>>(P, R, orp, oci, ova);
                else v5<<<g, 256>>>(P, R, orp, oci, ova);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep == 2) printf("v%d grid %d: %.3f ms  %.0f GB/s\n", v, g, ms, bytes / ms / 1e6);
            }
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
