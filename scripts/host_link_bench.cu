// Dev tool: host link (PCIe) bandwidth into / out of pinned host memory, as
// the e2e path uses it: one stream vs several streams each moving interleaved
// chunks, D2H alone, H2D alone and both directions at once.
// usage: host_link_bench [MB]
// Also: D2H into malloc'd memory registered with cudaHostRegister (what the
// bench's numpy buffers are), with and without transparent huge pages.
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t ev = (x);                                                          \
        if (ev != cudaSuccess) {                                                       \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(ev));          \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atoi(argv[1]) : 2048;
    const size_t bytes = mb << 20;
    void *d, *h, *d2, *h2;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMalloc(&d2, bytes));
    CK(cudaMallocHost(&h, bytes));
    CK(cudaMallocHost(&h2, bytes));
    CK(cudaMemset(d, 1, bytes));
    CK(cudaMemset(d2, 2, bytes));
    std::vector<cudaStream_t> st(8);
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    printf("%zu MB per direction\n", mb);
    // dir: 0 = D2H, 1 = H2D, 2 = both at once (same streams count each way)
    for (int dir = 0; dir < 3; ++dir)
        for (int ns : {1, 2, 4}) {
            for (size_t chunk : {size_t(64) << 20, bytes}) {
                if (chunk == bytes && ns > 1) continue;
                float best = 1e9;
                for (int it = 0; it < 4; ++it) {
                    CK(cudaDeviceSynchronize());
                    CK(cudaEventRecord(a, 0));
                    int k = 0;
                    for (size_t off = 0; off < bytes; off += chunk, ++k) {
                        const size_t n = bytes - off < chunk ? bytes - off : chunk;
                        cudaStream_t s = st[k % ns];
                        if (k < ns) CK(cudaStreamWaitEvent(s, a, 0));
                        if (dir != 1) CK(cudaMemcpyAsync((char*)h + off, (char*)d + off, n, cudaMemcpyDeviceToHost, s));
                        if (dir != 0) {
                            cudaStream_t s2 = dir == 2 ? st[4 + k % ns] : s;
                            if (dir == 2 && k < ns) CK(cudaStreamWaitEvent(s2, a, 0));
                            CK(cudaMemcpyAsync((char*)d2 + off, (char*)h2 + off, n, cudaMemcpyHostToDevice, s2));
                        }
                    }
                    for (int i = 0; i < 8; ++i) {
                        cudaEvent_t e;
                        CK(cudaEventCreate(&e));
                        CK(cudaEventRecord(e, st[i]));
                        CK(cudaStreamWaitEvent(0, e, 0));
                    }
                    CK(cudaEventRecord(b, 0));
                    CK(cudaEventSynchronize(b));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    if (it && ms < best) best = ms;
                }
                const char* nm[] = {"D2H", "H2D", "D2H+H2D"};
                printf("%-8s streams %d chunk %5zu MB  %8.2f ms  %6.1f GB/s per direction\n", nm[dir], ns, chunk >> 20,
                       best, bytes / (best * 1e-3) / 1e9);
            }
        }
    // D2H into registered (not cudaMallocHost) memory, 64 MB chunks over 4 streams
    for (int huge = 0; huge < 2; ++huge) {
        void* hr = nullptr;
        if (posix_memalign(&hr, size_t(2) << 20, bytes)) return 1;
        if (huge) madvise(hr, bytes, MADV_HUGEPAGE);
        memset(hr, 0, bytes);
        CK(cudaHostRegister(hr, bytes, cudaHostRegisterDefault));
        const size_t chunk = size_t(64) << 20;
        float best = 1e9;
        for (int it = 0; it < 4; ++it) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(a, 0));
            int k = 0;
            for (size_t off = 0; off < bytes; off += chunk, ++k) {
                cudaStream_t s = st[k % 4];
                if (k < 4) CK(cudaStreamWaitEvent(s, a, 0));
                CK(cudaMemcpyAsync((char*)hr + off, (char*)d + off, std::min(chunk, bytes - off), cudaMemcpyDeviceToHost, s));
            }
            for (int i = 0; i < 4; ++i) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                CK(cudaEventRecord(e, st[i]));
                CK(cudaStreamWaitEvent(0, e, 0));
            }
            CK(cudaEventRecord(b, 0));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (it && ms < best) best = ms;
        }
        printf("D2H into registered malloc memory (%s) streams 4 chunk 64 MB  %8.2f ms  %6.1f GB/s\n",
               huge ? "MADV_HUGEPAGE" : "4 KB pages", best, bytes / (best * 1e-3) / 1e9);
        CK(cudaHostUnregister(hr));
        free(hr);
    }
    return 0;
}
