// Dev tool: pull bandwidth from peer GPUs over NVLink, copy engines vs an
// SM-driven pull kernel (16-byte coalesced loads of the peer's memory).
// usage: peer_bench [MB per peer]   (uses every visible GPU: GPU 0 pulls from
// each of the others at once, like a trident rank pulling its B slices)
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                    \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void pull(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x, st = size_t(gridDim.x) * blockDim.x;
    for (; i + 3 * st < n; i += 4 * st) {
        int4 a = src[i], b = src[i + st], c = src[i + 2 * st], d = src[i + 3 * st];
        dst[i] = a;
        dst[i + st] = b;
        dst[i + 2 * st] = c;
        dst[i + 3 * st] = d;
    }
    for (; i < n; i += st) dst[i] = src[i];
}

// the same pull at narrower widths (a slice's destination offset is only
// 4- or 8-byte aligned in general)
template <typename V, int U>
__global__ void pull_w(const V* __restrict__ src, V* __restrict__ dst, size_t n) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x, st = size_t(gridDim.x) * blockDim.x;
    for (; i + (U - 1) * st < n; i += U * st) {
        V r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = src[i + u * st];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * st] = r[u];
    }
    for (; i < n; i += st) dst[i] = src[i];
}

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atoi(argv[1]) : 200;
    const size_t bytes = mb << 20;
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    printf("GPUs %d, %zu MB per peer\n", ng, mb);
    if (ng < 2) return 0;
    std::vector<void*> src(ng);
    for (int d = 1; d < ng; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&src[d], bytes));
        CK(cudaMemset(src[d], d, bytes));
    }
    CK(cudaSetDevice(0));
    for (int d = 1; d < ng; ++d) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, 0, d));
        if (ok) cudaDeviceEnablePeerAccess(d, 0);
        (void)cudaGetLastError();  // "already enabled" is not an error here
    }
    std::vector<void*> dst(ng);
    std::vector<cudaStream_t> st(ng);
    for (int d = 1; d < ng; ++d) {
        CK(cudaMalloc(&dst[d], bytes));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    }
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int npeer = 1; npeer < ng; ++npeer) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(a, 0));
                for (int d = 1; d <= npeer; ++d) {
                    CK(cudaStreamWaitEvent(st[d], a, 0));
                    if (mode == 0) {
                        CK(cudaMemcpyPeerAsync(dst[d], 0, src[d], d, bytes, st[d]));
                    } else if (mode == 1) {  // two copies per peer (two engines)
                        CK(cudaMemcpyPeerAsync(dst[d], 0, src[d], d, bytes / 2, st[d]));
                        CK(cudaMemcpyPeerAsync((char*)dst[d] + bytes / 2, 0, (char*)src[d] + bytes / 2, d, bytes / 2, 0));
                    } else {
                        pull<<<sms * 4 / npeer, 512, 0, st[d]>>>((const int4*)src[d], (int4*)dst[d], bytes / 16);
                    }
                    CK(cudaGetLastError());
                }
                for (int d = 1; d <= npeer; ++d) {
                    cudaEvent_t ev;
                    CK(cudaEventCreate(&ev));
                    CK(cudaEventRecord(ev, st[d]));
                    CK(cudaStreamWaitEvent(0, ev, 0));
                }
                CK(cudaEventRecord(b, 0));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                if (it && ms < best) best = ms;
            }
            const char* nm[] = {"copy engine", "copy engine x2", "SM pull kernel"};
            printf("peers %d  %-15s  %8.3f ms  %7.1f GB/s into GPU 0\n", npeer, nm[mode], best,
                   npeer * bytes / (best * 1e-3) / 1e9);
        }
    }
    // all-to-all: every GPU pulls bytes from each other GPU at once (the
    // trident exchange at q = 1: every rank pulls its node-mates' slices)
    {
        std::vector<std::vector<void*>> dd(ng, std::vector<void*>(ng, nullptr));
        std::vector<void*> sb(ng);
        std::vector<std::vector<cudaStream_t>> ss(ng, std::vector<cudaStream_t>(ng));
        for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            for (int h = 0; h < ng; ++h)
                if (h != g) {
                    int ok = 0;
                    CK(cudaDeviceCanAccessPeer(&ok, g, h));
                    if (ok) cudaDeviceEnablePeerAccess(h, 0);
        (void)cudaGetLastError();  // "already enabled" is not an error here
                    CK(cudaMalloc(&dd[g][h], bytes));
                    CK(cudaStreamCreateWithFlags(&ss[g][h], cudaStreamNonBlocking));
                }
            CK(cudaMalloc(&sb[g], bytes));
            CK(cudaMemset(sb[g], g, bytes));
        }
        for (int it = 0; it < 4; ++it) {
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaDeviceSynchronize());
            }
            cudaEvent_t e0, e1;
            CK(cudaSetDevice(0));
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            auto t0 = std::chrono::high_resolution_clock::now();
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                for (int h = 0; h < ng; ++h)
                    if (h != g) CK(cudaMemcpyPeerAsync(dd[g][h], g, sb[h], h, bytes, ss[g][h]));
            }
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaDeviceSynchronize());
            }
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::high_resolution_clock::now() - t0).count();
            if (it) printf("all-to-all %d GPUs: %8.3f ms (host clock)  %7.1f GB/s into each GPU\n", ng, ms,
                           (ng - 1) * bytes / (ms * 1e-3) / 1e9);
        }
        // the same all-to-all timed on each GPU with events (max over GPUs),
        // the way the trident exchange is timed: copy engines, one SM pull
        // kernel per peer, or a CE pull with an SM pull side by side
        std::vector<cudaStream_t> gs(ng);
        std::vector<cudaEvent_t> ga(ng), gb(ng);
        std::vector<int> gsm(ng);
        for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaStreamCreateWithFlags(&gs[g], cudaStreamNonBlocking));
            CK(cudaEventCreate(&ga[g]));
            CK(cudaEventCreate(&gb[g]));
            CK(cudaDeviceGetAttribute(&gsm[g], cudaDevAttrMultiProcessorCount, g));
        }
        const char* nm[] = {"copy engines", "SM pull kernels", "SM kernels, 2 per peer", "half CE half SM",
                            "SM pull 8-byte x8", "SM pull 4-byte x8", "SM pull 4-byte x16", "SM 16B x4 256thr"};
        for (int mode = 0; mode < 8; ++mode) {
            float best = 1e9;
            for (int it = 0; it < 6; ++it) {
                for (int g = 0; g < ng; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaDeviceSynchronize());
                }
                for (int g = 0; g < ng; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaEventRecord(ga[g], gs[g]));
                    for (int h = 0; h < ng; ++h) {
                        if (h == g) continue;
                        CK(cudaStreamWaitEvent(ss[g][h], ga[g], 0));
                        const int grid = gsm[g] * 4 / (ng - 1);
                        if (mode == 0) {
                            CK(cudaMemcpyPeerAsync(dd[g][h], g, sb[h], h, bytes, ss[g][h]));
                        } else if (mode == 1) {
                            pull<<<grid, 512, 0, ss[g][h]>>>((const int4*)sb[h], (int4*)dd[g][h], bytes / 16);
                        } else if (mode == 2) {
                            pull<<<grid / 2, 512, 0, ss[g][h]>>>((const int4*)sb[h], (int4*)dd[g][h], bytes / 32);
                            pull<<<grid / 2, 512, 0, ss[g][h]>>>((const int4*)((char*)sb[h] + bytes / 2),
                                                                 (int4*)((char*)dd[g][h] + bytes / 2), bytes / 32);
                        } else if (mode == 4) {
                            pull_w<int2, 8><<<grid, 512, 0, ss[g][h]>>>((const int2*)sb[h], (int2*)dd[g][h], bytes / 8);
                        } else if (mode == 5) {
                            pull_w<int, 8><<<grid, 512, 0, ss[g][h]>>>((const int*)sb[h], (int*)dd[g][h], bytes / 4);
                        } else if (mode == 6) {
                            pull_w<int, 16><<<grid, 512, 0, ss[g][h]>>>((const int*)sb[h], (int*)dd[g][h], bytes / 4);
                        } else if (mode == 7) {
                            pull_w<int4, 4><<<grid * 2, 256, 0, ss[g][h]>>>((const int4*)sb[h], (int4*)dd[g][h], bytes / 16);
                        } else {
                            CK(cudaMemcpyPeerAsync(dd[g][h], g, sb[h], h, bytes / 2, ss[g][h]));
                            pull<<<grid / 2, 512, 0, gs[g]>>>((const int4*)((char*)sb[h] + bytes / 2),
                                                             (int4*)((char*)dd[g][h] + bytes / 2), bytes / 32);
                        }
                        CK(cudaGetLastError());
                    }
                    for (int h = 0; h < ng; ++h) {
                        if (h == g) continue;
                        cudaEvent_t ev;
                        CK(cudaEventCreate(&ev));
                        CK(cudaEventRecord(ev, ss[g][h]));
                        CK(cudaStreamWaitEvent(gs[g], ev, 0));
                    }
                    CK(cudaEventRecord(gb[g], gs[g]));
                }
                float mx = 0;
                for (int g = 0; g < ng; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaEventSynchronize(gb[g]));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, ga[g], gb[g]));
                    if (ms > mx) mx = ms;
                }
                if (it && mx < best) best = mx;
            }
            printf("all-to-all %d GPUs, %-22s %8.3f ms (events, max over GPUs)  %7.1f GB/s into each GPU\n", ng,
                   nm[mode], best, (ng - 1) * bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
