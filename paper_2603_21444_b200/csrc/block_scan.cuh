// Block- and warp-level scan primitives (warp shuffles + one smem exchange).
#pragma once
#include <cstdint>

namespace spgb {

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Exclusive scan of one value per thread across a block of NT threads.
// `ws` is smem scratch of at least NT/32 + 1 elements. Returns the exclusive
// prefix; *total receives the block sum. Contains __syncthreads (all threads
// must call). Safe to call back-to-back.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* total, T* ws) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const T inc = warp_inclusive_scan(v);
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T s = lane < NW ? ws[lane] : T(0);
        s = warp_inclusive_scan(s);
        if (lane < NW) ws[lane] = s;
    }
    __syncthreads();
    const T before = wid > 0 ? ws[wid - 1] : T(0);
    *total = ws[NW - 1];
    __syncthreads();
    return before + inc - v;
}

// In-place exclusive scan of arr[0..n) (any memory space visible to the block),
// writing arr[n] = total. Processes NT*ITEMS elements per chunk with a carry.
template <int NT, int ITEMS, typename T, typename P>
__device__ void block_scan_array(P* arr, int64_t n, T* ws) {
    T carry = 0;
    for (int64_t base = 0; base < n; base += int64_t(NT) * ITEMS) {
        T vals[ITEMS];
        T sum = 0;
        const int64_t my = base + int64_t(threadIdx.x) * ITEMS;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            vals[k] = (my + k < n) ? T(arr[my + k]) : T(0);
            sum += vals[k];
        }
        T total;
        T pre = block_exclusive_scan<NT>(sum, &total, ws);
        pre += carry;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (my + k < n) arr[my + k] = P(pre);
            pre += vals[k];
        }
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) arr[n] = P(carry);
    __syncthreads();
}

}  // namespace spgb
