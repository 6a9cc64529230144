// GPU weight-spectrum enumeration and low-weight collection (SURVEY.md §8f
// row 1): the reference's `enumerate_spectrum` / `build_sphere`
// (wsphere.py:115-208) -- every one of the 2^K codewords is visited once as
// centre(h) ^ table[e], where table[e] is the XOR of the low LB generator rows
// selected by e (doubling table, wsphere.py:115-121) and centre(h) the XOR of
// the high rows selected by the Gray code of h (wsphere.py:124-144).  Each
// thread owns whole centres; weights are tallied with warp-aggregated shared
// atomics and codewords of weight <= cap appended to a global buffer (the host
// sorts them into CWS1 member order).
#pragma once
#include "common.cuh"

constexpr int ENUM_LB = 10;   // low message bits in the shared table

template <int NW>
__global__ void __launch_bounds__(256) enum_kernel(const uint32_t* __restrict__ gen, int k, int n, int lb,
                                                   const uint32_t* __restrict__ table, long long nhigh,
                                                   int cap, unsigned long long* spectrum, uint32_t* out,
                                                   unsigned long long* out_count, long long out_cap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tsize = 1 << lb;
    uint32_t* st = reinterpret_cast<uint32_t*>(smem_raw);                  // [tsize][NW]
    unsigned int* hist = reinterpret_cast<unsigned int*>(st + (size_t)tsize * NW);  // [n + 1]
    for (int i = threadIdx.x; i < tsize * NW; i += blockDim.x) st[i] = table[i];
    for (int i = threadIdx.x; i <= n; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long h0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long iters = (nhigh + stride - 1) / stride;       // uniform trip count per warp
    for (long long it = 0; it < iters; it++) {
        const long long h = h0 + it * stride;
        const bool valid = h < nhigh;
        uint32_t c[NW];
#pragma unroll
        for (int w = 0; w < NW; w++) c[w] = 0u;
        if (valid) {
            const unsigned long long g = (unsigned long long)h ^ ((unsigned long long)h >> 1);
            for (int b = 0; b < k - lb; b++)
                if ((g >> b) & 1ull) {
#pragma unroll
                    for (int w = 0; w < NW; w++) c[w] ^= gen[(size_t)(lb + b) * NW + w];
                }
        }
        for (int e = 0; e < tsize; e++) {
            uint32_t x[NW];
            int wt = 0;
#pragma unroll
            for (int w = 0; w < NW; w++) { x[w] = c[w] ^ st[e * NW + w]; wt += __popc(x[w]); }
            wt = valid ? wt : -1;
            const unsigned m = __match_any_sync(MPW_FULL, wt);
            if (wt >= 0 && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&hist[wt], (unsigned)__popc(m));
            if (wt > 0 && wt <= cap) {
                const unsigned long long slot = atomicAdd(out_count, 1ull);
                if ((long long)slot < out_cap) {
#pragma unroll
                    for (int w = 0; w < NW; w++) out[slot * NW + w] = x[w];
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= n; i += blockDim.x)
        if (hist[i]) atomicAdd(&spectrum[i], (unsigned long long)hist[i]);
}
