// tcgen05.mma kind::i8 M128 N256 K32 issue patterns (cycles per instruction, all SMs at once):
//   0  one accumulator, always accumulating (the peaks.cu measurement)
//   1  tiles of 8 MMAs, alternating two accumulators, first MMA of a tile overwrites
//   2  as 1, plus a tcgen05.commit to an mbarrier after every 4 MMAs and every tile
//   3  as 2, B operand cycling over five 32 KB stages, A over two 16 KB K-blocks
//   4  as 3, plus 8 warps reading the finished accumulator (tcgen05.ld x32 pack16, 128 columns per warp)
//   5  as 4, plus a producer thread re-arming each freed stage (empty -> full ping-pong, no copy) and the
//      issuer waiting for the stage
//   6  as 5, the readers also run ~150 ALU instructions, 3 volatile shared loads and 4 predicated shared
//      stores per tile (the scan loop's work)
//   7  as 6, the producer streams 32 KB stages of a 16 MB L2-resident buffer (cp.async.bulk)
//   8  as 7, but one barrier per accumulator collects the readers' releases and the tile's two stage
//      arrivals, so the issuer waits once per tile
//   9  as 7, with a second issuer thread (alternate tiles, own accumulator)
// Build and run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_tiles tools/micro/mma_tiles.cu && /tmp/mma_tiles
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(352, 1) k(int tiles, unsigned long long* out, const unsigned char* __restrict__ src) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar_e[5], bar_t[2], bar_r[2], bar_f[5];
    __shared__ uint32_t scratch[1024];
    unsigned char* a = sm;            // 2 x 16 KB
    unsigned char* b = sm + 32768;    // 5 x 32 KB
    for (int i = threadIdx.x; i < (32768 + 5 * 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 5; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_e[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_f[s])));
        }
        for (int s = 0; s < 2; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_t[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar_r[s])), "r"(MODE == 8 ? 9 : 8));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    if (threadIdx.x == 0 || (MODE == 9 && threadIdx.x == 32)) {
        const int first = threadIdx.x == 0 ? 0 : 1, step = MODE == 9 ? 2 : 1;
        const uint32_t idesc = (2u << 4) | (1u << 7) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const long long c0 = clock64();
        for (int t = first; t < tiles; t += step) {
            uint32_t u = 2 * t;
            const uint32_t buf = MODE >= 1 ? (t & 1) : 0;
            const uint32_t d = tm + buf * 256;
            if (MODE == 8) { wait(smem_u32(&bar_r[buf]), (t >> 1) & 1); asm volatile("tcgen05.fence::after_thread_sync;"); }
            else if (MODE >= 4 && t >= 2) { wait(smem_u32(&bar_r[buf]), ((t >> 1) & 1) ^ 1); asm volatile("tcgen05.fence::after_thread_sync;"); }
            for (int kb = 0; kb < 2; kb++, u++) {
                const uint32_t st = MODE >= 3 ? u % 5 : 0;
                if (MODE >= 5 && MODE != 8) { wait(smem_u32(&bar_f[st]), (u / 5) & 1); asm volatile("tcgen05.fence::after_thread_sync;"); }
                const uint64_t ad = sw128_desc(smem_u32(a) + (MODE >= 3 ? kb * 16384 : 0));
                const uint64_t bd = sw128_desc(smem_u32(b) + st * 32768);
#pragma unroll
                for (int ks = 0; ks < 4; ks++) mma_i8(d, ad + 2 * ks, bd + 2 * ks, idesc, MODE == 0 ? (uint32_t)(t | kb | ks) : (uint32_t)(kb | ks));
                if (MODE >= 2) commit(smem_u32(&bar_e[st]));
            }
            if (MODE >= 2) commit(smem_u32(&bar_t[buf]));
        }
        if (MODE < 2) commit(smem_u32(&bar_t[0]));
        // drain: the last tile's commit
        if (threadIdx.x == 0) {
            if (MODE >= 2) wait(smem_u32(&bar_t[(tiles - 1) & 1]), ((tiles - 1) >> 1) & 1);
            else wait(smem_u32(&bar_t[0]), 0);
            out[blockIdx.x] = (unsigned long long)(clock64() - c0);
        }
    } else if (MODE >= 5 && threadIdx.x == 320) {
        // producer: re-arm a stage as soon as the MMAs that read it completed
        for (uint32_t u = 0; u < (uint32_t)tiles * 2; u++) {
            const uint32_t st = u % 5;
            if (u >= 5) wait(smem_u32(&bar_e[st]), ((u / 5) & 1) ^ 1);
            const uint32_t fb = MODE == 8 ? smem_u32(&bar_r[(u >> 1) & 1]) : smem_u32(&bar_f[st]);
            if (MODE == 8) {
                // the accumulator barrier's previous phase must be complete before this tile's arrival joins the next
                if (!(u & 1) && u >= 4) wait(fb, (((u >> 1) >> 1) & 1) ^ 1);
                if (!(u & 1)) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(65536) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(b + st * 32768)), "l"(src + (size_t)((u * 7 + blockIdx.x * 13) % 512) * 32768), "r"(32768), "r"(fb) : "memory");
            } else if (MODE >= 7) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(32768) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(b + st * 32768)), "l"(src + (size_t)((u * 7 + blockIdx.x * 13) % 512) * 32768), "r"(32768), "r"(fb) : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
            }
        }
    } else if (MODE >= 4 && warp >= 2 && warp < 10) {
        // eight readers: two per lane quarter, 128 columns each, then release the accumulator
        const int g = warp & 3, half = (warp - 2) >> 2;
        uint32_t sink = 0;
        if (MODE == 8 && lane == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_r[0])) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_r[1])) : "memory");
        }
        for (int t = 0; t < tiles; t++) {
            const uint32_t buf = t & 1;
            wait(smem_u32(&bar_t[buf]), (t >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v[32], w[32];
            const uint32_t ta = tm + ((uint32_t)(g * 32) << 16) + buf * 256 + half * 128;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(ta));
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31]) : "r"(ta + 64));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_r[buf])) : "memory");
#pragma unroll
            for (int e = 0; e < 32; e++) sink ^= v[e] ^ w[e];
            if (MODE >= 6) {
                // the scan loop's per-tile work: min trees, control reads, predicated records
                volatile uint32_t* sc = scratch;
                uint32_t c0 = sc[threadIdx.x & 127], c1 = sc[128 + (threadIdx.x & 127)], c2 = sc[300];
                uint32_t m = 0xFFFFFFFFu;
#pragma unroll
                for (int e = 0; e < 32; e++) { m = min(m, v[e] + c0); m = min(m, w[e] ^ c1); m = min(m, (v[e] >> 3) + (w[e] << 2)); }
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (((m >> q) & 0xFFu) == 0x5Au + c2) sc[512 + ((threadIdx.x + q * 64) & 511)] = m;
                sink ^= m;
            }
        }
        if (sink == 0x12345678u) out[blockIdx.x] = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE>
static void run(int sms, int tiles, unsigned long long* d, const unsigned char* src) {
    const int smem = 32768 + 5 * 32768;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE><<<sms, 352, smem>>>(tiles, d, src);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double s = 0;
    for (auto x : h) s += (double)x;
    printf("  \"mode%d\": {\"cycles_per_mma\": %.1f, \"cycles_per_tile\": %.0f, \"error\": \"%s\"},\n", MODE,
           s / sms / tiles / 8.0, s / sms / tiles, cudaGetErrorString(e));
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount, tiles = 20000;
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    printf("{\n  \"device\": \"%s\", \"tiles\": %d, \"shape\": \"kind::i8 M128 N256 K32, 8 per tile\",\n", prop.name, tiles);
    unsigned char* src;
    cudaMalloc(&src, 16 << 20);
    cudaMemset(src, 1, 16 << 20);
    run<0>(sms, tiles, d, src);
    run<1>(sms, tiles, d, src);
    run<2>(sms, tiles, d, src);
    run<3>(sms, tiles, d, src);
    run<4>(sms, tiles, d, src);
    run<5>(sms, tiles, d, src);
    run<6>(sms, tiles, d, src);
    run<7>(sms, tiles, d, src);
    run<8>(sms, tiles, d, src);
    run<9>(sms, tiles, d, src);
    printf("  \"end\": 0\n}\n");
    return 0;
}
