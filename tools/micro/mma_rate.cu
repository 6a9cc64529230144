// Micro-benchmark: tcgen05.mma issue-to-completion rate per SM on B200 for the
// hop kernel's shapes (operand data is garbage; only timing matters).
//   kind::i8  M=128 N=256|224|128 K=32, A from shared memory or from TMEM
//   kind::f16 M=128 N=256 K=16, A from shared memory
// One CTA per SM, one thread issues ITERS instructions, then one commit to an
// mbarrier and waits for it; reports cycles per instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// SYNC: per 4 instructions (one K-block) the hop kernel's bookkeeping -- an
// mbarrier try_wait (on a completed phase), tcgen05.fence::after_thread_sync,
// and a tcgen05.commit to a stage barrier
template <int KIND, int N, bool ATMEM, int RING = 1, int SYNC = 0, int GRP = 4, int NW_ = 1, int NC_ = 1>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t done_bar, sink_bar;
    unsigned char* a = sm;            // 2 x 16 KB (two K-blocks)
    unsigned char* b = sm + 32768;    // RING x 32 KB
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (32768 + RING * 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&sink_bar)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t d = slot, at = slot + 448;
        const uint32_t idesc = (KIND == 0 ? (2u << 4) | (1u << 7) : (1u << 4)) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        const uint64_t ad = sw128_desc(smem_u32(a)), bd = sw128_desc(smem_u32(b));
        uint32_t phase = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            const int ks = it & 3;
            if ((SYNC & 8) && ks == 0) {   // plain shared-memory flag poll instead of an mbarrier
                volatile uint32_t* fl = reinterpret_cast<volatile uint32_t*>(&slot);
                while (*fl == 0xFFFFFFFFu) {}
            }
            if ((SYNC & 16) && ks == 0) {  // mbarrier.test_wait
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&done_bar)), "r"(0) : "memory");
            }
            if ((SYNC & 32) && (it % GRP) == 0) {   // NW_ try_waits + fence per group
                for (int w = 0; w < NW_; w++) {
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&done_bar)), "r"(0) : "memory");
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            if ((SYNC & 1) && ks == 0) {
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&done_bar)), "r"(0) : "memory");
            }
            if ((SYNC & 2) && ks == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int kb = (it >> 2) & 1;                 // A K-block
            const int stg = (it >> 2) % RING;             // B ring stage
            const uint64_t adk = ad + (uint64_t)(kb * 16384 >> 4), bdk = bd + (uint64_t)(stg * 32768 >> 4);
            if (KIND == 0) {
                if (ATMEM)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(at + kb * 32 + ks * 8), "l"(bdk + 2 * ks), "r"(idesc), "r"(it));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(d), "l"(adk + 2 * ks), "l"(bdk + 2 * ks), "r"(idesc), "r"(it));
            } else {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(adk + 2 * ks), "l"(bdk + 2 * ks), "r"(idesc), "r"(it));
            }
            if ((SYNC & 32) && (it % GRP) == GRP - 1)
                for (int c = 0; c < NC_; c++)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 ::"r"(smem_u32(&sink_bar)) : "memory");
            if ((SYNC & 4) && ks == 3)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&sink_bar)) : "memory");
        }
        // one commit after the last instruction tracks the completion of all of them
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)) : "memory");
        {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
        }
        long long t1 = clock64();
        out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int KIND, int N, bool ATMEM, int RING = 1, int SYNC = 0, int GRP = 4, int NW_ = 1, int NC_ = 1>
void run(const char* name, unsigned long long* d) {
    auto k = mma_rate<KIND, N, ATMEM, RING, SYNC, GRP, NW_, NC_>;
    const int smem = 32768 + RING * 32768 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 8 * 4096;
    k<<<148, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: error %s\n", name, cudaGetErrorString(e)); return; }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; i++) s += h[i];
    const double cyc = s / 148 / iters;
    const double ideal = (KIND == 0 ? 128.0 : 128.0) * N / 256.0;
    printf("%-28s %.1f cycles/instr (ideal %.0f, %.0f%%)\n", name, cyc, ideal, 100.0 * ideal / cyc);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<0, 256, false>("i8 N256 A smem", d);
    run<0, 256, true>("i8 N256 A tmem", d);
    run<0, 224, true>("i8 N224 A tmem", d);
    run<0, 224, false>("i8 N224 A smem", d);
    run<0, 128, false>("i8 N128 A smem", d);
    run<0, 128, true>("i8 N128 A tmem", d);
    run<1, 256, false>("f16 N256 A smem", d);
    run<0, 256, false, 6>("i8 N256 A smem ring6", d);
    run<0, 256, true, 6>("i8 N256 A tmem ring6", d);
    run<1, 256, false, 5>("f16 N256 A smem ring5", d);
    run<0, 256, false, 6, 32, 8, 3, 3>("i8 N256 per 8: 3 waits 3 commits", d);
    run<0, 256, false, 6, 32, 8, 1, 1>("i8 N256 per 8: 1 wait 1 commit", d);
    run<0, 256, false, 6, 32, 8, 1, 2>("i8 N256 per 8: 1 wait 2 commits", d);
    run<0, 256, false, 6, 32, 16, 1, 1>("i8 N256 per 16: 1 wait 1 commit", d);
    run<0, 160, false, 6, 32, 8, 1, 1>("i8 N160 per 8: 1 wait 1 commit", d);
    run<0, 256, false, 6, 7>("i8 N256 wait+fence+commit", d);
    run<0, 256, false, 6, 1>("i8 N256 try_wait", d);
    run<0, 256, false, 6, 16>("i8 N256 test_wait", d);
    run<0, 256, false, 6, 8>("i8 N256 lds poll", d);
    run<0, 256, true, 6, 1>("i8 N256 Atmem try_wait", d);
    run<0, 256, false, 6, 12>("i8 N256 lds poll+commit", d);
    return 0;
}
