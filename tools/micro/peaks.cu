// Measured denominators for the roofline: per-SM rates of
// the pipes the hop formulations are bound by, on all SMs at once, with the
// SM clock measured over the same interval (clock64 cycles / globaltimer ns).
//
//   tcgen05.mma kind::i8  M=128 N=256 K=32 (A, B in SW128 shared memory)
//   tcgen05.mma kind::f16 M=128 N=256 K=16
//   shared-memory loads   LDS.128, conflict-free, 1024 threads per SM
//   FP32 adds             FADD, 8 independent chains per thread, 1024 threads
//   L2 -> SM stream       cp.async.bulk of 32 KB stages of one 16 MB L2-resident
//                         buffer (the hop's P images) into a 6-stage ring on every
//                         SM: unicast with all SMs in step / staggered, and
//                         multicast to clusters of 2 and 4
//
// Build and run (one GPU):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//     -o peaks tools/micro/peaks.cu && ./peaks > profiles/r02_micro_peaks.json
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

struct Rec {
    unsigned long long cycles, ns, t_start, t_end;
    float sink;
};

// ---------------------------------------------------------------------------
// tensor core issue rate: one thread issues `iters` MMAs into one TMEM
// accumulator (operand contents are irrelevant to the rate)
template <int KIND, int M = 128, int N = 256>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, Rec* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    unsigned char* a = sm;            // 16 KB
    unsigned char* b = sm + 16384;    // 32 KB
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t d = slot;
        const uint32_t idesc = (KIND == 0 ? (2u << 4) | (1u << 7) : (1u << 4)) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = sw128_desc(smem_u32(a)), bd = sw128_desc(smem_u32(b));
        const uint64_t g0 = gtimer();
        const long long c0 = clock64();
        for (int it = 0; it < iters; it++) {
            const int ks = it & 3;
            if (KIND == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(ad + 2 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"(it));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(ad + 2 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"(it));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        const long long c1 = clock64();
        const uint64_t g1 = gtimer();
        out[blockIdx.x] = Rec{(unsigned long long)(c1 - c0), g1 - g0, g0, g1, 0.f};
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
}

// ---------------------------------------------------------------------------
// shared-memory load bandwidth: LDS.128, every warp reads 512 contiguous bytes
// per instruction (conflict-free), 4 independent loads in flight per thread
__global__ void __launch_bounds__(1024, 1) smem_kernel(int iters, Rec* out) {
    __shared__ __align__(16) float4 buf[2048];   // 32 KB
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const uint64_t g0 = gtimer();
    const long long c0 = clock64();
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int idx = threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; it++) {
        const float4 v0 = buf[idx & 2047];
        const float4 v1 = buf[(idx + 1024) & 2047];
        const float4 v2 = buf[(idx + 512) & 2047];
        const float4 v3 = buf[(idx + 1536) & 2047];
        acc0 ^= __float_as_uint(v0.x) ^ __float_as_uint(v0.y) ^ __float_as_uint(v0.z) ^ __float_as_uint(v0.w);
        acc1 ^= __float_as_uint(v1.x) ^ __float_as_uint(v1.y) ^ __float_as_uint(v1.z) ^ __float_as_uint(v1.w);
        acc2 ^= __float_as_uint(v2.x) ^ __float_as_uint(v2.y) ^ __float_as_uint(v2.z) ^ __float_as_uint(v2.w);
        acc3 ^= __float_as_uint(v3.x) ^ __float_as_uint(v3.y) ^ __float_as_uint(v3.z) ^ __float_as_uint(v3.w);
        idx += 32;
    }
    __syncthreads();
    const long long c1 = clock64();
    const uint64_t g1 = gtimer();
    if (threadIdx.x == 0) out[blockIdx.x] = Rec{(unsigned long long)(c1 - c0), g1 - g0, g0, g1, 0.f};
    if ((acc0 ^ acc1 ^ acc2 ^ acc3) == 0x12345678u) out[blockIdx.x].sink = 1.f;
}

// ---------------------------------------------------------------------------
// FP32 add rate: 8 independent FADD chains per thread
__global__ void __launch_bounds__(1024, 1) fadd_kernel(int iters, float seed, Rec* out) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = seed * (threadIdx.x + k);
    const float inc = seed * 1e-7f;
    __syncthreads();
    const uint64_t g0 = gtimer();
    const long long c0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 16; r++) {
#pragma unroll
            for (int k = 0; k < 8; k++) a[k] = __fadd_rn(a[k], inc);
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    const uint64_t g1 = gtimer();
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (threadIdx.x == 0) out[blockIdx.x] = Rec{(unsigned long long)(c1 - c0), g1 - g0, g0, g1, s};
}

// ---------------------------------------------------------------------------
// L2 -> shared memory stream of the hop's P operand
constexpr int L2_STAGES = 6, L2_STAGE = 32768;

__device__ __forceinline__ uint32_t cluster_rank_u32() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}

template <int CL>
__global__ void __launch_bounds__(32, 1) l2_kernel(const unsigned char* __restrict__ src, int nchunks, int iters,
                                                   int stagger, Rec* out) {
    extern __shared__ __align__(1024) unsigned char ring[];
    __shared__ __align__(8) uint64_t full[L2_STAGES], empty[L2_STAGES];
    const uint32_t crank = CL > 1 ? cluster_rank_u32() : 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < L2_STAGES; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CL));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (CL > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        const int cid = blockIdx.x / CL;
        const int start = stagger ? (cid * 7919) % nchunks : 0;
        const uint64_t g0 = gtimer();
        const long long c0 = clock64();
        // L2_STAGES - 1 copies in flight: issue copy i, then consume copy i - (L2_STAGES - 1)
        for (int i = 0; i < iters + L2_STAGES - 1; i++) {
            if (i < iters) {
                const int s = i % L2_STAGES;
                const uint32_t ph = (uint32_t)(i / L2_STAGES) & 1u;
                if (i >= L2_STAGES) while (!try_wait(smem_u32(&empty[s]), ph ^ 1u)) {}
                const uint32_t fb = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(L2_STAGE) : "memory");
                const unsigned char* g = src + (size_t)((start + i) % nchunks) * L2_STAGE;
                if (CL == 1) {
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(ring + s * L2_STAGE)), "l"(g), "r"(L2_STAGE), "r"(fb) : "memory");
                } else {
                    constexpr uint32_t PART = L2_STAGE / CL;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
                                 "[%0], [%1], %2, [%3], %4;"
                                 ::"r"(smem_u32(ring + s * L2_STAGE) + crank * PART), "l"(g + crank * PART), "r"(PART),
                                 "r"(fb), "h"((uint16_t)((1u << CL) - 1u)) : "memory");
                }
            }
            const int j = i - (L2_STAGES - 1);
            if (j >= 0) {
                // consume copy j: wait until its stage landed, then release it in every CTA of the cluster
                const int s = j % L2_STAGES;
                const uint32_t ph = (uint32_t)(j / L2_STAGES) & 1u;
                while (!try_wait(smem_u32(&full[s]), ph)) {}
                if (CL == 1) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
                } else {
                    for (int r = 0; r < CL; r++) {
                        uint32_t remote;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(r));
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                    }
                }
            }
        }
        const long long c1 = clock64();
        const uint64_t g1 = gtimer();
        out[blockIdx.x] = Rec{(unsigned long long)(c1 - c0), g1 - g0, g0, g1, 0.f};
    }
    __syncwarp();
    if (CL > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CL>
static void launch_l2(const unsigned char* src, int nchunks, int iters, int stagger, Rec* d, int sms) {
    const int smem = L2_STAGES * L2_STAGE;
    cudaFuncSetAttribute(l2_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sms / CL) * CL));
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, l2_kernel<CL>, src, nchunks, iters, stagger, d);
}

struct Result {
    double per_clk_per_sm;   // units per SM clock per SM
    double sm_mhz;           // measured over the interval
    double aggregate;        // units per second, all SMs (first start to last end)
};

static Result summarise(const std::vector<Rec>& r, double units_per_cta) {
    double cyc = 0, ns = 0;
    unsigned long long t0 = ~0ull, t1 = 0;
    for (const Rec& x : r) {
        cyc += x.cycles;
        ns += x.ns;
        t0 = x.t_start < t0 ? x.t_start : t0;
        t1 = x.t_end > t1 ? x.t_end : t1;
    }
    Result o;
    o.per_clk_per_sm = units_per_cta * r.size() / cyc;
    o.sm_mhz = cyc / ns * 1e3;
    o.aggregate = units_per_cta * r.size() / ((double)(t1 - t0) * 1e-9);
    return o;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    Rec* d;
    cudaMalloc(&d, sizeof(Rec) * sms);
    std::vector<Rec> h(sms);
    auto fetch = [&]() {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            fprintf(stderr, "error: %s\n", cudaGetErrorString(e));
            exit(1);
        }
        cudaMemcpy(h.data(), d, sizeof(Rec) * sms, cudaMemcpyDeviceToHost);
    };
    const int smem_mma = 49152 + 1024;
    cudaFuncSetAttribute(mma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mma);
    cudaFuncSetAttribute(mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mma);

    // warm-up (clocks ramp), then the measured runs of ~0.5-1 s each
    mma_kernel<0><<<sms, 128, smem_mma>>>(1 << 20, d);
    fetch();
    const int mma_iters = 1 << 23;
    mma_kernel<0><<<sms, 128, smem_mma>>>(mma_iters, d);
    fetch();
    Result i8 = summarise(h, 2.0 * 128 * 256 * 32 * (double)mma_iters);
    mma_kernel<1><<<sms, 128, smem_mma>>>(mma_iters, d);
    fetch();
    Result f16 = summarise(h, 2.0 * 128 * 256 * 16 * (double)mma_iters);
    // smaller int8 shapes: per-instruction cost of M = 64 and of N = 128 / 192
    cudaFuncSetAttribute(mma_kernel<0, 64, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mma);
    cudaFuncSetAttribute(mma_kernel<0, 128, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mma);
    cudaFuncSetAttribute(mma_kernel<0, 128, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mma);
    const int small_iters = 1 << 20;
    mma_kernel<0, 64, 256><<<sms, 128, smem_mma>>>(small_iters, d);
    fetch();
    Result i8m64 = summarise(h, 2.0 * 64 * 256 * 32 * (double)small_iters);
    mma_kernel<0, 128, 128><<<sms, 128, smem_mma>>>(small_iters, d);
    fetch();
    Result i8n128 = summarise(h, 2.0 * 128 * 128 * 32 * (double)small_iters);
    mma_kernel<0, 128, 192><<<sms, 128, smem_mma>>>(small_iters, d);
    fetch();
    Result i8n192 = summarise(h, 2.0 * 128 * 192 * 32 * (double)small_iters);
    const int lds_iters = 1 << 20;
    smem_kernel<<<sms, 1024>>>(lds_iters, d);
    fetch();
    Result lds = summarise(h, 1024.0 * 4 * 16 * (double)lds_iters);
    const int fadd_iters = 1 << 17;
    fadd_kernel<<<sms, 1024>>>(fadd_iters, 1.0f, d);
    fetch();
    Result fadd = summarise(h, 1024.0 * 16 * 8 * (double)fadd_iters);

    // L2 -> SM stream: 16 MB buffer (the int8 P images of cfg4), 32 KB stages
    const int nchunks = 512;
    unsigned char* src;
    cudaMalloc(&src, (size_t)nchunks * L2_STAGE);
    cudaMemset(src, 1, (size_t)nchunks * L2_STAGE);
    const int l2_iters = 1 << 14;
    double l2r[4][2];   // [variant] {bytes/clk/SM delivered, chip B/clk fetched from L2}
    int l2_ctas[4];
    for (int v = 0; v < 4; v++) {
        const int cl = v < 2 ? 1 : (v == 2 ? 2 : 4);
        if (cl == 1) launch_l2<1>(src, nchunks, l2_iters, v == 1, d, sms);
        else if (cl == 2) launch_l2<2>(src, nchunks, l2_iters, 1, d, sms);
        else launch_l2<4>(src, nchunks, l2_iters, 1, d, sms);
        fetch();
        l2_ctas[v] = (sms / cl) * cl;
        std::vector<Rec> hv(h.begin(), h.begin() + l2_ctas[v]);
        Result r = summarise(hv, (double)L2_STAGE * l2_iters);
        l2r[v][0] = r.per_clk_per_sm;
        l2r[v][1] = r.per_clk_per_sm * l2_ctas[v] / cl;   // every byte leaves L2 once per cluster
    }

    printf("{\n  \"device\": \"%s\", \"sms\": %d,\n", prop.name, sms);
    printf("  \"method\": \"all SMs at once, one CTA per SM; per-clock rates = units / clock64 cycles summed over "
           "CTAs; sm_mhz = cycles / globaltimer ns over the same interval; aggregate = units / (last end - first "
           "start)\",\n");
    printf("  \"tc_i8\": {\"shape\": \"tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32\", \"ops_per_clk_per_sm\": "
           "%.1f, \"nominal_ops_per_clk_per_sm\": 16384, \"sm_mhz\": %.0f, \"aggregate_tops\": %.1f},\n",
           i8.per_clk_per_sm, i8.sm_mhz, i8.aggregate * 1e-12);
    printf("  \"tc_f16\": {\"shape\": \"tcgen05.mma.cta_group::1.kind::f16 M128 N256 K16\", \"flop_per_clk_per_sm\": "
           "%.1f, \"nominal_flop_per_clk_per_sm\": 8192, \"sm_mhz\": %.0f, \"aggregate_tflops\": %.1f},\n",
           f16.per_clk_per_sm, f16.sm_mhz, f16.aggregate * 1e-12);
    printf("  \"tc_i8_shapes\": {\"M64_N256_ops_per_clk_per_sm\": %.1f, \"M128_N128_ops_per_clk_per_sm\": %.1f, "
           "\"M128_N192_ops_per_clk_per_sm\": %.1f},\n", i8m64.per_clk_per_sm, i8n128.per_clk_per_sm,
           i8n192.per_clk_per_sm);
    printf("  \"smem_lds128\": {\"bytes_per_clk_per_sm\": %.1f, \"nominal_bytes_per_clk_per_sm\": 128, \"sm_mhz\": "
           "%.0f, \"aggregate_gbs\": %.0f},\n",
           lds.per_clk_per_sm, lds.sm_mhz, lds.aggregate * 1e-9);
    printf("  \"fp32_fadd\": {\"adds_per_clk_per_sm\": %.1f, \"nominal_adds_per_clk_per_sm\": 128, \"sm_mhz\": %.0f, "
           "\"aggregate_gadds\": %.0f},\n",
           fadd.per_clk_per_sm, fadd.sm_mhz, fadd.aggregate * 1e-9);
    const char* l2names[4] = {"unicast_in_step", "unicast_staggered", "multicast_cluster2", "multicast_cluster4"};
    printf("  \"l2_to_smem_stream\": {\"buffer_mb\": 16, \"stage_bytes\": %d, \"stages\": %d,\n", L2_STAGE, L2_STAGES);
    for (int v = 0; v < 4; v++)
        printf("    \"%s\": {\"ctas\": %d, \"delivered_bytes_per_clk_per_sm\": %.1f, \"l2_read_bytes_per_clk_chip\": "
               "%.0f}%s\n", l2names[v], l2_ctas[v], l2r[v][0], l2r[v][1], v < 3 ? "," : "");
    printf("  }\n}\n");
    return 0;
}
