// Tensor-core hop: host side (operand images, launch).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hop_tc.cuh"
#include "hop_tc_api.h"

// ---------------------------------------------------------------------------
// host side

// Launch options (TcOpts, set per handle through mpw_set_option): the
// defaults are the production choices; the others are kept for A/B runs and
// the parity tests.  The per-tile clock trace (experiment bit 128) exists
// only in builds with -DMPW_PROFILE.

// fp32 certification pass bound: any summation order of at most wmax terms
// has |fl(S) - S| <= gamma_{wmax-1} sum|t_i| (gamma_k = k u / (1 - k u),
// u = 2^-24); with float64 inputs the fp32 rounding of y adds u sum|y|.
// Rounded up by 0.2 % (the float conversion and the product with sum|y|).
static float cert_gamma(int wmax, bool y64) {
    const double u = 5.9604644775390625e-8;
    const double k = wmax > 1 ? wmax - 1 : 0;
    double g = k * u / (1.0 - k * u);
    if (y64) g += u;
    return (float)(g * 1.002);
}

bool tc_supported(int n, int np) { return (n == 64 || n == 128 || n == 256) && np >= 1; }
bool tc_i8_supported(int n, int np) { return (n == 128 || n == 256) && np >= 1; }

void tc_release(TcPatterns& t) {
    if (t.tiles) cudaFree(t.tiles);
    if (t.tiles8) cudaFree(t.tiles8);
    if (t.ar_stat) cudaFree(t.ar_stat);
    t.ar_stat = nullptr;
    t.tiles = nullptr;
    t.tiles8 = nullptr;
    t.ready = false;
    t.ready8 = false;
}

// u8 0/1 images for the int8 screen: one 32 KB stage = 256 patterns x 128 positions
static int tc_build8(TcPatterns& t, const uint32_t* bits, int np, int n, int nw) {
    // packed (score, index) keys need |P| <= 2^17 and 127 * wmax < 8192
    int wmax = 0;
    for (int p = 0; p < np; p++) {
        int w = 0;
        for (int k = 0; k < nw; k++) w += __builtin_popcount(bits[(size_t)p * nw + k]);
        wmax = w > wmax ? w : wmax;
    }
    if (np > (1 << tc::KEY_IBITS) || 127 * wmax >= tc::KEY_BIAS) return 0;   // int8 screen unavailable
    const int kb = n / 128;
    const int ntiles = (np + tc::I8_TILE - 1) / tc::I8_TILE;
    const size_t bytes = (size_t)ntiles * kb * tc::I8_STAGE_BYTES;
    std::vector<uint8_t> img(bytes, 0);
    // the columns of the last tile past |P| repeat pattern 0: their scores are those of a real
    // pattern, so they never change a minimum and the asynchronous-row scan needs no tail mask
    // (its workers ignore pattern indices >= |P|; the synchronous screen masks the tail itself)
    for (int pp = 0; pp < ntiles * tc::I8_TILE; pp++) {
        const int p = pp < np ? pp : 0;
        const int j = pp / tc::I8_TILE, r = pp % tc::I8_TILE;
        for (int i = 0; i < n; i++) {
            if (!((bits[(size_t)p * nw + (i >> 5)] >> (i & 31)) & 1u)) continue;
            const int k = i / 128, col = i % 128;
            img[((size_t)j * kb + k) * tc::I8_STAGE_BYTES + tc::sw128_chunk(r, col >> 4) + (col & 15)] = 1;
        }
    }
    if (cudaMalloc(&t.tiles8, bytes) != cudaSuccess) return -1;
    if (cudaMemcpy(t.tiles8, img.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
    t.kb8 = kb;
    t.ntiles8 = ntiles;
    t.ready8 = true;
    if (cudaMalloc(&t.ar_stat, 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (cudaMemset(t.ar_stat, 0, 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    return 0;
}

int tc_build(TcPatterns& t, const uint32_t* bits, int np, int n, int nw) {
    tc_release(t);
    const int kb = n / tc::KBLK;
    const int ntiles = (np + tc::NT_COLS - 1) / tc::NT_COLS;
    const size_t bytes = (size_t)ntiles * kb * tc::B_STAGE_BYTES;
    std::vector<uint16_t> img(bytes / 2, 0);
    for (int p = 0; p < np; p++) {
        const int j = p / tc::NT_COLS, r = p % tc::NT_COLS;
        for (int i = 0; i < n; i++) {
            if (!((bits[(size_t)p * nw + (i >> 5)] >> (i & 31)) & 1u)) continue;
            const int k = i / tc::KBLK, col = i % tc::KBLK;
            const size_t off = ((size_t)j * kb + k) * tc::B_STAGE_BYTES + tc::sw128_off(r, col);
            img[off / 2] = 0x3C00;   // fp16 1.0
        }
    }
    if (cudaMalloc(&t.tiles, bytes) != cudaSuccess) return -1;
    if (cudaMemcpy(t.tiles, img.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
    t.np = np; t.ntiles = ntiles; t.kb = kb; t.ready = true;
    if (tc_i8_supported(n, np) && tc_build8(t, bits, np, n, nw)) return -1;
    return 0;
}

template <int KB, int NW, int LIMBS, int MODE, int CL = 1, int PM = 0>
static int tc_launch_t(const TcPatterns& t, int n, int nw, int A, int T, const float* y, const double* y64,
                       S2Dev s2, PatDev P, int num_sms, const TcOpts& o, cudaStream_t st) {
    tc::Params prm;
    prm.n = n; prm.nw = nw; prm.A = A; prm.T = T; prm.np = t.np; prm.ntiles = LIMBS == 0 ? t.ntiles8 : t.ntiles;
    prm.y = y; prm.y64 = MODE == 3 ? y64 : nullptr;
    prm.s2 = s2; prm.pbits = P.bits; prm.btiles = LIMBS == 0 ? t.tiles8 : t.tiles; prm.tie_rel = 1e-5f;
    prm.cert_g = cert_gamma(s2.wmax, MODE == 3);
    prm.experiment = (MODE == 1 || MODE == 2) ? o.experiment : 0;
    prm.trace = nullptr;
#ifdef MPW_PROFILE
    static long long* trace = nullptr;
    if (prm.experiment & 128) {
        const size_t tb = sizeof(long long) * tc::TRACE_W * tc::TRACE_TILES;
        if (!trace && cudaMallocManaged(&trace, tb) != cudaSuccess) trace = nullptr;
        if (trace) memset(trace, 0, tb);
        prm.trace = trace;
    }
#endif
    const size_t smem = tc::smem_bytes(KB, LIMBS, CL, PM);
    auto kern = tc::hop_tc_kernel<KB, NW, LIMBS, MODE, CL, PM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -(int)e;
    if (CL == 1) {
        kern<<<num_sms, tc::threads_for(LIMBS), smem, st>>>(prm);
    } else {
        // one CTA pair per two SMs (as many pairs as can be co-resident)
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(tc::threads_for(LIMBS));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3((unsigned)((num_sms / CL) * CL));
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) == cudaSuccess && clusters > 0)
            cfg.gridDim = dim3((unsigned)(clusters * CL));
        e = cudaLaunchKernelEx(&cfg, kern, prm);
        if (e != cudaSuccess) return -(int)e;
    }
    e = cudaGetLastError();
#ifdef MPW_PROFILE
    if (e == cudaSuccess && prm.trace) {
        // profiling only: dump the trace of this launch (CTA 0), overwriting the previous one
        cudaStreamSynchronize(st);
        const char* path = getenv("MPW_TC_TRACE");
        if (FILE* fh = fopen(path ? path : "gpurun_out/hop_trace.bin", "wb")) {
            fwrite(prm.trace, sizeof(long long), (size_t)tc::TRACE_W * tc::TRACE_TILES, fh);
            fclose(fh);
        }
    }
#endif
    return e == cudaSuccess ? 0 : -(int)e;
}

#define TCL(...) tc_launch_t<__VA_ARGS__>(t, n, nw, A, T, y, y64, s2, P, num_sms, o, st)

int tc_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, const double* y64, S2Dev s2,
              PatDev P, int num_sms, int limbs, const TcOpts& o, cudaStream_t st) {
    if (!t.ready) return 1;
    if (y64) {
        // float64 received words: one fp16 limb, exact re-scoring from y64
        if (limbs != 1) return 1;
        switch (n) {
            case 64: return TCL(1, 2, 1, 3);
            case 128: return TCL(2, 4, 1, 3);
            case 256: return TCL(4, 8, 1, 3);
            default: return 1;
        }
    }
    const int x = o.experiment;
#ifdef MPW_PROFILE
    if (x == 128) {   // per-tile clock trace of CTA 0
        if (limbs == 0 && n == 256)
            return o.i8_pair ? TCL(2, 8, 0, 1, 2, 1) : o.i8_cluster == 2 ? TCL(2, 8, 0, 1, 2) : TCL(2, 8, 0, 1);
        if (limbs == 1 && n == 256) return o.f16_cluster ? TCL(4, 8, 1, 1, 2) : TCL(4, 8, 1, 1);
    }
#endif
    if (limbs == 0) {
        if (!t.ready8) return 1;
        switch (n) {
            case 128: return x ? TCL(1, 4, 0, 2) : TCL(1, 4, 0, 0);
            case 256:
                // i8_cluster 2: CTA pairs sharing the P stream by multicast; i8_pair:
                // the cta_group::2 pair kernel (correct, but slower: the pair's MMAs
                // wait for the slower of two epilogues); default single CTAs
                if (x) return TCL(2, 8, 0, 2);
                if (o.i8_pair) return TCL(2, 8, 0, 0, 2, 1);
                return o.i8_cluster == 2 ? TCL(2, 8, 0, 0, 2) : TCL(2, 8, 0, 0);
            default: return 1;
        }
    }
    if (limbs == 1) {
        switch (n) {
            case 64: return TCL(1, 2, 1, 0);
            case 128: return TCL(2, 4, 1, 0);
            case 256:
                if (x) return TCL(4, 8, 1, 2);
                return o.f16_cluster ? TCL(4, 8, 1, 0, 2) : TCL(4, 8, 1, 0);
            default: return 1;
        }
    }
    switch (n) {
        case 64: return TCL(1, 2, 2, 0);
        case 128: return TCL(2, 4, 2, 0);
        case 256: return TCL(4, 8, 2, 0);
        default: return 1;
    }
}
