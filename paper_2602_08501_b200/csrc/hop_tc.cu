// Tensor-core hop: host side (operand images, launch).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hop_tc.cuh"
#include "hop_tc_api.h"

// ---------------------------------------------------------------------------
// host side

static int tc_experiment() {
    const char* e = getenv("MPW_TC_EXPERIMENT");
    return e ? atoi(e) : 0;
}


bool tc_supported(int n, int np) { return (n == 64 || n == 128 || n == 256) && np >= 1; }

void tc_release(TcPatterns& t) {
    if (t.tiles) cudaFree(t.tiles);
    t.tiles = nullptr;
    t.ready = false;
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
    return 0;
}

template <int KB, int NW, int LIMBS, int MODE>
static int tc_launch_t(const TcPatterns& t, int n, int nw, int A, int T, const float* y, S2Dev s2, PatDev P,
                       int num_sms, cudaStream_t st) {
    tc::Params prm;
    prm.n = n; prm.nw = nw; prm.A = A; prm.T = T; prm.np = t.np; prm.ntiles = t.ntiles;
    prm.y = y; prm.s2 = s2; prm.pbits = P.bits; prm.btiles = t.tiles; prm.tie_rel = 1e-5f;
    prm.err = 2e-3f;
    prm.experiment = tc_experiment();
    static long long* trace = nullptr;
    prm.trace = nullptr;
    if (prm.experiment & 128) {
        const size_t tb = sizeof(long long) * tc::TRACE_W * tc::TRACE_TILES;
        if (!trace && cudaMallocManaged(&trace, tb) != cudaSuccess) trace = nullptr;
        if (trace) memset(trace, 0, tb);
        prm.trace = trace;
    }
    const size_t smem = tc::smem_bytes(KB, LIMBS);
    cudaError_t e = cudaFuncSetAttribute(tc::hop_tc_kernel<KB, NW, LIMBS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return -(int)e;
    tc::hop_tc_kernel<KB, NW, LIMBS, MODE><<<num_sms, tc::THREADS, smem, st>>>(prm);
    e = cudaGetLastError();
    if (e == cudaSuccess && prm.trace) {
        // profiling only: dump the trace of this launch (CTA 0), overwriting the previous one
        cudaStreamSynchronize(st);
        const char* path = getenv("MPW_TC_TRACE");
        if (FILE* fh = fopen(path ? path : "gpurun_out/hop_trace.bin", "wb")) {
            fwrite(prm.trace, sizeof(long long), (size_t)tc::TRACE_W * tc::TRACE_TILES, fh);
            fclose(fh);
        }
    }
    return e == cudaSuccess ? 0 : -(int)e;
}

int tc_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, S2Dev s2, PatDev P,
                     int num_sms, int limbs, cudaStream_t st) {
    if (!t.ready) return 1;
    if (limbs == 1) {
        switch (n) {
            case 64: return tc_launch_t<1, 2, 1, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
            case 128: return tc_launch_t<2, 4, 1, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
            case 256: {
                // profiling builds of the cfg4 shape: 128 alone = trace only, other knobs = full
                const int x = tc_experiment();
                if (x == 128) return tc_launch_t<4, 8, 1, 1>(t, n, nw, A, T, y, s2, P, num_sms, st);
                if (x) return tc_launch_t<4, 8, 1, 2>(t, n, nw, A, T, y, s2, P, num_sms, st);
                return tc_launch_t<4, 8, 1, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
            }
            default: return 1;
        }
    }
    switch (n) {
        case 64: return tc_launch_t<1, 2, 2, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
        case 128: return tc_launch_t<2, 4, 2, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
        case 256: return tc_launch_t<4, 8, 2, 0>(t, n, nw, A, T, y, s2, P, num_sms, st);
        default: return 1;
    }
}
