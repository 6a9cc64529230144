// Host API of the tensor-core hop (definitions in hop_tc.cu, a separate
// translation unit so the kernel templates compile in parallel with the rest).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

struct TcPatterns {
    bool ready = false;
    uint8_t* tiles = nullptr;
    int np = 0, ntiles = 0, kb = 0;
    // int8 screen (N = 128, 256): u8 0/1 images [ntiles8][N/128][I8_TILE x 128] in the SW128 layout
    bool ready8 = false;
    uint8_t* tiles8 = nullptr;
    int kb8 = 0, ntiles8 = 0;   // int8 tiles are tc::I8_TILE patterns wide
    // asynchronous-row hop, launch statistics accumulated by the kernel: [0] tiles, [1] clock cycles of the
    // first MMA issuer thread, summed over CTAs (read by mpw_hop_tile_stats)
    unsigned long long* ar_stat = nullptr;
};

// Launch options of the tensor hop (per handle, mpw_set_option)
struct TcOpts {
    int experiment = 0;    // Params::experiment bits (profiling / test hooks; MODE 2 kernels)
    int i8_pair = 0;       // int8, N = 256: cta_group::2 pair kernel
    int i8_cluster = 1;    // int8, N = 256: 2 = CTA pairs sharing the P stream by multicast
    int f16_cluster = 1;   // 1-limb, N = 256: CTA pairs sharing the P stream (default on)
    int ar_hit_cap = 0;    // asynchronous-row hop: hit-list capacity per scan thread (0 = the compiled maximum)
};

bool tc_supported(int n, int np);
bool tc_i8_supported(int n, int np);
void tc_release(TcPatterns& t);
// P bits -> fp16 0/1 tile images [ntiles][KB][256 x 64] already in the SW128
// shared-memory layout, so one 32 KB bulk copy fills one pipeline stage.
int tc_build(TcPatterns& t, const uint32_t* bits, int np, int n, int nw);
// limbs: 1 or 2 fp16 limbs, 0 = int8 screen.
// 0 on launch, -cudaError on failure, 1 for an unsupported shape
// y64 (may be null): the caller's float64 received words, y their fp32
// rounding; only the 1-limb screen takes them.
int tc_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, const double* y64, S2Dev s2,
              PatDev P, int num_sms, int limbs, const TcOpts& o, cudaStream_t st);

// Asynchronous-row int8 hop (hop_ar.cuh): rows scan P in their own cycles, worker
// warps decide; needs the u8 images of TcPatterns.
// o.experiment != 0 launches the statistics build (one line on stderr per launch).
bool ar_supported(const TcPatterns& t, int n);
// y64 (may be null): the caller's float64 received words, y their fp32 rounding.
int ar_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, const double* y64, S2Dev s2, PatDev P,
              int num_sms, const TcOpts& o, cudaStream_t st);
