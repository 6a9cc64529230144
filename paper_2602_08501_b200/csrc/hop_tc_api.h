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
};

bool tc_supported(int n, int np);
bool tc_i8_supported(int n, int np);
void tc_release(TcPatterns& t);
// P bits -> fp16 0/1 tile images [ntiles][KB][256 x 64] already in the SW128
// shared-memory layout, so one 32 KB bulk copy fills one pipeline stage.
int tc_build(TcPatterns& t, const uint32_t* bits, int np, int n, int nw);
// limbs: 1 or 2 fp16 limbs, 0 = int8 screen.
// 0 on launch, -cudaError on failure, 1 for an unsupported shape
int tc_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, S2Dev s2, PatDev P,
              int num_sms, int limbs, cudaStream_t st);
