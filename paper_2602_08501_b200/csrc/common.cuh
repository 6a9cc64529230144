// Shared device-side definitions for the MP-WSD hot path (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#define MPW_FULL 0xffffffffu

// Code tables on the device (filled by mpw_set_code).  Bit layout of every
// packed vector: bit j in bit (j % 32) of uint32 word j / 32 (= the
// reference's uint64 layout read as little-endian uint32, binlin.py:1-8).
struct CodeDev {
    int n, m, nw;          // blocklength, log2 n, uint32 words per vector
    int k, kp;             // message bits, inner (precoded) bits
    int is_ca, crc_deg;    // CRC-concatenated?  CRC degree
    const int32_t* info;   // kp, ascending (codebook.py:225-238)
    const uint32_t* frozen;// nw words, bit = 1 if frozen
    const uint32_t* gen;   // k x nw: effective generator rows (codebook.py:261-271)
    const uint64_t* crc_h; // crc_deg masks over v: syndrome bit j = parity(v & crc_h[j])
    const int32_t* pivots; // k: message_of pivots (codebook.py:104-132)
    const uint64_t* mix;   // k: message_of mixing rows (k <= 64)
};

// Pattern set P on the device (filled by mpw_set_patterns).
struct PatDev {
    int np;                // |P| (nonzero sphere members, member order)
    int nw;
    const uint32_t* bits;  // np x nw
    const int32_t* off;    // np + 1 support offsets
    const uint16_t* idx;   // concatenated supports (ascending positions)
};

// Outputs of the stage-2 queue and trajectories.
struct S2Dev {
    int32_t* count;        // [1] number of queued stage-2 frames
    int32_t* frame;        // [cap] frame id of queue slot q
    int32_t* nanchor;      // [cap]
    uint32_t* anchors;     // [cap x A x nw]
    uint32_t* traj_cw;     // [cap x A x nw] final centres
    int32_t* traj_iters;   // [cap x A]
    int32_t* traj_hops;    // [cap x A x T] accepted pattern index per hop (-1 = none)
    uint8_t* traj_flags;   // [cap x A] bit0 near-tie argmin, bit1 near-tie accept
    int32_t* work_next;    // [1] persistent-kernel work counter
};

__device__ __forceinline__ int getbit32(const uint32_t* w, int j) { return (w[j >> 5] >> (j & 31)) & 1u; }

// Polar butterfly on packed words (codebook.py:166-178): for every h, first
// half of each 2h block ^= second half.  Bits >= n are zero so the in-word
// steps are harmless for n < 32.
template <int NW>
__device__ __forceinline__ void polar_transform_words(uint32_t (&x)[NW], int nw) {
    const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
#pragma unroll
    for (int s = 0; s < 5; s++) {
#pragma unroll
        for (int w = 0; w < NW; w++) x[w] ^= (x[w] >> (1 << s)) & masks[s];
    }
#pragma unroll
    for (int hw = 1; hw < NW; hw *= 2) {
#pragma unroll
        for (int w = 0; w < NW; w++)
            if (!(w & hw) && w + hw < nw) x[w] ^= x[w + hw];
    }
}
