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

// Per-frame flags (include/mpwsd.h)
#define MPW_F_TIE_ARGMIN 1u
#define MPW_F_TIE_ACCEPT 2u
#define MPW_F_TIE_FINAL 4u
#define MPW_F_UNRESOLVED 8u

// Running top-3 of a scan (values S_p, ascending; index order breaks ties
// because patterns are visited in increasing index, decoders.py:391).
struct Top3 {
    float b1, b2, b3;
    int i1, i2;
    __device__ __forceinline__ void reset() { b1 = b2 = b3 = CUDART_INF_F; i1 = i2 = 0; }
    __device__ __forceinline__ void push(float s, int p) {
        if (s < b3) {
            if (s < b2) {
                b3 = b2;
                if (s < b1) { b2 = b1; i2 = i1; b1 = s; i1 = p; }
                else { b2 = s; i2 = p; }
            } else {
                b3 = s;
            }
        }
    }
};

// Exact (float64) S_p = Σ_{i∈supp p} x_i y_i for the centre c (decoders.py:329-336).
template <int NW>
__device__ __forceinline__ double exact_score(const float* __restrict__ yrow, const uint32_t (&c)[NW],
                                              const uint32_t* __restrict__ pb, int nw, int n) {
    // y is read 32 values (8 x float4) per word, all loads issued before use,
    // so one exact score costs ~nw L2 round trips instead of one per set bit.
    double s = 0.0;

#pragma unroll
    for (int w = 0; w < NW; w++) {
        if (w >= nw) break;
        const uint32_t bits = pb[w];
        if (!bits) continue;
        const uint32_t cw = c[w];
        float v[32];
        if (n >= 32) {
            const float4* y4 = reinterpret_cast<const float4*>(yrow + w * 32);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const float4 t = y4[q];
                v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
            }
        }
#pragma unroll
        for (int b = 0; b < 32; b++) {
            if ((bits >> b) & 1u) {
                const double yi = (double)(n >= 32 ? v[b] : yrow[b]);
                s += ((cw >> b) & 1u) ? -yi : yi;
            }
        }
    }
    return s;
}

// End-of-scan decision with certification.  fp32 scores carry at most `err`
// absolute error; any pair inside the window is re-scored in float64, so the
// chosen pattern and the accept test match exact arithmetic unless a third
// candidate also falls inside the window (flagged MPW_F_UNRESOLVED).
// Near-tie report (north-star definition): exact relative gaps < tie_rel.
template <int NW>
__device__ __forceinline__ void certify_hop(const Top3& t, const float* __restrict__ yrow,
                                            const uint32_t (&c)[NW], const uint32_t* __restrict__ pbits,
                                            int nw, int n, float ed, float tie_rel, float err, int& best,
                                            bool& improve, uint8_t& flags) {
    const float thr = tie_rel * ed * 0.25f;          // 1e-5 relative ED gap, in S units
    const float win = thr + 2.0f * err;
    best = t.i1;
    improve = t.b1 < 0.0f;
    const bool pair = (t.b2 - t.b1) < win;
    const bool zero = fabsf(t.b1) < win;
    if (!pair && !zero) return;
    double e1 = exact_score<NW>(yrow, c, pbits + (size_t)t.i1 * nw, nw, n);
    double eb = e1;
    if (pair) {
        const double e2 = exact_score<NW>(yrow, c, pbits + (size_t)t.i2 * nw, nw, n);
        if (e2 < e1 || (e2 == e1 && t.i2 < t.i1)) { best = t.i2; eb = e2; }
        if (fabs(e2 - e1) < (double)thr) flags |= MPW_F_TIE_ARGMIN;
        if ((t.b3 - t.b1) < win) flags |= MPW_F_UNRESOLVED;
    }
    improve = eb < 0.0;
    if (fabs(eb) < (double)thr) flags |= MPW_F_TIE_ACCEPT;
}

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
