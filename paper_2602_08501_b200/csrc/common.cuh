// Shared device-side definitions for the MP-WSD hot path (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>
#include <cuda_fp16.h>

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
    float4* ebound;        // [cap] per-frame score error bounds (warp_error_bounds)
    float4* qscale;        // [cap] int8 quantisation of the frame (warp_i8_scale): inv_s, s, error bound
    int wmax;              // max pattern weight of P
};

__device__ __forceinline__ int getbit32(const uint32_t* w, int j) { return (w[j >> 5] >> (j & 31)) & 1u; }

// Per-frame flags (include/mpwsd.h)
#define MPW_F_TIE_ARGMIN 1u
#define MPW_F_TIE_ACCEPT 2u
#define MPW_F_TIE_FINAL 4u
#define MPW_F_UNRESOLVED 8u

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

// The same score from the caller's float64 received word (float64 inputs).
template <int NW>
__device__ __forceinline__ double exact_score64(const double* __restrict__ yrow, const uint32_t (&c)[NW],
                                                const uint32_t* __restrict__ pb, int nw, int n) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
        if (w >= nw) break;
        const uint32_t bits = pb[w], cw = c[w];
        for (uint32_t b = bits; b; b &= b - 1) {
            const int i = __ffs(b) - 1;
            const double yi = yrow[w * 32 + i];
            s += ((cw >> i) & 1u) ? -yi : yi;
        }
    }
    return s;
}

// Upper bound on the sum of the w largest of the values x[] spread over the
// warp (lane holds x[lane + 32 j]): for any tau with #{x > tau} <= w,
// sum_top_w <= sum_{x > tau} x + (w - #{x > tau}) * tau.  tau by bisection.
// CNT > 0: the lane's value count is a compile-time constant (n = 32 CNT), so the
// arrays of the callers stay in registers; CNT = 0: any n <= 1024.
template <int CNT = 0>
__device__ __forceinline__ float warp_topw_bound(const float* xv, int cnt_rt, int w) {
    constexpr int CAP = CNT ? CNT : 32;
    const int cnt = CNT ? CNT : cnt_rt;
    float mx = 0.0f;
#pragma unroll
    for (int j = 0; j < CAP; j++) if (j < cnt) mx = fmaxf(mx, xv[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(MPW_FULL, mx, o));
    float lo = 0.0f, hi = mx;
    for (int it = 0; it < 12; it++) {
        const float mid = 0.5f * (lo + hi);
        int c = 0;
#pragma unroll
        for (int j = 0; j < CAP; j++) if (j < cnt) c += xv[j] > mid;
        c = __reduce_add_sync(MPW_FULL, c);
        if (c <= w) hi = mid; else lo = mid;
    }
    float s = 0.0f;
    int c = 0;
#pragma unroll
    for (int j = 0; j < CAP; j++) if (j < cnt && xv[j] > hi) { s += xv[j]; c++; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(MPW_FULL, s, o);
    c = __reduce_add_sync(MPW_FULL, c);
    return (s + (float)(w - c) * hi) * 1.0001f;
}

// Per-frame score error bounds (S units) for the hop kernels, computed by one
// warp from y: |t_i| = |y_i| and the fp16 split errors of t_i = ±y_i do not
// depend on the sign pattern x, so one bound serves every hop of every anchor.
//   x: 1-limb tensor (fp16(t)),  y: 2-limb tensor (fp16 hi + fp16 lo),
//   z: fp32 gather,              w: sum of the wmax largest |y_i|.
// Each sums the wmax largest per-element representation errors and adds
// an fp32 accumulation bound of (terms) * 2^-23 * sum|t| (2^-23 = 2u per
// add: the tensor cores' fp32 accumulation is not guaranteed to round to
// nearest).
template <int CNT = 0>
__device__ __forceinline__ float4 warp_error_bounds(const float* __restrict__ yrow, int n, int wmax) {
    const int lane = threadIdx.x & 31;
    constexpr int CAP = CNT ? CNT : 32;
    float ay[CAP], e1[CAP], e2[CAP];
    const int cnt = CNT ? CNT : (n - lane + 31) / 32;
#pragma unroll
    for (int j = 0; j < CAP; j++) {
        if (j < cnt) {
            const float y = yrow[lane + 32 * j];
            const float h = __half2float(__float2half_rn(y));
            const float l = __half2float(__float2half_rn(y - h));
            ay[j] = fabsf(y);
            e1[j] = fabsf(y - h);
            e2[j] = fabsf((y - h) - l);
        }
    }
    const float A = warp_topw_bound<CNT>(ay, cnt, wmax);
    const float T1 = warp_topw_bound<CNT>(e1, cnt, wmax);
    const float T2 = warp_topw_bound<CNT>(e2, cnt, wmax);
    const float u = 1.1920929e-7f;   // 2^-23
    return make_float4(T1 + (float)wmax * u * A, T2 + 2.0f * (float)wmax * u * A,
                       (float)wmax * u * A, A);
}

// Per-frame int8 quantisation for the int8 tensor screen: t_i = ±y_i is
// represented as s·q_i with q_i = ±rint(|y_i|·inv_s) in [-127, 127],
// inv_s = 127 / max|y|, s = rcp_rn(inv_s) (the kernels repeat exactly these
// fp32 operations).  The MMA sums the q_i exactly (s32 accumulators), so the
// score error of every pattern is at most the sum of the wmax largest
// |(|y_i| - s·q_i)| plus the fp32 rounding of s·acc and of the window
// arithmetic (|acc| <= 127·wmax).  Returns {inv_s, s, bound, sum|y| (rounded up)}.
__device__ __forceinline__ float i8_inv_scale(float ymax) {
    return ymax > 1e-30f ? __fdiv_rn(127.0f, ymax) : 1.0f;
}
__device__ __forceinline__ int i8_quant(float ay, float inv_s) { return __float2int_rn(__fmul_rn(ay, inv_s)); }

template <int CNT = 0>
__device__ __forceinline__ float4 warp_i8_scale(const float* __restrict__ yrow, int n, int wmax) {
    const int lane = threadIdx.x & 31;
    constexpr int CAP = CNT ? CNT : 32;
    float ay[CAP], e8[CAP];
    const int cnt = CNT ? CNT : (n - lane + 31) / 32;
    float mx = 0.0f;
#pragma unroll
    for (int j = 0; j < CAP; j++) {
        if (j < cnt) {
            ay[j] = fabsf(yrow[lane + 32 * j]);
            mx = fmaxf(mx, ay[j]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(MPW_FULL, mx, o));
    const float inv_s = i8_inv_scale(mx);
    const float s = __frcp_rn(inv_s);
#pragma unroll
    for (int j = 0; j < CAP; j++) {
        if (j < cnt) {
            const int q = i8_quant(ay[j], inv_s);
            const double e = fabs((double)ay[j] - (double)s * (double)q);
            e8[j] = __double2float_ru(e);
        }
    }
    const float T8 = warp_topw_bound<CNT>(e8, cnt, wmax);
    const float u = 1.1920929e-7f;   // 2^-23
    float sa = 0.0f;                 // sum |y_i|, rounded up below (certification bound)
#pragma unroll
    for (int j = 0; j < CAP; j++) if (j < cnt) sa += ay[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sa += __shfl_xor_sync(MPW_FULL, sa, o);
    return make_float4(inv_s, s, T8 + 4.0f * u * s * 127.0f * (float)wmax, sa * 1.0001f);
}

// Running top-K (K small) of a scan; ascending values, index order breaks ties.
template <int K>
struct TopK {
    float b[K];
    int i[K];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < K; k++) { b[k] = CUDART_INF_F; i[k] = 0; }
    }
    __device__ __forceinline__ float last() const { return b[K - 1]; }
    __device__ __forceinline__ void push(float s, int p) {
        if (!(s < b[K - 1])) return;
        insert(s, p);
    }
    // precondition: s < b[K-1]; branch-free sorted insertion (registers only)
    __device__ __forceinline__ void insert_inline(float s, int p) {
#pragma unroll
        for (int k = K - 1; k > 0; k--) {
            const bool up = s < b[k - 1];          // s goes above slot k
            const bool here = !up && s < b[k];     // s lands in slot k
            const float nb = up ? b[k - 1] : (here ? s : b[k]);
            const int ni = up ? i[k - 1] : (here ? p : i[k]);
            b[k] = nb;
            i[k] = ni;
        }
        if (s < b[0]) { b[0] = s; i[0] = p; }
    }
    // precondition: s < b[K-1]
    __device__ __forceinline__ void insert(float s, int p) {
        // insertion from the back; strict < keeps earlier indices first on ties
#pragma unroll
        for (int k = K - 1; k > 0; k--) {
            if (s < b[k - 1]) { b[k] = b[k - 1]; i[k] = i[k - 1]; }
            else { b[k] = s; i[k] = p; return; }
        }
        b[0] = s; i[0] = p;
    }
};

// Certified decision from a top-K list whose scores carry at most `err_row`
// absolute error: every candidate within 2·err (+ the report threshold) of the
// best approximate score is re-scored in float64; the exact argmin (ties ->
// lowest index) and the exact accept test are used.  If the K-th score is
// also inside the window the scan is flagged MPW_F_UNRESOLVED.
// y64row (may be null): the caller's float64 received word, re-scored from
// instead of yrow (err_row then includes the fp32 rounding of y).
template <int K, int NW>
__device__ __forceinline__ void certify_topk(const TopK<K>& t, const float* __restrict__ yrow,
                                             const double* __restrict__ y64row,
                                             const uint32_t (&c)[NW], const uint32_t* __restrict__ pbits,
                                             int nw, int n, float ed, float tie_rel, float err_row, int& best,
                                             bool& improve, float& best_approx, uint8_t& flags) {
    auto score = [&](int p) {
        return y64row ? exact_score64<NW>(y64row, c, pbits + (size_t)p * nw, nw, n)
                      : exact_score<NW>(yrow, c, pbits + (size_t)p * nw, nw, n);
    };
    const float thr = tie_rel * ed * 0.25f;
    const float win = thr + 2.0f * err_row;
    best = t.i[0];
    best_approx = t.b[0];
    improve = t.b[0] < 0.0f;
    const bool pair = (t.b[1] - t.b[0]) < win;
    const bool zero = fabsf(t.b[0]) < err_row + thr;
    if (!pair && !zero) return;
    double eb = score(t.i[0]);
    double e_second = CUDART_INF;
#pragma unroll
    for (int k = 1; k < K - 1; k++) {
        if (!((t.b[k] - t.b[0]) < win)) break;
        const double e = score(t.i[k]);
        if (e < eb || (e == eb && t.i[k] < best)) {
            e_second = eb;
            eb = e;
            best = t.i[k];
            best_approx = t.b[k];
        } else if (e < e_second) {
            e_second = e;
        }
    }
    if ((t.b[K - 1] - t.b[0]) < win) flags |= MPW_F_UNRESOLVED;
    if (e_second - eb < (double)thr) flags |= MPW_F_TIE_ARGMIN;
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
