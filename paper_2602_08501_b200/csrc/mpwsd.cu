// libmpwsd: B200-native MP-WSD two-stage decoding, C-ABI (include/mpwsd.h).
//
// Pipeline of one batch (all on the caller's stream, no host sync):
//   scl_kernel       stage 1 + CRC gate + projection + stage-2 compaction
//   hop_*_kernel     stage 2 hops over the compacted trajectories
//   finalize_kernel  canonical float64 EDs, min over anchors, near-tie flags
//   frame_kernel     message_of, per-frame outputs, counters
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mpwsd.h"
#include "common.cuh"
#include "hop_gather.cuh"
#include "hop_tc_api.h"
#include "scl.cuh"
#include "scl_lane_api.h"
#include "channel.cuh"
#include "enum.cuh"
#include "osd.cuh"

#include <cub/device/device_segmented_sort.cuh>

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CK(expr)                                                                     \
    do {                                                                             \
        cudaError_t e_ = (expr);                                                     \
        if (e_ != cudaSuccess)                                                       \
            return fail(MPW_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                         \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t count) {
        if (count <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) cap = std::max<size_t>(count, 1);
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

struct mpw_handle {
    int device = 0;
    int num_sms = 148;
    // code
    bool has_code = false;
    int n = 0, m = 0, nw = 0, k = 0, kp = 0, is_ca = 0, crc_deg = 0;
    DevBuf<int32_t> info, pivots;
    DevBuf<uint32_t> frozen, gen;
    DevBuf<uint64_t> crc_h, mix;
    // patterns
    bool has_pat = false;
    int np = 0;
    int total_sup_u4 = 0;
    DevBuf<uint32_t> pbits;
    DevBuf<int32_t> poff, soff;
    DevBuf<uint16_t> pidx;
    DevBuf<uint4> sup;
    TcPatterns tcp;                 // tensor-core operand of P (hop_tc.cuh)
    // stage-2 scratch
    DevBuf<int32_t> s2_count, s2_frame, s2_nanchor, traj_iters, traj_hops, work_next;
    DevBuf<uint32_t> s2_anchors, traj_cw;
    DevBuf<uint8_t> traj_flags;
    DevBuf<float4> ebound;
    DevBuf<float4> qscale;
    DevBuf<uint8_t> s1_flags;       // OSD stage-1 near-tie flags
    // float64 inputs: fp32 rounding of y (screens) and float64 channel LLRs (stage 1)
    DevBuf<float> y32;
    DevBuf<double> llr64;
    // mpw_two_stage_batch_host staging (owned by the handle, so on its device)
    DevBuf<float> hy;
    DevBuf<uint32_t> htx, hbest;
    DevBuf<uint64_t> hmsg;
    DevBuf<double> hed;
    DevBuf<uint8_t> hstage, hflags;
    DevBuf<int32_t> hiters;
    DevBuf<unsigned long long> hctr;
    int wmax = 0;
    int scl_generic = 0;            // force the warp-per-frame SCL kernel
    TcOpts tco;                     // tensor-hop launch options (mpw_set_option)
    long long kernel_launches = 0;  // kernels this handle launched (mpw_launch_count)
    // timing
    int timing = 0;
    cudaEvent_t ev[8];
    bool ev_init = false;
    double acc_ms[4] = {0, 0, 0, 0};
    long long launches[4] = {0, 0, 0, 0};
    long long evals = 0;
};

namespace {

CodeDev code_dev(const mpw_handle* h) {
    CodeDev c;
    c.n = h->n; c.m = h->m; c.nw = h->nw; c.k = h->k; c.kp = h->kp;
    c.is_ca = h->is_ca; c.crc_deg = h->crc_deg;
    c.info = h->info.p; c.frozen = h->frozen.p; c.gen = h->gen.p; c.crc_h = h->crc_h.p;
    c.pivots = h->pivots.p; c.mix = h->mix.p;
    return c;
}

PatDev pat_dev(const mpw_handle* h) {
    PatDev p;
    p.np = h->np; p.nw = h->nw; p.bits = h->pbits.p; p.off = h->poff.p; p.idx = h->pidx.p;
    return p;
}

int set_device(mpw_handle* h) {
    CK(cudaSetDevice(h->device));
    return 0;
}

// ---------------------------------------------------------------------------
// finalize: canonical float64 EDs of the final centres, min over anchors with
// ties to the lowest anchor (decoders.py:505), near-tie flag for distinct
// codewords whose EDs differ by < tie_rel (relative).
struct FinalOut {
    uint32_t* best; double* best_ed; uint8_t* stage; int32_t* iters; int32_t* hops;
    uint32_t* anchors; uint8_t* flags; int32_t* best_k;
};

// CNT = n / 32 as a constant (n = 64 / 128 / 256): the frame's received word
// and the codeword words live in registers; CNT = 0: any n.  The float64 sums
// keep one order in both forms: lane-sequential over i = lane + 32 j, then the
// xor butterfly.
template <int CNT>
__global__ void finalize_kernel(int n, int nw, int A, int T, const float* __restrict__ y,
                                const double* __restrict__ y64, S2Dev s2, FinalOut out, float tie_rel) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int count = *s2.count;
    for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < count; q += warps) {
        const int f = s2.frame[q], na = s2.nanchor[q];
        // per-anchor outputs of the frame, copied in bulk
        if (out.iters)
            for (int a = lane; a < A; a += 32) out.iters[(size_t)f * A + a] = a < na ? s2.traj_iters[(size_t)q * A + a] : 0;
        if (out.hops)
            for (int i = lane; i < na * T; i += 32) out.hops[(size_t)f * A * T + i] = s2.traj_hops[(size_t)q * A * T + i];
        if (out.anchors)
            for (int i = lane; i < na * nw; i += 32) out.anchors[(size_t)f * A * nw + i] = s2.anchors[(size_t)q * A * nw + i];
        uint32_t flw = 0;
        for (int a = lane; a < na; a += 32) flw |= s2.traj_flags[(size_t)q * A + a];
        uint8_t fl = (uint8_t)__reduce_or_sync(MPW_FULL, flw);

        double best = CUDART_INF, second = CUDART_INF;
        int bk = 0;
        if constexpr (CNT > 0) {
            double yd[CNT];
#pragma unroll
            for (int j = 0; j < CNT; j++)
                yd[j] = y64 ? y64[(size_t)f * n + lane + 32 * j] : (double)y[(size_t)f * n + lane + 32 * j];
            uint32_t bw[CNT];
#pragma unroll
            for (int j = 0; j < CNT; j++) bw[j] = 0u;
            for (int a = 0; a < na; a++) {
                const uint32_t* cw = s2.traj_cw + ((size_t)q * A + a) * nw;
                uint32_t w[CNT];
                if constexpr (CNT % 4 == 0) {
#pragma unroll
                    for (int j = 0; j < CNT; j += 4) {
                        const uint4 v = *reinterpret_cast<const uint4*>(cw + j);
                        w[j] = v.x; w[j + 1] = v.y; w[j + 2] = v.z; w[j + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < CNT; j++) w[j] = cw[j];
                }
                double acc = 0.0;
                bool same = true;
#pragma unroll
                for (int j = 0; j < CNT; j++) {
                    const double x = ((w[j] >> lane) & 1u) ? -1.0 : 1.0;
                    const double d = yd[j] - x;
                    acc += d * d;
                    same = same && (w[j] == bw[j]);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(MPW_FULL, acc, o);
                if (a == 0) same = true;
                if (acc < best) {
                    if (a > 0 && !same) second = best;
                    best = acc;
                    bk = a;
#pragma unroll
                    for (int j = 0; j < CNT; j++) bw[j] = w[j];
                } else if (!same && acc < second) {
                    second = acc;
                }
            }
        } else {
            for (int a = 0; a < na; a++) {
                const uint32_t* cw = s2.traj_cw + ((size_t)q * A + a) * nw;
                double acc = 0.0;
                for (int i = lane; i < n; i += 32) {
                    const double x = ((cw[i >> 5] >> (i & 31)) & 1u) ? -1.0 : 1.0;
                    const double d = (y64 ? y64[(size_t)f * n + i] : (double)y[(size_t)f * n + i]) - x;
                    acc += d * d;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(MPW_FULL, acc, o);
                bool same = true;   // identical codeword to the current best?
                if (a > 0) {
                    const uint32_t* bc = s2.traj_cw + ((size_t)q * A + bk) * nw;
                    bool diff = false;
                    for (int w = lane; w < nw; w += 32) diff |= cw[w] != bc[w];
                    same = !__any_sync(MPW_FULL, diff);
                }
                if (acc < best) {
                    if (a > 0 && !same) second = best;
                    best = acc;
                    bk = a;
                } else if (!same && acc < second) {
                    second = acc;
                }
            }
        }
        if (second - best < (double)tie_rel * best) fl |= 4;
        for (int w = lane; w < nw; w += 32) out.best[(size_t)f * nw + w] = s2.traj_cw[((size_t)q * A + bk) * nw + w];
        if (lane == 0) {
            out.best_ed[f] = best;
            if (out.stage) out.stage[f] = 1;
            if (out.flags) out.flags[f] = fl;
            if (out.best_k) out.best_k[f] = bk;
        }
    }
}

// per-frame epilogue: message_of (codebook.py:123-132), stage-1 defaults, counters
struct FrameArgs {
    int F, A, T, nw, k, np;
    const uint32_t* best; const uint8_t* stage; const uint32_t* tx;
    int32_t* iters; int32_t* hops; uint8_t* flags; uint64_t* msg_out;
    const uint8_t* s1flags;         // per-frame stage-1 near-tie flags (OSD), may be null
    unsigned long long* counters;
    const int32_t* pivots; const uint64_t* mix;
};

__global__ void frame_kernel(FrameArgs fa) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c_err = 0, c_act = 0, c_it = 0, c_tie = 0, c_fr = 0, c_unr = 0;
    if (f < fa.F) {
        const uint32_t* b = fa.best + (size_t)f * fa.nw;
        if (fa.msg_out && fa.k <= 64) {
            uint64_t msg = 0;
            for (int j = 0; j < fa.k; j++) {
                const int p = fa.pivots[j];
                if ((b[p >> 5] >> (p & 31)) & 1u) msg ^= fa.mix[j];
            }
            fa.msg_out[f] = msg;
        }
        const bool s2 = fa.stage[f] == 1;
        if (!s2) {
            if (fa.iters) for (int a = 0; a < fa.A; a++) fa.iters[(size_t)f * fa.A + a] = 0;
            if (fa.hops) for (int a = 0; a < fa.A * fa.T; a++) fa.hops[(size_t)f * fa.A * fa.T + a] = -1;
            if (fa.flags) fa.flags[f] = 0;
        } else if (fa.iters) {
            for (int a = 0; a < fa.A; a++) c_it += (unsigned long long)fa.iters[(size_t)f * fa.A + a];
        }
        if (fa.flags && fa.s1flags) fa.flags[f] |= fa.s1flags[f];
        c_fr = 1;
        c_act = s2 ? 1 : 0;
        c_tie = (fa.flags && (fa.flags[f] & 23u)) ? 1 : 0;
        c_unr = (fa.flags && (fa.flags[f] & 8u)) ? 1 : 0;
        if (fa.tx) {
            bool diff = false;
            for (int w = 0; w < fa.nw; w++) diff |= b[w] != fa.tx[(size_t)f * fa.nw + w];
            c_err = diff ? 1 : 0;
        }
    }
    if (fa.counters) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c_fr += __shfl_xor_sync(MPW_FULL, c_fr, o);
            c_err += __shfl_xor_sync(MPW_FULL, c_err, o);
            c_act += __shfl_xor_sync(MPW_FULL, c_act, o);
            c_it += __shfl_xor_sync(MPW_FULL, c_it, o);
            c_tie += __shfl_xor_sync(MPW_FULL, c_tie, o);
            c_unr += __shfl_xor_sync(MPW_FULL, c_unr, o);
        }
        if ((threadIdx.x & 31) == 0 && c_fr) {
            atomicAdd(&fa.counters[MPW_CTR_FRAMES], c_fr);
            atomicAdd(&fa.counters[MPW_CTR_ERRORS], c_err);
            atomicAdd(&fa.counters[MPW_CTR_ACTIVATIONS], c_act);
            atomicAdd(&fa.counters[MPW_CTR_ITERATIONS], c_it);
            atomicAdd(&fa.counters[MPW_CTR_EVALS], c_it * (unsigned long long)fa.np);
            atomicAdd(&fa.counters[MPW_CTR_NEAR_TIE], c_tie);
            atomicAdd(&fa.counters[MPW_CTR_UNRESOLVED], c_unr);
        }
    }
}

// mp_wsd API: queue = identity over the given frames
// (warp per frame: also the per-frame score error bounds the hop kernels use)
// float64 inputs: every screen bound also covers sum_{supp}|y64_i - y_i| <=
// the sum of the wmax largest fp32 rounding errors of the frame
template <int CNT = 0>
__device__ __forceinline__ float y64_rounding_bound(const float* __restrict__ yrow, const double* __restrict__ y64row,
                                                    int n, int wmax) {
    constexpr int CAP = CNT ? CNT : 32;
    const int lane = threadIdx.x & 31;
    float r[CAP];
    const int cnt = CNT ? CNT : (n - lane + 31) / 32;
#pragma unroll
    for (int j = 0; j < CAP; j++)
        if (j < cnt) r[j] = __double2float_ru(fabs(y64row[lane + 32 * j] - (double)yrow[lane + 32 * j]));
    return warp_topw_bound<CNT>(r, cnt, wmax);
}

// Bounds of one queue entry (warp): the fp16 / fp32 screens' error bounds only where a
// hop that reads them will run (need_eb), the int8 quantisation always.
template <int CNT>
__device__ __forceinline__ void entry_bounds(const float* __restrict__ yr, const double* __restrict__ y64r, int n,
                                             int q, bool need_eb, S2Dev s2) {
    const int lane = threadIdx.x & 31;
    const float R = y64r ? y64_rounding_bound<CNT>(yr, y64r, n, s2.wmax) : 0.0f;
    if (need_eb) {
        float4 eb = warp_error_bounds<CNT>(yr, n, s2.wmax);
        if (y64r) eb = make_float4(eb.x + R, eb.y + R, eb.z + R, eb.w);
        if (lane == 0) s2.ebound[q] = eb;
    }
    float4 qs = warp_i8_scale<CNT>(yr, n, s2.wmax);
    qs.z += R;                                           // int8 screen of fp32(y64)
    if (lane == 0) s2.qscale[q] = qs;
}

template <int CNT>
__global__ void queue_identity_kernel(int F, int A, int n, const float* __restrict__ y,
                                      const double* __restrict__ y64, const int32_t* nanchor, S2Dev s2,
                                      bool need_eb) {
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q == 0 && lane == 0) *s2.count = F;
    if (q < F) {
        entry_bounds<CNT>(y + (size_t)q * n, y64 ? y64 + (size_t)q * n : nullptr, n, q, need_eb, s2);
        if (lane == 0) {
            s2.frame[q] = q;
            s2.nanchor[q] = nanchor ? min(nanchor[q], A) : A;
        }
    }
}

// per-frame score error bounds of the queued stage-2 frames (warp per entry)
template <int CNT>
__global__ void ebound_kernel(int n, const float* __restrict__ y, const double* __restrict__ y64, S2Dev s2,
                              bool need_eb) {
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int count = *s2.count;
    for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < count; q += warps) {
        const size_t f = (size_t)s2.frame[q];
        entry_bounds<CNT>(y + f * n, y64 ? y64 + f * n : nullptr, n, q, need_eb, s2);
    }
}

// launches with the per-lane value count as a constant for n = 64 / 128 / 256
#define MPW_BY_CNT(n_, CALL)                         \
    do {                                             \
        switch (n_) {                                \
            case 64: { constexpr int CNT = 2; CALL; break; }   \
            case 128: { constexpr int CNT = 4; CALL; break; }  \
            case 256: { constexpr int CNT = 8; CALL; break; }  \
            default: { constexpr int CNT = 0; CALL; break; }   \
        }                                            \
    } while (0)

// float64 inputs: fp32 rounding for the screens and float64 channel LLRs
// 2.0 * y / (sigma * sigma) with the reference's operation order (decoders.py:550)
__global__ void y64_prep_kernel(long long total, const double* __restrict__ y64, float* __restrict__ y32,
                                double* __restrict__ llr, double sigma) {
    const double sig2 = sigma * sigma;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = y64[i];
        y32[i] = __double2float_rn(v);
        if (llr) llr[i] = 2.0 * v / sig2;
    }
}

// float64 inputs: canonical squared EDs of the stage-1 (CRC-pass) frames from y64
__global__ void stage1_ed64_kernel(int F, int n, int nw, const double* __restrict__ y64, const uint8_t* stage,
                                   const uint32_t* __restrict__ best, double* best_ed) {
    const int lane = threadIdx.x & 31;
    const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (f >= F || stage[f] != 0) return;
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double x = ((best[(size_t)f * nw + (i >> 5)] >> (i & 31)) & 1u) ? -1.0 : 1.0;
        const double d = y64[(size_t)f * n + i] - x;
        acc += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(MPW_FULL, acc, o);
    if (lane == 0) best_ed[f] = acc;
}

// want_hops: the caller asked for the per-hop pattern log (else the hop
// kernels skip writing it: s2.traj_hops = null)
int ensure_s2(mpw_handle* h, int F, int A, int T, bool want_hops) {
    const size_t traj = (size_t)F * A;
    CK(h->s2_count.ensure(1));
    CK(h->work_next.ensure(1));
    CK(h->s2_frame.ensure(F));
    CK(h->s2_nanchor.ensure(F));
    CK(h->s2_anchors.ensure(traj * h->nw));
    CK(h->traj_cw.ensure(traj * h->nw));
    CK(h->traj_iters.ensure(traj));
    if (want_hops) CK(h->traj_hops.ensure(traj * T));
    CK(h->traj_flags.ensure(traj));
    CK(h->ebound.ensure(F));
    CK(h->qscale.ensure(F));
    return 0;
}

S2Dev s2_dev(mpw_handle* h, const uint32_t* anchors_override, bool want_hops) {
    S2Dev s;
    s.count = h->s2_count.p; s.frame = h->s2_frame.p; s.nanchor = h->s2_nanchor.p;
    s.anchors = anchors_override ? const_cast<uint32_t*>(anchors_override) : h->s2_anchors.p;
    s.traj_cw = h->traj_cw.p; s.traj_iters = h->traj_iters.p; s.traj_hops = want_hops ? h->traj_hops.p : nullptr;
    s.traj_flags = h->traj_flags.p; s.work_next = h->work_next.p;
    s.ebound = h->ebound.p; s.qscale = h->qscale.p; s.wmax = h->wmax;
    return s;
}

void timing_mark(mpw_handle* h, int slot, cudaStream_t st) {
    if (h->timing) cudaEventRecord(h->ev[slot], st);
}

int timing_close(mpw_handle* h) {
    if (!h->timing) return 0;
    CK(cudaEventSynchronize(h->ev[4]));
    float ms;
    for (int i = 0; i < 4; i++) {
        CK(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
        h->acc_ms[i] += ms;
        h->launches[i] += 1;
    }
    return 0;
}

template <int NW>
int launch_scl(mpw_handle* h, const float* y, const double* llr64, int F, double sigma, int L, int A,
               int mode, SclOut out, S2Dev s2, cudaStream_t st) {
    const SclLayout lay = scl_layout(h->n, L, h->nw);
    int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / lay.total));
    const size_t smem = lay.total * wpb;
    if (smem > 227 * 1024) return fail(MPW_ERR_UNSUPPORTED, "SCL shared memory %zu B exceeds the SM (n=%d, L=%d)", smem, h->n, L);
    CK(cudaFuncSetAttribute(scl_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scl_kernel<NW>, 32 * wpb, smem));
    per_sm = std::max(per_sm, 1);
    const long long need = ((long long)F + wpb - 1) / wpb;
    const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)per_sm * h->num_sms * 4));
    scl_kernel<NW><<<grid, 32 * wpb, smem, st>>>(code_dev(h), y, llr64, F, sigma, L, A, mode, out, s2);
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

int dispatch_scl(mpw_handle* h, const float* y, const double* llr64, int F, double sigma, int L, int A,
                 int mode, SclOut out, S2Dev s2, cudaStream_t st) {
    if (h->n & (h->n - 1)) return fail(MPW_ERR_UNSUPPORTED, "SCL needs a power-of-two length (n=%d)", h->n);
    // lane-per-path kernel for the common shapes (power-of-two L, N in {64,128,256}),
    // warp-per-frame kernel otherwise (or when MPW_SCL_GENERIC is set)
    const bool pow2 = L >= 1 && (L & (L - 1)) == 0 && L <= 32;
    if (pow2 && !h->scl_generic) {
        const int rc = scl_lane_launch(h->n, L, code_dev(h), y, llr64, F, sigma, A, mode, out, s2, h->num_sms, st);
        if (rc == 0) { h->kernel_launches++; return 0; }
        if (rc < 0) return fail(MPW_ERR_CUDA, "SCL lane kernel launch failed: %s", cudaGetErrorString((cudaError_t)-rc));
    }
    switch (h->nw) {
        case 1: return launch_scl<1>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        case 2: return launch_scl<2>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        case 4: return launch_scl<4>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        case 8: return launch_scl<8>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        case 16: return launch_scl<16>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        case 32: return launch_scl<32>(h, y, llr64, F, sigma, L, A, mode, out, s2, st);
        default: return fail(MPW_ERR_UNSUPPORTED, "blocklength %d unsupported", h->n);
    }
}

template <int NW>
int launch_gather(mpw_handle* h, HopParams hp, int max_traj, cudaStream_t st) {
    const size_t sup_bytes = ((sizeof(uint4) * (size_t)h->total_sup_u4 + sizeof(int32_t) * (size_t)(h->np + 1)) + 15) & ~(size_t)15;
    const size_t wsm = gather_warp_smem(h->n);
    int wpb = 8;
    while (wpb > 1 && wsm * wpb > 64 * 1024) wpb /= 2;
    hp.sup_in_smem = (sup_bytes + wsm * wpb <= 200 * 1024) ? 1 : 0;
    const size_t smem = (hp.sup_in_smem ? sup_bytes : 0) + wsm * wpb;
    CK(cudaFuncSetAttribute(hop_gather_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hop_gather_kernel<NW>, 32 * wpb, smem));
    per_sm = std::max(per_sm, 1);
    const long long tasks = ((long long)max_traj + 31) / 32;
    const long long need = (tasks + wpb - 1) / wpb;
    const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)per_sm * h->num_sms));
    hop_gather_kernel<NW><<<grid, 32 * wpb, smem, st>>>(hp);
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

// MPW_HOP_AUTO: the int8 screen where a scan streams enough of P to amortise
// its wider certification window (N = 256 and >= 32 tiles of 256 patterns), in
// its asynchronous-row form (hop_ar.cuh: cfg4 82 ms against 107 ms for the
// synchronous rounds of hop_tc.cuh); else one fp16 limb, else the gather kernel
// float64 inputs (f64): the asynchronous-row int8 hop where it applies (its
// workers re-score from the float64 words), else the 1-limb fp16 screen with
// float64 re-scoring, else the gather kernel
int resolve_variant(mpw_handle* h, int variant, bool f64 = false) {
    if (variant != MPW_HOP_AUTO) return variant;
    if (!(tc_supported(h->n, h->np) && h->tcp.ready)) return MPW_HOP_GATHER;
    if (h->tcp.ready8 && h->n >= 256 && h->tcp.ntiles >= 32) {
        if (ar_supported(h->tcp, h->n)) return MPW_HOP_TENSOR_I8_ASYNC;   // float32 and float64 received words
        if (!f64) return MPW_HOP_TENSOR_I8;
    }
    return MPW_HOP_TENSOR;
}

// the int8 screens read only the int8 quantisation bounds (qscale); the fp16 screens and
// the gather also the fp16 / fp32 score error bounds (ebound)
bool needs_fp_bounds(int resolved_variant) {
    return !(resolved_variant == MPW_HOP_TENSOR_I8 || resolved_variant == MPW_HOP_TENSOR_I8_ASYNC);
}

int run_hops(mpw_handle* h, const float* y, const double* y64, int Fmax, int A, int T, int variant, S2Dev s2,
             cudaStream_t st) {
    variant = resolve_variant(h, variant, y64 != nullptr);
    if (y64 && (variant == MPW_HOP_TENSOR_2LIMB || variant == MPW_HOP_TENSOR_I8))
        return fail(MPW_ERR_UNSUPPORTED, "float64 received words use the asynchronous-row int8, the 1-limb tensor or the gather hop");
    if (variant == MPW_HOP_TENSOR_I8_ASYNC) {
        if (!ar_supported(h->tcp, h->n))
            return fail(MPW_ERR_UNSUPPORTED, "asynchronous int8 tensor-core hop needs N = 128 or 256 and the u8 operand images");
        int rc = ar_launch(h->tcp, h->n, h->nw, A, T, y, y64, s2, pat_dev(h), h->num_sms, h->tco, st);
        if (rc) return fail(MPW_ERR_CUDA, "asynchronous tensor-core hop launch failed: %s",
                            rc < 0 ? cudaGetErrorString((cudaError_t)-rc) : "unsupported shape");
        h->kernel_launches++;
        return 0;
    }
    if (variant == MPW_HOP_TENSOR || variant == MPW_HOP_TENSOR_2LIMB || variant == MPW_HOP_TENSOR_I8) {
        if (!h->tcp.ready) return fail(MPW_ERR_UNSUPPORTED, "tensor-core hop operand not built for this pattern set");
        if (variant == MPW_HOP_TENSOR_I8 && !h->tcp.ready8)
            return fail(MPW_ERR_UNSUPPORTED, "int8 tensor-core hop needs N = 128 or 256");
        const int limbs = variant == MPW_HOP_TENSOR ? 1 : variant == MPW_HOP_TENSOR_2LIMB ? 2 : 0;
        int rc = tc_launch(h->tcp, h->n, h->nw, A, T, y, y64, s2, pat_dev(h), h->num_sms, limbs, h->tco, st);
        if (rc) return fail(MPW_ERR_CUDA, "tensor-core hop launch failed: %s",
                            rc < 0 ? cudaGetErrorString((cudaError_t)-rc) : "unsupported shape");
        h->kernel_launches++;
        return 0;
    }
    if (variant != MPW_HOP_GATHER) return fail(MPW_ERR_ARG, "unknown hop variant %d", variant);
    HopParams hp;
    hp.n = h->n; hp.nw = h->nw; hp.A = A; hp.T = T; hp.y = y; hp.y64 = y64; hp.s2 = s2; hp.P = pat_dev(h);
    hp.sup = h->sup.p; hp.soff = h->soff.p; hp.sup_in_smem = 0; hp.total_sup_u4 = h->total_sup_u4;
    hp.tie_rel = 1e-5f;
    const int max_traj = Fmax * A;
    switch (h->nw) {
        case 1: return launch_gather<1>(h, hp, max_traj, st);
        case 2: return launch_gather<2>(h, hp, max_traj, st);
        case 4: return launch_gather<4>(h, hp, max_traj, st);
        case 8: return launch_gather<8>(h, hp, max_traj, st);
        case 16: return launch_gather<16>(h, hp, max_traj, st);
        case 32: return launch_gather<32>(h, hp, max_traj, st);
        default: return fail(MPW_ERR_UNSUPPORTED, "blocklength %d unsupported", h->n);
    }
}

int finalize(mpw_handle* h, const float* y, const double* y64, int Fmax, int A, int T, S2Dev s2, FinalOut fo,
             cudaStream_t st) {
    const int grid = std::max(1, std::min((Fmax + 7) / 8, h->num_sms * 8));
    switch (h->n) {
        case 64: finalize_kernel<2><<<grid, 256, 0, st>>>(h->n, h->nw, A, T, y, y64, s2, fo, 1e-5f); break;
        case 128: finalize_kernel<4><<<grid, 256, 0, st>>>(h->n, h->nw, A, T, y, y64, s2, fo, 1e-5f); break;
        case 256: finalize_kernel<8><<<grid, 256, 0, st>>>(h->n, h->nw, A, T, y, y64, s2, fo, 1e-5f); break;
        default: finalize_kernel<0><<<grid, 256, 0, st>>>(h->n, h->nw, A, T, y, y64, s2, fo, 1e-5f); break;
    }
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

// float64 inputs: y32 = fp32(y64) into the handle's scratch (and the channel
// LLRs when llr is wanted)
int prep_y64(mpw_handle* h, const double* y64, int F, double sigma, bool llr, cudaStream_t st) {
    const size_t total = (size_t)F * h->n;
    CK(h->y32.ensure(total));
    if (llr) CK(h->llr64.ensure(total));
    const int grid = (int)std::max<size_t>(1, std::min<size_t>((total + 255) / 256, (size_t)h->num_sms * 16));
    y64_prep_kernel<<<grid, 256, 0, st>>>((long long)total, y64, h->y32.p, llr ? h->llr64.p : nullptr, sigma);
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* mpw_last_error(void) { return g_last_error.c_str(); }

int mpw_version(void) { return MPW_ABI_VERSION; }

int mpw_create(int device, mpw_handle** out) {
    if (!out) return fail(MPW_ERR_ARG, "null handle pointer");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(MPW_ERR_NO_DEVICE, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(MPW_ERR_ARG, "device %d out of range", device);
    mpw_handle* h = new mpw_handle();
    h->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        delete h;
        return fail(MPW_ERR_NO_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major, prop.minor);
    }
    h->num_sms = prop.multiProcessorCount;
    *out = h;
    return 0;
}

void mpw_destroy(mpw_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    h->info.release(); h->pivots.release(); h->frozen.release(); h->gen.release();
    h->crc_h.release(); h->mix.release(); h->pbits.release(); h->poff.release(); h->soff.release();
    h->pidx.release(); h->sup.release(); h->s2_count.release(); h->s2_frame.release();
    h->s2_nanchor.release(); h->traj_iters.release(); h->traj_hops.release(); h->work_next.release();
    h->s2_anchors.release(); h->traj_cw.release(); h->traj_flags.release(); h->ebound.release(); h->qscale.release(); h->s1_flags.release();
    h->y32.release(); h->llr64.release();
    h->hy.release(); h->htx.release(); h->hbest.release(); h->hmsg.release(); h->hed.release();
    h->hstage.release(); h->hflags.release(); h->hiters.release(); h->hctr.release();
    tc_release(h->tcp);
    if (h->ev_init) for (int i = 0; i < 8; i++) cudaEventDestroy(h->ev[i]);
    delete h;
}

int mpw_set_code(mpw_handle* h, int n, int k, int kp, const int32_t* info_set, const uint64_t* gen_words,
                 int is_ca, int crc_deg, uint32_t crc_poly) {
    if (!h || !info_set || !gen_words) return fail(MPW_ERR_ARG, "null argument");
    if (n < 2 || n > 1024) return fail(MPW_ERR_ARG, "n=%d must be in [2,1024]", n);
    if (k < 1 || kp < k || kp > n) return fail(MPW_ERR_ARG, "bad dimensions k=%d kp=%d", k, kp);
    if (k > 64) return fail(MPW_ERR_UNSUPPORTED, "k=%d > 64 is not supported on the device path", k);
    if (is_ca && (crc_deg < 1 || crc_deg > 32 || kp != k + crc_deg || kp > 64))
        return fail(MPW_ERR_ARG, "bad CRC parameters (deg=%d, k=%d, kp=%d)", crc_deg, k, kp);
    for (int i = 0; i < kp; i++)
        if (info_set[i] < 0 || info_set[i] >= n || (i && info_set[i] <= info_set[i - 1]))
            return fail(MPW_ERR_ARG, "info set must be ascending in [0,n)");
    if (set_device(h)) return MPW_ERR_CUDA;
    const int w64 = (n + 63) / 64, nw = (n + 31) / 32;
    h->n = n; h->m = __builtin_ctz(n); h->nw = nw; h->k = k; h->kp = kp; h->is_ca = is_ca; h->crc_deg = crc_deg;
    // frozen mask
    std::vector<uint32_t> frozen(nw, 0);
    for (int i = 0; i < n; i++) frozen[i >> 5] |= 1u << (i & 31);
    for (int i = 0; i < kp; i++) frozen[info_set[i] >> 5] &= ~(1u << (info_set[i] & 31));
    // generator as uint32 words
    std::vector<uint32_t> gen((size_t)k * nw, 0);
    for (int r = 0; r < k; r++)
        for (int j = 0; j < n; j++)
            if ((gen_words[(size_t)r * w64 + (j >> 6)] >> (j & 63)) & 1ull) gen[(size_t)r * nw + (j >> 5)] |= 1u << (j & 31);
    // CRC syndrome masks: v read MSB-first, remainder bit j = parity(v & H[j])
    std::vector<uint64_t> crc_h(std::max(crc_deg, 1), 0);
    if (is_ca) {
        for (int i = 0; i < kp; i++) {
            // r_i = x^(kp-1-i) mod g(x)
            uint64_t r = 1;  // polynomial, bit t = coeff x^t
            for (int e = 0; e < kp - 1 - i; e++) {
                r <<= 1;
                if ((r >> crc_deg) & 1ull) r ^= (uint64_t)crc_poly;
            }
            for (int j = 0; j < crc_deg; j++)
                if ((r >> j) & 1ull) crc_h[j] |= 1ull << i;
        }
    }
    // message_of tables: reduce [G | I] (codebook.py:104-117)
    const int W = n + k;
    std::vector<std::vector<uint8_t>> aug(k, std::vector<uint8_t>(W, 0));
    for (int r = 0; r < k; r++) {
        for (int j = 0; j < n; j++) aug[r][j] = (uint8_t)((gen_words[(size_t)r * w64 + (j >> 6)] >> (j & 63)) & 1ull);
        aug[r][n + r] = 1;
    }
    std::vector<int32_t> piv;
    int rank = 0;
    for (int col = 0; col < n && rank < k; col++) {
        int p = -1;
        for (int r = rank; r < k; r++) if (aug[r][col]) { p = r; break; }
        if (p < 0) continue;
        std::swap(aug[p], aug[rank]);
        for (int r = 0; r < k; r++)
            if (r != rank && aug[r][col])
                for (int j = 0; j < W; j++) aug[r][j] ^= aug[rank][j];
        piv.push_back(col);
        rank++;
    }
    if (rank != k) return fail(MPW_ERR_ARG, "generator rank %d < k=%d", rank, k);
    std::vector<uint64_t> mix(k, 0);
    for (int r = 0; r < k; r++)
        for (int j = 0; j < k; j++)
            if (aug[r][n + j]) mix[r] |= 1ull << j;

    CK(h->info.ensure(kp)); CK(h->frozen.ensure(nw)); CK(h->gen.ensure((size_t)k * nw));
    CK(h->crc_h.ensure(crc_h.size())); CK(h->pivots.ensure(k)); CK(h->mix.ensure(k));
    CK(cudaMemcpy(h->info.p, info_set, sizeof(int32_t) * kp, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->frozen.p, frozen.data(), sizeof(uint32_t) * nw, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->gen.p, gen.data(), sizeof(uint32_t) * gen.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->crc_h.p, crc_h.data(), sizeof(uint64_t) * crc_h.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->pivots.p, piv.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->mix.p, mix.data(), sizeof(uint64_t) * k, cudaMemcpyHostToDevice));
    h->has_code = true;
    h->has_pat = false;   // patterns must match the blocklength
    return 0;
}

int mpw_set_patterns(mpw_handle* h, const uint64_t* pattern_words, int np) {
    if (!h || (!pattern_words && np > 0) || np < 0) return fail(MPW_ERR_ARG, "bad pattern arguments");
    if (!h->has_code) return fail(MPW_ERR_STATE, "mpw_set_code must be called before mpw_set_patterns");
    if (set_device(h)) return MPW_ERR_CUDA;
    const int n = h->n, nw = h->nw, w64 = (n + 63) / 64;
    std::vector<uint32_t> bits((size_t)np * nw, 0);
    std::vector<int32_t> off(np + 1, 0), soff(np + 1, 0);
    std::vector<uint16_t> idx;
    std::vector<uint16_t> sup;
    for (int p = 0; p < np; p++) {
        off[p] = (int32_t)idx.size();
        soff[p] = (int32_t)(sup.size() / 8);
        int w = 0;
        for (int j = 0; j < n; j++)
            if ((pattern_words[(size_t)p * w64 + (j >> 6)] >> (j & 63)) & 1ull) {
                bits[(size_t)p * nw + (j >> 5)] |= 1u << (j & 31);
                idx.push_back((uint16_t)j);
                sup.push_back((uint16_t)j);
                w++;
            }
        if (w == 0) return fail(MPW_ERR_ARG, "pattern %d is the zero word (exclude member 0)", p);
        while (sup.size() % 8) sup.push_back((uint16_t)n);   // index n = zero row
    }
    off[np] = (int32_t)idx.size();
    soff[np] = (int32_t)(sup.size() / 8);
    h->np = np;
    h->total_sup_u4 = (int)(sup.size() / 8);
    h->wmax = 0;
    for (int p = 0; p < np; p++) h->wmax = std::max(h->wmax, off[p + 1] - off[p]);
    CK(h->pbits.ensure(bits.size())); CK(h->poff.ensure(off.size())); CK(h->soff.ensure(soff.size()));
    CK(h->pidx.ensure(std::max<size_t>(idx.size(), 1))); CK(h->sup.ensure(std::max<size_t>(sup.size() / 8, 1)));
    if (np) {
        CK(cudaMemcpy(h->pbits.p, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->pidx.p, idx.data(), sizeof(uint16_t) * idx.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->sup.p, sup.data(), sizeof(uint16_t) * sup.size(), cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(h->poff.p, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->soff.p, soff.data(), sizeof(int32_t) * soff.size(), cudaMemcpyHostToDevice));
    tc_release(h->tcp);
    if (tc_supported(n, np)) {
        if (tc_build(h->tcp, bits.data(), np, n, nw)) return fail(MPW_ERR_CUDA, "building the tensor-core operand failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    h->has_pat = true;
    return 0;
}

int mpw_scl_batch(mpw_handle* h, const float* y, const double* llr, int F, double sigma, int L,
                  int32_t* list_n, uint32_t* list_u, uint32_t* list_cw, double* list_pm, void* stream) {
    if (!h || F < 0) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y && !llr) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code) return fail(MPW_ERR_STATE, "no code set");
    if (L < 1 || L > SCL_MAX_L) return fail(MPW_ERR_UNSUPPORTED, "list size %d outside [1,%d]", L, SCL_MAX_L);
    if (F == 0) return 0;
    if (set_device(h)) return MPW_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    SclOut out{list_n, list_u, list_cw, list_pm, nullptr, nullptr, nullptr};
    S2Dev s2{};
    return dispatch_scl(h, y, llr, F, sigma, L, 0, 0, out, s2, st);
}

extern "C++" {
namespace {
int mpwsd_impl(mpw_handle* h, const float* y, const double* y64, const uint32_t* anchors, const int32_t* n_anchor,
               int F, int A, int T, int variant, uint32_t* best, double* best_ed, int32_t* iters, int32_t* hops,
               uint8_t* flags, cudaStream_t st) {
    if (!h->has_pat) return fail(MPW_ERR_STATE, "no pattern set");
    if (set_device(h)) return MPW_ERR_CUDA;
    if (y64) {
        if (int rc = prep_y64(h, y64, F, 1.0, false, st)) return rc;
        y = h->y32.p;
    }
    if (int rc = ensure_s2(h, F, A, T, hops != nullptr)) return rc;
    S2Dev s2 = s2_dev(h, anchors, hops != nullptr);
    CK(cudaMemsetAsync(s2.work_next, 0, sizeof(int32_t), st));
    const bool need_eb = needs_fp_bounds(resolve_variant(h, variant, y64 != nullptr));
    MPW_BY_CNT(h->n, (queue_identity_kernel<CNT><<<(F + 7) / 8, 256, 0, st>>>(F, A, h->n, y, y64, n_anchor, s2, need_eb)));
    CK(cudaGetLastError());
    h->kernel_launches++;
    if (int rc = run_hops(h, y, y64, F, A, T, variant, s2, st)) return rc;
    FinalOut fo{best, best_ed, nullptr, iters, hops, nullptr, flags, nullptr};
    return finalize(h, y, y64, F, A, T, s2, fo, st);
}
}  // namespace
}  // extern "C++"

int mpw_mpwsd_batch(mpw_handle* h, const float* y, const uint32_t* anchors, const int32_t* n_anchor,
                    int F, int A, int T, int variant, uint32_t* best, double* best_ed,
                    int32_t* iters, int32_t* hops, uint8_t* flags, void* stream) {
    if (!h || F < 0 || A < 1 || T < 1) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !anchors || !best || !best_ed) return fail(MPW_ERR_ARG, "bad arguments");
    return mpwsd_impl(h, y, nullptr, anchors, n_anchor, F, A, T, variant, best, best_ed, iters, hops, flags,
                      (cudaStream_t)stream);
}

int mpw_mpwsd_batch_f64(mpw_handle* h, const double* y, const uint32_t* anchors, const int32_t* n_anchor,
                        int F, int A, int T, int variant, uint32_t* best, double* best_ed,
                        int32_t* iters, int32_t* hops, uint8_t* flags, void* stream) {
    if (!h || F < 0 || A < 1 || T < 1) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !anchors || !best || !best_ed) return fail(MPW_ERR_ARG, "bad arguments");
    return mpwsd_impl(h, nullptr, y, anchors, n_anchor, F, A, T, variant, best, best_ed, iters, hops, flags,
                      (cudaStream_t)stream);
}

extern "C++" {
namespace {

struct Stage1 {
    int osd;                 // 0: CA-SCL (list size L), 1: OSD (order, list cap)
    double sigma;
    int L, order, cap;
};

long long osd_candidates(int K, int order) {
    long long c = 0, b = 1;
    for (int w = 0; w <= order && w <= K; w++) {
        c += b;
        b = b * (K - w) / (w + 1);
    }
    return c;
}

template <int NW>
int launch_osd_nw(mpw_handle* h, const OsdArgs& a, cudaStream_t st) {
    const size_t smem = osd_smem_bytes(h->n, NW);
    CK(cudaFuncSetAttribute(osd_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, osd_kernel<NW>, 32 * OSD_WARPS, smem));
    const int grid = std::max(1, std::min((a.F + OSD_WARPS - 1) / OSD_WARPS, h->num_sms * std::max(per_sm, 1)));
    osd_kernel<NW><<<grid, 32 * OSD_WARPS, smem, st>>>(a);
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

int launch_osd(mpw_handle* h, const OsdArgs& a, cudaStream_t st) {
    switch (h->nw) {
        case 1: return launch_osd_nw<1>(h, a, st);
        case 2: return launch_osd_nw<2>(h, a, st);
        case 4: return launch_osd_nw<4>(h, a, st);
        case 8: return launch_osd_nw<8>(h, a, st);
    }
    return fail(MPW_ERR_UNSUPPORTED, "OSD needs n in {32, 64, 128, 256}");
}

int osd_check(mpw_handle* h, int order) {
    if (order < 0) return fail(MPW_ERR_ARG, "order must be >= 0");
    if (h->k > OSD_MAX_K || order > OSD_MAX_ORDER)
        return fail(MPW_ERR_UNSUPPORTED, "OSD supports k <= %d and order <= %d", OSD_MAX_K, OSD_MAX_ORDER);
    if (h->nw != 1 && h->nw != 2 && h->nw != 4 && h->nw != 8)
        return fail(MPW_ERR_UNSUPPORTED, "OSD needs n in {32, 64, 128, 256}");
    if (osd_candidates(h->k, order) > (1ll << 31) - 1) return fail(MPW_ERR_UNSUPPORTED, "too many OSD candidates");
    return 0;
}

// y64 (may be null): float64 received words; y is then ignored and replaced by
// their fp32 rounding (screens), stage 1 runs from float64 LLRs, and the exact
// re-scoring and every reported ED use y64.
int two_stage_impl(mpw_handle* h, const float* y, const double* y64, int F, const Stage1& s1, int A, int T,
                   int mode, int variant, const uint32_t* tx_cw, uint32_t* best, uint64_t* best_msg,
                   double* best_ed, uint8_t* stage, int32_t* iters, int32_t* hops, uint32_t* anchors_out,
                   uint8_t* flags, unsigned long long* counters, cudaStream_t st) {
    if (mode != MPW_MODE_CRC_GATED && mode != MPW_MODE_ALWAYS_ON) return fail(MPW_ERR_ARG, "unknown activation mode %d", mode);
    if (mode == MPW_MODE_CRC_GATED && !h->is_ca) return fail(MPW_ERR_ARG, "crc_gated mode requires a CRC-concatenated code");
    if (y64 && s1.osd) return fail(MPW_ERR_UNSUPPORTED, "OSD stage 1 takes float32 received words");
    if (set_device(h)) return MPW_ERR_CUDA;
    if (int rc = ensure_s2(h, F, A, T, hops != nullptr)) return rc;
    S2Dev s2 = s2_dev(h, nullptr, hops != nullptr);
    if (h->timing && !h->ev_init) {
        for (int i = 0; i < 8; i++) CK(cudaEventCreate(&h->ev[i]));
        h->ev_init = true;
    }
    CK(cudaMemsetAsync(s2.count, 0, sizeof(int32_t), st));
    CK(cudaMemsetAsync(s2.work_next, 0, sizeof(int32_t), st));
    timing_mark(h, 0, st);
    if (y64) {
        if (int rc = prep_y64(h, y64, F, s1.sigma, true, st)) return rc;
        y = h->y32.p;
    }
    SclOut out{nullptr, nullptr, nullptr, nullptr, stage, best, best_ed};
    const int smode = (mode == MPW_MODE_CRC_GATED) ? 1 : 2;
    const uint8_t* s1flags = nullptr;
    if (!s1.osd) {
        if (int rc = dispatch_scl(h, y, y64 ? h->llr64.p : nullptr, F, s1.sigma, s1.L, A, smode, out, s2, st))
            return rc;
    } else {
        CK(h->s1_flags.ensure(F));
        OsdArgs a{};
        a.code = code_dev(h); a.y = y; a.F = F; a.order = s1.order; a.mode = smode;
        a.C = osd_candidates(h->k, s1.order);
        long long M = smode == 1 ? 1 : A;
        if (s1.cap > 0) M = std::min<long long>(M, s1.cap);
        a.M = (int)std::min<long long>(M, a.C);
        a.s1flags = h->s1_flags.p; a.out = out; a.s2 = s2; a.A = A;
        if (int rc = launch_osd(h, a, st)) return rc;
        s1flags = h->s1_flags.p;
    }
    const bool need_eb = needs_fp_bounds(resolve_variant(h, variant, y64 != nullptr));
    MPW_BY_CNT(h->n, (ebound_kernel<CNT><<<std::max(1, std::min((F + 7) / 8, h->num_sms * 16)), 256, 0, st>>>(
                         h->n, y, y64, s2, need_eb)));
    CK(cudaGetLastError());
    h->kernel_launches++;
    timing_mark(h, 1, st);
    if (int rc = run_hops(h, y, y64, F, A, T, variant, s2, st)) return rc;
    timing_mark(h, 2, st);
    FinalOut fo{best, best_ed, stage, iters, hops, anchors_out, flags, nullptr};
    if (int rc = finalize(h, y, y64, F, A, T, s2, fo, st)) return rc;
    if (y64) {
        stage1_ed64_kernel<<<(F + 7) / 8, 256, 0, st>>>(F, h->n, h->nw, y64, stage, best, best_ed);
        CK(cudaGetLastError());
        h->kernel_launches++;
    }
    timing_mark(h, 3, st);
    FrameArgs fa;
    fa.F = F; fa.A = A; fa.T = T; fa.nw = h->nw; fa.k = h->k; fa.np = h->np;
    fa.best = best; fa.stage = stage; fa.tx = tx_cw; fa.iters = iters; fa.hops = hops; fa.flags = flags;
    fa.msg_out = best_msg; fa.s1flags = s1flags; fa.counters = counters; fa.pivots = h->pivots.p; fa.mix = h->mix.p;
    frame_kernel<<<(F + 255) / 256, 256, 0, st>>>(fa);
    CK(cudaGetLastError());
    h->kernel_launches++;
    timing_mark(h, 4, st);
    return timing_close(h);
}

}  // namespace
}  // extern "C++"

int mpw_two_stage_batch(mpw_handle* h, const float* y, int F, double sigma, int L, int A, int T,
                        int mode, int variant, const uint32_t* tx_cw, uint32_t* best, uint64_t* best_msg,
                        double* best_ed, uint8_t* stage, int32_t* iters, int32_t* hops,
                        uint32_t* anchors_out, uint8_t* flags, unsigned long long* counters, void* stream) {
    if (!h || F < 0 || A < 1 || T < 1) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !best || !best_ed || !stage) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code || !h->has_pat) return fail(MPW_ERR_STATE, "code and pattern set must be set first");
    if (L < 1 || L > SCL_MAX_L) return fail(MPW_ERR_UNSUPPORTED, "list size %d outside [1,%d]", L, SCL_MAX_L);
    Stage1 s1{0, sigma, L, 0, 0};
    return two_stage_impl(h, y, nullptr, F, s1, A, T, mode, variant, tx_cw, best, best_msg, best_ed, stage, iters,
                          hops, anchors_out, flags, counters, (cudaStream_t)stream);
}

int mpw_two_stage_batch_f64(mpw_handle* h, const double* y, int F, double sigma, int L, int A, int T,
                            int mode, int variant, const uint32_t* tx_cw, uint32_t* best, uint64_t* best_msg,
                            double* best_ed, uint8_t* stage, int32_t* iters, int32_t* hops,
                            uint32_t* anchors_out, uint8_t* flags, unsigned long long* counters, void* stream) {
    if (!h || F < 0 || A < 1 || T < 1) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !best || !best_ed || !stage) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code || !h->has_pat) return fail(MPW_ERR_STATE, "code and pattern set must be set first");
    if (L < 1 || L > SCL_MAX_L) return fail(MPW_ERR_UNSUPPORTED, "list size %d outside [1,%d]", L, SCL_MAX_L);
    Stage1 s1{0, sigma, L, 0, 0};
    return two_stage_impl(h, nullptr, y, F, s1, A, T, mode, variant, tx_cw, best, best_msg, best_ed, stage, iters,
                          hops, anchors_out, flags, counters, (cudaStream_t)stream);
}

int mpw_two_stage_osd_batch(mpw_handle* h, const float* y, int F, int order, int list_cap, int A, int T,
                            int mode, int variant, const uint32_t* tx_cw, uint32_t* best, uint64_t* best_msg,
                            double* best_ed, uint8_t* stage, int32_t* iters, int32_t* hops,
                            uint32_t* anchors_out, uint8_t* flags, unsigned long long* counters, void* stream) {
    if (!h || F < 0 || A < 1 || T < 1) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !best || !best_ed || !stage) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code || !h->has_pat) return fail(MPW_ERR_STATE, "code and pattern set must be set first");
    if (int rc = osd_check(h, order)) return rc;
    if (A > OSD_MAX_KEEP - 1) return fail(MPW_ERR_UNSUPPORTED, "num_paths %d > %d", A, OSD_MAX_KEEP - 1);
    Stage1 s1{1, 1.0, 0, order, list_cap};
    return two_stage_impl(h, y, nullptr, F, s1, A, T, mode, variant, tx_cw, best, best_msg, best_ed, stage, iters,
                          hops, anchors_out, flags, counters, (cudaStream_t)stream);
}

extern "C++" {
namespace {
__global__ void osd_iota_kernel(int32_t* v, int32_t* offs, long long C, int F) {
    const long long total = C * F;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
        v[i] = (int32_t)(i % C);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= F) offs[t] = (int32_t)(C * t);
}

template <int NW>
int osd_full_list(mpw_handle* h, OsdArgs a, cudaStream_t st) {
    const size_t total = (size_t)a.F * (size_t)a.C;
    DevBuf<double> keys, keys_out;
    DevBuf<int32_t> vals, vals_out, offs;
    DevBuf<uint32_t> basis;
    DevBuf<unsigned char> temp;
    auto cleanup = [&]() { keys.release(); keys_out.release(); vals.release(); vals_out.release(); offs.release();
                           basis.release(); temp.release(); };
    cudaError_t e;
    if ((e = keys.ensure(total)) || (e = keys_out.ensure(total)) || (e = vals.ensure(total)) ||
        (e = vals_out.ensure(total)) || (e = offs.ensure(a.F + 1)) ||
        (e = basis.ensure((size_t)a.F * (h->k + 1) * NW))) {
        cleanup();
        return fail(MPW_ERR_CUDA, "allocation: %s", cudaGetErrorString(e));
    }
    a.keys = keys.p; a.basis = basis.p;
    if (int rc = launch_osd_nw<NW>(h, a, st)) { cleanup(); return rc; }
    osd_iota_kernel<<<std::max(1, std::min<int>((int)((total + 255) / 256), h->num_sms * 8)), 256, 0, st>>>(
        vals.p, offs.p, a.C, a.F);
    h->kernel_launches++;
    if (a.F + 1 > h->num_sms * 8 * 256) { cleanup(); return fail(MPW_ERR_UNSUPPORTED, "batch too large"); }
    size_t tb = 0;
    e = cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, keys.p, keys_out.p, vals.p, vals_out.p, (int)total,
                                                   a.F, offs.p, offs.p + 1, st);
    if (e == cudaSuccess) e = temp.ensure(tb);
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::StableSortPairs(temp.p, tb, keys.p, keys_out.p, vals.p, vals_out.p,
                                                       (int)total, a.F, offs.p, offs.p + 1, st);
    if (e == cudaSuccess) {
        const int grid = std::max(1, std::min((a.F + OSD_WARPS - 1) / OSD_WARPS, h->num_sms * 4));
        osd_materialize_kernel<NW><<<grid, 32 * OSD_WARPS, 0, st>>>(a, vals_out.p, keys_out.p);
        e = cudaGetLastError();
        h->kernel_launches++;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);    // scratch is freed below
    cleanup();
    if (e != cudaSuccess) return fail(MPW_ERR_CUDA, "OSD full list: %s", cudaGetErrorString(e));
    return 0;
}
}  // namespace
}  // extern "C++"

int mpw_osd_batch(mpw_handle* h, const float* y, int F, int order, int list_cap, int32_t* list_n,
                  uint32_t* list_cw, double* list_ed, uint8_t* flags, void* stream) {
    if (!h || F < 0) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y || !list_n || !list_cw || !list_ed) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code) return fail(MPW_ERR_STATE, "no code set");
    if (int rc = osd_check(h, order)) return rc;
    if (set_device(h)) return MPW_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    OsdArgs a{};
    a.code = code_dev(h); a.y = y; a.F = F; a.order = order; a.mode = 0;
    a.C = osd_candidates(h->k, order);
    a.M = (int)(list_cap > 0 ? std::min<long long>(list_cap, a.C) : a.C);
    a.list_n = list_n; a.list_cw = list_cw; a.list_ed = list_ed; a.s1flags = flags;
    if (a.M + 1 <= OSD_MAX_KEEP) return launch_osd(h, a, st);
    if ((long long)F * a.C > (1ll << 28)) return fail(MPW_ERR_UNSUPPORTED, "full OSD lists limited to F*C <= 2^28");
    switch (h->nw) {
        case 1: return osd_full_list<1>(h, a, st);
        case 2: return osd_full_list<2>(h, a, st);
        case 4: return osd_full_list<4>(h, a, st);
        default: return osd_full_list<8>(h, a, st);
    }
}

int mpw_two_stage_batch_host(mpw_handle* h, const float* y_host, int F, double sigma, int L, int A, int T,
                             int mode, int variant, const uint32_t* tx_host, uint32_t* best_host,
                             uint64_t* msg_host, double* ed_host, uint8_t* stage_host, int32_t* iters_host,
                             uint8_t* flags_host, unsigned long long* counters_host, void* stream) {
    if (!h || F < 0) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y_host) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (set_device(h)) return MPW_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int n = h->n, nw = h->nw;
    // staging buffers owned by the handle (allocated on its device)
    DevBuf<float>& dy = h->hy;
    DevBuf<uint32_t>&dtx = h->htx, &dbest = h->hbest;
    DevBuf<uint64_t>& dmsg = h->hmsg;
    DevBuf<double>& ded = h->hed;
    DevBuf<uint8_t>&dstage = h->hstage, &dflags = h->hflags;
    DevBuf<int32_t>& diters = h->hiters;
    DevBuf<unsigned long long>& dctr = h->hctr;
    CK(dy.ensure((size_t)F * n)); CK(dbest.ensure((size_t)F * nw)); CK(dmsg.ensure(F)); CK(ded.ensure(F));
    CK(dstage.ensure(F)); CK(dflags.ensure(F)); CK(diters.ensure((size_t)F * A)); CK(dctr.ensure(MPW_NUM_COUNTERS));
    CK(cudaMemcpyAsync(dy.p, y_host, sizeof(float) * (size_t)F * n, cudaMemcpyHostToDevice, st));
    if (tx_host) {
        CK(dtx.ensure((size_t)F * nw));
        CK(cudaMemcpyAsync(dtx.p, tx_host, sizeof(uint32_t) * (size_t)F * nw, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemsetAsync(dctr.p, 0, sizeof(unsigned long long) * MPW_NUM_COUNTERS, st));
    int rc = mpw_two_stage_batch(h, dy.p, F, sigma, L, A, T, mode, variant, tx_host ? dtx.p : nullptr, dbest.p,
                                 dmsg.p, ded.p, dstage.p, diters.p, nullptr, nullptr, dflags.p, dctr.p, stream);
    if (rc) return rc;
    if (best_host) CK(cudaMemcpyAsync(best_host, dbest.p, sizeof(uint32_t) * (size_t)F * nw, cudaMemcpyDeviceToHost, st));
    if (msg_host) CK(cudaMemcpyAsync(msg_host, dmsg.p, sizeof(uint64_t) * F, cudaMemcpyDeviceToHost, st));
    if (ed_host) CK(cudaMemcpyAsync(ed_host, ded.p, sizeof(double) * F, cudaMemcpyDeviceToHost, st));
    if (stage_host) CK(cudaMemcpyAsync(stage_host, dstage.p, F, cudaMemcpyDeviceToHost, st));
    if (iters_host) CK(cudaMemcpyAsync(iters_host, diters.p, sizeof(int32_t) * (size_t)F * A, cudaMemcpyDeviceToHost, st));
    if (flags_host) CK(cudaMemcpyAsync(flags_host, dflags.p, F, cudaMemcpyDeviceToHost, st));
    if (counters_host) CK(cudaMemcpyAsync(counters_host, dctr.p, sizeof(unsigned long long) * MPW_NUM_COUNTERS, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int mpw_channel_batch(mpw_handle* h, uint64_t seed, int snr_idx, long long first_frame, int F, double sigma,
                      float* y, uint32_t* tx, uint64_t* msg, void* stream) {
    if (!h || F < 0 || first_frame < 0 || !(sigma > 0)) return fail(MPW_ERR_ARG, "bad arguments");
    if (F == 0) return 0;
    if (!y) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code) return fail(MPW_ERR_STATE, "no code set");
    if (set_device(h)) return MPW_ERR_CUDA;
    ChannelArgs a;
    a.code = code_dev(h); a.seed = seed; a.snr_idx = (uint32_t)snr_idx; a.first_frame = first_frame;
    a.F = F; a.sigma = sigma; a.y = y; a.tx = tx; a.msg = msg;
    const int grid = std::max(1, std::min((F + 7) / 8, h->num_sms * 32));
    channel_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
    CK(cudaGetLastError());
    h->kernel_launches++;
    return 0;
}

extern "C++" {
namespace {
template <int NW>
cudaError_t launch_enum(const mpw_handle* h, int lb, const uint32_t* table, int cap, unsigned long long* spec,
                        uint32_t* out, unsigned long long* cnt, long long out_cap) {
    const size_t smem = ((size_t)NW << lb) * 4 + (size_t)(h->n + 1) * 4;
    cudaError_t e = cudaFuncSetAttribute(enum_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long nhigh = 1ll << (h->k - lb);
    const long long want = (nhigh + 255) / 256;
    const int grid = (int)std::max(1ll, std::min<long long>(want, (long long)h->num_sms * 8));
    enum_kernel<NW><<<grid, 256, smem>>>(h->gen.p, h->k, h->n, lb, table, nhigh, cap, spec, out, cnt, out_cap);
    const_cast<mpw_handle*>(h)->kernel_launches++;
    return cudaGetLastError();
}
}  // namespace
}  // extern "C++"

int64_t mpw_enumerate_lowweight_gpu(mpw_handle* h, int cap, int64_t* spectrum, uint64_t* out, int64_t out_cap) {
    if (!h || cap < 0 || out_cap < 0 || (out_cap > 0 && !out)) return fail(MPW_ERR_ARG, "bad arguments");
    if (!h->has_code) return fail(MPW_ERR_STATE, "no code set");
    if (h->k > 40) return fail(MPW_ERR_UNSUPPORTED, "exhaustive enumeration needs k <= 40 (k=%d)", h->k);
    const int nw = h->nw;
    if (nw != 1 && nw != 2 && nw != 4 && nw != 8) return fail(MPW_ERR_UNSUPPORTED, "n=%d", h->n);
    if (set_device(h)) return MPW_ERR_CUDA;
    const int lb = std::min(h->k, ENUM_LB);
    // doubling table of the low lb generator rows (wsphere.py:115-121)
    std::vector<uint32_t> gen((size_t)h->k * nw);
    CK(cudaMemcpy(gen.data(), h->gen.p, gen.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> table((size_t)nw << lb, 0u);
    for (int e = 1; e < (1 << lb); e++) {
        const int b = __builtin_ctz(e);
        for (int w = 0; w < nw; w++) table[(size_t)e * nw + w] = table[(size_t)(e & (e - 1)) * nw + w] ^ gen[(size_t)b * nw + w];
    }
    DevBuf<uint32_t> dtab, dout;
    DevBuf<unsigned long long> dspec, dcnt;
    const long long dcap = std::max<long long>(out_cap, 1);
    auto cleanup = [&]() { dtab.release(); dout.release(); dspec.release(); dcnt.release(); };
    cudaError_t e = cudaSuccess;
    if ((e = dtab.ensure(table.size())) != cudaSuccess || (e = dout.ensure((size_t)dcap * nw)) != cudaSuccess ||
        (e = dspec.ensure(h->n + 1)) != cudaSuccess || (e = dcnt.ensure(1)) != cudaSuccess) {
        cleanup();
        return fail(MPW_ERR_CUDA, "allocation: %s", cudaGetErrorString(e));
    }
    cudaMemcpy(dtab.p, table.data(), table.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dspec.p, 0, (h->n + 1) * sizeof(unsigned long long));
    cudaMemset(dcnt.p, 0, sizeof(unsigned long long));
    switch (nw) {
        case 1: e = launch_enum<1>(h, lb, dtab.p, cap, dspec.p, dout.p, dcnt.p, out_cap); break;
        case 2: e = launch_enum<2>(h, lb, dtab.p, cap, dspec.p, dout.p, dcnt.p, out_cap); break;
        case 4: e = launch_enum<4>(h, lb, dtab.p, cap, dspec.p, dout.p, dcnt.p, out_cap); break;
        default: e = launch_enum<8>(h, lb, dtab.p, cap, dspec.p, dout.p, dcnt.p, out_cap); break;
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long cnt = 0;
    std::vector<unsigned long long> spec(h->n + 1);
    if (e == cudaSuccess) e = cudaMemcpy(&cnt, dcnt.p, sizeof(cnt), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(spec.data(), dspec.p, spec.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> words;
    const long long got = std::min<long long>((long long)cnt, out_cap);
    if (e == cudaSuccess && got > 0) {
        words.resize((size_t)got * nw);
        e = cudaMemcpy(words.data(), dout.p, words.size() * 4, cudaMemcpyDeviceToHost);
    }
    cleanup();
    if (e != cudaSuccess) return fail(MPW_ERR_CUDA, "enumeration: %s", cudaGetErrorString(e));
    if (spectrum)
        for (int i = 0; i <= h->n; i++) spectrum[i] = (int64_t)spec[i];
    const int w64 = (h->n + 63) / 64;
    for (long long r = 0; r < got; r++)
        for (int w = 0; w < w64; w++) {
            const uint64_t lo = words[(size_t)r * nw + 2 * w];
            const uint64_t hi = 2 * w + 1 < nw ? words[(size_t)r * nw + 2 * w + 1] : 0u;
            out[(size_t)r * w64 + w] = lo | (hi << 32);
        }
    return (int64_t)cnt;
}

int mpw_set_option(mpw_handle* h, const char* key, int value) {
    if (!h || !key) return fail(MPW_ERR_ARG, "null argument");
    if (!strcmp(key, "scl_generic")) { h->scl_generic = value ? 1 : 0; return 0; }
    if (!strcmp(key, "timing")) { h->timing = value ? 1 : 0; return 0; }
    // tensor-hop launch options (TcOpts): A/B variants and test hooks
    if (!strcmp(key, "hop_experiment")) { h->tco.experiment = value; return 0; }
    if (!strcmp(key, "i8_pair")) { h->tco.i8_pair = value ? 1 : 0; return 0; }
    if (!strcmp(key, "i8_cluster")) {
        if (value != 1 && value != 2) return fail(MPW_ERR_ARG, "i8_cluster must be 1 or 2");
        h->tco.i8_cluster = value;
        return 0;
    }
    if (!strcmp(key, "f16_cluster")) { h->tco.f16_cluster = value ? 1 : 0; return 0; }
    if (!strcmp(key, "ar_hit_cap")) {   // asynchronous-row hop: hit-list entries per scan thread and cycle (tests: small values force re-scans)
        if (value < 0 || value > 30) return fail(MPW_ERR_ARG, "ar_hit_cap must be 0 (default) .. 30");
        h->tco.ar_hit_cap = value;
        return 0;
    }
    return fail(MPW_ERR_ARG, "unknown option '%s'", key);
}

int mpw_set_timing(mpw_handle* h, int enable) {
    if (!h) return fail(MPW_ERR_ARG, "null handle");
    h->timing = enable ? 1 : 0;
    return 0;
}

int mpw_read_timing(mpw_handle* h, double* ms_out /*4*/, long long* launches_out /*4*/, int reset) {
    if (!h) return fail(MPW_ERR_ARG, "null handle");
    for (int i = 0; i < 4; i++) {
        if (ms_out) ms_out[i] = h->acc_ms[i];
        if (launches_out) launches_out[i] = h->launches[i];
        if (reset) { h->acc_ms[i] = 0; h->launches[i] = 0; }
    }
    return 0;
}

int mpw_hop_tile_stats(mpw_handle* h, unsigned long long* out /*2*/, int reset) {
    if (!h || !out) return fail(MPW_ERR_ARG, "null argument");
    out[0] = out[1] = 0;
    if (!h->tcp.ar_stat) return 0;
    if (set_device(h)) return MPW_ERR_CUDA;
    CK(cudaMemcpy(out, h->tcp.ar_stat, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (reset) CK(cudaMemset(h->tcp.ar_stat, 0, 2 * sizeof(unsigned long long)));
    return 0;
}

int mpw_num_patterns(mpw_handle* h) { return h ? h->np : -1; }

long long mpw_launch_count(mpw_handle* h) { return h ? h->kernel_launches : -1; }

int mpw_tensor_path_ready(mpw_handle* h) { return (h && h->tcp.ready) ? 1 : 0; }

int mpw_hop_auto_variant(mpw_handle* h) { return h ? resolve_variant(h, MPW_HOP_AUTO) : MPW_ERR_ARG; }

}  // extern "C"
