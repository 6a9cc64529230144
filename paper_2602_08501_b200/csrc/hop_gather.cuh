// Stage 2, CUDA-core variant: MP-WSD hop by shared-memory gather-sum.
//
// Lanes over trajectories (SURVEY.md §7 layout G2): one warp owns 32
// (frame, anchor) trajectories; t = x ⊙ y lives in shared memory transposed,
// t[i][lane], so every lane's read of position i hits its own bank.  The
// pattern loop is warp-uniform: supports are broadcast 8 indices per 16-byte
// load (padded with index n -> a zero row), each lane accumulates
//   S_p = Σ_{i∈supp p} t_i ,   ΔED_p = 4·S_p   (decoders.py:329-336, 353-357)
// and keeps the running argmin (first index wins ties, decoders.py:391) plus
// the runner-up for the near-tie report.  A move flips t on the chosen
// support; a scan that does not strictly improve ends the trajectory and is
// counted (decoders.py:395-398, 441-451).
#pragma once
#include "common.cuh"

struct HopParams {
    int n, nw, A, T;
    const float* y;
    const double* y64;     // float64 inputs: the caller's received words (y = their fp32 rounding), else null
    S2Dev s2;
    PatDev P;
    const uint4* sup;      // padded supports, 8 x uint16 per uint4
    const int32_t* soff;   // np + 1 offsets in uint4 units
    int sup_in_smem;       // supports + offsets cached in shared memory
    int total_sup_u4;
    float tie_rel;         // near-tie threshold (relative), 1e-5
};

__host__ __device__ inline size_t gather_warp_smem(int n) { return sizeof(float) * (size_t)(n + 1) * 32; }

template <int NW>
__global__ void __launch_bounds__(256) hop_gather_kernel(HopParams hp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int n = hp.n, nw = hp.nw, A = hp.A, T = hp.T, np_ = hp.P.np;

    const uint4* sup = hp.sup;
    const int32_t* soff = hp.soff;
    size_t off_bytes = 0;
    if (hp.sup_in_smem) {
        uint4* ssup = reinterpret_cast<uint4*>(smem_raw);
        for (int i = threadIdx.x; i < hp.total_sup_u4; i += blockDim.x) ssup[i] = hp.sup[i];
        int32_t* soffs = reinterpret_cast<int32_t*>(ssup + hp.total_sup_u4);
        for (int i = threadIdx.x; i <= np_; i += blockDim.x) soffs[i] = hp.soff[i];
        sup = ssup; soff = soffs;
        off_bytes = ((sizeof(uint4) * (size_t)hp.total_sup_u4 + sizeof(int32_t) * (size_t)(np_ + 1)) + 15) & ~(size_t)15;
        __syncthreads();
    }
    float* t = reinterpret_cast<float*>(smem_raw + off_bytes) + (size_t)wib * (n + 1) * 32;
    t[n * 32 + lane] = 0.0f;   // padding row

    const int count = *hp.s2.count;
    const long long ntraj = (long long)count * A;
    const long long ntask = (ntraj + 31) / 32;
    for (long long task = (long long)blockIdx.x * wpb + wib; task < ntask; task += (long long)gridDim.x * wpb) {
        const long long tr = task * 32 + lane;
        const int q = (int)(tr / A), a = (int)(tr % A);
        const bool valid = tr < ntraj && a < hp.s2.nanchor[q < count ? q : 0];
        uint32_t c[NW];
        float ed = 0.0f;
        const int f = valid ? hp.s2.frame[q] : 0;
        const float err_row = valid ? hp.s2.ebound[q].z : 0.0f;
#pragma unroll
        for (int w = 0; w < NW; w++) c[w] = (valid && w < nw) ? hp.s2.anchors[(size_t)tr * nw + w] : 0u;
#pragma unroll
        for (int w = 0; w < NW; w++) {
            if (w >= nw) break;
            for (int b = 0; b < 32 && w * 32 + b < n; b++) {
                const int i = w * 32 + b;
                const float yi = valid ? hp.y[(size_t)f * n + i] : 0.0f;
                const float xi = ((c[w] >> b) & 1u) ? -1.0f : 1.0f;
                t[i * 32 + lane] = xi * yi;
                const float d = yi - xi;
                ed = fmaf(d, d, ed);
            }
        }
        __syncwarp();
        bool active = valid;
        int iters = 0;
        uint8_t flags = 0;
        for (int h = 0; h < T; h++) {
            if (!__any_sync(MPW_FULL, active)) break;
            TopK<4> top;
            top.reset();
            for (int p = 0; p < np_; p++) {
                const int q0 = soff[p], q1 = soff[p + 1];
                float s0 = 0.0f, s1 = 0.0f;
                for (int qq = q0; qq < q1; qq++) {
                    const uint4 v = sup[qq];
                    s0 += t[(v.x & 0xffffu) * 32 + lane];
                    s1 += t[(v.x >> 16) * 32 + lane];
                    s0 += t[(v.y & 0xffffu) * 32 + lane];
                    s1 += t[(v.y >> 16) * 32 + lane];
                    s0 += t[(v.z & 0xffffu) * 32 + lane];
                    s1 += t[(v.z >> 16) * 32 + lane];
                    s0 += t[(v.w & 0xffffu) * 32 + lane];
                    s1 += t[(v.w >> 16) * 32 + lane];
                }
                top.push(s0 + s1, p);
            }
            if (active) {
                iters++;
                int i1;
                bool improve;
                float sb;
                certify_topk<4, NW>(top, hp.y + (size_t)f * n, hp.y64 ? hp.y64 + (size_t)f * n : nullptr, c,
                                    hp.P.bits, nw, n, ed, hp.tie_rel, err_row, i1, improve, sb, flags);
                if (improve) {
                    for (int qq = soff[i1]; qq < soff[i1 + 1]; qq++) {
                        const uint4 v = sup[qq];
                        const uint32_t ids[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int i0 = ids[e] & 0xffffu, i1_ = ids[e] >> 16;
                            if (i0 < n) t[i0 * 32 + lane] = -t[i0 * 32 + lane];
                            if (i1_ < n) t[i1_ * 32 + lane] = -t[i1_ * 32 + lane];
                        }
                    }
#pragma unroll
                    for (int w = 0; w < NW; w++) if (w < nw) c[w] ^= hp.P.bits[(size_t)i1 * nw + w];
                    ed += 4.0f * sb;
                    if (hp.s2.traj_hops) hp.s2.traj_hops[(size_t)tr * T + h] = i1 + 1;
                } else {
                    active = false;
                }
            }
            __syncwarp();
        }
        if (valid) {
#pragma unroll
            for (int w = 0; w < NW; w++) if (w < nw) hp.s2.traj_cw[(size_t)tr * nw + w] = c[w];
            hp.s2.traj_iters[tr] = iters;
            hp.s2.traj_flags[tr] = flags;
            if (hp.s2.traj_hops) {
                // hops after the last accepted one are "none"
                int accepted = iters - (active ? 0 : 1);
                for (int h = accepted; h < T; h++) hp.s2.traj_hops[(size_t)tr * T + h] = -1;
            }
        }
        __syncwarp();
    }
}
