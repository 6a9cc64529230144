// Stage 1: batched CA-SCL, one warp per frame, float64 so that every decision
// and every path metric is bit-identical to the reference's numpy float64
// `scl_decode` (/root/reference/pkg/src/feclab/decoders.py:173-268):
//   f(a,b) = sign(a) sign(b) min(|a|,|b|)                (:173-174, exact)
//   g(a,b,u) = b + (1-2u) a                             (:177-178, one rounding)
//   frozen leaf: pm += |dm| [dm<0]                      (:216-218, one rounding)
//   info leaf:   candidates [pm, pm+|dm|], stable rank  (:219-228)
// The same IEEE operations in the same order give the same bits.
//
// Layout (per warp, shared memory):
//   llr0[n]          channel LLRs 2y/sigma^2 (decoders.py:550)
//   llr[L][n-1]      level l=1..m stored per "instance": every path writes its
//                    own instance; reads go through ptr[path][level] so that a
//                    clone at an info leaf copies m bytes instead of the
//                    arrays (all paths write a level at the same time, so the
//                    overwritten level is dead for everyone).
//   ps[L][nw]        partial-sum bits at absolute positions; live segments of
//                    different tree levels are disjoint, so one n-bit vector
//                    per path holds what the reference keeps in bit_mem[L][m+1][n].
//   u[L][nw]         leaf decisions.
// Fused epilogue: codewords (butterfly of u), CRC gate on v = u[info_set]
// (codebook.py:154-163, 287-297), projection encode(v[:K]) (decoders.py:572-579)
// and compaction of stage-2 frames into a queue.
#pragma once
#include "common.cuh"

constexpr int SCL_MAX_L = 32;
constexpr int SCL_MAX_LEVELS = 16;

struct SclOut {
    // list outputs (mode 0), any may be null
    int32_t* list_n; uint32_t* list_u; uint32_t* list_cw; double* list_pm;
    // two-stage outputs (mode 1 gated, 2 always-on)
    uint8_t* stage; uint32_t* best; double* best_ed;
};

struct SclLayout {
    size_t llr0, llr, pm, newpm, ptr, ps, u, src, bit, total;
};

__host__ __device__ inline size_t scl_align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline SclLayout scl_layout(int n, int L, int nw) {
    SclLayout o;
    o.llr0 = 0;
    o.llr = o.llr0 + sizeof(double) * (size_t)n;
    o.pm = o.llr + sizeof(double) * (size_t)L * (n - 1);
    o.newpm = o.pm + sizeof(double) * (size_t)L;
    o.ptr = scl_align16(o.newpm + sizeof(double) * (size_t)L);
    o.ps = o.ptr + (size_t)L * SCL_MAX_LEVELS;
    o.u = o.ps + sizeof(uint32_t) * (size_t)L * nw;
    o.src = o.u + sizeof(uint32_t) * (size_t)L * nw;
    o.bit = o.src + sizeof(int32_t) * (size_t)L;
    o.total = scl_align16(o.bit + sizeof(int32_t) * (size_t)L);
    return o;
}

// f(a,b) = sign(a)·sign(b)·min(|a|,|b|) with sign(0) = 0 (decoders.py:173-174),
// evaluated on the IEEE bit patterns with integer ops (exact: magnitudes of
// non-NaN doubles order like their unsigned bit patterns; a zero operand
// gives +0.0).  Keeps the float64 pipe free for the g additions.
__device__ __forceinline__ double scl_f(double a, double b) {
    const unsigned long long ia = (unsigned long long)__double_as_longlong(a);
    const unsigned long long ib = (unsigned long long)__double_as_longlong(b);
    const unsigned long long ma = ia & 0x7FFFFFFFFFFFFFFFull, mb = ib & 0x7FFFFFFFFFFFFFFFull;
    const unsigned long long mn = ma < mb ? ma : mb;
    const unsigned long long sg = (ia ^ ib) & 0x8000000000000000ull;
    return __longlong_as_double((long long)(mn ? (mn | sg) : 0ull));
}

template <int NW>
__global__ void __launch_bounds__(256) scl_kernel(CodeDev code, const float* __restrict__ y,
                                                  const double* __restrict__ llr64, int F,
                                                  double sigma, int L, int A, int mode, SclOut out,
                                                  S2Dev s2) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int n = code.n, m = code.m, nw = code.nw;
    const SclLayout lay = scl_layout(n, L, nw);
    unsigned char* base = smem_raw + lay.total * wib;
    double* llr0 = reinterpret_cast<double*>(base + lay.llr0);
    double* llr = reinterpret_cast<double*>(base + lay.llr);
    double* pm = reinterpret_cast<double*>(base + lay.pm);
    double* newpm = reinterpret_cast<double*>(base + lay.newpm);
    uint8_t* ptr = base + lay.ptr;
    uint32_t* ps = reinterpret_cast<uint32_t*>(base + lay.ps);
    uint32_t* ub = reinterpret_cast<uint32_t*>(base + lay.u);
    int32_t* src_of = reinterpret_cast<int32_t*>(base + lay.src);
    int32_t* bit_of = reinterpret_cast<int32_t*>(base + lay.bit);

    const int warps_total = gridDim.x * (blockDim.x >> 5);
    const double sig2 = sigma * sigma;
    for (int f = blockIdx.x * (blockDim.x >> 5) + wib; f < F; f += warps_total) {
        // ---- init (decoders.py:204-209)
        if (llr64) {
            for (int i = lane; i < n; i += 32) llr0[i] = llr64[(size_t)f * n + i];
        } else {
            for (int i = lane; i < n; i += 32) llr0[i] = 2.0 * (double)y[(size_t)f * n + i] / sig2;
        }
        for (int i = lane; i < L * nw; i += 32) { ps[i] = 0u; ub[i] = 0u; }
        for (int l = lane; l < L; l += 32) pm[l] = (l == 0) ? 0.0 : CUDART_INF;
        __syncwarp();

        for (int phi = 0; phi < n; phi++) {
            // ---- descend to leaf phi: g at depth m-1-t, then f down to m-1
            int dstart;
            if (phi == 0) {
                dstart = 0;
            } else {
                const int t = __ffs(phi) - 1;
                const int d = m - 1 - t;
                const int half = n >> (d + 1), lh = m - d - 1;
                const int lo = (phi >> (m - d)) << (m - d);
                const int poff = n - 2 * (n >> d), coff = n - 2 * half;
                for (int it = lane; it < L * half; it += 32) {
                    const int l = it >> lh, j = it & (half - 1);
                    const double* par = (d == 0) ? llr0 : llr + (size_t)ptr[l * SCL_MAX_LEVELS + d] * (n - 1) + poff;
                    const double a = par[j], b = par[j + half];
                    const int ubit = (ps[l * nw + ((lo + j) >> 5)] >> ((lo + j) & 31)) & 1u;
                    llr[(size_t)l * (n - 1) + coff + j] = b + (ubit ? -a : a);
                }
                for (int l = lane; l < L; l += 32) ptr[l * SCL_MAX_LEVELS + d + 1] = (uint8_t)l;
                __syncwarp();
                dstart = d + 1;
            }
            for (int d = dstart; d < m; d++) {
                const int half = n >> (d + 1), lh = m - d - 1;
                const int poff = n - 2 * (n >> d), coff = n - 2 * half;
                for (int it = lane; it < L * half; it += 32) {
                    const int l = it >> lh, j = it & (half - 1);
                    const double* par = (d == 0) ? llr0 : llr + (size_t)ptr[l * SCL_MAX_LEVELS + d] * (n - 1) + poff;
                    llr[(size_t)l * (n - 1) + coff + j] = scl_f(par[j], par[j + half]);
                }
                for (int l = lane; l < L; l += 32) ptr[l * SCL_MAX_LEVELS + d + 1] = (uint8_t)l;
                __syncwarp();
            }
            // ---- leaf phi
            double dm = 0.0, pml = CUDART_INF;
            if (lane < L) { dm = llr[(size_t)lane * (n - 1) + n - 2]; pml = pm[lane]; }
            const bool frozen = (code.frozen[phi >> 5] >> (phi & 31)) & 1u;
            if (frozen) {
                if (lane < L) pm[lane] = pml + fabs(dm) * (double)(dm < 0.0);
                __syncwarp();
            } else {
                // candidates c < L: (pm_c, natural); c >= L: (pm_{c-L} + |dm|, flipped)
                double v0 = CUDART_INF, v1 = CUDART_INF;
                const int c0 = lane, c1 = lane + 32;
                {
                    const int s = (c0 < L) ? c0 : c0 - L;
                    const double ps_ = __shfl_sync(MPW_FULL, pml, s & 31);
                    const double ds_ = __shfl_sync(MPW_FULL, dm, s & 31);
                    if (c0 < L) v0 = ps_;
                    else if (c0 < 2 * L) v0 = ps_ + fabs(ds_);
                }
                if (2 * L > 32) {
                    const int s = c1 - L;
                    const double ps_ = __shfl_sync(MPW_FULL, pml, s & 31);
                    const double ds_ = __shfl_sync(MPW_FULL, dm, s & 31);
                    if (c1 < 2 * L) v1 = ps_ + fabs(ds_);
                }
                int r0 = 0, r1 = 0;
                for (int c = 0; c < 2 * L; c++) {
                    const double vc = __shfl_sync(MPW_FULL, (c < 32) ? v0 : v1, c & 31);
                    r0 += (vc < v0) || (vc == v0 && c < c0);
                    r1 += (vc < v1) || (vc == v1 && c < c1);
                }
                const bool nat_self = dm < 0.0;
                const int natv = __ballot_sync(MPW_FULL, nat_self);
                if (c0 < 2 * L && r0 < L) {
                    const int s = c0 % L;
                    src_of[r0] = s;
                    bit_of[r0] = (int)(((natv >> s) & 1u) ^ (c0 >= L ? 1u : 0u));
                    newpm[r0] = v0;
                }
                if (c1 < 2 * L && r1 < L) {
                    const int s = c1 % L;
                    src_of[r1] = s;
                    bit_of[r1] = (int)(((natv >> s) & 1u) ^ 1u);
                    newpm[r1] = v1;
                }
                __syncwarp();
                // clone: slot j <- slot src_of[j]  (decoders.py:225-228)
                uint32_t rps[NW], ru[NW];
                uint4 rptr;
                int sj = 0, bj = 0;
                if (lane < L) {
                    sj = src_of[lane]; bj = bit_of[lane];
#pragma unroll
                    for (int w = 0; w < NW; w++) {
                        rps[w] = (w < nw) ? ps[sj * nw + w] : 0u;
                        ru[w] = (w < nw) ? ub[sj * nw + w] : 0u;
                    }
                    rptr = *reinterpret_cast<const uint4*>(ptr + sj * SCL_MAX_LEVELS);
                }
                __syncwarp();
                if (lane < L) {
                    if (bj) { rps[phi >> 5] |= 1u << (phi & 31); ru[phi >> 5] |= 1u << (phi & 31); }
#pragma unroll
                    for (int w = 0; w < NW; w++)
                        if (w < nw) { ps[lane * nw + w] = rps[w]; ub[lane * nw + w] = ru[w]; }
                    *reinterpret_cast<uint4*>(ptr + lane * SCL_MAX_LEVELS) = rptr;
                    pm[lane] = newpm[lane];
                }
                __syncwarp();
            }
            if (phi == n - 1) break;
            // ---- combine up through the trailing ones of phi (decoders.py:253-259)
            const int c = __ffs(~phi) - 1;
            for (int d = m - 1; d >= m - c; d--) {
                const int half = n >> (d + 1);
                const int lo = (phi >> (m - d)) << (m - d);
                if (half >= 32) {
                    const int hw = half >> 5, w0 = lo >> 5;
                    for (int it = lane; it < L * hw; it += 32) {
                        const int l = it / hw, i = it % hw;
                        ps[l * nw + w0 + i] ^= ps[l * nw + w0 + hw + i];
                    }
                } else {
                    const uint32_t mask = ((1u << half) - 1u) << (lo & 31);
                    for (int l = lane; l < L; l += 32) {
                        const uint32_t x = ps[l * nw + (lo >> 5)];
                        ps[l * nw + (lo >> 5)] = x ^ ((x >> half) & mask);
                    }
                }
                __syncwarp();
            }
        }

        // ---- output list: finite paths, stable by pm (decoders.py:261-268)
        const double mypm = (lane < L) ? pm[lane] : CUDART_INF;
        const bool fin = lane < L && isfinite(mypm);
        int rank = 0;
        for (int l = 0; l < L; l++) {
            const double pl = __shfl_sync(MPW_FULL, mypm, l);
            rank += isfinite(pl) && ((pl < mypm) || (pl == mypm && l < lane));
        }
        const unsigned finmask = __ballot_sync(MPW_FULL, fin);
        const int cnt = __popc(finmask);
        uint32_t cw[NW], uu[NW];
#pragma unroll
        for (int w = 0; w < NW; w++) { uu[w] = (lane < L && w < nw) ? ub[lane * nw + w] : 0u; cw[w] = uu[w]; }
        polar_transform_words<NW>(cw, nw);

        if (mode == 0) {
            if (lane == 0 && out.list_n) out.list_n[f] = cnt;
            if (fin) {
                const size_t o = ((size_t)f * L + rank) * nw;
#pragma unroll
                for (int w = 0; w < NW; w++)
                    if (w < nw) {
                        if (out.list_u) out.list_u[o + w] = uu[w];
                        if (out.list_cw) out.list_cw[o + w] = cw[w];
                    }
                if (out.list_pm) out.list_pm[(size_t)f * L + rank] = mypm;
            }
            continue;
        }

        // precoded v = u[info_set] (kp <= 64) and CRC syndrome
        uint64_t v = 0;
        if (code.is_ca && lane < L) {
            for (int j = 0; j < code.kp; j++) {
                const int pos = code.info[j];
                v |= (uint64_t)((ub[lane * nw + (pos >> 5)] >> (pos & 31)) & 1u) << j;
            }
        }
        int winner = 1 << 30;
        if (mode == 1) {
            uint32_t syn = 0;
            for (int j = 0; j < code.crc_deg; j++) syn |= (uint32_t)(__popcll(v & code.crc_h[j]) & 1) << j;
            winner = __reduce_min_sync(MPW_FULL, (fin && syn == 0) ? rank : (1 << 30));
        }
        if (winner < (1 << 30)) {
            // stage-1 CRC pass: best = the list codeword (== encode(msg)), decoders.py:559-570
            const int src = __ffs(__ballot_sync(MPW_FULL, fin && rank == winner)) - 1;
            if (lane == src) {
#pragma unroll
                for (int w = 0; w < NW; w++) if (w < nw) ps[w] = cw[w];   // ps is dead now: reuse
            }
            __syncwarp();
            double acc = 0.0;
            for (int i = lane; i < n; i += 32) {
                const double x = ((ps[i >> 5] >> (i & 31)) & 1u) ? -1.0 : 1.0;
                const double d = (double)y[(size_t)f * n + i] - x;
                acc += d * d;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(MPW_FULL, acc, o);
            if (lane < nw) out.best[(size_t)f * nw + lane] = ps[lane];
            __syncwarp();
            if (lane == 0) { out.stage[f] = 0; out.best_ed[f] = acc; }
            continue;
        }
        // ---- anchors: first A list entries, projected into the CRC subcode
        const int na = cnt < A ? cnt : A;
        int q = 0;
        if (lane == 0) q = atomicAdd(s2.count, 1);
        q = __shfl_sync(MPW_FULL, q, 0);
        if (fin && rank < na) {
            uint32_t an[NW];
            if (code.is_ca) {
#pragma unroll
                for (int w = 0; w < NW; w++) an[w] = 0u;
                const uint64_t msg = v & ((code.k >= 64) ? ~0ull : ((1ull << code.k) - 1ull));
                uint64_t rem = msg;
                while (rem) {
                    const int i = __ffsll((long long)rem) - 1;
                    rem &= rem - 1;
#pragma unroll
                    for (int w = 0; w < NW; w++) if (w < nw) an[w] ^= code.gen[(size_t)i * nw + w];
                }
            } else {
#pragma unroll
                for (int w = 0; w < NW; w++) an[w] = cw[w];
            }
            const size_t o = ((size_t)q * A + rank) * nw;
#pragma unroll
            for (int w = 0; w < NW; w++) if (w < nw) s2.anchors[o + w] = an[w];
        }
        if (lane == 0) { s2.frame[q] = f; s2.nanchor[q] = na; out.stage[f] = 1; }
    }
}
