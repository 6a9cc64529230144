// Stage 1, specialised: lane-per-path CA-SCL for power-of-two L <= 32 and
// N <= 256, templated on (N, L) so every loop bound and index is a constant.
//
// A warp holds FPW = 32 / L frames; lane = frame_in_warp * L + path.  Each
// lane runs its own path through the whole SC schedule (the f/g loops over a
// node's `half` elements are sequential per lane), so the per-element index
// arithmetic of the warp-per-frame kernel disappears.  Float64 operations and
// their order are exactly those of scl.cuh / the reference (decoders.py:173-268),
// so lists, orders and path metrics stay bit-identical.
//
// Shared memory per frame:
//   llr0[N]            channel LLRs (2y/sigma^2)
//   llr[L][INST]       per-path instances of stored levels 3..RL-1 (lazy clone via ptr)
//   ps[L][NW+1]        partial-sum bits (row padded against bank conflicts)
//   ptr[L][PTRW]       instance index per level (bytes)
//   sel[L]             info-leaf selection: source path | bit << 8 | flipped << 9
//   cand[L]            (pm, pm + |dm|) of every path at an info leaf
// The leaf decisions u are not stored: after the last leaf the partial sums
// are combined up to the root, giving the codeword, and u = its polar
// transform (the transform is an involution over GF(2)).
#pragma once
#include "common.cuh"
#include "scl.cuh"

// Levels 1 and 2 are "virtual": never stored, recomputed on demand from the
// channel LLRs and the path's own partial-sum bits with the same IEEE
// operations (so the values are bit-identical to stored ones).  Levels
// 3..RL-1 are stored per path instance in shared memory, levels RL..M in
// registers (SclLane below).
constexpr int SCL_VIRT = 2;
#ifndef MPW_SCL_D2_UNROLL
#define MPW_SCL_D2_UNROLL 1      // depth-2 node loop (measured on cfg4: 1: 7.35 ms, 2: 7.40, 4: 7.85, 8: 9.02: instruction fetch)
#endif
#ifndef MPW_SCL_RANK_UNROLL
#define MPW_SCL_RANK_UNROLL 4    // unroll factor of the info-leaf ranking loop (measured: 2: 7.89 ms, 4: 7.85, 8: 8.21, 16: 9.26 on cfg4)
#endif

template <int N, int L>
struct SclLane {
    static constexpr int M = (N >= 256) ? 8 : (N >= 128) ? 7 : (N >= 64) ? 6 : (N >= 32) ? 5 : (N >= 16) ? 4 : (N >= 8) ? 3 : (N >= 4) ? 2 : 1;
    static constexpr int NW = N >= 32 ? N / 32 : 1;
    static constexpr int NWP = NW + 1;
    static constexpr int PTRW = 1;                       // 4 bytes: instance index of shared levels 0..3
    static constexpr int FPW = 32 / L;
    // Levels of at most 16 values (RL..M) live in registers, one copy per lane
    // (= per path); a clone copies the source path's pending register levels
    // with shuffles.  Levels SCL_VIRT+1 .. RL-1 are stored per path instance in
    // shared memory (N = 256: level 3 only; N <= 128: none).
    static constexpr int RL = (M - 4 > SCL_VIRT + 1) ? M - 4 : SCL_VIRT + 1;
    static constexpr int INST = N / 4 - 2 * (N >> RL);   // stored doubles per instance (levels 3..RL-1)
    static constexpr int RT = 2 * (N >> RL) - 1;         // register doubles (levels RL..M)
    static constexpr size_t LLR0 = 0;
    static constexpr size_t LLR = LLR0 + 8 * (size_t)N;
    static constexpr size_t PS = LLR + 8 * (size_t)L * INST;
    static constexpr size_t PTR = PS + 4 * (size_t)L * NWP;
    static constexpr size_t SEL = PTR + 4 * (size_t)L * PTRW;
    static constexpr size_t CAND = (SEL + 4 * (size_t)L + 15) & ~(size_t)15;   // (pm, pm+|dm|) per path
    // Scratch of the cooperative frozen runs (SclCoop below): 3N/2 doubles.  Where the
    // instances of the dead paths can hold it (N = 256, L >= 16) it aliases them, else it is
    // a region of its own.
    static constexpr int SCRN = 3 * N / 2;
    static constexpr bool SCR_ALIAS = (L - 1) * INST >= SCRN;
    static constexpr size_t SCR = CAND + 16 * (size_t)L;
    static constexpr size_t TOTAL = SCR + (SCR_ALIAS ? 0 : 8 * (size_t)SCRN);
    // offset of stored level lvl (3..RL-1) inside an instance
    __host__ __device__ static constexpr int off(int lvl) { return N / 4 - 2 * (N >> (lvl > 0 ? lvl : 0)); }
    // offset of register level lvl (RL..M) inside the lane's register array
    __host__ __device__ static constexpr int roff(int lvl) { return 2 * (N >> RL) - 2 * (N >> lvl); }
};

// ---- node kernels with compile-time HALF (one lane = one path)
template <int HALF>
__device__ __forceinline__ void lane_f(const double* __restrict__ par, double* __restrict__ o) {
#pragma unroll (HALF < 8 ? HALF : 8)
    for (int j = 0; j < HALF; j++) o[j] = scl_f(par[j], par[j + HALF]);
}

template <int HALF>
__device__ __forceinline__ void lane_g(const double* __restrict__ par, double* __restrict__ o,
                                       const uint32_t* __restrict__ psrow, int lo) {
    if constexpr (HALF >= 32) {
#pragma unroll 1
        for (int jw = 0; jw < HALF / 32; jw++) {
            const uint32_t word = psrow[(lo >> 5) + jw];
#pragma unroll 8
            for (int b = 0; b < 32; b++) {
                const int j = jw * 32 + b;
                const double a = par[j], c = par[j + HALF];
                o[j] = c + (((word >> b) & 1u) ? -a : a);
            }
        }
    } else {
        const uint32_t word = psrow[lo >> 5] >> (lo & 31);
#pragma unroll
        for (int j = 0; j < HALF; j++) {
            const double a = par[j], c = par[j + HALF];
            o[j] = c + (((word >> j) & 1u) ? -a : a);
        }
    }
}

// virtual level 1: LLR j of depth-1 node `n1` (decoders.py:239-252 applied to llr0)
template <int N>
__device__ __forceinline__ double lv1(const double* __restrict__ llr0, const uint32_t* __restrict__ psrow,
                                      int n1, int j) {
    const double a = llr0[j], b = llr0[j + N / 2];
    if (n1 == 0) return scl_f(a, b);
    const uint32_t u = (psrow[j >> 5] >> (j & 31)) & 1u;       // left sibling's level-1 bits
    return b + (u ? -a : a);
}

// virtual level 2: LLR j of depth-2 node `n2`
template <int N>
__device__ __forceinline__ double lv2(const double* __restrict__ llr0, const uint32_t* __restrict__ psrow,
                                      int n2, int j) {
    const int n1 = n2 >> 1;
    const double a = lv1<N>(llr0, psrow, n1, j), b = lv1<N>(llr0, psrow, n1, j + N / 4);
    if (!(n2 & 1)) return scl_f(a, b);
    const int pos = n1 * (N / 2) + j;                           // left sibling's level-2 bits
    const uint32_t u = (psrow[pos >> 5] >> (pos & 31)) & 1u;
    return b + (u ? -a : a);
}

// depth-2 node: parent = virtual level 2, child = stored level 3
template <int N>
__device__ __forceinline__ void lane_node_d2(bool is_g, int n2, const double* __restrict__ llr0,
                                             const uint32_t* __restrict__ psrow, double* __restrict__ o,
                                             int lo) {
    constexpr int HALF = N / 8;
    if constexpr (N == 256) {
        // N = 256: element j of this node reads positions j + 32 k (k = 0..7) of llr0, and every
        // partial-sum bit it needs is bit j of one word: the words are read once, a sign flip is
        // an XOR of the sign bit (-a and a differ in nothing else), the f / g choices are
        // warp-uniform.  Same IEEE operations on the same operands as lv1 / lv2 above.
        const int n1 = n2 >> 1;
        const bool g1 = n1 != 0, g2 = (n2 & 1) != 0;
        uint32_t w1[4] = {0u, 0u, 0u, 0u}, w2[2] = {0u, 0u}, w3 = 0u;
        if (g1) {
#pragma unroll
            for (int k = 0; k < 4; k++) w1[k] = psrow[k];             // left half's level-1 bits
        }
        if (g2) { w2[0] = psrow[n1 * 4]; w2[1] = psrow[n1 * 4 + 1]; }   // left sibling's level-2 bits
        if (is_g) w3 = psrow[lo >> 5];                                // left sibling's level-3 bits
        auto flip = [](double a, uint32_t w, int j) {
            return __hiloint2double(__double2hiint(a) ^ (int)(((w >> j) & 1u) << 31), __double2loint(a));
        };
#pragma unroll 1
        for (int j = 0; j < HALF; j++) {
            double x[8];
#pragma unroll
            for (int k = 0; k < 8; k++) x[k] = llr0[j + 32 * k];
            double v1[4];
#pragma unroll
            for (int k = 0; k < 4; k++) v1[k] = g1 ? x[k + 4] + flip(x[k], w1[k], j) : scl_f(x[k], x[k + 4]);
            const double a = g2 ? v1[2] + flip(v1[0], w2[0], j) : scl_f(v1[0], v1[2]);
            const double c = g2 ? v1[3] + flip(v1[1], w2[1], j) : scl_f(v1[1], v1[3]);
            o[j] = is_g ? c + flip(a, w3, j) : scl_f(a, c);
        }
        return;
    }
    const uint32_t word = (HALF >= 32) ? 0u : (psrow[lo >> 5] >> (lo & 31));
    constexpr int DU = MPW_SCL_D2_UNROLL;
#pragma unroll (DU)
    for (int j = 0; j < HALF; j++) {
        const double a = lv2<N>(llr0, psrow, n2, j), c = lv2<N>(llr0, psrow, n2, j + HALF);
        if (!is_g) {
            o[j] = scl_f(a, c);
        } else {
            const int p = lo + j;
            const uint32_t u = (HALF >= 32) ? ((psrow[p >> 5] >> (p & 31)) & 1u) : ((word >> j) & 1u);
            o[j] = c + (u ? -a : a);
        }
    }
}

// One SC node at depth D (writes level D+1), the left (f) or right (g) child.
// Parent values come from the virtual level 2, a stored instance (via the
// path's instance pointer) or the lane's registers; the child goes to the
// path's own instance or to registers.  Same IEEE operations in every case.
template <int N, int L, int D>
__device__ __forceinline__ void lane_step(bool is_g, double (&r)[SclLane<N, L>::RT], const double* __restrict__ llr,
                                          double* __restrict__ myllr, uint8_t* ptrrow,
                                          const double* __restrict__ llr0, const uint32_t* __restrict__ psrow,
                                          int n2, int lo, int l) {
    using Lay = SclLane<N, L>;
    constexpr int RL = Lay::RL, HALF = N >> (D + 1);
    if constexpr (D < SCL_VIRT || D >= Lay::M) {
        return;                                                   // virtual child: nothing to do
    } else if constexpr (D + 1 < RL) {
        // shared -> shared
        if constexpr (D == SCL_VIRT) {
            lane_node_d2<N>(is_g, n2, llr0, psrow, myllr + Lay::off(3), lo);
        } else {
            const double* par = llr + (size_t)ptrrow[D] * Lay::INST + Lay::off(D);
            if (is_g) lane_g<HALF>(par, myllr + Lay::off(D + 1), psrow, lo);
            else lane_f<HALF>(par, myllr + Lay::off(D + 1));
        }
        ptrrow[D + 1] = (uint8_t)l;
        __syncwarp();
    } else {
        static_assert(HALF <= 16, "register levels hold at most 16 values");
        const double* par = nullptr;
        if constexpr (D > SCL_VIRT && D < RL) par = llr + (size_t)ptrrow[D] * Lay::INST + Lay::off(D);
        auto in = [&](int j) -> double {
            if constexpr (D == SCL_VIRT) return lv2<N>(llr0, psrow, n2, j);
            else if constexpr (D < RL) return par[j];
            else return r[Lay::roff(D) + j];
        };
        // f and g in separate loops (is_g is warp-uniform): no wasted half
        if (is_g) {
            const uint32_t word = psrow[lo >> 5] >> (lo & 31);
#pragma unroll
            for (int j = 0; j < HALF; j++) {
                const double a = in(j), c = in(j + HALF);
                r[Lay::roff(D + 1) + j] = c + (((word >> j) & 1u) ? -a : a);
            }
        } else {
#pragma unroll
            for (int j = 0; j < HALF; j++) r[Lay::roff(D + 1) + j] = scl_f(in(j), in(j + HALF));
        }
    }
}

// Descent to a leaf: the nodes at depths d0..M-1 (a g node at d0 unless this is
// leaf 0, f nodes below).  One jump on d0 per leaf, the node bodies fall through
// and exist once in the binary; each has its depth as a constant, so HALF and
// the register indices are constants.
template <int N, int L>
__device__ __forceinline__ void lane_descent(int d0, bool first_g, double (&r)[SclLane<N, L>::RT], const double* llr,
                                             double* myllr, uint8_t* ptrrow, const double* llr0,
                                             const uint32_t* psrow, int n2, int lo, int l) {
#define MPW_LANE_CASE(DD) \
    case DD: lane_step<N, L, DD>(first_g && d0 == DD, r, llr, myllr, ptrrow, llr0, psrow, n2, d0 == DD ? lo : 0, l);
    switch (d0 < SCL_VIRT ? SCL_VIRT : d0) {
        MPW_LANE_CASE(2) MPW_LANE_CASE(3) MPW_LANE_CASE(4) MPW_LANE_CASE(5) MPW_LANE_CASE(6) MPW_LANE_CASE(7)
        default: break;
    }
#undef MPW_LANE_CASE
}

template <int N, int L, int LVL>
__device__ __forceinline__ void clone_levels(double (&r)[SclLane<N, L>::RT], int phi, int srcl) {
    using Lay = SclLane<N, L>;
    if constexpr (LVL < Lay::M) {
        if (!((phi >> (Lay::M - 1 - LVL)) & 1)) {
#pragma unroll
            for (int j = 0; j < (N >> LVL); j++)
                r[Lay::roff(LVL) + j] = __shfl_sync(MPW_FULL, r[Lay::roff(LVL) + j], srcl);
        }
        clone_levels<N, L, LVL + 1>(r, phi, srcl);
    }
}

// first non-frozen leaf at or after phi (N if there is none)
template <int N>
__device__ __forceinline__ int next_info_leaf(const uint32_t* __restrict__ frozen, int phi) {
    constexpr int NW = N >= 32 ? N / 32 : 1;
    for (int w = phi >> 5; w < NW; w++) {
        uint32_t m = ~frozen[w];
        if (w == (phi >> 5)) m &= ~0u << (phi & 31);
        if (N < 32) m &= (1u << (N & 31)) - 1u;
        if (m) return w * 32 + __ffs(m) - 1;
    }
    return N;
}

// ---- cooperative frozen runs
// While only P < L paths are alive, the lanes of the dead paths would just
// repeat work.  A run of frozen leaves [phi0, phi0 + tau) that starts where the
// parent LLRs are virtual (phi0 = 0 or a multiple of N/8) is therefore computed
// by all L lanes of the frame together, G = L / P lanes per live path.  Every
// decision in the run is 0, so the left siblings of the path to leaf
// phi0 + tau are rate-0 subtrees: their leaf LLRs come from an in-place
// butterfly (f into the lower, g with u = 0 into the upper half of every node)
// and the penalties are added in leaf order (decoders.py:216-218).  Each value
// is produced by the same IEEE operation on the same operands as in the
// depth-first schedule (decoders.py:239-252), so the path metrics stay
// bit-identical.  The path's arrays of levels lev0..M end up in the scratch
// (stored levels: directly in instance p), from where the caller installs them.
//
// Scratch of path p (W = h0r + h0 + h0/2 doubles, h0 = N >> lev0, h0r = lev0 ? h0 : 0):
//   [0, h0r)                 root array (level lev0) unless it is a stored level
//   h0r + h0 - 2 (N >> k)    path array of level k > lev0
//   h0r + h0                 butterfly buffer (h0 / 2)
template <int N, int L>
struct SclCoop {
    using Lay = SclLane<N, L>;
    __device__ static __forceinline__ int h0r(int lev0) { return lev0 ? (N >> lev0) : 0; }
    __device__ static __forceinline__ int stride(int lev0) { return h0r(lev0) + (N >> lev0) + (N >> (lev0 + 1)); }
    __device__ static __forceinline__ double* level(double* base, double* inst, int lev0, int k) {
        if (k > SCL_VIRT && k < Lay::RL) return inst + Lay::off(k);
        return (k == lev0) ? base : base + h0r(lev0) + (N >> lev0) - 2 * (N >> k);
    }
    // in-place butterfly of a rate-0 subtree of h leaves by the G lanes of a path
    __device__ static __forceinline__ void butterfly(double* B, int h, int s, int G) {
        for (int sz = h; sz >= 2; sz >>= 1) {
            const int hh = sz >> 1;
            for (int t = s; t < (h >> 1); t += G) {
                const int j = t & (hh - 1), i0 = ((t - j) << 1) + j, i1 = i0 + hh;
                const double a = B[i0], c = B[i1];
                B[i0] = scl_f(a, c);
                B[i1] = c + a;
            }
            __syncwarp();
        }
    }
    __device__ static __forceinline__ double penalties(const double* B, int h, double pm) {
        for (int j = 0; j < h; j++) {
            const double dm = B[j];
            pm = pm + fabs(dm) * (double)(dm < 0.0);
        }
        return pm;
    }
    // returns the path metric of path p = l / G after the run
    __device__ static __forceinline__ double run(int phi0, int tau, int lev0, int P, double pm,
                                                 const double* __restrict__ llr0, const uint32_t* ps_all,
                                                 double* llr, double* scr, int l) {
        constexpr int M = Lay::M;
        const int G = L / P, p = l / G, s = l - p * G;
        const int h0 = N >> lev0;
        double* base = scr + (size_t)p * stride(lev0);
        double* inst = llr + (size_t)p * Lay::INST;
        double* B = base + h0r(lev0) + h0;
        const uint32_t* psrow = ps_all + p * Lay::NWP;
        const double* cur = llr0;
        if (lev0) {
            // root of the run = right child made by the g node at depth lev0 - 1 (virtual parent)
            double* root = level(base, inst, lev0, lev0);
            const int n2 = phi0 >> (M - 2);
            for (int j = s; j < h0; j += G) {
                double v;
                if (lev0 == 1) v = lv1<N>(llr0, psrow, 1, j);
                else if (lev0 == 2) v = lv2<N>(llr0, psrow, n2, j);
                else {
                    const double a = lv2<N>(llr0, psrow, n2, j), c = lv2<N>(llr0, psrow, n2, j + N / 8);
                    const int pos = n2 * (N / 4) + j;
                    v = c + (((psrow[pos >> 5] >> (pos & 31)) & 1u) ? -a : a);
                }
                root[j] = v;
            }
            __syncwarp();
            if (tau == h0) {                       // the whole subtree is frozen
                butterfly(root, h0, s, G);
                return penalties(root, h0, pm);
            }
            cur = root;
        }
        int sz = h0, lev = lev0, t = tau;
        while (sz > 1) {
            const int h = sz >> 1;
            double* child = level(base, inst, lev0, lev + 1);
            if (t < h) {
                for (int j = s; j < h; j += G) child[j] = scl_f(cur[j], cur[j + h]);
                __syncwarp();
            } else {
                for (int j = s; j < h; j += G) {
                    const double a = cur[j], c = cur[j + h];
                    B[j] = scl_f(a, c);
                    child[j] = c + a;
                }
                __syncwarp();
                butterfly(B, h, s, G);
                pm = penalties(B, h, pm);
                __syncwarp();
                t -= h;
            }
            cur = child;
            sz = h;
            lev++;
        }
        return pm;
    }
};

// register levels LVL..M of the lane := the path arrays a cooperative run left in the scratch
template <int N, int L, int LVL>
__device__ __forceinline__ void coop_install(double (&r)[SclLane<N, L>::RT], double* sb, double* si, int lev0) {
    using Lay = SclLane<N, L>;
    if constexpr (LVL <= Lay::M) {
        const double* a = SclCoop<N, L>::level(sb, si, lev0, LVL);
#pragma unroll
        for (int j = 0; j < (N >> LVL); j++) r[Lay::roff(LVL) + j] = a[j];
        coop_install<N, L, LVL + 1>(r, sb, si, lev0);
    }
}

template <int N, int L>
__global__ void __launch_bounds__(128, 4) scl_lane_kernel(CodeDev code, const float* __restrict__ y,
                                                       const double* __restrict__ llr64, int F,
                                                       double sigma, int A, int mode, SclOut out,
                                                       S2Dev s2) {
    using Lay = SclLane<N, L>;
    constexpr int M = Lay::M, NW = Lay::NW, NWP = Lay::NWP, FPW = Lay::FPW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int fi = lane / L, l = lane % L, g0 = fi * L;
    const unsigned gmask = (L == 32) ? MPW_FULL : (((1u << L) - 1u) << g0);
    unsigned char* base = smem_raw + (size_t)(wib * FPW + fi) * Lay::TOTAL;
    double* llr0 = reinterpret_cast<double*>(base + Lay::LLR0);
    double* llr = reinterpret_cast<double*>(base + Lay::LLR);
    uint32_t* ps_all = reinterpret_cast<uint32_t*>(base + Lay::PS);
    uint8_t* ptr_all = base + Lay::PTR;
    int32_t* sel = reinterpret_cast<int32_t*>(base + Lay::SEL);
    double2* cand = reinterpret_cast<double2*>(base + Lay::CAND);
    uint32_t* psrow = ps_all + l * NWP;
    uint8_t* ptrrow = ptr_all + l * Lay::PTRW * 4;
    double* myllr = llr + (size_t)l * Lay::INST;
    double* scrx = reinterpret_cast<double*>(base + Lay::SCR);      // (unused when the scratch aliases llr)
    const double sig2 = sigma * sigma;

    for (long long fb = ((long long)blockIdx.x * wpb + wib) * FPW; fb < F;
         fb += (long long)gridDim.x * wpb * FPW) {
        const long long f = fb + fi;
        const bool valid = f < F;
        // ---- init (decoders.py:204-209)
        for (int i = l; i < N; i += L) {
            double v = 0.0;
            if (valid) v = llr64 ? llr64[(size_t)f * N + i] : 2.0 * (double)y[(size_t)f * N + i] / sig2;
            llr0[i] = v;
        }
#pragma unroll
        for (int w = 0; w < NWP; w++) psrow[w] = 0u;
        double pm = (l == 0) ? 0.0 : CUDART_INF;
        double r[Lay::RT];                  // register levels RL..M of this path
#pragma unroll
        for (int j = 0; j < Lay::RT; j++) r[j] = 0.0;
        __syncwarp();

        // combine after leaf phi (:253-259); after the last leaf it runs up to the root
        auto combine = [&](int phi) {
            const int c = __ffs(~phi) - 1;
            // (rolled: this runs after every leaf, and the kernel is bound by instruction fetch)
#pragma unroll 1
            for (int d = M - 1; d >= M - c; d--) {
                const int half = N >> (d + 1);
                const int lo = (phi >> (M - d)) << (M - d);
                if (half >= 32) {
                    const int hw = half >> 5, w0 = lo >> 5;
#pragma unroll 1
                    for (int i = 0; i < hw; i++) psrow[w0 + i] ^= psrow[w0 + hw + i];
                } else {
                    const uint32_t mask = ((1u << half) - 1u) << (lo & 31);
                    const uint32_t x = psrow[lo >> 5];
                    psrow[lo >> 5] = x ^ ((x >> half) & mask);
                }
            }
        };
        int nlive = 1;                      // live paths = lanes 0..nlive-1 of the frame
        for (int phi = 0; phi < N; phi++) {
            if constexpr (N >= 64 && L >= 2) {
                // cooperative frozen run (coop_frozen_run above) while at most L/2 paths live
                if ((phi & (N / 8 - 1)) == 0 && 2 * nlive <= L && ((code.frozen[phi >> 5] >> (phi & 31)) & 1u)) {
                    const int lev0 = phi ? M - __ffs(phi) + 1 : 0;
                    const int h0 = N >> lev0;
                    const int tau = min(next_info_leaf<N>(code.frozen, phi) - phi, h0);
                    const int cap = Lay::SCR_ALIAS ? (L - nlive) * Lay::INST : Lay::SCRN;
                    if (tau >= 8 && (lev0 || tau < N) && nlive * SclCoop<N, L>::stride(lev0) <= cap) {
                        const int P = nlive, G = L / P;
                        double* scr = Lay::SCR_ALIAS ? llr + (size_t)P * Lay::INST : scrx;
                        const double pin = __shfl_sync(MPW_FULL, pm, g0 + l / G);
                        const double pout = SclCoop<N, L>::run(phi, tau, lev0, P, pin, llr0, ps_all, llr, scr, l);
                        const double pmine = __shfl_sync(MPW_FULL, pout, g0 + (l < P ? l * G : l));
                        if (l < P) pm = pmine;
                        if (tau == h0) {            // whole subtree done: only the last leaf's combine acts
                            combine(phi + h0 - 1);
                            __syncwarp();
                            phi += h0 - 1;
                            continue;
                        }
                        // install the arrays on the path to leaf phi + tau (an information leaf)
                        const int pl = l < P ? l : 0;
                        double* sb = scr + (size_t)pl * SclCoop<N, L>::stride(lev0);
                        double* si = llr + (size_t)pl * Lay::INST;
                        if constexpr (Lay::RL > SCL_VIRT + 1) {   // (dead paths point at path 0's arrays)
#pragma unroll
                            for (int k = SCL_VIRT + 1; k < Lay::RL; k++) ptrrow[k] = (uint8_t)pl;
                        }
                        coop_install<N, L, Lay::RL>(r, sb, si, lev0);
                        __syncwarp();
                        phi += tau;
                    }
                }
            }
            // descent to leaf phi: one g at depth M-1-ctz(phi), then f's.  Nodes
            // whose child level is virtual (depth < SCL_VIRT) need no work.
            // descent to leaf phi: one g at depth M-1-ctz(phi), then f's (one call
            // site, so the unrolled node bodies exist once in the binary)
            int d0 = SCL_VIRT, lo = 0;
            if (phi) {
                d0 = M - __ffs(phi);
                lo = (phi >> (M - d0)) << (M - d0);
            }
            lane_descent<N, L>(d0, phi != 0, r, llr, myllr, ptrrow, llr0, psrow, phi >> (M - 2), lo, l);
            const double dm = r[Lay::roff(M)];
            const bool frozen = (code.frozen[phi >> 5] >> (phi & 31)) & 1u;
            if (frozen) {
                pm = pm + fabs(dm) * (double)(dm < 0.0);                      // :216-218
            } else {
                // stable rank of the 2L candidates (pm_k natural, pm_k + |dm_k| flipped);
                // every path publishes its pair once, then reads all L pairs with
                // broadcast 16-byte loads (instead of 2L 64-bit shuffles)
                nlive = min(L, 2 * nlive);
                const double vn = pm, vf = pm + fabs(dm);
                cand[l] = make_double2(vn, vf);
                __syncwarp();
                int rn = 0, rf = 0;
                constexpr int RU = MPW_SCL_RANK_UNROLL < L ? MPW_SCL_RANK_UNROLL : L;
#pragma unroll (RU)
                for (int k = 0; k < L; k++) {
                    const double2 ck = cand[k];
                    const double pk = ck.x, fk = ck.y;
                    rn += (pk < vn) || (pk == vn && k < l);
                    rn += (fk < vn);
                    rf += (pk <= vf);
                    rf += (fk < vf) || (fk == vf && k < l);
                }
                const int nat = dm < 0.0 ? 1 : 0;
                if (rn < L) sel[rn] = l | (nat << 8);
                if (rf < L) sel[rf] = l | ((nat ^ 1) << 8) | (1 << 9);
                __syncwarp();
                const int sl = sel[l];
                const int src = sl & 0xFF;
                const int bit = (sl >> 8) & 1;
                {
                    const double2 cs = cand[src];
                    pm = (sl >> 9) ? cs.y : cs.x;
                }
                // register levels still to be read by a g node (this leaf is in the
                // left subtree of the depth-lvl node) come from the source path
                clone_levels<N, L, Lay::RL>(r, phi, g0 + src);
                uint32_t rps[NW], rp[Lay::PTRW];
                const uint32_t* sps = ps_all + src * NWP;
                const uint32_t* sp = reinterpret_cast<const uint32_t*>(ptr_all + src * Lay::PTRW * 4);
#pragma unroll
                for (int w = 0; w < NW; w++) rps[w] = sps[w];
#pragma unroll
                for (int w = 0; w < Lay::PTRW; w++) rp[w] = sp[w];
                __syncwarp();
#pragma unroll
                for (int w = 0; w < NW; w++) psrow[w] = rps[w];
                if (bit) psrow[phi >> 5] |= 1u << (phi & 31);     // the leaf's decision (one word, addressed)
                uint32_t* mp = reinterpret_cast<uint32_t*>(ptrrow);
#pragma unroll
                for (int w = 0; w < Lay::PTRW; w++) mp[w] = rp[w];
                __syncwarp();
            }
            combine(phi);
        }

        // ---- list: finite paths, stable by pm (decoders.py:261-268)
        const bool fin = isfinite(pm);
        int rank = 0;
#pragma unroll
        for (int k = 0; k < L; k++) {
            const double pk = __shfl_sync(MPW_FULL, pm, g0 + k);
            rank += isfinite(pk) && ((pk < pm) || (pk == pm && k < l));
        }
        const unsigned finmask = __ballot_sync(MPW_FULL, fin) & gmask;
        const int cnt = __popc(finmask);
        uint32_t cw[NW], uu[NW];
#pragma unroll
        for (int w = 0; w < NW; w++) { cw[w] = psrow[w]; uu[w] = cw[w]; }
        polar_transform_words<NW>(uu, NW);
        // own partial-sum row := u, read bit by bit by the CRC gate below
#pragma unroll
        for (int w = 0; w < NW; w++) psrow[w] = uu[w];

        if (mode == 0) {
            if (valid) {
                if (l == 0 && out.list_n) out.list_n[f] = cnt;
                if (fin) {
                    const size_t o = ((size_t)f * L + rank) * NW;
#pragma unroll
                    for (int w = 0; w < NW; w++) {
                        if (out.list_u) out.list_u[o + w] = uu[w];
                        if (out.list_cw) out.list_cw[o + w] = cw[w];
                    }
                    if (out.list_pm) out.list_pm[(size_t)f * L + rank] = pm;
                }
            }
            __syncwarp();
            continue;
        }

        // ---- CRC gate (decoders.py:559-570) on v = u[info_set] (codebook.py:154-163, 287-297)
        uint64_t v = 0;
        if (code.is_ca) {
#pragma unroll 1
            for (int j = 0; j < code.kp; j++) {
                const int pos = code.info[j];
                v |= (uint64_t)((psrow[pos >> 5] >> (pos & 31)) & 1u) << j;
            }
        }
        int gwin = 1 << 30;                 // lowest CRC-valid rank in this frame group
        if (mode == 1) {
            uint32_t syn = 0;
#pragma unroll 1
            for (int j = 0; j < code.crc_deg; j++) syn |= (uint32_t)(__popcll(v & code.crc_h[j]) & 1) << j;
            gwin = (fin && syn == 0) ? rank : (1 << 30);
#pragma unroll
            for (int o = 1; o < L; o <<= 1) gwin = min(gwin, __shfl_xor_sync(MPW_FULL, gwin, o));
        }
        const bool passed = gwin < (1 << 30);
        __syncwarp();
        // winner's codeword into scratch (ps rows are dead after the last leaf)
        if (passed && fin && rank == gwin) {
#pragma unroll
            for (int w = 0; w < NW; w++) ps_all[w] = cw[w];
        }
        __syncwarp();
        double acc = 0.0;
        if (passed) {
            for (int i = l; i < N; i += L) {
                const double x = ((ps_all[i >> 5] >> (i & 31)) & 1u) ? -1.0 : 1.0;
                const double dd = (valid ? (double)y[(size_t)f * N + i] : 0.0) - x;
                acc += dd * dd;
            }
        }
#pragma unroll
        for (int o = 1; o < L; o <<= 1) acc += __shfl_xor_sync(MPW_FULL, acc, o);
        // stage-2 queue slot (one atomic per failing frame), broadcast in the group
        const int na = cnt < A ? cnt : A;
        int q = 0;
        if (!passed && valid && l == 0) q = atomicAdd(s2.count, 1);
        q = __shfl_sync(MPW_FULL, q, g0);
        if (valid) {
            if (passed) {
                for (int w = l; w < NW; w += L) out.best[(size_t)f * NW + w] = ps_all[w];
                if (l == 0) { out.stage[f] = 0; out.best_ed[f] = acc; }
            } else {
                if (fin && rank < na) {
                    // anchors: first A entries projected into the CRC subcode (decoders.py:572-579)
                    uint32_t an[NW];
                    if (code.is_ca) {
#pragma unroll
                        for (int w = 0; w < NW; w++) an[w] = 0u;
                        uint64_t rem = v & ((code.k >= 64) ? ~0ull : ((1ull << code.k) - 1ull));
                        while (rem) {
                            const int i = __ffsll((long long)rem) - 1;
                            rem &= rem - 1;
#pragma unroll
                            for (int w = 0; w < NW; w++) an[w] ^= code.gen[(size_t)i * NW + w];
                        }
                    } else {
#pragma unroll
                        for (int w = 0; w < NW; w++) an[w] = cw[w];
                    }
                    const size_t o = ((size_t)q * A + rank) * NW;
#pragma unroll
                    for (int w = 0; w < NW; w++) s2.anchors[o + w] = an[w];
                }
                if (l == 0) { s2.frame[q] = (int)f; s2.nanchor[q] = na; out.stage[f] = 1; }
            }
        }
        __syncwarp();
    }
}
