// Order-k OSD stage 1 on the GPU (the paper's RM
// initialiser).  Restates `osd_decode` (decoders.py:274-317):
//   column order  = stable argsort(-|y|)                        (:287)
//   basis/pivots  = Gauss-Jordan over GF(2) in that column order (:288, binlin.py:209-247)
//   base          = XOR of basis rows whose pivot symbol is < 0   (:294-299)
//   candidates    = base ^ XOR(basis[c]) for every c in
//                   itertools.combinations(range(K), w), w = 1..order, in that
//                   order (:301-306, :320-323); candidate index = position
//   list          = stable argsort of squared ED, first list_cap (:310-317)
// One warp per frame.  Ranking by counting (N^2/32 per lane), elimination with
// ballot pivot search, then every lane walks a contiguous chunk of the
// candidate sequence: lexicographic order of combinations is decreasing order
// of the row mask with row j at bit K-1-j, so the successor is a
// reverse-Gosper step.  Candidates are scored by corr = sum_i x_i y_i in
// float64 (ED = |y|^2 + N - 2 corr) and kept in a warp-shared top-(M+1) list
// ordered by (-corr, index) -- the order of the reference's stable argsort.
// The kept M+1 entries are then re-sorted by their canonical squared ED
// (sequential float64, the oracle's arithmetic) so reported scores are the
// sort keys; the (M+1)-th entry certifies the list boundary: adjacent EDs
// closer than the rounding bound set MPW_F_TIE_STAGE1 (the reference's
// einsum sums in a different order).  The full-list path sorts every
// candidate by canonical ED directly.
#pragma once
#include "common.cuh"
#include "scl.cuh"

#define MPW_F_TIE_STAGE1 16u

constexpr int OSD_MAX_K = 63;
constexpr int OSD_MAX_ORDER = 16;
constexpr int OSD_MAX_KEEP = 96;     // M + 1 entries held in shared memory
constexpr int OSD_WARPS = 4;

struct OsdArgs {
    CodeDev code;
    const float* y;
    int F, order, M, mode;           // mode 0: list; 1: crc_gated two-stage; 2: always_on
    long long C;                     // sum_{w <= order} C(K, w)
    // list outputs (mode 0)
    int32_t* list_n; uint32_t* list_cw; double* list_ed;
    // all keys (mode 0, M > OSD_MAX_KEEP - 1): F x C, sorted on the device afterwards
    double* keys;
    uint32_t* basis;                 // F x (K + 1) x NW reduced rows + base (full-list path)
    uint8_t* s1flags;                // per-frame MPW_F_TIE_STAGE1
    SclOut out;
    S2Dev s2;
    int A;
};

__host__ __device__ inline size_t osd_warp_bytes(int n, int nw) {
    return scl_align16((size_t)nw * 32 * 4) + scl_align16((size_t)n * 2) + scl_align16((size_t)64 * nw * 4) +
           scl_align16((size_t)OSD_MAX_KEEP * 8) + scl_align16((size_t)OSD_MAX_KEEP * 4) + 16 * 8;
}
__host__ __device__ inline size_t osd_smem_bytes(int n, int nw) {
    return scl_align16((size_t)64 * (OSD_MAX_ORDER + 1) * 8) + OSD_WARPS * osd_warp_bytes(n, nw);
}

__device__ __forceinline__ uint64_t osd_kmask(int K) { return K >= 64 ? ~0ull : ((1ull << K) - 1ull); }

// Candidate index -> reversed row mask (row j at bit K-1-j).
__device__ inline uint64_t osd_unrank(long long idx, int K, int order, const unsigned long long* binom) {
    int w = 0;
    long long r = idx;
    while (w < order && r >= (long long)binom[K * (OSD_MAX_ORDER + 1) + w]) {
        r -= (long long)binom[K * (OSD_MAX_ORDER + 1) + w];
        w++;
    }
    uint64_t R = 0;
    int a = 0;
    for (int p = 0; p < w; p++) {
        for (;;) {
            const int rem = K - a - 1, kk = w - p - 1;
            const long long c = (rem >= kk) ? (long long)binom[rem * (OSD_MAX_ORDER + 1) + kk] : 0;
            if (c <= r) { r -= c; a++; } else break;
        }
        R |= 1ull << (K - 1 - a);
        a++;
    }
    return R;
}

// Next combination in lexicographic order (next smaller mask of equal popcount,
// else the first combination of the next weight).
__device__ __forceinline__ uint64_t osd_next(uint64_t R, int K) {
    const uint64_t km = osd_kmask(K);
    const int w = __popcll(R);
    const uint64_t v = ~R & km;
    if (v != 0 && R != ((1ull << w) - 1ull)) {
        const uint64_t t = v | (v - 1);
        const uint64_t nx = (t + 1) | (((~t & (t + 1)) - 1) >> (__ffsll((long long)v)));
        return ~nx & km;
    }
    return (w + 1 >= 64) ? km : (((1ull << (w + 1)) - 1ull) << (K - w - 1));
}

template <int NW>
__device__ __forceinline__ void osd_word(const uint32_t* rows, const uint32_t* base, uint64_t R, int K,
                                         uint32_t* c) {
#pragma unroll
    for (int w = 0; w < NW; w++) c[w] = base[w];
    while (R) {
        const int b = __ffsll((long long)R) - 1;
        R &= R - 1;
        const int row = K - 1 - b;
#pragma unroll
        for (int w = 0; w < NW; w++) c[w] ^= rows[row * NW + w];
    }
}

template <int NW>
__device__ __forceinline__ double osd_corr(const float* sy, const uint32_t* c, int n) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
        if (w * 32 >= n) break;
        const uint32_t bits = c[w];
#pragma unroll 8
        for (int b = 0; b < 32; b++) {
            const double v = (double)sy[w * 32 + b];
            acc += ((bits >> b) & 1u) ? -v : v;
        }
    }
    return acc;
}

// Canonical ||y - x(c)||^2: sequential float64, no contraction -- the same
// arithmetic as the oracle's sqdist (channel.py:90-93).
template <int NW>
__device__ __forceinline__ double osd_ced(const float* sy, const uint32_t* c, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; i++) {
        const double d = __dsub_rn((double)sy[i], ((c[i >> 5] >> (i & 31)) & 1u) ? -1.0 : 1.0);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return acc;
}

__device__ __forceinline__ bool osd_less(double ka, int ia, double kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__device__ inline void osd_binom_init(unsigned long long* binom) {
    for (int i = threadIdx.x; i < 64 * (OSD_MAX_ORDER + 1); i += blockDim.x) {
        const int nn = i / (OSD_MAX_ORDER + 1), kk = i % (OSD_MAX_ORDER + 1);
        unsigned long long c = kk <= nn ? 1ull : 0ull;
        for (int j = 0; j < kk && c; j++) c = c * (unsigned long long)(nn - j) / (unsigned long long)(j + 1);
        binom[i] = c;
    }
}

// Per-frame prologue (decoders.py:287-299): y row into sy, stable column
// order, Gauss-Jordan reduction of the generator in rows[K][NW], base word.
// Returns sum |y_i| (scale of the tie tolerance).
template <int NW>
__device__ inline double osd_prologue(const CodeDev& code, const float* yr, float* sy, uint16_t* sord,
                                      uint32_t* rows, uint32_t* base) {
    const int N = code.n, K = code.k, lane = threadIdx.x & 31;
    for (int i = lane; i < NW * 32; i += 32) sy[i] = i < N ? yr[i] : 0.0f;   // zero tail: +0 in corr
    for (int i = lane; i < K * NW; i += 32) rows[i] = code.gen[i];
    __syncwarp();
    // ---- column order: stable argsort(-|y|) (decoders.py:287)
    double yabs = 0.0;
    for (int i = lane; i < N; i += 32) {
        const float ai = fabsf(sy[i]);
        int r = 0;
        for (int j = 0; j < N; j++) {
            const float aj = fabsf(sy[j]);
            r += (aj > ai) || (aj == ai && j < i);
        }
        sord[r] = (uint16_t)i;
        yabs += (double)ai;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) yabs += __shfl_xor_sync(MPW_FULL, yabs, o);
    __syncwarp();
    // ---- Gauss-Jordan in column order (binlin.py:226-247)
    int rank = 0;
    uint64_t hard = 0;                     // bit r: y[pivot_r] < 0 (decoders.py:294)
    for (int t = 0; t < N && rank < K; t++) {
        const int col = sord[t], cw_ = col >> 5, cb = col & 31;
        const bool h0 = lane >= rank && lane < K && ((rows[lane * NW + cw_] >> cb) & 1u);
        const bool h1 = lane + 32 >= rank && lane + 32 < K && ((rows[(lane + 32) * NW + cw_] >> cb) & 1u);
        const unsigned b0 = __ballot_sync(MPW_FULL, h0), b1 = __ballot_sync(MPW_FULL, h1);
        if (!(b0 | b1)) continue;
        const int p = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
        if (p != rank && lane < NW) {
            const uint32_t tmp = rows[rank * NW + lane];
            rows[rank * NW + lane] = rows[p * NW + lane];
            rows[p * NW + lane] = tmp;
        }
        __syncwarp();
        uint32_t pr[NW];
#pragma unroll
        for (int w = 0; w < NW; w++) pr[w] = rows[rank * NW + w];
        __syncwarp();
        for (int rr = lane; rr < K; rr += 32) {
            if (rr != rank && ((rows[rr * NW + cw_] >> cb) & 1u)) {
#pragma unroll
                for (int w = 0; w < NW; w++) rows[rr * NW + w] ^= pr[w];
            }
        }
        if (sy[col] < 0.0f) hard |= 1ull << rank;
        rank++;
        __syncwarp();
    }
    // ---- base word (decoders.py:295-299)
    if (lane < NW) {
        uint32_t b = 0;
        uint64_t hm = hard;
        while (hm) {
            const int r = __ffsll((long long)hm) - 1;
            hm &= hm - 1;
            b ^= rows[r * NW + lane];
        }
        base[lane] = b;
    }
    __syncwarp();
    return yabs;
}

template <int NW>
__global__ void __launch_bounds__(32 * OSD_WARPS) osd_kernel(OsdArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.code.n, K = a.code.k, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long* binom = reinterpret_cast<unsigned long long*>(smem_raw);
    osd_binom_init(binom);
    unsigned char* wb = smem_raw + scl_align16((size_t)64 * (OSD_MAX_ORDER + 1) * 8) + wid * osd_warp_bytes(N, NW);
    float* sy = reinterpret_cast<float*>(wb);
    wb += scl_align16((size_t)NW * 32 * 4);
    uint16_t* sord = reinterpret_cast<uint16_t*>(wb);
    wb += scl_align16((size_t)N * 2);
    uint32_t* rows = reinterpret_cast<uint32_t*>(wb);
    wb += scl_align16((size_t)64 * NW * 4);
    double* tk = reinterpret_cast<double*>(wb);
    wb += scl_align16((size_t)OSD_MAX_KEEP * 8);
    int32_t* ti = reinterpret_cast<int32_t*>(wb);
    wb += scl_align16((size_t)OSD_MAX_KEEP * 4);
    uint32_t* base = reinterpret_cast<uint32_t*>(wb);
    __syncthreads();

    const int keep = a.keys ? 0 : (int)min((long long)a.M + 1, a.C);   // entries held (M + boundary)
    const int nwarps = gridDim.x * OSD_WARPS;
    for (int f = blockIdx.x * OSD_WARPS + wid; f < a.F; f += nwarps) {
        const double yabs = osd_prologue<NW>(a.code, a.y + (size_t)f * N, sy, sord, rows, base);
        if (a.keys) {            // full-list path: keep the basis for the materialise pass
            uint32_t* gb = a.basis + (size_t)f * (K + 1) * NW;
            for (int i = lane; i < K * NW; i += 32) gb[i] = rows[i];
            if (lane < NW) gb[K * NW + lane] = base[lane];
        }
        // ---- candidates: contiguous chunk per lane, lexicographic successor
        const long long chunk = (a.C + 31) / 32;
        const long long i0 = (long long)lane * chunk;
        const long long i1 = min(a.C, i0 + chunk);
        uint64_t R = i0 < i1 ? osd_unrank(i0, K, a.order, binom) : 0ull;
        int cnt = 0;
        double thr_k = CUDART_INF;
        int thr_i = 0x7fffffff;
        for (long long s = 0; s < chunk; s++) {
            const long long idx = i0 + s;
            const bool valid = idx < i1;
            double key = CUDART_INF;
            if (valid) {
                uint32_t c[NW];
                osd_word<NW>(rows, base, R, K, c);
                if (a.keys) a.keys[(size_t)f * a.C + idx] = osd_ced<NW>(sy, c, N);
                else key = -osd_corr<NW>(sy, c, N);
                R = osd_next(R, K);
            }
            if (a.keys) continue;
            bool pass = valid && (cnt < keep || osd_less(key, (int)idx, thr_k, thr_i));
            unsigned ball = __ballot_sync(MPW_FULL, pass);
            while (ball) {
                const int src = __ffs(ball) - 1;
                ball &= ball - 1;
                const double kk = __shfl_sync(MPW_FULL, key, src);
                const int ii = __shfl_sync(MPW_FULL, (int)idx, src);
                if (!(cnt < keep || osd_less(kk, ii, thr_k, thr_i))) continue;
                int below = 0;
                for (int e = lane; e < cnt; e += 32) below += osd_less(tk[e], ti[e], kk, ii) ? 1 : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(MPW_FULL, below, o);
                const int last = min(cnt, keep - 1);            // entries [below, last) shift right
                double mk[3];
                int mi[3];
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    const int e = lane + 32 * q;
                    if (e > below && e <= last) { mk[q] = tk[e - 1]; mi[q] = ti[e - 1]; }
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    const int e = lane + 32 * q;
                    if (e > below && e <= last) { tk[e] = mk[q]; ti[e] = mi[q]; }
                }
                if (lane == 0) { tk[below] = kk; ti[below] = ii; }
                cnt = min(cnt + 1, keep);
                __syncwarp();
                if (cnt == keep) { thr_k = tk[keep - 1]; thr_i = ti[keep - 1]; }
            }
        }
        if (a.keys) continue;
        // ---- canonical EDs of the kept entries; re-sort them by (ED, index) so the
        // reported scores are the sort keys, as in the reference (:310-316)
        double ced[3];
        int cid[3], pos[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const int e = lane + 32 * q;
            if (e < cnt) {
                uint32_t c[NW];
                cid[q] = ti[e];
                osd_word<NW>(rows, base, osd_unrank(cid[q], K, a.order, binom), K, c);
                ced[q] = osd_ced<NW>(sy, c, N);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 3; q++)
            if (lane + 32 * q < cnt) tk[lane + 32 * q] = ced[q];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 3; q++) {
            if (lane + 32 * q < cnt) {
                int r = 0;
                for (int j = 0; j < cnt; j++) r += osd_less(tk[j], ti[j], ced[q], cid[q]) ? 1 : 0;
                pos[q] = r;
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 3; q++)
            if (lane + 32 * q < cnt) { tk[pos[q]] = ced[q]; ti[pos[q]] = cid[q]; }
        __syncwarp();
        // ---- near-tie certification of the kept order and the M boundary
        const int m_eff = (int)min((long long)a.M, a.C);
        const double tol = 1e-12 * (yabs + 1.0) * (double)N;
        bool tie = false;
        for (int e = lane; e + 1 < cnt && e < m_eff; e += 32) tie |= (tk[e + 1] - tk[e]) <= tol;
        tie = __any_sync(MPW_FULL, tie);
        if (lane == 0 && a.s1flags) a.s1flags[f] = tie ? MPW_F_TIE_STAGE1 : 0;
        if (a.mode == 0) {
            if (lane == 0) a.list_n[f] = m_eff;
            for (int e = lane; e < m_eff; e += 32) {
                uint32_t c[NW];
                osd_word<NW>(rows, base, osd_unrank(ti[e], K, a.order, binom), K, c);
                uint32_t* o = a.list_cw + ((size_t)f * a.M + e) * NW;
#pragma unroll
                for (int w = 0; w < NW; w++) o[w] = c[w];
                a.list_ed[(size_t)f * a.M + e] = tk[e];
            }
        } else if (a.mode == 1) {
            // every candidate is a codeword of `code`, so the CRC gate
            // (decoders.py:559-570) passes on the first entry, kept as-is
            uint32_t c[NW];
            osd_word<NW>(rows, base, osd_unrank(ti[0], K, a.order, binom), K, c);
            if (lane == 0) {
#pragma unroll
                for (int w = 0; w < NW; w++) a.out.best[(size_t)f * NW + w] = c[w];
                a.out.stage[f] = 0;
                a.out.best_ed[f] = tk[0];
            }
        } else {
            // always_on: anchors = first A entries, already in the subcode (decoders.py:572-576)
            const int na = min(a.A, m_eff);
            int q = 0;
            if (lane == 0) q = atomicAdd(a.s2.count, 1);
            q = __shfl_sync(MPW_FULL, q, 0);
            for (int e = lane; e < na; e += 32) {
                uint32_t c[NW];
                osd_word<NW>(rows, base, osd_unrank(ti[e], K, a.order, binom), K, c);
                uint32_t* o = a.s2.anchors + ((size_t)q * a.A + e) * NW;
#pragma unroll
                for (int w = 0; w < NW; w++) o[w] = c[w];
            }
            if (lane == 0) { a.s2.frame[q] = f; a.s2.nanchor[q] = na; a.out.stage[f] = 1; }
        }
        __syncwarp();
    }
}

// Full-list path (list_cap > OSD_MAX_KEEP - 1): osd_kernel wrote every key and
// the reduced basis; the caller sorted (key, index) stably per frame; one warp
// per frame writes the first M words and canonical EDs.
template <int NW>
__global__ void __launch_bounds__(32 * OSD_WARPS) osd_materialize_kernel(OsdArgs a, const int32_t* sorted_idx,
                                                                        const double* sorted_key) {
    __shared__ unsigned long long binom[64 * (OSD_MAX_ORDER + 1)];
    osd_binom_init(binom);
    __syncthreads();
    const int N = a.code.n, K = a.code.k, lane = threadIdx.x & 31;
    const int m_eff = (int)min((long long)a.M, a.C);
    const int nwarps = gridDim.x * OSD_WARPS;
    for (int f = blockIdx.x * OSD_WARPS + (threadIdx.x >> 5); f < a.F; f += nwarps) {
        const uint32_t* gb = a.basis + (size_t)f * (K + 1) * NW;
        const float* yr = a.y + (size_t)f * N;
        double yabs = 0.0;
        for (int i = lane; i < N; i += 32) yabs += fabs((double)yr[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) yabs += __shfl_xor_sync(MPW_FULL, yabs, o);
        const double tol = 1e-12 * (yabs + 1.0) * (double)N;
        bool tie = false;
        for (long long e = lane; e + 1 < a.C && e < m_eff; e += 32)
            tie |= (sorted_key[(size_t)f * a.C + e + 1] - sorted_key[(size_t)f * a.C + e]) <= tol;
        tie = __any_sync(MPW_FULL, tie);
        if (lane == 0 && a.s1flags) a.s1flags[f] = tie ? MPW_F_TIE_STAGE1 : 0;
        if (lane == 0) a.list_n[f] = m_eff;
        for (int e = lane; e < m_eff; e += 32) {
            uint32_t c[NW];
            osd_word<NW>(gb, gb + K * NW, osd_unrank(sorted_idx[(size_t)f * a.C + e], K, a.order, binom), K, c);
            uint32_t* o = a.list_cw + ((size_t)f * a.M + e) * NW;
#pragma unroll
            for (int w = 0; w < NW; w++) o[w] = c[w];
            a.list_ed[(size_t)f * a.M + e] = sorted_key[(size_t)f * a.C + e];
        }
    }
}
