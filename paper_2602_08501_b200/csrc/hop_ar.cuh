// Stage 2, asynchronous-row int8 tensor hop (MPW_HOP_TENSOR_I8_ASYNC).
//
// Same contraction as the int8 screen of hop_tc.cuh (decoders.py:329-357):
//     Q[r, p] = Σ_i q[r, i] · P[p, i],   t = x ⊙ y ≈ s·q,   ΔED = 4 S
// with tcgen05.mma.kind::i8 into s32 TMEM accumulators, but without rounds:
// the P tiles stream cyclically and never stop, and every trajectory row runs
// its own scan cycle (ntiles consecutive tiles starting at any tile).  The
// scan warps do no insertion and take no data-dependent branch per tile: per
// 32-pattern group they keep the group minimum, update the row's running
// minimum, and append the groups whose minimum lies inside the certification
// window of the running minimum to a per-thread hit list in shared memory (a
// predicated store).  When a row's cycle ends its bit is set in a ready mask;
// any of the worker warps takes it, keeps the hit groups inside the window of
// the final minimum m, recomputes the exact integer scores Q_p of their
// patterns (lane = pattern: popcounts of the pattern words against the eight bit
// planes of the row's int8 image, no cross-lane reduction), scores every pattern with
// Q_p < m + wq from y in fp32, certifies the argmin / accept decision
// (decoders.py:385-398) with the recursive-summation bound or re-scores the
// finalists in float64, applies the move to the row's int8 image (or stores the
// trajectory and builds the next one of the stage-2 queue), and publishes the
// tile at which the row's next cycle starts.  Rows are dead only between their
// cycle end and that tile (about ten tiles of 244 at cfg4); no CTA-wide round
// end exists, so the MMA stream is continuous.
//
// Exactness: a pattern outside every kept group has Q_p >= m + wq for the
// row's final minimum m, hence S_p > S_best + thr by the frame's quantisation
// bound (same window as the synchronous int8 screen, common.cuh warp_i8_scale);
// every pattern with Q_p < m + wq is scored from y, so the decision is the
// exact one.  A hit list that overflows (CAP entries per thread and cycle)
// makes the row scan once more with the achieved minimum as the seed of the
// running minimum (then only true window groups are recorded); the extra scan
// is not counted in iterations_used.
//
// CTA = 20 warps (NCOL = 2), persistent, one per SM:
//   warp 0        producer: cp.async.bulk of 32 KB pre-swizzled u8 P stages
//   warps 1, 2    TMEM allocator + two tcgen05.mma issuer threads on alternate tiles (warp 3
//                 idle: it fills the warpgroup)
//   warps 4..11   scan: NCOL per TMEM lane quarter, 256 / NCOL columns of every tile each
//   warps 12..19  workers: decisions, moves, refills
// Register budgets (setmaxnreg; the CTA's pool is what its own warps release): warps 0..3
// drop from 96 to 40 registers, the workers take 120, the scan warps stay at 96.  (NCOL = 4,
// 16 scan warps of 64 columns at 64 registers with workers at 104, compiles and is correct but
// measured slower: seven warps per scheduler.)
#pragma once
#include "hop_tc.cuh"

namespace ar {
using namespace tc;

#ifndef MPW_AR_NWORK
#define MPW_AR_NWORK 8
#endif
constexpr int NWORK = MPW_AR_NWORK;            // worker warps (any worker takes any ready row)
#ifndef MPW_AR_NCOL
#define MPW_AR_NCOL 2
#endif
constexpr int NCOL = MPW_AR_NCOL;              // scan threads per row: each scans 256 / NCOL columns of every tile
static_assert(NCOL == 2 || NCOL == 4, "column parts per row");
constexpr int SCAN_T = ROWS * NCOL;            // scan threads
constexpr int NLD = I8_TILE / NCOL / 64;       // 64-column TMEM loads per scan thread and tile
constexpr int NGRP = I8_TILE / NCOL / 32;      // 32-pattern groups per scan thread and tile
// warps 0..3: producer, two MMA issuers, one idle (one warpgroup, so the register budgets
// can be set per warpgroup); then the scan warps; then the workers
constexpr int SCAN_W0 = 4;
constexpr int WORK_W0 = SCAN_W0 + SCAN_T / 32;
constexpr int THREADS = 32 * (WORK_W0 + NWORK);
static_assert(NWORK % 4 == 0, "worker warps in whole warpgroups");
constexpr int CAP = NCOL == 2 ? 22 : 11;       // hit-list entries per scan thread and cycle
constexpr int RSW = 16;                        // 32-bit words of a row's state in shared memory
constexpr int AR_STAGES = 5;                   // P ring stages (one 128-position K-block of a tile each)
constexpr int Q_INF = 0x7FFF;                  // s16 maximum: "no score"
#ifndef MPW_AR_NISS
#define MPW_AR_NISS 2
#endif
constexpr int NISS = MPW_AR_NISS;             // MMA issuer threads (alternate tiles)
static_assert(NISS == 1 || NISS == 2, "one issuer per accumulator");
constexpr int MARGIN = 2;                      // tiles between the issue counter read and a row's first live tile
static_assert(CAP <= 32, "one hit entry per worker lane");
// a hit entry names a group of 32 patterns in 16 bits: |P| <= 2^17 gives 4096 groups

struct Params {
    int n, nw, A, T, np, ntiles;
    const float* y;
    const double* y64;           // float64 inputs: the caller's received words (y = their fp32 rounding), else null
    S2Dev s2;
    const uint32_t* pbits;       // np x nw
    const uint8_t* btiles;       // [ntiles][KB][256 x 128 u8] swizzled images
    float tie_rel;
    int cap;                     // hit-list entries per scan thread and cycle in use (<= CAP)
    float cert_g;                // fp32 summation bound factor (cert_gamma)
    unsigned long long* stats;   // STATS builds: counters (see hop_ar.cu)
    unsigned long long* tilestat;   // optional (any build): [0] += tiles, [1] += clock64 cycles of issuer 0, per CTA
    int experiment;              // STATS builds, timing probes (results wrong): 2 workers decide "no move" without
                                 // scoring, 4 the producer stops copying once the ring is full, 8 scan skips the TMEM loads,
                                 // 16 workers skip the proxy fence, 64 workers skip the fp32 scoring of the window patterns,
                                 // 128 workers skip the bit-plane filter
};

__host__ __device__ constexpr size_t smem_bytes(int kb) {
    return (size_t)kb * A_KBLK_BYTES + (size_t)AR_STAGES * I8_STAGE_BYTES + (size_t)CAP * SCAN_T * 4 +
           ROWS * 8 /*row_ctl*/ + ROWS * 4 /*row_best*/ + ROWS * 4 /*row_done*/ + SCAN_T /*hit_cnt*/ +
           ROWS * RSW * 4 /*row state*/ + 16 /*ready mask*/ +
           (2 * AR_STAGES + 4) * 8 /*barriers*/ + 16 /*tmem slot, stop tile, issue counter, rows left*/ +
           NWORK * 256 /*bit planes of the row a worker is deciding*/;
}

__device__ __forceinline__ uint2 ld_shared_volatile_v2(const uint2* p) {
    uint2 v;
    asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void st_shared_volatile_v2(uint2* p, uint2 v) {
    asm volatile("st.volatile.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_volatile_u32(const volatile uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(const_cast<const uint32_t*>(p))));
    return v;
}
__device__ __forceinline__ void st_shared_volatile_u32(volatile uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(const_cast<uint32_t*>(p))), "r"(v) : "memory");
}

// predicated shared-memory store / minimum / trap: one predicated instruction each, no branch
// (the compiler turns the equivalent `if` into a divergent branch with a reconvergence barrier)
__device__ __forceinline__ void st_shared_if(uint32_t addr, uint32_t v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void red_min_shared_if(uint32_t addr, int v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.min.s32 [%0], %1;\n\t}" ::"r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void trap_if(bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q trap;\n\t}" ::"r"((uint32_t)p));
}

// minimum of 32 packed s16 values (registers o .. o + 15): 8 three-input instructions
template <int NV>
__device__ __forceinline__ int min32_s16_b(const uint32_t (&v)[NV], int o) {
    if constexpr (NV < 32) {
        return 0x7FFF;
    } else {
        const uint32_t a = min3_s16x2(v[o], v[o + 1], v[o + 2]), b = min3_s16x2(v[o + 3], v[o + 4], v[o + 5]);
        const uint32_t c = min3_s16x2(v[o + 6], v[o + 7], v[o + 8]), d = min3_s16x2(v[o + 9], v[o + 10], v[o + 11]);
        const uint32_t e = min3_s16x2(v[o + 12], v[o + 13], v[o + 14]);
        const uint32_t f = min3_s16x2(a, b, c), g = min3_s16x2(d, e, v[o + 15]);
        uint32_t r;
        asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(f), "r"(g));
        return min((int)(short)(r & 0xFFFFu), (int)(short)(r >> 16));
    }
}
__device__ __forceinline__ int min32_s16(const uint32_t (&v)[32], int o) {
    const uint32_t a = min3_s16x2(v[o], v[o + 1], v[o + 2]), b = min3_s16x2(v[o + 3], v[o + 4], v[o + 5]);
    const uint32_t c = min3_s16x2(v[o + 6], v[o + 7], v[o + 8]), d = min3_s16x2(v[o + 9], v[o + 10], v[o + 11]);
    const uint32_t e = min3_s16x2(v[o + 12], v[o + 13], v[o + 14]);
    const uint32_t f = min3_s16x2(a, b, c), g = min3_s16x2(d, e, v[o + 15]);
    uint32_t r;
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(f), "r"(g));
    return min((int)(short)(r & 0xFFFFu), (int)(short)(r >> 16));
}

// minimum of 64 packed s16 values (32 registers): 16 three-input instructions
__device__ __forceinline__ int min64_s16_only(const uint32_t (&v)[32]) {
    uint32_t m[11];
#pragma unroll
    for (int e = 0; e < 10; e++) m[e] = min3_s16x2(v[3 * e], v[3 * e + 1], v[3 * e + 2]);
    uint32_t r;
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(v[30]), "r"(v[31]));
    m[10] = r;
    const uint32_t q0 = min3_s16x2(m[0], m[1], m[2]), q1 = min3_s16x2(m[3], m[4], m[5]);
    const uint32_t q2 = min3_s16x2(m[6], m[7], m[8]), q3 = min3_s16x2(m[9], m[10], q0);
    const uint32_t f = min3_s16x2(q1, q2, q3);
    return min((int)(short)(f & 0xFFFFu), (int)(short)(f >> 16));
}

// barrier waits of the producer and the issuer: 1 = spin on try_wait, 0 = try_wait with a
// suspend-time hint (the thread sleeps until the phase completes)
#ifndef MPW_AR_SPIN
#define MPW_AR_SPIN 0
#endif
__device__ __forceinline__ void ar_wait(uint32_t bar, uint32_t parity) {
#if MPW_AR_SPIN
    mbar_wait(bar, parity);
#else
    while (!mbar_try_hint(bar, parity)) {}
#endif
}

#ifndef MPW_AR_BACKOFF
#define MPW_AR_BACKOFF 1000
#endif

// stats slots
enum { ST_TILES = 0, ST_LIVE, ST_ROWCYC, ST_CHUNKS, ST_F64, ST_OVF, ST_BUSY, ST_FINISHED, ST_ENTRIES,
       ST_SCAN_WAIT, ST_SCAN_TOT, ST_ISS_FULL, ST_ISS_TEMPTY, ST_ISS_TOT, ST_W_LIST, ST_W_CHUNK, ST_W_DECIDE, ST_W_CLAIM,
       ST_W_PUBLISH, ST_W_POCKET, ST_ISS_MMA, ST_DEAD, ST_N };

template <int KB, int NW, bool STATS>
__global__ void __launch_bounds__(THREADS, 1) hop_ar_kernel(Params prm) {
    constexpr int STAGES = AR_STAGES;
    constexpr int STB = I8_STAGE_BYTES;
    extern __shared__ __align__(1024) unsigned char sm[];
    if ((smem_u32(sm) & 1023u) != 0u) __trap();   // SW128 operands need 1024-byte alignment
    unsigned char* a_rows = sm;
    unsigned char* b_ring = sm + KB * A_KBLK_BYTES;
    uint32_t* hits = reinterpret_cast<uint32_t*>(b_ring + STAGES * STB);    // [CAP][SCAN_T], slot-major
    uint2* row_ctl = reinterpret_cast<uint2*>(hits + CAP * SCAN_T);         // [ROWS] {start tile, wq << 16 | seed + 8192}
    int* row_best = reinterpret_cast<int*>(row_ctl + ROWS);                 // [ROWS] running minimum over both halves
    int* row_done = row_best + ROWS;                                        // [ROWS] halves that finished the cycle
    uint8_t* hit_cnt = reinterpret_cast<uint8_t*>(row_done + ROWS);         // [SCAN_T] entries recorded in the cycle
    uint32_t* row_state = reinterpret_cast<uint32_t*>(hit_cnt + SCAN_T);    // [ROWS][RSW]: c[8], trajectory, frame, iters | flags | recyc, ed, err, inv_s, sum|y|, wq
    uint32_t* ready_mask = row_state + ROWS * RSW;                          // [4]: rows whose cycle ended (or that await their first trajectory)
    uint64_t* bars = reinterpret_cast<uint64_t*>(ready_mask + 4);
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    volatile uint32_t* stop_tile = tmem_slot + 1;    // first tile nobody processes (0xFFFFFFFF while rows are left)
    volatile uint32_t* issue_ctr = tmem_slot + 2;    // tile whose MMAs the issuer is about to issue
    int* rows_left = reinterpret_cast<int*>(tmem_slot + 3);
    unsigned char* planes = reinterpret_cast<unsigned char*>(tmem_slot + 4);   // [NWORK][8 planes][32 bytes]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = prm.n, A = prm.A, T = prm.T, np_ = prm.np, ntiles = prm.ntiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) { mbar_init(smem_u32(&empty[s]), 1); }
        for (int b = 0; b < 2; b++) { mbar_init(smem_u32(&tfull[b]), 1); mbar_init(smem_u32(&tempty[b]), 4 * NCOL + 1); }   // tempty: the scan warps' releases + the producer's arrival with the tile's bytes
        *stop_tile = 0xFFFFFFFFu;
        *issue_ctr = 0u;
        *rows_left = ROWS;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int r = threadIdx.x; r < ROWS; r += THREADS) {
        row_ctl[r] = make_uint2(0x80000000u, 0u);
        row_best[r] = 0x7FFFFFFF;
        row_done[r] = 0;
    }
    for (int r = threadIdx.x; r < SCAN_T; r += THREADS) hit_cnt[r] = 0;
    for (int r = threadIdx.x; r < ROWS * RSW; r += THREADS) row_state[r] = (r % RSW) == 8 ? 0xFFFFFFFFu : 0u;   // no trajectory yet
    if (threadIdx.x < 4) ready_mask[threadIdx.x] = 0xFFFFFFFFu;   // every row awaits its first trajectory
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // register budgets per warpgroup (an increase can only take what decreases in the same CTA
    // released: NCOL = 2, from 96: 4 x 32 x 56 >= 8 x 32 x 24; NCOL = 4, from 72: 4 x 32 x 32 + 16 x 32 x 8 = 8 x 32 x 32)
    if (warp < SCAN_W0) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      if (warp == 0) {
        // ===== producer: the P tiles, cyclically, until the stop tile
        if (lane == 0) {
            int stage = 0, j = 0;
            uint32_t phase = 0;
            for (uint32_t gt = 0;; gt++) {
                if (gt >= ld_shared_volatile_u32(stop_tile)) break;
                // One barrier per accumulator collects what tile gt's MMAs wait for: the scan
                // warps' releases of tile gt - 2 and both stages of tile gt.  Its previous phase
                // (tile gt - 2) must be complete before this tile's arrival joins the next.
                const uint32_t gb = smem_u32(&tempty[gt & 1u]);
                if (gt >= 2) ar_wait(gb, (((gt >> 1) & 1u) ^ 1u));
                const bool probe = STATS && (prm.experiment & 4) && gt >= 4;   // timing probe: no P traffic
                if (probe) mbar_arrive(gb);
                else mbar_expect_tx(gb, KB * STB);
                for (int kb = 0; kb < KB; kb++) {
                    ar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    if (!probe) bulk_g2s(smem_u32(b_ring + stage * STB), prm.btiles + ((size_t)j * KB + kb) * STB, STB, gb);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (++j == ntiles) j = 0;
            }
        }
      } else if (warp == 1 || (NISS == 2 && warp == 2)) {
        // ===== MMA issuers: one M128 N256 tile per step, K = 32 per instruction.  Two
        // threads (warps 1 and 2) take alternate tiles, each with its own accumulator:
        // while one runs through the barrier check of its next tile, the other's MMAs keep
        // the tensor pipe fed (one thread alone leaves the pipe idle ~20 % of the time: its
        // per-tile waits, fences and commits outlast the few MMAs the pipe can queue).  A
        // tile waits on one barrier only (the accumulator's: releases + the tile's bytes)
        if (lane == 0) {
            const uint32_t which = (uint32_t)(warp - 1);
            const uint32_t idesc = (2u << 4) | (1u << 7) | ((uint32_t)(I8_TILE >> 3) << 17) | ((uint32_t)(ROWS >> 4) << 24);
            const uint32_t abase = smem_u32(a_rows), bring = smem_u32(b_ring);
            const uint32_t ictr = smem_u32(const_cast<uint32_t*>(issue_ctr));
            long long w_full = 0, w_tempty = 0, w_mma = 0, t_0 = 0, t_a = 0;
            if (STATS || prm.tilestat) t_0 = clock64();
            uint32_t gt_end = 0;
            for (uint32_t gt = which;; gt += NISS) {
                gt_end = gt;
                if (gt >= ld_shared_volatile_u32(stop_tile)) break;
                const uint32_t buf = gt & 1u;
                if (STATS) t_a = clock64();
                ar_wait(smem_u32(&tempty[buf]), (gt >> 1) & 1u);
                if (STATS) w_tempty += clock64() - t_a;
                tc_fence_after();
                // published (as a running maximum) before the tile's MMAs are issued: a
                // worker that reads v knows that no MMA of a tile beyond v has been issued yet
                asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(ictr), "r"(gt) : "memory");
                const uint32_t d = tmem_base + buf * I8_TILE;
                for (int kb = 0; kb < KB; kb++) {
                    const uint32_t u = gt * KB + kb;           // K-block number -> ring stage and phase
                    const uint32_t stage = u % STAGES;
                    const uint64_t bd = sw128_desc(bring + stage * STB);
                    const uint64_t ad = sw128_desc(abase + kb * A_KBLK_BYTES);
                    if (STATS) t_a = clock64();
#pragma unroll
                    for (int ks = 0; ks < 4; ks++) tc_mma_i8(d, ad + 2 * ks, bd + 2 * ks, idesc, (kb | ks) != 0);
                    tc_commit(smem_u32(&empty[stage]));
                    if (STATS) w_mma += clock64() - t_a;
                }
                tc_commit(smem_u32(&tfull[buf]));
            }
            if (prm.tilestat && which == 0) {
                atomicAdd(&prm.tilestat[0], (unsigned long long)gt_end);
                atomicAdd(&prm.tilestat[1], (unsigned long long)(clock64() - t_0));
            }
            if (STATS && which == 0) {
                atomicAdd(&prm.stats[ST_ISS_FULL], (unsigned long long)w_full);
                atomicAdd(&prm.stats[ST_ISS_TEMPTY], (unsigned long long)w_tempty);
                atomicAdd(&prm.stats[ST_ISS_MMA], (unsigned long long)w_mma);
                atomicAdd(&prm.stats[ST_ISS_TOT], (unsigned long long)(clock64() - t_0));
            }
        }
      }
    } else if (warp < WORK_W0) {
        if (NCOL == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        // ===== scan: thread = (row, column part); no data-dependent branch per tile
        const int g = warp & 3;                      // TMEM lane quarter of this warp
        const int colq = (warp - SCAN_W0) >> 2;      // column part of this warp
        const int row = g * 32 + lane;
        const int thr = colq * ROWS + row;
        const int col0 = colq * (I8_TILE / NCOL);
        const uint32_t t_lane = tmem_base + ((uint32_t)(g * 32) << 16);
        const int cap = prm.cap;
        if (lane == 0) {   // no release precedes the first two tiles: the scan warps arrive for them up front
            mbar_arrive(smem_u32(&tempty[0]));
            mbar_arrive(smem_u32(&tempty[1]));
        }
        uint32_t seen = 0x80000000u;                 // start tile of the cycle this thread knows
        const uint32_t hits_addr = smem_u32(hits) + (uint32_t)thr * 4u, best_addr = smem_u32(&row_best[row]);
        int cnt = 0, m_run = Q_INF, pub = 0x7FFFFFFF, wq = 0;
        int j = 0;
        unsigned long long st_live = 0, st_tiles = 0, st_entries = 0;
        long long sw_wait = 0, sw_0 = 0, sw_a = 0;
        if (STATS) sw_0 = clock64();
        for (uint32_t gt = 0;; gt++) {
            if (gt >= ld_shared_volatile_u32(stop_tile)) break;
            const uint32_t buf = gt & 1u;
            if (STATS) sw_a = clock64();
            while (!mbar_try_hint(smem_u32(&tfull[buf]), (gt >> 1) & 1u)) {}
            if (STATS) sw_wait += clock64() - sw_a;
            tc_fence_after();
            uint32_t va[32], vb[NLD == 2 ? 32 : 1];
            const uint32_t tbase = t_lane + buf * I8_TILE + col0;
            if (STATS && (prm.experiment & 8)) {
#pragma unroll
                for (int e = 0; e < 32; e++) { va[e] = 0x00010001u * (uint32_t)(e + lane); if (NLD == 2) vb[e] = va[e]; }
            } else {
                TC_LD32P(tbase, va);
                if constexpr (NLD == 2) TC_LD32P(tbase + 64, vb);
            }
            // the row's control word, then the other half's published minimum (in this
            // order: a new control word implies the reset of the minimum is visible)
            const uint2 ctl = ld_shared_volatile_v2(&row_ctl[row]);
            const int shb = ld_shared_volatile(&row_best[row]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // the accumulator goes back to the issuer; the scan below overlaps the next MMAs
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty[buf]));
            const int pa = j * I8_TILE + col0;
            // (no tail mask: the image columns past |P| repeat pattern 0, hop_tc.cu tc_build8)
            // minima of the thread's 32-pattern groups (16 packed registers each)
            int mg[NGRP];
            mg[0] = min32_s16(va, 0);
            mg[1] = min32_s16(va, 16);
            if constexpr (NLD == 2) {
                mg[2] = min32_s16_b(vb, 0);
                mg[3] = min32_s16_b(vb, 16);
            }
            const bool isnew = ctl.x != seen;
            seen = ctl.x;
            // a new cycle: counters reset, the running minimum starts from the seed
            cnt = isnew ? 0 : cnt;
            m_run = isnew ? (int)(ctl.y & 0xFFFFu) - KEY_BIAS : m_run;
            pub = isnew ? 0x7FFFFFFF : pub;
            wq = isnew ? (int)(ctl.y >> 16) : wq;
            trap_if(isnew && gt > ctl.x);   // the start tile was observed late: protocol violation, fail the launch
            const uint32_t age = gt - seen;
            const bool live = age < (uint32_t)ntiles;
            int mt = min(mg[0], mg[1]);
            if constexpr (NLD == 2) mt = min(mt, min(mg[2], mg[3]));
            m_run = live ? min(m_run, min(mt, shb)) : m_run;
            const int lim = m_run + wq;
            const uint32_t grp0 = (uint32_t)pa >> 5;
            auto record = [&](int m, uint32_t grp) {
                const bool h = live && m < lim && !(STATS && (prm.experiment & 8));
                st_shared_if(hits_addr + (uint32_t)cnt * (SCAN_T * 4), ((uint32_t)(m + KEY_BIAS) << 16) | grp, h && cnt < cap);
                cnt += h ? 1 : 0;
            };
#pragma unroll
            for (int k = 0; k < NGRP; k++) record(mg[k], grp0 + (uint32_t)k);
            const bool lower = live && mt < pub;
            red_min_shared_if(best_addr, mt, lower);
            pub = lower ? mt : pub;
            if (STATS) { st_tiles++; st_live += live ? 1 : 0; }
            if (live && age == (uint32_t)(ntiles - 1)) {
                // cycle end: hand the hit list to the row's worker
                if (STATS) st_entries += cnt;
                hit_cnt[thr] = (uint8_t)min(cnt, 255);
                __threadfence_block();
                if (atomicAdd(&row_done[row], 1) == NCOL - 1) atomicOr(&ready_mask[row >> 5], 1u << (row & 31));   // all parts done
            }
            if (++j == ntiles) j = 0;
        }
        if (STATS) {
            atomicAdd(&prm.stats[ST_TILES], st_tiles);
            atomicAdd(&prm.stats[ST_LIVE], st_live);
            atomicAdd(&prm.stats[ST_ENTRIES], st_entries);
            if (lane == 0) {
                atomicAdd(&prm.stats[ST_SCAN_WAIT], (unsigned long long)sw_wait);
                atomicAdd(&prm.stats[ST_SCAN_TOT], (unsigned long long)(clock64() - sw_0));
            }
        }
    } else {
        if (NCOL == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 120;");
        // ===== workers: any worker takes any ready row (a bit mask of rows whose cycle
        // ended); the row's state lives in shared memory between its cycles
        const int w = warp - WORK_W0;
        const int count = *prm.s2.count;
        const int ntraj = count * A;
        // next trajectory of the stage-2 queue (queue slot x anchor; short lists skip), claimed
        // when a row needs one.  (Claiming ahead into a per-worker pocket saved ~1.5k cycles per
        // trajectory but could strand the pocket of a worker that gets no more rows at the end.)
        auto claim_next = [&](int& nq) -> int {
            int ntr = -1;
            nq = 0;
            if (lane == 0) {
                for (;;) {
                    const int cand = atomicAdd(prm.s2.work_next, 1);
                    if (cand >= ntraj) break;
                    const int q = cand / A, a = cand - q * A;
                    if (a >= prm.s2.nanchor[q]) continue;
                    ntr = cand;
                    nq = q;
                    break;
                }
            }
            nq = __shfl_sync(MPW_FULL, nq, 0);
            return __shfl_sync(MPW_FULL, ntr, 0);
        };
        unsigned long long st_rowcyc = 0, st_chunks = 0, st_f64 = 0, st_ovf = 0, st_busy = 0, st_fin = 0, st_dead = 0;
        long long ph[6] = {0, 0, 0, 0, 0, 0}, t_ph = 0;
#define PH(k) if (STATS) { const long long t_ = clock64(); ph[k] += t_ - t_ph; t_ph = t_; }
        for (;;) {
            if (ld_shared_volatile_u32(stop_tile) != 0xFFFFFFFFu) break;
            // a ready row: every worker starts its search at a different word of the mask
            const int wi_l = (lane + w) & 3;
            const uint32_t mw = lane < 4 ? ld_shared_volatile_u32(ready_mask + wi_l) : 0u;
            const unsigned has = __ballot_sync(MPW_FULL, mw != 0u);
            // (workers on the MMA issuers' schedulers, warps 1 and 2 mod 4, yield to the others)
            if (!has) { __nanosleep(((warp & 3) == 1 || (warp & 3) == 2) ? MPW_AR_BACKOFF : 100); continue; }
            long long t_busy0 = 0;
            if (STATS) { t_busy0 = clock64(); t_ph = t_busy0; }
            const int srcl = __ffs(has) - 1;
            const int wi = (srcl + w) & 3;
            const uint32_t mword = __shfl_sync(MPW_FULL, mw, srcl);
            const int bit = (w & 1) ? 31 - __clz(mword) : __ffs(mword) - 1;   // two search directions: fewer collisions
            uint32_t old = 0u;
            if (lane == 0) old = atomicAnd(&ready_mask[wi], ~(1u << bit));
            old = __shfl_sync(MPW_FULL, old, 0);
            if (!((old >> bit) & 1u)) continue;   // another worker took it
            const int row = wi * 32 + bit;
            __threadfence_block();
            // the row's state
            const uint32_t sw = lane < RSW ? row_state[row * RSW + lane] : 0u;
            uint32_t c_[NW];
#pragma unroll
            for (int k = 0; k < NW; k++) c_[k] = __shfl_sync(MPW_FULL, sw, k);
            int tr_ = (int)__shfl_sync(MPW_FULL, sw, 8), frame_ = (int)__shfl_sync(MPW_FULL, sw, 9);
            const uint32_t packed = __shfl_sync(MPW_FULL, sw, 10);
            int iters_ = (int)(packed & 0xFFFFu);
            uint32_t flags_ = (packed >> 16) & 0xFFu;
            bool recyc_ = (packed >> 24) != 0u;
            float ed_ = __uint_as_float(__shfl_sync(MPW_FULL, sw, 11)), err_ = __uint_as_float(__shfl_sync(MPW_FULL, sw, 12));
            float inv_ = __uint_as_float(__shfl_sync(MPW_FULL, sw, 13)), ay_ = __uint_as_float(__shfl_sync(MPW_FULL, sw, 14));
            int wq_ = (int)__shfl_sync(MPW_FULL, sw, 15);
            int seed = Q_INF;
            bool need_claim = tr_ < 0;
            bool exhausted_ = false;
            if (tr_ >= 0) {
                // the frame's y (this lane's 8 positions) is on its way while the hit lists are read
                const float* yr = prm.y + (size_t)frame_ * n;
                float4 ya = make_float4(0.f, 0.f, 0.f, 0.f), yb = ya;
                const bool pos_on = lane * 8 < n;      // this lane holds positions 8 lane .. 8 lane + 7
                if (pos_on) {
                    const float4* y4 = reinterpret_cast<const float4*>(yr) + lane * 2;
                    ya = __ldg(y4);
                    yb = __ldg(y4 + 1);
                }
                __threadfence_block();
                // everything the decision reads from shared memory, issued together: the final
                // minimum, both halves' entry counts and entries, this lane's 8 int8 values
                uint2* const qptr = reinterpret_cast<uint2*>(a_rows + (lane >> 4) * A_KBLK_BYTES +
                                                             sw128_chunk(row, (lane & 15) >> 1) + (lane & 1) * 8);
                const int mfin = ld_shared_volatile(&row_best[row]);
                int cntq[NCOL];
                uint32_t entq[NCOL];
                const int hl = lane < CAP ? lane : 0;
#pragma unroll
                for (int q = 0; q < NCOL; q++) {
                    cntq[q] = hit_cnt[q * ROWS + row];
                    entq[q] = hits[hl * SCAN_T + q * ROWS + row];
                }
                uint2 q2 = make_uint2(0u, 0u);
                if (pos_on) q2 = *qptr;
                bool ovf = false;
#pragma unroll
                for (int q = 0; q < NCOL; q++) ovf = ovf || cntq[q] > prm.cap;
                if (STATS) st_rowcyc++;
                if (ovf && !recyc_) {
                    // hit list overflow: scan once more, recording only the groups inside
                    // the window of the achieved minimum
                    if (STATS) st_ovf++;
                    recyc_ = true;
                    seed = mfin;
                } else {
                    if (ovf) flags_ |= MPW_F_UNRESOLVED;
                    recyc_ = false;
                    const int limit = mfin + wq_;
                    PH(0);
                    // |fl(S) - S| of the fp32 sums (rounded up), the tie threshold, and the margin
                    // inside which two fp32 scores are not told apart
                    const float bnd = ay_ * prm.cert_g * 1.000001f;
                    const float thr = prm.tie_rel * ed_ * 0.25f;
                    const float Mf = (2.0f * bnd + thr) * 1.000001f;
                    // t = x ⊙ y of this lane's positions
                    float tv[8];
                    const uint32_t cw8 = select_word<NW>(c_, (lane >> 2) & (NW - 1)) >> ((lane & 3) * 8);
                    float Bs = CUDART_INF_F;
                    int Bi = 0x7FFFFFFF, nf = 0;
                    float fs = CUDART_INF_F;   // finalist `lane`: fp32 score, pattern
                    int fi = 0x7FFFFFFF;
                    bool tv_ready = false;
                    uint32_t pw = 0u;          // lanes < NW: word `lane` of the running best pattern
                    // Per hit group (32 patterns): lane j holds pattern j of the group (its NW
                    // words, one row-major load) and computes the exact integer score
                    // Q_j = sum_i q_i P[j, i] from the bit planes of the row's int8 image:
                    // Q_j = sum_{b < 7} 2^b popc(P_j & plane_b) - 128 popc(P_j & plane_7)
                    // (two's complement), planes read by broadcast from shared memory; no
                    // cross-lane reduction.  The patterns inside the window of the final minimum
                    // are then scored from y in fp32 (8 positions per lane, butterfly sum).
                    unsigned char* const pl = planes + (warp - WORK_W0) * 256;
                    bool planes_ready = false;
                    auto load_group = [&](int grp, uint4& t0, uint4& t1) {
                        t0 = make_uint4(0u, 0u, 0u, 0u);
                        t1 = t0;
                        const int pc = grp * 32 + lane;
                        if (pc < np_) {
                            const uint4* s4 = reinterpret_cast<const uint4*>(prm.pbits + (size_t)pc * NW);
                            t0 = __ldg(s4);
                            if (NW > 4) t1 = __ldg(s4 + 1);
                        }
                    };
                    auto do_group = [&](int grp, const uint4& t0, const uint4& t1) {
                        if (!planes_ready) {
                            // plane b, byte `lane` = bit b of this lane's 8 values (positions 8 lane ..)
#pragma unroll
                            for (int b = 0; b < 8; b++) {
                                const uint32_t lo4 = (((q2.x >> b) & 0x01010101u) * 0x01020408u) >> 24;
                                const uint32_t hi4 = (((q2.y >> b) & 0x01010101u) * 0x01020408u) >> 24;
                                pl[b * 32 + lane] = (unsigned char)(lo4 | (hi4 << 4));
                            }
                            __syncwarp();
                            planes_ready = true;
                        }
                        int Q = 0;
#pragma unroll
                        for (int b = 0; b < 8; b++) {   // (unrolled: 27.11 M cycles per launch; rolled 27.19, by 2 or 4: 27.16)
                            if (STATS && (prm.experiment & 128)) break;   // (128: timing probe without the filter)
                            const uint4 a0 = *reinterpret_cast<const uint4*>(pl + b * 32);
                            int c = __popc(t0.x & a0.x) + __popc(t0.y & a0.y) + __popc(t0.z & a0.z) + __popc(t0.w & a0.w);
                            if (NW > 4) {
                                const uint4 a1 = *reinterpret_cast<const uint4*>(pl + b * 32 + 16);
                                c += __popc(t1.x & a1.x) + __popc(t1.y & a1.y) + __popc(t1.z & a1.z) + __popc(t1.w & a1.w);
                            }
                            Q += (b == 7 ? -c : c) << b;
                        }
                        unsigned cm = __ballot_sync(MPW_FULL, grp * 32 + lane < np_ && Q < limit);
                        if (STATS && (prm.experiment & 64)) cm = 0u;          // timing probe: filter only
                        if (STATS) st_chunks++;
                        if (cm && !tv_ready) {
                            const float yv[8] = {ya.x, ya.y, ya.z, ya.w, yb.x, yb.y, yb.z, yb.w};
#pragma unroll
                            for (int k = 0; k < 8; k++)
                                tv[k] = __uint_as_float(__float_as_uint(yv[k]) ^ (((cw8 >> k) & 1u) << 31));
                            tv_ready = true;
                        }
                        while (cm) {
                            const int j = __ffs(cm) - 1;
                            cm &= cm - 1;
                            const int pc = grp * 32 + j;
                            const uint32_t byte =
                                pos_on ? (uint32_t)__ldg(reinterpret_cast<const unsigned char*>(prm.pbits) + (size_t)pc * (NW * 4) + lane) : 0u;
                            float sp = 0.f;
#pragma unroll
                            for (int k = 0; k < 8; k++)
                                if ((byte >> k) & 1u) sp += tv[k];
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(MPW_FULL, sp, o);
                            if (sp < Bs || (sp == Bs && pc < Bi)) {
                                Bs = sp;
                                Bi = pc;
                                // the running best's bits are fetched now; a move needs them later
                                if (lane < NW) pw = __ldg(prm.pbits + (size_t)pc * NW + lane);
                            }
                            // finalists: everything within the certification margin of the running best
                            // (the difference of two close floats is exact)
                            if (sp - Bs < Mf) {
                                if (lane == nf) { fs = sp; fi = pc; }
                                nf++;
                            }
                        }
                    };
                    // the row's hit groups: per column part a mask over its list slots; the next
                    // group's bytes are in flight while a group is scored
                    uint32_t mq[NCOL];
#pragma unroll
                    for (int q = 0; q < NCOL; q++)
                        mq[q] = __ballot_sync(MPW_FULL, lane < min(cntq[q], prm.cap) && (int)(entq[q] >> 16) - KEY_BIAS < limit);
                    if (STATS && (prm.experiment & 2)) {   // timing probe: no scoring
#pragma unroll
                        for (int q = 0; q < NCOL; q++) mq[q] = 0u;
                    }
                    // first pending (part, slot): its group, -1 if none; pop() removes it
                    auto peek = [&]() -> int {
                        int g = -1;
#pragma unroll
                        for (int q = NCOL - 1; q >= 0; q--)
                            if (mq[q]) g = (int)(__shfl_sync(MPW_FULL, entq[q], __ffs(mq[q]) - 1) & 0xFFFFu);
                        return g;
                    };
                    auto pop = [&]() {
                        bool done = false;
#pragma unroll
                        for (int q = 0; q < NCOL; q++)
                            if (!done && mq[q]) { mq[q] &= mq[q] - 1; done = true; }
                    };
                    uint4 n0, n1;
                    int gnext = peek();
                    if (gnext >= 0) load_group(gnext, n0, n1);
#pragma unroll 1
                    while (gnext >= 0) {
                        const int grp = gnext;
                        pop();
                        const uint4 t0 = n0, t1 = n1;
                        gnext = peek();
                        if (gnext >= 0) load_group(gnext, n0, n1);
                        do_group(grp, t0, t1);
                    }
                    PH(1);
                    if (nf > 32) flags_ |= MPW_F_UNRESOLVED;   // more near-equal scores than lanes
                    const bool keep = fs - Bs < Mf;
                    const int nk = __popc(__ballot_sync(MPW_FULL, keep));
                    int best = Bi;
                    bool improve = false;
                    float sb = 0.f;
                    const float aB = fabsf(Bs);
                    if (nk == 1 && aB > bnd && fabsf(aB - thr) > bnd * 1.000001f) {
                        // the fp32 decision is the exact one
                        improve = Bs < 0.f;
                        sb = Bs;
                        if (aB < thr) flags_ |= MPW_F_TIE_ACCEPT;
                    } else if (nk >= 1) {
                        // float64 scores of the finalists (ascending positions), one per lane
                        if (STATS) st_f64++;
                        double e = CUDART_INF;
                        if (keep) {
                            // rolled loops (same ascending-position sum as exact_score in common.cuh):
                            // this path decides 0.1 % of the row cycles, and its unrolled form was
                            // half of the kernel's code
                            e = 0.0;
                            const uint32_t* pb = prm.pbits + (size_t)fi * NW;
#pragma unroll 1
                            for (int wd = 0; wd < NW; wd++) {
                                const uint32_t cwd = select_word<NW>(c_, wd);
#pragma unroll 1
                                for (uint32_t b = __ldg(pb + wd); b; b &= b - 1) {
                                    const int i = __ffs(b) - 1;
                                    const double yi = prm.y64 ? __ldg(prm.y64 + (size_t)frame_ * n + wd * 32 + i)
                                                              : (double)__ldg(yr + wd * 32 + i);
                                    e += ((cwd >> i) & 1u) ? -yi : yi;
                                }
                            }
                        }
                        double be = e;
                        int bi = keep ? fi : 0x7FFFFFFF;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double oe = __shfl_xor_sync(MPW_FULL, be, o);
                            const int oi = __shfl_xor_sync(MPW_FULL, bi, o);
                            if (oe < be || (oe == be && oi < bi)) { be = oe; bi = oi; }
                        }
                        double e2 = (keep && fi != bi) ? e : CUDART_INF;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) e2 = fmin(e2, __shfl_xor_sync(MPW_FULL, e2, o));
                        best = bi;
                        if (e2 - be < (double)thr) flags_ |= MPW_F_TIE_ARGMIN;
                        improve = be < 0.0;
                        if (fabs(be) < (double)thr) flags_ |= MPW_F_TIE_ACCEPT;
                        sb = (float)be;
                    }
                    iters_++;
                    if (improve) {
                        // the move: c ^= p, the moved positions' int8 values negated
                        if (best != Bi) pw = lane < NW ? __ldg(prm.pbits + (size_t)best * NW + lane) : 0u;
#pragma unroll
                        for (int k = 0; k < NW; k++) c_[k] ^= __shfl_sync(MPW_FULL, pw, k);
                        const uint32_t word = __shfl_sync(MPW_FULL, pw, (lane >> 2) & (NW - 1));
                        const uint32_t b8 = (word >> ((lane & 3) * 8)) & 0xFFu;
                        if (b8 && pos_on) {
                            uint32_t m = byte_mask4(b8 & 0xFu);
                            q2.x = (q2.x & ~m) | (__vsub4(0u, q2.x) & m);
                            m = byte_mask4(b8 >> 4);
                            q2.y = (q2.y & ~m) | (__vsub4(0u, q2.y) & m);
                            *qptr = q2;
                        }
                        ed_ += 4.f * sb;
                        if (prm.s2.traj_hops && lane == 0) prm.s2.traj_hops[(size_t)tr_ * T + iters_ - 1] = best + 1;
                    }
                    if (!improve || iters_ == T) {
                        // the trajectory is complete (decoders.py:441-451)
                        if (prm.s2.traj_hops && lane == 0)
                            for (int h = iters_ - (improve ? 0 : 1); h < T; h++) prm.s2.traj_hops[(size_t)tr_ * T + h] = -1;
                        if (lane < NW) prm.s2.traj_cw[(size_t)tr_ * NW + lane] = select_word<NW>(c_, lane);
                        if (lane == 0) {
                            prm.s2.traj_iters[tr_] = iters_;
                            prm.s2.traj_flags[tr_] = (uint8_t)flags_;
                        }
                        if (STATS) st_fin++;
                        need_claim = true;
                    }
                }
            }
            PH(2);
            if (need_claim) {
                int nq;
                tr_ = claim_next(nq);
                if (tr_ < 0) {
                    exhausted_ = true;
                    if (lane == 0 && atomicSub(rows_left, 1) == 1) {
                        // the CTA's last row: everybody stops a few tiles past the issuer
                        // (beyond the producer's look-ahead of STAGES / KB tiles)
                        st_shared_volatile_u32(stop_tile, ld_shared_volatile_u32(issue_ctr) + 4u + STAGES);
                    }
                } else {
                    frame_ = prm.s2.frame[nq];
                    const float4 qs = prm.s2.qscale[nq];
                    inv_ = qs.x;
                    err_ = qs.z;
                    ay_ = qs.w;
                    const uint32_t aw = lane < NW ? __ldg(prm.s2.anchors + (size_t)tr_ * NW + lane) : 0u;
                    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
                    if (lane * 8 < n) {
                        const float4* y4 = reinterpret_cast<const float4*>(prm.y + (size_t)frame_ * n) + lane * 2;
                        a = __ldg(y4);
                        b = __ldg(y4 + 1);
                    }
#pragma unroll
                    for (int k = 0; k < NW; k++) c_[k] = __shfl_sync(MPW_FULL, aw, k);
                    // the row's int8 image q_i = ±rint(|y_i| inv_s) and the fp32 canonical ED
                    float syy = 0.f, sxy = 0.f;
                    if (lane * 8 < n) {
                        const float yv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                        const uint32_t cw = select_word<NW>(c_, lane >> 2) >> ((lane & 3) * 8);
                        uint32_t qw[2] = {0u, 0u};
#pragma unroll
                        for (int b_ = 0; b_ < 8; b_++) {
                            const float v = yv[b_];
                            const int q = i8_quant(fabsf(v), inv_);
                            const bool neg = (((cw >> b_) & 1u) != 0u) != (v < 0.0f);
                            qw[b_ >> 2] |= ((uint32_t)(neg ? -q : q) & 0xFFu) << (8 * (b_ & 3));
                            syy = fmaf(v, v, syy);
                            sxy += __uint_as_float(__float_as_uint(v) ^ (((cw >> b_) & 1u) << 31));
                        }
                        *reinterpret_cast<uint2*>(a_rows + (lane >> 4) * A_KBLK_BYTES + sw128_chunk(row, (lane & 15) >> 1) +
                                                  (lane & 1) * 8) = make_uint2(qw[0], qw[1]);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        syy += __shfl_xor_sync(MPW_FULL, syy, o);
                        sxy += __shfl_xor_sync(MPW_FULL, sxy, o);
                    }
                    ed_ = syy + (float)n - 2.0f * sxy;
                    iters_ = 0;
                    flags_ = 0u;
                    recyc_ = false;
                }
            }
            PH(3);
            if (!exhausted_) {
                // window of the next cycle in q units (rounded up; >= 16384 records everything)
                const float wf = (2.0f * err_ + prm.tie_rel * ed_ * 0.25f) * inv_ * 1.00001f + 1.0f;
                wq_ = wf < 16384.f ? __float2int_ru(wf) : 16384;
                // the row's state back to shared memory (whichever worker decides its next cycle)
                {
                    uint32_t ow = select_word<NW>(c_, lane & (NW - 1));
                    if (lane == 8) ow = (uint32_t)tr_;
                    if (lane == 9) ow = (uint32_t)frame_;
                    if (lane == 10) ow = (uint32_t)iters_ | (flags_ << 16) | ((recyc_ ? 1u : 0u) << 24);
                    if (lane == 11) ow = __float_as_uint(ed_);
                    if (lane == 12) ow = __float_as_uint(err_);
                    if (lane == 13) ow = __float_as_uint(inv_);
                    if (lane == 14) ow = __float_as_uint(ay_);
                    if (lane == 15) ow = (uint32_t)wq_;
                    if (lane < RSW) row_state[row * RSW + lane] = ow;
                }
                // the row image is complete and visible to the tensor core's reads of
                // every MMA issued from now on
                if (!(STATS && (prm.experiment & 16))) fence_proxy_async();   // (16: timing probe without the fence)
                __syncwarp();
                if (lane == 0) {
                    row_best[row] = 0x7FFFFFFF;
                    row_done[row] = 0;
                    __threadfence_block();
                    const uint32_t v = ld_shared_volatile_u32(issue_ctr);
                    if (STATS) {
                        const uint32_t prev = ld_shared_volatile_v2(&row_ctl[row]).x;
                        if (prev != 0x80000000u) st_dead += (v + MARGIN) - (prev + (uint32_t)ntiles);
                    }
                    st_shared_volatile_v2(&row_ctl[row],
                                          make_uint2(v + MARGIN, ((uint32_t)wq_ << 16) | (uint32_t)(seed + KEY_BIAS)));
                }
            }
            PH(4);
            PH(5);
            if (STATS) st_busy += clock64() - t_busy0;
        }
#undef PH
        if (STATS && lane == 0) {
            atomicAdd(&prm.stats[ST_ROWCYC], st_rowcyc);
            atomicAdd(&prm.stats[ST_CHUNKS], st_chunks);
            atomicAdd(&prm.stats[ST_F64], st_f64);
            atomicAdd(&prm.stats[ST_OVF], st_ovf);
            atomicAdd(&prm.stats[ST_BUSY], st_busy);
            atomicAdd(&prm.stats[ST_FINISHED], st_fin);
            atomicAdd(&prm.stats[ST_DEAD], st_dead);
            for (int k = 0; k < 6; k++) atomicAdd(&prm.stats[ST_W_LIST + k], (unsigned long long)ph[k]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

}  // namespace ar
