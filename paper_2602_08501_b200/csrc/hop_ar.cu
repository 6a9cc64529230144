// Asynchronous-row int8 tensor hop: host side (launch, statistics).
#include <cstdio>
#include <cstring>
#include <mutex>

#include "hop_ar.cuh"
#include "hop_tc_api.h"

static float ar_cert_gamma(int wmax, bool y64) {
    // any summation order of at most wmax terms: |fl(S) - S| <= gamma_{wmax-1} sum|t_i|;
    // with float64 inputs the fp32 rounding of y adds u sum|y|
    const double u = 5.9604644775390625e-8;
    const double k = wmax > 1 ? wmax - 1 : 0;
    double g = k * u / (1.0 - k * u);
    if (y64) g += u;
    return (float)(g * 1.002);
}

bool ar_supported(const TcPatterns& t, int n) {
    // u8 images present (|P| <= 2^17, 127 wmax < 8192), 32-pattern group ids fit 16 bits
    return t.ready8 && (n == 128 || n == 256) && t.np <= (1 << 17);
}

template <int KB, int NW, bool STATS>
static int ar_launch_t(const TcPatterns& t, int n, int A, int T, const float* y, const double* y64, S2Dev s2, PatDev P, int num_sms,
                       int experiment, int hit_cap, cudaStream_t st) {
    ar::Params prm;
    prm.n = n; prm.nw = NW; prm.A = A; prm.T = T; prm.np = t.np; prm.ntiles = t.ntiles8;
    prm.y = y; prm.y64 = y64; prm.s2 = s2; prm.pbits = P.bits; prm.btiles = t.tiles8;
    prm.tie_rel = 1e-5f;
    prm.cap = hit_cap > 0 && hit_cap < ar::CAP ? hit_cap : ar::CAP;
    prm.cert_g = ar_cert_gamma(s2.wmax, y64 != nullptr);
    prm.stats = nullptr;
    prm.experiment = 0;
    prm.tilestat = t.ar_stat;   // accumulated over launches (mpw_hop_tile_stats)
    // statistics buffers (instrumented / hop_experiment = 32 launches only) are shared by all
    // handles of the process: such launches are serialised
    static std::mutex stat_mutex;
    std::unique_lock<std::mutex> stat_lock(stat_mutex, std::defer_lock);
    if (STATS || experiment == 32) stat_lock.lock();
    static unsigned long long* tilestat = nullptr;
    if (experiment == 32) {   // light statistic of the production kernel: cycles per tile
        if (!tilestat && cudaMallocManaged(&tilestat, 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
        tilestat[0] = tilestat[1] = 0;
        prm.tilestat = tilestat;
    }
    static unsigned long long* stats = nullptr;
    if (STATS) {
        if (!stats && cudaMallocManaged(&stats, sizeof(unsigned long long) * ar::ST_N) != cudaSuccess) return -1;
        memset(stats, 0, sizeof(unsigned long long) * ar::ST_N);
        prm.stats = stats;
        prm.experiment = experiment;
    }
    const size_t smem = ar::smem_bytes(KB);
    auto kern = ar::hop_ar_kernel<KB, NW, STATS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -(int)e;
    kern<<<num_sms, ar::THREADS, smem, st>>>(prm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return -(int)e;
    if (experiment == 32 && prm.tilestat == tilestat) {
        cudaStreamSynchronize(st);
        fprintf(stderr, "[hop_ar] production kernel: %.0f tiles per CTA, %.1f cycles per tile\n", (double)tilestat[0] / num_sms,
                tilestat[0] ? (double)tilestat[1] / (double)tilestat[0] : 0.0);
    }
    if (STATS) {
        cudaStreamSynchronize(st);
        const unsigned long long* s = stats;
        const double tiles = (double)s[ar::ST_TILES] / 32.0 / (ar::SCAN_T / 32);   // per-lane counts of the scan warps
        fprintf(stderr,
                "[hop_ar] CTA-tiles %.0f, live row-halves %.4f, row cycles %llu (finished %llu), hit chunks/cycle %.3f, "
                "entries/thread-cycle %.2f, f64 decisions %llu, overflow re-scans %llu, worker busy cycles/row-cycle %.0f\n",
                tiles, s[ar::ST_TILES] ? (double)s[ar::ST_LIVE] / (double)s[ar::ST_TILES] : 0.0, s[ar::ST_ROWCYC],
                s[ar::ST_FINISHED], s[ar::ST_ROWCYC] ? (double)s[ar::ST_CHUNKS] / (double)s[ar::ST_ROWCYC] : 0.0,
                s[ar::ST_ROWCYC] ? (double)s[ar::ST_ENTRIES] / ((double)ar::NCOL * (double)s[ar::ST_ROWCYC]) : 0.0, s[ar::ST_F64],
                s[ar::ST_OVF], s[ar::ST_ROWCYC] ? (double)s[ar::ST_BUSY] / (double)s[ar::ST_ROWCYC] : 0.0);
        fprintf(stderr,
                "[hop_ar] cycles per tile %.0f; issuer: B stage wait %.3f, accumulator wait %.3f, MMA issue + commit %.3f of its time; scan warps wait "
                "for the accumulator %.3f of their time\n",
                tiles > 0 ? (double)s[ar::ST_ISS_TOT] / tiles : 0.0,   // issuer 0's clock over all tiles
                s[ar::ST_ISS_TOT] ? (double)s[ar::ST_ISS_FULL] / (double)s[ar::ST_ISS_TOT] : 0.0,
                s[ar::ST_ISS_TOT] ? (double)s[ar::ST_ISS_TEMPTY] / (double)s[ar::ST_ISS_TOT] : 0.0,
                s[ar::ST_ISS_TOT] ? (double)s[ar::ST_ISS_MMA] / (double)s[ar::ST_ISS_TOT] : 0.0,
                s[ar::ST_SCAN_TOT] ? (double)s[ar::ST_SCAN_WAIT] / (double)s[ar::ST_SCAN_TOT] : 0.0);
        const double rc = s[ar::ST_ROWCYC] ? (double)s[ar::ST_ROWCYC] : 1.0;
        fprintf(stderr,
                "[hop_ar] worker cycles per row cycle: lists+t %.0f, chunk scores %.0f, decision+move %.0f, claim+build %.0f, "
                "publish %.0f, pocket refill %.0f; tiles per row cycle "
                "between cycle end and next start %.2f\n",
                s[ar::ST_W_LIST] / rc, s[ar::ST_W_CHUNK] / rc, s[ar::ST_W_DECIDE] / rc, s[ar::ST_W_CLAIM] / rc,
                s[ar::ST_W_PUBLISH] / rc, s[ar::ST_W_POCKET] / rc, s[ar::ST_DEAD] / rc);
    }
    return 0;
}

int ar_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, const double* y64, S2Dev s2, PatDev P,
              int num_sms, const TcOpts& o, cudaStream_t st) {
    if (!ar_supported(t, n) || nw != n / 32) return 1;
    const bool stats = o.experiment != 0 && o.experiment != 32;
    if (n == 256)
        return stats ? ar_launch_t<2, 8, true>(t, n, A, T, y, y64, s2, P, num_sms, o.experiment, o.ar_hit_cap, st)
                     : ar_launch_t<2, 8, false>(t, n, A, T, y, y64, s2, P, num_sms, o.experiment, o.ar_hit_cap, st);
    return stats ? ar_launch_t<1, 4, true>(t, n, A, T, y, y64, s2, P, num_sms, o.experiment, o.ar_hit_cap, st)
                 : ar_launch_t<1, 4, false>(t, n, A, T, y, y64, s2, P, num_sms, o.experiment, o.ar_hit_cap, st);
}
