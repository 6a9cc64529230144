// Lane-per-path SCL: host side (launch configuration per (N, L)).
#include <algorithm>

#include "scl_lane.cuh"
#include "scl_lane_api.h"

#define CKL(expr)                                   \
    do {                                            \
        const cudaError_t e_ = (expr);              \
        if (e_ != cudaSuccess) return -(int)e_;     \
    } while (0)

template <int N, int L>
static int launch_scl_lane(CodeDev cd, const float* y, const double* llr64, int F, double sigma, int A, int mode,
                           SclOut out, S2Dev s2, int num_sms, cudaStream_t st) {
    using Lay = SclLane<N, L>;
    const size_t per_warp = Lay::TOTAL * Lay::FPW;
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / per_warp));
    const size_t smem = per_warp * wpb;
    if (smem > 227 * 1024) return 1;
    CKL(cudaFuncSetAttribute(scl_lane_kernel<N, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CKL(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scl_lane_kernel<N, L>, 32 * wpb, smem));
    per_sm = std::max(per_sm, 1);
    const long long frames_per_block = (long long)wpb * Lay::FPW;
    const long long need = ((long long)F + frames_per_block - 1) / frames_per_block;
    const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)per_sm * num_sms * 8));
    scl_lane_kernel<N, L><<<grid, 32 * wpb, smem, st>>>(cd, y, llr64, F, sigma, A, mode, out, s2);
    CKL(cudaGetLastError());
    return 0;
}

template <int N>
static int dispatch_l(int L, CodeDev cd, const float* y, const double* llr64, int F, double sigma, int A, int mode,
                      SclOut out, S2Dev s2, int num_sms, cudaStream_t st) {
    switch (L) {
        case 4: return launch_scl_lane<N, 4>(cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        case 8: return launch_scl_lane<N, 8>(cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        case 16: return launch_scl_lane<N, 16>(cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        case 32: return launch_scl_lane<N, 32>(cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        default: return 1;
    }
}

int scl_lane_launch(int n, int L, CodeDev cd, const float* y, const double* llr64, int F, double sigma, int A,
                    int mode, SclOut out, S2Dev s2, int num_sms, cudaStream_t st) {
    switch (n) {
        case 64: return dispatch_l<64>(L, cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        case 128: return dispatch_l<128>(L, cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        case 256: return dispatch_l<256>(L, cd, y, llr64, F, sigma, A, mode, out, s2, num_sms, st);
        default: return 1;
    }
}
