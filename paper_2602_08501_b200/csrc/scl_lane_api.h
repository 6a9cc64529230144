// Host API of the lane-per-path SCL kernel (definitions in scl_lane.cu, a
// separate translation unit so its (N, L) instantiations compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "scl.cuh"

// Returns 0 on launch, 1 if (n, L) has no lane-kernel instantiation (the
// caller falls back to the warp-per-frame kernel), -cudaError on failure.
int scl_lane_launch(int n, int L, CodeDev cd, const float* y, const double* llr64, int F, double sigma, int A,
                    int mode, SclOut out, S2Dev s2, int num_sms, cudaStream_t st);
