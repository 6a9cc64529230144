// Stage 2, tensor-core variant (tcgen05) -- placeholder until the kernel lands.
#pragma once
#include "common.cuh"

struct TcPatterns {
    bool ready = false;
};

inline bool tc_supported(int n, int np) { return false; }
inline int tc_build(TcPatterns& t, const uint32_t* bits, int np, int n, int nw) { t.ready = false; return 0; }
inline int tc_launch(const TcPatterns& t, int n, int nw, int A, int T, const float* y, S2Dev s2, PatDev P,
                     int num_sms, cudaStream_t st) { return -1; }
inline void tc_release(TcPatterns& t) { t.ready = false; }
