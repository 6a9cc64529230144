// Device-side channel generator: seeded, counter-based
// inputs for 10^6-10^7-frame sweeps without host traffic.
//
// Frame g of stream (seed, snr_idx) draws from Philox4x32-10 with
//   key     = (seed_lo, seed_hi ^ (snr_idx * 0x9E3779B9))
//   counter = (g_lo, g_hi, word, 0x4D505753)
// word 0 -> message bits (4 x 32 random bits, bit j of the message = bit j of
// the 128-bit block), word 1 + c -> symbols 4c..4c+3 by Box-Muller on
// u = (x + 0.5) 2^-32 in float64.  Codeword = XOR of generator rows selected
// by the message (codebook.py:282-284), x = 1 - 2c (channel.py:44-50),
// y = float32(x + sigma z).  channel.py's `keyed_inputs_host` is the numpy
// mirror of the same recipe.  This keying is our own (the reference keys one
// numpy Philox stream per trial, simharness.py:220-222); it is used for bulk
// runs and documented as such.
#pragma once
#include "common.cuh"

struct Philox4 {
    uint32_t v[4];
};

__host__ __device__ inline Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.v[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.v[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        Philox4 n;
        n.v[0] = hi1 ^ c.v[1] ^ k0;
        n.v[1] = lo1;
        n.v[2] = hi0 ^ c.v[3] ^ k1;
        n.v[3] = lo0;
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

struct ChannelArgs {
    CodeDev code;
    uint64_t seed;
    uint32_t snr_idx;
    long long first_frame;
    int F;
    double sigma;
    float* y;          // F x n
    uint32_t* tx;      // F x nw (may be null)
    uint64_t* msg;     // F (k <= 64, may be null)
};

// one warp per frame: lane j handles symbols j, j+32, ...
__global__ void channel_kernel(ChannelArgs a) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int n = a.code.n, nw = a.code.nw, k = a.code.k;
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32) ^ (a.snr_idx * 0x9E3779B9u);
    for (int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); f < a.F; f += warps) {
        const unsigned long long g = (unsigned long long)(a.first_frame + f);
        Philox4 c0 = {{(uint32_t)g, (uint32_t)(g >> 32), 0u, 0x4D505753u}};
        const Philox4 mb = philox4x32_10(c0, k0, k1);
        // codeword: lane w < nw accumulates word w over the message's generator rows
        uint32_t cwl = 0;
        for (int i = 0; i < k; i++) {
            const uint32_t bit = (mb.v[i >> 5] >> (i & 31)) & 1u;
            if (bit && lane < nw) cwl ^= a.code.gen[(size_t)i * nw + lane];
        }
        if (a.tx && lane < nw) a.tx[(size_t)f * nw + lane] = cwl;
        if (a.msg && lane == 0) {
            uint64_t m = ((uint64_t)mb.v[1] << 32) | mb.v[0];
            if (k < 64) m &= (1ull << k) - 1ull;
            a.msg[f] = m;
        }
        for (int base = 0; base < n; base += 128) {
            // lane handles symbols base + 4*lane .. +3 (one Philox call); the
            // codeword word is shuffled from its owner before any divergence
            const int s0 = base + 4 * lane;
            const int wsrc = min(s0 >> 5, nw - 1);
            const uint32_t word = __shfl_sync(MPW_FULL, cwl, wsrc);
            if (s0 >= n) continue;
            Philox4 cc = {{(uint32_t)g, (uint32_t)(g >> 32), 1u + (uint32_t)(s0 >> 2), 0x4D505753u}};
            const Philox4 r = philox4x32_10(cc, k0, k1);
            double z[4];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const double u1 = ((double)r.v[2 * h] + 0.5) * 2.3283064365386963e-10;
                const double u2 = ((double)r.v[2 * h + 1] + 0.5) * 2.3283064365386963e-10;
                const double rad = sqrt(-2.0 * log(u1));
                double sv, cv;
                sincospi(2.0 * u2, &sv, &cv);
                z[2 * h] = rad * cv;
                z[2 * h + 1] = rad * sv;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int s = s0 + q;
                if (s < n) {
                    const double x = ((word >> (s & 31)) & 1u) ? -1.0 : 1.0;
                    a.y[(size_t)f * n + s] = (float)(x + a.sigma * z[q]);
                }
            }
        }
    }
}
