// Host-side pattern-set generation (off the timed path).
//
//  * mpw_enumerate_lowweight: exhaustive walk of all 2^K codewords (K <= 40)
//    in Gray-code order over the high message bits with a doubling table for
//    the low bits -- the same enumeration the reference's
//    `enumerate_spectrum`/`build_sphere` performs (wsphere.py:115-208), split
//    across threads by high-bit ranges.  Collects every nonzero codeword of
//    weight <= cap and tallies the full weight spectrum.
//  * mpw_collect_lowweight: seeded information-set search (Lee-Brickell,
//    p <= 2) for codes whose 2^K walk is out of reach (BASELINE config 4,
//    K = 53).  The result is the union over a fixed, seeded iteration set, so
//    it is deterministic for any thread count; completeness is not proven.
//
// Both write unsorted words; the Python side sorts into CWS1 member order.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

constexpr int kMaxW = 16;  // up to 1024 bits

struct Word {
    uint64_t w[kMaxW];
    int nw;
    bool operator==(const Word& o) const { return std::memcmp(w, o.w, sizeof(uint64_t) * nw) == 0; }
};
struct WordHash {
    size_t operator()(const Word& x) const {
        uint64_t h = 0x9e3779b97f4a7c15ull;
        for (int i = 0; i < x.nw; i++) { h ^= x.w[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); }
        return (size_t)h;
    }
};

inline int popc_row(const uint64_t* w, int nw) {
    int s = 0;
    for (int i = 0; i < nw; i++) s += __builtin_popcountll(w[i]);
    return s;
}

uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

}  // namespace

extern "C" {

// Returns the number of collected words (all of them are written if
// out_cap >= return value), or -1 on bad arguments.  spectrum: n+1 counts.
int64_t mpw_enumerate_lowweight(const uint64_t* gen, int k, int n, int cap, int64_t* spectrum,
                                uint64_t* out, int64_t out_cap, int nthreads) {
    const int nw = (n + 63) / 64;
    if (k < 1 || k > 40 || nw > kMaxW || n < 1) return -1;
    if (nthreads < 1) nthreads = 1;
    const int low = std::min(k, 16);
    const int high = k - low;
    const size_t tsize = (size_t)1 << low;
    std::vector<uint64_t> table(tsize * nw, 0);
    for (int i = 0; i < low; i++) {  // doubling table: entry e = XOR of rows in bits of e
        size_t half = (size_t)1 << i;
        for (size_t e = 0; e < half; e++)
            for (int w = 0; w < nw; w++) table[(half + e) * nw + w] = table[e * nw + w] ^ gen[(size_t)i * nw + w];
    }
    const uint64_t nhigh = (uint64_t)1 << high;
    int T = (int)std::min<uint64_t>((uint64_t)nthreads, nhigh);
    std::vector<std::vector<int64_t>> tallies(T, std::vector<int64_t>(n + 1, 0));
    std::vector<std::vector<uint64_t>> found(T);
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++) {
        th.emplace_back([&, t]() {
            uint64_t h0 = nhigh * (uint64_t)t / T, h1 = nhigh * (uint64_t)(t + 1) / T;
            uint64_t center[kMaxW] = {0};
            // center = XOR of high rows selected by gray(h0)
            uint64_t g0 = h0 ^ (h0 >> 1);
            for (int b = 0; b < high; b++)
                if ((g0 >> b) & 1)
                    for (int w = 0; w < nw; w++) center[w] ^= gen[(size_t)(low + b) * nw + w];
            auto& tally = tallies[t];
            auto& fw = found[t];
            uint64_t tmp[kMaxW];
            for (uint64_t h = h0; h < h1; h++) {
                if (h != h0) {
                    int flip = __builtin_ctzll(h);  // Gray step h-1 -> h flips bit ctz(h)
                    for (int w = 0; w < nw; w++) center[w] ^= gen[(size_t)(low + flip) * nw + w];
                }
                for (size_t e = 0; e < tsize; e++) {
                    const uint64_t* te = &table[e * nw];
                    int wt = 0;
                    for (int w = 0; w < nw; w++) { tmp[w] = te[w] ^ center[w]; wt += __builtin_popcountll(tmp[w]); }
                    tally[wt]++;
                    if (wt > 0 && wt <= cap) fw.insert(fw.end(), tmp, tmp + nw);
                }
            }
        });
    }
    for (auto& x : th) x.join();
    int64_t total = 0;
    if (spectrum) std::memset(spectrum, 0, sizeof(int64_t) * (n + 1));
    for (int t = 0; t < T; t++) {
        if (spectrum) for (int i = 0; i <= n; i++) spectrum[i] += tallies[t][i];
        total += (int64_t)(found[t].size() / nw);
    }
    if (out && out_cap >= total) {
        int64_t pos = 0;
        for (int t = 0; t < T; t++) {
            std::memcpy(out + pos * nw, found[t].data(), found[t].size() * sizeof(uint64_t));
            pos += (int64_t)(found[t].size() / nw);
        }
    }
    return total;
}

// Seeded Lee-Brickell search over `iterations` random information sets.
// Writes up to out_cap words; returns the number of distinct words found.
int64_t mpw_collect_lowweight(const uint64_t* gen, int k, int n, int cap, int64_t iterations,
                              uint64_t seed, int p_max, uint64_t* out, int64_t out_cap,
                              int nthreads) {
    const int nw = (n + 63) / 64;
    if (k < 1 || k > 256 || nw > kMaxW || p_max < 1 || p_max > 3) return -1;
    if (nthreads < 1) nthreads = 1;
    std::unordered_set<Word, WordHash> global;
    std::mutex mu;
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; t++) {
        th.emplace_back([&, t]() {
            std::unordered_set<Word, WordHash> local;
            std::vector<uint64_t> g((size_t)k * nw);
            std::vector<int> perm(n);
            Word cand; cand.nw = nw;
            auto consider = [&](const uint64_t* w) {
                int wt = popc_row(w, nw);
                if (wt > 0 && wt <= cap) {
                    std::memcpy(cand.w, w, sizeof(uint64_t) * nw);
                    for (int i = nw; i < kMaxW; i++) cand.w[i] = 0;
                    local.insert(cand);
                }
            };
            for (int64_t it = t; it < iterations; it += nthreads) {
                uint64_t s = seed ^ (0xd1b54a32d192ed03ull * (uint64_t)(it + 1));
                for (int i = 0; i < n; i++) perm[i] = i;
                for (int i = n - 1; i > 0; i--) {
                    int j = (int)(splitmix64(s) % (uint64_t)(i + 1));
                    std::swap(perm[i], perm[j]);
                }
                std::memcpy(g.data(), gen, sizeof(uint64_t) * g.size());
                int rank = 0;
                for (int ci = 0; ci < n && rank < k; ci++) {
                    int col = perm[ci], cw = col >> 6; uint64_t bit = 1ull << (col & 63);
                    int piv = -1;
                    for (int r = rank; r < k; r++) if (g[(size_t)r * nw + cw] & bit) { piv = r; break; }
                    if (piv < 0) continue;
                    if (piv != rank)
                        for (int w = 0; w < nw; w++) std::swap(g[(size_t)piv * nw + w], g[(size_t)rank * nw + w]);
                    for (int r = 0; r < k; r++)
                        if (r != rank && (g[(size_t)r * nw + cw] & bit))
                            for (int w = 0; w < nw; w++) g[(size_t)r * nw + w] ^= g[(size_t)rank * nw + w];
                    rank++;
                }
                uint64_t a[kMaxW], b[kMaxW];
                for (int i = 0; i < rank; i++) {
                    const uint64_t* ri = &g[(size_t)i * nw];
                    consider(ri);
                    if (p_max < 2) continue;
                    for (int j = i + 1; j < rank; j++) {
                        const uint64_t* rj = &g[(size_t)j * nw];
                        for (int w = 0; w < nw; w++) a[w] = ri[w] ^ rj[w];
                        consider(a);
                        if (p_max < 3) continue;
                        for (int l = j + 1; l < rank; l++) {
                            const uint64_t* rl = &g[(size_t)l * nw];
                            for (int w = 0; w < nw; w++) b[w] = a[w] ^ rl[w];
                            consider(b);
                        }
                    }
                }
            }
            std::lock_guard<std::mutex> lk(mu);
            global.insert(local.begin(), local.end());
        });
    }
    for (auto& x : th) x.join();
    int64_t total = (int64_t)global.size();
    if (out) {
        int64_t pos = 0;
        for (const auto& x : global) {
            if (pos >= out_cap) break;
            std::memcpy(out + pos * nw, x.w, sizeof(uint64_t) * nw);
            pos++;
        }
    }
    return total;
}

}  // extern "C"
