// host_rng.cpp -- CounterRng (rng.hpp:15-64) for synthetic host inputs.
// Input generation only (x[i] = normal_at(i) as in router.hpp:357-360); the
// Box-Muller transform needs libm log/cos, so it stays on the host where it is
// bitwise equal to the reference.  Threads split the index range; every
// element is a pure function of (seed, i), so the split does not matter.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/scmoe.h"

namespace {
uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}
uint64_t hash2(uint64_t seed, uint64_t ctr) {
    return mix64(mix64(seed + 0x9e3779b97f4a7c15ULL) ^ mix64(ctr + 0xbf58476d1ce4e5b9ULL));
}
double uniform01(uint64_t seed, uint64_t ctr) {
    return (static_cast<double>(hash2(seed, ctr) >> 11) + 1.0) * 0x1.0p-53;
}
double normal(uint64_t seed, uint64_t ctr) {
    const double u1 = uniform01(seed, 2 * ctr);
    const double u2 = uniform01(seed, 2 * ctr + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}
}  // namespace

extern "C" {

uint64_t scmoe_rng_stream_seed(uint64_t seed, uint64_t id) {
    return hash2(seed, id ^ 0xa5a5a5a5a5a5a5a5ULL);
}

void scmoe_rng_fill_normal_host(uint64_t seed, uint64_t first, size_t n, float* out, int threads) {
    if (threads < 1) threads = 1;
    if (n < 65536) threads = 1;
    std::vector<std::thread> pool;
    const size_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const size_t a = t * per, b = std::min(n, a + per);
        if (a >= b) break;
        pool.emplace_back([=] {
            for (size_t i = a; i < b; ++i) out[i] = static_cast<float>(normal(seed, first + i));
        });
    }
    for (auto& th : pool) th.join();
}

}  // extern "C"
