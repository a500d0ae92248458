// Seeded inputs with the reference's generator, quasar::Rng
// (/root/reference/proj/include/quasar/rng.hpp:29-103): splitmix64 over a
// keyed counter, fnv1a stream labels, Box-Muller normals with a cached spare.
//
// The generator is counter-based (draw c = mix(key + phi * c)), so a stream of
// `count` draws splits across host threads and still reproduces the
// sequential stream bit for bit. Normal draws come in (cos, sin) pairs from
// counters (2j+1, 2j+2); the reference's u1 == 0 rejection (rng.hpp:59, p =
// 2^-53 per pair) would shift every later counter, so if any chunk meets it
// the whole fill is redone sequentially.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>
#include <vector>

#include "qsv_internal.hpp"

namespace qsv {

namespace {
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;

inline uint64_t mix(uint64_t z) {
    z += kPhi;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
inline uint64_t fnv1a(const char *s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ull;
    }
    return h;
}
inline double to_unit(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

struct Seq { // sequential reference semantics (used on the rejection path)
    uint64_t key, counter = 0;
    double spare = 0;
    bool have = false;
    double uniform() { return to_unit(mix(key + kPhi * ++counter)); }
    double normal() {
        if (have) {
            have = false;
            return spare;
        }
        double u1 = 0.0;
        while (u1 == 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare = r * std::sin(2.0 * 3.141592653589793 * u2);
        have = true;
        return r * std::cos(2.0 * 3.141592653589793 * u2);
    }
};
} // namespace

int rng_fill(uint64_t seed, const char *label, int kind, uint64_t count, void *out, int nthreads,
             uint64_t offset) {
    require(kind >= 0 && kind <= 2, "rng_fill: kind must be 0 (u64), 1 (uniform) or 2 (normal)");
    require(kind != 2 || offset % 2 == 0, "rng_fill: normal draws start at an even offset (Box-Muller pairs)");
    if (label) seed ^= fnv1a(label);
    const uint64_t key = mix(seed ^ kPhi); // Rng(uint64_t) constructor
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned T = nthreads > 0 ? static_cast<unsigned>(nthreads) : hw;
    T = std::max(1u, std::min<unsigned>(T, static_cast<unsigned>(std::max<uint64_t>(1, count >> 16))));
    std::atomic<bool> rejected{false};
    // work unit: one draw (kinds 0/1) or one normal pair (kind 2); the
    // stream starts `offset` draws in (counter-based: no sequential skip)
    const uint64_t units = kind == 2 ? (count + 1) / 2 : count;
    const uint64_t c0 = offset;
    auto work = [&](uint64_t b, uint64_t e) {
        for (uint64_t j = b; j < e; ++j) {
            if (kind == 0) static_cast<uint64_t *>(out)[j] = mix(key + kPhi * (c0 + j + 1));
            else if (kind == 1) static_cast<double *>(out)[j] = to_unit(mix(key + kPhi * (c0 + j + 1)));
            else {
                const double u1 = to_unit(mix(key + kPhi * (c0 + 2 * j + 1)));
                const double u2 = to_unit(mix(key + kPhi * (c0 + 2 * j + 2)));
                if (u1 == 0.0) {
                    rejected = true;
                    return;
                }
                const double r = std::sqrt(-2.0 * std::log(u1));
                double *o = static_cast<double *>(out);
                o[2 * j] = r * std::cos(2.0 * 3.141592653589793 * u2);
                if (2 * j + 1 < count) o[2 * j + 1] = r * std::sin(2.0 * 3.141592653589793 * u2);
            }
        }
    };
    if (T == 1) work(0, units);
    else {
        std::vector<std::thread> pool;
        const uint64_t per = (units + T - 1) / T;
        for (unsigned t = 0; t < T; ++t) {
            const uint64_t b = std::min<uint64_t>(units, t * per), e = std::min<uint64_t>(units, b + per);
            pool.emplace_back(work, b, e);
        }
        for (auto &th : pool) th.join();
    }
    if (rejected) { // p ~ 2^-53 per pair: replay the sequential stream exactly
        Seq s{key};
        double *o = static_cast<double *>(out);
        for (uint64_t i = 0; i < offset; ++i) s.normal();
        for (uint64_t i = 0; i < count; ++i) o[i] = s.normal();
    }
    return 0;
}

// measure()'s sampling (circuit.hpp:217-236) over given marginals: shots
// draws of Rng(seed, label).uniform() * total starting after *counter draws,
// lower_bound over the running sums; counts per outcome index.
void sample_counts(const double *probs, int k, int shots, uint64_t seed, const char *label, uint64_t *counter,
                   uint64_t *counts) {
    if (label) seed ^= fnv1a(label);
    const uint64_t key = mix(seed ^ kPhi);
    const size_t np = size_t(1) << k;
    std::vector<double> cdf(np);
    double acc = 0.0;
    for (size_t i = 0; i < np; ++i) {
        acc += probs[i];
        cdf[i] = acc;
    }
    std::fill(counts, counts + np, 0ull);
    const uint64_t c0 = counter ? *counter : 0;
    // shot s draws the stream's (c0 + s + 1)-th value (counter-based), so
    // shot ranges are independent: large batches fan out over host threads
    // and the histogram is the same as the sequential loop's
    auto run = [&](int s0, int s1, bool atomic) {
        for (int s = s0; s < s1; ++s) {
            const double u = to_unit(mix(key + kPhi * (c0 + static_cast<uint64_t>(s) + 1))) * acc;
            const size_t idx = std::min<size_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin(), np - 1);
            if (atomic) __atomic_fetch_add(&counts[idx], 1ull, __ATOMIC_RELAXED);
            else counts[idx] += 1;
        }
    };
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int nt = shots >= (1 << 16) ? std::min(hw, 16) : 1;
    if (nt == 1) run(0, shots, false);
    else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                run(static_cast<int>(static_cast<int64_t>(shots) * t / nt),
                    static_cast<int>(static_cast<int64_t>(shots) * (t + 1) / nt), true);
            });
        for (auto &x : th) x.join();
    }
    if (counter) *counter = c0 + static_cast<uint64_t>(shots);
}

} // namespace qsv
