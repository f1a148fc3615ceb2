// Synthetic bench inputs, host C++.
//
// Built on the reference's own deterministic RNG -- SplitMix64 streams keyed
// by an FNV-1a hash of a tag (rng.hpp:17-72) -- so the product, the C oracle
// and the reference-side harness generate bit-identical scenes, receivers
// and conditioning states (pinned by tests/test_capi_host.py).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "rxgs_b200.h"

namespace {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

struct Stream {
    uint64_t s;
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
    double normal() {
        double u1 = u01();
        while (u1 <= 0.0) u1 = u01();
        const double u2 = u01();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.28318530717958647692 * u2);
    }
};

uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

Stream stream(uint64_t seed, const std::string& tag, uint64_t counter = 0) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char c : tag) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    h = mix(h ^ mix(seed));
    h = mix(h ^ mix(counter ^ 0xa5a5a5a5a5a5a5a5ull));
    return Stream{h};
}

}  // namespace

namespace rxgs_b200 {
// initial state of derive_stream(seed, tag, counter) (rng.hpp:67-72)
uint64_t derive_stream_state(uint64_t seed, const char* tag, uint64_t counter) {
    return stream(seed, tag, counter).s;
}
}  // namespace rxgs_b200

extern "C" {

int rxgs_synth_scene(int k, int l_max, int channels, uint64_t seed, double* pos, double* ls,
                     double* q, double* tau, double* coeffs) {
    Stream r = stream(seed, "bench.scene");
    const double base = std::log(0.554 * std::cbrt(144.0 / static_cast<double>(k)));
    for (int i = 0; i < k; ++i) {
        pos[3 * i + 0] = r.uniform(-4.0, 4.0);
        pos[3 * i + 1] = r.uniform(-3.0, 3.0);
        pos[3 * i + 2] = r.uniform(-1.5, 1.5);
        for (int a = 0; a < 3; ++a) ls[3 * i + a] = base + r.uniform(-0.3, 0.3);
        double v[4];
        for (double& x : v) x = r.normal();
        const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
        for (int a = 0; a < 4; ++a) q[4 * i + a] = v[a] / n;
        tau[i] = r.uniform(-2.0, 1.0);
    }
    Stream cr = stream(seed, "bench.scene.coeffs");
    const size_t n = static_cast<size_t>(k) * (l_max + 1) * (l_max + 1) * channels * 2;
    for (size_t i = 0; i < n; ++i) coeffs[i] = cr.normal();
    return RXGS_OK;
}

int rxgs_synth_points(int n, uint64_t seed, const char* tag, const double lo[3], const double hi[3],
                      double margin, double* out) {
    Stream r = stream(seed, tag ? tag : "");
    double a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        const double ext = hi[d] - lo[d];
        a[d] = lo[d] + margin * ext;
        b[d] = hi[d] - margin * ext;
    }
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) out[3 * i + d] = r.uniform(a[d], b[d]);
    return RXGS_OK;
}

// init_conditioning (conditioning.cpp:217-253) + the bench overwrite.
int64_t rxgs_synth_cond(const int32_t cfg[9], int l_max, int channels, const double lo[3],
                        const double hi[3], uint64_t seed, int randomize, double* p) {
    const int F = cfg[0], d = cfg[1], dc = cfg[2], C = channels;
    const int L = (l_max + 1) * (l_max + 1);
    const int gin = 6 * F + 2 + dc;
    size_t o = 0;
    const size_t o_freq = o; o += static_cast<size_t>(F) * 3;
    const size_t o_gw1 = o; o += static_cast<size_t>(d) * gin;
    const size_t o_gb1 = o; o += d;
    const size_t o_gw2 = o; o += static_cast<size_t>(d) * d;
    const size_t o_gb2 = o; o += d;
    const size_t o_gw3 = o; o += static_cast<size_t>(4) * C * d;
    const size_t o_gb3 = o; o += 4 * C;
    const size_t o_emb = o; o += static_cast<size_t>(L) * dc;
    const size_t o_lw1 = o; o += static_cast<size_t>(d) * 6;
    const size_t o_lb1 = o; o += d;
    const size_t o_lw2 = o; o += static_cast<size_t>(d) * d;
    const size_t o_lb2 = o; o += d;
    const size_t o_lw3 = o; o += static_cast<size_t>(4) * C * d;
    const size_t o_lb3 = o; o += 4 * C;
    if (!p) return static_cast<int64_t>(o);
    std::memset(p, 0, o * sizeof(double));
    for (int band = 0; band < F; ++band)
        for (int a = 0; a < 3; ++a) {
            const double ext = hi[a] - lo[a];
            p[o_freq + static_cast<size_t>(band) * 3 + a] = std::pow(2.0, band) * kTwoPi / (ext > 0.0 ? ext : 1.0);
        }
    struct Init { const char* tag; size_t off; int in, out; };
    const Init init[4] = {{"cond.global.w1", o_gw1, gin, d}, {"cond.global.w2", o_gw2, d, d},
                          {"cond.local.w1", o_lw1, 6, d}, {"cond.local.w2", o_lw2, d, d}};
    for (const Init& it : init) {
        Stream r = stream(seed, it.tag);
        const double sc = 1.0 / std::sqrt(static_cast<double>(it.in));
        for (int e = 0; e < it.in * it.out; ++e) p[it.off + e] = r.uniform(-sc, sc);
    }
    Stream er = stream(seed, "cond.embed");
    for (int e = 0; e < L * dc; ++e) p[o_emb + e] = 0.1 * er.normal();
    if (randomize) {
        const char* names[2] = {"global", "local"};
        const size_t ow[2][3] = {{o_gw1, o_gw2, o_gw3}, {o_lw1, o_lw2, o_lw3}};
        const size_t ob[2][3] = {{o_gb1, o_gb2, o_gb3}, {o_lb1, o_lb2, o_lb3}};
        const int fin[2][3] = {{gin, d, d}, {6, d, d}};
        const int fout[3] = {d, d, 4 * C};
        for (int m = 0; m < 2; ++m)
            for (int li = 0; li < 3; ++li) {
                const std::string pre = std::string("bench.cond.") + names[m] + ".";
                Stream rw = stream(seed, pre + "w" + std::to_string(li + 1));
                Stream rb = stream(seed, pre + "b" + std::to_string(li + 1));
                const double sc = 1.0 / std::sqrt(static_cast<double>(fin[m][li]));
                for (int e = 0; e < fin[m][li] * fout[li]; ++e) p[ow[m][li] + e] = rw.uniform(-1.0, 1.0) * sc;
                for (int e = 0; e < fout[li]; ++e) p[ob[m][li] + e] = li < 2 ? 0.1 * rb.normal() : 0.0;
            }
    }
    return static_cast<int64_t>(o);
}

}  // extern "C"
