// synth.cpp — deterministic synthetic SIFT-like datasets (libchsynth.so, host only).
//
// Recipe of SURVEY.md §8(d), modelled on the reference's fixtures
// (proj/tests/support/synthetic.hpp:48-61 uniform_descriptor / noisy_copy, :75-94 make_noisy_pair):
//   pool[p], p < ceil(rho*N): i.i.d. uniform u8[128] from mt19937_64(stream_seed(seed, 0xba5e, 0))
//   image i, generator mt19937_64(stream_seed(seed, 0x1396, i)):
//     slots s < ceil(rho*N): clamp(pool[s] + sigma*N(0,1), 0, 255) truncated to u8  (a twin of the
//                            same pool entry in every image => about rho*N true matches per pair)
//     remaining slots      : i.i.d. uniform u8
//   "sift" shape: |N(0,1)| components, L2-normalised to 512, clipped to 255 (bucket-skew stress).
// Used by tests and bench.py to make inputs; it is not part of the matching path.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace {

inline uint64_t fin(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline uint64_t stream_seed(uint64_t seed, uint64_t a, uint64_t b) {
    return fin(fin(seed ^ fin(a)) ^ fin(b ^ 0xd6e8feb86659fd93ULL));
}
inline double unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
inline double normal(std::mt19937_64& g) {
    const double u1 = 1.0 - unit(g), u2 = unit(g);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

void fill_uniform(std::mt19937_64& g, uint8_t* d) {
    for (int c = 0; c < 128; c += 8) {  // 8 bytes per generator word; any fixed rule is fine for a fixture
        uint64_t w = g();
        for (int k = 0; k < 8; ++k) d[c + k] = static_cast<uint8_t>(w >> (8 * k));
    }
}

void fill_sift_like(std::mt19937_64& g, uint8_t* d) {
    double v[128], norm = 0;
    for (int c = 0; c < 128; ++c) {
        v[c] = std::fabs(normal(g));
        norm += v[c] * v[c];
    }
    const double s = 512.0 / std::sqrt(norm);
    for (int c = 0; c < 128; ++c) d[c] = static_cast<uint8_t>(std::min(255.0, v[c] * s));
}

}  // namespace

extern "C" {

// shape: 0 = uniform, 1 = sift-like.  pool must hold ceil(rho*n)*128 bytes.
int chsynth_pool(uint64_t seed, uint32_t n, double rho, int shape, uint8_t* pool) {
    const uint32_t twins = static_cast<uint32_t>(std::ceil(rho * n));
    std::mt19937_64 g(stream_seed(seed, 0xba5e, 0));
    for (uint32_t p = 0; p < twins; ++p) {
        if (shape == 1) fill_sift_like(g, pool + size_t(p) * 128);
        else fill_uniform(g, pool + size_t(p) * 128);
    }
    return 0;
}

int chsynth_image(uint64_t seed, uint32_t image_index, uint32_t n, double rho, double sigma, int shape,
                  const uint8_t* pool, uint8_t* desc) {
    const uint32_t twins = static_cast<uint32_t>(std::ceil(rho * n));
    std::mt19937_64 g(stream_seed(seed, 0x1396, image_index));
    for (uint32_t s = 0; s < n; ++s) {
        uint8_t* d = desc + size_t(s) * 128;
        if (s < twins) {
            const uint8_t* base = pool + size_t(s) * 128;
            for (int c = 0; c < 128; ++c) {
                const double v = static_cast<double>(base[c]) + sigma * normal(g);
                d[c] = static_cast<uint8_t>(std::clamp(v, 0.0, 255.0));
            }
        } else if (shape == 1) {
            fill_sift_like(g, d);
        } else {
            fill_uniform(g, d);
        }
    }
    return 0;
}

// Whole dataset, images [first, first+count) into desc (count*n*128 bytes), on `threads` threads.
int chsynth_dataset(uint64_t seed, uint32_t first, uint32_t count, uint32_t n, double rho, double sigma,
                    int shape, uint32_t threads, uint8_t* desc) {
    const uint32_t twins = static_cast<uint32_t>(std::ceil(rho * n));
    std::vector<uint8_t> pool(size_t(std::max(twins, 1u)) * 128);
    chsynth_pool(seed, n, rho, shape, pool.data());
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    threads = std::min(threads, std::max(count, 1u));
    std::vector<std::thread> pool_threads;
    for (uint32_t w = 0; w < threads; ++w)
        pool_threads.emplace_back([&, w] {
            for (uint32_t i = w; i < count; i += threads)
                chsynth_image(seed, first + i, n, rho, sigma, shape, pool.data(), desc + size_t(i) * n * 128);
        });
    for (auto& t : pool_threads) t.join();
    return 0;
}

}  // extern "C"
