// fg_internal.hpp — shared host-side plumbing of libfgb200: error state,
// checked CUDA calls, small helpers.  Not part of the ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fg_b200.h"

namespace fgb {

// Error carrying the reference's machine code (error.hpp:11-20): what() is
// "<code>: <message>", exactly like fusegraph::Error.
class Error : public std::runtime_error {
public:
    Error(std::string code, const std::string& message)
        : std::runtime_error(code + ": " + message), code_(std::move(code)) {}
    const std::string& code() const noexcept { return code_; }

private:
    std::string code_;
};

void set_last_error(const std::string& code, const std::string& what);
void clear_last_error();

// Runs fn, mapping exceptions to FG_ERR + thread-local last error.
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        clear_last_error();
        return FG_OK;
    } catch (const Error& e) {
        set_last_error(e.code(), e.what());
    } catch (const std::bad_alloc&) {
        set_last_error("out-of-memory", "out-of-memory: host allocation failed");
    } catch (const std::exception& e) {
        set_last_error("internal", std::string("internal: ") + e.what());
    }
    return FG_ERR;
}

// SplitMix64 exactly as rng.hpp:17-41 (same constants, same order), plus
// random access: draw j of a stream seeded with s is mix(s + (j+1)*gamma).
struct SplitMix64 {
    static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
    uint64_t state = 0;
    explicit SplitMix64(uint64_t seed = 0) : state(seed) {}
    static inline uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    inline uint64_t next() { return mix(state += kGamma); }
};

inline uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    SplitMix64 m(seed ^ (0xA0761D6478BD642FULL * (stream + 1)));
    return m.next();
}
inline uint64_t bounded(SplitMix64& rng, uint64_t bound) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(rng.next()) * bound) >> 64);
}
inline double uniform01_bits(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }
inline double uniform01(SplitMix64& rng) { return uniform01_bits(rng.next()); }

}  // namespace fgb

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace fgb {
// Dev tool: FGB_HOST_TIMING=1 prints per-phase wall times of host entry
// points (each mark synchronises the device first, so phases include their
// GPU work); =2 prints the same marks without synchronising.  Off by
// default: no syncs, no output.
struct HostTimer {
    const char* scope;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit HostTimer(const char* s) : scope(s), on(enabled()), t(std::chrono::steady_clock::now()) {}
    static int mode() {
        static const int e = [] {
            const char* v = std::getenv("FGB_HOST_TIMING");
            return v ? std::atoi(v) : 0;
        }();
        return e;
    }
    static bool enabled() { return mode() != 0; }
    void mark(const char* what);
};
}  // namespace fgb
