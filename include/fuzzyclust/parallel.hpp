// fuzzyclust/parallel.hpp -- the reduction-block constant of parallel.hpp:15-31.
// The reference's std::thread pool (parallel_for_blocks) is replaced by the GPU
// grid; its fixed 1024-column block order is kept by every device reduction,
// which is why results are bitwise identical to the reference for any worker
// or GPU count.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <thread>

namespace fuzzyclust {

inline constexpr std::size_t kReductionBlock = 1024;

inline std::size_t block_count(std::size_t n) { return (n + kReductionBlock - 1) / kReductionBlock; }

/// Kept for signature parity (SolverConfig::workers); the device ignores it.
inline unsigned resolve_workers(unsigned requested = 0) {
    if (requested > 0) return requested;
    if (const char* env = std::getenv("FUZZYCLUST_THREADS")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v > 0) return static_cast<unsigned>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? hw : 1;
}

}  // namespace fuzzyclust
