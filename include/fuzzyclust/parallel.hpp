// fuzzyclust/parallel.hpp -- the reduction-block partition of parallel.hpp:15-68.
// On the solver path the reference's std::thread pool is replaced by the GPU grid;
// its fixed 1024-column block order is kept by every device reduction, which is why
// results are bitwise identical to the reference for any worker or GPU count.
// parallel_for_blocks itself is kept for host callers (the reference's suites and any
// host-side per-block loop): same partition and callback contract, a static cyclic
// block-to-thread assignment.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

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

/// fn(block, begin, end) for every kReductionBlock-sized block of [0, n).  The partition
/// is fixed, so per-block outputs do not depend on `workers` (<= 1: the calling thread
/// alone).  Worker t takes blocks t, t + w, t + 2w, ...; the first exception is rethrown.
template <class Fn>
void parallel_for_blocks(std::size_t n, unsigned workers, Fn&& fn) {
    const std::size_t nb = block_count(n);
    if (nb == 0) return;
    const std::size_t w = std::min<std::size_t>(workers > 1 ? workers : 1, nb);
    auto lane = [&](std::size_t t) {
        for (std::size_t b = t; b < nb; b += w) fn(b, b * kReductionBlock, std::min(n, (b + 1) * kReductionBlock));
    };
    if (w == 1) {
        lane(0);
        return;
    }
    std::exception_ptr first;
    std::mutex mu;
    std::vector<std::thread> pool;
    pool.reserve(w - 1);
    for (std::size_t t = 1; t < w; ++t)
        pool.emplace_back([&, t] {
            try {
                lane(t);
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                if (!first) first = std::current_exception();
            }
        });
    try {
        lane(0);
    } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
    }
    for (auto& th : pool) th.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace fuzzyclust
