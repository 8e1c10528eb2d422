// generator.cpp -- synthetic similarity graphs for the benchmark configurations
// (SURVEY.md section 8(d)).  New code: the reference's only generator is the
// paper's two-cluster Erdos-Renyi model, O(n^2) Bernoulli draws
// (generator.hpp:46-97), which cannot produce the BASELINE shapes.
//
// Every random decision is a pure function of (seed, counter) through the
// reference's splitmix64 mix (rng.hpp:21-26), so the output is identical for
// any thread count.  The result is build_similarity's A + I pattern
// (sparse.hpp:66-75): symmetric, diagonal present, duplicates merged, rows
// sorted ascending, all values 1.0.
//
// kind 0 -- stochastic block model: `blocks` equal blocks; each of m edge draws
//   picks u uniformly, then v inside u's block with probability p_in, else
//   uniformly over all nodes (v != u).
// kind 1 -- power-law citation-like: node u (time order) cites d_u older nodes,
//   d_u ~ Pareto(alpha) (stochastically rounded, capped at 4096, mean m/n); each
//   cited node is floor(u * r^gamma), r ~ U[0,1): gamma > 1 biases citations to
//   old nodes and yields a power-law in-degree (gamma = 2: tail exponent ~3,
//   max in-degree ~ 2 (m/n) sqrt(n)).
// locality 0 relabels nodes by a keyed Feistel permutation (random ids);
// locality 1 keeps block / time order (neighbours close in id space).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fuzzyclust_cuda.h"

namespace {

inline uint64_t mix64(uint64_t z) {   // splitmix64 finaliser, rng.hpp:23-25
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// draw #k of stream `stream` under `seed` (counter-based)
inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t k) {
    return mix64(seed + 0x9E3779B97F4A7C15ULL * (mix64(stream * 0xD1B54A32D192ED03ULL + 1) + k + 1));
}
inline double unit(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53; }
inline uint64_t below(uint64_t r, uint64_t bound) {   // multiply-high, unbiased enough
    return static_cast<uint64_t>((static_cast<unsigned __int128>(r) * bound) >> 64);
}

struct Feistel {   // bijection of [0, n) by cycle-walking a balanced Feistel network
    uint64_t n, key;
    unsigned half;
    uint64_t mask;
    Feistel(uint64_t n_, uint64_t key_) : n(n_), key(key_) {
        unsigned bits = 1;
        while ((1ULL << bits) < n) ++bits;
        half = (bits + 1) / 2;
        mask = (1ULL << half) - 1;
    }
    uint64_t once(uint64_t x) const {
        uint64_t l = x >> half, r = x & mask;
        for (int round = 0; round < 4; ++round) {
            const uint64_t f = mix64(key + 0x9E3779B97F4A7C15ULL * (r + 1 + (uint64_t)round * (mask + 1))) & mask;
            const uint64_t nl = r;
            r = l ^ f;
            l = nl;
        }
        return (l << half) | r;
    }
    uint64_t operator()(uint64_t x) const {
        do { x = once(x); } while (x >= n);
        return x;
    }
};

void parallel_for(uint64_t n, int threads, const std::function<void(uint64_t, uint64_t)>& fn) {
    if (n == 0) return;
    const uint64_t t = std::max<uint64_t>(1, std::min<uint64_t>(threads, n));
    std::vector<std::thread> pool;
    for (uint64_t k = 0; k < t; ++k) {
        const uint64_t a = n * k / t, b = n * (k + 1) / t;
        pool.emplace_back([&fn, a, b] { fn(a, b); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int fc_generate_graph_impl(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out,
                                      uint32_t** col_idx_out, std::string* err) {
    const uint64_t n = spec->n;
    if (n == 0 || n > 0xFFFFFFFFULL) { *err = "generator: n must be in [1, 2^32)"; return FC_INVALID; }
    int threads = spec->threads > 0 ? spec->threads : (int)std::thread::hardware_concurrency();
    if (threads <= 0) threads = 1;
    const uint64_t seed = spec->seed;

    // ---- 1. edge endpoints, in a fixed order -------------------------------
    std::vector<uint32_t> src, dst;
    if (spec->kind == 0) {
        if (spec->blocks == 0 || spec->blocks > n) { *err = "generator: bad block count"; return FC_INVALID; }
        if (n < 2) { *err = "generator: SBM needs n >= 2"; return FC_INVALID; }
        const uint64_t m = spec->m;
        src.resize(m);
        dst.resize(m);
        const uint64_t nb = spec->blocks;
        parallel_for(m, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t e = a; e < b; ++e) {
                const uint64_t u = below(draw(seed, 1, e), n);
                const uint64_t blk = u * nb / n;
                const uint64_t lo = (blk * n + nb - 1) / nb, hi = ((blk + 1) * n + nb - 1) / nb;  // [lo, hi)
                uint64_t v;
                const bool inside = unit(draw(seed, 2, e)) < spec->p_in && hi - lo >= 2;
                for (uint64_t k = 0;; ++k) {
                    const uint64_t r = draw(seed, 3, e * 64 + k);
                    v = inside ? lo + below(r, hi - lo) : below(r, n);
                    if (v != u) break;
                }
                src[e] = (uint32_t)u;
                dst[e] = (uint32_t)v;
            }
        });
    } else if (spec->kind == 1) {
        const double alpha = spec->alpha > 2.0 ? spec->alpha : 2.5;
        const double gamma = spec->gamma >= 1.0 ? spec->gamma : 2.0;
        const double mean = (double)spec->m / (double)n;
        const double dmin = mean * (alpha - 2.0) / (alpha - 1.0);
        const double cap = 4096.0;
        std::vector<uint64_t> off(n + 1, 0);
        parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t u = a; u < b; ++u) {
                if (u == 0) { off[1] = 0; continue; }
                const double x = dmin * std::pow(1.0 - unit(draw(seed, 4, u)), -1.0 / (alpha - 1.0));
                double d = std::floor(std::min(x, cap) + unit(draw(seed, 5, u)));
                off[u + 1] = (uint64_t)std::min<double>(d, (double)u);
            }
        });
        for (uint64_t u = 0; u < n; ++u) off[u + 1] += off[u];
        const uint64_t m = off[n];
        src.resize(m);
        dst.resize(m);
        parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t u = a; u < b; ++u) {
                for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
                    const double r = unit(draw(seed, 6, k));
                    uint64_t v = (uint64_t)std::floor((double)u * std::pow(r, gamma));
                    if (v >= u) v = u - 1;
                    src[k] = (uint32_t)u;
                    dst[k] = (uint32_t)v;
                }
            }
        });
    } else {
        *err = "generator: unknown kind";
        return FC_INVALID;
    }
    const uint64_t m = src.size();

    // ---- 2. optional random relabel ----------------------------------------
    if (!spec->locality) {
        const Feistel perm(n, mix64(seed ^ 0x5EED5EED5EEDULL));
        parallel_for(m, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t e = a; e < b; ++e) {
                src[e] = (uint32_t)perm(src[e]);
                dst[e] = (uint32_t)perm(dst[e]);
            }
        });
    }

    // ---- 3. symmetric A + I: count, scatter, sort + unique per row ------------
    std::vector<uint64_t> deg(n, 1);   // diagonal
    {
        auto* d = deg.data();
        parallel_for(m, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t e = a; e < b; ++e) {
                __atomic_fetch_add(d + src[e], 1, __ATOMIC_RELAXED);
                __atomic_fetch_add(d + dst[e], 1, __ATOMIC_RELAXED);
            }
        });
    }
    std::vector<uint64_t> start(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) start[i + 1] = start[i] + deg[i];
    std::vector<uint32_t> col(start[n]);
    std::vector<uint64_t> cur(n);
    parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            col[start[i]] = (uint32_t)i;
            cur[i] = start[i] + 1;
        }
    });
    {
        auto* c = cur.data();
        parallel_for(m, threads, [&](uint64_t a, uint64_t b) {
            for (uint64_t e = a; e < b; ++e) {
                col[__atomic_fetch_add(c + src[e], 1, __ATOMIC_RELAXED)] = dst[e];
                col[__atomic_fetch_add(c + dst[e], 1, __ATOMIC_RELAXED)] = src[e];
            }
        });
    }
    src.clear(); src.shrink_to_fit();
    dst.clear(); dst.shrink_to_fit();
    std::vector<uint64_t> len(n);
    parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            uint32_t* p = col.data() + start[i];
            uint32_t* q = col.data() + start[i + 1];
            std::sort(p, q);
            len[i] = (uint64_t)(std::unique(p, q) - p);
        }
    });
    int64_t* rp = static_cast<int64_t*>(std::malloc((n + 1) * sizeof(int64_t)));
    if (!rp) { *err = "generator: out of host memory"; return FC_DEVICE; }
    rp[0] = 0;
    for (uint64_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + (int64_t)len[i];
    const uint64_t nnz = (uint64_t)rp[n];
    uint32_t* ci = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(nnz, 1) * sizeof(uint32_t)));
    if (!ci) { std::free(rp); *err = "generator: out of host memory"; return FC_DEVICE; }
    parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i)
            std::memcpy(ci + rp[i], col.data() + start[i], len[i] * sizeof(uint32_t));
    });
    *nnz_out = nnz;
    *row_ptr_out = rp;
    *col_idx_out = ci;
    return FC_OK;
}

// dense.hpp:40-46 frob_inner: one sequential sum over the storage order (host; the
// order is the contract, so it is not parallelised).  Compiled without FMA contraction.
extern "C" double fc_frob_inner(const double* a, const double* b, uint64_t count) {
    double acc = 0.0;
    for (uint64_t k = 0; k < count; ++k) acc += a[k] * b[k];
    return acc;
}
