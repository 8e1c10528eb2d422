// fuzzyclust/graph.hpp -- the Graph value type build_similarity consumes
// (graph.hpp:18-52).  Edge-list ingestion, LCC and 2-core pruning are outside
// the hot path and are not part of this build.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace fuzzyclust {

struct Graph {
    std::size_t num_nodes = 0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;   ///< u < v, sorted, unique
};

inline void normalize_edges(std::vector<std::pair<std::uint32_t, std::uint32_t>>& edges) {
    for (auto& e : edges)
        if (e.first > e.second) std::swap(e.first, e.second);
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
}

}  // namespace fuzzyclust
