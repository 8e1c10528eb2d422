// fuzzyclust/graph.hpp -- drop-in for graph.hpp (graph.hpp:18-224).  Graph and
// normalize_edges are the reference's value types; parse_edge_list, the largest
// connected component and the 2-core run on the device (libfuzzyclust_cuda.so,
// fc_ingest.cu) with the reference's semantics: ids compacted
// by first appearance, LCC ties to the component with the smallest id, the same
// IoError messages and line numbers.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <istream>
#include <iterator>
#include <ostream>
#include <string>
#include <utility>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/device.hpp"

namespace fuzzyclust {

struct Graph {
    std::size_t num_nodes = 0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;   ///< u < v, sorted, unique

    std::vector<std::size_t> degrees() const {
        std::vector<std::size_t> deg(num_nodes, 0);
        for (const auto& [u, v] : edges) {
            ++deg[u];
            ++deg[v];
        }
        return deg;
    }
    std::vector<std::vector<std::uint32_t>> adjacency() const {
        std::vector<std::vector<std::uint32_t>> adj(num_nodes);
        for (const auto& [u, v] : edges) {
            adj[u].push_back(v);
            adj[v].push_back(u);
        }
        return adj;
    }
};

inline void normalize_edges(std::vector<std::pair<std::uint32_t, std::uint32_t>>& edges) {
    for (auto& e : edges)
        if (e.first > e.second) std::swap(e.first, e.second);
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
}

struct ParsedGraph {
    Graph graph;
    std::vector<std::int64_t> original_ids;   ///< input id of compacted node k (first appearance)
};

namespace detail {
inline std::vector<std::uint32_t> flat_edges(const Graph& g) {
    std::vector<std::uint32_t> e(2 * g.edges.size());
    for (std::size_t k = 0; k < g.edges.size(); ++k) {
        e[2 * k] = g.edges[k].first;
        e[2 * k + 1] = g.edges[k].second;
    }
    return e;
}
inline std::vector<std::uint32_t> take_nodes(uint32_t* p, uint64_t count) {
    std::vector<std::uint32_t> v(p, p + count);
    fc_free(p);
    return v;
}
}  // namespace detail

/// graph.hpp:63-103 -- "u v" lines, '#' comments; text read whole, parsed by all
/// host cores, compacted / deduplicated on the device.
inline ParsedGraph parse_edge_list(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    auto& d = device::context();
    fc_ingest_result r{};
    device::check(fc_ingest_edge_list(d.ctx, text.data(), text.size(), 0, &r), d.ctx);
    ParsedGraph out;
    out.graph.num_nodes = r.num_nodes;
    out.graph.edges.resize(r.num_edges);
    for (std::size_t k = 0; k < r.num_edges; ++k) out.graph.edges[k] = {r.edges[2 * k], r.edges[2 * k + 1]};
    out.original_ids.assign(r.original_ids, r.original_ids + r.num_nodes);
    fc_free(r.edges);
    fc_free(r.original_ids);
    return out;
}

/// graph.hpp:107-120 (host: order-preserving recompaction keeps the list sorted).
inline Graph induced_subgraph(const Graph& g, const std::vector<std::uint32_t>& nodes) {
    std::vector<std::uint32_t> new_id(g.num_nodes, UINT32_MAX);
    for (std::size_t k = 0; k < nodes.size(); ++k) new_id[nodes[k]] = static_cast<std::uint32_t>(k);
    Graph out;
    out.num_nodes = nodes.size();
    for (const auto& [u, v] : g.edges)
        if (new_id[u] != UINT32_MAX && new_id[v] != UINT32_MAX) out.edges.emplace_back(new_id[u], new_id[v]);
    normalize_edges(out.edges);
    return out;
}

/// graph.hpp:146-169 on the device (union-find, min-id roots).
inline std::vector<std::uint32_t> largest_connected_component_nodes(const Graph& g) {
    if (g.num_nodes == 0) throw InvalidInput("largest_connected_component: empty graph");
    auto& d = device::context();
    const auto e = detail::flat_edges(g);
    uint32_t* nodes = nullptr;
    uint64_t count = 0;
    device::check(fc_graph_lcc_nodes(d.ctx, g.num_nodes, g.edges.size(), e.data(), &nodes, &count), d.ctx);
    return detail::take_nodes(nodes, count);
}

inline Graph largest_connected_component(const Graph& g) {
    return induced_subgraph(g, largest_connected_component_nodes(g));
}

inline bool is_connected(const Graph& g) {
    if (g.num_nodes == 0) return false;
    return largest_connected_component_nodes(g).size() == g.num_nodes;
}

/// graph.hpp:206-213 on the device (frontier peeling of degree <= 1 nodes).
inline std::vector<std::uint32_t> two_core_nodes(const Graph& g) {
    auto& d = device::context();
    const auto e = detail::flat_edges(g);
    uint32_t* nodes = nullptr;
    uint64_t count = 0;
    device::check(fc_graph_two_core_nodes(d.ctx, g.num_nodes, g.edges.size(), e.data(), &nodes, &count), d.ctx);
    return detail::take_nodes(nodes, count);
}

/// graph.hpp:185-204: true for every node peeled away.
inline std::vector<bool> degree_one_peel_mask(const Graph& g) {
    std::vector<bool> removed(g.num_nodes, true);
    for (std::uint32_t v : two_core_nodes(g)) removed[v] = false;
    return removed;
}

inline Graph prune_degree_one(const Graph& g) { return induced_subgraph(g, two_core_nodes(g)); }

/// graph.hpp:222-224
inline void write_edge_list(const Graph& g, std::ostream& out) {
    for (const auto& [u, v] : g.edges) out << u << ' ' << v << '\n';
}

}  // namespace fuzzyclust
