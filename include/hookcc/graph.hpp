#pragma once
// Input data model — header-compatible with the reference graph.hpp
// (/root/reference/proj/include/hookcc/graph.hpp:9-96).
//
// Graph keeps the reference's host AoS layout (16 B/edge, stored order,
// duplicates and self-loops kept).  The device layout is packed u32 pairs
// (8 B/edge), produced by DeviceGraph at upload time (hcc_graph_from_*).
// compute_stats runs on the GPU (radix sort + unique, hcc_graph_compute_stats)
// instead of the reference's O(m log m) host sort.

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "hookcc/detail.hpp"

namespace hookcc {

using Vertex = std::uint64_t;

struct Edge {
  Vertex u;
  Vertex v;

  friend bool operator==(const Edge&, const Edge&) = default;
};

/// Undirected graph: vertex count plus ordered edge records (graph.hpp:20-31).
struct Graph {
  Vertex n = 0;
  std::vector<Edge> edges;

  std::uint64_t m_stored() const { return edges.size(); }

  friend bool operator==(const Graph&, const Graph&) = default;
};

struct GraphStats {
  Vertex n = 0;
  std::uint64_t m_stored = 0;
  std::uint64_t m_unique = 0;   // unique undirected adjacencies, no loops
  double avg_degree = 0.0;      // 2 * m_unique / n
  std::uint64_t max_degree = 0;
};

/// Device-resident copy of a Graph (packed u32 pairs in HBM).  Upload
/// validates endpoints (check_endpoints semantics, graph.hpp:89-94).
class DeviceGraph {
 public:
  DeviceGraph() = default;
  explicit DeviceGraph(const Graph& g) {
    static_assert(sizeof(Edge) == 2 * sizeof(std::uint64_t));
    detail::check(hcc_graph_from_edges_u64(
        detail::ctx(), reinterpret_cast<const std::uint64_t*>(g.edges.data()),
        g.edges.size(), g.n, &h_));
  }
  /// Adopt a handle produced by the C-ABI (generators, CSR ingestion).
  explicit DeviceGraph(hcc_graph* h) : h_(h) {}
  /// Device generator spec: "rmatx:...", "erx:...", "grid:RxC".
  static DeviceGraph generate(const std::string& spec,
                              std::uint64_t default_seed = 1) {
    hcc_graph* h = nullptr;
    detail::check(
        hcc_graph_generate(detail::ctx(), spec.c_str(), default_seed, &h));
    return DeviceGraph(h);
  }
  /// CSR: entry j of row u is edge (u, col[j]) (north-star CSR loading).
  static DeviceGraph from_csr(const std::vector<std::uint64_t>& row_ptr,
                              const std::vector<std::uint32_t>& col) {
    if (row_ptr.empty()) throw std::invalid_argument("empty row_ptr");
    hcc_graph* h = nullptr;
    detail::check(hcc_graph_from_csr(detail::ctx(), row_ptr.data(),
                                     col.data(), row_ptr.size() - 1, &h));
    return DeviceGraph(h);
  }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
  DeviceGraph(DeviceGraph&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceGraph& operator=(DeviceGraph&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  ~DeviceGraph() {
    if (h_) hcc_graph_free(h_);
  }

  hcc_graph* handle() const { return h_; }
  Vertex n() const {
    std::uint64_t n = 0, m = 0;
    hcc_graph_info(h_, &n, &m);
    return n;
  }
  std::uint64_t m_stored() const {
    std::uint64_t n = 0, m = 0;
    hcc_graph_info(h_, &n, &m);
    return m;
  }
  /// Download as a host Graph (u32 ids widened to u64).
  Graph to_host() const {
    Graph g;
    g.n = n();
    std::uint64_t m = m_stored();
    std::vector<std::uint32_t> uv(2 * m);
    detail::check(hcc_graph_download_u32(detail::ctx(), h_, uv.data(), 0, m));
    g.edges.resize(m);
    for (std::uint64_t i = 0; i < m; ++i) g.edges[i] = {uv[2 * i], uv[2 * i + 1]};
    return g;
  }

 private:
  hcc_graph* h_ = nullptr;
};

inline GraphStats stats_of(const DeviceGraph& dg) {
  hcc_graph_stats st{};
  detail::check(hcc_graph_compute_stats(detail::ctx(), dg.handle(), &st));
  GraphStats out;
  out.n = st.n;
  out.m_stored = st.m_stored;
  out.m_unique = st.m_unique;
  out.avg_degree = st.avg_degree;
  out.max_degree = st.max_degree;
  return out;
}

/// Degree statistics over the deduplicated adjacency (graph.hpp:43-68),
/// computed on the device.
inline GraphStats compute_stats(const Graph& g) {
  if (g.n == 0) {
    GraphStats st;
    st.m_stored = g.edges.size();
    return st;
  }
  return stats_of(DeviceGraph(g));
}

/// Deduplicated, loop-free, canonical (u < v), sorted copy (graph.hpp:72-87).
/// A host utility for cross-checks; no engine calls it.
inline Graph normalize(const Graph& g) {
  Graph out;
  out.n = g.n;
  out.edges.reserve(g.edges.size());
  for (const Edge& e : g.edges)
    if (e.u != e.v) out.edges.push_back({std::min(e.u, e.v), std::max(e.u, e.v)});
  std::sort(out.edges.begin(), out.edges.end(), [](const Edge& a, const Edge& b) {
    return a.u != b.u ? a.u < b.u : a.v < b.v;
  });
  out.edges.erase(std::unique(out.edges.begin(), out.edges.end()), out.edges.end());
  return out;
}

/// Endpoint validation (graph.hpp:89-94).
inline void check_endpoints(const Graph& g) {
  for (const Edge& e : g.edges)
    if (e.u >= g.n || e.v >= g.n)
      throw std::invalid_argument("edge endpoint out of range");
}

}  // namespace hookcc
