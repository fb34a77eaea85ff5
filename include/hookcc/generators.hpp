#pragma once
// Synthetic inputs — API-compatible with the reference generators.hpp
// (/root/reference/proj/include/hookcc/generators.hpp:10-89).
//
// erdos_renyi / rmat / grid reproduce the reference graphs bit-for-bit on
// the host (same std::mt19937_64 stream and libstdc++ uniform_real mapping;
// the ids are unpermuted; duplicates and self-loops are kept).  They are
// sequential by construction.  rmatx / erx are the counter-based twins
// (include/hookcc_gen.h) that the device generates in parallel
// (DeviceGraph::generate); the host versions here exist for parity checks
// and for host-side consumers.

#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>

#include "hookcc/graph.hpp"
#include "hookcc_gen.h"

namespace hookcc {

/// G(n, m): both endpoints uniform with replacement (generators.hpp:14-26).
inline Graph erdos_renyi(Vertex n, std::uint64_t m, std::uint64_t seed) {
  if (n == 0) throw std::invalid_argument("erdos_renyi: zero vertices");
  Graph g;
  g.n = n;
  g.edges.resize(m);
  std::mt19937_64 draw(seed);
  for (Edge& e : g.edges) {
    e.u = draw() % n;
    e.v = draw() % n;
  }
  return g;
}

/// Recursive-quadrant generator, probabilities applied un-perturbed at
/// every level, MSB first (generators.hpp:31-62).
inline Graph rmat(unsigned scale, std::uint64_t edge_factor, double a, double b,
                  double c, double d, std::uint64_t seed) {
  if (std::fabs(a + b + c + d - 1.0) > 1e-9)
    throw std::invalid_argument("rmat: quadrant probabilities must sum to 1");
  Graph g;
  g.n = Vertex{1} << scale;
  g.edges.resize(edge_factor * g.n);
  std::mt19937_64 draw(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  const double ab = a + b, abc = a + b + c;
  for (Edge& e : g.edges) {
    Vertex u = 0, v = 0;
    for (unsigned level = 0; level < scale; ++level) {
      const double p = unit(draw);
      const bool row = p >= ab;                   // quadrants (1,0), (1,1)
      const bool col = (p >= a && p < ab) || p >= abc;  // (0,1), (1,1)
      u = (u << 1) | row;
      v = (v << 1) | col;
    }
    e = {u, v};
  }
  return g;
}

inline Graph rmat(unsigned scale, std::uint64_t edge_factor, std::uint64_t seed) {
  return rmat(scale, edge_factor, 0.57, 0.19, 0.19, 0.05, seed);
}

/// 4-neighbour lattice, row-major ids; row edges first, then column edges
/// (generators.hpp:71-87).
inline Graph grid(Vertex rows, Vertex cols) {
  if (rows == 0 || cols == 0) throw std::invalid_argument("grid: zero vertices");
  Graph g;
  g.n = rows * cols;
  g.edges.resize(rows * (cols - 1) + (rows - 1) * cols);
  for (std::uint64_t i = 0; i < g.edges.size(); ++i) {
    std::uint32_t u = 0, v = 0;
    hcc::grid_edge(rows, cols, i, &u, &v);
    g.edges[i] = {u, v};
  }
  return g;
}

/// Counter-based RMAT twin (host side of DeviceGraph::generate("rmatx:...")).
inline Graph rmatx(unsigned scale, std::uint64_t edge_factor, double a, double b,
                   double c, double d, std::uint64_t seed) {
  if (std::fabs(a + b + c + d - 1.0) > 1e-9)
    throw std::invalid_argument("rmat: quadrant probabilities must sum to 1");
  if (scale > 31) throw std::invalid_argument("rmatx: scale > 31");
  Graph g;
  g.n = Vertex{1} << scale;
  g.edges.resize(edge_factor * g.n);
  const std::uint64_t key = hcc::gen_key(seed);
  const std::uint32_t ta = hcc::prob_threshold(a), tab = hcc::prob_threshold(a + b),
                      tabc = hcc::prob_threshold(a + b + c);
  for (std::uint64_t i = 0; i < g.edges.size(); ++i) {
    std::uint32_t u = 0, v = 0;
    hcc::rmatx_edge(key, i, scale, ta, tab, tabc, &u, &v);
    g.edges[i] = {u, v};
  }
  return g;
}

/// Counter-based Erdos-Renyi twin ("erx:...").
inline Graph erx(Vertex n, std::uint64_t m, std::uint64_t seed) {
  if (n == 0) throw std::invalid_argument("erdos_renyi: zero vertices");
  if (n > 0xffffffffull) throw std::invalid_argument("erx: n >= 2^32");
  Graph g;
  g.n = n;
  g.edges.resize(m);
  const std::uint64_t key = hcc::gen_key(seed);
  for (std::uint64_t i = 0; i < m; ++i) {
    std::uint32_t u = 0, v = 0;
    hcc::erx_edge(key, i, n, &u, &v);
    g.edges[i] = {u, v};
  }
  return g;
}

}  // namespace hookcc
