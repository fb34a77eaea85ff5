#pragma once
// Device-side verification: O(n) / O(m) checks that avoid
// the std::map partitions_equal of the reference (oracle.hpp:112-126,
// bench.hpp:351-372) at 2^24-2^28 vertices.

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "hookcc/detail.hpp"
#include "hookcc/engines.hpp"
#include "hookcc/forest.hpp"
#include "hookcc/graph.hpp"

namespace hookcc {

struct ForestCheck {
  std::uint64_t split_edges = 0;     // edges (u, v) with pi(u) != pi(v)
  std::uint64_t noncanonical = 0;    // v with pi(v) > v or pi(pi(v)) != pi(v)
  bool ok() const { return split_edges == 0 && noncanonical == 0; }
};

/// Size-independent correctness properties of a finished forest.
inline ForestCheck verify_forest(const DeviceGraph& g, ParentForest& pi) {
  ForestCheck r;
  detail::check(hcc_forest_verify(detail::ctx(), g.handle(), pi.handle(), &r.split_edges,
                                  &r.noncanonical));
  return r;
}

/// partitions_equal computed on the device (labels must be < 2^32).
inline bool device_partitions_equal(const ComponentLabeling& a, const ComponentLabeling& b) {
  if (a.label.size() != b.label.size())
    throw std::invalid_argument("partitions_equal: length mismatch");
  std::vector<std::uint32_t> x(a.label.size()), y(b.label.size());
  for (std::size_t i = 0; i < x.size(); ++i) {
    if (a.label[i] > 0xffffffffull || b.label[i] > 0xffffffffull)
      throw std::invalid_argument("device_partitions_equal: label >= 2^32");
    x[i] = static_cast<std::uint32_t>(a.label[i]);
    y[i] = static_cast<std::uint32_t>(b.label[i]);
  }
  int pe = 0, ex = 0;
  detail::check(hcc_labels_compare(detail::ctx(), x.data(), y.data(), x.size(), &pe, &ex));
  return pe != 0;
}

}  // namespace hookcc
