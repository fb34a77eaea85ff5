// B200-specific additions to the header API (not in the reference suite):
// device graphs, device verification, CSR ingestion, counter-based twins.
#include <catch_amalgamated.hpp>

#include "hookcc/engines.hpp"
#include "hookcc/generators.hpp"
#include "hookcc/oracle.hpp"
#include "hookcc/verify.hpp"

using namespace hookcc;

TEST_CASE("rmatx host twin equals the device generator") {
  Graph h = rmatx(12, 8, 0.57, 0.19, 0.19, 0.05, 3);
  DeviceGraph d = DeviceGraph::generate("rmatx:scale=12,ef=8,seed=3");
  CHECK(d.to_host() == h);
  Graph e = erx(5000, 20000, 9);
  CHECK(DeviceGraph::generate("erx:n=5000,m=20000,seed=9").to_host() == e);
}

TEST_CASE("device verification of a finished forest") {
  Graph g = rmat(12, 8, 5);
  DeviceGraph dg(g);
  ParentForest pi(g.n);
  baseline_mj_cc_into(g, pi);
  CHECK(verify_forest(dg, pi).ok());
  pi.store(5, 5);  // break it
  CHECK_FALSE(verify_forest(dg, pi).ok());
}

TEST_CASE("device partitions_equal agrees with the host checker") {
  Graph g = erdos_renyi(3000, 4000, 7);
  ComponentLabeling a = oracle_cc(g), b = bfs_cc(g);
  CHECK(device_partitions_equal(a, b));
  ComponentLabeling c = a;
  for (auto& x : c.label) x = x * 3 + 1;  // renamed
  CHECK(device_partitions_equal(a, c));
  c.label[0] = c.label[1] == c.label[0] ? c.label[0] + 2 : c.label[1];
  CHECK(device_partitions_equal(a, c) == partitions_equal(a, c));
}

TEST_CASE("CSR ingestion matches the edge list") {
  Graph g = grid(7, 9);
  std::vector<std::uint64_t> rp(g.n + 1, 0);
  for (const Edge& e : g.edges) ++rp[e.u + 1];
  for (Vertex v = 0; v < g.n; ++v) rp[v + 1] += rp[v];
  std::vector<std::uint32_t> col(g.edges.size());
  std::vector<std::uint64_t> fill(rp.begin(), rp.end() - 1);
  for (const Edge& e : g.edges) col[fill[e.u]++] = static_cast<std::uint32_t>(e.v);
  DeviceGraph d = DeviceGraph::from_csr(rp, col);
  CHECK(d.m_stored() == g.edges.size());
  Graph back = d.to_host();
  CHECK(oracle_cc(back).label == oracle_cc(g).label);
}

TEST_CASE("edge-partitioned multi-GPU drivers (DriverOptions::devices)") {
  // four shards on device 0 (the builder's single GPU): the same code path
  // as four GPUs, minus the NVLink hop
  Graph g = rmat(13, 8, 11);
  const ComponentLabeling truth = oracle_cc(g);
  DriverOptions opts;
  opts.devices = {0, 0, 0, 0};
  DriverResult a = baseline_mj_cc(g, opts);
  CHECK(a.labels.label == truth.label);
  DriverResult b = adaptive_cc(g, 0, opts);
  CHECK(b.labels.label == truth.label);
  ParentForest pi(g.n);
  baseline_mj_cc_into(g, pi, opts);
  CHECK(pi.snapshot() == truth.label);
}
