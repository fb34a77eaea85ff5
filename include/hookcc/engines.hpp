#pragma once
// CC drivers — header-compatible with the reference engines.hpp
// (/root/reference/proj/include/hookcc/engines.hpp:17-340): the same entry
// points, in-place *_into variants, segment plan helpers and result types.
//
// Each driver uploads the graph (untimed, like the reference's in-memory
// Graph) and runs the whole algorithm on the B200 through hcc_cc: pi init,
// hook/compress phases and the convergence loop execute as one CUDA graph
// with device-side conditional loops.  Timings are device times.
//   baseline_cc     Fig. 1 (atomic-free hook + jump-until-fixpoint)
//   baseline_mj_cc  north-star engine: topology pass + worklist passes
//   single_hook_cc  one CAS-hook segment + Multi-Jump
//   adaptive_cc     s CAS-hook segments, Multi-Jump after each
// DriverOptions::workers caps the device threads (1 = one device thread:
// the reference's deterministic workers=1 schedule; 0 = whole GPU).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hookcc/forest.hpp"
#include "hookcc/graph.hpp"
#include "hookcc/metrics.hpp"
#include "hookcc/parallel.hpp"

namespace hookcc {

struct ComponentLabeling {
  std::vector<Vertex> label;
  bool canonical = false;

  Vertex n() const { return label.size(); }
};

struct SegmentPlan {
  std::uint64_t s = 1;
  bool clamped = false;
  std::vector<std::uint64_t> boundaries;  // s+1 offsets
};

/// Average degree rounded half-up, >= 1, <= m (engines.hpp:35-41).
inline std::uint64_t choose_segment_count(const GraphStats& stats) {
  hcc_graph_stats st{stats.n, stats.m_stored, stats.m_unique, stats.avg_degree,
                     stats.max_degree};
  return hcc_choose_segment_count(&st);
}

/// s contiguous balanced segments; the first m % s get one extra edge
/// (engines.hpp:43-58).
inline SegmentPlan partition_edges(std::uint64_t m, std::uint64_t s) {
  SegmentPlan plan;
  const std::uint64_t want = std::max<std::uint64_t>(s, 1);
  plan.clamped = want > m && m > 0;
  plan.s = std::clamp<std::uint64_t>(want, 1, std::max<std::uint64_t>(m, 1));
  const std::uint64_t q = m / plan.s, r = m % plan.s;
  plan.boundaries.assign(plan.s + 1, 0);
  for (std::uint64_t i = 0; i < plan.s; ++i)
    plan.boundaries[i + 1] = plan.boundaries[i] + q + (i < r ? 1 : 0);
  return plan;
}

inline SegmentPlan partition_edges(const Graph& g, std::uint64_t s) {
  return partition_edges(g.edges.size(), s);
}

/// Converged forest -> labeling; throws std::logic_error unless every tree
/// is a star (engines.hpp:66-75; checked on the device in every build).
inline ComponentLabeling extract_labels(const ParentForest& pi) {
  if (!is_star(pi))
    throw std::logic_error("extract_labels: forest is not star-shaped");
  ComponentLabeling out;
  out.label = pi.snapshot();
  out.canonical = true;
  return out;
}

inline std::uint64_t count_components(const ComponentLabeling& labeling) {
  std::uint64_t roots = 0;
  for (Vertex v = 0; v < labeling.label.size(); ++v) roots += labeling.label[v] == v;
  return roots;
}

enum class Phase { Hook, Compress };

struct DriverOptions {
  unsigned workers = 0;  // device thread cap; 0 = whole GPU
  // Called with the quiesced forest after every phase barrier.  Setting it
  // switches the engine to a host-stepped loop (one sync per phase).
  std::function<void(const ParentForest&, Phase)> phase_observer;
  // B200 options
  std::uint64_t first_pass_segments = 0;  // baseline-mj topology segments (0 = auto)
  std::uint32_t flags = 0;                // HCC_FLAG_*
  // Edge-partitioned multi-GPU run (hcc_create_multi): one shard per entry
  // (partition_edges(m, devices.size()), engines.hpp:43-58), local CC on
  // every device, NVLink P2P merge.  Empty = the calling thread's device.
  std::vector<int> devices;
};

struct DriverResult {
  ComponentLabeling labels;
  RunMetrics metrics;
};

namespace detail {

inline void observer_trampoline(void* user, int phase, hcc_forest* f) {
  const auto& fn =
      *static_cast<const std::function<void(const ParentForest&, Phase)>*>(user);
  ParentForest view = ParentForest::view_with_snapshot(f);
  fn(view, phase == HCC_PHASE_HOOK ? Phase::Hook : Phase::Compress);
}

inline RunMetrics run_device(const Graph& g, int algo, const char* name,
                             std::uint64_t segments, ParentForest& pi,
                             const DriverOptions& opts) {
  if (pi.size() != g.n)
    throw std::invalid_argument("forest size does not match the graph");
  RunMetrics mx;
  mx.algo = name;
  mx.n = g.n;
  mx.m = g.edges.size();
  mx.workers = opts.workers;
  if (g.n == 0) {
    SegmentPlan plan = partition_edges(g.edges.size(), segments ? segments : 1);
    mx.s = algo == HCC_ALGO_ADAPTIVE ? plan.s : 1;
    mx.outer_iterations = algo == HCC_ALGO_ADAPTIVE ? mx.s : 0;
    return mx;
  }
  DeviceGraph dg = opts.devices.empty() ? DeviceGraph(g) : DeviceGraph();
  hcc_opts o{};
  o.algo = algo;
  o.segments = segments;
  o.first_pass_segments = opts.first_pass_segments;
  o.max_threads = opts.workers;
  o.flags = opts.flags;
  if (opts.phase_observer) {
    o.observer = &observer_trampoline;
    o.observer_user = const_cast<void*>(static_cast<const void*>(&opts.phase_observer));
  }
  hcc_metrics hm{};
  if (!opts.devices.empty()) {
    // sharded over opts.devices; the merged labels are copied into pi
    if (opts.phase_observer)
      throw std::invalid_argument("phase_observer needs a single-device run");
    hcc_ctx* mc = multi_ctx(opts.devices);
    hcc_graph* mg = nullptr;
    check(hcc_graph_from_edges_u64(mc, reinterpret_cast<const std::uint64_t*>(g.edges.data()),
                                   g.edges.size(), g.n, &mg));
    std::vector<std::uint64_t> lab(g.n);
    const int st = hcc_cc_u64(mc, mg, &o, nullptr, lab.data(), &hm);
    hcc_graph_free(mg);
    check(st);
    check(hcc_forest_upload_u64(pi.handle(), lab.data()));
    mx.s = hm.s;
    mx.segments_clamped = hm.segments_clamped != 0;
    mx.total_ms = hm.total_ms;
    mx.hook_ms = hm.hook_ms;
    mx.compress_ms = hm.compress_ms;
    mx.outer_iterations = hm.outer_iterations;
    mx.counters = {hm.counters.hook_traversal_steps, hm.counters.cas_failures,
                   hm.counters.jump_steps};
    mx.passes = hm.passes;
    mx.edges_processed = hm.edges_processed;
    mx.device_loop = hm.used_device_loop != 0;
    return mx;
  }
  check(hcc_cc(ctx(), dg.handle(), &o, pi.handle(), nullptr, &hm));
  mx.s = hm.s;
  mx.segments_clamped = hm.segments_clamped != 0;
  mx.total_ms = hm.total_ms;
  mx.hook_ms = hm.hook_ms;
  mx.compress_ms = hm.compress_ms;
  mx.outer_iterations = hm.outer_iterations;
  mx.counters = {hm.counters.hook_traversal_steps, hm.counters.cas_failures,
                 hm.counters.jump_steps};
  mx.passes = hm.passes;
  mx.edges_processed = hm.edges_processed;
  mx.device_loop = hm.used_device_loop != 0;
  std::uint64_t nrec = 0;
  check(hcc_ctx_segments(ctx(), nullptr, 0, &nrec));
  std::vector<hcc_segment_rec> recs(nrec);
  check(hcc_ctx_segments(ctx(), recs.data(), nrec, &nrec));
  for (const hcc_segment_rec& r : recs) {
    mx.segment_ms.push_back({r.hook_ms, r.compress_ms});
    mx.segment_counters.push_back({r.counters.hook_traversal_steps,
                                   r.counters.cas_failures, r.counters.jump_steps});
    mx.worklist_sizes.push_back(r.edges_out);
  }
  return mx;
}

template <typename Driver>
DriverResult run_driver(const Graph& g, Driver&& driver) {
  ParentForest pi(g.n);
  DriverResult result;
  result.metrics = driver(pi);
  result.labels = extract_labels(pi);
  result.metrics.components = count_components(result.labels);
  return result;
}

}  // namespace detail

// ---- in-place drivers (caller owns pi; it is reset inside) ----------------

inline RunMetrics baseline_cc_into(const Graph& g, ParentForest& pi,
                                   const DriverOptions& opts = {}) {
  return detail::run_device(g, HCC_ALGO_BASELINE, "baseline", 0, pi, opts);
}

inline RunMetrics baseline_mj_cc_into(const Graph& g, ParentForest& pi,
                                      const DriverOptions& opts = {}) {
  return detail::run_device(g, HCC_ALGO_BASELINE_MJ, "baseline-mj", 0, pi, opts);
}

/// segments == 0 selects choose_segment_count(compute_stats(g)), computed on
/// the device before the timed region (engines.hpp:245-247).
inline RunMetrics adaptive_cc_into(const Graph& g, std::uint64_t segments,
                                   ParentForest& pi,
                                   const DriverOptions& opts = {}) {
  return detail::run_device(g, HCC_ALGO_ADAPTIVE, "adaptive", segments, pi, opts);
}

inline RunMetrics single_hook_cc_into(const Graph& g, ParentForest& pi,
                                      const DriverOptions& opts = {}) {
  return detail::run_device(g, HCC_ALGO_ATOMIC, "atomic", 1, pi, opts);
}

// ---- entry points (engines.hpp:316-338) -------------------------------------

inline DriverResult baseline_cc(const Graph& g, const DriverOptions& opts = {}) {
  return detail::run_driver(g, [&](ParentForest& pi) { return baseline_cc_into(g, pi, opts); });
}

inline DriverResult baseline_mj_cc(const Graph& g, const DriverOptions& opts = {}) {
  return detail::run_driver(g, [&](ParentForest& pi) { return baseline_mj_cc_into(g, pi, opts); });
}

inline DriverResult single_hook_cc(const Graph& g, const DriverOptions& opts = {}) {
  return detail::run_driver(g, [&](ParentForest& pi) { return single_hook_cc_into(g, pi, opts); });
}

inline DriverResult adaptive_cc(const Graph& g, std::uint64_t segments = 0,
                                const DriverOptions& opts = {}) {
  return detail::run_driver(
      g, [&](ParentForest& pi) { return adaptive_cc_into(g, segments, pi, opts); });
}

}  // namespace hookcc
