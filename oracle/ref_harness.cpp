// ref_harness.cpp — C wrapper around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY.  oracle/Makefile compiles this
// file against the read-only reference headers in
// /root/reference/proj/include (header-only C++20; nothing is copied) into
// oracle/_ref/libhookcc_ref.so.  tests/ use it to pin the C restatement and
// the CUDA path; bench.py's `--impl reference` arm and `cpu_baseline` time
// the reference's own engines through it, on the host cores.
//
// Every entry point is a thin call into the reference's public API:
//   generators.hpp (erdos_renyi, rmat, grid), oracle.hpp (oracle_cc,
//   bfs_cc), engines.hpp (baseline_cc, baseline_mj_cc, single_hook_cc,
//   adaptive_cc), graph.hpp (compute_stats), forest.hpp (element kernels).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "hookcc/engines.hpp"
#include "hookcc/forest.hpp"
#include "hookcc/generators.hpp"
#include "hookcc/graph.hpp"
#include "hookcc/oracle.hpp"

using namespace hookcc;

namespace {

Graph make_graph(uint64_t n, const uint64_t* uv, uint64_t m) {
  Graph g;
  g.n = n;
  g.edges.resize(m);
  if (m) std::memcpy(g.edges.data(), uv, m * sizeof(Edge));
  return g;
}

Graph make_graph32(uint64_t n, const uint32_t* uv, uint64_t m) {
  Graph g;
  g.n = n;
  g.edges.resize(m);
  for (uint64_t i = 0; i < m; ++i) g.edges[i] = {uv[2 * i], uv[2 * i + 1]};
  return g;
}

ParentForest make_forest(const uint64_t* pi, uint64_t n) {
  ParentForest f(n);
  for (uint64_t v = 0; v < n; ++v) f.store(v, pi[v]);
  return f;
}

void read_forest(const ParentForest& f, uint64_t* pi) {
  for (uint64_t v = 0; v < f.size(); ++v) pi[v] = f.load(v);
}

}  // namespace

extern "C" {

struct ref_metrics {
  double total_ms, hook_ms, compress_ms;
  uint64_t s, outer_iterations, hook_traversal_steps, cas_failures,
      jump_steps, components;
  int segments_clamped;
  unsigned workers;
};

unsigned ref_hardware_workers() { return hardware_workers(); }

// ---- generators ---------------------------------------------------------
int ref_gen_er(uint64_t n, uint64_t m, uint64_t seed, uint64_t* uv) {
  try {
    Graph g = erdos_renyi(n, m, seed);
    std::memcpy(uv, g.edges.data(), m * sizeof(Edge));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_gen_rmat(unsigned scale, uint64_t ef, double a, double b, double c,
                 double d, uint64_t seed, uint64_t* uv) {
  try {
    Graph g = rmat(scale, ef, a, b, c, d, seed);
    std::memcpy(uv, g.edges.data(), g.edges.size() * sizeof(Edge));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_gen_grid(uint64_t rows, uint64_t cols, uint64_t* uv) {
  try {
    Graph g = grid(rows, cols);
    std::memcpy(uv, g.edges.data(), g.edges.size() * sizeof(Edge));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// ---- oracles --------------------------------------------------------------
int ref_oracle_cc(uint64_t n, const uint64_t* uv, uint64_t m, uint64_t* labels) {
  Graph g = make_graph(n, uv, m);
  ComponentLabeling l = oracle_cc(g);
  std::memcpy(labels, l.label.data(), n * sizeof(uint64_t));
  return 0;
}

int ref_bfs_cc(uint64_t n, const uint64_t* uv, uint64_t m, uint64_t* labels) {
  Graph g = make_graph(n, uv, m);
  ComponentLabeling l = bfs_cc(g);
  std::memcpy(labels, l.label.data(), n * sizeof(uint64_t));
  return 0;
}

int ref_stats(uint64_t n, const uint64_t* uv, uint64_t m, uint64_t* m_unique,
              double* avg_degree, uint64_t* max_degree) {
  Graph g = make_graph(n, uv, m);
  GraphStats st = compute_stats(g);
  *m_unique = st.m_unique;
  *avg_degree = st.avg_degree;
  *max_degree = st.max_degree;
  return 0;
}

uint64_t ref_choose_segment_count(uint64_t n, uint64_t m_stored,
                                  double avg_degree) {
  GraphStats st;
  st.n = n;
  st.m_stored = m_stored;
  st.avg_degree = avg_degree;
  return choose_segment_count(st);
}

// ---- engines --------------------------------------------------------------
// algo: 0 baseline, 1 baseline-mj, 2 atomic, 3 adaptive (bench.hpp:23).
// labels may be null.  seg_counters (3 per segment, capacity seg_cap) may be
// null.
static int run(int algo, const Graph& g, uint64_t segments, unsigned workers,
               uint64_t* labels, ref_metrics* out, uint64_t* seg_counters,
               uint64_t seg_cap) {
  try {
    DriverOptions opts;
    opts.workers = workers;
    DriverResult r;
    switch (algo) {
      case 0: r = baseline_cc(g, opts); break;
      case 1: r = baseline_mj_cc(g, opts); break;
      case 2: r = single_hook_cc(g, opts); break;
      case 3: r = adaptive_cc(g, segments, opts); break;
      default: return 1;
    }
    if (labels) std::memcpy(labels, r.labels.label.data(), g.n * sizeof(uint64_t));
    const RunMetrics& mx = r.metrics;
    if (out) {
      out->total_ms = mx.total_ms;
      out->hook_ms = mx.hook_ms;
      out->compress_ms = mx.compress_ms;
      out->s = mx.s;
      out->outer_iterations = mx.outer_iterations;
      out->hook_traversal_steps = mx.counters.hook_traversal_steps;
      out->cas_failures = mx.counters.cas_failures;
      out->jump_steps = mx.counters.jump_steps;
      out->components = mx.components;
      out->segments_clamped = mx.segments_clamped;
      out->workers = mx.workers;
    }
    if (seg_counters)
      for (uint64_t i = 0; i < mx.segment_counters.size() && i < seg_cap; ++i) {
        seg_counters[3 * i] = mx.segment_counters[i].hook_traversal_steps;
        seg_counters[3 * i + 1] = mx.segment_counters[i].cas_failures;
        seg_counters[3 * i + 2] = mx.segment_counters[i].jump_steps;
      }
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

int ref_run(int algo, uint64_t n, const uint64_t* uv, uint64_t m,
            uint64_t segments, unsigned workers, uint64_t* labels,
            ref_metrics* out, uint64_t* seg_counters, uint64_t seg_cap) {
  Graph g = make_graph(n, uv, m);
  return run(algo, g, segments, workers, labels, out, seg_counters, seg_cap);
}

// Graph handle so repeated timed runs do not rebuild the 16 B/edge Graph.
void* ref_graph_new32(uint64_t n, const uint32_t* uv, uint64_t m) {
  try {
    return new Graph(make_graph32(n, uv, m));
  } catch (...) {
    return nullptr;
  }
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

int ref_run_graph(int algo, void* gh, uint64_t segments, unsigned workers,
                  uint64_t* labels, ref_metrics* out) {
  return run(algo, *static_cast<Graph*>(gh), segments, workers, labels, out,
             nullptr, 0);
}

// ---- per-element kernels on a host forest ---------------------------------
int ref_hook(uint64_t* pi, uint64_t n, uint64_t u, uint64_t v) {
  ParentForest f = make_forest(pi, n);
  bool r = hook(u, v, f);
  read_forest(f, pi);
  return r ? 1 : 0;
}

int ref_jump(uint64_t* pi, uint64_t n, uint64_t v) {
  ParentForest f = make_forest(pi, n);
  bool r = jump(v, f);
  read_forest(f, pi);
  return r ? 1 : 0;
}

void ref_atomic_hook(uint64_t* pi, uint64_t n, uint64_t u, uint64_t v,
                     uint64_t* counters) {
  ParentForest f = make_forest(pi, n);
  KernelCounters c{counters[0], counters[1], counters[2]};
  atomic_hook(u, v, f, c);
  counters[0] = c.hook_traversal_steps;
  counters[1] = c.cas_failures;
  counters[2] = c.jump_steps;
  read_forest(f, pi);
}

void ref_multi_jump(uint64_t* pi, uint64_t n, uint64_t v, uint64_t* counters) {
  ParentForest f = make_forest(pi, n);
  KernelCounters c{counters[0], counters[1], counters[2]};
  multi_jump(v, f, c);
  counters[0] = c.hook_traversal_steps;
  counters[1] = c.cas_failures;
  counters[2] = c.jump_steps;
  read_forest(f, pi);
}

int ref_is_star(const uint64_t* pi, uint64_t n) {
  ParentForest f = make_forest(pi, n);
  return is_star(f) ? 1 : 0;
}

}  // extern "C"
