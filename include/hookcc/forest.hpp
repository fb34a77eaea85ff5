#pragma once
// Parent forest and per-element kernels — header-compatible with the
// reference forest.hpp (/root/reference/proj/include/hookcc/forest.hpp:12-148).
//
// B200 design: the forest lives in HBM as u32[n] (hcc_forest).  Every
// element operation (load/store/cas and the Fig. 2/3 kernels hook, jump,
// atomic_hook, multi_jump) is a device kernel launched on the calling
// thread's per-thread stream, so concurrent host threads race on the device
// exactly as the reference's threads race on std::atomic slots.  The engines
// (engines.hpp) run their whole loop on the device over the same buffer.
// A forest handed to a phase observer carries a host snapshot, so observer
// loops over load(v) cost no device round trips.

#include <cstdint>
#include <memory>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "hookcc/detail.hpp"
#include "hookcc/graph.hpp"

namespace hookcc {

class ParentForest {
 public:
  explicit ParentForest(Vertex n) {
    detail::check(hcc_forest_create(detail::ctx(), n, &f_));
    n_ = n;
    owned_ = true;
  }
  ParentForest(const ParentForest&) = delete;
  ParentForest& operator=(const ParentForest&) = delete;
  ParentForest(ParentForest&& o) noexcept { swap(o); }
  ParentForest& operator=(ParentForest&& o) noexcept {
    swap(o);
    return *this;
  }
  ~ParentForest() {
    if (owned_ && f_) hcc_forest_free(f_);
  }

  Vertex size() const { return n_; }

  /// pi(v) = v for all v (forest.hpp:25-28).
  void reset() {
    mirror_.reset();
    detail::check(hcc_forest_reset(f_));
  }

  Vertex load(Vertex v) const {
    if (mirror_) return (*mirror_)[v];
    std::uint64_t out = 0;
    detail::check(hcc_forest_load(f_, v, &out));
    return out;
  }

  void store(Vertex v, Vertex parent) {
    mirror_.reset();
    detail::check(hcc_forest_store(f_, v, parent));
  }

  /// On failure `expected` holds the observed value (forest.hpp:39-43).
  bool cas(Vertex v, Vertex& expected, Vertex desired) {
    mirror_.reset();
    int ok = 0;
    std::uint64_t e = expected;
    detail::check(hcc_forest_cas(f_, v, &e, desired, &ok));
    expected = e;
    return ok != 0;
  }

  std::vector<Vertex> snapshot() const {
    if (mirror_) return *mirror_;
    std::vector<Vertex> out(n_);
    detail::check(hcc_forest_download_u64(f_, out.data()));
    return out;
  }

  std::string dump() const {
    std::ostringstream os;
    std::vector<Vertex> s = snapshot();
    for (Vertex v = 0; v < s.size(); ++v) os << (v ? " " : "") << s[v];
    return os.str();
  }

  hcc_forest* handle() const { return f_; }

  /// Non-owning view of a device forest with a host snapshot (observer use).
  static ParentForest view_with_snapshot(hcc_forest* f) {
    ParentForest p;
    p.f_ = f;
    p.owned_ = false;
    std::uint64_t n = 0;
    detail::check(hcc_forest_size(f, &n));
    p.n_ = n;
    auto snap = std::make_shared<std::vector<Vertex>>(n);
    detail::check(hcc_forest_download_u64(f, snap->data()));
    p.mirror_ = std::move(snap);
    return p;
  }
  bool has_snapshot() const { return static_cast<bool>(mirror_); }

 private:
  ParentForest() = default;
  void swap(ParentForest& o) noexcept {
    std::swap(f_, o.f_);
    std::swap(n_, o.n_);
    std::swap(owned_, o.owned_);
    std::swap(mirror_, o.mirror_);
  }

  hcc_forest* f_ = nullptr;
  Vertex n_ = 0;
  bool owned_ = false;
  std::shared_ptr<std::vector<Vertex>> mirror_;
};

/// Work counters (forest.hpp:65-75).
struct KernelCounters {
  std::uint64_t hook_traversal_steps = 0;
  std::uint64_t cas_failures = 0;
  std::uint64_t jump_steps = 0;

  void merge(const KernelCounters& o) {
    hook_traversal_steps += o.hook_traversal_steps;
    cas_failures += o.cas_failures;
    jump_steps += o.jump_steps;
  }
};

inline ParentForest init_forest(Vertex n) { return ParentForest(n); }

/// Atomic-free hook (Fig. 2; forest.hpp:83-89): one device thread.
inline bool hook(Vertex u, Vertex v, ParentForest& pi) {
  int changed = 0;
  detail::check(hcc_forest_hook(pi.handle(), u, v, &changed));
  return changed != 0;
}

/// Single-level shortcut (forest.hpp:93-99).
inline bool jump(Vertex v, ParentForest& pi) {
  int changed = 0;
  detail::check(hcc_forest_jump(pi.handle(), v, &changed));
  return changed != 0;
}

/// CAS-verified hook walking down to a root (Fig. 3; forest.hpp:107-122).
inline void atomic_hook(Vertex u, Vertex v, ParentForest& pi,
                        KernelCounters& counters) {
  hcc_counters c{0, 0, 0};
  detail::check(hcc_forest_atomic_hook(pi.handle(), u, v, &c));
  counters.hook_traversal_steps += c.hook_traversal_steps;
  counters.cas_failures += c.cas_failures;
}

/// Multi-Jump with eager writes (Fig. 3; forest.hpp:127-136).
inline void multi_jump(Vertex v, ParentForest& pi, KernelCounters& counters) {
  hcc_counters c{0, 0, 0};
  detail::check(hcc_forest_multi_jump(pi.handle(), v, &c));
  counters.jump_steps += c.jump_steps;
}

/// Every tree has depth <= 1 (forest.hpp:140-146): a device reduction, or
/// the host snapshot of an observer view.
inline bool is_star(const ParentForest& pi) {
  if (pi.has_snapshot()) {
    std::vector<Vertex> s = pi.snapshot();
    for (Vertex v = 0; v < s.size(); ++v)
      if (s[s[v]] != s[v]) return false;
    return true;
  }
  if (pi.size() == 0) return true;
  int ok = 0;
  detail::check(hcc_forest_is_star(pi.handle(), &ok));
  return ok != 0;
}

}  // namespace hookcc
