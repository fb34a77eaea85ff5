#pragma once
// Reference parallel.hpp (/root/reference/proj/include/hookcc/parallel.hpp)
// provided the fork-join ThreadPool that launched every phase on host
// threads.  On B200 that role is taken by device kernel launches inside a
// CUDA graph (csrc/hcc_capi.cu), so only the worker-count query remains for
// API compatibility (acceptance.cpp uses it to pick worker settings).

#include <thread>

namespace hookcc {

/// Host hardware concurrency (parallel.hpp:13-16); never 0.
inline unsigned hardware_workers() {
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? hc : 1u;
}

}  // namespace hookcc
