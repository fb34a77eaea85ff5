#pragma once
// Shared plumbing of the header-compatible C++ API: error mapping from the
// C-ABI status codes back to the reference's exception types
// (SURVEY.md §8b "Errors"), and the per-thread default device context
// (one hcc_ctx per host thread, replacing the per-call ThreadPool of
// engines.hpp:125-126).

#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "hookcc_c.h"

namespace hookcc {

/// A CUDA / device failure surfaced through the C-ABI (no reference
/// equivalent: the reference has no device).
class DeviceError : public std::runtime_error {
 public:
  DeviceError(int code, const std::string& what)
      : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

namespace detail {

[[noreturn]] inline void throw_status(int code) {
  std::string msg = hcc_last_error();
  switch (code) {
    case HCC_EINVAL:
    case HCC_ERANGE:
      throw std::invalid_argument(msg);
    case HCC_ENOTSTAR:
      throw std::logic_error(msg);
    case HCC_ENOMEM:
      throw std::bad_alloc();
    default:
      throw DeviceError(code, msg);
  }
}

inline void check(int code) {
  if (code != HCC_OK) throw_status(code);
}

/// Device used by the header API: $HOOKCC_DEVICE or 0.
inline int default_device() {
  const char* e = std::getenv("HOOKCC_DEVICE");
  return e ? std::atoi(e) : 0;
}

/// The calling thread's context (created on first use, destroyed at thread
/// exit).  Contexts are not shared between threads.
inline hcc_ctx* ctx() {
  struct Holder {
    hcc_ctx* c = nullptr;
    ~Holder() {
      if (c) hcc_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) {
    // structs cross the boundary by value: refuse a library built against
    // another revision of hookcc_c.h
    if (hcc_abi_version() != HCC_ABI_VERSION)
      throw std::runtime_error("libhookcc_cuda.so ABI " + std::to_string(hcc_abi_version()) +
                               " != header ABI " + std::to_string(HCC_ABI_VERSION) +
                               " (rebuild the binary)");
    check(hcc_create(default_device(), &h.c));
  }
  return h.c;
}

/// The calling thread's multi-device context for a device list (created on
/// first use, kept for the thread's lifetime: the shard buffers and cached
/// CUDA graphs are reused across calls).
inline hcc_ctx* multi_ctx(const std::vector<int>& devices) {
  struct Holder {
    std::map<std::vector<int>, hcc_ctx*> m;
    ~Holder() {
      for (auto& kv : m) hcc_destroy(kv.second);
    }
  };
  thread_local Holder h;
  auto it = h.m.find(devices);
  if (it != h.m.end()) return it->second;
  ctx();  // ABI check
  hcc_ctx* c = nullptr;
  check(hcc_create_multi(devices.data(), static_cast<int>(devices.size()), &c));
  h.m.emplace(devices, c);
  return c;
}

}  // namespace detail
}  // namespace hookcc
