// Host-side internals shared by the C-ABI translation units of
// libhookcc_cuda.so (not installed; the public boundary is hookcc_c.h):
//   hcc_capi.cu        contexts, graphs, forests, the CC engines
//   hcc_multi_host.cu  multi-device contexts (hcc_create_multi)
//   hcc_peer.cu        multi-process merge over CUDA IPC (hcc_peer_*)
// Error plumbing: helpers throw CudaFail (HCC_CUDA) and every extern "C"
// entry point converts it back to a status code (HCC_GUARD_*), with the
// message in the thread-local g_err (hcc_last_error).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "hcc_internal.cuh"
#include "hookcc_c.h"

// (internal header: the translation units that include it all work in the
// kernel namespace)
using namespace hcc;

namespace hcc {
namespace host {

extern thread_local std::string g_err;
int fail(int code, const std::string& msg);

struct CudaFail {
  int code;
};

// Device-side narrowing works on 32-bit ids.
constexpr u64 kMaxN = 0xffffffffull;
// Topology segments unrolled into the root graph (with per-launch events).
constexpr u64 kMaxUnrolledSegments = 64;

}  // namespace host
}  // namespace hcc

#define HCC_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
      throw CudaFail{e_ == cudaErrorMemoryAllocation ? HCC_ENOMEM           \
                                                      : HCC_ECUDA};         \
    }                                                                        \
  } while (0)

#define HCC_GUARD_BEGIN try {
#define HCC_GUARD_END                                                        \
  }                                                                          \
  catch (const CudaFail& f) {                                                \
    return f.code;                                                           \
  }                                                                          \
  catch (const std::bad_alloc&) {                                            \
    return fail(HCC_ENOMEM, "host allocation failed");                       \
  }                                                                          \
  catch (const std::exception& ex) {                                         \
    return fail(HCC_ECUDA, ex.what());                                       \
  }

// ---------------------------------------------------------------------------
// handles

// Per-shard state of a multi-device merge (hcc_create_multi).
struct MergeShard {
  u32* bits = nullptr;       // export bitmap, ceil(n/32) words
  u64 bits_words = 0;
  uint2* pairs = nullptr;    // export pairs
  u64 cap = 0;
  u64* cnt = nullptr;        // device: pairs the export produced
  PeerTab* tab = nullptr;    // device: every shard's export buffers
  bool tab_dirty = true;
  cudaEvent_t ev_exp = nullptr, ev_t0 = nullptr, ev_m0 = nullptr, ev_t1 = nullptr;
  hcc_forest* forest = nullptr;  // local forest (shard 0 may use the caller's)
  double local_ms = 0, merge_ms = 0, total_ms = 0;
  u64 passes = 0, records = 0, exported = 0, linked = 0;
};

struct GraphKey {
  int algo = -1;
  const void* edges = nullptr;
  const void* pi = nullptr;
  const void* wl0 = nullptr;
  const void* wl1 = nullptr;
  const void* s0b = nullptr;
  const void* s0f = nullptr;
  u64 wl_cap = 0;
  u64 n = 0, m = 0, nseg = 0, max_threads = 0;
  u32 flags = 0;
  int walk = 0;
  u64 plan = 0;
  bool s0b_on = false;
  bool sum = false;
  bool operator==(const GraphKey& o) const {
    return algo == o.algo && edges == o.edges && pi == o.pi && wl0 == o.wl0 &&
           wl1 == o.wl1 && s0b == o.s0b && s0f == o.s0f && wl_cap == o.wl_cap &&
           n == o.n && m == o.m && nseg == o.nseg &&
           max_threads == o.max_threads && flags == o.flags && walk == o.walk &&
           plan == o.plan && s0b_on == o.s0b_on && sum == o.sum;
  }
};

struct hcc_ctx {
  int dev = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  DevCtrl* d_ctrl = nullptr;
  DevRec* d_recs = nullptr;
  DevCtrl* h_ctrl = nullptr;  // pinned
  DevRec* h_recs = nullptr;   // pinned
  u32* scratch_pi = nullptr;
  u64 scratch_n = 0;
  uint2* wl[2] = {nullptr, nullptr};
  u64 wl_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int occ_hook = 1, occ_vert = 1, occ_hook_sum = 1, occ_hook_cas = 1, occ_hook_sum_cas = 1,
      occ_hook_sumd = 1, occ_hook_cas_sumd = 1;
  // cached executable graph for repeated calls with identical arguments,
  // plus the previous one (two graphs used alternately, e.g. a pipelined
  // upload into one while the other runs, keep both instantiated)
  cudaGraphExec_t exec = nullptr;
  GraphKey key;
  cudaGraphExec_t alt_exec = nullptr;
  GraphKey alt_key;
  u64 alt_seg_ev = 0;
  std::vector<int> alt_slot_kernel;
  int alt_wl_kernel = 0;
  cudaStream_t copy_stream = nullptr;  // hcc_graph_upload_async
  cudaEvent_t order_ev = nullptr;      // copy stream after the context stream
  cudaStream_t check_stream = nullptr; // endpoint checks of landed chunks
  std::vector<cudaEvent_t> chunk_ev;   // one per in-flight upload chunk
  std::vector<hcc_segment_rec> last_recs;
  // CUDA events around the unrolled topology hook launches
  std::vector<cudaEvent_t> seg_ev;   // 2 per segment
  u64 seg_ev_used = 0;
  u64 exec_seg_ev = 0;  // seg_ev_used of the cached executable graph
  // hook kernel per unrolled slot (HCC_HOOK_KERNEL_*; SUM means "voted:
  // summary or streaming") and of the worklist passes, as enqueued
  std::vector<int> slot_kernel, exec_slot_kernel;
  int wl_kernel = 0, exec_wl_kernel = 0;
  u32* s0b = nullptr;  // star-0 bitmap
  u32* s0b_base = nullptr;  // its allocation
  u64 s0b_words = 0;
  u32* s0f = nullptr;  // star-0 summary (one bit per group of bitmap words)
  u64 s0f_words = 0;
  // a worklist overflowed once: size the lists to m from now on
  bool wl_full = false;
  // multi-device context (hcc_create_multi): one sub-context per edge
  // shard (devices may repeat), merge buffers per shard
  std::vector<hcc_ctx*> subs;
  std::vector<MergeShard> merge;
  int peer_access = 0;
  // multi-process merge over CUDA IPC (hcc_peer_*)
  struct hcc_peer_state* peer = nullptr;
};

struct hcc_graph {
  hcc_ctx* ctx = nullptr;
  u64 n = 0, m = 0;
  u64 first = 0;  // global index of edge 0 (ranged / shard graphs)
  // multi-device graph: shard r (partition_edges(m, shards)) on ctx->subs[r]
  std::vector<hcc_graph*> shards;
  std::vector<u64> bounds;
  uint2* d_edges = nullptr;
  bool has_stats = false;
  hcc_graph_stats stats{};
  // hcc_graph_upload_async: copy + endpoint check in flight on the
  // context's copy stream; every reader waits for it (graph_ready)
  mutable bool pending = false;
  cudaEvent_t up_ev = nullptr;
  u32* d_err = nullptr;  // device endpoint-check flag
  u32* h_err = nullptr;  // pinned copy of it
};

struct hcc_forest {
  hcc_ctx* ctx = nullptr;
  int dev = 0;
  u64 n = 0;
  u32* d_pi = nullptr;
};

namespace hcc {
namespace host {

// hcc_capi.cu
void drop_exec(hcc_ctx* c);
void ensure_wl(hcc_ctx* c, u64 cap);
unsigned grid_for(u64 work, unsigned block, u64 cap);
int ctx_enter(hcc_ctx* c);
int graph_ready(const hcc_graph* g);
int compute_stats_dev(hcc_ctx* c, hcc_graph* g);
std::vector<u64> uniform_bounds(u64 m, u64 s);
int run_cc_sized(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o, hcc_forest* f,
                 hcc_metrics* mx);
// Re-hook the worklist records already in wl[0] (ctrl->wl_count[0]) into pi
// with the worklist engine, host-stepped (rehook_plan + rehook_loop).
void enqueue_rehook(hcc_ctx* c, u32* pi, u64 n);

// hcc_multi_host.cu
int multi_from_edges(hcc_ctx* c, const void* uv, bool wide, u64 m, u64 n, hcc_graph** out);
int multi_generate(hcc_ctx* c, const char* spec, u64 seed, u64 n, u64 first, u64 count,
                   hcc_graph** out);
int multi_range_io(hcc_ctx* c, hcc_graph* g, uint32_t* uv, u64 first, u64 count, int op);
int multi_stats(hcc_ctx* c, const hcc_graph* g, hcc_graph_stats* out);
int multi_cc(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o, hcc_forest* f, uint32_t* lab32,
             uint64_t* lab64, hcc_metrics* mx);

// hcc_peer.cu
void peer_release(hcc_ctx* c);

}  // namespace host
}  // namespace hcc
