// C-ABI implementation of libhookcc_cuda.so: contexts, graph handles,
// device forests and the CC engines.  (Multi-device contexts:
// hcc_multi_host.cu; the multi-process IPC merge: hcc_peer.cu; shared
// handles and helpers: hcc_host.cuh.)
//
// Engines (reference drivers, /root/reference/proj/include/hookcc/engines.hpp):
//   BASELINE     (123-179)  loop { hook all edges ; loop { jump } } until no
//                           hook changed
//   BASELINE_MJ  (183-231)  north-star engine: segmented topology-driven
//                           hook pass, then data-driven passes over the
//                           device-compacted worklist of (H, L) pairs, each
//                           followed by Multi-Jump; converged when a pass
//                           appends nothing.  HCC_FLAG_FULL_PASSES gives the
//                           reference's literal "re-hook every edge" loop.
//   ATOMIC/ADAPTIVE (238-300) per segment: CAS hook + Multi-Jump.
//
// Every loop runs on the device: the body is captured into the body graph
// of a CUDA-graph conditional WHILE node and the last kernel of the body
// sets the condition, so an hcc_cc call is one cudaGraphLaunch with no
// host round trip per iteration (HCC_FLAG_HOST_LOOP / observer mode drive
// the same kernels from the host instead).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "hookcc_gen.h"
#include "hcc_host.cuh"

using namespace hcc::host;

// ---------------------------------------------------------------------------
// errors

namespace hcc {
namespace host {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace host
}  // namespace hcc

namespace {

// Root-walk steps of the atomic-free hook before an unconditional store
// (HCC_WALK overrides, for tuning).
// Root-walk bound (HCC_WALK) and the steady slot's (HCC_WALK_LAST).  In
// lockstep one long walk holds its whole warp-tile, so shorter bounds defer
// the rare long walks to the worklist pass instead (after a compress they
// are short): grid 4096^2 1.06 -> 0.87 ms; RMAT-24 and ER-2^24 unchanged
// (ER's forming slots need 16: at 8 their deferrals inflate the store ratio).
constexpr int kDefaultWalk = 16;
constexpr int kDefaultWalkLast = 4;
// Fig. 3's walk runs until it links (the streaming CAS hook of the adaptive
// engine has no worklist to defer to).
constexpr int kUnboundedWalk = 1 << 30;
// Unrolled adaptive chains run the star pick in segments 1..kAdaptivePicks
// (the giant has formed by then; HCC_ADAPT_PICKS overrides).
constexpr int kAdaptivePicks = 4;
// First adaptive topology segment = m >> kAdaptShift (HCC_PLAN=adapt:<k>).
constexpr u32 kAdaptShift = 7;
// Unrolled adaptive slots (HCC_PLAN=adapt:<k>:<slots>); the last takes every
// remaining edge, so a plan never needs an empty trailing launch.
constexpr int kAdaptSlots = 4;
// Floor of the first adaptive segment: n >> kAdaptNShift edges
// (HCC_PLAN_NSHIFT; 0 disables, the default).  n/8 takes sparse ER (2^25
// vertices, 4 edges each) from 5.2 to 4.0 ms but costs grid 4096^2 0.1 ms
// (a lattice wants a small first segment); the BASELINE configs are dense.
constexpr u32 kAdaptNShift = 0;

int usable_devices() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int usable = 0;
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10)
      ++usable;
  }
  return usable;
}

}  // namespace

namespace hcc {
namespace host {

// Per-host-thread scratch for element operations (ParentForest API):
// results travel through a pinned buffer on the thread's default stream.
struct ThreadScratch {
  int dev = -1;
  u64* d_res = nullptr;
  u64* h_res = nullptr;
  ~ThreadScratch() {
    // process teardown: leaking is harmless and avoids calls into a
    // possibly-destroyed runtime
  }
};
thread_local ThreadScratch t_scratch;

u64* thread_scratch(int dev, u64** host) {
  if (t_scratch.dev != dev) {
    HCC_CUDA(cudaSetDevice(dev));
    u64* d = nullptr;
    u64* h = nullptr;
    HCC_CUDA(cudaMalloc(&d, 8 * sizeof(u64)));
    HCC_CUDA(cudaMallocHost(&h, 8 * sizeof(u64)));
    t_scratch.dev = dev;
    t_scratch.d_res = d;
    t_scratch.h_res = h;
  }
  *host = t_scratch.h_res;
  return t_scratch.d_res;
}

void drop_exec(hcc_ctx* c);

// Every buffer an executable graph bakes into its kernel arguments (pi,
// worklists, star bitmap and summary) is sized here; a reallocation drops
// the cached graphs, whose arguments would otherwise point at freed memory.
void ensure_pi(hcc_ctx* c, u64 n) {
  if (c->scratch_n >= n && c->scratch_pi) return;
  drop_exec(c);
  if (c->scratch_pi) HCC_CUDA(cudaFree(c->scratch_pi));
  c->scratch_pi = nullptr;
  c->scratch_n = 0;
  HCC_CUDA(cudaMalloc(&c->scratch_pi, std::max<u64>(n, 4) * sizeof(u32)));
  c->scratch_n = n;
}

void ensure_wl(hcc_ctx* c, u64 cap) {
  cap = std::max<u64>(cap, 1024);
  if (c->wl_cap >= cap) return;
  drop_exec(c);
  for (int i = 0; i < 2; ++i) {
    if (c->wl[i]) HCC_CUDA(cudaFree(c->wl[i]));
    c->wl[i] = nullptr;
  }
  c->wl_cap = 0;
  for (int i = 0; i < 2; ++i) HCC_CUDA(cudaMalloc(&c->wl[i], cap * sizeof(uint2)));
  c->wl_cap = cap;
}

void ensure_s0b(hcc_ctx* c, u64 nwords) {
  if (c->s0b_words >= nwords) return;
  drop_exec(c);
  if (c->s0b_base) HCC_CUDA(cudaFree(c->s0b_base));
  c->s0b = c->s0b_base = nullptr;
  c->s0b_words = 0;
  // HCC_S0B_PAD (bytes, experiment): offset of the bitmap inside its
  // allocation (L2 set aliasing against pi)
  const u64 pad = std::getenv("HCC_S0B_PAD") ? std::strtoull(std::getenv("HCC_S0B_PAD"), nullptr, 0) : 0;
  HCC_CUDA(cudaMalloc(&c->s0b_base, std::max<u64>(nwords, 1) * sizeof(u32) + pad));
  c->s0b = reinterpret_cast<u32*>(reinterpret_cast<char*>(c->s0b_base) + (pad & ~15ull));
  c->s0b_words = nwords;
}

void ensure_s0f(hcc_ctx* c, u64 nwords) {
  if (c->s0f_words >= nwords) return;
  drop_exec(c);
  if (c->s0f) HCC_CUDA(cudaFree(c->s0f));
  c->s0f = nullptr;
  c->s0f_words = 0;
  HCC_CUDA(cudaMalloc(&c->s0f, std::max<u64>(nwords, 1) * sizeof(u32)));
  c->s0f_words = nwords;
}

void drop_exec(hcc_ctx* c) {
  if (c->exec) cudaGraphExecDestroy(c->exec);
  c->exec = nullptr;
  c->key = GraphKey{};
  if (c->alt_exec) cudaGraphExecDestroy(c->alt_exec);
  c->alt_exec = nullptr;
  c->alt_key = GraphKey{};
}

unsigned grid_for(u64 work, unsigned block, u64 cap) {
  u64 g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  if (g > 0x7fffffffull) g = 0x7fffffffull;
  return (unsigned)g;
}

// ---- sequence builder: CUDA-graph capture or host-driven loop -------------

struct Seq {
  hcc_ctx* c;
  bool graph_mode;
  std::vector<cudaStream_t> streams;  // streams[d] captures nesting depth d
  int depth = 0;
  std::function<void(int)> on_phase;  // observer hook (host mode only)

  cudaStream_t s() const { return streams[depth]; }

  void phase_done(int phase) {
    if (!graph_mode && on_phase) on_phase(phase);
  }

  // Event record usable both eagerly and inside a stream capture (an
  // external event-record node of the root graph).
  void record(cudaEvent_t ev) {
    if (graph_mode)
      HCC_CUDA(cudaEventRecordWithFlags(ev, s(), cudaEventRecordExternal));
    else
      HCC_CUDA(cudaEventRecord(ev, s()));
  }

  // while (cond) body(h, use_cond); the body's last kernel sets the
  // condition. The body always executes at least once.
  void loop(const std::function<void(cudaGraphConditionalHandle, int)>& body) {
    if (!graph_mode) {
      for (;;) {
        body(0, 0);
        HCC_CUDA(cudaMemcpyAsync(&c->h_ctrl->cond, &c->d_ctrl->cond,
                                 sizeof(u32), cudaMemcpyDeviceToHost, s()));
        HCC_CUDA(cudaStreamSynchronize(s()));
        if (!c->h_ctrl->cond) break;
      }
      return;
    }
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    HCC_CUDA(cudaStreamGetCaptureInfo(s(), &st, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    if (depth == 0) {
      // top-level loop: the default value 1 is applied at every launch of
      // the root graph, so the body runs at least once without a kernel
      HCC_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    } else {
      // An upstream kernel arms the condition on every entry, so a nested
      // loop re-runs after an earlier pass left its condition at 0 (default
      // values are only applied at top-level graph launch).
      HCC_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
      k_set_cond<<<1, 1, 0, s()>>>(h, 1u);
      HCC_CUDA(cudaGetLastError());
      HCC_CUDA(cudaStreamGetCaptureInfo(s(), &st, nullptr, &g, &deps, &nd));
    }
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    HCC_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
    HCC_CUDA(cudaStreamUpdateCaptureDependencies(
        s(), &node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body_graph = p.conditional.phGraph_out[0];
    if ((int)streams.size() <= depth + 1) {
      cudaStream_t ns;
      HCC_CUDA(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
      streams.push_back(ns);
    }
    ++depth;
    HCC_CUDA(cudaStreamBeginCaptureToGraph(s(), body_graph, nullptr, nullptr,
                                           0, cudaStreamCaptureModeRelaxed));
    body(h, 1);
    cudaGraph_t out = nullptr;
    HCC_CUDA(cudaStreamEndCapture(s(), &out));
    --depth;
  }
};

struct Plan {
  int algo;
  bool full_passes;
  u64 n, m;
  const uint2* edges;
  u32* pi;
  uint2* wl0;
  uint2* wl1;
  u64 nseg;
  std::vector<u64> bounds;  // unrolled topology segment boundaries (nseg+1)
  int walk;
  int walk_last = 0;        // root-walk bound of the last (steady) topology slot
  bool s0b;                 // star-0 bitmap for hook passes after a compress
  bool sum = false;         // star-0 summary staged in the hook's shared memory
  bool chunked = false;     // streaming hooks with per-warp chunked appends
  bool small_slots = true;  // forming slots below two tiles use k_hook_small
  // HCC_HOOK_CAS: root stores by CAS (no record, no re-check) in 0: no
  // launch; 1: the worklist passes (stores are rare there); 2: also the
  // last topology slot
  int cas_mode = 1;
  u32 sum_words = 0, sum_shift = 0;
  bool hook_events = false;  // CUDA events around unrolled hook launches
  bool adapt;               // device-side adaptive topology plan
  u32 adapt_shift;          // first adaptive segment = m >> adapt_shift ...
  u64 adapt_first = 0;      // ... or n >> kAdaptNShift if larger (edges)
  u32 forming_pct;          // store ratio (%) above which a segment is forming
  unsigned grid_hook, block_hook, grid_vert, block_vert;
  unsigned grid_cas = 1;    // k_hook_cas grid (kHookCasCta threads per CTA)
  bool cas_stream = false;  // atomic / adaptive on the streaming CAS hook
  bool dyn = true;          // streaming hooks take tiles dynamically (HCC_DYN=0: static)
  bool wide_compress = false;  // k_compress_s0b_w (n >= 2^26; HCC_COMP_WIDE overrides)
  // The steady slot's hook: k_hook_sumd (summary-predicated lookups: RMAT-24
  // 1.59 -> 1.47 ms, ER 2.19 -> 2.06, grid unchanged) instead of the device
  // vote between k_hook_sum and the plain k_hook (HCC_SUM_VOTE=1 restores
  // the vote, HCC_SUMD=0 the plain hook; 2: sumd in every streaming slot
  // after the first, measured slower).
  int sumd = 1;
  bool sum_vote = false;
  bool wl_sumd = true;         // worklist passes follow the steady slot's choice (HCC_WL_SUMD)
  // star pick in the streaming hook's last block instead of a k_star_pick
  // node (HCC_FOLD_PICK=1): measured no gain for the worklist engine
  // (RMAT-24 1.474 vs 1.477 ms, ER and grid slightly slower: the pick's
  // dependent chases then extend the hook's tail instead of a node)
  bool fold_pick = false;
  // HCC_SUMD_ANY=1: any streaming slot >= 2 (not only the one taking the
  // remaining edges) runs k_hook_sumd when the summary covers its sample
  bool sumd_any = false;
  // compress L2 prefetch distance in blocks (0: off), for pi beyond L2
  u32 comp_pf = 0;
  // sixteen vertices per compress thread (k_compress_s0b16; HCC_COMP16)
  bool comp16 = false;
  // middle topology slots on the two-sided streaming hook (k_hook_both;
  // HCC_HOOK_BOTH=0: the one-sided k_hook)
  bool hook_both = true;
};

HookArgs hook_args(hcc_ctx* c, const Plan& P, int mode, int append) {
  HookArgs a;
  a.edges = P.edges;
  a.m = P.m;
  a.b = 0;
  a.e = P.m;
  a.mode = mode;
  a.append = append;
  a.walk = append ? P.walk : 0;  // the literal full-pass loops keep Fig. 2
  a.s0b = nullptr;
  a.s0f = nullptr;
  a.s0f_words = a.s0f_shift = 0;
  a.pi = P.pi;
  a.wl0 = P.wl0;
  a.wl1 = P.wl1;
  a.wl_cap = c->wl_cap;
  a.chunked = 0;
  a.gate = kGateAlways;
  a.cas = 0;
  a.ctrl = c->d_ctrl;
  a.recs = c->d_recs;
  a.n = P.n;
  a.rec_idx = -1;
  a.dslot = -1;
  a.pick = 0;
  a.dyn = 0;
  return a;
}

// Star-0 lookups for a hook launch (bitmap, plus the summary table when the
// plan has one).
void use_s0b(hcc_ctx* c, const Plan& P, HookArgs& a) {
  a.s0b = c->s0b;
  if (P.sum) {
    a.s0f = c->s0f;
    a.s0f_words = P.sum_words;
    a.s0f_shift = P.sum_shift;
  }
}

// k_hook dynamic shared memory: the summary table, then one slow-path queue
// of 32 * kHookEPT edges per warp (hook_stream).
size_t hook_smem(const HookArgs& a, unsigned block) {
  if (!a.s0f) return 0;
  return (size_t)sum_region_words(a.s0f_words) * 4 + (size_t)((block + 31) / 32) * 32 * kHookEPT * 8;
}
constexpr size_t kHookSmemMax =
    (size_t)sum_region_words(kSumTableMaxBytes / 4) * 4 + (size_t)kHookSumCta * kHookEPT * 8;

// Unrolled topology slot that runs the small-segment hook (forming regime).
bool slot_small(const Plan& P, u64 sgi) {
  const u64 seg_edges = P.bounds[sgi + 1] - P.bounds[sgi];  // adaptive: estimate
  return P.small_slots && P.block_hook == kHookCta &&
         seg_edges < (u64)P.grid_hook * P.block_hook * kHookEPT * 2;
}

// Sixteen vertices per compress thread (k_compress_s0b16): measured RMAT-24
// 1.377 -> 1.381 ms, adaptive 2.659 -> 2.674, ER equal, RMAT-28 -0.06 ms,
// grid's adaptive engine 1.08 -> 0.855 ms (its row chains resolve in the
// thread's second half).  Off by default; HCC_COMP16=1.
#ifndef HCC_COMP16
#define HCC_COMP16 0
#endif
#ifndef HCC_S0B_MIN_LOG2
#define HCC_S0B_MIN_LOG2 20
#endif
constexpr u32 kS0bMinLog2 = HCC_S0B_MIN_LOG2;
// Star-bitmap compress over the full grid (a persistent grid with cp.async
// prefetch was slower: DESIGN.md §3.2).
void launch_compress_s0b(hcc_ctx* c, const Plan& P, cudaStream_t s, int rec_idx = -1,
                         int dslot = -1) {
  if (P.comp16 && (!P.sum || P.sum_shift == kSumHalfShift || P.sum_shift == 0))
    k_compress_s0b16<<<grid_for((P.n + 15) / 16, kVertThreads, 0x7fffffffull), kVertThreads, 0,
                       s>>>(P.pi, P.n, c->d_ctrl, c->d_recs, c->s0b, kCompressIfDirty,
                            P.sum ? c->s0f : nullptr, P.sum_words, P.sum_shift, rec_idx, dslot,
                            P.comp_pf ? P.comp_pf / 2 : 0u);
  else if (P.wide_compress)
    k_compress_s0b_w<<<grid_for((P.n + 7) / 8, kVertThreadsWide, 0x7fffffffull), kVertThreadsWide,
                       0, s>>>(P.pi, P.n, c->d_ctrl, c->d_recs, c->s0b, kCompressIfDirty,
                               P.sum ? c->s0f : nullptr, P.sum_words, P.sum_shift, rec_idx, dslot,
                               P.comp_pf);
  else
    k_compress_s0b<<<grid_for((P.n + 7) / 8, kVertThreads, 0x7fffffffull), kVertThreads, 0, s>>>(
        P.pi, P.n, c->d_ctrl, c->d_recs, c->s0b, kCompressIfDirty, P.sum ? c->s0f : nullptr,
        P.sum_words, P.sum_shift, rec_idx, dslot, P.comp_pf);
}

// Preferred shared-memory carveout (percent) of the forming-slot hook.  RMAT's
// first slot is contention-bound on the hubs' lines, and a carveout of 5-10%
// runs it in 0.14 ms instead of 0.18 ms (0%: 0.18, 25-100%: 0.22; ER and grid
// unchanged).  -1 leaves the driver's choice; HCC_HOOK_CARVE / HCC_COMP_CARVE
// (the streaming hooks / the compress) are experiment knobs, off by default
// (10% cost the steady hook 0.02 ms and ER's compresses 0.07 ms).
#ifndef HCC_SMALL_CARVE
#define HCC_SMALL_CARVE 8
#endif
#ifndef HCC_HOOK_CARVE
#define HCC_HOOK_CARVE -1
#endif
#ifndef HCC_COMP_CARVE
#define HCC_COMP_CARVE -1
#endif
// Streaming hook (chunked appends, full warps) or the block-aggregated one.
void launch_hook(const Plan& P, cudaStream_t s, const HookArgs& a) {
  if (a.chunked && (P.block_hook & 31u) == 0) {
    if (a.cas)
      k_hook_cas<<<P.grid_cas, kHookCasCta, 0, s>>>(a);
    else
      k_hook<<<P.grid_hook, P.block_hook, 0, s>>>(a);
  } else {
    k_hook_legacy<<<P.grid_hook, P.block_hook, 0, s>>>(a);
  }
}

// Summary-predicated streaming hook (the summary in shared memory, no
// queues).
void launch_hook_sumd(hcc_ctx* c, const Plan& P, cudaStream_t s, const HookArgs& a) {
  const size_t smem = (size_t)sum_region_words(a.s0f_words) * 4;
  if (P.sum_shift == kSumShiftFixed)
    k_hook_sumd<<<c->sms * c->occ_hook_sumd, kHookSumdCta, smem, s>>>(a);
  else
    k_hook_sumd_sh<<<c->sms * c->occ_hook_sumd, kHookSumdCta, smem, s>>>(a);
}

// Segment hook of the adaptive / atomic engines (no appends).  HCC_SEG_CAS=0
// uses the worklist passes' 768-thread k_hook_cas instead.
// With a one-bit-per-word star summary, the summary-predicated build
// (k_hook_seg_cas_sumd; HCC_SEG_SUMD=0 disables).
void launch_seg_cas(const Plan& P, cudaStream_t s, const HookArgs& a) {
  static const int v = std::getenv("HCC_SEG_CAS") ? std::atoi(std::getenv("HCC_SEG_CAS")) : 1;
  static const int sd = std::getenv("HCC_SEG_SUMD") ? std::atoi(std::getenv("HCC_SEG_SUMD")) : 1;
  if (v && sd && P.sum && P.sum_shift == 0 && a.s0f) {
    k_hook_seg_cas_sumd<<<P.grid_hook, kHookCta, (size_t)sum_region_words(a.s0f_words) * 4, s>>>(a);
  } else if (v && sd && P.sum && a.s0f) {
    k_hook_seg_cas_sumd_sh<<<P.grid_hook, kHookCta, (size_t)sum_region_words(a.s0f_words) * 4,
                             s>>>(a);
  } else if (v) {
    k_hook_seg_cas<<<P.grid_hook, kHookCta, 0, s>>>(a);
  } else {
    k_hook_cas<<<P.grid_cas, kHookCasCta, 0, s>>>(a);
  }
}

// The summary hook (one CTA per SM, the summary and queues in shared memory).
void launch_hook_sum(hcc_ctx* c, cudaStream_t s, const HookArgs& a) {
  if (a.cas)
    k_hook_sum_cas<<<c->sms * c->occ_hook_sum_cas, kHookCasCta, hook_smem(a, kHookCasCta), s>>>(a);
  else
    k_hook_sum<<<c->sms * c->occ_hook_sum, kHookSumCta, hook_smem(a, kHookSumCta), s>>>(a);
}

// Topology slot whose hook is voted between the summary and the plain
// streaming hook: the last one (the steady segment).  Earlier slots are in
// the forming regime, where no measured graph covers half of its summary
// groups, and a voted slot costs a second (gated) launch.
bool sum_slot(const Plan& P, u64 sgi) {
  return P.sum && P.adapt && sgi >= 1 && sgi + 1 == P.nseg && !slot_small(P, sgi);
}

// Unrolled adaptive-plan slot whose hook is chosen on the device between the
// summary-predicated k_hook_sumd (the slot that takes every remaining edge)
// and the plain k_hook (forming slots).
// (The step before the slot also checks the summary's coverage of a sample
// of the slot's endpoints, k_step_adapt: a coarse summary covers little of
// RMAT's lookups at n > 2^24, and the kernel's 64 KB of shared memory then
// only costs L1 -- RMAT-28's steady slot 27.4 -> 32.4 ms unconditionally --
// while it pays for ER at n = 2^26: 17.3 -> 14.5 ms.)
bool remainder_slot(const Plan& P, u64 sgi) {
  // (slot 1 would be the remainder only if the first m/128 edges left the
  // graph out of the forming regime: no gated pair there)
  return P.sumd == 1 && !P.sum_vote && P.sum && P.adapt &&
         P.chunked && sgi >= 2 && !slot_small(P, sgi) && !(P.cas_mode >= 2 && sgi + 1 == P.nseg);
}

// Enqueue one full CC run (pi init through convergence) on seq.
void enqueue_run(hcc_ctx* c, const Plan& P, Seq& q) {
  c->seg_ev_used = 0;
  c->slot_kernel.clear();
  c->wl_kernel = HCC_HOOK_KERNEL_LEGACY;
  // grid-stride init with 8 CTAs per SM: the 16 K-block vertex grid took
  // 21 us from run start to the first hook, this one 11 us (RMAT-24)
  const unsigned start_grid =
      std::min<unsigned>(P.grid_vert, (unsigned)c->sms * 8u);
  k_start<<<std::max(start_grid, 1u), P.block_vert, 0, q.s()>>>(
      P.pi, P.n, P.s0b ? c->s0b : nullptr, c->d_ctrl, c->d_recs, P.nseg, P.m,
      P.adapt ? P.adapt_first : 0, P.sum ? c->s0f : nullptr, P.sum_words);
  HCC_CUDA(cudaGetLastError());
  DevCtrl* ctrl = c->d_ctrl;
  DevRec* recs = c->d_recs;

  switch (P.algo) {
    case HCC_ALGO_BASELINE: {
      q.loop([&](cudaGraphConditionalHandle ho, int uo) {
        launch_hook(P, q.s(), 
            hook_args(c, P, kSrcRange, 0));
        q.phase_done(HCC_PHASE_HOOK);
        q.loop([&](cudaGraphConditionalHandle hi, int ui) {
          k_jump<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl, recs);
          k_step_jump<<<1, 1, 0, q.s()>>>(ctrl, hi, ui);
        });
        q.phase_done(HCC_PHASE_COMPRESS);
        k_step_outer<<<1, 1, 0, q.s()>>>(ctrl, recs, ho, uo);
      });
      break;
    }
    case HCC_ALGO_BASELINE_MJ: {
      if (P.full_passes) {
        q.loop([&](cudaGraphConditionalHandle h, int u) {
          launch_hook(P, q.s(), 
              hook_args(c, P, kSrcRange, 0));
          q.phase_done(HCC_PHASE_HOOK);
          k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl,
                                                              recs, 0);
          q.phase_done(HCC_PHASE_COMPRESS);
          k_step_outer<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
        });
        break;
      }
      // topology-driven first pass, segmented.  Few segments: unrolled in
      // the root graph with CUDA events around every hook launch (the
      // dominant kernel's per-launch time); many: a device loop.
      c->seg_ev_used = 0;
      if (P.nseg <= kMaxUnrolledSegments) {
        while (c->seg_ev.size() < 2 * P.nseg) {
          cudaEvent_t ev;
          HCC_CUDA(cudaEventCreate(&ev));
          c->seg_ev.push_back(ev);
        }
        for (u64 sgi = 0; sgi < P.nseg; ++sgi) {
          HookArgs ha = hook_args(c, P, P.adapt ? kSrcCtrlRange : kSrcRange, 1);
          ha.b = P.bounds[sgi];
          ha.e = P.bounds[sgi + 1];
          if (P.s0b && sgi >= 1) use_s0b(c, P, ha);
          // star of the next bitmap (the giant need not contain vertex 0),
          // not after the last slot (only the worklist passes would see
          // it): the streaming hooks' last block runs the pick (no
          // k_star_pick node), the small forming-slot hook gets the kernel
          const bool pick = P.s0b && P.adapt && sgi >= 1 && sgi + 1 < P.nseg;
          const bool pick_in_hook = pick && !slot_small(P, sgi) && P.fold_pick;
          ha.pick = pick_in_hook ? 1 : 0;
          if (P.hook_events) q.record(c->seg_ev[2 * sgi]);
          c->slot_kernel.push_back(slot_small(P, sgi)       ? HCC_HOOK_KERNEL_SMALL
                                   : remainder_slot(P, sgi) ? HCC_HOOK_KERNEL_SUMD
                                   : sum_slot(P, sgi) && !P.sum_vote ? HCC_HOOK_KERNEL_STREAM
                                   : sum_slot(P, sgi)   ? HCC_HOOK_KERNEL_SUM
                                   : P.chunked          ? HCC_HOOK_KERNEL_STREAM
                                                        : HCC_HOOK_KERNEL_LEGACY);
          if (slot_small(P, sgi)) {
            // forming-regime segment: EPT 2 over a full grid
            ha.s0f = nullptr;
            const u64 seg_edges = ha.e - ha.b;  // adaptive: the static estimate
            k_hook_small<<<grid_for((seg_edges + kSmallEPT - 1) / kSmallEPT + 1, kHookThreads,
                                    0x7fffffffull),
                           kHookThreads, 0, q.s()>>>(ha);
          } else {
            ha.chunked = P.chunked ? 1 : 0;
            ha.dyn = P.dyn && P.chunked ? 1 : 0;
            ha.cas = P.cas_mode >= 2 && sgi + 1 == P.nseg ? 1 : 0;
            if (P.adapt && sgi + 1 == P.nseg) ha.walk = P.walk_last;
            HookArgs hp = ha;  // plain streaming hook: bitmap only, full L1
            hp.s0f = nullptr;
            if (remainder_slot(P, sgi)) {
              // the slot that takes every remaining edge (decided on the
              // device by the previous step, which sets use_sum) streams
              // with summary-predicated lookups (k_hook_sumd), any other
              // with the plain hook; the one not chosen exits at entry
              HookArgs hd = ha;
              hd.gate = kGateIfSum;
              hp.gate = kGateIfPlain;
              launch_hook_sumd(c, P, q.s(), hd);
              launch_hook(P, q.s(), hp);
            } else if (sum_slot(P, sgi) && !P.sum_vote) {
              launch_hook(P, q.s(), hp);
            } else if (sum_slot(P, sgi)) {
              // the previous step's device vote picks the summary hook or
              // the plain one; the other launch exits at entry (cheaper
              // than an IF/ELSE graph node, measured ~20 us per slot)
              ha.gate = kGateIfSum;
              hp.gate = kGateIfPlain;
              launch_hook_sum(c, q.s(), ha);
              launch_hook(P, q.s(), hp);
            } else if (P.sumd >= 2 && P.sum && sgi >= 1 && !ha.cas) {
              HookArgs hd = ha;
              hd.gate = kGateAlways;
              launch_hook_sumd(c, P, q.s(), hd);
            } else if (P.hook_both && !hp.cas && hp.chunked) {
              // forming-side streaming slots: two-sided walks (768-thread
              // CTAs for their registers) leave shallower trees for the
              // compress (ER 1.876 -> 1.850 ms, grid -1%, RMAT unchanged)
              k_hook_both<<<(unsigned)c->sms, kHookBothCta, 0, q.s()>>>(hp);
            } else {
              launch_hook(P, q.s(), hp);
            }
          }
          if (P.hook_events) q.record(c->seg_ev[2 * sgi + 1]);
          q.phase_done(HCC_PHASE_HOOK);
          if (pick && !pick_in_hook) k_star_pick<<<1, 32, 0, q.s()>>>(P.pi, P.n, ctrl);
          // compress (+ star-0 bitmap, initialised by k_start)
          if (P.s0b)
            launch_compress_s0b(c, P, q.s());
          else
            k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl,
                                                                recs, 1);
          q.phase_done(HCC_PHASE_COMPRESS);
          // (a step folded into the compress's last block costs one
          // single-address atomic per compress block: slower than a launch)
          if (P.adapt) {
            // the next hook's summary vote rides on the step kernel (the
            // worklist passes reuse the last one: coverage only grows)
            // and so does the bitmap-use decision (a 2048-endpoint sample)
            const bool vote = sgi + 1 < P.nseg && sum_slot(P, sgi + 1) && P.sum_vote;
            const bool rvote = sgi + 1 < P.nseg && remainder_slot(P, sgi + 1);
            if (P.s0b)
              k_step_adapt<<<1, 1024, 0, q.s()>>>(ctrl, recs, P.m, P.forming_pct,
                                                 vote ? c->s0f : nullptr, P.sum_words,
                                                 P.edges, c->s0b, rvote ? c->s0f : nullptr,
                                                 P.sum_shift, P.sumd_any ? 1 : 0);
            else
              k_step_adapt<<<1, 1, 0, q.s()>>>(ctrl, recs, P.m, P.forming_pct, nullptr, 0,
                                              nullptr, nullptr, nullptr, 0, 0);
          } else
            k_step_segment<<<1, 1, 0, q.s()>>>(ctrl, recs, 0, 0);
        }
        c->seg_ev_used = P.hook_events ? P.nseg : 0;
      } else {
        q.loop([&](cudaGraphConditionalHandle h, int u) {
          launch_hook(P, q.s(), 
              hook_args(c, P, kSrcSegment, 1));
          q.phase_done(HCC_PHASE_HOOK);
          k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl,
                                                              recs, 1);
          q.phase_done(HCC_PHASE_COMPRESS);
          k_step_segment<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
        });
      }
      // data-driven passes over the compacted worklist
      q.loop([&](cudaGraphConditionalHandle h, int u) {
        HookArgs wa = hook_args(c, P, kSrcWorklist, 1);
        if (P.s0b && !P.bounds.empty()) use_s0b(c, P, wa);
        wa.chunked = P.chunked ? 1 : 0;
        wa.dyn = P.dyn && P.chunked ? 1 : 0;
        wa.cas = P.cas_mode >= 1 && P.chunked ? 1 : 0;
        c->wl_kernel = wa.cas ? HCC_HOOK_KERNEL_CAS
                              : (P.chunked ? HCC_HOOK_KERNEL_STREAM : HCC_HOOK_KERNEL_LEGACY);
        if (wa.s0f && P.adapt && !P.sum_vote && P.sumd == 1 && wa.cas && P.wl_sumd) {
          // after a steady slot that streamed with summary-predicated
          // lookups (use_sum still set), the worklist passes do too
          HookArgs wp = wa;
          wa.gate = kGateIfSum;
          wp.gate = kGateIfPlain;
          wp.s0f = nullptr;
          if (P.sum_shift == kSumShiftFixed)
            k_hook_cas_sumd<<<c->sms * c->occ_hook_cas_sumd, kHookCasCta,
                              (size_t)sum_region_words(wa.s0f_words) * 4, q.s()>>>(wa);
          else
            k_hook_cas_sumd_sh<<<c->sms * c->occ_hook_cas_sumd, kHookCasCta,
                                 (size_t)sum_region_words(wa.s0f_words) * 4, q.s()>>>(wa);
          launch_hook(P, q.s(), wp);
        } else if (wa.s0f && P.adapt && P.sum_vote) {
          HookArgs wp = wa;
          wa.gate = kGateIfSum;
          wp.gate = kGateIfPlain;
          wp.s0f = nullptr;
          launch_hook_sum(c, q.s(), wa);
          launch_hook(P, q.s(), wp);
        } else {
          wa.s0f = nullptr;
          launch_hook(P, q.s(), wa);
        }
        q.phase_done(HCC_PHASE_HOOK);
        if (P.s0b && !P.bounds.empty())
          launch_compress_s0b(c, P, q.s());
        else
          k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl,
                                                              recs, 1);
        q.phase_done(HCC_PHASE_COMPRESS);
        k_step_worklist<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
      });
      break;
    }
    default: {  // ATOMIC / ADAPTIVE
      if (P.cas_stream && P.nseg <= kMaxUnrolledSegments && P.bounds.size() == P.nseg + 1) {
        // unrolled: two launches per segment.  The hook's last block runs
        // the star pick of the early segments, the compress clears the next
        // segment's dirty flag, records are indexed by segment: no pick or
        // step launches, no loop node (31 segments on RMAT-24: 125 -> 63
        // kernels)
        int picks = kAdaptivePicks;
        if (const char* e = std::getenv("HCC_ADAPT_PICKS")) picks = std::atoi(e);
        for (u64 i = 0; i < P.nseg; ++i) {
          HookArgs a = hook_args(c, P, kSrcRange, 0);
          a.b = P.bounds[i];
          a.e = P.bounds[i + 1];
          a.walk = kUnboundedWalk;
          a.cas = 1;
          a.chunked = 1;
          a.s0b = c->s0b;
          a.rec_idx = (int)i;
          a.dslot = (int)(i & 1);
          a.dyn = P.dyn ? 1 : 0;
          if (P.sum) use_s0b(c, P, a);
          a.pick = i >= 1 && (int)i <= picks && i + 1 < P.nseg ? 1 : 0;
          c->slot_kernel.push_back(HCC_HOOK_KERNEL_CAS);
          launch_seg_cas(P, q.s(), a);
          q.phase_done(HCC_PHASE_HOOK);
          launch_compress_s0b(c, P, q.s(), (int)i, (int)(i & 1));
          q.phase_done(HCC_PHASE_COMPRESS);
        }
        break;
      }
      if (P.cas_stream) {
        // the paper's engine on the streaming machinery: per segment, the
        // CAS-storing streaming hook (16-byte edge loads, star-bitmap
        // lookups, lockstep walks that CAS only where they meet a root,
        // walks unbounded as in Fig. 3, no worklist), then the star pick and
        // the bitmap-building Multi-Jump compress (skipped when the segment
        // linked nothing)
        q.loop([&](cudaGraphConditionalHandle h, int u) {
          HookArgs a = hook_args(c, P, kSrcSegment, 0);
          a.walk = kUnboundedWalk;
          a.cas = 1;
          a.chunked = 1;
          a.s0b = c->s0b;
          a.dyn = P.dyn ? 1 : 0;
          if (P.sum) use_s0b(c, P, a);
          launch_seg_cas(P, q.s(), a);
          q.phase_done(HCC_PHASE_HOOK);
          k_star_pick<<<1, 32, 0, q.s()>>>(P.pi, P.n, ctrl);
          launch_compress_s0b(c, P, q.s());
          q.phase_done(HCC_PHASE_COMPRESS);
          k_step_segment<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
        });
        break;
      }
      q.loop([&](cudaGraphConditionalHandle h, int u) {
        k_cas_hook<<<P.grid_hook, P.block_hook, 0, q.s()>>>(
            hook_args(c, P, kSrcSegment, 0));
        q.phase_done(HCC_PHASE_HOOK);
        k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl,
                                                            recs, 0);
        q.phase_done(HCC_PHASE_COMPRESS);
        k_step_segment<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
      });
      break;
    }
  }
  HCC_CUDA(cudaGetLastError());
}

int ctx_enter(hcc_ctx* c) {
  if (!c) return fail(HCC_EINVAL, "null context");
  cudaError_t e = cudaSetDevice(c->dev);
  if (e != cudaSuccess) return fail(HCC_ECUDA, cudaGetErrorString(e));
  return HCC_OK;
}

// Device compute_stats (graph.hpp:43-68): keys (min<<32|max) of non-loop
// edges, radix sort, unique, degree histogram over the unique pairs.
__global__ void k_stat_keys(const uint2* e, u64 m, u64* keys) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    uint2 x = e[i];
    keys[i] = x.x == x.y ? ~0ull
                         : ((u64)min(x.x, x.y) << 32) | (u64)max(x.x, x.y);
  }
}

__global__ void k_stat_unique(const u64* k, u64 m, u32* deg, u64* uniq) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 cnt = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    u64 x = k[i];
    if (x == ~0ull) continue;
    if (i > 0 && k[i - 1] == x) continue;
    ++cnt;
    atomicAdd(deg + (x >> 32), 1u);
    atomicAdd(deg + (x & 0xffffffffull), 1u);
  }
  if (cnt) atomicAdd(uniq, cnt);
}

__global__ void k_stat_max(const u32* deg, u64 n, u32* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u32 mx = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    mx = max(mx, deg[i]);
  if (mx) atomicMax(out, mx);
}

int compute_stats_dev(hcc_ctx* c, hcc_graph* g) {
  hcc_graph_stats st{};
  st.n = g->n;
  st.m_stored = g->m;
  if (g->n == 0) {
    g->stats = st;
    g->has_stats = true;
    return HCC_OK;
  }
  u64 *keys = nullptr, *keys2 = nullptr, *d_uniq = nullptr;
  u32 *deg = nullptr, *d_max = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaStream_t s = c->stream;
  const u64 m = g->m;
  auto cleanup = [&] {
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(d_uniq);
    cudaFree(deg);
    cudaFree(d_max);
    cudaFree(tmp);
  };
  try {
    HCC_CUDA(cudaMalloc(&deg, std::max<u64>(g->n, 1) * sizeof(u32)));
    HCC_CUDA(cudaMalloc(&d_uniq, sizeof(u64)));
    HCC_CUDA(cudaMalloc(&d_max, sizeof(u32)));
    HCC_CUDA(cudaMemsetAsync(deg, 0, g->n * sizeof(u32), s));
    HCC_CUDA(cudaMemsetAsync(d_uniq, 0, sizeof(u64), s));
    HCC_CUDA(cudaMemsetAsync(d_max, 0, sizeof(u32), s));
    if (m > 0) {
      HCC_CUDA(cudaMalloc(&keys, m * sizeof(u64)));
      HCC_CUDA(cudaMalloc(&keys2, m * sizeof(u64)));
      k_stat_keys<<<grid_for(m, 256, 65536), 256, 0, s>>>(g->d_edges, m, keys);
      // radix sort in chunks of at most 2^31 keys per call is not needed for
      // CUB's 64-bit offset overload; use it directly.
      HCC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys2,
                                               (int64_t)m, 0, 64, s));
      HCC_CUDA(cudaMalloc(&tmp, tmp_bytes));
      HCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys2,
                                               (int64_t)m, 0, 64, s));
      k_stat_unique<<<grid_for(m, 256, 65536), 256, 0, s>>>(keys2, m, deg,
                                                            d_uniq);
    }
    k_stat_max<<<grid_for(g->n, 256, 65536), 256, 0, s>>>(deg, g->n, d_max);
    HCC_CUDA(cudaGetLastError());
    u64 uniq = 0;
    u32 mx = 0;
    HCC_CUDA(cudaMemcpyAsync(&uniq, d_uniq, sizeof(u64), cudaMemcpyDeviceToHost, s));
    HCC_CUDA(cudaMemcpyAsync(&mx, d_max, sizeof(u32), cudaMemcpyDeviceToHost, s));
    HCC_CUDA(cudaStreamSynchronize(s));
    st.m_unique = uniq;
    st.avg_degree = 2.0 * (double)uniq / (double)g->n;
    st.max_degree = mx;
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  g->stats = st;
  g->has_stats = true;
  return HCC_OK;
}

// Parse "k=v,k=v" parameters of a generator spec.
bool spec_get(const std::string& params, const std::string& key,
              std::string* out) {
  size_t pos = 0;
  while (pos <= params.size()) {
    size_t comma = params.find(',', pos);
    std::string item = params.substr(
        pos, comma == std::string::npos ? std::string::npos : comma - pos);
    size_t eq = item.find('=');
    if (eq != std::string::npos && item.substr(0, eq) == key) {
      *out = item.substr(eq + 1);
      return true;
    }
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return false;
}

bool parse_u64(const std::string& s, u64* out) {
  if (s.empty()) return false;
  u64 v = 0;
  for (char ch : s) {
    if (ch < '0' || ch > '9') return false;
    v = v * 10 + (u64)(ch - '0');
  }
  *out = v;
  return true;
}

// Worklist engine over re-hook records already in wl[0] (remote relations
// of a multi-GPU merge): the block-append hook, since the list sizes are
// exact (count + n), then Multi-Jump; host-stepped (a merge needs 1-3).
Plan rehook_plan(hcc_ctx* c, u32* pi, u64 n) {
  Plan P;
  P.algo = HCC_ALGO_BASELINE_MJ;
  P.full_passes = false;
  P.n = n;
  P.m = 0;
  P.edges = nullptr;
  P.pi = pi;
  P.wl0 = c->wl[0];
  P.wl1 = c->wl[1];
  P.nseg = 1;
  P.walk = kDefaultWalk;
  P.s0b = false;
  P.adapt = false;
  P.adapt_shift = 0;
  P.forming_pct = 0;
  P.block_hook = kHookCta;
  P.grid_hook = (unsigned)(c->sms * c->occ_hook);
  P.block_vert = kVertThreads;
  // grid-stride compress over a few CTAs per SM: after a merge the trees
  // are stars plus a few remote links, and a pass that finds the forest
  // clean exits at once (a full grid took 0.45 ms to do nothing at n = 2^28)
  P.grid_vert = grid_for((n + 3) / 4, kVertThreads, (u64)c->sms * 16);
  return P;
}

void rehook_loop(hcc_ctx* c, const Plan& P) {
  Seq q;
  q.c = c;
  q.graph_mode = false;
  q.streams.push_back(c->stream);
  DevCtrl* ctrl = c->d_ctrl;
  DevRec* recs = c->d_recs;
  q.loop([&](cudaGraphConditionalHandle h, int u) {
    // CAS stores and unbounded walks: no link is lost, so nothing is
    // re-recorded and one pass (plus the compress) converges (the plain
    // hook took a second pass and compress: 0.23 ms per merge at n = 2^28)
    HookArgs a = hook_args(c, P, kSrcWorklist, 1);
    a.cas = 1;
    a.chunked = 1;
    a.walk = kUnboundedWalk;
    k_hook_cas<<<(unsigned)(c->sms * c->occ_hook_cas), kHookCasCta, 0, q.s()>>>(a);
    k_compress<<<P.grid_vert, P.block_vert, 0, q.s()>>>(P.pi, P.n, ctrl, recs, 1);
    k_step_worklist<<<1, 1, 0, q.s()>>>(ctrl, recs, h, u);
  });
}

// (plan + host-stepped loop: the multi-GPU merges)
void enqueue_rehook(hcc_ctx* c, u32* pi, u64 n) { rehook_loop(c, rehook_plan(c, pi, n)); }

}  // namespace host
}  // namespace hcc

namespace hcc {
namespace host {

// Wait for a graph's pending asynchronous upload and report its endpoint
// check (check_endpoints, graph.hpp:89-94).  Every entry point that reads a
// graph's edges calls this first.
int graph_ready(const hcc_graph* g) {
  if (g)
    for (const hcc_graph* sh : g->shards)
      if (int r = graph_ready(sh)) return r;
  if (!g || !g->pending) return HCC_OK;
  const cudaError_t e = cudaEventSynchronize(g->up_ev);
  g->pending = false;
  if (e != cudaSuccess)
    return fail(HCC_ECUDA, std::string("graph upload: ") + cudaGetErrorString(e));
  if (*g->h_err) return fail(HCC_ERANGE, "edge endpoint out of range");
  return HCC_OK;
}

// partition_edges(m, s) boundaries (engines.hpp:43-58).
std::vector<u64> uniform_bounds(u64 m, u64 s) {
  std::vector<u64> b(s + 1, 0);
  const u64 q = m / s, r = m % s;
  for (u64 i = 0; i < s; ++i) b[i + 1] = b[i] + q + (i < r ? 1 : 0);
  return b;
}

// Auto plan for the topology pass: a short first segment
// builds the hub structure while trees are still forming (the expensive,
// walk-heavy regime), then each boundary grows by `growth` so the bulk of the
// edges streams in the cheap regime where both endpoints already share a
// star.  Every segment costs one compress over n, so few segments are used.
// HCC_PLAN="geo:<k>:<growth>" overrides (first boundary m / 2^k).
std::vector<u64> geometric_bounds(u64 m) {
  int k = 7, growth = 8;
  if (const char* e = std::getenv("HCC_PLAN")) {
    int kk = 0, gg = 0;
    if (std::sscanf(e, "geo:%d:%d", &kk, &gg) == 2 && kk >= 0 && gg >= 2) {
      k = kk;
      growth = gg;
    }
  }
  std::vector<u64> b{0};
  u64 cur = k >= 63 ? 0 : (m >> k);
  if (cur == 0) cur = std::min<u64>(m, 1);
  while (cur < m && b.size() < kMaxUnrolledSegments) {
    if (cur > b.back()) b.push_back(cur);
    const u64 next = cur * (u64)growth;
    cur = next / (u64)growth == cur ? next : m;  // overflow guard
  }
  if (b.back() != m || b.size() == 1) b.push_back(m);
  return b;
}

// run_cc's internal "worklist overflowed, repeat" code (never returned).
constexpr int kRerun = -1;

int run_cc(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o,
                  hcc_forest* f, hcc_metrics* mx);

// run_cc, repeated once with m-sized worklists after an overflow.
int run_cc_sized(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o, hcc_forest* f,
                        hcc_metrics* mx) {
  int r = run_cc(c, g, o, f, mx);
  if (r == kRerun) {
    r = run_cc(c, g, o, f, mx);
    if (mx) mx->wl_reruns = 1;
    if (r == kRerun) r = fail(HCC_ECUDA, "worklist capacity exceeded");
  }
  return r;
}

int run_cc(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o,
                  hcc_forest* f, hcc_metrics* mx) {
  if (int r = graph_ready(g)) return r;
  if (!g->shards.empty())
    return fail(HCC_EINVAL, "sharded graph: run it on its multi-device context");
  const hcc_opts defaults = {HCC_ALGO_BASELINE_MJ, 0, 0, 0, 0, nullptr, nullptr};
  if (!o) o = &defaults;
  if (o->algo < HCC_ALGO_BASELINE || o->algo > HCC_ALGO_ADAPTIVE)
    return fail(HCC_EINVAL, "unknown algorithm");
  const u64 n = g->n, m = g->m;
  if (f && f->n != n)
    return fail(HCC_EINVAL, "forest size does not match the graph");
  if (f && f->ctx && f->dev != c->dev)
    return fail(HCC_EINVAL, "forest lives on another device");

  hcc_metrics out{};
  out.n = n;
  out.m = m;
  c->last_recs.clear();

  // segments (engines.hpp:243-247 and partition_edges 43-62)
  u64 requested = 1;
  bool geo_plan = false;
  if (o->algo == HCC_ALGO_ADAPTIVE) {
    requested = o->segments;
    if (requested == 0) {
      hcc_graph_stats st;
      if (int r = hcc_graph_compute_stats(c, g, &st)) return r;
      requested = hcc_choose_segment_count(&st);
    }
  } else if (o->algo == HCC_ALGO_BASELINE_MJ &&
             !(o->flags & HCC_FLAG_FULL_PASSES)) {
    requested = o->first_pass_segments;
    if (requested == 0) geo_plan = true;
  }
  if (requested < 1) requested = 1;
  u64 nseg = std::max<u64>(1, std::min(requested, std::max<u64>(m, 1)));
  std::vector<u64> bounds;
  bool adapt = false;
  u32 adapt_shift = kAdaptShift;
  u64 adapt_first = 0;
  u32 adapt_growth = kAdaptGrowth;
  if (geo_plan) {
    const char* pe = std::getenv("HCC_PLAN");
    int sh = 0;
    if (!pe || std::strncmp(pe, "adapt", 5) == 0) {
      // device-side adaptive plan: launches are unrolled up to the number a
      // x4-growth schedule can need; ranges past the end are empty no-ops
      adapt = true;
      int slots = kAdaptSlots;
      if (pe) {
        int sl = 0;
        const int got = std::sscanf(pe, "adapt:%d:%d", &sh, &sl);
        if (got >= 1 && sh >= 0 && sh < 40) adapt_shift = (u32)sh;
        if (got == 2 && sl >= 1 && sl <= (int)kMaxUnrolledSegments) slots = sl;
      }
      // at most `slots` launches; the device gives the last one every
      // remaining edge (k_step_adapt)
      // first segment: m/128, optionally at least n >> nshift edges.
      // Forming lasts a number of edges proportional to n (the giant
      // emerges near n/2), so sparse graphs (m = 4n) would want the
      // n-relative floor for the forming slots to finish before the last
      // slot takes the rest (see kAdaptNShift).
      u32 nshift = kAdaptNShift;
      if (const char* e2 = std::getenv("HCC_PLAN_NSHIFT")) nshift = (u32)std::atoi(e2);
      const u64 nfloor = nshift && nshift < 64 ? (n >> nshift) : 0;
      u64 first = std::min<u64>(std::max<u64>(std::max<u64>(1, m >> adapt_shift), nfloor),
                                std::max<u64>(m, 1));
      adapt_first = first;
      u64 len = first, covered = first;
      nseg = 1;
      u32 growth = kAdaptGrowth;
      if (const char* e2 = std::getenv("HCC_ADAPT_GROWTH")) growth = (u32)std::max(2, std::atoi(e2));
      adapt_growth = growth;
      while (covered < m && nseg < (u64)slots) {
        len = std::min<u64>(len * growth, m - covered);
        covered += len;
        ++nseg;
      }
      // the static bounds only size the launch of each slot (small vs
      // streaming hook kernel); the device decides the real ranges
      bounds.assign(nseg + 1, 0);
      u64 b = 0, l = first;
      for (u64 i = 0; i < nseg; ++i) {
        bounds[i] = b;
        b = std::min<u64>(m, b + l);
        l *= growth;
      }
      bounds[nseg] = m;
      if (nseg >= 2) bounds[nseg - 1] = std::min(bounds[nseg - 1], m);
    } else {
      bounds = geometric_bounds(m);
      nseg = bounds.size() - 1;
    }
  } else if (nseg <= kMaxUnrolledSegments) {
    bounds = uniform_bounds(m, nseg);
  }
  out.s = nseg;
  out.segments_clamped = requested > m && m > 0;

  if (n == 0) {  // nothing to launch (test_engines.cpp:124)
    if (mx) *mx = out;
    return HCC_OK;
  }

  HCC_GUARD_BEGIN
  u32* pi;
  if (f) {
    pi = f->d_pi;
  } else {
    ensure_pi(c, n);
    pi = c->scratch_pi;
  }
  const bool uses_wl =
      o->algo == HCC_ALGO_BASELINE_MJ && !(o->flags & HCC_FLAG_FULL_PASSES);
  if (uses_wl && o->max_threads != 0) ensure_wl(c, m);  // exact block appends
  // atomic / adaptive on the streaming CAS hook (HCC_CAS_STREAM=0: the
  // scalar k_cas_hook + k_compress of the one-thread reference schedule)
  bool cas_stream = (o->algo == HCC_ALGO_ADAPTIVE || o->algo == HCC_ALGO_ATOMIC) &&
                    o->max_threads == 0 && n >= (1ull << 16);
  if (const char* e = std::getenv("HCC_CAS_STREAM")) cas_stream = cas_stream && std::atoi(e) != 0;
  // The worklist engine's star bitmap from n = 2^20 (HCC_S0B_MIN_LOG2):
  // below, its compress and sampling steps cost more than the lookups save
  // (RMAT-16 0.120 -> 0.101 ms without it, RMAT-18 0.19 -> 0.17, grid 512^2
  // 0.20 -> 0.13; RMAT-20 and ER 2^20 still gain from it).  The adaptive
  // chain always keeps it.
  u32 s0b_min_log2 = kS0bMinLog2;
  if (const char* e = std::getenv("HCC_S0B_MIN_LOG2")) s0b_min_log2 = (u32)std::atoi(e);
  bool s0b = ((uses_wl && s0b_min_log2 < 64 && n >= (1ull << s0b_min_log2)) || cas_stream) &&
             o->max_threads == 0 && n >= (1ull << 16);
  if (const char* e = std::getenv("HCC_S0B")) s0b = s0b && std::atoi(e) != 0;

  Plan P;
  P.algo = o->algo;
  P.full_passes = (o->flags & HCC_FLAG_FULL_PASSES) != 0;
  P.n = n;
  P.m = m;
  P.edges = g->d_edges;
  P.pi = pi;
  P.wl0 = uses_wl ? c->wl[0] : nullptr;
  P.wl1 = uses_wl ? c->wl[1] : nullptr;
  P.nseg = nseg;
  P.bounds = bounds;
  P.s0b = s0b && (!bounds.empty() || cas_stream);
  P.cas_stream = cas_stream && P.s0b;
  P.adapt = adapt;
  P.adapt_shift = adapt_shift;
  P.adapt_first = adapt_first;
  P.hook_events = (o->flags & HCC_FLAG_HOOK_EVENTS) != 0;
  if (const char* e = std::getenv("HCC_HOOK_SMALL")) P.small_slots = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_HOOK_CAS")) P.cas_mode = std::atoi(e);
  if (const char* e = std::getenv("HCC_DYN")) P.dyn = std::atoi(e) != 0;
  P.wide_compress = false;  // measured: no gain at n = 2^28 (33.89 vs 33.81 ms)
  if (const char* e = std::getenv("HCC_COMP_WIDE")) P.wide_compress = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_SUMD")) P.sumd = std::atoi(e);
  P.forming_pct = std::getenv("HCC_FORMING_PCT") ? (u32)std::atoi(std::getenv("HCC_FORMING_PCT"))
                                                  : kAdaptFormingPct;
  P.forming_pct = (P.forming_pct & 0xffu) |
                  (adapt_growth != kAdaptGrowth ? (adapt_growth & 0xffu) << 8 : 0u);
  if (P.s0b) {
    ensure_s0b(c, (n + 31) / 32);
  }
  if (P.s0b && (uses_wl || cas_stream)) {
    // star-0 summary: the smallest group (2^shift bitmap words per bit)
    // whose table fits the hook's shared-memory budget; groups larger than
    // a compress block's 64 words are not built
    const u64 nwords = (n + 31) / 32;
    u32 sh = 0;
    while (((nwords + (1ull << sh) - 1) >> sh) > (u64)kS0fMaxBytes * 8) ++sh;
    // (one bit per 16 words or more, n > 2^27: the steady slot's coverage
    // vote never picks the summary there, and building it cost RMAT-28's
    // compresses 0.13 ms of block barriers)
    bool sum_ok = sh <= kSumMaxShift;
    if (const char* e = std::getenv("HCC_S0F")) sum_ok = sum_ok && std::atoi(e) != 0;
    // one bit per 16 vertices while that table fits (HCC_SUM_HALF=0: per word)
    // (not for the adaptive engine's 31 short segment hooks, whose L1 the
    // 132 KB table costs more: RMAT-24 2.81 vs 2.66 ms)
    bool half = HCC_SUM_HALF && (n + 15) / 16 <= (u64)kSumHalfMaxBytes * 8 && !cas_stream;
    if (const char* e = std::getenv("HCC_SUM_HALF")) half = half && std::atoi(e) != 0;
    if (sum_ok) {
      P.sum = true;
      P.sum_shift = half ? kSumHalfShift : sh;
      P.sum_words = half ? (u32)(((n + 15) / 16 + 31) / 32)
                         : (u32)std::min<u64>((((nwords + (1ull << sh) - 1) >> sh) + 31) / 32,
                                              kS0fMaxBytes / 4);
      ensure_s0f(c, P.sum_words);
    }
  }
  // (HCC_SUM_VOTE=1: round 1's device vote between k_hook_sum and the
  // plain hook on word coverage, instead of the k_hook_sumd choice)
  P.sum_vote = false;
  if (const char* e = std::getenv("HCC_SUM_VOTE")) P.sum_vote = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_WL_SUMD")) P.wl_sumd = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_FOLD_PICK")) P.fold_pick = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_SUMD_ANY")) P.sumd_any = std::atoi(e) != 0;
  // pi beyond L2: the compress prefetches one residency wave (6 blocks per
  // SM) ahead (RMAT-28's compresses 1.94 -> 1.89 ms in total)
  P.comp_pf = n >= (1ull << 26) ? (u32)c->sms * 6u : 0u;
  if (const char* e = std::getenv("HCC_COMP_PF")) P.comp_pf = (u32)std::atoi(e);
  P.comp16 = HCC_COMP16 != 0;
  // (not when pi exceeds L2: RMAT-28's steady slot then ran 27.5 -> 28.7 ms
  // after two-sided middle slots, 2-shard ranks 11.6 -> 12.1 ms)
  P.hook_both = n < (1ull << 26);
  if (const char* e = std::getenv("HCC_HOOK_BOTH")) P.hook_both = std::atoi(e) != 0;
  if (const char* e = std::getenv("HCC_COMP16")) P.comp16 = std::atoi(e) != 0;
  {
    const char* w = std::getenv("HCC_WALK");
    P.walk = w ? std::atoi(w) : kDefaultWalk;
    const char* wl = std::getenv("HCC_WALK_LAST");
    P.walk_last = wl ? std::atoi(wl) : (w ? P.walk : kDefaultWalkLast);
  }
  if (o->max_threads == 0) {
    P.block_hook = kHookCta;
    P.grid_hook = (unsigned)(c->sms * c->occ_hook);
    P.grid_cas = (unsigned)(c->sms * c->occ_hook_cas);
    P.block_vert = kVertThreads;
    // k_compress / k_init_pi take four vertices per thread.  The grid covers
    // n exactly: blocks start in ascending order and a new block starts as
    // soon as any finishes, so the compress front stays ascending even when
    // some chases are long (a persistent grid-stride loop lets fast blocks
    // overtake stalled ancestors: grid 4096^2 compress went 0.5 -> 28 ms).
    P.grid_vert = grid_for((n + 3) / 4, kVertThreads, 0x7fffffffull);
  } else {
    u64 t = o->max_threads;
    unsigned blk = (unsigned)std::min<u64>(t, 256);
    if (blk >= 32) blk &= ~31u;
    unsigned grd = (unsigned)std::max<u64>(1, std::min<u64>(t / blk, 1u << 20));
    P.block_hook = P.block_vert = blk;
    P.grid_hook = P.grid_vert = grd;
  }
  if (uses_wl && o->max_threads == 0) {
    // streaming hooks (unrolled topology slots, worklist passes) append in
    // per-warp chunks and pad every warp's last chunk of a launch with
    // no-op records: room for all launches appending to one list (the
    // unrolled slots; the looped-segment path keeps exact block appends)
    P.chunked = true;
    const u64 warps = std::max<u64>(
        std::max<u64>((u64)P.grid_hook * (P.block_hook / 32),
                      (u64)c->sms * c->occ_hook_sum * (kHookSumCta / 32)),
        std::max<u64>(std::max<u64>((u64)P.grid_cas * (kHookCasCta / 32),
                                    (u64)c->sms * c->occ_hook_sum_cas * (kHookCasCta / 32)),
                      (u64)c->sms * c->occ_hook_sumd * (kHookSumdCta / 32)));
    const u64 launches = (P.nseg <= kMaxUnrolledSegments ? P.nseg : 0) + 2;
    // Records: every store of the topology slots plus deferred walks, all
    // slots into one list.  Stores link distinct roots up to benign races,
    // so ~n at most (grid 4096^2: 16.7 M of 33.5 M edges; RMAT-24: 9.1 M of
    // 268 M).  max(m/8, 2n) keeps RMAT-28 at 2 x 4.3 GB instead of 2 x 34
    // GB; an overflow is caught on the device (err bit 4) and the run is
    // repeated with m-sized lists (wl_full).  HCC_WL_DIV overrides the 8.
    u64 div = 8;
    if (const char* e = std::getenv("HCC_WL_DIV")) div = std::max<u64>(1, std::strtoull(e, nullptr, 10));
    const u64 recs_cap = c->wl_full ? m : std::min<u64>(m, std::max<u64>(m / div, div > 8 ? 0 : 2 * n));
    ensure_wl(c, recs_cap + launches * warps * kWlChunk);
    P.wl0 = c->wl[0];
    P.wl1 = c->wl[1];
  }

  const bool observer = o->observer != nullptr;
  // HCC_LAUNCH=eager: launch every kernel directly (host-driven loops) so a
  // profiler that cannot see inside conditional graphs (ncu) lists them.
  const char* launch_env = std::getenv("HCC_LAUNCH");
  const bool eager_env = launch_env && std::strcmp(launch_env, "eager") == 0;
  const bool graph_mode = !observer && !eager_env &&
                          !(o->flags & (HCC_FLAG_HOST_LOOP | HCC_FLAG_NO_GRAPH));
  out.used_device_loop = graph_mode ? 1 : 0;

  // HCC_APW=1 (experiment): persisting L2 access-policy window over the star
  // bitmap on the launch stream (applies to eager launches)
  if (const char* e = std::getenv("HCC_APW")) {
    if (std::atoi(e) && P.s0b) {
      const size_t bytes = (size_t)((n + 31) / 32) * 4;
      HCC_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
      cudaStreamAttrValue v = {};
      v.accessPolicyWindow.base_ptr = c->s0b;
      v.accessPolicyWindow.num_bytes = bytes;
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      HCC_CUDA(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v));
    }
  }
  Seq q;
  q.c = c;
  q.graph_mode = graph_mode;
  q.streams.push_back(c->stream);
  if (observer) {
    hcc_forest view;
    view.ctx = c;
    view.dev = c->dev;
    view.n = n;
    view.d_pi = pi;
    q.on_phase = [&, view](int phase) mutable {
      HCC_CUDA(cudaStreamSynchronize(c->stream));
      o->observer(o->observer_user, phase, &view);
    };
  }

  GraphKey key;
  key.algo = o->algo;
  key.edges = g->d_edges;
  key.pi = pi;
  key.wl0 = P.wl0;
  key.wl1 = P.wl1;
  key.s0b = c->s0b;
  key.s0f = c->s0f;
  key.wl_cap = c->wl_cap;
  key.n = n;
  key.m = m;
  key.nseg = nseg;
  key.max_threads = o->max_threads;
  key.flags = o->flags;
  key.walk = P.walk;
  key.s0b_on = P.s0b;
  key.sum = P.sum;
  key.plan = key.plan * 7 + (P.small_slots ? 1 : 0);
  key.plan = key.plan * 131 + (u64)P.walk_last;
  key.plan = key.plan * 5 + (u64)P.cas_mode;
  key.plan = key.plan * 3 + (P.cas_stream ? 1 : 0);
  key.plan = key.plan * 3 + (P.dyn ? 1 : 0);
  key.plan = key.plan * 3 + (P.wide_compress ? 1 : 0);
  key.plan = key.plan * 3 + (u64)P.sumd;
  key.plan = key.plan * 3 + (P.sum_vote ? 1 : 0);
  key.plan = key.plan * 3 + (P.wl_sumd ? 1 : 0);
  key.plan = key.plan * 3 + (P.fold_pick ? 1 : 0);
  key.plan = key.plan * 3 + (P.sumd_any ? 1 : 0);
  key.plan = key.plan * 1000003ull + P.comp_pf;
  key.plan = key.plan * 3 + (P.comp16 ? 1 : 0);
  key.plan = key.plan * 3 + (P.hook_both ? 1 : 0);
  key.plan = key.plan * 1000003ull + P.sum_words * 64ull + P.sum_shift;
  key.plan = key.plan * 31 + (P.adapt ? 1000 + P.adapt_shift + 100000ull * P.forming_pct : 0);
  key.plan = key.plan * 1000003ull + P.adapt_first;
  for (u64 x : P.bounds) key.plan = key.plan * 1000003ull + x;

  if (graph_mode) {
    if (!(c->exec && c->key == key) && c->alt_exec && c->alt_key == key) {
      std::swap(c->exec, c->alt_exec);
      std::swap(c->key, c->alt_key);
      std::swap(c->exec_seg_ev, c->alt_seg_ev);
      std::swap(c->exec_slot_kernel, c->alt_slot_kernel);
      std::swap(c->exec_wl_kernel, c->alt_wl_kernel);
    }
    if (!(c->exec && c->key == key)) {
      // keep the current executable graph as the alternate
      if (c->alt_exec) cudaGraphExecDestroy(c->alt_exec);
      c->alt_exec = c->exec;
      c->alt_key = c->key;
      c->alt_seg_ev = c->exec_seg_ev;
      c->alt_slot_kernel = c->exec_slot_kernel;
      c->alt_wl_kernel = c->exec_wl_kernel;
      c->exec = nullptr;
      c->key = GraphKey{};
      cudaGraph_t graph = nullptr;
      HCC_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
      try {
        enqueue_run(c, P, q);
      } catch (...) {
        // end the open captures innermost first (loop bodies capture into
        // conditional-node graphs on streams[1..depth]), then the root
        cudaGraph_t tmp = nullptr;
        for (int d = q.depth; d >= 1; --d) {
          tmp = nullptr;
          cudaStreamEndCapture(q.streams[d], &tmp);
        }
        tmp = nullptr;
        cudaStreamEndCapture(c->stream, &tmp);
        if (tmp) cudaGraphDestroy(tmp);
        cudaGetLastError();
        for (size_t i = 1; i < q.streams.size(); ++i)
          cudaStreamDestroy(q.streams[i]);
        throw;
      }
      HCC_CUDA(cudaStreamEndCapture(c->stream, &graph));
      cudaError_t ie = cudaGraphInstantiate(&c->exec, graph, 0);
      cudaGraphDestroy(graph);
      for (size_t i = 1; i < q.streams.size(); ++i)
        cudaStreamDestroy(q.streams[i]);
      q.streams.resize(1);
      if (ie != cudaSuccess) {
        c->exec = nullptr;
        return fail(HCC_ECUDA, std::string("cudaGraphInstantiate: ") +
                                   cudaGetErrorString(ie));
      }
      c->key = key;
      c->exec_seg_ev = c->seg_ev_used;
      c->exec_slot_kernel = c->slot_kernel;
      c->exec_wl_kernel = c->wl_kernel;
    }
    c->seg_ev_used = c->exec_seg_ev;
    c->slot_kernel = c->exec_slot_kernel;
    c->wl_kernel = c->exec_wl_kernel;
    HCC_CUDA(cudaEventRecord(c->ev0, c->stream));
    HCC_CUDA(cudaGraphLaunch(c->exec, c->stream));
    HCC_CUDA(cudaEventRecord(c->ev1, c->stream));
  } else {
    HCC_CUDA(cudaEventRecord(c->ev0, c->stream));
    enqueue_run(c, P, q);
    HCC_CUDA(cudaEventRecord(c->ev1, c->stream));
  }
  HCC_CUDA(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  HCC_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  out.total_ms = ms;

  // roots = components (count_components, engines.hpp:77-82), untimed
  k_count_roots<<<grid_for(n, 256, (u64)c->sms * 16), 256, 0, c->stream>>>(
      pi, n, c->d_ctrl);
  if (o->flags & HCC_FLAG_CHECK_STAR)
    k_is_star<<<grid_for(n, 256, (u64)c->sms * 16), 256, 0, c->stream>>>(
        pi, n, &c->d_ctrl->flag);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(c->h_ctrl, c->d_ctrl, sizeof(DevCtrl),
                           cudaMemcpyDeviceToHost, c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  const bool chain = P.cas_stream && P.nseg <= kMaxUnrolledSegments && P.bounds.size() == P.nseg + 1;
  const u64 nrec = chain ? std::min<u64>(nseg, kMaxRecs) : std::min<u64>(c->h_ctrl->rec, kMaxRecs);
  if (nrec)
    HCC_CUDA(cudaMemcpyAsync(c->h_recs, c->d_recs, nrec * sizeof(DevRec),
                             cudaMemcpyDeviceToHost, c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  const DevCtrl& hc = *c->h_ctrl;
  out.components = hc.components;
  out.passes = chain ? nseg : hc.passes;
  out.edges_processed = hc.edges_processed;
  out.records = nrec;
  c->last_recs.resize(nrec);
  for (u64 i = 0; i < nrec; ++i) {
    const DevRec& r = c->h_recs[i];
    hcc_segment_rec sr{};
    if (r.hook_t1 > r.hook_t0 && r.hook_t0 != ~0ull)
      sr.hook_ms = (double)(r.hook_t1 - r.hook_t0) * 1e-6;
    if (r.comp_t1 > r.comp_t0 && r.comp_t0 != ~0ull)
      sr.compress_ms = (double)(r.comp_t1 - r.comp_t0) * 1e-6;
    sr.counters.hook_traversal_steps = r.traversal;
    sr.counters.cas_failures = r.cas_fail;
    sr.counters.jump_steps = r.jump_total();
    sr.edges_in = r.edges_in;
    sr.edges_out = r.edges_out;
    auto rel = [&](u64 t) {
      return (t == 0 || t == ~0ull || hc.t_start == 0) ? -1.0
                                                       : (double)(int64_t)(t - hc.t_start) * 1e-6;
    };
    const bool hk = r.hook_t1 > r.hook_t0 && r.hook_t0 != ~0ull;
    const bool cp = r.comp_t1 > r.comp_t0 && r.comp_t0 != ~0ull;
    sr.hook_start_ms = hk ? rel(r.hook_t0) : -1.0;
    sr.hook_end_ms = hk ? rel(r.hook_t1) : -1.0;
    sr.compress_start_ms = cp ? rel(r.comp_t0) : -1.0;
    sr.compress_end_ms = cp ? rel(r.comp_t1) : -1.0;
    if (P.adapt || !P.bounds.empty()) {
      if (i < c->slot_kernel.size()) {
        sr.hook_kernel = c->slot_kernel[i];
        if (sr.hook_kernel == HCC_HOOK_KERNEL_SUM && !hc.use_sum)
          sr.hook_kernel = HCC_HOOK_KERNEL_STREAM;  // the vote chose the plain hook
        if (r.kind) sr.hook_kernel = (int32_t)r.kind;  // what actually ran
      } else if (o->algo == HCC_ALGO_BASELINE_MJ && !P.full_passes) {
        sr.hook_kernel = c->wl_kernel;
      }
    }
    sr.hook_event_ms = -1.0;
    if (i < c->seg_ev_used) {
      float ems = 0.f;
      if (cudaEventElapsedTime(&ems, c->seg_ev[2 * i], c->seg_ev[2 * i + 1]) ==
          cudaSuccess)
        sr.hook_event_ms = ems;
      else
        cudaGetLastError();
    }
    c->last_recs[i] = sr;
    out.hook_ms += sr.hook_ms;
    out.compress_ms += sr.compress_ms;
    out.counters.hook_traversal_steps += r.traversal;
    out.counters.cas_failures += r.cas_fail;
    out.counters.jump_steps += r.jump_total();
  }
  out.star0_bitmap = P.s0b ? 1 : 0;
  {
    // kernels launched by the run (loop iterations from the device records)
    const u64 iters = nrec;
    u64 k = 1;  // k_start
    if (o->algo == HCC_ALGO_BASELINE_MJ && !P.full_passes && !P.bounds.empty()) {
      const u64 wl = nrec > nseg ? nrec - nseg : 0;
      k += 3 * nseg + 3 * wl;  // hook+compress+step per slot and per wl pass
      for (u64 sgi = 1; sgi < nseg && nseg <= kMaxUnrolledSegments; ++sgi) {
        const bool pick = P.s0b && P.adapt && sgi + 1 < nseg;
        k += pick && !(P.fold_pick && !slot_small(P, sgi)) ? 1 : 0;  // k_star_pick
        // gated pairs (two launches, one exits at entry)
        k += remainder_slot(P, sgi) || (P.sum && P.adapt && P.sum_vote && sum_slot(P, sgi)) ? 1 : 0;
      }
      // gated worklist pairs
      if (P.sum && P.adapt && ((P.sum_vote) || (P.sumd == 1 && P.wl_sumd && P.cas_mode >= 1)))
        k += wl;
    } else {
      k += (chain ? 2 : P.cas_stream ? 4 : 3) * iters;  // hook/(pick)/compress(or jump)/step
    }
    out.kernels = k;
  }
  out.wl_capacity = uses_wl ? c->wl_cap : 0;
  if (o->algo == HCC_ALGO_BASELINE_MJ && !P.full_passes)
    out.outer_iterations = 1 + (nrec > nseg ? nrec - nseg : 0);
  else if (o->algo == HCC_ALGO_ADAPTIVE || o->algo == HCC_ALGO_ATOMIC)
    out.outer_iterations = nseg;  // engines.hpp:288
  else
    out.outer_iterations = nrec;
  if (mx) *mx = out;
  if (hc.err & 2u)
    return fail(HCC_ECUDA, "device loop exceeded its step cap (runaway loop)");
  if (hc.err & 4u) {
    if (!c->wl_full) {
      c->wl_full = true;  // hcc_cc repeats the run with m-sized worklists
      return kRerun;
    }
    return fail(HCC_ECUDA, "worklist capacity exceeded");
  }
  if ((o->flags & HCC_FLAG_CHECK_STAR) && hc.flag)
    return fail(HCC_ENOTSTAR, "extract_labels: forest is not star-shaped");
  return HCC_OK;
  HCC_GUARD_END
}

}  // namespace host
}  // namespace hcc

// ===========================================================================
// C-ABI

extern "C" {

int hcc_abi_version(void) { return HCC_ABI_VERSION; }

const char* hcc_last_error(void) { return g_err.c_str(); }

int hcc_device_count(void) { return usable_devices(); }

int hcc_create(int device, hcc_ctx** out) {
  if (!out) return fail(HCC_EINVAL, "null output");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(HCC_ENODEV, "no CUDA device visible (libhookcc_cuda has no "
                            "CPU fallback)");
  }
  if (device < 0 || device >= count)
    return fail(HCC_EINVAL, "device index out of range");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(HCC_ECUDA, "cudaGetDeviceProperties failed");
  if (prop.major != 10)
    return fail(HCC_ENODEV, std::string("device ") + prop.name +
                                " is not sm_100 (this build targets sm_100a)");
  hcc_ctx* c = new hcc_ctx;
  HCC_GUARD_BEGIN
  c->dev = device;
  HCC_CUDA(cudaSetDevice(device));
  c->sms = prop.multiProcessorCount;
  HCC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  HCC_CUDA(cudaMalloc(&c->d_ctrl, sizeof(DevCtrl)));
  HCC_CUDA(cudaMalloc(&c->d_recs, sizeof(DevRec) * kMaxRecs));
  HCC_CUDA(cudaMallocHost(&c->h_ctrl, sizeof(DevCtrl)));
  HCC_CUDA(cudaMallocHost(&c->h_recs, sizeof(DevRec) * kMaxRecs));
  HCC_CUDA(cudaMemset(c->d_ctrl, 0, sizeof(DevCtrl)));
  HCC_CUDA(cudaEventCreate(&c->ev0));
  HCC_CUDA(cudaEventCreate(&c->ev1));
  int occ = 0;
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook, kHookCta, 0));
  c->occ_hook = std::max(occ, 1);
  // the summary hook stages the star-0 summary and its slow-path queues
  HCC_CUDA(cudaFuncSetAttribute(k_hook_sum, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kHookSmemMax));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_sum_cas, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kHookSmemMax));
  const int sumd_smem = (int)sum_region_words(kSumTableMaxBytes / 4) * 4;
  HCC_CUDA(cudaFuncSetAttribute(k_hook_sumd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_seg_cas_sumd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_cas_sumd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_cas_sumd_sh, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_seg_cas_sumd_sh, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_sumd_sh, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                sumd_smem));
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook_cas_sumd, kHookCasCta,
                                                          sumd_smem));
  c->occ_hook_cas_sumd = std::max(occ, 1);
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook_sumd, kHookSumdCta,
                                                          sumd_smem));
  c->occ_hook_sumd = std::max(occ, 1);
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook_sum, kHookSumCta,
                                                          kHookSmemMax));
  c->occ_hook_sum = std::max(occ, 1);
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook_sum_cas, kHookCasCta,
                                                          kHookSmemMax));
  c->occ_hook_sum_cas = std::max(occ, 1);
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hook_cas, kHookCasCta, 0));
  c->occ_hook_cas = std::max(occ, 1);
#if HCC_SMALL_CARVE >= 0
  HCC_CUDA(cudaFuncSetAttribute(k_hook_small, cudaFuncAttributePreferredSharedMemoryCarveout,
                                HCC_SMALL_CARVE));
#endif
#if HCC_HOOK_CARVE >= 0
  HCC_CUDA(cudaFuncSetAttribute(k_hook, cudaFuncAttributePreferredSharedMemoryCarveout,
                                HCC_HOOK_CARVE));
  HCC_CUDA(cudaFuncSetAttribute(k_hook_cas, cudaFuncAttributePreferredSharedMemoryCarveout,
                                HCC_HOOK_CARVE));
#endif
#if HCC_COMP_CARVE >= 0
  HCC_CUDA(cudaFuncSetAttribute(k_compress_s0b, cudaFuncAttributePreferredSharedMemoryCarveout,
                                HCC_COMP_CARVE));
#endif
  HCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_compress,
                                                          kVertThreads, 0));
  c->occ_vert = std::max(occ, 1);
  *out = c;
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    hcc_destroy(c);
    return f.code;
  }
}

int hcc_destroy(hcc_ctx* c) {
  if (!c) return HCC_OK;
  peer_release(c);
  for (size_t r = 0; r < c->merge.size(); ++r) {
    MergeShard& ms = c->merge[r];
    if (r < c->subs.size()) cudaSetDevice(c->subs[r]->dev);
    if (ms.forest) hcc_forest_free(ms.forest);
    cudaFree(ms.bits);
    cudaFree(ms.pairs);
    cudaFree(ms.cnt);
    cudaFree(ms.tab);
    for (cudaEvent_t ev : {ms.ev_exp, ms.ev_t0, ms.ev_m0, ms.ev_t1})
      if (ev) cudaEventDestroy(ev);
  }
  for (hcc_ctx* sc : c->subs) hcc_destroy(sc);
  cudaSetDevice(c->dev);
  drop_exec(c);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_ctrl);
  cudaFree(c->d_recs);
  cudaFreeHost(c->h_ctrl);
  cudaFreeHost(c->h_recs);
  cudaFree(c->scratch_pi);
  cudaFree(c->wl[0]);
  cudaFree(c->wl[1]);
  cudaFree(c->s0b_base);
  cudaFree(c->s0f);
  for (cudaEvent_t ev : c->seg_ev) cudaEventDestroy(ev);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->check_stream) {
    cudaStreamSynchronize(c->check_stream);
    cudaStreamDestroy(c->check_stream);
  }
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  for (cudaEvent_t ev : c->chunk_ev) cudaEventDestroy(ev);
  delete c;
  return HCC_OK;
}

int hcc_ctx_segments(hcc_ctx* c, hcc_segment_rec* out, uint64_t cap,
                     uint64_t* count) {
  if (!c) return fail(HCC_EINVAL, "null context");
  u64 k = std::min<u64>(cap, c->last_recs.size());
  if (out)
    for (u64 i = 0; i < k; ++i) out[i] = c->last_recs[i];
  if (count) *count = c->last_recs.size();
  return HCC_OK;
}

int hcc_ctx_sm_count(hcc_ctx* c, int* out) {
  if (!c || !out) return fail(HCC_EINVAL, "null argument");
  *out = c->sms;
  return HCC_OK;
}

// ---- graphs ----------------------------------------------------------------

int hcc_graph_from_edges_u64(hcc_ctx* c, const uint64_t* uv, uint64_t m,
                             uint64_t n, hcc_graph** out) {
  if (!out) return fail(HCC_EINVAL, "null output");
  *out = nullptr;
  if (int r = ctx_enter(c)) return r;
  if (n > kMaxN)
    return fail(HCC_EINVAL, "vertex count >= 2^32 is not supported by the "
                            "device forest (u32 ids)");
  if (m > 0 && !uv) return fail(HCC_EINVAL, "null edge buffer");
  if (!c->subs.empty()) return multi_from_edges(c, uv, true, m, n, out);
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = m;
  u64* stage = nullptr;
  u32* d_err = nullptr;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&g->d_edges, std::max<u64>(m, 2) * sizeof(uint2)));
  HCC_CUDA(cudaMalloc(&d_err, sizeof(u32)));
  HCC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(u32), c->stream));
  const u64 chunk = std::min<u64>(m, 1ull << 26);  // 1 GiB of u64 pairs
  if (m > 0) HCC_CUDA(cudaMalloc(&stage, chunk * 2 * sizeof(u64)));
  for (u64 off = 0; off < m; off += chunk) {
    u64 k = std::min(chunk, m - off);
    HCC_CUDA(cudaMemcpyAsync(stage, uv + 2 * off, k * 2 * sizeof(u64),
                             cudaMemcpyHostToDevice, c->stream));
    k_narrow_u64<<<grid_for(k, 256, 65536), 256, 0, c->stream>>>(
        stage, g->d_edges + off, k, n, d_err);
    HCC_CUDA(cudaGetLastError());
  }
  u32 err = 0;
  HCC_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(stage);
  cudaFree(d_err);
  stage = nullptr;
  d_err = nullptr;
  if (err) {
    hcc_graph_free(g);
    return fail(HCC_ERANGE, "edge endpoint out of range");
  }
  *out = g;
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    cudaFree(stage);
    cudaFree(d_err);
    hcc_graph_free(g);
    return f.code;
  }
}

int hcc_graph_from_edges_u32(hcc_ctx* c, const uint32_t* uv, uint64_t m,
                             uint64_t n, hcc_graph** out) {
  if (!out) return fail(HCC_EINVAL, "null output");
  *out = nullptr;
  if (int r = ctx_enter(c)) return r;
  if (n > kMaxN) return fail(HCC_EINVAL, "vertex count >= 2^32");
  if (m > 0 && !uv) return fail(HCC_EINVAL, "null edge buffer");
  if (!c->subs.empty()) return multi_from_edges(c, uv, false, m, n, out);
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = m;
  u32* d_err = nullptr;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&g->d_edges, std::max<u64>(m, 2) * sizeof(uint2)));
  HCC_CUDA(cudaMalloc(&d_err, sizeof(u32)));
  HCC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(u32), c->stream));
  if (m > 0) {
    HCC_CUDA(cudaMemcpyAsync(g->d_edges, uv, m * sizeof(uint2),
                             cudaMemcpyHostToDevice, c->stream));
    k_check_u32<<<grid_for(m, 256, 65536), 256, 0, c->stream>>>(g->d_edges, m,
                                                                n, d_err);
    HCC_CUDA(cudaGetLastError());
  }
  u32 err = 0;
  HCC_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(d_err);
  d_err = nullptr;
  if (err) {
    hcc_graph_free(g);
    return fail(HCC_ERANGE, "edge endpoint out of range");
  }
  *out = g;
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    cudaFree(d_err);
    hcc_graph_free(g);
    return f.code;
  }
}

int hcc_graph_upload_async(hcc_ctx* c, hcc_graph* g, const uint32_t* uv, uint64_t first,
                           uint64_t count) {
  if (!g || (count && !uv)) return fail(HCC_EINVAL, "null argument");
  if (first > g->m || count > g->m - first)
    return fail(HCC_EINVAL, "range out of bounds");
  if (int r = ctx_enter(c)) return r;
  if (!g->shards.empty()) return multi_range_io(c, g, const_cast<uint32_t*>(uv), first, count, 0);
  if (int r = graph_ready(g)) return r;  // one upload in flight per graph
  HCC_GUARD_BEGIN
  if (!c->copy_stream) {
    HCC_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    HCC_CUDA(cudaStreamCreateWithFlags(&c->check_stream, cudaStreamNonBlocking));
  }
  if (!g->up_ev) {
    HCC_CUDA(cudaEventCreateWithFlags(&g->up_ev, cudaEventDisableTiming));
    HCC_CUDA(cudaMalloc(&g->d_err, sizeof(u32)));
    HCC_CUDA(cudaMallocHost(&g->h_err, sizeof(u32)));
  }
  // the graph's previous readers ran on the context stream
  if (!c->order_ev) HCC_CUDA(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
  HCC_CUDA(cudaEventRecord(c->order_ev, c->stream));
  HCC_CUDA(cudaStreamWaitEvent(c->copy_stream, c->order_ev, 0));
  HCC_CUDA(cudaMemsetAsync(g->d_err, 0, sizeof(u32), c->copy_stream));
  // chunked copy; each chunk's endpoint check runs on the check stream while
  // the next chunk copies, so only the last check follows the transfer
  constexpr u64 kChunk = 16ull << 20;  // edges (128 MiB)
  const u64 nch = (count + kChunk - 1) / kChunk;
  while (c->chunk_ev.size() < nch) {
    cudaEvent_t ev;
    HCC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->chunk_ev.push_back(ev);
  }
  HCC_CUDA(cudaEventRecord(c->order_ev, c->copy_stream));
  HCC_CUDA(cudaStreamWaitEvent(c->check_stream, c->order_ev, 0));
  for (u64 k = 0; k < nch; ++k) {
    const u64 b = first + k * kChunk, cnt = std::min<u64>(kChunk, count - k * kChunk);
    HCC_CUDA(cudaMemcpyAsync(g->d_edges + b, uv + 2 * (b - first), cnt * sizeof(uint2),
                             cudaMemcpyHostToDevice, c->copy_stream));
    HCC_CUDA(cudaEventRecord(c->chunk_ev[k], c->copy_stream));
    HCC_CUDA(cudaStreamWaitEvent(c->check_stream, c->chunk_ev[k], 0));
    k_check_u32<<<grid_for(cnt, 256, 65536), 256, 0, c->check_stream>>>(g->d_edges + b, cnt,
                                                                        g->n, g->d_err);
    HCC_CUDA(cudaGetLastError());
  }
  HCC_CUDA(cudaMemcpyAsync(g->h_err, g->d_err, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->check_stream));
  HCC_CUDA(cudaEventRecord(g->up_ev, c->check_stream));
  g->pending = true;
  g->has_stats = false;
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_graph_assign_edges_u32(hcc_ctx* c, hcc_graph* g, const uint32_t* uv,
                               uint64_t first, uint64_t count) {
  // the chunked upload with overlapped endpoint checks, then wait for it
  if (int r = hcc_graph_upload_async(c, g, uv, first, count)) return r;
  return graph_ready(g);
}

int hcc_graph_from_csr(hcc_ctx* c, const uint64_t* row_ptr, const uint32_t* col,
                       uint64_t n, hcc_graph** out) {
  if (!out) return fail(HCC_EINVAL, "null output");
  *out = nullptr;
  if (int r = ctx_enter(c)) return r;
  if (n > kMaxN) return fail(HCC_EINVAL, "vertex count >= 2^32");
  if (!row_ptr) return fail(HCC_EINVAL, "null row_ptr");
  if (row_ptr[0] != 0) return fail(HCC_EINVAL, "row_ptr[0] must be 0");
  for (u64 i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i])
      return fail(HCC_EINVAL, "row_ptr must be non-decreasing");
  const u64 m = row_ptr[n];
  if (m > 0 && !col) return fail(HCC_EINVAL, "null col");
  if (!c->subs.empty()) {
    // sharded: expand on the host (row order), then partition the edge list
    std::vector<u32> uv;
    try {
      uv.resize(2 * m);
    } catch (const std::bad_alloc&) {
      return fail(HCC_ENOMEM, "host allocation failed");
    }
    for (u64 u = 0; u < n; ++u)
      for (u64 j = row_ptr[u]; j < row_ptr[u + 1]; ++j) {
        if (col[j] >= n) return fail(HCC_ERANGE, "column index out of range");
        uv[2 * j] = (u32)u;
        uv[2 * j + 1] = col[j];
      }
    return multi_from_edges(c, uv.data(), false, m, n, out);
  }
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = m;
  u64* d_rp = nullptr;
  u32 *d_col = nullptr, *d_err = nullptr;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&g->d_edges, std::max<u64>(m, 2) * sizeof(uint2)));
  HCC_CUDA(cudaMalloc(&d_err, sizeof(u32)));
  HCC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(u32), c->stream));
  if (m > 0) {
    HCC_CUDA(cudaMalloc(&d_rp, (n + 1) * sizeof(u64)));
    HCC_CUDA(cudaMalloc(&d_col, m * sizeof(u32)));
    HCC_CUDA(cudaMemcpyAsync(d_rp, row_ptr, (n + 1) * sizeof(u64),
                             cudaMemcpyHostToDevice, c->stream));
    HCC_CUDA(cudaMemcpyAsync(d_col, col, m * sizeof(u32),
                             cudaMemcpyHostToDevice, c->stream));
    k_csr_expand<<<grid_for(m, 256, 65536), 256, 0, c->stream>>>(
        d_rp, d_col, n, g->d_edges, m, d_err);
    HCC_CUDA(cudaGetLastError());
  }
  u32 err = 0;
  HCC_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(d_rp);
  cudaFree(d_col);
  cudaFree(d_err);
  d_rp = nullptr;
  d_col = nullptr;
  d_err = nullptr;
  if (err) {
    hcc_graph_free(g);
    return fail(HCC_ERANGE, "column index out of range");
  }
  *out = g;
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    cudaFree(d_rp);
    cudaFree(d_col);
    cudaFree(d_err);
    hcc_graph_free(g);
    return f.code;
  }
}

static int generate_impl(hcc_ctx* c, const char* spec_c, uint64_t default_seed,
                         bool ranged, u64 first, u64 count, hcc_graph** out) {
  if (!out || !spec_c) return fail(HCC_EINVAL, "null argument");
  *out = nullptr;
  if (int r = ctx_enter(c)) return r;
  std::string spec(spec_c);
  size_t colon = spec.find(':');
  if (colon == std::string::npos)
    return fail(HCC_EINVAL, "generator spec needs the form kind:params");
  std::string kind = spec.substr(0, colon), params = spec.substr(colon + 1);
  u64 n = 0, m = 0, rows = 0, cols = 0, seed = default_seed, scale = 0, ef = 0;
  double a = 0.57, b = 0.19, cc = 0.19, d = 0.05;
  std::string v;
  if (kind == "grid") {
    size_t x = params.find('x');
    if (x == std::string::npos || !parse_u64(params.substr(0, x), &rows) ||
        !parse_u64(params.substr(x + 1), &cols))
      return fail(HCC_EINVAL, "grid spec needs RxC");
    if (rows == 0 || cols == 0) return fail(HCC_EINVAL, "grid: zero vertices");
    n = rows * cols;
    m = rows * (cols - 1) + (rows - 1) * cols;
  } else if (kind == "rmatx") {
    if (!spec_get(params, "scale", &v) || !parse_u64(v, &scale) ||
        !spec_get(params, "ef", &v) || !parse_u64(v, &ef))
      return fail(HCC_EINVAL, "rmatx spec needs scale= and ef=");
    if (scale > 32) return fail(HCC_EINVAL, "rmatx: scale > 32");
    if (spec_get(params, "seed", &v) && !parse_u64(v, &seed))
      return fail(HCC_EINVAL, "rmatx: bad seed");
    if (spec_get(params, "a", &v)) a = atof(v.c_str());
    if (spec_get(params, "b", &v)) b = atof(v.c_str());
    if (spec_get(params, "c", &v)) cc = atof(v.c_str());
    if (spec_get(params, "d", &v)) d = atof(v.c_str());
    if (std::fabs(a + b + cc + d - 1.0) > 1e-9)
      return fail(HCC_EINVAL, "rmat: quadrant probabilities must sum to 1");
    n = 1ull << scale;
    m = ef * n;
  } else if (kind == "erx") {
    if (!spec_get(params, "n", &v) || !parse_u64(v, &n) ||
        !spec_get(params, "m", &v) || !parse_u64(v, &m))
      return fail(HCC_EINVAL, "erx spec needs n= and m=");
    if (spec_get(params, "seed", &v) && !parse_u64(v, &seed))
      return fail(HCC_EINVAL, "erx: bad seed");
    if (n == 0) return fail(HCC_EINVAL, "erdos_renyi: zero vertices");
  } else {
    return fail(HCC_EINVAL, "unknown device generator kind `" + kind + "`");
  }
  if (n > kMaxN + 1 || (kind != "rmatx" && n > kMaxN))
    return fail(HCC_EINVAL, "vertex count >= 2^32");
  if (kind == "rmatx" && n > kMaxN)
    return fail(HCC_EINVAL, "rmatx: scale 32 needs 2^32 vertices (> u32)");
  if (ranged) {
    if (first > m || count > m - first)
      return fail(HCC_EINVAL, "generator range out of bounds");
  } else {
    first = 0;
    count = m;
  }
  if (!c->subs.empty()) return multi_generate(c, spec_c, default_seed, n, first, count, out);
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = count;
  g->first = first;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&g->d_edges, std::max<u64>(count, 2) * sizeof(uint2)));
  if (count > 0) {
    unsigned grid = grid_for(count, 256, (u64)c->sms * 32);
    if (kind == "grid") {
      k_gen_grid<<<grid, 256, 0, c->stream>>>(g->d_edges, rows, cols, first, count);
    } else if (kind == "rmatx") {
      k_gen_rmatx<<<grid, 256, 0, c->stream>>>(
          g->d_edges, first, count, (u32)scale, seed, prob_threshold(a),
          prob_threshold(a + b), prob_threshold(a + b + cc));
    } else {
      k_gen_erx<<<grid, 256, 0, c->stream>>>(g->d_edges, first, count, n, seed);
    }
    HCC_CUDA(cudaGetLastError());
  }
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  *out = g;
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    hcc_graph_free(g);
    return f.code;
  }
}

int hcc_graph_generate(hcc_ctx* c, const char* spec, uint64_t default_seed,
                       hcc_graph** out) {
  return generate_impl(c, spec, default_seed, false, 0, 0, out);
}

int hcc_graph_generate_range(hcc_ctx* c, const char* spec, uint64_t default_seed,
                             uint64_t first, uint64_t count, hcc_graph** out) {
  return generate_impl(c, spec, default_seed, true, first, count, out);
}

int hcc_graph_info(const hcc_graph* g, uint64_t* n, uint64_t* m) {
  if (!g) return fail(HCC_EINVAL, "null graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  return HCC_OK;
}

int hcc_graph_download_u32(hcc_ctx* c, const hcc_graph* g, uint32_t* uv,
                           uint64_t first, uint64_t count) {
  if (int r = graph_ready(g)) return r;
  if (!g || (count && !uv)) return fail(HCC_EINVAL, "null argument");
  if (first > g->m || count > g->m - first)
    return fail(HCC_EINVAL, "range out of bounds");
  if (int r = ctx_enter(c)) return r;
  if (!g->shards.empty())
    return multi_range_io(c, const_cast<hcc_graph*>(g), uv, first, count, 2);
  HCC_GUARD_BEGIN
  if (count)
    HCC_CUDA(cudaMemcpy(uv, g->d_edges + first, count * sizeof(uint2),
                        cudaMemcpyDeviceToHost));
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_graph_checksum(hcc_ctx* c, const hcc_graph* g, uint64_t* out) {
  if (int r = graph_ready(g)) return r;
  if (!g || !out) return fail(HCC_EINVAL, "null argument");
  if (int r = ctx_enter(c)) return r;
  if (!g->shards.empty()) {  // position-keyed terms: the shard sums add up
    u64 sum = 0;
    for (size_t r = 0; r < g->shards.size(); ++r) {
      uint64_t x = 0;
      if (int e = hcc_graph_checksum(c->subs[r], g->shards[r], &x)) return e;
      sum += x;
    }
    *out = sum;
    return HCC_OK;
  }
  u64* d = nullptr;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&d, sizeof(u64)));
  HCC_CUDA(cudaMemsetAsync(d, 0, sizeof(u64), c->stream));
  if (g->m)
    k_checksum<<<grid_for(g->m, 256, (u64)c->sms * 16), 256, 0, c->stream>>>(
        g->d_edges, g->m, g->first, d);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(out, d, sizeof(u64), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(d);
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    cudaFree(d);
    return f.code;
  }
}

int hcc_graph_compute_stats(hcc_ctx* c, const hcc_graph* g_c,
                            hcc_graph_stats* out) {
  if (int r = graph_ready(g_c)) return r;
  if (!g_c || !out) return fail(HCC_EINVAL, "null argument");
  if (int r = ctx_enter(c)) return r;
  hcc_graph* g = const_cast<hcc_graph*>(g_c);
  if (!g->shards.empty() && !g->has_stats) {
    if (int r = multi_stats(c, g, &g->stats)) return r;
    g->has_stats = true;
  }
  HCC_GUARD_BEGIN
  if (!g->has_stats)
    if (int r = compute_stats_dev(c, g)) return r;
  *out = g->stats;
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_graph_free(hcc_graph* g) {
  if (!g) return HCC_OK;
  if (!g->shards.empty()) {
    for (hcc_graph* sh : g->shards) hcc_graph_free(sh);
    delete g;
    return HCC_OK;
  }
  if (g->ctx) {
    cudaSetDevice(g->ctx->dev);
    // the cached executable graph may reference these edges
    if (g->ctx->key.edges == g->d_edges || g->ctx->alt_key.edges == g->d_edges)
      drop_exec(g->ctx);
    if (g->pending) cudaEventSynchronize(g->up_ev);
  }
  if (g->up_ev) cudaEventDestroy(g->up_ev);
  cudaFree(g->d_err);
  cudaFreeHost(g->h_err);
  cudaFree(g->d_edges);
  delete g;
  return HCC_OK;
}

uint64_t hcc_choose_segment_count(const hcc_graph_stats* st) {
  // engines.hpp:35-41
  if (!st || st->n == 0) return 1;
  u64 s = (u64)std::floor(st->avg_degree + 0.5);
  if (s < 1) s = 1;
  if (st->m_stored > 0 && s > st->m_stored) s = st->m_stored;
  return s;
}

// ---- the CC engine -----------------------------------------------------------

int hcc_cc(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o, hcc_forest* f,
           uint32_t* labels_out, hcc_metrics* mx) {
  if (!g) return fail(HCC_EINVAL, "null graph");
  if (int r = ctx_enter(c)) return r;
  if (!c->subs.empty()) return multi_cc(c, g, o, f, labels_out, nullptr, mx);
  if (int r = run_cc_sized(c, g, o, f, mx)) return r;
  if (labels_out && g->n) {
    const u32* pi = f ? f->d_pi : c->scratch_pi;
    HCC_GUARD_BEGIN
    HCC_CUDA(cudaMemcpy(labels_out, pi, g->n * sizeof(u32),
                        cudaMemcpyDeviceToHost));
    HCC_GUARD_END
  }
  return HCC_OK;
}

int hcc_cc_u64(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o,
               hcc_forest* f, uint64_t* labels_out, hcc_metrics* mx) {
  if (!g) return fail(HCC_EINVAL, "null graph");
  if (int r = ctx_enter(c)) return r;
  if (!c->subs.empty()) return multi_cc(c, g, o, f, nullptr, labels_out, mx);
  if (int r = run_cc_sized(c, g, o, f, mx)) return r;
  if (labels_out && g->n) {
    const u32* pi = f ? f->d_pi : c->scratch_pi;
    HCC_GUARD_BEGIN
    // widen in place from the top: copy u32 labels into the upper half of
    // the caller's u64 buffer, then expand forward-safely from the end.
    uint32_t* tmp = reinterpret_cast<uint32_t*>(labels_out) + g->n;
    HCC_CUDA(cudaMemcpy(tmp, pi, g->n * sizeof(u32), cudaMemcpyDeviceToHost));
    for (u64 i = 0; i < g->n; ++i) labels_out[i] = tmp[i];
    HCC_GUARD_END
  }
  return HCC_OK;
}

// ---- forests -----------------------------------------------------------------

int hcc_forest_create(hcc_ctx* c, uint64_t n, hcc_forest** out) {
  if (!out) return fail(HCC_EINVAL, "null output");
  *out = nullptr;
  if (int r = ctx_enter(c)) return r;
  if (n > kMaxN) return fail(HCC_EINVAL, "forest size >= 2^32");
  hcc_forest* f = new hcc_forest;
  f->ctx = c;
  f->dev = c->dev;
  f->n = n;
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaMalloc(&f->d_pi, std::max<u64>(n, 4) * sizeof(u32)));
  *out = f;
  int r = hcc_forest_reset(f);
  if (r) {
    hcc_forest_free(f);
    *out = nullptr;
  }
  return r;
  }
  catch (const CudaFail& fl) {
    hcc_forest_free(f);
    return fl.code;
  }
}

int hcc_forest_free(hcc_forest* f) {
  if (!f) return HCC_OK;
  cudaSetDevice(f->dev);
  if (f->ctx && (f->ctx->key.pi == f->d_pi || f->ctx->alt_key.pi == f->d_pi))
    drop_exec(f->ctx);
  cudaFree(f->d_pi);
  delete f;
  return HCC_OK;
}

int hcc_forest_size(const hcc_forest* f, uint64_t* n) {
  if (!f || !n) return fail(HCC_EINVAL, "null argument");
  *n = f->n;
  return HCC_OK;
}

int hcc_forest_reset(hcc_forest* f) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaSetDevice(f->dev));
  if (f->n) {
    k_init_pi<<<grid_for(f->n, 256, 65536), 256, 0, cudaStreamPerThread>>>(
        f->d_pi, f->n, nullptr);
    HCC_CUDA(cudaGetLastError());
  }
  HCC_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_forest_download_u32(hcc_forest* f, uint32_t* out) {
  if (!f || (f->n && !out)) return fail(HCC_EINVAL, "null argument");
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaSetDevice(f->dev));
  if (f->n)
    HCC_CUDA(cudaMemcpyAsync(out, f->d_pi, f->n * sizeof(u32),
                             cudaMemcpyDeviceToHost, cudaStreamPerThread));
  HCC_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_forest_download_u64(hcc_forest* f, uint64_t* out) {
  if (!f || (f->n && !out)) return fail(HCC_EINVAL, "null argument");
  std::vector<u32> tmp(f->n);
  if (int r = hcc_forest_download_u32(f, tmp.data())) return r;
  for (u64 i = 0; i < f->n; ++i) out[i] = tmp[i];
  return HCC_OK;
}

int hcc_forest_upload_u64(hcc_forest* f, const uint64_t* in) {
  if (!f || (f->n && !in)) return fail(HCC_EINVAL, "null argument");
  std::vector<u32> tmp(f->n);
  for (u64 i = 0; i < f->n; ++i) {
    if (in[i] >= f->n) return fail(HCC_EINVAL, "parent out of range");
    tmp[i] = (u32)in[i];
  }
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaSetDevice(f->dev));
  if (f->n)
    HCC_CUDA(cudaMemcpyAsync(f->d_pi, tmp.data(), f->n * sizeof(u32),
                             cudaMemcpyHostToDevice, cudaStreamPerThread));
  HCC_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  return HCC_OK;
  HCC_GUARD_END
}

static int elem(hcc_forest* f, int op, u64 a, u64 b, u64 cc, u64 res[3]) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaSetDevice(f->dev));
  u64* h = nullptr;
  u64* d = thread_scratch(f->dev, &h);
  k_elem<<<1, 1, 0, cudaStreamPerThread>>>(f->d_pi, op, a, b, cc, d);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(h, d, 3 * sizeof(u64), cudaMemcpyDeviceToHost,
                           cudaStreamPerThread));
  HCC_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  res[0] = h[0];
  res[1] = h[1];
  res[2] = h[2];
  return HCC_OK;
  HCC_GUARD_END
}

#define HCC_CHECK_V(x)                                                      \
  if ((x) >= f->n) return fail(HCC_EINVAL, "vertex out of range")

int hcc_forest_load(hcc_forest* f, uint64_t v, uint64_t* out) {
  if (!f || !out) return fail(HCC_EINVAL, "null argument");
  HCC_CHECK_V(v);
  u64 r[3];
  if (int e = elem(f, kOpLoad, v, 0, 0, r)) return e;
  *out = r[0];
  return HCC_OK;
}

int hcc_forest_store(hcc_forest* f, uint64_t v, uint64_t p) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_CHECK_V(v);
  HCC_CHECK_V(p);
  u64 r[3];
  return elem(f, kOpStore, v, p, 0, r);
}

int hcc_forest_cas(hcc_forest* f, uint64_t v, uint64_t* expected,
                   uint64_t desired, int* ok) {
  if (!f || !expected || !ok) return fail(HCC_EINVAL, "null argument");
  HCC_CHECK_V(v);
  HCC_CHECK_V(desired);
  u64 r[3];
  if (*expected > kMaxN) {  // can never match a u32 slot
    if (int e = hcc_forest_load(f, v, expected)) return e;
    *ok = 0;
    return HCC_OK;
  }
  if (int e = elem(f, kOpCas, v, *expected, desired, r)) return e;
  *ok = (int)r[1];
  if (!r[1]) *expected = r[0];
  return HCC_OK;
}

int hcc_forest_hook(hcc_forest* f, uint64_t u, uint64_t v, int* changed) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_CHECK_V(u);
  HCC_CHECK_V(v);
  u64 r[3];
  if (int e = elem(f, kOpHook, u, v, 0, r)) return e;
  if (changed) *changed = (int)r[0];
  return HCC_OK;
}

int hcc_forest_jump(hcc_forest* f, uint64_t v, int* changed) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_CHECK_V(v);
  u64 r[3];
  if (int e = elem(f, kOpJump, v, 0, 0, r)) return e;
  if (changed) *changed = (int)r[0];
  return HCC_OK;
}

int hcc_forest_atomic_hook(hcc_forest* f, uint64_t u, uint64_t v,
                           hcc_counters* c) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_CHECK_V(u);
  HCC_CHECK_V(v);
  u64 r[3];
  if (int e = elem(f, kOpAtomicHook, u, v, 0, r)) return e;
  if (c) {
    c->hook_traversal_steps += r[0];
    c->cas_failures += r[1];
  }
  return HCC_OK;
}

int hcc_forest_multi_jump(hcc_forest* f, uint64_t v, hcc_counters* c) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  HCC_CHECK_V(v);
  u64 r[3];
  if (int e = elem(f, kOpMultiJump, v, 0, 0, r)) return e;
  if (c) c->jump_steps += r[2];
  return HCC_OK;
}

int hcc_forest_multi_jump_range(hcc_forest* f, uint64_t begin, uint64_t end,
                                int descending, hcc_counters* c) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  if (begin > end || end > f->n) return fail(HCC_EINVAL, "bad range");
  if (begin == end) return HCC_OK;
  u64 r[3];
  if (int e = elem(f, kOpMultiJumpRange, begin, end, descending ? 1 : 0, r))
    return e;
  if (c) c->jump_steps += r[2];
  return HCC_OK;
}

static int forest_flag_kernel(hcc_forest* f, bool star, int* out) {
  if (!f || !out) return fail(HCC_EINVAL, "null argument");
  if (f->n == 0) {
    *out = 1;
    return HCC_OK;
  }
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaSetDevice(f->dev));
  u64* h = nullptr;
  u64* d = thread_scratch(f->dev, &h);  // per-thread device scratch word
  u32* flag = reinterpret_cast<u32*>(d + 3);
  HCC_CUDA(cudaMemsetAsync(flag, 0, sizeof(u32), cudaStreamPerThread));
  const unsigned grid = grid_for(f->n, 256, 4096);
  if (star)
    k_is_star<<<grid, 256, 0, cudaStreamPerThread>>>(f->d_pi, f->n, flag);
  else
    k_check_bound<<<grid, 256, 0, cudaStreamPerThread>>>(f->d_pi, f->n, flag);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(h + 3, flag, sizeof(u32), cudaMemcpyDeviceToHost,
                           cudaStreamPerThread));
  HCC_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  *out = (*reinterpret_cast<u32*>(h + 3)) ? 0 : 1;
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_forest_is_star(hcc_forest* f, int* out) {
  return forest_flag_kernel(f, true, out);
}

int hcc_forest_check_bound(hcc_forest* f, int* ok) {
  return forest_flag_kernel(f, false, ok);
}

// ---- device-side verification ----------------------------------------------------

int hcc_forest_verify(hcc_ctx* c, const hcc_graph* g, hcc_forest* f,
                      uint64_t* bad_edges, uint64_t* bad_vertices) {
  if (int r = graph_ready(g)) return r;
  if (!g || !f || !bad_edges || !bad_vertices) return fail(HCC_EINVAL, "null argument");
  if (f->n != g->n) return fail(HCC_EINVAL, "forest size does not match the graph");
  if (int r = ctx_enter(c)) return r;
  if (!g->shards.empty()) {
    // each shard's edges on its own device against f (peer reads); the
    // vertex check once
    u64 be = 0, bv = 0;
    for (size_t r = 0; r < g->shards.size(); ++r) {
      uint64_t e = 0, v = 0;
      if (int st = hcc_forest_verify(c->subs[r], g->shards[r], f, &e, &v)) return st;
      be += e;
      if (r == 0) bv = v;
    }
    *bad_edges = be;
    *bad_vertices = bv;
    return HCC_OK;
  }
  HCC_GUARD_BEGIN
  u64* d = reinterpret_cast<u64*>(&c->d_ctrl->wl_count[0]);  // two u64 scratch slots
  HCC_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(u64), c->stream));
  if (g->m)
    k_verify_edges<<<grid_for(g->m, 256, (u64)c->sms * 32), 256, 0, c->stream>>>(
        g->d_edges, g->m, f->d_pi, d);
  if (f->n)
    k_verify_canonical<<<grid_for(f->n, 256, (u64)c->sms * 32), 256, 0, c->stream>>>(
        f->d_pi, f->n, d + 1);
  HCC_CUDA(cudaGetLastError());
  u64 h[2] = {0, 0};
  HCC_CUDA(cudaMemcpyAsync(h, d, 2 * sizeof(u64), cudaMemcpyDeviceToHost, c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  *bad_edges = h[0];
  *bad_vertices = h[1];
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_labels_compare(hcc_ctx* c, const uint32_t* a, const uint32_t* b, uint64_t n,
                       int* partition_equal, int* exact) {
  if (!partition_equal || !exact || (n && (!a || !b))) return fail(HCC_EINVAL, "null argument");
  if (int r = ctx_enter(c)) return r;
  if (n == 0) {
    *partition_equal = *exact = 1;
    return HCC_OK;
  }
  u32 *da = nullptr, *db = nullptr;
  u64 *k1 = nullptr, *k2 = nullptr, *cnt = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&] {
    cudaFree(da); cudaFree(db); cudaFree(k1); cudaFree(k2); cudaFree(cnt); cudaFree(tmp);
  };
  try {
    cudaStream_t s = c->stream;
    HCC_CUDA(cudaMalloc(&da, n * sizeof(u32)));
    HCC_CUDA(cudaMalloc(&db, n * sizeof(u32)));
    HCC_CUDA(cudaMalloc(&k1, n * sizeof(u64)));
    HCC_CUDA(cudaMalloc(&k2, n * sizeof(u64)));
    HCC_CUDA(cudaMalloc(&cnt, 4 * sizeof(u64)));
    HCC_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(u64), s));
    HCC_CUDA(cudaMemcpyAsync(da, a, n * sizeof(u32), cudaMemcpyHostToDevice, s));
    HCC_CUDA(cudaMemcpyAsync(db, b, n * sizeof(u32), cudaMemcpyHostToDevice, s));
    const unsigned grid = grid_for(n, 256, (u64)c->sms * 32);
    size_t tb = 0;
    // pairs (a, b): distinct pairs and distinct a
    k_pair_keys<<<grid, 256, 0, s>>>(da, db, n, k1, cnt + 3);
    HCC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, k1, k2, (int64_t)n, 0, 64, s));
    HCC_CUDA(cudaMalloc(&tmp, tb));
    HCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, k1, k2, (int64_t)n, 0, 64, s));
    k_count_distinct<<<grid, 256, 0, s>>>(k2, n, 0, cnt + 0);
    k_count_distinct<<<grid, 256, 0, s>>>(k2, n, 32, cnt + 1);
    // pairs (b, a): distinct b
    k_pair_keys<<<grid, 256, 0, s>>>(db, da, n, k1, cnt + 3);
    HCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, k1, k2, (int64_t)n, 0, 64, s));
    k_count_distinct<<<grid, 256, 0, s>>>(k2, n, 32, cnt + 2);
    HCC_CUDA(cudaGetLastError());
    u64 h[4];
    HCC_CUDA(cudaMemcpyAsync(h, cnt, 4 * sizeof(u64), cudaMemcpyDeviceToHost, s));
    HCC_CUDA(cudaStreamSynchronize(s));
    *partition_equal = h[0] == h[1] && h[0] == h[2];
    *exact = h[3] == 0;
  } catch (const CudaFail& f) {
    cleanup();
    return f.code;
  }
  cleanup();
  return HCC_OK;
}

// ---- multi-GPU merge primitives (kernels in hcc_multi.cu) ---------------------

int hcc_forest_export(hcc_ctx* c, hcc_forest* f, uint32_t* dev_bits,
                      uint32_t* dev_pairs, uint64_t cap, uint64_t* count) {
  if (!f || !count || (!dev_bits && f->n)) return fail(HCC_EINVAL, "null argument");
  if (cap && !dev_pairs) return fail(HCC_EINVAL, "null pair buffer");
  if (int r = ctx_enter(c)) return r;
  HCC_GUARD_BEGIN
  u64* d_cnt = reinterpret_cast<u64*>(&c->d_ctrl->wl_count[0]);
  HCC_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(u64), c->stream));
  if (f->n) {
    const u64 nwords = (f->n + 31) / 32;
    k_export<<<grid_for(nwords * 32, 256, (u64)c->sms * 32), 256, 0, c->stream>>>(
        f->d_pi, f->n, dev_bits, reinterpret_cast<uint2*>(dev_pairs), cap, d_cnt);
    HCC_CUDA(cudaGetLastError());
  }
  u64 h = 0;
  HCC_CUDA(cudaMemcpyAsync(&h, d_cnt, sizeof(u64), cudaMemcpyDeviceToHost, c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  *count = h;
  return HCC_OK;
  HCC_GUARD_END
}

// Re-hook remote relations into a star forest with the worklist engine
// (host-driven passes: the merge needs only a few).
int hcc_rehook(hcc_ctx* c, hcc_forest* f, const uint32_t* dev_bits_or,
               const uint32_t* dev_pairs, uint64_t count, hcc_metrics* mx) {
  const uint64_t nwords = f ? (f->n + 31) / 32 : 0;
  return hcc_rehook_rows(c, f, dev_bits_or, dev_bits_or ? 1 : 0, nwords, ~0ull, dev_pairs,
                         count, mx);
}

int hcc_rehook_rows(hcc_ctx* c, hcc_forest* f, const uint32_t* dev_bit_rows, uint64_t nrows,
                    uint64_t row_stride_words, uint64_t skip_row, const uint32_t* dev_pairs,
                    uint64_t count, hcc_metrics* mx) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  if (nrows && !dev_bit_rows) return fail(HCC_EINVAL, "null bitmap rows");
  if (nrows && row_stride_words < (f->n + 31) / 32)
    return fail(HCC_EINVAL, "bitmap row stride below ceil(n/32)");
  if (count && !dev_pairs) return fail(HCC_EINVAL, "null pair buffer");
  if (int r = ctx_enter(c)) return r;
  hcc_metrics out{};
  out.n = f->n;
  out.m = count;
  HCC_GUARD_BEGIN
  const u64 n = f->n;
  ensure_wl(c, count + n + 1);
  const Plan P = rehook_plan(c, f->d_pi, n);
  HCC_CUDA(cudaEventRecord(c->ev0, c->stream));
  k_begin<<<1, 1, 0, c->stream>>>(c->d_ctrl, c->d_recs, 1);
  u64* d_cnt = reinterpret_cast<u64*>(&c->d_ctrl->wl_count[0]);
  if (count) {
    HCC_CUDA(cudaMemcpyAsync(c->wl[0], dev_pairs, count * sizeof(uint2),
                             cudaMemcpyDeviceToDevice, c->stream));
    c->h_ctrl->wl_count[0] = count;
    HCC_CUDA(cudaMemcpyAsync(d_cnt, &c->h_ctrl->wl_count[0], sizeof(u64),
                             cudaMemcpyHostToDevice, c->stream));
  }
  if (nrows && n)
    k_decode_bits<<<grid_for((n + 31) / 32 * 32, 256, (u64)c->sms * 32), 256, 0,
                    c->stream>>>(dev_bit_rows, nrows, row_stride_words, skip_row, f->d_pi, n,
                                 c->wl[0], d_cnt);
  HCC_CUDA(cudaGetLastError());
  rehook_loop(c, P);
  HCC_CUDA(cudaEventRecord(c->ev1, c->stream));
  HCC_CUDA(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  HCC_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  HCC_CUDA(cudaMemcpy(c->h_ctrl, c->d_ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost));
  out.total_ms = ms;
  out.passes = c->h_ctrl->passes;
  out.outer_iterations = c->h_ctrl->passes;
  out.edges_processed = c->h_ctrl->edges_processed;
  out.kernels = 2 + 3 * c->h_ctrl->passes;
  if (mx) *mx = out;
  return HCC_OK;
  HCC_GUARD_END
}

}  // extern "C"
