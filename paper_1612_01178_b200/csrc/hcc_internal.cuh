// Internal declarations shared by the hookcc CUDA translation units.
//
// Device data layout:
//   edges  : uint2[m]      packed (u, v) u32 pairs, stored order preserved
//                          (reference Graph.edges, graph.hpp:24-31, 16 B/edge
//                          AoS u64 -> 8 B/edge here)
//   pi     : uint32[n]     parent forest (reference ParentForest slots,
//                          forest.hpp:62), pi(v) <= v always
//   wl[2]  : uint2[cap]    ping-pong worklists of (H, L) root pairs
//   ctrl   : DevCtrl       device-side loop state (counts, parity, flags)
//   recs   : DevRec[]      per-phase timing / counter records
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hookcc_c.h"

namespace hcc {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kMaxRecs = 4096;    // per-run phase records kept on device
#ifndef HCC_SMALL_CTA
#define HCC_SMALL_CTA 1024
#endif
constexpr int kHookThreads = HCC_SMALL_CTA;  // k_hook_small CTA (full grid)
#ifndef HCC_SMALL_EPT
#define HCC_SMALL_EPT 2
#endif
constexpr int kSmallEPT = HCC_SMALL_EPT;  // k_hook_small edges per thread
// Streaming hook CTA (k_hook): threads per CTA; its shared-memory star-0
// summary table holds at most HCC_S0F_MAX_BYTES.
#ifndef HCC_HOOK_CTA
#define HCC_HOOK_CTA 1024
#endif
#ifndef HCC_S0F_MAX_BYTES
#define HCC_S0F_MAX_BYTES 65536
#endif
constexpr int kHookCta = HCC_HOOK_CTA;
#ifndef HCC_HOOK_SUM_CTA
#define HCC_HOOK_SUM_CTA 1024
#endif
constexpr int kHookSumCta = HCC_HOOK_SUM_CTA;  // k_hook_sum (one CTA per SM)
// CAS-storing worklist hooks (k_hook_cas, k_hook_sum_cas): 768-thread CTAs
// give them 80 registers instead of 64 (at 1024 threads ptxas spilled
// 32 B / 12 B of stores per thread).
#ifndef HCC_HOOK_CAS_CTA
#define HCC_HOOK_CAS_CTA 768
#endif
constexpr int kHookCasCta = HCC_HOOK_CAS_CTA;
// Two-sided streaming hook (k_hook_both): CTA size and edges per thread
// (768 / 4: ER 2^24/2^28 1.877 -> 1.836 ms, RMAT-24 1.353 -> 1.345 against
// 768 / 8; 1024 / 8 spilled 160 B, 1024 / 4 measured no gain).
#ifndef HCC_BOTH_CTA
#define HCC_BOTH_CTA 768
#endif
#ifndef HCC_BOTH_EPT
#define HCC_BOTH_EPT 4
#endif
constexpr int kHookBothCta = HCC_BOTH_CTA;
// Summary-predicated streaming hook (k_hook_sumd).
#ifndef HCC_HOOK_SUMD_CTA
#define HCC_HOOK_SUMD_CTA 1024
#endif
constexpr int kHookSumdCta = HCC_HOOK_SUMD_CTA;
constexpr u32 kS0fMaxBytes = HCC_S0F_MAX_BYTES;
// Half-word summary (one bit per 16 vertices: RMAT-24's lookups are 76%
// covered instead of 63% at one bit per 32), used while its table fits
// kSumHalfMaxBytes (n <= 2^24).  Its shift is ~0u: consumers index bit
// x >> (5 + shift), and 5 + ~0u wraps to 4.
#ifndef HCC_SUM_HALF
#define HCC_SUM_HALF 1
#endif
constexpr u32 kSumHalfShift = ~0u;
// Coarsest summary built (2^shift bitmap words per bit).
#ifndef HCC_SUM_MAX_SHIFT
#define HCC_SUM_MAX_SHIFT 3
#endif
constexpr u32 kSumMaxShift = HCC_SUM_MAX_SHIFT;
constexpr u32 kSumHalfMaxBytes = 128u * 1024u;
// Largest staged table (shared-memory budgets of the summary hooks).
constexpr u32 kSumTableMaxBytes = kSumHalfMaxBytes > kS0fMaxBytes ? kSumHalfMaxBytes : kS0fMaxBytes;
// The shift the summary-predicated kernels compile in (their _sh builds take
// it at run time).
constexpr u32 kSumShiftFixed = HCC_SUM_HALF ? kSumHalfShift : 0u;
// Shared-memory words the staged summary of `w` words occupies (32-word rows
// padded to 33 words, sum_swz).
__host__ __device__ constexpr u32 sum_region_words(u32 w) { return ((w + 31) >> 5) * 33; }
constexpr int kHookSlow = 4;
// HookArgs.gate: k_hook_sum and k_hook are launched back to back for a
// voted slot and the one not chosen (DevCtrl.use_sum) exits at entry.
constexpr int kGateAlways = 0, kGateIfSum = 1, kGateIfPlain = 2;     // queued edges per lane per slow-path round
#ifndef HCC_WL_CHUNK
#define HCC_WL_CHUNK 256
#endif
constexpr u32 kWlChunk = HCC_WL_CHUNK;  // worklist records a warp reserves at once
#ifndef HCC_HOOK_EPT
#define HCC_HOOK_EPT 8
#endif
constexpr int kHookEPT = HCC_HOOK_EPT;  // edges per thread per tile (4 x uint4)
constexpr int kVertThreads = 256;
constexpr int kVertThreadsWide = 512;  // k_compress_s0b_w (n >= 2^26)

// One record per hook+compress phase pair (segment, outer iteration or
// worklist pass).  Times are %globaltimer nanoseconds (first block start,
// last block end).
// Compress jump counters are striped over kJumpStripes words (by block):
// tens of thousands of per-warp atomics on one address serialise in its L2
// slice.  The host sums the stripes.
#ifndef HCC_JUMP_STRIPES
#define HCC_JUMP_STRIPES 16
#endif
constexpr int kJumpStripes = HCC_JUMP_STRIPES;
struct DevRec {
  u64 hook_t0, hook_t1, comp_t0, comp_t1;
  u64 traversal, cas_fail, jump_steps;
  u64 edges_in, edges_out;
  u64 kind;          // HCC_HOOK_KERNEL_* of the hook that did this record's pass
  u64 jump_stripe[kJumpStripes];
  u64 jump_total() const {
    u64 t = jump_steps;
    for (int i = 0; i < kJumpStripes; ++i) t += jump_stripe[i];
    return t;
  }
};

struct DevCtrl {
  u64 wl_count[2];   // worklist fill counts
  u64 seg;           // current segment (segmented loops)
  u64 nseg;          // number of segments
  u64 passes;        // hook passes executed
  u64 edges_processed;
  u64 components;
  u32 parity;        // worklist index that is the NEXT hook input
  u32 rec;           // current record index
  u32 dirty;         // a hook in the current phase wrote pi
  u32 changed;       // baseline: some hook saw pi(u) != pi(v)
  u32 jchanged;      // baseline: some jump changed a slot
  u32 cond;          // last loop condition (host-loop mode reads it)
  u32 err;           // sticky device error bits
  u32 flag;          // scratch result flag (is_star / bound checks)
  u64 loop_steps;    // loop-step kernels executed (runaway guard)
  u64 seg_b, seg_e;  // adaptive topology plan: current segment range
  u64 t_start;       // globaltimer at k_start (span timeline origin)
  u32 use_sum;       // last summary vote (k_step_adapt): next hook uses k_hook_sum
  u32 star_hint;     // a vertex of the component the star bitmap tracks
  u32 star;          // its root at the last compress: bit v of the bitmap
                     // means pi(v) == star (k_compress_s0b)
  u32 use_bits;      // next plain hook looks the bitmap up (k_step_adapt)
  // unrolled segment chains without step kernels (the adaptive engine):
  // segment i's hook sets dirtyp[i & 1], its compress reads it and clears
  // the other slot for segment i + 1
  u32 dirtyp[2];
  u32 pick_count;    // blocks of a hook that finished (last one runs the pick)
  u64 merged_links;  // roots a multi-GPU merge linked to 0 in place
  u32 tile_ctr;      // next warp tile of a dynamically scheduled hook; every
                     // compress (and k_start) resets it for the next hook
};

// k_compress_s0b modes.
enum CompressMode : int {
  kCompressAlways = 0,
  kCompressIfDirty = 1,
};

// Device loops stop (and report HCC_ECUDA) after this many steps; the
// reference's own bound is 4*ceil(log2(n+2))+2 outer iterations
// (test_engines.cpp:179-187), so this only catches bugs.
constexpr u64 kMaxLoopSteps = 1ull << 22;

// Source of a hook phase.
enum HookMode : int {
  kSrcRange = 0,     // edges[b, e)
  kSrcSegment = 1,   // segment ctrl->seg of partition_edges(m, ctrl->nseg)
  kSrcWorklist = 2,  // wl[ctrl->parity][0, wl_count[parity])
  kSrcCtrlRange = 3, // edges[ctrl->seg_b, ctrl->seg_e) (adaptive plan)
};

// Adaptive topology plan: the first segment is m >> shift;
// while a segment stores for more than kAdaptFormingPct% of its edges (trees
// still forming) the next one is kAdaptGrowth times larger, otherwise the
// next segment takes every remaining edge.
constexpr u32 kAdaptGrowth = 4;
constexpr u32 kAdaptFormingPct = 20;

struct HookArgs {
  const uint2* edges;
  u64 m;
  u64 n;             // vertices (the in-kernel star pick)
  u64 b, e;
  int mode;
  int append;        // append (H, L) of every write to the next worklist
  int walk;          // max root-walk steps before a store (0 = Fig. 2 hook)
  const u32* s0b;    // star-0 bitmap (bit v = pi(v) == 0 after the last
                     // compress), or null
  const u32* s0f;    // star-0 summary: bit i = bitmap words
                     // [i << s0f_shift, (i + 1) << s0f_shift) are all ones;
                     // staged in shared memory by k_hook; or null
  u32 s0f_words;     // u32 words of s0f
  u32 s0f_shift;
  u64 wl_cap;        // records each worklist buffer holds
  int chunked;       // full-warp launch with per-warp chunked appends
                     // (padding records; the host sized the worklists)
  int gate;          // kGate*: run only if ctrl->use_sum says so
  int cas;           // launch the CAS-storing kernel (k_hook_cas /
                     // k_hook_sum_cas): links are not recorded
  u32* pi;
  uint2* wl0;
  uint2* wl1;
  DevCtrl* ctrl;
  DevRec* recs;
  int rec_idx;       // record of this launch (-1: ctrl->rec)
  int dslot;         // dirty flag: -1 ctrl->dirty, else ctrl->dirtyp[dslot]
  int pick;          // the hook's last block runs the star pick (no k_star_pick node)
  int dyn;           // warps take tiles from ctrl->tile_ctr (reset by the next
                     // compress) instead of a static round-robin
};

// Launch shape chosen on the host.
struct Launch {
  int grid_hook;     // persistent hook grid
  int block_hook;
  int grid_vert;     // vertex-parallel grid (0 = cover n)
  int block_vert;
  u64 max_threads;   // 0 = unlimited
};

// ---- kernels (hcc_kernels.cu) -------------------------------------------
__global__ void k_begin(DevCtrl* ctrl, DevRec* recs, u64 nseg);
__global__ void k_init_pi(u32* pi, u64 n, u32* bits);
__global__ void k_hook(HookArgs a);
__global__ void k_hook_small(HookArgs a);
__global__ void k_hook_sum(HookArgs a);
__global__ void k_hook_legacy(HookArgs a);
__global__ void k_hook_cas(HookArgs a);
__global__ void k_hook_both(HookArgs a);
__global__ void k_hook_sum_cas(HookArgs a);
__global__ void k_hook_seg_cas(HookArgs a);
__global__ void k_hook_sumd(HookArgs a);
__global__ void k_hook_sumd_sh(HookArgs a);
__global__ void k_hook_cas_sumd_sh(HookArgs a);
__global__ void k_hook_seg_cas_sumd(HookArgs a);
__global__ void k_hook_seg_cas_sumd_sh(HookArgs a);
__global__ void k_hook_cas_sumd(HookArgs a);
__global__ void k_star_pick(const u32* pi, u64 n, DevCtrl* ctrl);
__global__ void k_cas_hook(HookArgs a);
__global__ void k_compress(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                           int skip_if_clean);
__global__ void k_compress_s0b(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                               u32* bits, int skip_if_clean, u32* sum, u32 sum_words,
                               u32 sum_shift, int rec_idx, int dslot, u32 pf_blocks);
__global__ void k_compress_s0b16(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                                 u32* bits, int skip_if_clean, u32* sum, u32 sum_words,
                                 u32 sum_shift, int rec_idx, int dslot, u32 pf_blocks);
__global__ void k_compress_s0b_w(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                                 u32* bits, int skip_if_clean, u32* sum, u32 sum_words,
                                 u32 sum_shift, int rec_idx, int dslot, u32 pf_blocks);
__global__ void k_start(u32* pi, u64 n, u32* bits, DevCtrl* ctrl, DevRec* recs, u64 nseg,
                        u64 m, u64 plan_first, u32* sum, u32 sum_words);
__global__ void k_jump(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs);
__global__ void k_step_worklist(DevCtrl* ctrl, DevRec* recs,
                                cudaGraphConditionalHandle h, int use_cond);
__global__ void k_step_segment(DevCtrl* ctrl, DevRec* recs,
                               cudaGraphConditionalHandle h, int use_cond);
__global__ void k_step_adapt(DevCtrl* ctrl, DevRec* recs, u64 m, u32 forming_pct,
                             const u32* sum, u32 sum_words, const uint2* edges,
                             const u32* bits, const u32* rsum, u32 rshift, int rany);
__global__ void k_step_outer(DevCtrl* ctrl, DevRec* recs,
                             cudaGraphConditionalHandle h, int use_cond);
__global__ void k_step_jump(DevCtrl* ctrl, cudaGraphConditionalHandle h,
                            int use_cond);
__global__ void k_set_cond(cudaGraphConditionalHandle h, u32 value);
__global__ void k_count_roots(const u32* pi, u64 n, DevCtrl* ctrl);
__global__ void k_is_star(const u32* pi, u64 n, u32* flag);
__global__ void k_check_bound(const u32* pi, u64 n, u32* flag);

// Element kernels (single thread) for the ParentForest API.
enum ElemOp : int {
  kOpLoad = 0, kOpStore, kOpCas, kOpHook, kOpJump, kOpAtomicHook,
  kOpMultiJump, kOpMultiJumpRange
};
__global__ void k_elem(u32* pi, int op, u64 a, u64 b, u64 c, u64* res);

// Ingestion / generators (hcc_graph.cu).
__global__ void k_narrow_u64(const u64* uv, uint2* out, u64 m, u64 n,
                             u32* err);
__global__ void k_check_u32(const uint2* e, u64 m, u64 n, u32* err);
__global__ void k_csr_expand(const u64* row_ptr, const u32* col, u64 n,
                             uint2* out, u64 m, u32* err);
__global__ void k_gen_grid(uint2* out, u64 rows, u64 cols, u64 first, u64 count);
__global__ void k_gen_rmatx(uint2* out, u64 first, u64 count, u32 scale,
                            u64 seed, u32 ta, u32 tab, u32 tabc);
__global__ void k_gen_erx(uint2* out, u64 first, u64 count, u64 n, u64 seed);
__global__ void k_checksum(const uint2* e, u64 m, u64 base, u64* out);

// Verification (hcc_graph_kernels.cu).
__global__ void k_verify_edges(const uint2* e, u64 m, const u32* pi, u64* bad);
__global__ void k_verify_canonical(const u32* pi, u64 n, u64* bad);
__global__ void k_pair_keys(const u32* a, const u32* b, u64 n, u64* keys, u64* diff);
__global__ void k_count_distinct(const u64* k, u64 n, int shift, u64* out);

// Multi-GPU merge (hcc_multi.cu).
__global__ void k_export(const u32* pi, u64 n, u32* bits, uint2* pairs, u64 cap,
                         u64* count);
// Peer export buffers of a multi-device merge (device-resident table).
constexpr u32 kMaxShards = 64;
struct PeerTab {
  u32 npeers;
  const u32* bits[kMaxShards];    // export bitmap of rank r
  const uint2* pairs[kMaxShards]; // export pairs of rank r
  const u64* count[kMaxShards];   // pairs rank r produced (may exceed cap)
  u64 cap[kMaxShards];
};
__global__ void k_merge_gather(const PeerTab* tab, u32 self, u32* pi, u64 n, uint2* wl,
                               u64* count, u64 cap, u32* err, u32* dirty, u64* linked);
__global__ void k_decode_bits(const u32* rows, u64 nrows, u64 stride, u64 skip, const u32* pi,
                              u64 n, uint2* wl, u64* count);

}  // namespace hcc
