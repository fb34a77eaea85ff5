// Hook-Compress kernels for sm_100a.
//
// Reference semantics (all paths relative to /root/reference):
//   hook         proj/include/hookcc/forest.hpp:83-89   (paper Fig. 2)
//   jump         proj/include/hookcc/forest.hpp:93-99
//   atomic_hook  proj/include/hookcc/forest.hpp:107-122 (paper Fig. 3)
//   multi_jump   proj/include/hookcc/forest.hpp:127-136 (paper Fig. 3)
//   is_star      proj/include/hookcc/forest.hpp:140-146
//   loops        proj/include/hookcc/engines.hpp:123-291
//
// B200 design:
//   * The hook is the atomic-free Hook (Fig. 2) with Fig. 3's root walk and
//     a plain load in place of the CAS.  Edges stream as packed u32 pairs in
//     16-byte loads (8 per thread per tile, the next tile prefetched); the
//     star bitmap answers pi(x) == star for most endpoints; the walks of a
//     thread advance in lockstep; a stored link is recorded in the worklist
//     (resolve_edges).
//       k_hook        persistent, one 1024-thread CTA per SM, per-warp
//                     chunked appends (no block barriers), full L1
//       k_hook_sum    + the star summary in shared memory (device vote)
//       k_hook_cas /  root stores by atomicCAS: worklist passes, where a
//       k_hook_sum_cas  record would only be re-checked
//       k_hook_small  forming slots: full grid, 2 edges per thread, two-sided
//                     walks
//       k_hook_legacy block-aggregated appends (non-chunked launches)
//     The same kernels serve the topology slots and the worklist passes; the
//     worklist length lives on the device, so passes chain without host
//     round trips.
//   * k_compress_s0b is Multi-Jump with eager writes in ascending vertex
//     order (8 vertices per thread, chases in lockstep, in-group parents
//     resolved from their roots, chase loads through L1), and builds the
//     star bitmap and summary for the next hook.  k_compress is the ordered
//     variant without them (one-thread reference schedule, other engines).
//   * k_star_pick, k_step_* advance device-side plan state (next range,
//     tracked star, bitmap use, summary vote) and set the CUDA-graph
//     conditional-node value.
#include <cuda_runtime.h>

#include "hcc_internal.cuh"

namespace hcc {

namespace {

__device__ __forceinline__ u64 gtime() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Streaming 16-byte edge load: read once, do not allocate in L1, evict first
// from L2 so the edge stream does not push pi out of the 126 MB L2.
__device__ __forceinline__ u64 policy_evict_first() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;"
               : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ld_stream16(const uint4* p, u64 pol) {
  uint4 r;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, "
      "[%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}

// pi gather that may hit a stale L1 line; fine for the atomic-free hook
// (any value ever held by the slot is a valid ancestor).
__device__ __forceinline__ u32 ld_pi(const u32* p) { return *p; }

// Star-0 bitmap read: the bitmap is written only by the compress kernel,
// never during a hook launch, so the read-only path is legal; evict-last
// keeps hot words resident against the pi gathers.  HCC_BITLOAD selects the
// variant at compile time for experiments (0 = plain, 1 = nc + evict_last).
#ifndef HCC_BITLOAD
#define HCC_BITLOAD 0
#endif
__device__ __forceinline__ u32 ld_bits(const u32* p) {
#if HCC_BITLOAD == 1
  u32 r;
  asm volatile("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
#elif HCC_BITLOAD == 2
  // L2 evict-last: keep the (32 MiB at RMAT-28) bitmap resident against
  // the random pi sectors of the large-pi regime
  u32 r;
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
#else
  return *p;
#endif
}

// First pi gather of an endpoint outside the star: in the large-pi regime
// (pi >> L2) these sectors are rarely reused; HCC_PIGATHER=1 tags them L2
// evict-first.
#ifndef HCC_PIGATHER
#define HCC_PIGATHER 0
#endif
__device__ __forceinline__ u32 ld_pi_gather(const u32* p) {
#if HCC_PIGATHER == 1
  u32 r;
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
#else
  return *p;
#endif
}

// Template shift of the summary-predicated kernels (kSumShiftFixed).
constexpr int kSumFixSh = HCC_SUM_HALF ? -2 : 0;

// Shared-memory slot of summary word i: 32-word rows padded to 33 words, so
// consecutive rows start in consecutive banks.  Skewed graphs hit summary
// words whose indices have few one bits (RMAT hubs: 0, 32, 64, ...), which
// would all sit in bank 0 unpadded.  (Round 1 XOR-permuted each row by a
// hash of its index, 5 instructions a lookup against 2: RMAT-24 1.431 ->
// 1.414 ms, ER 2^24 2.00 -> 1.90 ms with the padding.)
__device__ __forceinline__ u32 sum_swz(u32 i) { return i + (i >> 5); }

__device__ __forceinline__ bool sum_covered(const u32* s_sum, u32 x, u32 shift) {
  const u32 g = x >> (5u + shift);
  return (s_sum[sum_swz(g >> 5)] >> (g & 31u)) & 1u;
}

// Control words a kernel reads at entry (dirty, star, use_sum) are written
// only by earlier kernels, so they are read through the non-coherent path:
// a volatile (L2) load by every thread of a 16K-block grid piles onto one
// L2 slice (measured: +5-8 us per compress).

// Coherent (L2) read: sees other threads' stores made during this kernel.
__device__ __forceinline__ u32 ld_fresh(const u32* p) { return __ldcg(p); }

// Compress chase step.  During a compress no root changes, so a stale value
// (an older ancestor) is safe and a root always reads as itself.  Through L1:
// chases into a giant component all end on the same few root lines, and as
// coherent L2 loads they queued on one L2 slice (ER-2^24's forming
// compresses 0.25 -> 0.13 ms, grid -46 us).  HCC_CHASE_L1=0 restores them.
#ifndef HCC_CHASE_L1
#define HCC_CHASE_L1 1
#endif
__device__ __forceinline__ u32 ld_chase(const u32* p) {
#if HCC_CHASE_L1
  return ld_pi(p);
#else
  return ld_fresh(p);
#endif
}

__device__ __forceinline__ void rec_clear(DevRec& r) {
  r.hook_t0 = ~0ull;
  r.hook_t1 = 0;
  r.comp_t0 = ~0ull;
  r.comp_t1 = 0;
  r.traversal = r.cas_fail = r.jump_steps = 0;
  r.edges_in = r.edges_out = 0;
  r.kind = 0;
  for (int i = 0; i < kJumpStripes; ++i) r.jump_stripe[i] = 0;
}

__device__ __forceinline__ DevRec* cur_rec(DevCtrl* c, DevRec* recs) {
  u32 i = c->rec;
  return recs + (i < (u32)kMaxRecs ? i : (u32)kMaxRecs - 1);
}

// Record of a launch: explicit (unrolled chains) or the control block's.
__device__ __forceinline__ DevRec* rec_of(DevCtrl* c, DevRec* recs, int idx) {
  return idx >= 0 ? recs + (idx < kMaxRecs ? idx : kMaxRecs - 1) : cur_rec(c, recs);
}

__device__ __forceinline__ void set_dirty(DevCtrl* c, int dslot) {
  if (dslot < 0)
    c->dirty = 1;
  else
    c->dirtyp[dslot] = 1;
}

__device__ __forceinline__ void next_rec(DevCtrl* c, DevRec* recs) {
  if (c->rec + 1 < (u32)kMaxRecs) {
    c->rec += 1;
    rec_clear(recs[c->rec]);
  }
}

// Phase spans: sampled blocks only (every 32nd block plus the last 32), so
// a kernel with tens of thousands of blocks does not serialize on two L2
// atomics per block.  Block 0 starts first and the tail blocks finish last.
__device__ __forceinline__ bool timer_block() {
  return (blockIdx.x & 31u) == 0 || blockIdx.x + 32u >= gridDim.x;
}

__device__ __forceinline__ void block_t0(u64* t0) {
  if (threadIdx.x == 0 && timer_block()) atomicMin(t0, gtime());
}

__device__ __forceinline__ void block_t1(u64* t1) {
  if (!timer_block()) return;  // uniform per block
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(t1, gtime());
}

// Adds a per-thread counter into a global u64.  Must be reached by every
// thread of the block (uniform control flow).
__device__ __forceinline__ void add_counter(u64* dst, u64 v) {
  if ((blockDim.x & 31u) == 0) {
    if (!__any_sync(0xffffffffu, v != 0)) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31u) == 0 && v) atomicAdd(dst, v);
  } else if (v) {
    atomicAdd(dst, v);
  }
}

__device__ __forceinline__ void resolve_src(const HookArgs& a, const uint2*& src,
                                            u64& b, u64& e, u32& out) {
  const DevCtrl* c = a.ctrl;
  if (a.mode == kSrcRange) {
    src = a.edges;
    b = a.b;
    e = a.e;
    out = c->parity;
  } else if (a.mode == kSrcSegment) {
    // partition_edges(m, s) (engines.hpp:43-58): the first m % s segments
    // get one extra edge.
    u64 s = c->nseg ? c->nseg : 1, seg = c->seg;
    u64 base = a.m / s, rem = a.m % s;
    b = seg * base + (seg < rem ? seg : rem);
    e = b + base + (seg < rem ? 1 : 0);
    if (e > a.m) e = a.m;
    if (b > e) b = e;
    src = a.edges;
    out = c->parity;
  } else if (a.mode == kSrcCtrlRange) {
    src = a.edges;
    b = c->seg_b;
    e = c->seg_e;
    out = c->parity;
  } else {
    u32 p = c->parity;
    src = p ? a.wl1 : a.wl0;
    b = 0;
    e = c->wl_count[p];
    // an overflowed list (device error bit 4; the host re-runs with full-size
    // worklists) counts past its capacity: never read beyond it
    if (e > a.wl_cap) e = a.wl_cap;
    out = p ^ 1u;
  }
}

// Reserve space for `c` entries of this thread in the output worklist with
// one global atomic per block; returns this thread's first slot.
// `appended` (meaningful in the thread that reserves: warp 0 lane 31, or
// each thread of a tiny launch) accumulates this block's appends; the block
// publishes it once per launch (block_publish), so a launch costs one
// counter atomic and one dirty store per block instead of one per tile.
__device__ __forceinline__ bool block_reserve(u32 c, u64* cnt, u64& pos,
                                              u64& appended) {
  __shared__ u32 s_w[32];
  __shared__ u64 s_base;
  if (!__syncthreads_or(c != 0)) return false;
  if ((blockDim.x & 31u) != 0) {
    // Tiny launches (max_threads < 32): per-thread reservation, in thread
    // order so a single-thread launch is deterministic.
    for (u32 t = 0; t < blockDim.x; ++t) {
      if (t == threadIdx.x && c) {
        pos = atomicAdd(cnt, (u64)c);
        appended += c;
      }
      __syncthreads();
    }
    return c != 0;
  }
  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  u32 x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (u32)o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const u32 nw = blockDim.x >> 5;
    u32 w = lane < nw ? s_w[lane] : 0u;
    u32 inc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (u32)o) inc += y;
    }
    if (lane < nw) s_w[lane] = inc - w;
    if (lane == 31) {
      s_base = atomicAdd(cnt, (u64)inc);
      appended += inc;
    }
  }
  __syncthreads();
  pos = s_base + s_w[warp] + (x - c);
  return c != 0;
}

__device__ __forceinline__ void block_publish(u64 appended, DevRec* r, DevCtrl* ctrl) {
  if (appended) {
    atomicAdd(&r->edges_out, appended);
    ctrl->dirty = 1;
  }
}

}  // namespace

// ---------------------------------------------------------------------------

__global__ void k_begin(DevCtrl* ctrl, DevRec* recs, u64 nseg) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevCtrl c = {};
    c.nseg = nseg ? nseg : 1;
    *ctrl = c;
    rec_clear(recs[0]);
  }
}

// Run start: control block + first record (k_begin), the adaptive plan's
// first range (plan_first > 0), and pi(v) = v + the star bitmap and
// summary (k_init_pi), in one launch.
__global__ void k_start(u32* pi, u64 n, u32* bits, DevCtrl* ctrl, DevRec* recs, u64 nseg,
                        u64 m, u64 plan_first, u32* sum, u32 sum_words) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevCtrl c = {};
    c.nseg = nseg ? nseg : 1;
    c.t_start = gtime();
    c.use_bits = 1;
    if (plan_first) {  // adaptive plan: the first range (the host sized it)
      u64 first = plan_first < m ? plan_first : m;
      if (c.nseg <= 1) first = m;  // a single slot takes every edge
      c.seg_e = first;
    }
    *ctrl = c;
    rec_clear(recs[0]);
  }
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  // records of the unrolled segments (chains without step kernels index
  // them directly)
  for (u64 i = 1 + tid; i < (nseg < (u64)kMaxRecs ? nseg : (u64)kMaxRecs); i += stride)
    rec_clear(recs[i]);
  if (bits)
    for (u64 w = tid; w < ((n + 31) >> 5); w += stride) bits[w] = w == 0 ? 1u : 0u;
  if (sum)
    for (u64 w = tid; w < sum_words; w += stride) sum[w] = 0u;
  const u64 n4 = n >> 2;
  uint4* p4 = reinterpret_cast<uint4*>(pi);
  for (u64 i = tid; i < n4; i += stride) {
    const u32 v = (u32)(i << 2);
    p4[i] = make_uint4(v, v + 1, v + 2, v + 3);
  }
  for (u64 v = (n4 << 2) + tid; v < n; v += stride) pi[v] = (u32)v;
}

// pi(v) = v (ParentForest::reset, forest.hpp:25-28), 16-byte stores.  With
// a star-0 bitmap, also its initial state (only vertex 0 is in star 0).
__global__ void k_init_pi(u32* pi, u64 n, u32* bits) {
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  if (bits)
    for (u64 w = tid; w < ((n + 31) >> 5); w += stride) bits[w] = w == 0 ? 1u : 0u;
  const u64 n4 = n >> 2;
  uint4* p4 = reinterpret_cast<uint4*>(pi);
  for (u64 i = tid; i < n4; i += stride) {
    u32 v = (u32)(i << 2);
    p4[i] = make_uint4(v, v + 1, v + 2, v + 3);
  }
  for (u64 v = (n4 << 2) + tid; v < n; v += stride) pi[v] = (u32)v;
}

// Lookups, root walk and stores for S edges of one thread (the body of a
// hook tile).  Returns the mask of edges whose (h, l) pair in (pu, pv)
// must be appended to the worklist (stored links and deferred walks).
// FIXSH: the summary's shift as a compile-time constant (>= 0, or -2 for
// the half-word table's ~0u), -1 = the run-time a.s0f_shift.
template <int S, bool SUM, bool BOTH = false, bool CAS = false, int FIXSH = -1>
__device__ __forceinline__ u32 resolve_edges(const HookArgs& a, u32& links, u32& tries,
                                             const u32* bits,
                                             const u32* s_sum, u32 star,
                                             const uint2 (&ed)[S], u32 (&pu)[S],
                                             u32 (&pv)[S]) {
  u32* pi = a.pi;
  if (bits) {
    // Star bitmap: one L1-friendly word read answers pi(x) == star for
    // the tracked component's vertices; only the rest gather pi.
    u32 wu[S], wv[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const u32 xu = ed[k].x >> 5, xv = ed[k].y >> 5;
      if (SUM) {
        // (a compile-time shift: the steady slot 0.825 -> 0.790 ms on
        // RMAT-24 at one bit per word)
        const u32 sh = FIXSH == -2 ? kSumHalfShift : FIXSH >= 0 ? (u32)FIXSH : a.s0f_shift;
        wu[k] = sum_covered(s_sum, ed[k].x, sh) ? ~0u : ld_bits(bits + xu);
        wv[k] = sum_covered(s_sum, ed[k].y, sh) ? ~0u : ld_bits(bits + xv);
      } else {
        wu[k] = ld_bits(bits + xu);
        wv[k] = ld_bits(bits + xv);
      }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      pu[k] = (wu[k] >> (ed[k].x & 31u)) & 1u ? star : ld_pi_gather(pi + ed[k].x);
      pv[k] = (wv[k] >> (ed[k].y & 31u)) & 1u ? star : ld_pi_gather(pi + ed[k].y);
    }
  } else {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      pu[k] = ld_pi(pi + ed[k].x);
      pv[k] = ld_pi(pi + ed[k].y);
    }
  }
  // Candidates (pu != pv) walk down like Fig. 3's atomic hook, but with a
  // plain load in place of the CAS: read pi[h]; already linked -> drop;
  // h still a root -> plain store; otherwise continue from (pi[h], l).
  // Every value met is a root of the forest at the start of the pass, so
  // only pass-start roots are ever stored to, and every store is recorded
  // in the worklist.  A walk that runs out of `walk`
  // steps is deferred to the worklist unstored (below).  This removes the
  // redundant stores that single-level reads make to hub slots while the
  // hub structure forms.
  // The S walks of a thread advance in lockstep, one level per round
  // with all their loads in flight (in the forming segments a walk is
  // several dependent round trips).
  u32 walking = 0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const u32 x = pu[k], y = pv[k];
    pu[k] = max(x, y);  // h
    pv[k] = min(x, y);  // l
    walking |= x != y ? 1u << k : 0u;
  }
  u32 act = walking, roots = a.walk == 0 ? walking : 0u;
  for (int step = 0; step < a.walk && walking; ++step) {
    // L1-cached read: any value the slot ever held is a recorded link
    // (pass-start link or a worklist pair), so a stale value is a safe
    // basis for both "drop" and "descend"; reading through L1 keeps the
    // hub slots every edge touches off the L2 slices.
    u32 ph[S], pl[S];
#pragma unroll
    for (int k = 0; k < S; ++k) ph[k] = walking & (1u << k) ? ld_pi(pi + pu[k]) : 0u;
    // BOTH (the small forming-slot hook): the low side descends in the same
    // round and a store needs both sides observed as roots, so it links h
    // to l's current root rather than to an l an earlier store of this pass
    // already hooked.  RMAT's first compress 0.10 -> 0.05 ms; in the
    // register-bound streaming hook the extra state spills (measured loss).
    if (BOTH) {
#pragma unroll
      for (int k = 0; k < S; ++k) pl[k] = walking & (1u << k) ? ld_pi(pi + pv[k]) : 0u;
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      if (!(walking & (1u << k))) continue;
      const u32 p = ph[k];
      if (BOTH) {
        const u32 q = pl[k];
        if (p == pu[k] && q == pv[k]) {  // both roots: store now
          pi[pu[k]] = pv[k];
          walking &= ~(1u << k);
        } else if (p == q) {             // one tree
          act &= ~(1u << k);
          walking &= ~(1u << k);
        } else {                         // one level down on both sides
          pu[k] = max(p, q);
          pv[k] = min(p, q);
        }
        continue;
      }
      if (p == pu[k]) {               // root: store now
        if (CAS) {
          // CAS (k_hook_cas: worklist passes, where stores are rare): a
          // link made this way is never lost, so it is not recorded and no
          // further pass has to re-check it
          const u32 old = atomicCAS(pi + pu[k], pu[k], pv[k]);
          ++tries;
          if (old == pu[k]) {
            ++links;
            act &= ~(1u << k);
            walking &= ~(1u << k);
          } else if (old == pv[k]) {  // someone linked h to l
            act &= ~(1u << k);
            walking &= ~(1u << k);
          } else {                    // h got a parent: descend from it
            const u32 l = pv[k];
            pu[k] = max(old, l);
            pv[k] = min(old, l);
          }
          continue;
        }
        pi[pu[k]] = pv[k];
        walking &= ~(1u << k);
      } else if (p == pv[k]) {        // already linked
        act &= ~(1u << k);
        walking &= ~(1u << k);
      } else {
        const u32 l = pv[k];
        pu[k] = max(p, l);
        pv[k] = min(p, l);
      }
    }
  }
  // A walk that ran out of steps defers the pair to the worklist without
  // storing: h may be an interior vertex whose link existed at pass start
  // (the forest need not be a star), and only slots observed as roots may
  // be written.
#pragma unroll
  for (int k = 0; k < S; ++k)
    if (roots & (1u << k)) pi[pu[k]] = pv[k];
  return act;
}

// Copy the star-0 summary into shared memory (swizzled rows).
// 16-byte reads, eight in flight per thread before their stores: a
// one-word load-store loop waited an L2 round trip per word (~5 us per
// launch for the 64 KB table, 12% of the stall samples of an adaptive
// segment hook).
__device__ __forceinline__ void store_summary4(u32* s_sum, u32 j, uint4 v) {
  // j is a multiple of 4: the four words share one padded row
  const u32 p = sum_swz(j);
  s_sum[p] = v.x;
  s_sum[p + 1] = v.y;
  s_sum[p + 2] = v.z;
  s_sum[p + 3] = v.w;
}

__device__ __forceinline__ void load_summary(const HookArgs& a, u32* s_sum) {
  const u32 w = a.s0f_words, n16 = w >> 2, bd = blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(a.s0f);
  u32 i = threadIdx.x;
  for (; i + 7 * bd < n16; i += 8 * bd) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(src + i + k * bd);
#pragma unroll
    for (int k = 0; k < 8; ++k) store_summary4(s_sum, (i + k * bd) << 2, v[k]);
  }
  for (; i < n16; i += bd) store_summary4(s_sum, i << 2, __ldcg(src + i));
  for (u32 j = (n16 << 2) + threadIdx.x; j < w; j += bd) s_sum[sum_swz(j)] = __ldcg(a.s0f + j);
  __syncthreads();
}

// Atomic-free Hook (forest.hpp:83-89) over an edge range, a segment or the
// current worklist.  See the file comment for the design.  EPT edges per
// thread per tile; the next tile's edge loads are issued before the current
// tile's dependent gathers (software pipelining).
template <int EPT, bool SUM, bool BOTH = false>
__device__ __forceinline__ void hook_impl(const HookArgs& a) {
  const uint2* src;
  u64 b, e;
  u32 out;
  resolve_src(a, src, b, e, out);
  DevCtrl* ctrl = a.ctrl;
  DevRec* r = cur_rec(ctrl, a.recs);
  // root of the star the bitmap tracks (set by the last compress), and
  // whether the last step found the bitmap worth a lookup
  const u32 star = a.s0b ? __ldg(&ctrl->star) : 0u;
  const u32* bits = (a.s0b && (SUM || __ldg(&ctrl->use_bits))) ? a.s0b : nullptr;
  block_t0(&r->hook_t0);
  if (blockIdx.x == 0 && threadIdx.x == 0 && e > b) {
    atomicAdd(&r->edges_in, e - b);
    atomicAdd(&ctrl->edges_processed, e - b);
  }
  u32* pi = a.pi;
  uint2* wl_out = out ? a.wl1 : a.wl0;
  u64* cnt_out = &ctrl->wl_count[out];

  // One-thread launch (max_threads = 1): strictly sequential ascending edge
  // order with read-after-write between edges, i.e. exactly the reference's
  // workers = 1 schedule (parallel.hpp:29, 52-55).
  if (gridDim.x * blockDim.x == 1) {
    u32 wrote = 0;
    for (u64 i = b; i < e; ++i) {
      const uint2 ed = src[i];
      u32 x = ld_fresh(pi + ed.x), y = ld_fresh(pi + ed.y);
      if (x == y) continue;
      u32 h = max(x, y), l = min(x, y);
      bool store = true, at_root = a.walk == 0;
      for (int step = 0; step < a.walk; ++step) {
        const u32 ph = ld_fresh(pi + h);
        if (ph == h) {
          at_root = true;
          break;
        }
        if (ph == l) {
          store = false;
          break;
        }
        h = max(ph, l);
        l = min(ph, l);
      }
      if (!store) continue;
      if (at_root) {
        pi[h] = l;
        wrote = 1;
      }
      if (a.append) {
        const u64 pos = atomicAdd(cnt_out, 1ull);
        if (pos < a.wl_cap)
          wl_out[pos] = make_uint2(h, l);
        else
          atomicOr(&ctrl->err, 4u);
        atomicAdd(&r->edges_out, 1ull);
      }
    }
    if (wrote) {
      ctrl->dirty = 1;
      if (!a.append) ctrl->changed = 1;
    }
    block_t1(&r->hook_t1);
    return;
  }

  // Head / tail edges that do not fill a 16-byte pair: thread 0 of block 0.
  u64 b2 = b + (b & 1ull);
  if (b2 > e) b2 = e;
  const u64 n4 = (e - b2) >> 1;
  u32 any_change = 0;
  u64 appended = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    u64 idx[2];
    int k = 0;
    if (b2 != b) idx[k++] = b;
    if ((e - b2) & 1ull) idx[k++] = e - 1;
    for (int j = 0; j < k; ++j) {
      uint2 ed = src[idx[j]];
      u32 pu = ld_pi(pi + ed.x), pv = ld_pi(pi + ed.y);
      if (pu != pv) {
        u32 h = max(pu, pv), l = min(pu, pv);
        pi[h] = l;
        any_change = 1;
        if (a.append) {
          u64 pos = atomicAdd(cnt_out, 1ull);
          if (pos < a.wl_cap)
            wl_out[pos] = make_uint2(h, l);
          else
            atomicOr(&ctrl->err, 4u);
          atomicAdd(&r->edges_out, 1ull);
          ctrl->dirty = 1;
        }
      }
    }
  }

  // Star-0 summary staged in shared memory: a lane whose endpoint's
  // 32-vertex word is known all-ones skips the bitmap gather (the L1 miss /
  // wavefront that bounds the steady segments).
  extern __shared__ u32 s_sum[];
  if (SUM) load_summary(a, s_sum);
  const uint4* s4 = reinterpret_cast<const uint4*>(src + b2);
  const u64 pol = policy_evict_first();
  const u64 tile = (u64)blockDim.x * (EPT / 2);
  const u64 ntiles = (n4 + tile - 1) / tile;
  // Out-of-range slots become the self-loop (0,0): a no-op hook.
  auto load_tile = [&](u64 t, uint4* q) {
#pragma unroll
    for (int j = 0; j < EPT / 2; ++j) {
      const u64 i = t * tile + (u64)j * blockDim.x + threadIdx.x;
      q[j] = i < n4 ? ld_stream16(s4 + i, pol) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  uint4 nq[EPT / 2];
  if ((u64)blockIdx.x < ntiles) load_tile(blockIdx.x, nq);
  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint2 ed[EPT];
#pragma unroll
    for (int j = 0; j < EPT / 2; ++j) {
      ed[2 * j] = make_uint2(nq[j].x, nq[j].y);
      ed[2 * j + 1] = make_uint2(nq[j].z, nq[j].w);
    }
    if (t + gridDim.x < ntiles) load_tile(t + gridDim.x, nq);
    u32 pu[EPT], pv[EPT];
    u32 links_unused = 0, tries_unused = 0;
    const u32 act = resolve_edges<EPT, SUM, BOTH>(a, links_unused, tries_unused, bits, s_sum, star,
                                                  ed, pu, pv);
    if (a.append) {
      u64 pos;
      if (block_reserve(__popc(act), cnt_out, pos, appended)) {
        if (pos + __popc(act) <= a.wl_cap) {
#pragma unroll
          for (int k = 0; k < EPT; ++k)
            if (act & (1u << k)) wl_out[pos++] = make_uint2(pu[k], pv[k]);
        } else {
          atomicOr(&ctrl->err, 4u);  // sized on the host; the host re-runs
        }
      }
    } else {
      any_change |= act;
    }
  }
  if (!a.append) {
    if (__syncthreads_or(any_change != 0) && threadIdx.x == 0) {
      ctrl->changed = 1;
      ctrl->dirty = 1;
    }
  } else {
    block_publish(appended, r, ctrl);
  }
  block_t1(&r->hook_t1);
}


__device__ void star_pick_warp(const u32* pi, u64 n, DevCtrl* ctrl, u32 dirty);

// The hook's last block to finish runs the star pick (the kernel's stores
// are all visible to it: each block fences before it counts itself), so an
// unrolled chain needs no k_star_pick launch between hook and compress.
__device__ __forceinline__ void last_block_pick(const HookArgs& a) {
  // (__syncthreads_or broadcasts the verdict: no static shared memory, so
  // the plain streaming hook keeps its full-L1 configuration)
  int last = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&a.ctrl->pick_count, 1u) == gridDim.x - 1;
  }
  if (!__syncthreads_or(last)) return;
  __threadfence();
  if (threadIdx.x < 32) {
    const u32 d = a.dslot < 0 ? __ldcg(&a.ctrl->dirty) : __ldcg(&a.ctrl->dirtyp[a.dslot]);
    if (d != 0 && a.n) star_pick_warp(a.pi, a.n, a.ctrl, d);
  }
  if (threadIdx.x == 0) a.ctrl->pick_count = 0;
}

// Per-warp output of the streaming hook: the warp's current chunk of the
// output worklist [pos, end), its real appends and its change flag (all
// warp-uniform).
struct WarpOut {
  u64 pos = 0, end = 0;
  u32 appended = 0, changed = 0;
};

// Append the (h, l) pairs selected by each lane's `act` mask (at most N per
// lane) to the warp's chunk; a full chunk is padded with (0, 0) no-op
// records and a new one is reserved with one global atomic.
template <int N>
__device__ __forceinline__ void warp_emit(const HookArgs& a, WarpOut& w, uint2* wl_out,
                                          u64* cnt_out, u32 lane, u32 act,
                                          const u32 (&h)[N], const u32 (&l)[N]) {
  static_assert(32 * N <= (int)kWlChunk, "a warp's appends must fit one chunk");
  const u32 cnt = __popc(act);
  u32 incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (u32)o) incl += y;
  }
  const u32 total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  if (!a.append) {
    w.changed = 1;
    return;
  }
  if (w.pos + total > w.end) {
    for (u64 i = w.pos + lane; i < w.end; i += 32) wl_out[i] = make_uint2(0u, 0u);
    u64 base = 0;
    if (lane == 0) base = atomicAdd(cnt_out, (u64)kWlChunk);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + kWlChunk > a.wl_cap) {  // sized on the host; never expected
      if (lane == 0) atomicOr(&a.ctrl->err, 4u);
      w.pos = w.end = 0;
      return;
    }
    w.pos = base;
    w.end = base + kWlChunk;
  }
  u64 pos = w.pos + (incl - cnt);
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (act & (1u << k)) wl_out[pos++] = make_uint2(h[k], l[k]);
  w.pos += total;
  w.appended += total;
}

// warp_emit, or (a launch that appends nothing: the adaptive engine's CAS
// segments) only the change flag.
template <int N, bool APPEND>
__device__ __forceinline__ void emit(const HookArgs& a, WarpOut& w, uint2* wl_out, u64* cnt_out,
                                     u32 lane, u32 act, const u32 (&h)[N], const u32 (&l)[N]) {
  if (APPEND)
    warp_emit<N>(a, w, wl_out, cnt_out, lane, act, h, l);
  else if (__any_sync(0xffffffffu, act != 0))
    w.changed = 1;
}

// Streaming hook for full-warp launches: no block barriers after the
// prologue; appends go to per-warp chunks of the output worklist (one
// global atomic per kWlChunk records; a chunk's unused tail is padded with
// (0, 0) self-loops, which the next pass skips as no-ops).
//
// SUM (k_hook_sum, chosen on the device when the star-0 summary covers at
// least half of its groups): each thread first tests its EPT edges against
// the summary staged in shared memory (two shared loads per edge, no global
// traffic when both endpoints' words are all in star 0); the warp compacts
// the rest into its shared-memory queue and resolves them kHookSlow per
// lane per round.  Otherwise (k_hook: no shared memory, so L1 keeps its full
// size for the bitmap's hot words; e.g. RMAT, whose isolated vertices break
// most words) every edge takes the bitmap / gather path directly.
template <int EPT, bool SUM, bool CAS = false, bool APPEND = true, bool SUMD = false,
          bool DYNOK = true, int FIXSH = -1, bool BOTH = false>
__device__ __forceinline__ void hook_stream(const HookArgs& a) {
  constexpr int S = kHookSlow;
  const uint2* src;
  u64 b, e;
  u32 out;
  resolve_src(a, src, b, e, out);
  DevCtrl* ctrl = a.ctrl;
  DevRec* r = rec_of(ctrl, a.recs, a.rec_idx);
  // root of the star the bitmap tracks (set by the last compress), and
  // whether the last step found the bitmap worth a lookup
  const u32 star = a.s0b ? __ldg(&ctrl->star) : 0u;
  const u32* bits = (a.s0b && (SUM || __ldg(&ctrl->use_bits))) ? a.s0b : nullptr;
  block_t0(&r->hook_t0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    r->kind = SUMD ? HCC_HOOK_KERNEL_SUMD
              : CAS ? HCC_HOOK_KERNEL_CAS
              : SUM ? HCC_HOOK_KERNEL_SUM
                    : HCC_HOOK_KERNEL_STREAM;
    if (e > b) {
      atomicAdd(&r->edges_in, e - b);
      atomicAdd(&ctrl->edges_processed, e - b);
    }
  }
  uint2* wl_out = out ? a.wl1 : a.wl0;
  u64* cnt_out = &ctrl->wl_count[out];
  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;

  extern __shared__ u32 s_sum[];
  if (SUM || SUMD) load_summary(a, s_sum);
  uint2* s_q = reinterpret_cast<uint2*>(s_sum + sum_region_words(a.s0f_words)) +
               (size_t)warp * (32 * EPT);
  WarpOut wo;
  u32 links = 0, tries = 0;  // CAS links made / CAS attempts of this thread

  // head / tail edges that do not fill a 16-byte pair: warp 0 of block 0
  u64 b2 = b + (b & 1ull);
  if (b2 > e) b2 = e;
  const u64 n4 = (e - b2) >> 1;
  if (blockIdx.x == 0 && warp == 0) {
    uint2 ed[1] = {make_uint2(0u, 0u)};
    if (lane == 0 && b2 != b) ed[0] = src[b];
    if (lane == 1 && ((e - b2) & 1ull)) ed[0] = src[e - 1];
    u32 h[1], l[1];
    const u32 act = resolve_edges<1, false, false, CAS>(a, links, tries, bits, s_sum, star, ed, h, l);
    emit<1, APPEND>(a, wo, wl_out, cnt_out, lane, act, h, l);
  }

  const uint4* s4 = reinterpret_cast<const uint4*>(src + b2);
  const u64 pol = policy_evict_first();
  // Warp tiles: 32 lanes x EPT/2 16-byte loads (256 edges), the block's
  // warps on consecutive tiles (a 128 KB stretch per block and round).  A
  // warp that runs out of tiles frees its SM's issue slots to the others, so
  // a short launch (an adaptive segment: ~7 block tiles per SM) no longer
  // idles whole blocks behind the last round's stragglers.
  const u64 tile = 32ull * (EPT / 2);
  // tile indices fit 32 bits (a tile is 256 edges)
  const u32 ntiles = (u32)((n4 + tile - 1) / tile);
  const u32 wpb = blockDim.x >> 5;
  const u32 gw = blockIdx.x * wpb + warp, wstride = gridDim.x * wpb;
  // Out-of-range slots become the self-loop (0,0): a no-op hook.
  auto load_tile = [&](u32 t, uint4* q) {
#pragma unroll
    for (int j = 0; j < EPT / 2; ++j) {
      const u64 i = (u64)t * tile + (u64)j * 32 + lane;
      q[j] = i < n4 ? ld_stream16(s4 + i, pol) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  // Dynamic schedule (a.dyn, launches of >= 32 tiles per warp): each warp
  // starts on a static chunk of kch tiles, then takes further chunks from a
  // global counter; the next chunk is requested halfway through the current
  // one, so the atomic's latency hides behind work and the requests of a
  // launch's warps do not arrive as one burst.  A static round-robin let
  // warps on slow SMs trail: RMAT-28's steady hook ran 5.5 ms past its
  // median block for some placements of the star bitmap.
  const u32 tpw = ntiles / wstride;
  const bool dyn = DYNOK && a.dyn && tpw >= 32;
  const u32 kch = tpw / 16 < 4 ? 4 : tpw / 16 > 64 ? 64 : tpw / 16;
  u32 cbase = gw * kch;  // current chunk
  u32 nreq = 0;          // lane 0: reply for the next chunk
  auto next_of = [&](u32 t) -> u32 {
    if (!dyn) return t + wstride;
    const u32 k = t + 1 - cbase;
    if (k == kch / 2 && lane == 0) nreq = atomicAdd(&ctrl->tile_ctr, kch);
    if (k < kch) return t + 1;
    cbase = wstride * kch + __shfl_sync(0xffffffffu, nreq, 0);
    return cbase;
  };
  const u32 t0 = dyn ? cbase : gw;
  uint4 nq[EPT / 2];
  if (t0 < ntiles) load_tile(t0, nq);
  for (u32 t = t0; t < ntiles;) {
    uint2 ed[EPT];
#pragma unroll
    for (int j = 0; j < EPT / 2; ++j) {
      ed[2 * j] = make_uint2(nq[j].x, nq[j].y);
      ed[2 * j + 1] = make_uint2(nq[j].z, nq[j].w);
    }
    const u32 tn = next_of(t);
    if (tn < ntiles) load_tile(tn, nq);
    t = tn;
    if (SUMD) {
      // summary-predicated lookups, no compaction: a lane whose endpoint's
      // 32-vertex word is all in the star (one shared-memory load) skips
      // its bitmap gather, so the gather instruction touches fewer lines
#if HCC_SUMD_HALVES
      // (two halves of EPT/2 edges: fewer live registers)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint2 e2[EPT / 2];
#pragma unroll
        for (int k = 0; k < EPT / 2; ++k) e2[k] = ed[hf * (EPT / 2) + k];
        u32 h[EPT / 2], l[EPT / 2];
        const u32 act =
            resolve_edges<EPT / 2, true, false, CAS>(a, links, tries, bits, s_sum, star, e2, h, l);
        emit<EPT / 2, APPEND>(a, wo, wl_out, cnt_out, lane, act, h, l);
      }
#else
      u32 h[EPT], l[EPT];
      const u32 act =
          resolve_edges<EPT, true, false, CAS, FIXSH>(a, links, tries, bits, s_sum, star, ed, h, l);
      emit<EPT, APPEND>(a, wo, wl_out, cnt_out, lane, act, h, l);
#endif
      continue;
    }
    if (!SUM) {
      u32 h[EPT], l[EPT];
      const u32 act = resolve_edges<EPT, false, BOTH, CAS>(a, links, tries, bits, s_sum, star, ed, h, l);
      emit<EPT, APPEND>(a, wo, wl_out, cnt_out, lane, act, h, l);
      continue;
    }
    // fast path: both endpoints in summary-covered words (or a self loop)
    u32 need = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const bool done = ed[k].x == ed[k].y ||
                        (sum_covered(s_sum, ed[k].x, a.s0f_shift) &&
                         sum_covered(s_sum, ed[k].y, a.s0f_shift));
      need |= done ? 0u : 1u << k;
    }
    const u32 nneed = __popc(need);
    u32 incl = nneed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (u32)o) incl += y;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    u32 o = incl - nneed;
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (need & (1u << k)) s_q[o++] = ed[k];
    __syncwarp();
    for (u32 base = 0; base < total; base += 32u * S) {
      uint2 q2[S];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const u32 idx = base + (u32)j * 32u + lane;
        q2[j] = idx < total ? s_q[idx] : make_uint2(0u, 0u);
      }
      u32 h[S], l[S];
      const u32 act = resolve_edges<S, true, false, CAS>(a, links, tries, bits, s_sum, star, q2, h, l);
      emit<S, APPEND>(a, wo, wl_out, cnt_out, lane, act, h, l);
    }
    __syncwarp();
  }
  // pad this warp's chunk tail; publish the real appends (CAS links count
  // as stores for the plan and need a compress too)
  for (u64 i = wo.pos + lane; i < wo.end; i += 32) wl_out[i] = make_uint2(0u, 0u);
  if (CAS) {
    // reference KernelCounters (forest.hpp:65-75): a CAS attempt is one
    // traversal step, a CAS that did not link is a failure
    add_counter(&r->traversal, tries);
    add_counter(&r->cas_fail, tries - links);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xffffffffu, links, o);
  }
  if (lane == 0) {
    if (wo.appended || links) {
      atomicAdd(&r->edges_out, (u64)wo.appended + links);
      set_dirty(ctrl, a.dslot);
    }
    if (wo.changed) {
      ctrl->changed = 1;
      set_dirty(ctrl, a.dslot);
    }
  }
  if (a.pick) last_block_pick(a);
  block_t1(&r->hook_t1);
}

#ifndef HCC_HOOK_MINB
#define HCC_HOOK_MINB (1024 / HCC_HOOK_CTA)
#endif
// Two-sided walks (k_hook_small's BOTH) in the streaming hook, at 768
// threads for the registers they need: the middle topology slots (at 1024
// threads the extra state spilled).
__global__ void __launch_bounds__(kHookBothCta, 1) k_hook_both(HookArgs a) {
  if (a.gate == kGateIfPlain && __ldg(&a.ctrl->use_sum)) return;
  hook_stream<HCC_BOTH_EPT, false, false, true, false, true, -1, true>(a);
}

__global__ void __launch_bounds__(kHookCta, HCC_HOOK_MINB) k_hook(HookArgs a) {
  // (the summary path is k_hook_sum; s0f is ignored here)
  if (a.gate == kGateIfPlain && __ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false>(a);
}

// Block-aggregated hook (per-tile block scan for appends): launches that are
// not full warps or not sized for chunk padding (baseline passes, the
// looped-segment path, re-hook, max_threads launches).
__global__ void __launch_bounds__(kHookCta, HCC_HOOK_MINB) k_hook_legacy(HookArgs a) {
  hook_impl<kHookEPT, false>(a);
}

// CAS-storing variants (separate kernels: the runtime branch in k_hook cost
// it spills).
__global__ void __launch_bounds__(kHookCasCta, 1) k_hook_cas(HookArgs a) {
  if (a.gate == kGateIfPlain && __ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false, true>(a);
}

__global__ void __launch_bounds__(kHookCasCta, 1) k_hook_sum_cas(HookArgs a) {
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, true, true>(a);
}

// Segment hook of the adaptive / atomic engines: CAS stores, unbounded
// walks, nothing appended (no chunk state), so it fits 1024-thread CTAs.
__global__ void __launch_bounds__(kHookCta, HCC_HOOK_MINB) k_hook_seg_cas(HookArgs a) {
  hook_stream<kHookEPT, false, true, false>(a);
}

#ifndef HCC_SUMD_HALVES
#define HCC_SUMD_HALVES 0
#endif
// Worklist pass (CAS stores) with summary-predicated lookups.
__global__ void __launch_bounds__(kHookCasCta, 1) k_hook_cas_sumd(HookArgs a) {
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false, true, true, true, false, kSumFixSh>(a);
}

__global__ void __launch_bounds__(kHookCasCta, 1) k_hook_cas_sumd_sh(HookArgs a) {
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false, true, true, true, false>(a);
}

// Adaptive / atomic segment hook with summary-predicated lookups.
__global__ void __launch_bounds__(kHookCta, 1) k_hook_seg_cas_sumd(HookArgs a) {
  hook_stream<kHookEPT, false, true, false, true, false, 0>(a);
}

__global__ void __launch_bounds__(kHookCta, 1) k_hook_seg_cas_sumd_sh(HookArgs a) {
  hook_stream<kHookEPT, false, true, false, true, false>(a);
}

// Streaming hook with summary-predicated lookups (the summary in shared
// memory, no slow-path queues: 64 KB instead of 128 KB of shared memory).
// Static schedule: the dynamic one's state made it spill 40 B, and the
// kernel only serves n <= 2^24, where the static schedule is as fast.
__global__ void __launch_bounds__(kHookSumdCta, 1) k_hook_sumd(HookArgs a) {
  if (a.gate == kGateIfPlain && __ldg(&a.ctrl->use_sum)) return;
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false, false, true, true, false, kSumFixSh>(a);
}

// A coarser summary (n > 2^24: one bit per 2^shift words).
__global__ void __launch_bounds__(kHookSumdCta, 1) k_hook_sumd_sh(HookArgs a) {
  if (a.gate == kGateIfPlain && __ldg(&a.ctrl->use_sum)) return;
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, false, false, true, true, false>(a);
}



// Streaming hook with the star-0 summary in shared memory (full warps,
// chunked appends, s0f set).
// Static schedule (HCC_SUM_DYN=1: dynamic, which spilled 12 B and measured
// the same: ER n = 2^24 + 1 2.34 vs 2.32 ms, n = 2^26 16.15 vs 16.14 ms).
#ifndef HCC_SUM_DYN
#define HCC_SUM_DYN 0
#endif
__global__ void __launch_bounds__(kHookSumCta, 1) k_hook_sum(HookArgs a) {
  if (a.gate == kGateIfSum && !__ldg(&a.ctrl->use_sum)) return;
  hook_stream<kHookEPT, true, false, true, false, HCC_SUM_DYN != 0>(a);
}

// Small segments (the forming regime): kSmallEPT (2) edges per thread, one
// tile per block over a full grid, two-sided walks.
__global__ void __launch_bounds__(kHookThreads) k_hook_small(HookArgs a) {
  hook_impl<kSmallEPT, false, true>(a);
}

// CAS-verified hook (forest.hpp:107-122): walks down until it acquires a
// root slot; counters follow the reference definitions.
__global__ void __launch_bounds__(kHookCta) k_cas_hook(HookArgs a) {
  const uint2* src;
  u64 b, e;
  u32 out;
  resolve_src(a, src, b, e, out);
  DevCtrl* ctrl = a.ctrl;
  DevRec* r = cur_rec(ctrl, a.recs);
  block_t0(&r->hook_t0);
  if (blockIdx.x == 0 && threadIdx.x == 0 && e > b) {
    atomicAdd(&r->edges_in, e - b);
    atomicAdd(&ctrl->edges_processed, e - b);
  }
  u32* pi = a.pi;
  u64 trav = 0, fails = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = b + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < e;
       i += stride) {
    uint2 ed = src[i];
    u32 u = ed.x, v = ed.y;
    for (;;) {
      u32 pu = ld_fresh(pi + u), pv = ld_fresh(pi + v);
      if (pu == pv) break;
      ++trav;
      u32 h = max(pu, pv), l = min(pu, pv);
      u32 old = atomicCAS(pi + h, h, l);
      if (old == h) break;
      ++fails;
      u = old;
      v = l;
    }
  }
  add_counter(&r->traversal, trav);
  add_counter(&r->cas_fail, fails);
  if (threadIdx.x == 0 && blockIdx.x == 0) ctrl->dirty = 1;
  block_t1(&r->hook_t1);
}

// Multi-Jump compress (forest.hpp:127-136) over all vertices in ascending
// block order, eager writes.  A vertex that is a root or already points at a
// root costs one coalesced read and one (usually L1/L2-hot) gather; warps
// whose lanes are all in that state exit the chase loop together.
__global__ void __launch_bounds__(kVertThreads)
    k_compress(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs, int skip_if_clean) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->tile_ctr = 0;  // next hook's schedule
  if (skip_if_clean && __ldg(&ctrl->dirty) == 0) return;
  DevRec* r = cur_rec(ctrl, recs);
  block_t0(&r->comp_t0);
  u64 steps = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  // Four consecutive vertices per thread: one 16-byte coalesced read, then
  // up to four independent parent gathers in flight before any chase.
  const u64 n4 = n >> 2;
  const uint4* p4 = reinterpret_cast<const uint4*>(pi);
  for (u64 q = tid; q < n4; q += stride) {
    const uint4 pp = __ldcg(p4 + q);
    const u32 v0 = (u32)(q << 2);
    u32 p[4] = {pp.x, pp.y, pp.z, pp.w};
    u32 gp[4];
#pragma unroll
    // First parent read through L1: during a compress no root changes and
    // non-root slots only move to other ancestors, so a stale value is safe
    // (it just lengthens the chase), while a fresh read would send every
    // warp to the one L2 sector holding the giant component's root.
    for (int j = 0; j < 4; ++j) gp[j] = p[j] != v0 + j ? ld_pi(pi + p[j]) : p[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u32 a = p[j], b = gp[j];
      // parent inside this group: re-read after the earlier chases wrote it
      // (keeps the one-thread schedule identical to the reference's
      // sequential ascending pass, forest.hpp:127-136 / parallel.hpp:52-55)
      // (own writes are visible to the L1-cached reads, so a one-thread
      // launch reads exactly what the reference's sequential pass reads)
      if (j > 0 && a >= v0 && a != v0 + j) b = ld_chase(pi + a);
      while (b != a) {  // eager writes: every step is visible to other chasers
        pi[v0 + j] = b;
        ++steps;
        a = b;
        b = ld_chase(pi + a);
      }
    }
  }
  for (u64 v = (n4 << 2) + tid; v < n; v += stride) {
    u32 a = ld_chase(pi + v);
    if (a == (u32)v) continue;
    u32 b = ld_chase(pi + a);
    while (b != a) {
      pi[v] = b;
      ++steps;
      a = b;
      b = ld_chase(pi + a);
    }
  }
  add_counter(&r->jump_stripe[blockIdx.x & (kJumpStripes - 1)], steps);
  block_t1(&r->comp_t1);
}

// Star choice after a topology hook (one warp): the bitmap built by the
// next compress tracks the component of ctrl->star_hint.  A fixed 32-vertex
// sample is chased to its roots; when one component clearly outnumbers the
// tracked one (ER: the giant forms around vertex 1 while vertex 0 is still
// isolated; any graph whose vertex 0 is isolated), the hint moves to it.
constexpr int kStarChase = 32;

__device__ void star_pick_warp(const u32* pi, u64 n, DevCtrl* ctrl, u32 dirty);

__global__ void k_star_pick(const u32* pi, u64 n, DevCtrl* ctrl) {
  if (threadIdx.x >= 32 || n == 0) return;
  star_pick_warp(pi, n, ctrl, __ldcg(&ctrl->dirty));
}

// The pick itself (one full warp).  `dirty`: the slot's hook stored
// something; a slot that stored nothing skips its compress
// (kCompressIfDirty), so the bitmap keeps tracking the current star: it must
// not move.
__device__ void star_pick_warp(const u32* pi, u64 n, DevCtrl* ctrl, u32 dirty) {
  const u32 lane = threadIdx.x & 31u;
  if (dirty == 0) return;
  u64 hsh = (u64)(lane + 1) * 0x9E3779B97F4A7C15ull;
  hsh ^= hsh >> 29;
  hsh *= 0xBF58476D1CE4E5B9ull;
  hsh ^= hsh >> 32;
  // bounded chases: before a compress the trees can be long chains (grid
  // rows); a sample that does not reach its root within the bound counts
  // as unknown (~0); an unresolved current star (~0) leaves the next
  // bitmap empty unless a candidate wins
  u32 x = (u32)(hsh % n);
  // the sample's first parents and the control words are independent
  // loads: issue them together (one round trip, not three)
  const u32 px = ld_fresh(pi + x);
  const u32 star0 = __ldcg(&ctrl->star);
  u32 cur = __ldcg(&ctrl->star_hint);
  // the tracked star already holds a quarter of the sample: keep it (leaf
  // slots are not written by a hook, so pi(x) == star still marks it)
  if (star0 < n && ld_fresh(pi + star0) == star0 &&
      __popc(__ballot_sync(0xffffffffu, px == star0)) >= 8)
    return;
  bool rooted = px == x;
  x = px;
  for (int i = 1; i < kStarChase && !rooted; ++i) {
    const u32 p = ld_fresh(pi + x);
    rooted = p == x;
    x = p;
  }
  if (!rooted) x = ~0u;
  bool cur_rooted = false;
  for (int i = 0; i < kStarChase && !cur_rooted; ++i) {
    const u32 p = ld_fresh(pi + cur);
    cur_rooted = p == cur;
    cur = p;
  }
  if (!cur_rooted) cur = ~0u;
  const u32 same = __match_any_sync(0xffffffffu, x);
  unsigned long long best = x == ~0u ? 0ull : ((unsigned long long)__popc(same) << 32) | x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  const u32 n_cand = (u32)(best >> 32), cand = (u32)best;
  const u32 n_cur = __popc(__ballot_sync(0xffffffffu, cur != ~0u && x == cur));
  if (lane == 0) {
    // publish the root the next compress builds the bitmap for
    const u32 star = (n_cand >= 6 && n_cand > 2 * n_cur) ? cand : cur;
    if (star != ~0u) ctrl->star_hint = star;
    ctrl->star = star;
  }
}

// Multi-Jump compress of vertices [v0, v0 + 8) (one thread; pa, pb hold
// pi of the group when it is whole).  Returns bit j = (root(v0 + j) ==
// star) and counts written levels in `steps`.
__device__ __forceinline__ u32 compress8(u32* pi, u64 n, u64 v0, bool whole, uint4 pa,
                                         uint4 pb, u32 star, bool star_root, u64& steps) {
  u32 byte = 0;
  if (whole) {
    u32 a[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
    // Settled group (most groups once the giant is a star): every vertex
    // is its own root or a child of the star's root, which is still a
    // root.  No gathers, no writes.
    if (star_root) {
      u32 settled = 1, sb = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        settled &= (a[j] == (u32)v0 + j) | (a[j] == star);
        sb |= (u32)(a[j] == star) << j;
      }
      if (settled) return sb;
    }
    // pi(v) <= v, so a parent inside this group is an earlier vertex of it:
    // those vertices take their parent's root after the chases (ascending,
    // as the reference's sequential pass would; grid rows chain this way).
    u32 dep = 0;
#pragma unroll
    for (int j = 1; j < 8; ++j)
      dep |= (a[j] >= (u32)v0 && a[j] < (u32)v0 + j) ? 1u << j : 0u;
    u32 b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      b[j] = (a[j] != (u32)v0 + j && !(dep & (1u << j)) && !(star_root && a[j] == star))
                 ? ld_pi(pi + a[j])
                 : a[j];
    // The remaining chases advance in lockstep (one level per round, up to
    // eight independent loads in flight) instead of one after another: in
    // the forming segments the trees are deep and a serial chase is one
    // dependent L2 round trip per level.  Each level is still written
    // eagerly; values read from other chasers' slots are ancestors, so a
    // stale read only costs an extra round.
    u32 act = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) act |= (b[j] != a[j]) ? 1u << j : 0u;
    while (act) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (act & (1u << j)) {
          pi[v0 + j] = b[j];
          ++steps;
          a[j] = b[j];
          b[j] = ld_chase(pi + a[j]);
        }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (b[j] == a[j]) act &= ~(1u << j);
    }
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      if (dep & (1u << j)) {
        u32 root = a[0];
#pragma unroll
        for (int k = 1; k < j; ++k)
          if (a[j] == (u32)v0 + k) root = a[k];
        if (root != a[j]) {
          pi[v0 + j] = root;
          ++steps;
          a[j] = root;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) byte |= (a[j] == star) ? 1u << j : 0u;
  } else if (v0 < n) {
    for (u64 v = v0; v < n; ++v) {
      u32 a = ld_chase(pi + v);
      if (a != (u32)v) {
        u32 b = ld_chase(pi + a);
        while (b != a) {
          pi[v] = b;
          ++steps;
          a = b;
          b = ld_chase(pi + a);
        }
      }
      byte |= (a == star) ? 1u << (u32)(v - v0) : 0u;
    }
  }
  return byte;
}

// Store the bitmap words and star summary of one 2048-vertex chunk (one
// block's groups; byte = this thread's 8 bits).  Uniform per block.
__device__ __forceinline__ void emit_bits(u64 chunk, u64 n, u64 v0, u32 byte, u32* bits,
                                          u32* sum, u32 sum_words, u32 sum_shift,
                                          u32* s_full) {
  // four lanes = one 32-vertex word
  const u32 lane = threadIdx.x & 31u;
  u32 w = byte << (8u * (lane & 3u));
  w |= __shfl_xor_sync(0xffffffffu, w, 1);
  w |= __shfl_xor_sync(0xffffffffu, w, 2);
  if ((lane & 3u) == 0 && v0 < n) bits[v0 >> 5] = w;
  if (!sum) return;
  if (sum_shift == kSumHalfShift) {
    // one bit per 16 vertices = two neighbouring threads' bytes all in the
    // star: one ballot, then the pairs' bits packed into the warp's 16-bit
    // summary halfword (was eight shuffles)
    const u32 f8 = __ballot_sync(0xffffffffu, v0 < n && byte == 0xffu);
    u32 x = f8 & (f8 >> 1) & 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0f0f0f0fu;
    x = (x | (x >> 4)) & 0x00ff00ffu;
    x = (x | (x >> 8)) & 0x0000ffffu;
    const u64 hw_idx = (chunk * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0 && hw_idx < (u64)sum_words * 2)
      reinterpret_cast<unsigned short*>(sum)[hw_idx] = (unsigned short)x;
    return;
  }
  // Star-0 summary: this chunk's 64 words -> 64 >> sum_shift bits (bit =
  // every word of its group is all ones).  Groups shared with other chunks
  // are merged with atomics (clear, then set), whole summary words stored.
  const u32 full = __ballot_sync(0xffffffffu, (lane & 3u) == 0 && v0 < n && w == ~0u);
  // bit j = word (warp * 8 + j) is all ones: every 4th bit of `full`
  u32 b8 = full & 0x11111111u;
  b8 = (b8 | (b8 >> 3)) & 0x03030303u;
  b8 = (b8 | (b8 >> 6)) & 0x000f000fu;
  b8 = (b8 | (b8 >> 12)) & 0xffu;
  if (sum_shift == 0) {
    // one summary bit per word: a warp's 8 words are one summary byte
    const u64 byte_idx = (chunk * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0 && byte_idx < (u64)sum_words * 4)
      reinterpret_cast<unsigned char*>(sum)[byte_idx] = (unsigned char)b8;
    return;
  }
  if (lane == 0) s_full[threadIdx.x >> 5] = b8;
  __syncthreads();
  // a 64-word chunk is 8 warps (256 threads); a wider block holds several,
  // the first lane of each chunk's first warp assembles it
  if ((threadIdx.x & 255u) == 0 && (blockDim.x & 255u) == 0) {
    const u32 c8 = threadIdx.x >> 5;
    chunk = chunk * (blockDim.x >> 8) + (threadIdx.x >> 8);
    u64 f = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) f |= (u64)s_full[c8 + i] << (8 * i);
    const u32 g = 1u << sum_shift, nb = 64u >> sum_shift;
    u64 bitsg = 0;
    for (u32 i = 0; i < nb; ++i) {
      const u64 mask = (g == 64 ? ~0ull : ((1ull << g) - 1)) << (i * g);
      if ((f & mask) == mask) bitsg |= 1ull << i;
    }
    const u64 pos = chunk * nb;  // first summary bit of this chunk
    if (nb >= 32) {
      for (u32 k = 0; k < nb / 32; ++k)
        if ((pos >> 5) + k < sum_words) sum[(pos >> 5) + k] = (u32)(bitsg >> (32 * k));
    } else if ((pos >> 5) < sum_words) {
      // this chunk owns nb bits of a shared word: clear, then set (the
      // star may have moved since the last compress)
      const u32 mask = (u32)((1ull << nb) - 1) << (pos & 31);
      const u32 val = (u32)bitsg << (pos & 31);
      if (~val & mask) atomicAnd(sum + (pos >> 5), ~(mask & ~val));
      if (val) atomicOr(sum + (pos >> 5), val);
    }
  }
}

// Multi-Jump compress fused with the star-0 bitmap build (HC engine, full
// grid): thread q owns vertices [8q, 8q+8); after the chases every thread
// knows its vertices' roots, so bit v = (root(v) == star) is assembled with
// two warp shuffles (4 lanes = one 32-vertex word) and stored once.
#ifndef HCC_COMP_MINB
#define HCC_COMP_MINB 6
#endif
template <int BS>
__device__ __forceinline__ void compress_s0b_body(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                                                  u32* bits, int mode, u32* sum, u32 sum_words,
                                                  u32 sum_shift, int rec_idx, int dslot,
                                                  u32 pf_blocks);

__global__ void __launch_bounds__(kVertThreads, HCC_COMP_MINB)
    k_compress_s0b(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs, u32* bits,
                   int mode, u32* sum, u32 sum_words, u32 sum_shift, int rec_idx, int dslot,
                   u32 pf_blocks) {
  compress_s0b_body<kVertThreads>(pi, n, ctrl, recs, bits, mode, sum, sum_words, sum_shift,
                                  rec_idx, dslot, pf_blocks);
}

// 512-thread blocks, half as many (HCC_COMP_WIDE=1; off by default): at
// n = 2^28 a compress is 131 K blocks of 256 threads that each read 8 KB of
// pi, which suggested block turnover as the bound; measured, it is not
// (RMAT-28 33.89 vs 33.81 ms, adaptive 41.7 vs 40.7 ms).
__global__ void __launch_bounds__(kVertThreadsWide, 3)
    k_compress_s0b_w(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs, u32* bits,
                     int mode, u32* sum, u32 sum_words, u32 sum_shift, int rec_idx, int dslot,
                     u32 pf_blocks) {
  compress_s0b_body<kVertThreadsWide>(pi, n, ctrl, recs, bits, mode, sum, sum_words, sum_shift,
                                      rec_idx, dslot, pf_blocks);
}

template <int BS>
__device__ __forceinline__ void compress_s0b_body(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs,
                                                  u32* bits, int mode, u32* sum, u32 sum_words,
                                                  u32 sum_shift, int rec_idx, int dslot,
                                                  u32 pf_blocks) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->tile_ctr = 0;  // next hook's schedule
  if (dslot >= 0) {
    // unrolled chain: this segment's flag; clear the next segment's
    if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->dirtyp[dslot ^ 1] = 0;
    if (mode && __ldg(&ctrl->dirtyp[dslot]) == 0) return;
  } else if (mode && __ldg(&ctrl->dirty) == 0) {
    return;
  }
  DevRec* r = rec_of(ctrl, recs, rec_idx);
  block_t0(&r->comp_t0);
  u64 steps = 0;
  // Two 16-byte reads and eight parent gathers in flight before any chase
  // (ascending order is kept: a thread's vertices are consecutive and
  // blocks start in ascending order).  The bitmap tracks the star rooted
  // at ctrl->star: k_star_pick resolved it after the last hook (vertex 0,
  // the initial star, is never hooked).  Should it have been hooked since
  // (a slot without a pick), no root equals it and this bitmap is empty.
  const u32 star = __ldg(&ctrl->star);
  const u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 v0 = q << 3;
  const bool whole = v0 + 8 <= n;
  uint4 pa = make_uint4(0u, 0u, 0u, 0u), pb = pa;
  if (whole) {
    const uint4* p4 = reinterpret_cast<const uint4*>(pi) + (q << 1);
    pa = __ldcg(p4);
    pb = __ldcg(p4 + 1);
  }
  // pi larger than L2 (n >= 2^26): pull the line the block pf_blocks later
  // in launch order (about one residency wave ahead) will read into L2, so
  // its first read does not wait on DRAM
  if (pf_blocks && (threadIdx.x & 3u) == 0) {
    const u64 vn = v0 + ((u64)pf_blocks * BS << 3);
    if (vn + 8 <= n) asm volatile("prefetch.global.L2 [%0];" ::"l"(pi + vn));
  }
  // the star's root is read once per thread (one L1 line for the grid):
  // a compress never moves a root, so the answer holds for the whole pass
  const bool star_root = star < n && ld_pi(pi + star) == star;
  const u32 byte = compress8(pi, n, v0, whole, pa, pb, star, star_root, steps);
  __shared__ u32 s_full[BS / 32];
  emit_bits(blockIdx.x, n, v0, byte, bits, sum, sum_words, sum_shift, s_full);
  add_counter(&r->jump_stripe[blockIdx.x & (kJumpStripes - 1)], steps);
  block_t1(&r->comp_t1);
}

// Sixteen vertices per thread (four 16-byte reads in flight): the control
// reads, index math and bitmap emission are paid once per 16 vertices, and
// a settled group of 16 (the common case once the giant is a star) is one
// compare chain.  Otherwise the two halves run compress8 one after the
// other (the second sees the first's writes).  Serves the star summaries
// whose bits map onto a warp without block merging: none, one bit per word,
// one bit per 16 vertices.
__device__ __forceinline__ void emit_bits16(u64 q, u64 n, u64 v0, u32 b16, u32* bits, u32* sum,
                                            u32 sum_words, u32 sum_shift) {
  const u32 lane = threadIdx.x & 31u;
  u32 w = b16 << (16u * (lane & 1u));
  w |= __shfl_xor_sync(0xffffffffu, w, 1);
  if ((lane & 1u) == 0 && v0 < n) bits[v0 >> 5] = w;
  if (!sum) return;
  if (sum_shift == kSumHalfShift) {
    // one bit per 16 vertices = one bit per thread: a warp is one word
    const u32 ball = __ballot_sync(0xffffffffu, v0 < n && b16 == 0xffffu);
    if (lane == 0 && (q >> 5) < sum_words) sum[q >> 5] = ball;
    return;
  }
  // one bit per word (two lanes): a warp's 16 words are one halfword
  u32 x = __ballot_sync(0xffffffffu, (lane & 1u) == 0 && v0 < n && w == ~0u) & 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0f0f0f0fu;
  x = (x | (x >> 4)) & 0x00ff00ffu;
  x = (x | (x >> 8)) & 0x0000ffffu;
  if (lane == 0 && (q >> 5) < (u64)sum_words * 2)
    reinterpret_cast<unsigned short*>(sum)[q >> 5] = (unsigned short)x;
}

#ifndef HCC_COMP16_MINB
#define HCC_COMP16_MINB 4
#endif
__global__ void __launch_bounds__(kVertThreads, HCC_COMP16_MINB)
    k_compress_s0b16(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs, u32* bits, int mode, u32* sum,
                     u32 sum_words, u32 sum_shift, int rec_idx, int dslot, u32 pf_blocks) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->tile_ctr = 0;  // next hook's schedule
  if (dslot >= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->dirtyp[dslot ^ 1] = 0;
    if (mode && __ldg(&ctrl->dirtyp[dslot]) == 0) return;
  } else if (mode && __ldg(&ctrl->dirty) == 0) {
    return;
  }
  DevRec* r = rec_of(ctrl, recs, rec_idx);
  block_t0(&r->comp_t0);
  u64 steps = 0;
  const u32 star = __ldg(&ctrl->star);
  const u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 v0 = q << 4;
  const bool whole = v0 + 16 <= n;
  uint4 pa = make_uint4(0u, 0u, 0u, 0u), pb = pa, pc = pa, pd = pa;
  if (whole) {
    const uint4* p4 = reinterpret_cast<const uint4*>(pi) + (q << 2);
    pa = __ldcg(p4);
    pb = __ldcg(p4 + 1);
    pc = __ldcg(p4 + 2);
    pd = __ldcg(p4 + 3);
  }
  if (pf_blocks && (threadIdx.x & 1u) == 0) {
    const u64 vn = v0 + ((u64)pf_blocks * kVertThreads << 4);
    if (vn + 16 <= n) asm volatile("prefetch.global.L2 [%0];" ::"l"(pi + vn));
  }
  const bool star_root = star < n && ld_pi(pi + star) == star;
  u32 b16 = 0;
  bool done = false;
  if (whole && star_root) {
    const u32 a[16] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w,
                       pc.x, pc.y, pc.z, pc.w, pd.x, pd.y, pd.z, pd.w};
    u32 settled = 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      settled &= (a[j] == (u32)v0 + j) | (a[j] == star);
      b16 |= (u32)(a[j] == star) << j;
    }
    done = settled != 0;
  }
  if (!done) {
    const u32 lo = compress8(pi, n, v0, v0 + 8 <= n, pa, pb, star, star_root, steps);
    const u32 hi = compress8(pi, n, v0 + 8, whole, pc, pd, star, star_root, steps);
    b16 = lo | (hi << 8);
  }
  emit_bits16(q, n, v0, b16, bits, sum, sum_words, sum_shift);
  add_counter(&r->jump_stripe[blockIdx.x & (kJumpStripes - 1)], steps);
  block_t1(&r->comp_t1);
}

// Single-level jump pass (forest.hpp:93-99) with a device change flag.
__global__ void __launch_bounds__(kVertThreads)
    k_jump(u32* pi, u64 n, DevCtrl* ctrl, DevRec* recs) {
  DevRec* r = cur_rec(ctrl, recs);
  block_t0(&r->comp_t0);
  u64 steps = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    u32 p = ld_fresh(pi + v);
    u32 gp = ld_fresh(pi + p);
    if (gp != p) {
      pi[v] = gp;
      ++steps;
    }
  }
  if (__syncthreads_or(steps != 0) && threadIdx.x == 0) ctrl->jchanged = 1;
  add_counter(&r->jump_stripe[blockIdx.x & (kJumpStripes - 1)], steps);
  block_t1(&r->comp_t1);
}

// ---- loop-step kernels (single thread) ------------------------------------

__device__ __forceinline__ u32 guard(DevCtrl* c, u32 cond) {
  if (++c->loop_steps > kMaxLoopSteps) {
    c->err |= 2u;
    return 0u;
  }
  return cond;
}

__global__ void k_set_cond(cudaGraphConditionalHandle h, u32 value) {
  cudaGraphSetConditional(h, value);
}

// Worklist pass finished: the output becomes the next input.
__global__ void k_step_worklist(DevCtrl* c, DevRec* recs,
                                cudaGraphConditionalHandle h, int use_cond) {
  const u32 in = c->parity, out = in ^ 1u;
  const u64 produced = c->wl_count[out];
  c->parity = out;
  c->wl_count[in] = 0;
  c->passes += 1;
  c->dirty = 0;
  next_rec(c, recs);
  // a worklist overflow ends the run (the host re-runs with full-size lists)
  const u32 cond = guard(c, produced > 0 && !(c->err & 4u) ? 1u : 0u);
  c->cond = cond;
  if (use_cond) cudaGraphSetConditional(h, cond);
}

// Segment finished (topology pass / adaptive segments).
__global__ void k_step_segment(DevCtrl* c, DevRec* recs,
                               cudaGraphConditionalHandle h, int use_cond) {
  c->seg += 1;
  c->passes += 1;
  c->dirty = 0;
  next_rec(c, recs);
  const u32 cond = guard(c, c->seg < c->nseg ? 1u : 0u);
  c->cond = cond;
  if (use_cond) cudaGraphSetConditional(h, cond);
}

// Adaptive segment finished: choose the next range from this segment's
// store ratio (records are per segment).
__global__ void k_step_adapt(DevCtrl* c, DevRec* recs, u64 m, u32 forming_pct,
                             const u32* sum, u32 sum_words, const uint2* edges,
                             const u32* bits, const u32* rsum, u32 rshift, int rany) {
  // Every thread derives the next range from the pass-start control words
  // (same addresses: broadcast reads), so the sample loads below issue
  // without waiting for thread 0's bookkeeping; thread 0 writes after the
  // barrier, once every thread has read.
  const u32 ri = c->rec < (u32)kMaxRecs ? c->rec : (u32)kMaxRecs - 1;
  const u64 r_in = recs[ri].edges_in, r_out = recs[ri].edges_out;
  const u64 seg = c->seg, nseg = c->nseg, old_b = c->seg_b, old_e = c->seg_e;
  const u64 len = old_e - old_b;
  // (forming_pct bits 8-15: the growth factor, 0 = kAdaptGrowth)
  const u32 growth = (forming_pct >> 8) & 0xffu ? (forming_pct >> 8) & 0xffu : kAdaptGrowth;
  const bool forming = r_in > 0 && r_out * 100 > r_in * (forming_pct & 0xffu);
  u64 next = forming ? len * growth : m;
  if (next < 1) next = 1;
  if (seg + 2 >= nseg) next = m;  // the next slot is the last one
  const u64 s_b = old_e;
  const u64 s_e = (m - s_b) <= next ? m : s_b + next;
  // Bitmap use for the next hook (one block): a lookup pays only when it
  // usually answers; the share of the next segment's endpoints in the star
  // decides (RMAT: 81-98% with hub words L1-resident; ER's giant at 37%
  // made its bitmap lookups a net loss, 0.63 vs 0.51 ms).
  const bool sample = blockDim.x > 1 && bits && s_e > s_b;
  uint2 ed = make_uint2(0u, 0u);
  if (sample) {
    u64 hsh = (((seg + 1) << 32) + threadIdx.x + 1) * 0x9E3779B97F4A7C15ull;
    hsh ^= hsh >> 29;
    hsh *= 0xBF58476D1CE4E5B9ull;
    hsh ^= hsh >> 32;
    ed = edges[s_b + hsh % (s_e - s_b)];
  }
  if (blockDim.x > 1) __syncthreads();
  if (threadIdx.x == 0) {
    c->seg_b = s_b;
    c->seg_e = s_e;
    c->seg = seg + 1;
    if (rsum) c->use_sum = 0u;  // set below for the remainder slot
    c->passes += (len > 0);
    c->dirty = 0;
    next_rec(c, recs);
  }
  if (blockDim.x == 1) return;
  if (sample) {
    const u32 hits = ((bits[ed.x >> 5] >> (ed.x & 31u)) & 1u) + ((bits[ed.y >> 5] >> (ed.y & 31u)) & 1u);
    const int n_hit = __syncthreads_count(hits == 2) * 2 + __syncthreads_count(hits == 1);
    if (threadIdx.x == 0) c->use_bits = (u32)n_hit * 2 >= 2 * blockDim.x ? 1u : 0u;
    // The slot that takes every remaining edge (the steady regime) streams
    // with summary-predicated lookups (k_hook_sumd) when the summary
    // answers at least a quarter of its sampled endpoints (RMAT-24: 63%;
    // RMAT-28 with one bit per 16 words: little, and the kernel's 64 KB of
    // shared memory would only cost L1); otherwise the plain hook.
    if (rsum) {
      const u32 gx = ed.x >> (5u + rshift), gy = ed.y >> (5u + rshift);
      const u32 cov = ((rsum[gx >> 5] >> (gx & 31u)) & 1u) + ((rsum[gy >> 5] >> (gy & 31u)) & 1u);
      const int n_cov = __syncthreads_count(cov == 2) * 2 + __syncthreads_count(cov == 1);
      if (threadIdx.x == 0 && (s_e == m || rany))
        c->use_sum = (u32)n_cov * 4 >= 2 * blockDim.x ? 1u : 0u;
    }
  }
  // Star summary vote for the next hook launch: the summary path pays off
  // when at least half of the groups are covered.
  if (sum) {
    __shared__ u32 s_cov;
    if (threadIdx.x == 0) s_cov = 0;
    __syncthreads();
    // 16-byte loads, four in flight per thread (the table is 64 KB at most;
    // a serial word loop was ~10 us of the step)
    u32 cov = 0;
    const uint4* s4 = reinterpret_cast<const uint4*>(sum);
    const u32 n4 = sum_words / 4;
    for (u32 i = threadIdx.x; i < n4; i += 4 * blockDim.x) {
      uint4 q[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const u32 k = i + (u32)j * blockDim.x;
        q[j] = k < n4 ? __ldg(s4 + k) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) cov += __popc(q[j].x) + __popc(q[j].y) + __popc(q[j].z) + __popc(q[j].w);
    }
    for (u32 i = n4 * 4 + threadIdx.x; i < sum_words; i += blockDim.x) cov += __popc(sum[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cov += __shfl_xor_sync(0xffffffffu, cov, o);
    if ((threadIdx.x & 31u) == 0 && cov) atomicAdd(&s_cov, cov);
    __syncthreads();
    if (threadIdx.x == 0) c->use_sum = (u64)s_cov * 2 >= (u64)sum_words * 32 ? 1u : 0u;
  }
}

// Baseline outer iteration finished: loop while some hook changed.
__global__ void k_step_outer(DevCtrl* c, DevRec* recs,
                             cudaGraphConditionalHandle h, int use_cond) {
  const u32 cond = guard(c, c->changed ? 1u : 0u);
  c->changed = 0;
  c->passes += 1;
  c->dirty = 0;
  next_rec(c, recs);
  c->cond = cond;
  if (use_cond) cudaGraphSetConditional(h, cond);
}

// Baseline inner jump loop: repeat while a jump changed a slot.
__global__ void k_step_jump(DevCtrl* c, cudaGraphConditionalHandle h,
                            int use_cond) {
  const u32 cond = guard(c, c->jchanged ? 1u : 0u);
  c->jchanged = 0;
  c->cond = cond;
  if (use_cond) cudaGraphSetConditional(h, cond);
}

// ---- reductions -----------------------------------------------------------

__global__ void k_count_roots(const u32* pi, u64 n, DevCtrl* ctrl) {
  u64 cnt = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    cnt += (pi[v] == (u32)v);
  add_counter(&ctrl->components, cnt);
}

// *flag != 0 iff some v has pi(pi(v)) != pi(v).
__global__ void k_is_star(const u32* pi, u64 n, u32* flag) {
  u32 bad = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    u32 p = pi[v];
    bad |= (pi[p] != p);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// *flag != 0 iff some v has pi(v) > v.
__global__ void k_check_bound(const u32* pi, u64 n, u32* flag) {
  u32 bad = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    bad |= (pi[v] > (u32)v);
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// ---- element kernels for the ParentForest API ------------------------------
// One device thread; results in res[0..3]: res[0] = value / changed / steps,
// res[1] = ok / cas failures, res[2] = jump steps.
__global__ void k_elem(u32* pi, int op, u64 a, u64 b, u64 c, u64* res) {
  volatile u32* vp = pi;
  u64 r0 = 0, r1 = 0, r2 = 0;
  switch (op) {
    case kOpLoad:
      r0 = vp[a];
      break;
    case kOpStore:
      vp[a] = (u32)b;
      break;
    case kOpCas: {
      u32 old = atomicCAS(pi + a, (u32)b, (u32)c);
      r0 = old;
      r1 = old == (u32)b;
      break;
    }
    case kOpHook: {  // forest.hpp:83-89
      u32 pu = vp[a], pv = vp[b];
      if (pu != pv) {
        vp[max(pu, pv)] = min(pu, pv);
        r0 = 1;
      }
      break;
    }
    case kOpJump: {  // forest.hpp:93-99
      u32 p = vp[a], gp = vp[p];
      if (gp != p) {
        vp[a] = gp;
        r0 = 1;
      }
      break;
    }
    case kOpAtomicHook: {  // forest.hpp:107-122
      u32 u = (u32)a, v = (u32)b;
      for (;;) {
        u32 pu = vp[u], pv = vp[v];
        if (pu == pv) break;
        ++r0;
        u32 h = max(pu, pv), l = min(pu, pv);
        u32 old = atomicCAS(pi + h, h, l);
        if (old == h) break;
        ++r1;
        u = old;
        v = l;
      }
      break;
    }
    case kOpMultiJump:
    case kOpMultiJumpRange: {  // forest.hpp:127-136
      u64 lo = a, hi = op == kOpMultiJump ? a + 1 : b;
      const bool desc = op == kOpMultiJumpRange && c != 0;
      for (u64 k = 0; k < hi - lo; ++k) {
        u64 v = desc ? hi - 1 - k : lo + k;
        u32 p = vp[v];
        for (;;) {
          u32 gp = vp[p];
          if (gp == p) break;
          vp[v] = gp;
          ++r2;
          p = gp;
        }
      }
      break;
    }
    default:
      break;
  }
  res[0] = r0;
  res[1] = r1;
  res[2] = r2;
}

}  // namespace hcc
