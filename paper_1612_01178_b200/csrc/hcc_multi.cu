// Multi-GPU merge kernels (north-star (5); SURVEY.md §8e shape 3).
//
// Each rank runs the single-GPU engine on its partition_edges(m, world)
// shard (engines.hpp:43-58 semantics) into a full local forest.  The forest
// of a rank is a set of stars, so it is fully described by the pairs
// (v, pi(v)) with pi(v) != v.  On skewed graphs almost all of those point at
// vertex 0 (the giant component's minimum), so the export is split into
//   bits  : bit v = (pi(v) == 0 && v != 0)          n/8 bytes, dense
//   pairs : (v, pi(v)) for pi(v) not in {v, 0}      8 bytes each, sparse
// The host exchanges the payloads (NCCL allgather through torch.distributed
// in bench.py; any transport works) and hcc_rehook re-hooks the remote
// relations into the local forest as edges, with the same worklist kernels
// as the single-GPU engine.  One exchange round suffices: after it every
// rank holds the union of all shards' relations.
#include <cuda_runtime.h>

#include "hcc_internal.cuh"

namespace hcc {

namespace {

// Warp-aggregated append of one pair per active lane; returns via `pos`.
__device__ __forceinline__ void warp_append(bool want, uint2 pr, uint2* out, u64 cap,
                                            u64* count) {
  const u32 mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return;
  const u32 lane = threadIdx.x & 31u;
  u64 base = 0;
  if (lane == 0) base = atomicAdd(count, (u64)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (want) {
    const u64 pos = base + __popc(mask & ((1u << lane) - 1u));
    if (pos < cap) out[pos] = pr;
  }
}

}  // namespace

// One warp per 32-vertex word, four words per round (four 128-byte reads in
// flight per warp).  Requires blockDim.x % 32 == 0.
__global__ void k_export(const u32* pi, u64 n, u32* bits, uint2* pairs, u64 cap,
                         u64* count) {
  constexpr u32 kW = 4;
  const u32 lane = threadIdx.x & 31u;
  const u64 nwords = (n + 31) >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w0 = (((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kW; w0 < nwords;
       w0 += warps * kW) {
    u32 p[kW];
#pragma unroll
    for (u32 k = 0; k < kW; ++k) {
      const u64 v = ((w0 + k) << 5) + lane;
      p[k] = v < n ? __ldcg(pi + v) : (u32)v;
    }
#pragma unroll
    for (u32 k = 0; k < kW; ++k) {
      if (w0 + k >= nwords) break;  // warp-uniform
      const u64 v = ((w0 + k) << 5) + lane;
      const u32 b = __ballot_sync(0xffffffffu, v < n && v != 0 && p[k] == 0u);
      if (lane == 0) bits[w0 + k] = b;
      warp_append(v < n && p[k] != (u32)v && p[k] != 0u, make_uint2((u32)v, p[k]), pairs, cap,
                  count);
    }
  }
}

// Append (v, 0) for every v set in the OR of the remote bitmaps that is not
// already in the local star of 0.
__global__ void k_decode_bits(const u32* rows, u64 nrows, u64 stride, u64 skip, const u32* pi,
                              u64 n, uint2* wl, u64* count) {
  // bit v of the OR over the gathered rows (every rank's bitmap but this
  // one's: `skip`), decoded to (v, 0) worklist edges where v is not yet in 0
  constexpr u32 kW = 4;
  const u32 lane = threadIdx.x & 31u;
  const u64 nwords = (n + 31) >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w0 = (((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kW; w0 < nwords;
       w0 += warps * kW) {
    u32 b[kW] = {0u, 0u, 0u, 0u};
    for (u64 r = 0; r < nrows; ++r) {
      if (r == skip) continue;
#pragma unroll
      for (u32 k = 0; k < kW; ++k)
        if (w0 + k < nwords) b[k] |= rows[r * stride + w0 + k];
    }
#pragma unroll
    for (u32 k = 0; k < kW; ++k) {
      if (b[k] == 0u) continue;  // warp-uniform
      const u64 v = ((w0 + k) << 5) + lane;
      const bool want = ((b[k] >> lane) & 1u) && v < n && __ldcg(pi + v) != 0u;
      warp_append(want, make_uint2((u32)v, 0u), wl, ~0ull, count);
    }
  }
}

// Fused exchange + decode of the single-process multi-device merge
// (hcc_create_multi): rank r's kernel reads every peer's export buffers
// directly over NVLink (peer access; shards on the same device read plain
// device memory), so no payload is staged and no host reads a size:
//   * bitmaps  OR of the peers' rows, 32 words per warp round; a set bit
//              whose vertex is not yet in r's star of 0 links its root to 0
//              in place;
//   * pairs    the peers' (v, parent) pairs, count read from peer memory;
//              pairs already joined in r's forest (pi(v) == pi(parent): the
//              forest is a set of stars after the local CC) are dropped.
// Records go to r's worklist; the worklist engine then re-hooks them.
__global__ void k_merge_gather(const PeerTab* tab, u32 self, u32* pi, u64 n, uint2* wl,
                               u64* count, u64 cap, u32* err, u32* dirty, u64* linked) {
  const u32 lane = threadIdx.x & 31u;
  const u32 np = tab->npeers;
  const u64 nwords = (n + 31) >> 5;
  const u64 gwarp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  // 32 words per warp round: lane j ORs word w0 + j of every peer row (one
  // 128-byte read per peer), then the warp decodes the words one by one
  for (u64 w0 = gwarp * 32; w0 < nwords; w0 += warps * 32) {
    u32 x = 0;
    if (w0 + lane < nwords) {
      for (u32 r = 0; r < np; ++r)
        if (r != self) x |= __ldcg(tab->bits[r] + w0 + lane);
      // vertices already in this rank's star of 0 (its own exported row)
      // need nothing: their pi is not even read (at 8 GPUs on RMAT-28 about
      // half of the peers' star members)
      x &= ~__ldcg(tab->bits[self] + w0 + lane);
    }
    // Every set bit is a vertex of the global star of 0.  The local forest
    // is a set of stars (a converged local CC, or the end of a re-hook
    // pass), so pi(v) is v's root: link that root to 0 in place (every
    // writer stores the same value 0, the minimum id, so the races are
    // benign and pi(x) <= x holds).  No worklist records: at 8 GPUs on
    // RMAT-28 each rank learned ~61 M vertices this way, and re-hooking them
    // as (v, 0) records cost a worklist pass over all of them.  Eight words'
    // pi reads in flight per group.
    u32 links = 0;
    for (u32 k0 = 0; k0 < 32; k0 += 8) {
      u32 b[8], p[8];
#pragma unroll
      for (u32 j = 0; j < 8; ++j) {
        b[j] = __shfl_sync(0xffffffffu, x, k0 + j);
        const u64 v = ((w0 + k0 + j) << 5) + lane;
        p[j] = ((b[j] >> lane) & 1u) && v < n ? __ldcg(pi + v) : 0u;
      }
#pragma unroll
      for (u32 j = 0; j < 8; ++j)
        if (p[j] != 0u) {
          pi[p[j]] = 0u;
          ++links;
        }
    }
    if (__any_sync(0xffffffffu, links != 0)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xffffffffu, links, o);
      if (lane == 0) {
        atomicAdd(linked, (u64)links);
        *dirty = 1u;
      }
    }
  }
  // pairs: one global index space over the peers' lists
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u32 r = 0; r < np; ++r) {
    if (r == self) continue;
    u64 k = __ldcg(tab->count[r]);
    if (k > tab->cap[r]) k = tab->cap[r];  // the host detects the overflow
    const uint2* pr = tab->pairs[r];
    for (u64 i = tid; i < ((k + 31) & ~31ull); i += stride) {
      uint2 x = make_uint2(0u, 0u);
      bool want = false;
      if (i < k) {
        x = __ldcg(pr + i);
        want = x.x < n && x.y < n && __ldcg(pi + x.x) != __ldcg(pi + x.y);
      }
      const u32 mask = __ballot_sync(0xffffffffu, want);
      if (!mask) continue;
      u64 base = 0;
      if (lane == 0) base = atomicAdd(count, (u64)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (want) {
        const u64 pos = base + __popc(mask & ((1u << lane) - 1u));
        if (pos < cap)
          wl[pos] = x;
        else
          atomicOr(err, 4u);
      }
    }
  }
}

}  // namespace hcc
