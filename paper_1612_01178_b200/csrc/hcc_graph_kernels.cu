// Ingestion, generator and checksum kernels.  Input production is outside
// the reference timing boundary (bench.hpp:163-167): these run
// when a graph handle is created, never inside hcc_cc's timed region.
#include <cuda_runtime.h>

#include "hookcc_gen.h"
#include "hcc_internal.cuh"

namespace hcc {

// u64 (u, v) pairs -> packed u32 pairs with check_endpoints semantics
// (graph.hpp:89-94): err bit 1 on an endpoint >= n.
__global__ void k_narrow_u64(const u64* uv, uint2* out, u64 m, u64 n,
                             u32* err) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u32 bad = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    u64 u = uv[2 * i], v = uv[2 * i + 1];
    bad |= (u >= n) | (v >= n);
    out[i] = make_uint2((u32)u, (u32)v);
  }
  if (bad) atomicOr(err, 1u);
}

__global__ void k_check_u32(const uint2* e, u64 m, u64 n, u32* err) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u32 bad = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    uint2 x = e[i];
    bad |= ((u64)x.x >= n) | ((u64)x.y >= n);
  }
  if (bad) atomicOr(err, 1u);
}

// CSR -> edge records in row order: entry j of row u becomes (u, col[j]).
// The row of entry j is found by binary search over row_ptr.
__global__ void k_csr_expand(const u64* row_ptr, const u32* col, u64 n,
                             uint2* out, u64 m, u32* err) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u32 bad = 0;
  for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    // largest u with row_ptr[u] <= j
    u64 lo = 0, hi = n;  // invariant: row_ptr[lo] <= j < row_ptr[hi]
    while (hi - lo > 1) {
      u64 mid = (lo + hi) >> 1;
      if (row_ptr[mid] <= j) lo = mid; else hi = mid;
    }
    u32 c = col[j];
    bad |= ((u64)c >= n);
    out[j] = make_uint2((u32)lo, c);
  }
  if (bad) atomicOr(err, 1u);
}

__global__ void k_gen_grid(uint2* out, u64 rows, u64 cols, u64 first, u64 count) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    u32 u, v;
    grid_edge(rows, cols, first + i, &u, &v);
    out[i] = make_uint2(u, v);
  }
}

__global__ void k_gen_rmatx(uint2* out, u64 first, u64 count, u32 scale,
                            u64 seed, u32 ta, u32 tab, u32 tabc) {
  const u64 key = gen_key(seed);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    u32 u, v;
    rmatx_edge(key, first + i, scale, ta, tab, tabc, &u, &v);
    out[i] = make_uint2(u, v);
  }
}

__global__ void k_gen_erx(uint2* out, u64 first, u64 count, u64 n, u64 seed) {
  const u64 key = gen_key(seed);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    u32 u, v;
    erx_edge(key, first + i, n, &u, &v);
    out[i] = make_uint2(u, v);
  }
}

__global__ void k_checksum(const uint2* e, u64 m, u64 base, u64* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 s = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    uint2 x = e[i];
    s += checksum_term(base + i, x.x, x.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31u) == 0) atomicAdd(out, s);
}

__global__ void k_verify_edges(const uint2* e, u64 m, const u32* pi, u64* bad) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 cnt = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 x = e[i];
    cnt += __ldcg(pi + x.x) != __ldcg(pi + x.y);
  }
  if (cnt) atomicAdd(bad, cnt);
}

__global__ void k_verify_canonical(const u32* pi, u64 n, u64* bad) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 cnt = 0;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    const u32 l = __ldcg(pi + v);
    cnt += (l > (u32)v) || (__ldcg(pi + l) != l);
  }
  if (cnt) atomicAdd(bad, cnt);
}

// keys[i] = a[i] << 32 | b[i]; diff counts label mismatches (exactness)
__global__ void k_pair_keys(const u32* a, const u32* b, u64 n, u64* keys, u64* diff) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 cnt = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    keys[i] = ((u64)a[i] << 32) | b[i];
    cnt += a[i] != b[i];
  }
  if (cnt) atomicAdd(diff, cnt);
}

// distinct counts over sorted keys: [0] pairs, [1] first components
__global__ void k_count_distinct(const u64* k, u64 n, int shift, u64* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 cnt = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 x = shift ? (k[i] >> shift) : k[i];
    cnt += i == 0 || (shift ? (k[i - 1] >> shift) : k[i - 1]) != x;
  }
  if (cnt) atomicAdd(out, cnt);
}

}  // namespace hcc
