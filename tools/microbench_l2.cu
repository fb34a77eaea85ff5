// Microbenchmark: does a 32 MiB random-lookup table (RMAT-28's star bitmap)
// stay L2-resident while a persistent kernel streams a 32 GiB array through
// L2 with an evict-first policy (the steady hook's edge stream)?
//   mode 0: stream only (16-byte evict-first loads)
//   mode 1: stream + 2 random 4-byte lookups per 8 streamed bytes into the table
//   mode 2: lookups only (same count as mode 1)
// Prints ms and the lookup rate; compare with ncu's lts hit rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_l2 tools/microbench_l2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint4 ld16(const uint4* p, unsigned long long pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__global__ void k_bench(const uint4* stream, unsigned long long n16, const unsigned* table,
                        unsigned mask_words, int mode, unsigned* out) {
  const unsigned long long pol = pol_first();
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (unsigned long long i = tid; i < n16; i += stride) {
    uint4 q = make_uint4((unsigned)i * 2654435761u, (unsigned)(i >> 7) * 40503u, (unsigned)i ^ 0x9e3779b9u,
                         (unsigned)i * 97u);
    if (mode != 2) q = ld16(stream + i, pol);
    if (mode == 0) {
      acc += q.x ^ q.w;
      continue;
    }
    // 4 lookups per 16 bytes (2 per 8-byte edge), RMAT-like skew: a third
    // of them into the first 1/16 of the table
    // keys: the streamed words mixed with the position (the stream's
    // contents are constant here)
    unsigned k[4] = {q.x ^ (unsigned)i * 2246822519u, q.y ^ (unsigned)(i >> 3) * 3266489917u,
                     q.z ^ (unsigned)i * 668265263u, q.w ^ (unsigned)(i * 374761393u + 7u)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned h = k[j] * 2654435761u;
      unsigned w = (h % 3u == 0u) ? ((h >> 4) & (mask_words >> 4)) : ((h >> 2) & mask_words);
      acc += __ldg(table + w);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
  const unsigned long long bytes = 32ull << 30;
  const unsigned table_words = (32u << 20) / 4;  // 32 MiB
  uint4* stream = nullptr;
  unsigned *table = nullptr, *out = nullptr;
  if (cudaMalloc(&stream, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&table, table_words * 4ull);
  cudaMalloc(&out, 4);
  cudaMemset(stream, 1, bytes);
  cudaMemset(table, 2, table_words * 4ull);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned long long n16 = bytes / 16;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_bench<<<sms * 2, 1024>>>(stream, n16, table, table_words - 1, mode, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("mode %d: %.3f ms  stream %.1f GB/s  lookups %.1f G/s\n", mode, ms,
               mode == 2 ? 0.0 : bytes / (ms * 1e-3) / 1e9,
               mode == 0 ? 0.0 : n16 * 4 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
