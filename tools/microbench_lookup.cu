// Microbenchmark: random 4-byte lookup throughput on B200 from
//   (a) a 2 MiB global array (the star-0 bitmap; L1/L2 resident),
//   (b) distributed shared memory of an 8-CTA cluster (ld.shared::cluster),
//   (c) local shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_lookup tools/microbench_lookup.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned lcg(unsigned x) { return x * 1664525u + 1013904223u; }

constexpr int kUnroll = 8;

__global__ void k_global(const unsigned* arr, unsigned mask, int iters, unsigned* out) {
  unsigned x[kUnroll], acc = 0;
  for (int j = 0; j < kUnroll; ++j) x[j] = (blockIdx.x * blockDim.x + threadIdx.x) * 7919u + j * 104729u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      x[j] = lcg(x[j]);
      acc += arr[(x[j] >> 7) & mask];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) k_dsmem(unsigned words, int iters, unsigned* out) {
  extern __shared__ unsigned sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (unsigned i = threadIdx.x; i < words; i += blockDim.x) sm[i] = i * 2654435761u;
  cl.sync();
  unsigned x[kUnroll], acc = 0;
  for (int j = 0; j < kUnroll; ++j) x[j] = (blockIdx.x * blockDim.x + threadIdx.x) * 7919u + j * 104729u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      x[j] = lcg(x[j]);
      const unsigned rank = (x[j] >> 28) & 7u;
      const unsigned off = (x[j] >> 7) % words;
      const unsigned* p = cl.map_shared_rank(sm, rank);
      acc += p[off];
    }
  }
  cl.sync();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_smem(unsigned words, int iters, unsigned* out) {
  extern __shared__ unsigned sm[];
  for (unsigned i = threadIdx.x; i < words; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  unsigned x[kUnroll], acc = 0;
  for (int j = 0; j < kUnroll; ++j) x[j] = (blockIdx.x * blockDim.x + threadIdx.x) * 7919u + j * 104729u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      x[j] = lcg(x[j]);
      acc += sm[(x[j] >> 7) % words];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 1024, iters = 2000;
  unsigned *arr, *out;
  const unsigned words2m = (2u << 20) / 4;
  cudaMalloc(&arr, 64u << 20);
  cudaMemset(arr, 1, 64u << 20);
  cudaMalloc(&out, (size_t)sms * 16 * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  auto report = [&](const char* name, double lookups, float t) {
    printf("%-28s %8.3f ms  %7.1f G lookups/s  %.3f lookups/SM/cycle@1.965GHz\n", name, t,
           lookups / t / 1e6, lookups / (t * 1e-3) / sms / 1.965e9);
  };
  for (unsigned mb : {2u, 64u}) {
    const unsigned mask = (mb << 20) / 4 - 1;
    for (int blocks_per_sm : {2, 4}) {
      int nb = sms * blocks_per_sm, nt = 256;
      k_global<<<nb, nt>>>(arr, mask, 10, out);
      cudaEventRecord(a);
      k_global<<<nb, nt>>>(arr, mask, iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      char nm[64];
      snprintf(nm, sizeof nm, "global %u MiB (%dx256/SM)", mb, blocks_per_sm);
      report(nm, (double)nb * nt * iters * kUnroll, ms);
    }
  }
  const unsigned smem_bytes = 200u << 10, words = smem_bytes / 4;
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  {
    int nb = (sms / 8) * 8;
    k_dsmem<<<nb, threads, smem_bytes>>>(words, 10, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("dsmem launch: %s\n", cudaGetErrorString(e));
    cudaEventRecord(a);
    k_dsmem<<<nb, threads, smem_bytes>>>(words, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    e = cudaGetLastError();
    if (e != cudaSuccess) printf("dsmem: %s\n", cudaGetErrorString(e));
    cudaEventElapsedTime(&ms, a, b);
    report("dsmem cluster8 x 200KiB", (double)nb * threads * iters * kUnroll, ms);
  }
  {
    int nb = sms;
    k_smem<<<nb, threads, smem_bytes>>>(words, 10, out);
    cudaEventRecord(a);
    k_smem<<<nb, threads, smem_bytes>>>(words, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    report("local smem 200KiB", (double)nb * threads * iters * kUnroll, ms);
  }
  printf("done\n");
  return 0;
}
