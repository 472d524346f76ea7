// Microbenchmark: cost of cluster barriers, block barriers and dependent
// L2 / DRAM load chains on one SM (calibrates the update-kernel model).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(8, 1, 1) k_cluster_sync(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = clock64() - t0;
}
__global__ void k_block_sync(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) out[1] = clock64() - t0;
}
__global__ void k_chain(const int* next, int iters, long long* out, int* sink) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = next[p];
  long long t1 = clock64();
  sink[0] = p;
  out[2] = t1 - t0;
}
__global__ void k_atomic_chain(int* a, int iters, long long* out) {
  int v = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = atomicAdd(&a[(v & 1023) * 32], 1);
  out[3] = clock64() - t0;
  a[1] = v;
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 8 * sizeof(long long));
  int n = 1 << 22;  // 16 MB ring: L2-resident;   64M ints = 256 MB: DRAM
  for (int big = 0; big < 2; ++big) {
    int N = big ? (1 << 26) : n;
    int* next;
    cudaMalloc(&next, sizeof(int) * N);
    int* h = (int*)malloc(sizeof(int) * N);
    // random cyclic permutation with stride to defeat prefetch
    for (int i = 0; i < N; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % N);
    cudaMemcpy(next, h, sizeof(int) * N, cudaMemcpyHostToDevice);
    int* sink;
    cudaMalloc(&sink, 64);
    k_chain<<<1, 1>>>(next, 1000, out, sink);
    cudaDeviceSynchronize();
    k_chain<<<1, 1>>>(next, 1000, out, sink);
    cudaDeviceSynchronize();
    printf("dependent load chain (%s): %.0f cycles/load\n", big ? "256 MB, DRAM" : "16 MB, L2",
           out[2] / 1000.0);
    cudaFree(next);
    free(h);
  }
  k_cluster_sync<<<8, 1024>>>(1000, out);
  cudaDeviceSynchronize();
  k_cluster_sync<<<8, 1024>>>(1000, out);
  k_block_sync<<<1, 1024>>>(1000, out);
  cudaDeviceSynchronize();
  int* a;
  cudaMalloc(&a, 1024 * 32 * sizeof(int) * 2);
  cudaMemset(a, 0, 1024 * 32 * sizeof(int) * 2);
  k_atomic_chain<<<1, 1>>>(a, 1000, out);
  cudaDeviceSynchronize();
  printf("cluster.sync (8 CTAs x 1024 thr): %.0f cycles\n", out[0] / 1000.0);
  printf("__syncthreads (1024 thr): %.0f cycles\n", out[1] / 1000.0);
  printf("dependent atomicAdd (returning): %.0f cycles\n", out[3] / 1000.0);
  return 0;
}
