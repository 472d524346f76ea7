// Microbenchmark: cost of cluster barriers (with and without pending global
// stores, relaxed vs release/acquire), block barriers, dependent L2 / DRAM /
// L1 load chains and shared-atomic contention on one SM (calibrates the
// update-kernel model).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o sync_lat sync_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void cl_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(8, 1, 1) k_cluster_sync(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = clock64() - t0;
}
// cluster.sync with one pending global store per thread before each barrier
__global__ void __cluster_dims__(8, 1, 1) k_cluster_sync_st(int iters, long long* out, int* buf) {
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank() * blockDim.x + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[g * 32 + (i & 31)] = i;
    cl.sync();
  }
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[4] = clock64() - t0;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster_relaxed(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    cl_arrive_relaxed();
    cl_wait();
  }
  if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) out[5] = clock64() - t0;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster_fence(int iters, long long* out, int* buf) {
  const int g = cg::this_cluster().block_rank() * blockDim.x + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[g * 32 + (i & 31)] = i;
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
    cl_arrive_relaxed();
    cl_wait();
  }
  if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) out[6] = clock64() - t0;
}
__global__ void k_block_sync(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) out[1] = clock64() - t0;
}
__global__ void k_chain(const int* next, int iters, long long* out, int* sink, int slot) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = next[p];
  long long t1 = clock64();
  sink[0] = p;
  out[slot] = t1 - t0;
}
__global__ void k_atomic_chain(int* a, int iters, long long* out) {
  int v = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = atomicAdd(&a[(v & 1023) * 32], 1);
  out[3] = clock64() - t0;
  a[1] = v;
}
// 1024 threads x 8 adds on ONE shared counter, plain vs warp-aggregated
__global__ void k_smem_atomics(long long* out, int* sink) {
  __shared__ int ctr;
  if (threadIdx.x == 0) ctr = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 8; ++i) atomicAdd(&ctr, 1);
  __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) {
    const unsigned m = __activemask();
    const int leader = __ffs(m) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(&ctr, __popc(m));
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    out[7] = t1 - t0;
    out[8] = t2 - t1;
    sink[1] = ctr;
  }
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 16 * sizeof(long long));
  int n = 1 << 22;  // 16 MB ring: L2-resident;   64M ints = 256 MB: DRAM;  4K ints: L1
  const int sizes[3] = {1 << 12, n, 1 << 26};
  const char* names[3] = {"16 KB, L1", "16 MB, L2", "256 MB, DRAM"};
  for (int big = 0; big < 3; ++big) {
    int N = sizes[big];
    int* next;
    cudaMalloc(&next, sizeof(int) * N);
    int* h = (int*)malloc(sizeof(int) * N);
    for (int i = 0; i < N; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % N);
    cudaMemcpy(next, h, sizeof(int) * N, cudaMemcpyHostToDevice);
    int* sink;
    cudaMalloc(&sink, 64);
    k_chain<<<1, 1>>>(next, 1000, out, sink, 2);
    cudaDeviceSynchronize();
    k_chain<<<1, 1>>>(next, 1000, out, sink, 2);
    cudaDeviceSynchronize();
    printf("dependent load chain (%s): %.0f cycles/load\n", names[big], out[2] / 1000.0);
    cudaFree(next);
    free(h);
  }
  int* buf;
  cudaMalloc(&buf, 8 * 1024 * 32 * sizeof(int));
  for (int rep = 0; rep < 2; ++rep) {
    k_cluster_sync<<<8, 1024>>>(1000, out);
    k_cluster_sync_st<<<8, 1024>>>(1000, out, buf);
    k_cluster_relaxed<<<8, 1024>>>(1000, out);
    k_cluster_fence<<<8, 1024>>>(1000, out, buf);
    k_block_sync<<<1, 1024>>>(1000, out);
    cudaDeviceSynchronize();
  }
  int* a;
  cudaMalloc(&a, 1024 * 32 * sizeof(int) * 2);
  cudaMemset(a, 0, 1024 * 32 * sizeof(int) * 2);
  k_atomic_chain<<<1, 1>>>(a, 1000, out);
  k_smem_atomics<<<1, 1024>>>(out, a);
  cudaDeviceSynchronize();
  printf("cluster.sync (8 CTAs x 1024 thr): %.0f cycles\n", out[0] / 1000.0);
  printf("cluster.sync after a global store: %.0f cycles\n", out[4] / 1000.0);
  printf("relaxed cluster barrier: %.0f cycles\n", out[5] / 1000.0);
  printf("store + fence.acq_rel.cluster + relaxed barrier: %.0f cycles\n", out[6] / 1000.0);
  printf("__syncthreads (1024 thr): %.0f cycles\n", out[1] / 1000.0);
  printf("dependent atomicAdd (returning): %.0f cycles\n", out[3] / 1000.0);
  printf("8192 smem atomicAdds on one address: %lld cycles; warp-aggregated: %lld cycles\n",
         out[7], out[8]);
  return 0;
}
