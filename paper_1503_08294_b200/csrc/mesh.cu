// mesh.cu -- mesh validation on the device.
//
// The reference validates a reconstructed surface on the host
// (metrics.py:165-240): every face edge's face count (_edge_face_counts),
// the manifold class (manifold_check: closed / with_boundary /
// non_manifold), connectivity of the face-edge graph (_is_connected) and the
// Euler genus.  Here one call reduces a face list to the counts those
// decisions need:
//   edge keys (min << 32 | max) of every face side -> radix sort -> run-length
//   encode (distinct edges and their face counts) -> per edge: > 2 faces,
//   boundary (1 face: both ends' boundary degree += 1), union-find hook of
//   its ends -> per vertex: boundary degree not in {0, 2}, root count.
// O(F log F) on the device instead of Python dict loops over 3F edges.

#include <cub/cub.cuh>

#include "common.cuh"

namespace gs {
namespace {

__global__ void k_edge_keys(const int64_t* __restrict__ faces, int64_t F, int64_t V,
                            unsigned long long* __restrict__ keys, int* __restrict__ bad) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int64_t a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
  if (a < 0 || b < 0 || c < 0 || a >= V || b >= V || c >= V) {
    atomicExch(bad, 1);
    keys[3 * f] = keys[3 * f + 1] = keys[3 * f + 2] = 0ull;
    return;
  }
  auto key = [](int64_t u, int64_t v) {
    const unsigned long long lo = (unsigned long long)(u < v ? u : v);
    const unsigned long long hi = (unsigned long long)(u < v ? v : u);
    return (lo << 32) | hi;
  };
  keys[3 * f] = key(a, b);
  keys[3 * f + 1] = key(a, c);
  keys[3 * f + 2] = key(b, c);
}

__device__ __forceinline__ int uf_root(int* parent, int v) {
  while (true) {
    const int p = ((volatile int*)parent)[v];
    if (p == v) return v;
    const int gp = ((volatile int*)parent)[p];
    if (gp != p) parent[v] = gp;  // path halving: always an ancestor
    v = p;
  }
}

__device__ __forceinline__ void uf_union(int* parent, int u, int v) {
  while (true) {
    u = uf_root(parent, u);
    v = uf_root(parent, v);
    if (u == v) return;
    if (u > v) {
      const int t = u;
      u = v;
      v = t;
    }
    // hook the larger root under the smaller one
    if (atomicCAS(&parent[v], v, u) == v) return;
  }
}

// counters: [0] > 2 faces, [1] boundary edges
__global__ void k_edge_runs(const unsigned long long* __restrict__ ukeys,
                            const int* __restrict__ counts, const int* __restrict__ nruns,
                            int* __restrict__ bdeg, int* __restrict__ parent,
                            unsigned long long* __restrict__ ctr) {
  const int n = *nruns;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = ukeys[i];
    const int u = (int)(k >> 32), v = (int)(k & 0xffffffffull);
    const int c = counts[i];
    if (c > 2) atomicAdd(&ctr[0], 1ull);
    if (c == 1) {
      atomicAdd(&ctr[1], 1ull);
      atomicAdd(&bdeg[u], 1);
      atomicAdd(&bdeg[v], 1);
    }
    uf_union(parent, u, v);
  }
}

// counters: [2] vertices with boundary degree not in {0, 2}, [3] components
__global__ void k_vertex_pass(const int* __restrict__ bdeg, int* parent, int64_t V,
                              unsigned long long* __restrict__ ctr) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int d = bdeg[v];
    if (d != 0 && d != 2) atomicAdd(&ctr[2], 1ull);
    if (uf_root(parent, (int)v) == (int)v) atomicAdd(&ctr[3], 1ull);
  }
}

__global__ void k_iota(int* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

}  // namespace

// faces: device (F x 3 int64, indices into [0, V)); out[6]: distinct face
// edges, edges with > 2 faces, boundary edges (1 face), vertices whose
// boundary degree is not 0 or 2, connected components of the face-edge graph
// over the V vertices, bad indices (1 = some index outside [0, V)).
void mesh_topology_device(Ctx& ctx, const int64_t* d_faces, int64_t F, int64_t V, int64_t out[6],
                          cudaStream_t st) {
  for (int q = 0; q < 6; ++q) out[q] = 0;
  GS_CHECK(V >= 0 && V < (1LL << 31) && F >= 0 && F < (1LL << 29), GS_VALUE_ERROR,
           "mesh too large");
  const int64_t E3 = 3 * F;
  const int threads = 256;
  const int grid = 4 * ctx.sm_count;
  // scratch layout (one allocation)
  size_t temp_sort = 0, temp_rle = 0;
  unsigned long long* nk = nullptr;
  GS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp_sort, nk, nk, (int)E3, 0, 64, st));
  GS_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, temp_rle, nk, nk, (int*)nullptr,
                                             (int*)nullptr, (int)E3, st));
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t b_keys = al(sizeof(unsigned long long) * (size_t)(E3 + 1));
  const size_t b_cnt = al(sizeof(int) * (size_t)(E3 + 1));
  const size_t b_v = al(sizeof(int) * (size_t)(V + 1));
  const size_t total = 3 * b_keys + b_cnt + 2 * b_v + al(64) + al(std::max(temp_sort, temp_rle));
  char* base = (char*)dmalloc(total, st);
  unsigned long long* keys = (unsigned long long*)base;
  unsigned long long* sorted = (unsigned long long*)(base + b_keys);
  unsigned long long* ukeys = (unsigned long long*)(base + 2 * b_keys);
  int* counts = (int*)(base + 3 * b_keys);
  int* bdeg = (int*)(base + 3 * b_keys + b_cnt);
  int* parent = (int*)(base + 3 * b_keys + b_cnt + b_v);
  int* small = (int*)(base + 3 * b_keys + b_cnt + 2 * b_v);  // [0] nruns, [1] bad
  unsigned long long* ctr = (unsigned long long*)(small + 4);  // 4 counters
  void* temp = base + 3 * b_keys + b_cnt + 2 * b_v + al(64);
  GS_CUDA(cudaMemsetAsync(small, 0, 64, st));
  if (V) GS_CUDA(cudaMemsetAsync(bdeg, 0, sizeof(int) * (size_t)V, st));
  if (V) {
    k_iota<<<grid, threads, 0, st>>>(parent, V);
    ++g_launches;
  }
  if (F) {
    k_edge_keys<<<(unsigned)((F + threads - 1) / threads), threads, 0, st>>>(d_faces, F, V, keys,
                                                                           small + 1);
    ++g_launches;
    size_t ts = temp_sort;
    GS_CUDA(cub::DeviceRadixSort::SortKeys(temp, ts, keys, sorted, (int)E3, 0, 64, st));
    size_t tr = temp_rle;
    GS_CUDA(cub::DeviceRunLengthEncode::Encode(temp, tr, sorted, ukeys, counts, small, (int)E3,
                                               st));
    g_launches += 4;
    k_edge_runs<<<grid, threads, 0, st>>>(ukeys, counts, small, bdeg, parent, ctr);
    ++g_launches;
  }
  if (V) {
    k_vertex_pass<<<grid, threads, 0, st>>>(bdeg, parent, V, ctr);
    ++g_launches;
  }
  GS_CUDA(cudaGetLastError());
  int h_small[2];
  unsigned long long h_ctr[4];
  GS_CUDA(cudaMemcpyAsync(h_small, small, sizeof(h_small), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  dfree(base, st);
  out[0] = F ? h_small[0] : 0;
  out[1] = (int64_t)h_ctr[0];
  out[2] = (int64_t)h_ctr[1];
  out[3] = (int64_t)h_ctr[2];
  out[4] = (int64_t)h_ctr[3];
  out[5] = h_small[1];
}

}  // namespace gs

using namespace gs;

extern "C" gs_status gs_mesh_topology(gs_ctx* ctx, const int64_t* faces, int64_t n_faces,
                                      int64_t n_vertices, int64_t out[6]) {
  return guarded([&] {
    GS_CHECK(ctx && out && (faces || n_faces == 0), GS_VALUE_ERROR, "null argument");
    GS_CHECK(n_faces >= 0 && n_vertices >= 0, GS_VALUE_ERROR, "negative size");
    std::lock_guard<std::mutex> lk(ctx->mu);
    GS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    int64_t* d_faces = nullptr;
    if (n_faces) {
      d_faces = (int64_t*)dmalloc(sizeof(int64_t) * 3 * (size_t)n_faces, st);
      GS_CUDA(cudaMemcpyAsync(d_faces, faces, sizeof(int64_t) * 3 * (size_t)n_faces,
                              cudaMemcpyHostToDevice, st));
    }
    try {
      mesh_topology_device(*ctx, d_faces, n_faces, n_vertices, out, st);
    } catch (...) {
      dfree(d_faces, st);
      throw;
    }
    dfree(d_faces, st);
    GS_CHECK(out[5] == 0, GS_VALUE_ERROR, "face index out of range");
  });
}
