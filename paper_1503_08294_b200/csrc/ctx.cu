// ctx.cu -- context lifetime, error strings, launch accounting.
#include <cstdio>
#include <cstring>
#include <map>
#include <unordered_map>

#include "common.cuh"

namespace gs {

unsigned long long g_launches = 0;

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64] = {};
static std::multimap<size_t, void*> g_host_free;
static std::unordered_map<void*, size_t> g_host_size;

static cudaMemPool_t device_pool() {
  int dev = 0;
  GS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) throw Fail{GS_CUDA_ERROR};
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    GS_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t keep = ~0ull;
    GS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    g_pool[dev] = pool;
  }
  return g_pool[dev];
}

void* dmalloc(size_t bytes, cudaStream_t st) {
  void* p = nullptr;
  GS_CUDA(cudaMallocFromPoolAsync(&p, bytes ? bytes : 1, device_pool(), st));
  return p;
}

void dfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

void* hmalloc(size_t bytes) {
  bytes = (bytes + 4095) & ~(size_t)4095;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_host_free.lower_bound(bytes);
    if (it != g_host_free.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      g_host_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  GS_CUDA(cudaMallocHost(&p, bytes));
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_host_size[p] = bytes;
  return p;
}

void hfree(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_host_size.find(p);
  if (it == g_host_size.end()) return;
  g_host_free.emplace(it->second, p);
}

void* Ctx::ensure_device(size_t bytes) {
  if (bytes > d_cap) {
    if (d_buf) GS_CUDA(cudaFree(d_buf));
    d_buf = nullptr;
    d_cap = bytes + bytes / 2 + 4096;
    GS_CUDA(cudaMalloc(&d_buf, d_cap));
  }
  return d_buf;
}

void* Ctx::ensure_host(size_t bytes) {
  if (bytes > h_cap) {
    if (h_buf) GS_CUDA(cudaFreeHost(h_buf));
    h_buf = nullptr;
    h_cap = bytes + bytes / 2 + 4096;
    GS_CUDA(cudaMallocHost(&h_buf, h_cap));
  }
  return h_buf;
}

}  // namespace gs

using namespace gs;

extern "C" const char* gs_last_error(void) { return t_last_error.c_str(); }

extern "C" const char* gs_version(void) { return "growsurf-b200 0.1.0 (sm_100a)"; }

extern "C" gs_status gs_ctx_create(int device, gs_ctx** out) {
  return guarded([&] {
    GS_CHECK(out, GS_VALUE_ERROR, "null output pointer");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    GS_CHECK(e == cudaSuccess && count > 0, GS_CUDA_ERROR,
             std::string("no CUDA device available: ") + cudaGetErrorString(e));
    GS_CHECK(device >= 0 && device < count, GS_VALUE_ERROR, "device ordinal out of range");
    cudaDeviceProp prop;
    GS_CUDA(cudaGetDeviceProperties(&prop, device));
    GS_CHECK(prop.major >= 10, GS_CUDA_ERROR,
             std::string("growsurf-b200 is built for sm_100a; device is ") + prop.name);
    GS_CUDA(cudaSetDevice(device));
    gs_ctx* c = new gs_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) {
      delete c;
      GS_CUDA(se);
    }
    *out = c;
  });
}

extern "C" void gs_ctx_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_buf) cudaFree(ctx->d_buf);
  if (ctx->h_buf) cudaFreeHost(ctx->h_buf);
  if (ctx->d_fallbacks) cudaFree(ctx->d_fallbacks);
  ctx->find_work.release();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

extern "C" int gs_ctx_sm_count(const gs_ctx* ctx) { return ctx ? ctx->sm_count : 0; }

// ---------------------------------------------------------------------------
// FP32 peak probe (the find roofline's denominator, measured on the box):
// every thread runs 8 independent chains of packed FFMA2 (2 FMA = 4 FLOP
// each); one CTA of 512 threads per SM slot, 4 per SM.

namespace {
__global__ void __launch_bounds__(512) k_ffma2_peak(float* out, int iters, float seed) {
  float2 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    a[k] = make_float2(seed * (threadIdx.x + k), seed * (blockIdx.x + k));
  const float2 b = make_float2(0.9999999f, 1.0000001f), c = make_float2(1e-7f, -1e-7f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __ffma2_rn(a[k], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k].x + a[k].y;
  if (s == 1234.5f) out[0] = s;  // never true; keeps the chains alive
}
}  // namespace

extern "C" gs_status gs_fp32_peak(gs_ctx* ctx, double* tflops, double* ms) {
  return guarded([&] {
    GS_CHECK(ctx && tflops, GS_VALUE_ERROR, "null argument");
    GS_CUDA(cudaSetDevice(ctx->device));
    float* out = (float*)ctx->ensure_device(sizeof(float));
    const int blocks = 4 * ctx->sm_count, threads = 512, iters = 1 << 15;
    cudaEvent_t e0, e1;
    GS_CUDA(cudaEventCreate(&e0));
    GS_CUDA(cudaEventCreate(&e1));
    k_ffma2_peak<<<blocks, threads, 0, ctx->stream>>>(out, 256, 1e-3f);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      GS_CUDA(cudaEventRecord(e0, ctx->stream));
      k_ffma2_peak<<<blocks, threads, 0, ctx->stream>>>(out, iters, 1e-3f);
      GS_CUDA(cudaEventRecord(e1, ctx->stream));
      GS_CUDA(cudaEventSynchronize(e1));
      float t = 0.f;
      GS_CUDA(cudaEventElapsedTime(&t, e0, e1));
      best = t < best ? t : best;
    }
    GS_CUDA(cudaGetLastError());
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flop = 4.0 * 8.0 * (double)iters * blocks * threads;
    *tflops = flop / (best * 1e-3) / 1e12;
    if (ms) *ms = best;
  });
}
