// ctx.cu -- context lifetime, error strings, launch accounting.
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace gs {

unsigned long long g_launches = 0;

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

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
