// sample.cu -- device-side CloudSource sampler, bit-identical to numpy.
//
// Reference: CloudSource.sample (pkg/src/growsurf/sampling.py:175-177) is
//   idx = rng.integers(0, N, size=m); return points[idx]
// with rng = numpy.random.Generator(Philox(seed)) (multi.py:151).  numpy
// draws each index with Lemire's bounded method on 32-bit halves of the
// Philox4x64-10 output stream (low half first; a pending high half is kept
// in the bit generator as has_uint32 / uinteger):
//   m64 = u32 * N;  reject while (m64 mod 2^32) < (2^32 - N) mod N;  idx = m64 >> 32.
// (Verified against numpy 2.3.5 by tests/test_sampler.py's pure-Python model.)
//
// The generator state lives on the device, so a run samples every batch
// without host work: one CTA generates candidate draws in parallel (a
// thread's eight consecutive draws), flags the rare rejections, ranks the
// accepted ones with a block scan, gathers points[idx] for the first m, and
// advances the state past the last draw it consumed -- exactly as numpy's
// sequential loop would.

#include "common.cuh"

namespace gs {

struct PhiloxState {
  unsigned long long ctr[4], key[2], buf[4];
  int pos;       // next unread word of buf (4 = empty)
  int has;       // a pending high half is stored in u
  unsigned u;
  int pad_;
};

__device__ __forceinline__ void philox4x64_10(const unsigned long long c_in[4],
                                              const unsigned long long k_in[2],
                                              unsigned long long out[4]) {
  unsigned long long c0 = c_in[0], c1 = c_in[1], c2 = c_in[2], c3 = c_in[3];
  unsigned long long k0 = k_in[0], k1 = k_in[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const unsigned long long hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const unsigned long long lo1 = 0xCA5A826395121157ULL * c2;
    const unsigned long long hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// 256-bit counter + b
__device__ __forceinline__ void ctr_add(const unsigned long long c[4], unsigned long long b,
                                        unsigned long long o[4]) {
  o[0] = c[0] + b;
  unsigned long long carry = o[0] < b ? 1ULL : 0ULL;
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    o[i] = c[i] + carry;
    carry = (carry && o[i] == 0ULL) ? 1ULL : 0ULL;
  }
}

// word q (0-based) of the uint64 stream that follows the state's position
__device__ unsigned long long stream_u64(const PhiloxState& s, unsigned long long q) {
  const unsigned long long r = 4ULL - (unsigned long long)s.pos;
  if (q < r) return s.buf[s.pos + q];
  const unsigned long long t = q - r;
  unsigned long long c[4], o[4];
  ctr_add(s.ctr, t / 4 + 1, c);
  philox4x64_10(c, s.key, o);
  return o[t % 4];
}

// 32-bit draw i of the stream that follows the state's position
__device__ __forceinline__ unsigned stream_u32(const PhiloxState& s, unsigned long long i) {
  if (s.has) {
    if (i == 0) return s.u;
    --i;
  }
  const unsigned long long v = stream_u64(s, i >> 1);
  return (i & 1) ? (unsigned)(v >> 32) : (unsigned)(v & 0xffffffffULL);
}

// state after consuming C 32-bit draws (numpy's next_uint32 / next_uint64)
__device__ void advance_state(PhiloxState& s, unsigned long long C) {
  if (C == 0) return;
  if (s.has) {
    s.has = 0;
    --C;
    if (C == 0) return;
  }
  const unsigned long long Q = (C + 1) / 2;  // uint64 words touched
  const bool half = (C & 1ULL) != 0;        // the last word's high half is pending
  const unsigned long long last = stream_u64(s, Q - 1);
  const unsigned long long r = 4ULL - (unsigned long long)s.pos;
  if (Q <= r) {
    s.pos += (int)Q;
  } else {
    const unsigned long long t = Q - r;
    const unsigned long long blocks = (t + 3) / 4;
    unsigned long long c[4];
    ctr_add(s.ctr, blocks, c);
    philox4x64_10(c, s.key, s.buf);
    for (int i = 0; i < 4; ++i) s.ctr[i] = c[i];
    s.pos = (int)(t - 4 * (blocks - 1));
  }
  s.has = half ? 1 : 0;
  s.u = half ? (unsigned)(last >> 32) : 0u;
}

constexpr int kSampThreads = 1024;
constexpr int kSampPer = 8;  // one Philox block (4 words = 8 draws) per thread per round

// One CTA per batch.  The stream after the state's position is: the pending
// high half (if any), the halves of the buffered words, then whole Philox
// blocks ctr+1, ctr+2, ...  Thread 0 handles that short prefix (<= 9
// draws); then every thread computes ONE block per round -- eight
// consecutive draws -- the rare rejections are flagged, a block scan ranks
// the accepted draws in stream order, and the first m gather points[idx].
__global__ void __launch_bounds__(kSampThreads) k_cloud_sample(PhiloxState* st, const double* pts,
                                                               unsigned npts, int m,
                                                               double* out, int64_t* out_idx) {
  __shared__ int s_warp[32];
  __shared__ int s_total;
  __shared__ int s_pre;
  __shared__ unsigned long long s_consumed;
  if (npts == 1u) {  // integers(0, 1) returns zeros without drawing
    for (int j = threadIdx.x; j < m; j += kSampThreads) {
      if (out) {
        out[3 * (size_t)j] = pts[0];
        out[3 * (size_t)j + 1] = pts[1];
        out[3 * (size_t)j + 2] = pts[2];
      }
      if (out_idx) out_idx[j] = 0;
    }
    return;
  }
  const PhiloxState s = *st;
  const unsigned rng = npts - 1u;
  const unsigned excl = npts;
  const unsigned thr = (0xffffffffu - rng) % excl;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  auto emit = [&](int rank, unsigned v) {
    if (out) {
      const size_t p = (size_t)v * 3;
      out[3 * (size_t)rank] = pts[p];
      out[3 * (size_t)rank + 1] = pts[p + 1];
      out[3 * (size_t)rank + 2] = pts[p + 2];
    }
    if (out_idx) out_idx[rank] = (int64_t)v;
  };
  // ---- prefix: pending half + buffered words (no Philox needed)
  const int npre = s.has + 2 * (4 - s.pos);
  if (tid == 0) {
    int produced = 0;
    s_consumed = 0;
    for (int i = 0; i < npre && produced < m; ++i) {
      unsigned u32;
      if (s.has && i == 0) {
        u32 = s.u;
      } else {
        const int k = i - s.has;
        const unsigned long long word = s.buf[s.pos + (k >> 1)];
        u32 = (k & 1) ? (unsigned)(word >> 32) : (unsigned)word;
      }
      const unsigned long long mm = (unsigned long long)u32 * excl;
      if ((unsigned)mm >= thr) {
        emit(produced, (unsigned)(mm >> 32));
        if (++produced == m) s_consumed = (unsigned long long)i + 1;
      }
    }
    s_pre = produced;
  }
  __syncthreads();
  int produced = s_pre;
  unsigned long long block0 = 0;  // blocks already handed out (ctr + 1 + block index)
  while (produced < m) {          // uniform: produced is block-wide
    const unsigned long long b = block0 + (unsigned long long)tid;
    unsigned long long c[4], o[4];
    ctr_add(s.ctr, b + 1, c);
    philox4x64_10(c, s.key, o);
    unsigned vals[kSampPer];
    unsigned acc = 0;  // bit e: draw e accepted
#pragma unroll
    for (int e = 0; e < kSampPer; ++e) {
      const unsigned long long word = o[e >> 1];
      const unsigned u32 = (e & 1) ? (unsigned)(word >> 32) : (unsigned)word;
      const unsigned long long mm = (unsigned long long)u32 * excl;
      vals[e] = (unsigned)(mm >> 32);
      if ((unsigned)mm >= thr) acc |= 1u << e;
    }
    // block exclusive scan of accepted counts (thread order == stream order)
    const int cnt = __popc(acc);
    int inc = cnt;
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o2);
      if (lane >= o2) inc += t;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    if (w == 0) {
      const int x = s_warp[lane];
      int xi = x;
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, xi, o2);
        if (lane >= o2) xi += t;
      }
      s_warp[lane] = xi - x;
      if (lane == 31) s_total = xi;
    }
    __syncthreads();
    int rank = produced + s_warp[w] + inc - cnt;
#pragma unroll
    for (int e = 0; e < kSampPer; ++e) {
      if (!((acc >> e) & 1u)) continue;
      if (rank < m) {
        emit(rank, vals[e]);
        if (rank == m - 1) s_consumed = (unsigned long long)npre + b * kSampPer + e + 1;
      }
      ++rank;
    }
    produced += s_total;
    block0 += kSampThreads;
    __syncthreads();
  }
  if (tid == 0) {
    PhiloxState n = s;
    advance_state(n, s_consumed);
    *st = n;
  }
}

}  // namespace gs

using namespace gs;

struct gs_sampler {
  gs_ctx* ctx = nullptr;
  double* d_pts = nullptr;
  unsigned long long npts = 0;
  PhiloxState* d_state = nullptr;
  bool owns_pts = false;
  gs::DevBuf idx_tmp;  // indices for gs_sampler_draw's parallel gather
};

namespace gs {
__global__ void k_sample_gather(const int64_t* idx, const double* pts, double* out, int64_t m) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const size_t src = 3 * (size_t)idx[j];
  out[3 * j] = pts[src];
  out[3 * j + 1] = pts[src + 1];
  out[3 * j + 2] = pts[src + 2];
}
}  // namespace gs

extern "C" gs_status gs_sampler_create(gs_ctx* ctx, const double* points, int64_t npts,
                                       int points_on_device, gs_sampler** out) {
  return guarded([&] {
    GS_CHECK(ctx && out, GS_VALUE_ERROR, "null argument");
    GS_CHECK(npts >= 1 && npts <= 0xffffffffLL, GS_VALUE_ERROR,
             "point count must be in [1, 2^32) (numpy's 32-bit bounded path)");
    GS_CUDA(cudaSetDevice(ctx->device));
    gs_sampler* s = new gs_sampler();
    s->ctx = ctx;
    s->npts = (unsigned long long)npts;
    try {
      s->d_state = (PhiloxState*)dmalloc(sizeof(PhiloxState), ctx->stream);
      if (!points) {
        s->d_pts = nullptr;  // index-only sampler (rng.integers(0, npts, m))
      } else if (points_on_device) {
        s->d_pts = const_cast<double*>(points);
      } else {
        s->d_pts = (double*)dmalloc(sizeof(double) * 3 * (size_t)npts, ctx->stream);
        s->owns_pts = true;
        GS_CUDA(cudaMemcpyAsync(s->d_pts, points, sizeof(double) * 3 * (size_t)npts,
                                cudaMemcpyHostToDevice, ctx->stream));
      }
      GS_CUDA(cudaStreamSynchronize(ctx->stream));  // draws run on other streams
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      dfree(s->d_state, ctx->stream);
      if (s->owns_pts) dfree(s->d_pts, ctx->stream);
      delete s;
      throw;
    }
    *out = s;
  });
}

extern "C" void gs_sampler_destroy(gs_sampler* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  // draws run on caller streams: wait for them before the memory returns to the pool
  cudaDeviceSynchronize();
  dfree(s->d_state, s->ctx->stream);
  if (s->owns_pts) dfree(s->d_pts, s->ctx->stream);
  s->idx_tmp.release();
  delete s;
}

// state layout (uint64[15]): ctr[4], key[2], buf[4], pos, has_uint32, uinteger, 0, 0
extern "C" gs_status gs_sampler_set_state(gs_sampler* s, const uint64_t* state) {
  return guarded([&] {
    GS_CHECK(s && state, GS_VALUE_ERROR, "null argument");
    GS_CHECK(state[10] >= 1 && state[10] <= 4 && state[11] <= 1 && state[12] <= 0xffffffffULL,
             GS_VALUE_ERROR, "bad Philox state");
    PhiloxState h;
    for (int i = 0; i < 4; ++i) h.ctr[i] = state[i];
    h.key[0] = state[4];
    h.key[1] = state[5];
    for (int i = 0; i < 4; ++i) h.buf[i] = state[6 + i];
    h.pos = (int)state[10];
    h.has = (int)state[11];
    h.u = (unsigned)state[12];
    h.pad_ = 0;
    GS_CUDA(cudaMemcpyAsync(s->d_state, &h, sizeof(h), cudaMemcpyHostToDevice, s->ctx->stream));
    GS_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

extern "C" gs_status gs_sampler_get_state(gs_sampler* s, uint64_t* state) {
  return guarded([&] {
    GS_CHECK(s && state, GS_VALUE_ERROR, "null argument");
    GS_CUDA(cudaDeviceSynchronize());
    PhiloxState h;
    GS_CUDA(cudaMemcpy(&h, s->d_state, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; ++i) state[i] = h.ctr[i];
    state[4] = h.key[0];
    state[5] = h.key[1];
    for (int i = 0; i < 4; ++i) state[6 + i] = h.buf[i];
    state[10] = (uint64_t)h.pos;
    state[11] = (uint64_t)h.has;
    state[12] = (uint64_t)h.u;
    state[13] = state[14] = 0;
  });
}

static void sampler_launch(gs_sampler* s, int64_t m, double* d_out, int64_t* d_idx,
                           cudaStream_t st) {
  GS_CHECK(m >= 0 && m <= 0x7fffffffLL, GS_VALUE_ERROR, "bad sample count");
  if (m == 0) return;
  k_cloud_sample<<<1, kSampThreads, 0, st>>>(s->d_state, s->d_pts, (unsigned)s->npts, (int)m,
                                            d_out, d_idx);
  GS_CUDA(cudaGetLastError());
  ++g_launches;
}

// indices from the one-CTA generator, then a full-grid gather
void gs::sampler_draw(gs_sampler* s, int64_t m, double* d_out, cudaStream_t st) {
  GS_CHECK(s && d_out, GS_VALUE_ERROR, "null argument");
  GS_CHECK(s->d_pts, GS_VALUE_ERROR, "index-only sampler has no points");
  if (m <= 0) return;
  int64_t* idx = (int64_t*)s->idx_tmp.get(sizeof(int64_t) * (size_t)m);
  sampler_launch(s, m, nullptr, idx, st);
  k_sample_gather<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(idx, s->d_pts, d_out, m);
  GS_CUDA(cudaGetLastError());
  ++g_launches;
}

void gs::sampler_indices(gs_sampler* s, int64_t m, int64_t* d_idx, cudaStream_t st) {
  GS_CHECK(s && d_idx, GS_VALUE_ERROR, "null argument");
  GS_CHECK(s->d_pts, GS_VALUE_ERROR, "index-only sampler has no points");
  sampler_launch(s, m, nullptr, d_idx, st);
}

const double* gs::sampler_points(const gs_sampler* s) { return s->d_pts; }

extern "C" gs_status gs_sampler_draw_indices(gs_sampler* s, int64_t m, int64_t* d_idx,
                                             void* stream) {
  return guarded([&] {
    GS_CHECK(s && d_idx, GS_VALUE_ERROR, "null argument");
    sampler_launch(s, m, nullptr, d_idx, stream ? (cudaStream_t)stream : s->ctx->stream);
  });
}

extern "C" gs_status gs_sampler_draw(gs_sampler* s, int64_t m, double* d_out, void* stream) {
  return guarded([&] {
    GS_CHECK(s, GS_VALUE_ERROR, "null sampler");
    sampler_draw(s, m, d_out, stream ? (cudaStream_t)stream : s->ctx->stream);
  });
}
