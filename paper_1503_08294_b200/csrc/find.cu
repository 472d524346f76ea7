// find.cu -- batched best-two ("find winners") kernels for sm_100a.
//
// Reference semantics: scan_best_two_into, pkg/src/growsurf/kernels/_scan.pyx:39-98.
// For every signal j: the rows of the nearest and second-nearest unit and
// their squared distances, lexicographic on (d2, row), with
// d2 = ((dx*dx + dy*dy) + dz*dz) in binary64 and dx = p - s.
//
// Exact path (GS_FIND_EXACT): every pair in FP64 with the reference rounding
// sequence.  The m x n pair space is split two ways: CTAs over signal tiles
// (each thread keeps FS signals in registers) and, when m alone cannot fill
// the 148 SMs, over contiguous row chunks ("split-n").  Unit rows are staged
// through shared memory tile by tile and read as broadcasts.  Per-chunk
// best-two partials are merged in chunk (= row) order with the same strict-<
// rule, which is exactly the lexicographic (d2, row) top-2 of the union, so
// the result is independent of the chunking (as it is of the reference's
// `tile`, test_kernels.py:74-86).
//
// Filter path (GS_FIND_FILTER, filter.cu): FP32 top-3 filter and a certified
// FP64 re-check; bit-identical outputs.

#include <algorithm>

#include "common.cuh"

namespace gs {

constexpr int kFT = 128;    // threads per CTA
constexpr int kMinChunk = 64; // fewest unit rows per split-n chunk
constexpr int kFTile = 256; // unit rows per shared-memory tile

struct Part {
  double d1, d2;
  int32_t i1, i2;
};

template <int kFS>  // signals per thread
__global__ void __launch_bounds__(kFT) find_exact_kernel(FindArgs a, int64_t rows_per_chunk,
                                                         Part* part) {
  __shared__ double sx[kFTile], sy[kFTile], sz[kFTile];
  const int tid = threadIdx.x;
  const int64_t sig0 = (int64_t)blockIdx.x * (kFT * kFS);
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_chunk;
  const int64_t n = a.n_dev ? (int64_t)*a.n_dev : a.n;
  // the last chunk takes every row past the host's estimate
  const int64_t r_end = blockIdx.y + 1 == gridDim.y ? n : min(n, r_begin + rows_per_chunk);

  double qx[kFS], qy[kFS], qz[kFS];
  Best2 best[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const int64_t j = sig0 + tid + k * kFT;
    best[k].init();
    if (j < a.m) {
      qx[k] = a.sig[3 * j];
      qy[k] = a.sig[3 * j + 1];
      qz[k] = a.sig[3 * j + 2];
    } else {
      qx[k] = qy[k] = qz[k] = 0.0;
    }
  }
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kFTile) {
    __syncthreads();
    for (int i = tid; i < kFTile; i += kFT) {
      const int64_t r = r0 + i;
      double x = kInf, y = kInf, z = kInf;
      if (r < r_end && !load_row(a, r, x, y, z)) x = y = z = kInf;
      sx[i] = x;
      sy[i] = y;
      sz[i] = z;
    }
    __syncthreads();
    const int cnt = (int)(r_end - r0 < kFTile ? r_end - r0 : kFTile);
    for (int i = 0; i < cnt; ++i) {
      const double px = sx[i], py = sy[i], pz = sz[i];
      const int32_t row = (int32_t)(r0 + i);
#pragma unroll
      for (int k = 0; k < kFS; ++k) best[k].push(dist2_exact(px, py, pz, qx[k], qy[k], qz[k]), row);
    }
  }
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const int64_t j = sig0 + tid + k * kFT;
    if (j >= a.m) continue;
    if (part) {
      Part p;
      p.d1 = best[k].d1;
      p.d2 = best[k].d2;
      p.i1 = best[k].i1;
      p.i2 = best[k].i2;
      part[(int64_t)blockIdx.y * a.m + j] = p;
    } else {
      write_result(a, j, best[k]);
    }
  }
}

__global__ void find_merge_kernel(FindArgs a, int nchunks, const Part* part) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.m) return;
  Best2 b;
  b.init();
  for (int c = 0; c < nchunks; ++c) {
    const Part p = part[(int64_t)c * a.m + j];
    if (p.i1 >= 0) b.push(p.d1, p.i1);
    if (p.i2 >= 0) b.push(p.d2, p.i2);
  }
  write_result(a, j, b);
}

// ---------------------------------------------------------------------------
// Small-n exact find (the engine's regime: a few thousand units): one kernel,
// no partial buffer.  Every CTA stages ALL rows in shared memory (24 B per
// row) and owns 16*FS signals; the 16 lanes of a half-warp split the rows of
// one signal (lane l scans rows l, l+16, ..., ascending) and merge their
// best-two lexicographically on (d2, row) with xor shuffles -- the result is
// the same for any split.

constexpr int kSmallThreads = 256;
constexpr int kSmallSlices = 16;
constexpr int kSmallMaxRows = 6144;  // 144 KB of shared memory


template <int kFS>
__global__ void __launch_bounds__(kSmallThreads) find_small_kernel(FindArgs a, int tile_rows) {
  extern __shared__ double s_rows[];  // [3][tile_rows]
  const int64_t n = a.n_dev ? (int64_t)*a.n_dev : a.n;
  const bool compact = a.rowpos && *a.rowpos_n == n;
  double* sx = s_rows;
  double* sy = s_rows + tile_rows;
  double* sz = s_rows + 2 * tile_rows;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const int slice = threadIdx.x & (kSmallSlices - 1);
  const int sl = threadIdx.x / kSmallSlices;  // 0..15
  const int64_t sig0 = (int64_t)blockIdx.x * (kSmallThreads / kSmallSlices) * kFS;
  double qx[kFS], qy[kFS], qz[kFS];
  Best2 b[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const int64_t j = sig0 + sl + k * (kSmallThreads / kSmallSlices);
    b[k].init();
    qx[k] = qy[k] = qz[k] = 0.0;
    if (j < a.m) {
      if (a.sig_idx) {  // fused sampling: gather the signal, one lane stores it
        const size_t src = 3 * (size_t)a.sig_idx[j];
        qx[k] = a.sig_pts[src];
        qy[k] = a.sig_pts[src + 1];
        qz[k] = a.sig_pts[src + 2];
        if (slice == 0) {
          double* o = const_cast<double*>(a.sig);
          o[3 * j] = qx[k];
          o[3 * j + 1] = qy[k];
          o[3 * j + 2] = qz[k];
        }
      } else {
        qx[k] = a.sig[3 * j];
        qy[k] = a.sig[3 * j + 1];
        qz[k] = a.sig[3 * j + 2];
      }
    }
  }
  // one tile in the common case; more when the device's row count has grown
  // past the host's estimate (batches in flight)
  for (int64_t t0 = 0; t0 < n; t0 += tile_rows) {
    const int nr = (int)min((int64_t)tile_rows, n - t0);
    if (t0 > 0) __syncthreads();
    if (compact) {  // the update left row-ordered positions: coalesced copies
      const double* X = a.rowpos + t0;
      for (int r = threadIdx.x; r < nr; r += kSmallThreads) {
        sx[r] = X[r];
        sy[r] = X[a.rowpos_stride + r];
        sz[r] = X[2 * a.rowpos_stride + r];
      }
    } else {
      for (int r0 = 0; r0 < nr; r0 += 4 * kSmallThreads) {  // four rows in flight per thread
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + q * kSmallThreads + threadIdx.x;
          if (r < nr) {
            double x = kInf, y = kInf, z = kInf;
            if (!load_row(a, t0 + r, x, y, z)) x = y = z = kInf;
            sx[r] = x;
            sy[r] = y;
            sz[r] = z;
          }
        }
      }
    }
    __syncthreads();
    // four rows per step: independent FP64 chains, one rarely-taken branch
    int r = slice;
    for (; r + 3 * kSmallSlices < nr; r += 4 * kSmallSlices) {
#pragma unroll
      for (int k = 0; k < kFS; ++k) {
        double d[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = r + q * kSmallSlices;
          d[q] = dist2_exact(sx[rr], sy[rr], sz[rr], qx[k], qy[k], qz[k]);
        }
        if (fmin(fmin(d[0], d[1]), fmin(d[2], d[3])) < b[k].d2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) b[k].push(d[q], (int32_t)(t0 + r + q * kSmallSlices));
        }
      }
    }
    for (; r < nr; r += kSmallSlices) {
      const double px = sx[r], py = sy[r], pz = sz[r];
#pragma unroll
      for (int k = 0; k < kFS; ++k)
        b[k].push(dist2_exact(px, py, pz, qx[k], qy[k], qz[k]), (int32_t)(t0 + r));
    }
  }
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
#pragma unroll
    for (int o = kSmallSlices / 2; o > 0; o >>= 1) {
      const double od1 = __shfl_xor_sync(0xffffffffu, b[k].d1, o);
      const double od2 = __shfl_xor_sync(0xffffffffu, b[k].d2, o);
      const int32_t oi1 = __shfl_xor_sync(0xffffffffu, b[k].i1, o);
      const int32_t oi2 = __shfl_xor_sync(0xffffffffu, b[k].i2, o);
      best2_lex(b[k], od1, oi1);
      best2_lex(b[k], od2, oi2);
    }
    const int64_t j = sig0 + sl + k * (kSmallThreads / kSmallSlices);
    if (slice == 0 && j < a.m) write_result(a, j, b[k]);
  }
}

// ---------------------------------------------------------------------------
// Small-n screened find (GS_FIND_SMALL; AUTO for n <= 4096): one kernel, the
// same output bit for bit.  Every CTA stages all rows in shared memory as FP32
// unit pairs relative to a centre c (row 0 rounded to FP32, so c is exact in
// binary64): {-2P'x, -2P'y, -2P'z, |P'|^2}, P' = fl32(p - c).  A warp owns FS
// signals; lane l owns the unit pairs l, l+32, ... .
//   pass 1  e = |P'|^2 - 2 P'.Q' with three packed FFMA2 per two units and a
//           running minimum: no indices, no branches.
//   screen  e2 = the second smallest of the 32 lane minima.  Two distinct
//           units have e_fp32 <= e2, so with f >= |e_fp32 - e_real| for every
//           unit (filter.cu's bound with a = Pmax) the reference's best two
//           both have e_fp32 <= T = e2 + 2f (+ FP64 slack).  Only lanes whose
//           minimum is <= T can hold one; their units are re-screened one by
//           one and those with e_fp32 <= T form the warp's candidate list
//           (usually two or three per signal).
//   exact   every candidate is evaluated in FP64 with the reference rounding
//           (one per lane) and lane k merges signal k's candidates in
//           lexicographic (d2, row) order.
// Whenever the bound does not apply (fewer than two finite FP32 values,
// non-finite or huge coordinates) or the list overflows (mass ties), the
// warp scans every row exactly instead.

constexpr int kSfMaxRows = 4096;  // 16 B per row in shared memory
constexpr int kSfCand = 128;      // candidate list per warp

__device__ __forceinline__ void warp_best2_merge(Best2& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od1 = __shfl_xor_sync(0xffffffffu, b.d1, o);
    const double od2 = __shfl_xor_sync(0xffffffffu, b.d2, o);
    const int32_t oi1 = __shfl_xor_sync(0xffffffffu, b.i1, o);
    const int32_t oi2 = __shfl_xor_sync(0xffffffffu, b.i2, o);
    best2_lex(b, od1, oi1);
    best2_lex(b, od2, oi2);
  }
}

__device__ __forceinline__ bool sf_row(const FindArgs& a, bool compact, int64_t r, double& x,
                                       double& y, double& z) {
  if (compact) {
    x = a.rowpos[r];
    y = a.rowpos[a.rowpos_stride + r];
    z = a.rowpos[2 * a.rowpos_stride + r];
    return true;
  }
  return load_row(a, r, x, y, z);
}

// fused sampling: the gathered signals are stored for the update (last, so
// the stores never wait on the gather ahead of the row staging)
template <int kFS>
__device__ __forceinline__ void sf_store_signals(const FindArgs& a, int64_t sig0, int lane,
                                                 const double* qx, const double* qy,
                                                 const double* qz) {
  if (!a.sig_idx) return;
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const int64_t j = sig0 + k;
    if (lane == k && j < a.m) {
      double* o = const_cast<double*>(a.sig);
      o[3 * j] = qx[k];
      o[3 * j + 1] = qy[k];
      o[3 * j + 2] = qz[k];
    }
  }
}

#ifndef GS_POLL_NS
#define GS_POLL_NS 32  // back-off between polls of the update's flags
#endif
#ifndef GS_POLL_ACQ
#define GS_POLL_ACQ 0  // acquire loads in the poll instead of a fence after it
#endif
#ifdef GS_PROF_TL
// timeline profiling builds: globaltimer stamps of every CTA for launches
// [GS_PROF_TL - 100, GS_PROF_TL + 3), printed (tools/timeline.py parses them)
__device__ unsigned g_sf_seq;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SF_TL(k) if (threadIdx.x == 0) tl[k] = gtimer()
// per batch: wait released (CTA 0), last CTA's end, CTA count
__device__ unsigned long long g_tlf[8192][3];
// per batch, CTA 0's entry and poll start; the latest CTA's poll start
__device__ unsigned long long g_tlf2[8192][3];
extern "C" int gs_debug_tl_find2(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_tlf2, sizeof(unsigned long long) * 3 * (size_t)n);
}
extern "C" int gs_debug_tl_find(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_tlf, sizeof(unsigned long long) * 3 * (size_t)n);
}
#else
#define SF_TL(k)
#endif

// the screen's threshold T = e2 + 2 f + slack, every operation rounded up
// (an upper bound of the same expression evaluated exactly; filter.cu's
// error bound with a = Pmax, Q = |q - c|)
// delta > 0 (speculative screen against the snapshot before the last update,
// delta >= every unit's displacement since): every unit whose distance may be
// within the second-best one after the moves, i.e. old distance <= D2 + 2 delta
// with D2 bounded by sqrt(e2 + f + Q^2):  T = (D2 + 2 delta)^2 - Q^2 + f
__device__ __forceinline__ float sf_threshold(float e2, float pmaxf, double Qx, double Qy,
                                              double Qz, bool& ok, float delta = 0.f) {
  const float ax = __double2float_ru(fabs(Qx)), ay = __double2float_ru(fabs(Qy)),
              az = __double2float_ru(fabs(Qz));
  const float q2 = __fmaf_ru(az, az, __fmaf_ru(ay, ay, __fmul_ru(ax, ax)));
  ok = e2 < INFINITY && pmaxf * pmaxf <= 1e30f && q2 <= 1e30f;
  const float u = 0x1p-24f, Q = __fsqrt_ru(q2), av = pmaxf;
  const float dl = __fmaf_ru(u, av, __fmul_ru(__fmul_ru(u, 1.0f + 0x1p-23f), pmaxf));
  float t = __fmul_ru(__fmul_ru(2.0f, dl), __fadd_ru(av, Q));
  t = __fmaf_ru(dl, dl, t);
  t = __fmaf_ru(__fmul_ru(6.02f * u, av), av, t);
  t = __fmaf_ru(__fmul_ru(8.03f * u, av), Q, t);
  const float fb = __fadd_ru(__fmul_ru(t, 1.0f + 1e-6f), 1e-38f);
  if (delta > 0.f) {
    const float qx = __double2float_rd(fabs(Qx)), qy = __double2float_rd(fabs(Qy)),
                qz = __double2float_rd(fabs(Qz));
    const float q2lo = __fmaf_rd(qz, qz, __fmaf_rd(qy, qy, __fmul_rd(qx, qx)));
    const float d2 = __fsqrt_ru(fmaxf(0.f, __fadd_ru(__fadd_ru(e2, fb), q2)));
    const float R = __fadd_ru(d2, __fmul_ru(2.0f, delta));
    const float RR = __fmul_ru(R, R);
    const float slack = __fmul_ru(1e-14f, __fadd_ru(RR, q2));
    ok = ok && RR <= 1e30f;
    return __fadd_ru(__fadd_ru(__fsub_ru(RR, q2lo), fb), slack);
  }
  const float slack = __fmul_ru(1e-14f, __fadd_ru(__fadd_ru(fabsf(e2), fb), q2));
  return __fadd_ru(__fadd_ru(e2, __fmul_ru(2.0f, fb)), slack);
}

// pass 1 (lane minima of e), the thresholds and the candidate list of one
// warp's kFS signals against nr staged rows (swizzled pairs A0 / A1, centre c,
// max-norm pm); returns the candidate count, full_scan when the bound does
// not apply
template <int kFS>
__device__ __forceinline__ int sf_screen(const float4* A0, const float4* A1, int nr, double cx,
                                         double cy, double cz, float pm, float delta,
                                         const double (&qx)[kFS], const double (&qy)[kFS],
                                         const double (&qz)[kFS], int lane, int32_t* cand,
                                         double (*sq)[3], bool& full_scan) {
  // |p - c| <= sqrt(3) * max_k |P'_k| / (1 - u), rounded up generously
  const float pmaxf = __fmul_ru(pm, 1.7320508075688774f * (1.0f + 1e-6f));
  float2 fq[kFS][3];
  float m1[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const float fx = __double2float_rn(qx[k] - cx), fy = __double2float_rn(qy[k] - cy),
                fz = __double2float_rn(qz[k] - cz);
    fq[k][0] = make_float2(fx, fx);
    fq[k][1] = make_float2(fy, fy);
    fq[k][2] = make_float2(fz, fz);
    m1[k] = INFINITY;
  }
  const int np64 = (((nr + 1) / 2) + 63) & ~63;  // padded pairs are +inf
#pragma unroll 1
  for (int p = lane; p < np64; p += 64) {
    const int sa = sf_swz(p), sc = sf_swz(p + 32);
    const float4 a0 = A0[sa], a1 = A1[sa];
    const float4 c0 = A0[sc], c1 = A1[sc];
#pragma unroll
    for (int k = 0; k < kFS; ++k) {
      float2 ea = __ffma2_rn(make_float2(a0.x, a0.y), fq[k][0], make_float2(a1.z, a1.w));
      float2 ec = __ffma2_rn(make_float2(c0.x, c0.y), fq[k][0], make_float2(c1.z, c1.w));
      ea = __ffma2_rn(make_float2(a0.z, a0.w), fq[k][1], ea);
      ec = __ffma2_rn(make_float2(c0.z, c0.w), fq[k][1], ec);
      ea = __ffma2_rn(make_float2(a1.x, a1.y), fq[k][2], ea);
      ec = __ffma2_rn(make_float2(c1.x, c1.y), fq[k][2], ec);
      m1[k] = fminf(m1[k], fminf(fminf(ea.x, ea.y), fminf(ec.x, ec.y)));
    }
  }
  // screen: every signal's threshold (independent chains, issued together),
  // then the surviving lanes' units one by one
  float T[kFS];
  unsigned tasks[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    float v1 = m1[k], v2 = INFINITY;  // two smallest lane minima
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float o1 = __shfl_xor_sync(0xffffffffu, v1, o);
      const float o2 = __shfl_xor_sync(0xffffffffu, v2, o);
      v2 = fminf(fmaxf(v1, o1), fminf(v2, o2));
      v1 = fminf(v1, o1);
    }
    bool ok;
    T[k] = sf_threshold(v2, pmaxf, qx[k] - cx, qy[k] - cy, qz[k] - cz, ok, delta);
    full_scan |= !ok;  // warp-uniform
    tasks[k] = __ballot_sync(0xffffffffu, m1[k] <= T[k]);
  }
  int cnt = 0;
  if (!full_scan) {
#pragma unroll
    for (int k = 0; k < kFS; ++k) {
      unsigned tk = tasks[k];
      while (tk) {
        const int l = __ffs(tk) - 1;
        tk &= tk - 1;
        for (int i0 = 0; i0 < np64 / 32; i0 += 32) {  // lane l's pairs l + 32 i, one per lane
          const int p = 32 * (i0 + lane) + l;
          const bool in = p < np64;
          const int sp = sf_swz(p);  // conflict-free: lane i reads row i, column l ^ i
          const float4 a0 = in ? A0[sp] : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 a1 = in ? A1[sp] : make_float4(0.f, 0.f, INFINITY, INFINITY);
          float2 e = __ffma2_rn(make_float2(a0.x, a0.y), fq[k][0], make_float2(a1.z, a1.w));
          e = __ffma2_rn(make_float2(a0.z, a0.w), fq[k][1], e);
          e = __ffma2_rn(make_float2(a1.x, a1.y), fq[k][2], e);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool pass = in && (h ? e.y : e.x) <= T[k];
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            const int at = cnt + __popc(bal & ((1u << lane) - 1u));
            if (pass && at < kSfCand) cand[at] = ((2 * p + h) << 3) | k;
            cnt += __popc(bal);
          }
        }
      }
      if (lane == 0) {
        sq[k][0] = qx[k];
        sq[k][1] = qy[k];
        sq[k][2] = qz[k];
      }
    }
  }
  return cnt;
}

// kFS signals per warp, kW warps per CTA
template <int kFS, int kW>
__global__ void __launch_bounds__(32 * kW, 2) find_small_f32_kernel(FindArgs a, int tile_rows) {
  static_assert(kFS == 1 || kFS == 2 || kFS == 4 || kFS == 8, "signals per warp");
  // A0[npad] {ax0,ax1,ay0,ay1}, A1[npad] {az0,az1,w0,w1}, pair p at sf_swz(p)
  extern __shared__ __align__(16) float4 s_u[];
  __shared__ float s_pm[kW];
  __shared__ int32_t s_cand[kW][kSfCand];  // (row << 3) | signal slot
  __shared__ double s_d[kW][kSfCand];
  __shared__ int32_t s_cid[kW][kSfCand];  // speculative path: the candidates' unit ids
  __shared__ double s_q[kW][kFS][3];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ bool s_ok, s_verdict;
#ifdef GS_PROF_TL
  unsigned long long tl[6] = {0, 0, 0, 0, 0, 0};
  SF_TL(0);
#endif
  const int npad = tile_rows / 2;  // unit pairs (tile_rows is a multiple of 128)
  float4* A0 = s_u;
  float4* A1 = s_u + npad;
  const bool tma = a.rowpos && a.rowf;
  if (threadIdx.x == 0 && tma) {
    mbar_init(&s_bar, 1);
    fence_barrier_init();
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sig0 = ((int64_t)blockIdx.x * kW + warp) * kFS;
  // signals (FP64, as the reference reads them): the sampled indices and the
  // cloud do not depend on the update, so the gather overlaps it (the
  // engine's signal buffer is written only at the end, after the update)
  double qx[kFS], qy[kFS], qz[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    const int64_t j = sig0 + k;
    qx[k] = qy[k] = qz[k] = 0.0;
    if (j < a.m) {
      if (a.sig_idx) {  // fused sampling: gather (stored for the update at the end)
        const size_t src = 3 * (size_t)a.sig_idx[j];
        qx[k] = a.sig_pts[src];
        qy[k] = a.sig_pts[src + 1];
        qz[k] = a.sig_pts[src + 2];
      } else {
        qx[k] = a.sig[3 * j];
        qy[k] = a.sig[3 * j + 1];
        qz[k] = a.sig[3 * j + 2];
      }
    }
  }
  // ---- speculative screen (the engine's batches): while the update that
  //      precedes runs, screen against the snapshot before it with the
  //      threshold widened by a bound on that update's moves (twice the
  //      previous update's largest displacement); after the update the
  //      candidates stand if it changed no row and moved nothing further
  bool spec = false;
  float dspec = 0.f;
  int n_prev = 0;
  int cnt = 0;
  bool full_scan = false;
  uint32_t par = 0;
  const int ncopy = (int)(npad < a.rowf_stride ? (int64_t)npad : a.rowf_stride);
  if (a.rowf_prev && tma) {
    n_prev = *a.rowpos_n_prev;
    const float dprev = __uint_as_float(*a.disp_prev);
    dspec = __fadd_ru(__fmul_ru(2.f, dprev), 1e-30f);
    spec = n_prev >= 2 && n_prev <= tile_rows && dprev < 1e30f;  // (inf: rows changed)
    if (spec) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&s_bar, 2u * 16u * (uint32_t)ncopy);
        tma_bulk_g2s(A0, a.rowf_prev, 16u * (uint32_t)ncopy, &s_bar);
        tma_bulk_g2s(A1, a.rowf_prev + a.rowf_stride, 16u * (uint32_t)ncopy, &s_bar);
      }
      mbar_wait(&s_bar, 0);
      par = 1;
      cnt = sf_screen<kFS>(A0, A1, n_prev, a.fcen_prev[0], a.fcen_prev[1], a.fcen_prev[2],
                           __uint_as_float(*a.fpm_prev), dspec, qx, qy, qz, lane, s_cand[warp],
                           s_q[warp], full_scan);
      // the candidates' unit ids now (the rows stand if the candidates do):
      // the records need no row -> id load after the update
      __syncwarp();
      if (!full_scan && cnt <= kSfCand)
        for (int c = lane; c < cnt; c += 32) s_cid[warp][c] = a.rows[s_cand[warp][c] >> 3];
    }
  }
  // launched as a programmatic dependent of the previous kernel (the update):
  // every CTA may already be resident; start once the update's row snapshot
  // is published (its token), or when that grid has completed
#ifdef GS_PROF_TL
  if (threadIdx.x == 0 && a.tl_batch >= 0) {
    const unsigned long long tp = gtimer();
    unsigned long long* g2 = g_tlf2[a.tl_batch & 8191];
    if (blockIdx.x == 0) {
      g2[0] = tl[0];
      g2[1] = tp;
    }
    atomicMax(&g2[2], tp);
  }
#endif
  bool waited = false;
  bool verdict = false;  // the update's: the speculative candidates stand
  if (a.snap_token) {
    if (threadIdx.x < 32) {  // warp 0: lane q polls the flag of update CTA q
      const int lane = threadIdx.x;
      const bool mine = lane < a.snap_parts;
      int spins = 0;
      int t = 0;
      bool done;
      do {
        if (mine) {
#if GS_POLL_ACQ
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(t) : "l"(a.snap_token + lane) : "memory");
#else
          asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(t) : "l"(a.snap_token + lane) : "memory");
#endif
        }
        done = __all_sync(0xffffffffu, !mine || (t >> 1) - a.snap_target >= 0);
        if (done) break;
#if GS_POLL_NS > 0
        __nanosleep(GS_POLL_NS);
#endif
      } while (++spins < (1 << 20));
#if !GS_POLL_ACQ
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire after the flags
#endif
      const bool v = __all_sync(0xffffffffu, !mine || ((t >> 1) == a.snap_target && (t & 1)));
      if (lane == 0) {
        s_ok = done;
        s_verdict = done && v;
      }
    }
    __syncthreads();
    waited = !s_ok;
    verdict = s_verdict;
  } else {
    waited = true;
  }
  if (waited) asm volatile("griddepcontrol.wait;" ::: "memory");
  // ... and let the update (16 SMs) become resident on the SMs this grid
  // leaves free; it waits for this grid's records in turn
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  SF_TL(1);
  // the speculative candidates hold if the update changed no row and moved
  // none by more than the bound: its verdict, in the token (CTA-uniform)
  const bool spec_ok = spec && verdict;
  const int64_t n = spec_ok ? n_prev : a.n_dev ? (int64_t)*a.n_dev : a.n;
  const bool compact = spec_ok || (a.rowpos && *a.rowpos_n == n);
  if (!spec_ok) {
    if (spec) {
      full_scan = false;
      cnt = 0;
    }
    // the update left the rows as swizzled FP32 unit pairs: two bulk copies of
    // the whole tile (at most rowf_stride pairs); used only if that snapshot
    // describes the current rows
    if (threadIdx.x == 0 && tma) {
      if (spec) fence_proxy_async_smem();  // the speculative screen's reads come first
      mbar_expect_tx(&s_bar, 2u * 16u * (uint32_t)ncopy);
      tma_bulk_g2s(A0, a.rowf, 16u * (uint32_t)ncopy, &s_bar);
      tma_bulk_g2s(A1, a.rowf + a.rowf_stride, 16u * (uint32_t)ncopy, &s_bar);
    }
    full_scan = n > tile_rows;  // the host estimate went stale (batches in flight)
    // the copies complete on the mbarrier whatever path follows
    if (tma) mbar_wait(&s_bar, par);
  }
  if (!spec_ok && !full_scan) {
    const int nr = (int)n;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    float pm = 0.f;
    if (compact && tma) {
      // the update kernel left these rows as FP32 unit pairs (same centre
      // rule, same bound, same swizzle): already staged
      cx = a.fcen[0];
      cy = a.fcen[1];
      cz = a.fcen[2];
      pm = __uint_as_float(*a.fpm_bits);
    } else {
      __syncthreads();  // every thread saw the copies land before they are overwritten
      // centre: row 0 rounded to FP32 (any centre is valid; the bound uses Pmax)
      if (nr > 0) {
        double x, y, z;
        if (sf_row(a, compact, 0, x, y, z) && fabs(x) < 1e30 && fabs(y) < 1e30 && fabs(z) < 1e30) {
          cx = (double)__double2float_rn(x);
          cy = (double)__double2float_rn(y);
          cz = (double)__double2float_rn(z);
        }
      }
      // stage the FP32 unit pairs; max-norm of P' for Pmax.  Four pairs per
      // thread per step with every load issued before any use (one memory
      // latency per step, not one per row).
      const double kInf = __longlong_as_double(0x7ff0000000000000LL);
      for (int p0 = threadIdx.x; p0 < npad; p0 += 4 * 32 * kW) {
        double X[8], Y[8], Z[8];
  #pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int r = 2 * (p0 + (t >> 1) * 32 * kW) + (t & 1);
          X[t] = Y[t] = Z[t] = kInf;
          if (r < nr) {
            if (compact) {
              X[t] = a.rowpos[r];
              Y[t] = a.rowpos[a.rowpos_stride + r];
              Z[t] = a.rowpos[2 * a.rowpos_stride + r];
            } else if (!load_row(a, r, X[t], Y[t], Z[t])) {
              X[t] = kInf;
            }
          }
        }
  #pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = p0 + q * 32 * kW;
          if (p >= npad) break;
          float ax[2], ay[2], az[2], w[2];
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double x = X[2 * q + h], y = Y[2 * q + h], z = Z[2 * q + h];
            ax[h] = ay[h] = az[h] = 0.f;
            w[h] = INFINITY;
            // a row with a non-finite coordinate has d2 = inf or NaN for every
            // signal and is never selected (nor are dead rows, +inf here and
            // in the update's row snapshot): it is left out like a dead one
            if (isfinite(x) && isfinite(y) && isfinite(z)) {
              const float px = __double2float_rn(x - cx), py = __double2float_rn(y - cy),
                          pz = __double2float_rn(z - cz);
              ax[h] = -2.f * px;
              ay[h] = -2.f * py;
              az[h] = -2.f * pz;
              w[h] = __double2float_rn((double)px * px + (double)py * py + (double)pz * pz);
              const float mn = fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz)));
              pm = (mn == mn) ? fmaxf(pm, mn) : INFINITY;  // NaN poisons Pmax
            }
          }
          A0[sf_swz(p)] = make_float4(ax[0], ax[1], ay[0], ay[1]);
          A1[sf_swz(p)] = make_float4(az[0], az[1], w[0], w[1]);
        }
      }
  #pragma unroll
      for (int o = 16; o > 0; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
      if (lane == 0) s_pm[warp] = pm;
      __syncthreads();
      pm = s_pm[0];
  #pragma unroll
      for (int k = 1; k < kW; ++k) pm = fmaxf(pm, s_pm[k]);
    }
    SF_TL(2);
    cnt = sf_screen<kFS>(A0, A1, nr, cx, cy, cz, pm, 0.f, qx, qy, qz, lane, s_cand[warp], s_q[warp],
                         full_scan);
    SF_TL(3);
  }
  {
    if (!full_scan && cnt <= kSfCand) {
      __syncwarp();
      SF_TL(4);
      for (int c = lane; c < cnt; c += 32) {  // exact FP64 distance per candidate
        const int code = s_cand[warp][c];
        const int r = code >> 3, k = code & 7;
        double x, y, z;
        double d = __longlong_as_double(0x7ff8000000000000LL);  // NaN: never selected
        if (sf_row(a, compact, r, x, y, z))
          d = dist2_exact(x, y, z, s_q[warp][k][0], s_q[warp][k][1], s_q[warp][k][2]);
        s_d[warp][c] = d;
      }
      __syncwarp();
      if (lane < kFS) {
        Best2 b;
        b.init();
        int c1 = -1, c2 = -1;  // candidate slots of the best two (best2_lex, tracked)
        for (int c = 0; c < cnt; ++c) {
          const int code = s_cand[warp][c];
          if ((code & 7) != lane) continue;
          const double d = s_d[warp][c];
          const int32_t i = code >> 3;
          if (d < b.d1 || (d == b.d1 && i < b.i1)) {
            b.d2 = b.d1;
            b.i2 = b.i1;
            c2 = c1;
            b.d1 = d;
            b.i1 = i;
            c1 = c;
          } else if (i != b.i1 && (d < b.d2 || (d == b.d2 && i < b.i2))) {
            b.d2 = d;
            b.i2 = i;
            c2 = c;
          }
        }
        const int64_t j = sig0 + lane;
        if (j < a.m) {
          if (spec_ok && a.out_win && !a.out_idx) {  // ids staged with the candidates
            WinRec w;
            w.b = c1 >= 0 ? s_cid[warp][c1] : -1;
            w.s = c2 >= 0 ? s_cid[warp][c2] : -1;
            w.dwin = __dsqrt_rn(b.d1);  // math.sqrt (correctly rounded): multi.py:72-78
            a.out_win[j] = w;
            if (a.firstwin && j < a.fw_limit && w.b >= 0 && w.s >= 0 && w.b != w.s)
              atomicMin(&a.firstwin[w.b], (int32_t)j);
          } else {
            write_result(a, j, b);
          }
        }
      }
      sf_store_signals<kFS>(a, sig0, lane, qx, qy, qz);
#ifdef GS_PROF_TL
      SF_TL(5);
      if (threadIdx.x == 0 && a.tl_batch >= 0) {
        unsigned long long* g = g_tlf[a.tl_batch & 8191];
        if (blockIdx.x == 0) g[0] = tl[1];
        atomicMax(&g[1], tl[5]);
        atomicAdd(&g[2], 1ull);
      }
      __shared__ unsigned s_seq;
      if (threadIdx.x == 0) s_seq = *(volatile unsigned*)&g_sf_seq;
      __syncthreads();
      if (threadIdx.x == 0 && s_seq + 100 >= GS_PROF_TL && s_seq < GS_PROF_TL + 3 && GS_PROF_TL > 0) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        printf("F %u %u %u %llu %llu %llu %llu %llu %llu\n", s_seq, blockIdx.x, smid, tl[0],
               tl[1], tl[2], tl[3], tl[4], tl[5]);
      }
      if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_sf_seq, 1u);
#endif
      // complete only after the update grid has (the next update relies on it)
      if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
      return;
    }
    full_scan = true;
  }
  // exact FP64 scan of every row (stale estimate, degenerate inputs, mass ties)
  Best2 b[kFS];
#pragma unroll
  for (int k = 0; k < kFS; ++k) b[k].init();
  for (int64_t r = lane; r < n; r += 32) {
    double x, y, z;
    if (!sf_row(a, compact, r, x, y, z)) continue;
#pragma unroll
    for (int k = 0; k < kFS; ++k) b[k].push(dist2_exact(x, y, z, qx[k], qy[k], qz[k]), (int32_t)r);
  }
#pragma unroll
  for (int k = 0; k < kFS; ++k) {
    warp_best2_merge(b[k]);
    const int64_t j = sig0 + k;
    if (lane == 0 && j < a.m) write_result(a, j, b[k]);
  }
  sf_store_signals<kFS>(a, sig0, lane, qx, qy, qz);
  if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// materialise sampled signals (sig[j] = pts[idx[j]]) for the non-fused finds
__global__ void k_gather_signals(const int64_t* idx, const double* pts, double* sig, int64_t m) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const size_t src = 3 * (size_t)idx[j];
  sig[3 * j] = pts[src];
  sig[3 * j + 1] = pts[src + 1];
  sig[3 * j + 2] = pts[src + 2];
}

void gather_signals_launch(const int64_t* idx, const double* pts, double* sig, int64_t m,
                           cudaStream_t stream) {
  if (m <= 0) return;
  k_gather_signals<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(idx, pts, sig, m);
  GS_CUDA(cudaGetLastError());
  ++g_launches;
}

// forward declarations (filter.cu, grid.cu)
bool find_filter_launch(Ctx& ctx, const FindArgs& a, cudaStream_t stream, DevBuf& work);
void find_grid_launch(Ctx& ctx, const FindArgs& a, cudaStream_t stream, DevBuf& work);

void find_launch(Ctx& ctx, const FindArgs& a_in, cudaStream_t stream, DevBuf& work) {
  if (a_in.m <= 0) return;
  FindArgs a = a_in;
  // AUTO: the grid for large scans (its ~10 launches are amortised), which
  // is where the FP32 filter ran before it (1e6 signals: 0.7-0.8 ms at any
  // n from 1e4 to 1e6 against 1.8-147 ms)
  const bool use_grid = a.mode == GS_FIND_GRID ||
                    (a.mode == GS_FIND_AUTO && a.n > kSfMaxRows && (double)a.n * (double)a.m >= 6.0e7);
  const bool small = !use_grid && a.n <= kSmallMaxRows &&
                     !((a.mode == GS_FIND_FILTER) || (a.mode == GS_FIND_AUTO && a.n >= 4096 &&
                                                      (double)a.n * (double)a.m >= 6.0e7));
  if (a.sig_idx && !small) {  // only the small kernel gathers in place
    k_gather_signals<<<(unsigned)((a.m + 255) / 256), 256, 0, stream>>>(
        a.sig_idx, a.sig_pts, const_cast<double*>(a.sig), a.m);
    GS_CUDA(cudaGetLastError());
    ++g_launches;
    a.sig_idx = nullptr;
    a.sig_pts = nullptr;
  }
  if (use_grid) {
    find_grid_launch(ctx, a, stream, work);
    return;
  }
  if ((a.mode == GS_FIND_FILTER || a.mode == GS_FIND_AUTO) &&
      find_filter_launch(ctx, a, stream, work))
    return;
  if (a.mode != GS_FIND_EXACT && a.n <= kSfMaxRows) {
    // signals per warp and warps per CTA: enough CTAs for every SM, each
    // staged row pair feeding as many signals as that allows (pass 1 is
    // bound by shared-memory wavefronts: 8 signals per load at cfg3's m)
    static int fs_env = -1;
    if (fs_env < 0) {
      const char* e = getenv("GS_SF_FS");
      fs_env = e ? atoi(e) : 0;
    }
    const int64_t sms = ctx.sm_count;
    int fs = fs_env, w = 8;
    if (fs != 1 && fs != 2 && fs != 4 && fs != 8) {
      // the most signals per warp that still gives most SMs two 8-warp CTAs
      // (the second hides the first one's staging; measured on cfg3: 2 at
      // m = 4096 beats 4 and 8)
      fs = 1;
      for (int c : {8, 4, 2})
        if (a.m * 100 >= (int64_t)170 * 8 * c * sms) { fs = c; break; }
    }
    if (fs >= 4) w = 4;
    // rows staged: the estimate plus headroom for growth in flight, a
    // multiple of 128 (whole 64-pair steps)
    const int tile_rows = (int)std::min<int64_t>(
        kSfMaxRows, ((std::max<int64_t>(a.n, 1) + 512 + 127) / 128) * 128);
    const size_t smem = 16 * (size_t)tile_rows;
    const unsigned grid = (unsigned)((a.m + w * fs - 1) / (w * fs));  // a warp owns fs signals
    // programmatic dependent launch: the CTAs become resident while the
    // previous kernel (the 16-SM update) still runs and wait in-kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * w);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool sf_attr = false;
    if (!sf_attr) {
      for (auto kern : {find_small_f32_kernel<8, 4>, find_small_f32_kernel<4, 4>,
                        find_small_f32_kernel<2, 8>, find_small_f32_kernel<2, 4>,
                        find_small_f32_kernel<1, 8>, find_small_f32_kernel<1, 4>})
        GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     16 * kSfMaxRows));
      sf_attr = true;
    }
    auto go = [&](void (*kern)(FindArgs, int)) {
      GS_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tile_rows));
    };
    if (fs == 8) go(find_small_f32_kernel<8, 4>);
    else if (fs == 4) go(find_small_f32_kernel<4, 4>);
    else if (fs == 2 && w == 8) go(find_small_f32_kernel<2, 8>);
    else if (fs == 2) go(find_small_f32_kernel<2, 4>);
    else if (w == 8) go(find_small_f32_kernel<1, 8>);
    else go(find_small_f32_kernel<1, 4>);
    GS_CUDA(cudaGetLastError());
    ++g_launches;
    return;
  }
  if (a.n <= kSmallMaxRows) {
    static bool attr_set = false;
    if (!attr_set) {
      const int bytes = 24 * kSmallMaxRows;
      GS_CUDA(cudaFuncSetAttribute(find_small_kernel<1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      GS_CUDA(cudaFuncSetAttribute(find_small_kernel<2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      GS_CUDA(cudaFuncSetAttribute(find_small_kernel<4>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      attr_set = true;
    }
    // rows staged per tile: the estimate plus headroom for growth in flight
    const int tile_rows = (int)std::min<int64_t>(kSmallMaxRows, std::max<int64_t>(a.n, 1) + 512);
    const size_t smem = 24 * (size_t)tile_rows;
    const int64_t per1 = kSmallThreads / kSmallSlices;
    // signals per thread: the fewest CTAs that still cover every SM once
    // (each CTA re-stages all rows, so fewer, fuller CTAs win)
    const int64_t sms = ctx.sm_count;
    if (a.m >= 4 * per1 * sms) {
      find_small_kernel<4><<<(unsigned)((a.m + 4 * per1 - 1) / (4 * per1)), kSmallThreads, smem,
                             stream>>>(a, tile_rows);
    } else if (a.m >= 2 * per1 * sms * 2) {
      find_small_kernel<2><<<(unsigned)((a.m + 2 * per1 - 1) / (2 * per1)), kSmallThreads, smem,
                             stream>>>(a, tile_rows);
    } else {
      find_small_kernel<1><<<(unsigned)((a.m + per1 - 1) / per1), kSmallThreads, smem, stream>>>(
          a, tile_rows);
    }
    GS_CUDA(cudaGetLastError());
    ++g_launches;
    return;
  }
  // few signals -> one per thread and more row chunks; many -> 4 per thread
  const int fs = a.m >= 4LL * ctx.sm_count * kFT * 4 ? 4 : 1;
  const int64_t per_cta = (int64_t)kFT * fs;
  const int64_t gx = (a.m + per_cta - 1) / per_cta;
  const int64_t target = 4LL * ctx.sm_count;
  int64_t nchunks = std::max<int64_t>(1, (target + gx - 1) / gx);
  nchunks = std::min<int64_t>(nchunks, std::max<int64_t>(1, (a.n + kMinChunk - 1) / kMinChunk));
  nchunks = std::min<int64_t>(nchunks, 65535);
  int64_t rows_per_chunk = (a.n + nchunks - 1) / nchunks;
  if (rows_per_chunk < 1) rows_per_chunk = 1;
  nchunks = std::max<int64_t>(1, (a.n + rows_per_chunk - 1) / rows_per_chunk);
  if (a.n == 0) nchunks = 1;
  Part* part = nullptr;
  if (nchunks > 1) part = (Part*)work.get(sizeof(Part) * (size_t)nchunks * (size_t)a.m);
  dim3 grid((unsigned)gx, (unsigned)nchunks);
  if (fs == 4)
    find_exact_kernel<4><<<grid, kFT, 0, stream>>>(a, rows_per_chunk, part);
  else
    find_exact_kernel<1><<<grid, kFT, 0, stream>>>(a, rows_per_chunk, part);
  GS_CUDA(cudaGetLastError());
  ++g_launches;
  if (nchunks > 1) {
    find_merge_kernel<<<(unsigned)((a.m + 255) / 256), 256, 0, stream>>>(a, (int)nchunks, part);
    GS_CUDA(cudaGetLastError());
    ++g_launches;
  }
}

}  // namespace gs

using namespace gs;

// ---------------------------------------------------------------------------
// kernel-backend protocol (kernels/__init__.py:6-7): host buffers in and out.

extern "C" gs_status gs_scan_best_two_into(gs_ctx* ctx, const double* pos, int64_t n_rows,
                                           int64_t n, const double* signals, int64_t m,
                                           int64_t* out_idx, int64_t out_rows, double* out_d2,
                                           int64_t out_d2_rows, int64_t tile) {
  return guarded([&] {
    GS_CHECK(ctx, GS_VALUE_ERROR, "null context");
    GS_CHECK(n >= 0 && n <= n_rows, GS_VALUE_ERROR, "n exceeds the position array");
    GS_CHECK(m >= 0 && out_rows >= m && out_d2_rows >= m, GS_VALUE_ERROR,
             "output arrays are smaller than the signal batch");
    GS_CHECK(tile >= 1, GS_VALUE_ERROR, "tile must be >= 1");
    if (m == 0) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    GS_CUDA(cudaSetDevice(ctx->device));
    const size_t pos_b = sizeof(double) * 3 * (size_t)std::max<int64_t>(n, 1);
    const size_t sig_b = sizeof(double) * 3 * (size_t)m;
    const size_t idx_b = sizeof(int64_t) * 2 * (size_t)m;
    const size_t d2_b = sizeof(double) * 2 * (size_t)m;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char* d = (char*)ctx->ensure_device(al(pos_b) + al(sig_b) + al(idx_b) + al(d2_b));
    double* d_pos = (double*)d;
    double* d_sig = (double*)(d + al(pos_b));
    int64_t* d_idx = (int64_t*)(d + al(pos_b) + al(sig_b));
    double* d_d2 = (double*)(d + al(pos_b) + al(sig_b) + al(idx_b));
    cudaStream_t st = ctx->stream;
    if (n > 0) GS_CUDA(cudaMemcpyAsync(d_pos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    GS_CUDA(cudaMemcpyAsync(d_sig, signals, sig_b, cudaMemcpyHostToDevice, st));
    FindArgs a;
    a.pos = d_pos;
    a.n = n;
    a.sig = d_sig;
    a.m = m;
    a.out_idx = d_idx;
    a.out_d2 = d_d2;
    a.mode = GS_FIND_AUTO;
    find_launch(*ctx, a, st, ctx->find_work);
    GS_CUDA(cudaMemcpyAsync(out_idx, d_idx, idx_b, cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaMemcpyAsync(out_d2, d_d2, d2_b, cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" gs_status gs_best_two_single(gs_ctx* ctx, const double* pos, int64_t n_rows, int64_t n,
                                        double x, double y, double z, int64_t* r1, int64_t* r2,
                                        double* d2_1, double* d2_2) {
  const double sig[3] = {x, y, z};
  int64_t idx[2];
  double d2[2];
  gs_status st = gs_scan_best_two_into(ctx, pos, n_rows, n, sig, 1, idx, 1, d2, 1, 1);
  if (st != GS_OK) return st;
  *r1 = idx[0];
  *r2 = idx[1];
  *d2_1 = d2[0];
  *d2_2 = d2[1];
  return GS_OK;
}

extern "C" gs_status gs_find_device(gs_ctx* ctx, const double* d_pos, int64_t n,
                                    const double* d_sig, int64_t m, int64_t* d_idx, double* d_d2,
                                    int mode, void* stream) {
  return guarded([&] {
    GS_CHECK(ctx, GS_VALUE_ERROR, "null context");
    GS_CHECK(n >= 0 && m >= 0, GS_VALUE_ERROR, "negative size");
    GS_CHECK(mode >= 0 && mode <= 4, GS_VALUE_ERROR, "bad find mode");
    FindArgs a;
    a.pos = d_pos;
    a.n = n;
    a.sig = d_sig;
    a.m = m;
    a.out_idx = d_idx;
    a.out_d2 = d_d2;
    a.mode = mode;
    std::lock_guard<std::mutex> lk(ctx->mu);
    find_launch(*ctx, a, stream ? (cudaStream_t)stream : ctx->stream, ctx->find_work);
  });
}

extern "C" gs_status gs_find_last_fallbacks(gs_ctx* ctx, int64_t* count) {
  int64_t both[2];
  const gs_status st = gs_find_last_fallback_counts(ctx, both);
  if (st == GS_OK && count) *count = both[0];
  return st;
}

extern "C" gs_status gs_find_last_fallback_counts(gs_ctx* ctx, int64_t out[2]) {
  return guarded([&] {
    GS_CHECK(ctx && out, GS_VALUE_ERROR, "null argument");
    unsigned v[2] = {0u, 0u};
    if (ctx->d_fallbacks) {
      GS_CUDA(cudaDeviceSynchronize());
      GS_CUDA(cudaMemcpy(v, ctx->d_fallbacks, sizeof(v), cudaMemcpyDeviceToHost));
    }
    out[0] = (int64_t)v[0];
    out[1] = (int64_t)v[1];
  });
}
