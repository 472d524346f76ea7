// filter.cu -- FP32 find-winners filter with a certified FP64 re-check (sm_100a).
//
// Output is bit-identical to the exact path (find.cu) and so to the reference
// scan_best_two_into (pkg/src/growsurf/kernels/_scan.pyx:39-98): rows of the
// lexicographic (d2, row) best two, d2 = ((dx*dx + dy*dy) + dz*dz) in binary64.
//
// Pipeline (all on one stream, no host synchronisation):
//   1 k_bbox      bounding box of the live rows -> centre c (an FP32 value).
//   2 k_prep      every row r -> P = p - c, stored as FP32 "unit pairs"
//                 {-2Px, -2Py, -2Pz, |P|^2} for rows (2i, 2i+1) and
//                 Pmax = max |P| (rounded up).  Dead rows get |P|^2 = +inf.
//   3 k_filter    per signal Q = q - c in FP32 registers; for every unit
//                 e = |P|^2 - 2 P.Q (= d - |Q|^2) with three packed FFMA2
//                 per two units; keeps the lexicographic (e, row) top-3.
//                 Unit tiles are streamed into shared memory by TMA bulk
//                 copies (cp.async.bulk + mbarrier, double-buffered) and
//                 read as broadcasts.  Split over unit chunks when m alone
//                 cannot fill the GPU; k_filter_merge merges the partial
//                 top-3s in chunk (= row) order.
//   4 certify     the two FP32 candidates are re-evaluated EXACTLY (FP64,
//                 reference rounding).  They are the exact top-2 if every
//                 other unit is provably farther: with E = 8u(Pmax+|Q|)^2
//                 bounding |e_fp32 - e_real| (u = 2^-24; derivation in
//                 DESIGN.md), every non-candidate has
//                 d_real >= e3 - E + |Q|^2, and we require that bound to
//                 exceed both candidates' FP64 distances with margin for
//                 the FP64 roundings.  Otherwise the signal is appended to
//                 a fallback list.
//   5 k_fallback  one CTA per listed signal scans all rows in FP64 (exact
//                 reference arithmetic) and reduces the lexicographic top-2.
//
// Algorithmic work: 8 FLOP per (signal, unit) pair as in the reference
// (3 sub, 3 mul, 2 add); this kernel issues 3 FMA lanes per pair.

#include <algorithm>

#include "common.cuh"

namespace gs {

constexpr int kQT = 256;           // threads per filter CTA
constexpr int kQS = 4;             // signals per thread
constexpr int kSigPerCta = kQT * kQS;
constexpr int kTilePairs = 512;    // unit pairs (1024 units) per shared-memory tile
constexpr int kFbThreads = 256;    // fallback CTA
constexpr int kMinChunkTiles = 16; // fewest tiles (16k units) per split-n chunk: each chunk
                                   // restarts the top-3, and the warm-up inserts are slow
constexpr int kCellBits = 4;       // signal ordering: 16^3 cells in Morton order
constexpr int kCells = 1 << (3 * kCellBits);

struct __align__(16) UPair {
  float ax0, ax1, ay0, ay1;  // -2 P.x, -2 P.y for rows 2i, 2i+1
  float az0, az1, w0, w1;    // -2 P.z, |P|^2
};

struct FilterMeta {
  unsigned long long bbox[6];  // ordered-int encoded min x,y,z / max x,y,z
  double cx, cy, cz;           // centre (FP32-representable)
  unsigned int pmax_bits;      // float bits of max |P| (rounded up)
  unsigned int nlive;          // live rows scanned
  unsigned int nfb;            // fallback list length (signals the filter could not certify)
  unsigned int nexact;         // listed signals that also needed the FP64 scan
  unsigned int overflow;       // more rows than the pair array holds (host estimate stale):
                               // every signal takes the exact FP64 scan
};

struct Top3 {
  float e1, e2, e3;
  int32_t i1, i2, i3;
};

__device__ __forceinline__ unsigned long long ord_enc(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_dec(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ bool filter_row(const FindArgs& a, int64_t nrows, int64_t r, double& x,
                                           double& y, double& z) {
  if (r >= nrows) return false;
  if (a.pos4) {
    const int32_t slot = a.rows ? a.rows[r] : (int32_t)r;
    if (a.alive && !a.alive[slot]) return false;
    const double4 p = a.pos4[slot];
    x = p.x;
    y = p.y;
    z = p.z;
    return true;
  }
  x = a.pos[3 * r];
  y = a.pos[3 * r + 1];
  z = a.pos[3 * r + 2];
  return true;
}

__device__ __forceinline__ int64_t rows_of(const FindArgs& a) {
  return a.n_dev ? (int64_t)*a.n_dev : a.n;
}

__global__ void k_filter_init(FilterMeta* M, int* hist) {
  for (int i = threadIdx.x; i < kCells; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x < 3) {
    M->bbox[threadIdx.x] = ~0ULL;
    M->bbox[3 + threadIdx.x] = 0ULL;
  }
  if (threadIdx.x == 0) {
    M->pmax_bits = 0u;
    M->nfb = 0u;
    M->nlive = 0u;
    M->nexact = 0u;
    M->overflow = 0u;
  }
}

__global__ void k_bbox(FindArgs a, FilterMeta* M) {
  const int64_t nrows = rows_of(a);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double p[3];
    if (!filter_row(a, nrows, r, p[0], p[1], p[2])) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], p[k]);
      hi[k] = fmax(hi[k], p[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (lo[k] <= hi[k]) {
        atomicMin(&M->bbox[k], ord_enc(lo[k]));
        atomicMax(&M->bbox[3 + k], ord_enc(hi[k]));
      }
    }
  }
}

__device__ __forceinline__ void centre_of(const FilterMeta* M, double& cx, double& cy, double& cz) {
  double c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned long long lo = M->bbox[k], hi = M->bbox[3 + k];
    c[k] = (lo == ~0ULL) ? 0.0 : (double)__double2float_rn(0.5 * (ord_dec(lo) + ord_dec(hi)));
  }
  cx = c[0];
  cy = c[1];
  cz = c[2];
}

// rows -> FP32 unit pairs (npairs_alloc pairs; rows past the live count are +inf)
__global__ void k_prep(FindArgs a, FilterMeta* M, UPair* U, int64_t npairs_alloc) {
  const int64_t nrows = rows_of(a);
  double cx, cy, cz;
  centre_of(M, cx, cy, cz);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    M->cx = cx;
    M->cy = cy;
    M->cz = cz;
    if (nrows > 2 * npairs_alloc) M->overflow = 1u;
  }
  float pm = 0.f;
  unsigned live = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs_alloc;
       i += (int64_t)gridDim.x * blockDim.x) {
    float ax[2], ay[2], az[2], w[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double x, y, z;
      if (filter_row(a, nrows, 2 * i + h, x, y, z)) {
        const float px = __double2float_rn(x - cx), py = __double2float_rn(y - cy),
                    pz = __double2float_rn(z - cz);
        ax[h] = -2.f * px;
        ay[h] = -2.f * py;
        az[h] = -2.f * pz;
        const double n2 = (double)px * px + (double)py * py + (double)pz * pz;
        w[h] = __double2float_rn(n2);
        const double dx = x - cx, dy = y - cy, dz = z - cz;
        pm = fmaxf(pm, __double2float_ru(sqrt(dx * dx + dy * dy + dz * dz)));
        ++live;
      } else {
        ax[h] = ay[h] = az[h] = 0.f;
        w[h] = INFINITY;
      }
    }
    UPair u;
    u.ax0 = ax[0];
    u.ax1 = ax[1];
    u.ay0 = ay[0];
    u.ay1 = ay[1];
    u.az0 = az[0];
    u.az1 = az[1];
    u.w0 = w[0];
    u.w1 = w[1];
    U[i] = u;
  }
  for (int o = 16; o > 0; o >>= 1) {
    pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
    live += __shfl_xor_sync(0xffffffffu, live, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (pm > 0.f) atomicMax(&M->pmax_bits, __float_as_uint(pm));
    if (live) atomicAdd(&M->nlive, live);
  }
}

// ---------------------------------------------------------------------------
// Signal ordering.  A warp keeps going only while no lane's top-3 changes;
// the warm-up inserts (about 3 ln n per signal) make that branch common when
// a warp's signals are scattered.  Signals are therefore visited in the
// Morton order of a 16^3 grid over the units' bounding box (counting sort:
// histogram -> scan -> scatter), so a warp's signals are near each other and
// insert at the same units.  Results are written at the original indices,
// so the order never affects the output.

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 4 bits -> every third bit
  v &= 0xF;
  v = (v | (v << 4)) & 0x0C3;
  v = (v | (v << 2)) & 0x249;
  return v;
}

__device__ __forceinline__ int signal_cell(const FilterMeta* M, double x, double y, double z) {
  int c[3];
  const double q[3] = {x, y, z};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned long long lk = M->bbox[k], hk = M->bbox[3 + k];
    int v = 0;
    if (lk != ~0ULL) {
      const double lo = ord_dec(lk), hi = ord_dec(hk);
      const double t = hi > lo ? (q[k] - lo) / (hi - lo) : 0.0;
      v = (int)(t * (1 << kCellBits));  // NaN -> 0
      v = v < 0 ? 0 : (v >= (1 << kCellBits) ? (1 << kCellBits) - 1 : v);
    }
    c[k] = v;
  }
  return (int)(spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2));
}

__global__ void k_sig_hist(FindArgs a, const FilterMeta* M, int* hist) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.m;
       j += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[signal_cell(M, a.sig[3 * j], a.sig[3 * j + 1], a.sig[3 * j + 2])], 1);
}

// exclusive scan of the 4096 cell counts, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_sig_scan(int* hist) {
  __shared__ int s[1024];
  const int t = threadIdx.x;
  const int4 v = reinterpret_cast<int4*>(hist)[t];
  const int tot = v.x + v.y + v.z + v.w;
  s[t] = tot;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int add = t >= o ? s[t - o] : 0;
    __syncthreads();
    s[t] += add;
    __syncthreads();
  }
  const int base = s[t] - tot;
  reinterpret_cast<int4*>(hist)[t] = make_int4(base, base + v.x, base + v.x + v.y,
                                               base + v.x + v.y + v.z);
}

__global__ void k_sig_scatter(FindArgs a, const FilterMeta* M, int* offs, int32_t* perm) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int c = signal_cell(M, a.sig[3 * j], a.sig[3 * j + 1], a.sig[3 * j + 2]);
    perm[atomicAdd(&offs[c], 1)] = (int32_t)j;
  }
}

__device__ __forceinline__ void top3_push(Top3& t, float e, int32_t r) {
  if (e < t.e3) {
    if (e < t.e2) {
      t.e3 = t.e2;
      t.i3 = t.i2;
      if (e < t.e1) {
        t.e2 = t.e1;
        t.i2 = t.i1;
        t.e1 = e;
        t.i1 = r;
      } else {
        t.e2 = e;
        t.i2 = r;
      }
    } else {
      t.e3 = e;
      t.i3 = r;
    }
  }
}

__device__ __forceinline__ void top3_init(Top3& t) {
  t.e1 = t.e2 = t.e3 = INFINITY;
  t.i1 = t.i2 = t.i3 = -1;
}

// FP64 reference distance of row r (dead rows: +inf, never selected)
__device__ __forceinline__ double exact_d2(const FindArgs& a, int64_t nrows, int32_t r, double qx,
                                           double qy, double qz) {
  double x, y, z;
  if (!filter_row(a, nrows, r, x, y, z)) return INFINITY;
  return dist2_exact(x, y, z, qx, qy, qz);
}

__device__ __forceinline__ void write_best(const FindArgs& a, int64_t j, const Best2& b) {
  if (a.out_idx) {
    a.out_idx[2 * j] = b.i1;
    a.out_idx[2 * j + 1] = b.i2;
    a.out_d2[2 * j] = b.d1;
    a.out_d2[2 * j + 1] = b.d2;
  }
  if (a.out_win) {
    WinRec w;
    w.b = (b.i1 >= 0 && a.rows) ? a.rows[b.i1] : b.i1;
    w.s = (b.i2 >= 0 && a.rows) ? a.rows[b.i2] : b.i2;
    w.dwin = __dsqrt_rn(b.d1);  // math.sqrt: multi.py:72-78
    a.out_win[j] = w;
    if (a.firstwin && j < a.fw_limit && w.b >= 0 && w.s >= 0 && w.b != w.s)
      atomicMin(&a.firstwin[w.b], (int32_t)j);
  }
}

// Certify the FP32 top-3 of signal j and write its exact result, or list it
// for the exact fallback scan.
// Certify the FP32 top-3 of signal j and write its exact result, or list it
// for the fallback scans.  e values are relative to the signal tile's centre
// cT = c + D (D an FP32 vector, so cT is exact in binary64): e = |PT|^2 -
// 2 PT.QT with PT = p - cT, QT = q - cT.  Bound: the stored
// P' = fl32(p - c) is off by at most u(1+u)Pmax, the tile shift PT' =
// fl32(P' - D) by u|PT|, so with a >= |PT|, Q = |QT|:
//   |e_fp32 - e_real| <= f = 2 dl (a + Q) + dl^2 + 6.02u a^2 + 8.03u a Q,
//   dl = u(1+u) Pmax + u a.
// For a unit outside the top-3, e >= e3; its distance d = e + Q^2 satisfies
// d >= S - f(S) with S = e3 + Q^2 and a = sqrt(S) + Q (f grows with d).  If
// that exceeds both candidates' exact FP64 distances (less FP64 slack), the
// two candidates are the reference's best two.
__device__ void certify(const FindArgs& a, const FilterMeta* M, int64_t j, const Top3& t,
                        float Dx, float Dy, float Dz, int32_t* fb_list) {
  const int64_t nrows = rows_of(a);
  const double qx = a.sig[3 * j], qy = a.sig[3 * j + 1], qz = a.sig[3 * j + 2];
  Best2 b;
  b.init();
  // candidates in row order so strict-< gives the lexicographic (d, row) order
  int32_t c0 = t.i1, c1 = t.i2;
  if (c1 >= 0 && c1 < c0) {
    const int32_t tmp = c0;
    c0 = c1;
    c1 = tmp;
  }
  double d0 = INFINITY, d1 = INFINITY;
  if (c0 >= 0) b.push(d0 = exact_d2(a, nrows, c0, qx, qy, qz), c0);
  if (c1 >= 0) b.push(d1 = exact_d2(a, nrows, c1, qx, qy, qz), c1);
  const double Qx = qx - (M->cx + (double)Dx), Qy = qy - (M->cy + (double)Dy),
               Qz = qz - (M->cz + (double)Dz);
  const double q2 = Qx * Qx + Qy * Qy + Qz * Qz;
  const double Q = sqrt(q2);
  const double pmax = (double)__uint_as_float(M->pmax_bits);
  // FP32 values stay far from overflow below 1e30; beyond it, go exact
  bool ok = pmax * pmax <= 1e30 && q2 <= 1e30 && !M->overflow;
  if (t.i3 < 0) {
    // fewer than three finite FP32 values: certified only if every live
    // row is among the candidates
    ok = ok && M->nlive == (unsigned)((c0 >= 0) + (c1 >= 0));
  } else if (ok) {
    const double u = 0x1p-24;
    const double S = (double)t.e3 + q2;
    const double av = sqrt(fmax(S, 0.0)) + Q;
    const double dl = u * (1.0 + u) * pmax + u * av;
    // 1e-44 covers FP32 subnormal rounding (absolute, not relative)
    const double f = (2.0 * dl * (av + Q) + dl * dl + 6.02 * u * av * av + 8.03 * u * av * Q) *
                         (1.0 + 1e-6) + 1e-44;
    // FP64 slack for S, q2 and the reference's own rounding of d
    const double lower = (S - f - 1e-14 * (fabs(S) + q2 + f)) * (1.0 - 1e-14);
    ok = (b.i2 >= 0) && lower > fmax(d0, d1);
  }
  if (ok) {
    write_best(a, j, b);
  } else {
    const unsigned k = atomicAdd((unsigned*)&((FilterMeta*)M)->nfb, 1u);
    fb_list[k] = (int32_t)j;
  }
}

// The FP32 filter: grid (signal tiles, unit chunks)
__global__ void __launch_bounds__(kQT, 3)
    k_filter(FindArgs a, const FilterMeta* __restrict__ M, const UPair* __restrict__ U,
             int64_t npairs, int64_t pairs_per_chunk, const int32_t* __restrict__ perm,
             float4* __restrict__ shift, Top3* __restrict__ part, int32_t* __restrict__ fb_list) {
  __shared__ __align__(128) UPair tile[2][kTilePairs];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double s_red[6][kQT / 32];
  __shared__ float s_D[3];
  const int tid = threadIdx.x;
  const int64_t sig0 = (int64_t)blockIdx.x * kSigPerCta;
  const int64_t p_begin = (int64_t)blockIdx.y * pairs_per_chunk;
  const int64_t p_end = min(npairs, p_begin + pairs_per_chunk);
  const int ntiles = (int)((p_end - p_begin + kTilePairs - 1) / kTilePairs);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int t) {
    const int64_t p0 = p_begin + (int64_t)t * kTilePairs;
    const int cnt = (int)min((int64_t)kTilePairs, p_end - p0);
    const uint32_t bytes = (uint32_t)cnt * (uint32_t)sizeof(UPair);
    mbar_expect_tx(&bar[t & 1], bytes);
    tma_bulk_g2s(&tile[t & 1][0], U + p0, bytes, &bar[t & 1]);
  };
  if (tid == 0) {
    if (ntiles > 0) issue(0);
    if (ntiles > 1) issue(1);
  }

  // tile centre: the bounding box of this CTA's signals (spatially sorted,
  // so it is small) -> D = fl32(mid - c); every chunk of the tile computes
  // the same D, so partial e values are comparable
  const double cx = M->cx, cy = M->cy, cz = M->cz;
  {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int k = 0; k < kQS; ++k) {
      const int64_t jj = sig0 + tid + k * kQT;
      if (jj < a.m) {
        const int64_t j = perm[jj];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double v = a.sig[3 * j + d];
          lo[d] = fmin(lo[d], v);
          hi[d] = fmax(hi[d], v);
        }
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      for (int o = 16; o > 0; o >>= 1) {
        lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
        hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
      }
      if ((tid & 31) == 0) {
        s_red[d][tid >> 5] = lo[d];
        s_red[3 + d][tid >> 5] = hi[d];
      }
    }
    __syncthreads();
    if (tid < 3) {
      double l = INFINITY, h = -INFINITY;
      for (int w = 0; w < kQT / 32; ++w) {
        l = fmin(l, s_red[tid][w]);
        h = fmax(h, s_red[3 + tid][w]);
      }
      const double c = tid == 0 ? cx : (tid == 1 ? cy : cz);
      const float D = (l <= h) ? __double2float_rn(0.5 * (l + h) - c) : 0.f;
      s_D[tid] = isfinite(D) ? D : 0.f;
    }
    __syncthreads();
  }
  const float Dx = s_D[0], Dy = s_D[1], Dz = s_D[2];
  if (shift && blockIdx.y == 0 && tid == 0) shift[blockIdx.x] = make_float4(Dx, Dy, Dz, 0.f);
  const double tcx = cx + (double)Dx, tcy = cy + (double)Dy, tcz = cz + (double)Dz;  // exact
  float2 qx[kQS], qy[kQS], qz[kQS];
  Top3 t[kQS];
#pragma unroll
  for (int k = 0; k < kQS; ++k) {
    const int64_t jj = sig0 + tid + k * kQT;
    top3_init(t[k]);
    float x = 0.f, y = 0.f, z = 0.f;
    if (jj < a.m) {
      const int64_t j = perm[jj];
      x = __double2float_rn(a.sig[3 * j] - tcx);
      y = __double2float_rn(a.sig[3 * j + 1] - tcy);
      z = __double2float_rn(a.sig[3 * j + 2] - tcz);
    }
    qx[k] = make_float2(x, x);
    qy[k] = make_float2(y, y);
    qz[k] = make_float2(z, z);
  }

  for (int ti = 0; ti < ntiles; ++ti) {
    const int buf = ti & 1;
    mbar_wait(&bar[buf], (uint32_t)((ti >> 1) & 1));
    const int64_t p0 = p_begin + (int64_t)ti * kTilePairs;
    const int cnt = (int)min((int64_t)kTilePairs, p_end - p0);
    // re-centre the tile on this CTA's signals: PT = fl32(P' - D),
    // a = -2 PT, w = |PT|^2 (FP32); P' = -a/2 exactly
    for (int i = tid; i < cnt; i += kQT) {
      UPair u = tile[buf][i];
      if (u.w0 != INFINITY) {
        const float px = -0.5f * u.ax0 - Dx, py = -0.5f * u.ay0 - Dy, pz = -0.5f * u.az0 - Dz;
        u.ax0 = -2.f * px;
        u.ay0 = -2.f * py;
        u.az0 = -2.f * pz;
        u.w0 = __fmaf_rn(pz, pz, __fmaf_rn(py, py, __fmul_rn(px, px)));
      }
      if (u.w1 != INFINITY) {
        const float px = -0.5f * u.ax1 - Dx, py = -0.5f * u.ay1 - Dy, pz = -0.5f * u.az1 - Dz;
        u.ax1 = -2.f * px;
        u.ay1 = -2.f * py;
        u.az1 = -2.f * pz;
        u.w1 = __fmaf_rn(pz, pz, __fmaf_rn(py, py, __fmul_rn(px, px)));
      }
      tile[buf][i] = u;
    }
    __syncthreads();
    const UPair* T = tile[buf];
    const int32_t row0 = (int32_t)(2 * p0);
    // two unit pairs (4 units) per step: 24 independent FFMA2 chains between
    // branches; one predicate over all kQS signals keeps the common path
    // branch-free (cnt is even: the pair array is padded to an even count)
#pragma unroll 1
    for (int i = 0; i < cnt; i += 2) {
      const float4 a0 = *reinterpret_cast<const float4*>(&T[i].ax0);
      const float4 a1 = *reinterpret_cast<const float4*>(&T[i].az0);
      const float4 b0 = *reinterpret_cast<const float4*>(&T[i + 1].ax0);
      const float4 b1 = *reinterpret_cast<const float4*>(&T[i + 1].az0);
      float2 ea[kQS], eb[kQS];
      bool any = false;
#pragma unroll
      for (int k = 0; k < kQS; ++k) {
        ea[k] = __ffma2_rn(make_float2(a0.x, a0.y), qx[k], make_float2(a1.z, a1.w));
        eb[k] = __ffma2_rn(make_float2(b0.x, b0.y), qx[k], make_float2(b1.z, b1.w));
        ea[k] = __ffma2_rn(make_float2(a0.z, a0.w), qy[k], ea[k]);
        eb[k] = __ffma2_rn(make_float2(b0.z, b0.w), qy[k], eb[k]);
        ea[k] = __ffma2_rn(make_float2(a1.x, a1.y), qz[k], ea[k]);
        eb[k] = __ffma2_rn(make_float2(b1.x, b1.y), qz[k], eb[k]);
        any |= fminf(fminf(ea[k].x, ea[k].y), fminf(eb[k].x, eb[k].y)) < t[k].e3;
      }
      if (any) {
        const int32_t r = row0 + 2 * i;
#pragma unroll
        for (int k = 0; k < kQS; ++k) {
          top3_push(t[k], ea[k].x, r);
          top3_push(t[k], ea[k].y, r + 1);
          top3_push(t[k], eb[k].x, r + 2);
          top3_push(t[k], eb[k].y, r + 3);
        }
      }
    }
    __syncthreads();  // every thread is done with this buffer
    if (tid == 0 && ti + 2 < ntiles) {
      // generic-proxy writes (the re-centring) before the async-proxy refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(ti + 2);
    }
  }

#pragma unroll
  for (int k = 0; k < kQS; ++k) {
    const int64_t jj = sig0 + tid + k * kQT;
    if (jj >= a.m) continue;
    if (part)
      part[(int64_t)blockIdx.y * a.m + jj] = t[k];  // sorted position
    else
      certify(a, M, perm[jj], t[k], Dx, Dy, Dz, fb_list);
  }
}

__global__ void k_filter_merge(FindArgs a, const FilterMeta* M, int nchunks, const Top3* part,
                               const int32_t* perm, const float4* shift, int32_t* fb_list) {
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj >= a.m) return;
  Top3 t;
  top3_init(t);
  for (int c = 0; c < nchunks; ++c) {
    const Top3 p = part[(int64_t)c * a.m + jj];
    if (p.i1 >= 0) top3_push(t, p.e1, p.i1);
    if (p.i2 >= 0) top3_push(t, p.e2, p.i2);
    if (p.i3 >= 0) top3_push(t, p.e3, p.i3);
  }
  const float4 D = shift[jj / kSigPerCta];
  certify(a, M, perm[jj], t, D.x, D.y, D.z, fb_list);
}

// lexicographic (d, row) merge of two best-two records
__device__ __forceinline__ void best2_merge(Best2& b, double d, int32_t i) {
  if (i < 0) return;
  if (d < b.d1 || (d == b.d1 && i < b.i1)) {
    b.d2 = b.d1;
    b.i2 = b.i1;
    b.d1 = d;
    b.i1 = i;
  } else if (i != b.i1 && (d < b.d2 || (d == b.d2 && i < b.i2))) {
    b.d2 = d;
    b.i2 = i;
  }
}

// lexicographic (e, row) top-3 insert; rows may arrive in any order
__device__ __forceinline__ void top3_lex(Top3& t, float e, int32_t r) {
  if (r < 0) return;
  if (e < t.e3 || (e == t.e3 && r < t.i3)) {
    if (e < t.e2 || (e == t.e2 && r < t.i2)) {
      t.e3 = t.e2;
      t.i3 = t.i2;
      if (e < t.e1 || (e == t.e1 && r < t.i1)) {
        t.e2 = t.e1;
        t.i2 = t.i1;
        t.e1 = e;
        t.i1 = r;
      } else {
        t.e2 = e;
        t.i2 = r;
      }
    } else {
      t.e3 = e;
      t.i3 = r;
    }
  }
}

// Listed signals, one CTA per signal (persistent).  Tier 1: FP32 DIRECT form
// d~ = (P'-Q')^2 from the FP32 unit pairs (P' = -a/2 exactly), whose error
// grows with sqrt(d) instead of |P|^2:
//   |d~ - d| <= E(d) = 2.01u R sqrt(d) + 5.1u d + 3.1u^2 (R + sqrt(d))^2
// (R = Pmax + |Q|), so the lexicographic top-3 is certified when
// d~3 - E(d~3) exceeds both candidates' FP64 distances.  Tier 2 (rare): the
// exact FP64 scan over the rows.
__global__ void __launch_bounds__(kFbThreads) k_fallback(FindArgs a, const FilterMeta* M,
                                                         const UPair* __restrict__ U,
                                                         int64_t npairs,
                                                         const int32_t* fb_list) {
  __shared__ double s_d[2][kFbThreads / 32];
  __shared__ int32_t s_i[2][kFbThreads / 32];
  __shared__ float s_e[3][kFbThreads / 32];
  __shared__ int32_t s_r[3][kFbThreads / 32];
  __shared__ int s_ok;
  const int64_t nrows = rows_of(a);
  const unsigned nfb = M->nfb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (unsigned f = blockIdx.x; f < nfb; f += gridDim.x) {
    const int64_t j = fb_list[f];
    const double qx = a.sig[3 * j], qy = a.sig[3 * j + 1], qz = a.sig[3 * j + 2];
    // ---- tier 1: FP32 direct form
    const double Qx = qx - M->cx, Qy = qy - M->cy, Qz = qz - M->cz;
    const float fx = __double2float_rn(Qx), fy = __double2float_rn(Qy), fz = __double2float_rn(Qz);
    Top3 t;
    top3_init(t);
    for (int64_t p = threadIdx.x; p < (M->overflow ? 0 : npairs); p += kFbThreads) {
      const UPair u = U[p];
      if (u.w0 != INFINITY) {
        const float dx = -0.5f * u.ax0 - fx, dy = -0.5f * u.ay0 - fy, dz = -0.5f * u.az0 - fz;
        top3_push(t, dx * dx + dy * dy + dz * dz, (int32_t)(2 * p));
      }
      if (u.w1 != INFINITY) {
        const float dx = -0.5f * u.ax1 - fx, dy = -0.5f * u.ay1 - fy, dz = -0.5f * u.az1 - fz;
        top3_push(t, dx * dx + dy * dy + dz * dz, (int32_t)(2 * p + 1));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Top3 o3;
      o3.e1 = __shfl_xor_sync(0xffffffffu, t.e1, o);
      o3.e2 = __shfl_xor_sync(0xffffffffu, t.e2, o);
      o3.e3 = __shfl_xor_sync(0xffffffffu, t.e3, o);
      o3.i1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
      o3.i2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
      o3.i3 = __shfl_xor_sync(0xffffffffu, t.i3, o);
      top3_lex(t, o3.e1, o3.i1);
      top3_lex(t, o3.e2, o3.i2);
      top3_lex(t, o3.e3, o3.i3);
    }
    if (lane == 0) {
      s_e[0][w] = t.e1;
      s_e[1][w] = t.e2;
      s_e[2][w] = t.e3;
      s_r[0][w] = t.i1;
      s_r[1][w] = t.i2;
      s_r[2][w] = t.i3;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Top3 m;
      top3_init(m);
      for (int k = 0; k < kFbThreads / 32; ++k)
        for (int q = 0; q < 3; ++q) top3_lex(m, s_e[q][k], s_r[q][k]);
      Best2 b;
      b.init();
      int32_t c0 = m.i1, c1 = m.i2;
      if (c1 >= 0 && c1 < c0) {
        const int32_t tmp = c0;
        c0 = c1;
        c1 = tmp;
      }
      double d0 = INFINITY, d1 = INFINITY;
      if (c0 >= 0) b.push(d0 = exact_d2(a, nrows, c0, qx, qy, qz), c0);
      if (c1 >= 0) b.push(d1 = exact_d2(a, nrows, c1, qx, qy, qz), c1);
      const double q2 = Qx * Qx + Qy * Qy + Qz * Qz;
      const double R = (double)__uint_as_float(M->pmax_bits) + sqrt(q2);
      bool ok = R * R <= 1e30 && !M->overflow;
      if (m.i3 < 0) {
        ok = ok && M->nlive == (unsigned)((c0 >= 0) + (c1 >= 0));
      } else if (ok) {
        const double u = 0x1p-24, s3 = (double)m.e3, rs = sqrt(fmax(s3, 0.0));
        const double E = (2.01 * u * R * rs + 5.1 * u * s3 + 3.1 * u * u * (R + rs) * (R + rs)) *
                             (1.0 + 1e-6) + 1e-44;
        const double lower = (s3 - E - 1e-13 * R * R) * (1.0 - 1e-14);
        ok = (b.i2 >= 0) && lower > fmax(d0, d1);
      }
      if (ok) write_best(a, j, b);
      s_ok = ok ? 1 : 0;
    }
    __syncthreads();
    if (s_ok) continue;  // uniform across the CTA
    // ---- tier 2: exact FP64 scan
    Best2 b;
    b.init();
    for (int64_t r = threadIdx.x; r < nrows; r += kFbThreads) {
      double x, y, z;
      if (!filter_row(a, nrows, r, x, y, z)) continue;
      b.push(dist2_exact(x, y, z, qx, qy, qz), (int32_t)r);  // rows ascend per thread
    }
    // warp reduction (lexicographic: order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od1 = __shfl_xor_sync(0xffffffffu, b.d1, o);
      const double od2 = __shfl_xor_sync(0xffffffffu, b.d2, o);
      const int32_t oi1 = __shfl_xor_sync(0xffffffffu, b.i1, o);
      const int32_t oi2 = __shfl_xor_sync(0xffffffffu, b.i2, o);
      best2_merge(b, od1, oi1);
      best2_merge(b, od2, oi2);
    }
    if (lane == 0) {
      s_d[0][w] = b.d1;
      s_d[1][w] = b.d2;
      s_i[0][w] = b.i1;
      s_i[1][w] = b.i2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Best2 r;
      r.init();
      for (int k = 0; k < kFbThreads / 32; ++k) {
        best2_merge(r, s_d[0][k], s_i[0][k]);
        best2_merge(r, s_d[1][k], s_i[1][k]);
      }
      write_best(a, j, r);
      atomicAdd((unsigned*)&((FilterMeta*)M)->nexact, 1u);
    }
    __syncthreads();
  }
}

static int g_filter_ctas_per_sm = 0;

bool find_filter_launch(Ctx& ctx, const FindArgs& a, cudaStream_t stream, DevBuf& work) {
  if (a.m <= 0) return true;
  // AUTO: the filter pays for its extra passes only on large scans
  if (a.mode == GS_FIND_AUTO && (a.n < 4096 || (double)a.n * (double)a.m < 6.0e7)) return false;
  if (a.n < 3) return false;
  if (g_filter_ctas_per_sm == 0) {
    int occ = 0;
    GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter, kQT, 0));
    g_filter_ctas_per_sm = std::max(1, occ);
  }
  const int64_t npairs = ((a.n + 3) / 4) * 2;  // even: the filter steps two pairs at a time
  const int64_t gx = (a.m + kSigPerCta - 1) / kSigPerCta;
  const int64_t ntiles_total = (npairs + kTilePairs - 1) / kTilePairs;
  // split-n: the fewest chunks whose wave quantisation keeps >= 92% of the
  // slots busy (more chunks = more top-3 warm-ups and partial traffic)
  const double resident = (double)ctx.sm_count * g_filter_ctas_per_sm;
  int64_t best_c = 1;
  double best_eff = -1.0;
  const int64_t max_c = std::max<int64_t>(1, std::min<int64_t>(64, ntiles_total / kMinChunkTiles));
  for (int64_t c = 1; c <= max_c; ++c) {
    const double waves = (double)(gx * c) / resident;
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff) {
      best_eff = eff;
      best_c = c;
    }
    if (eff >= 0.92) break;
  }
  const int64_t tiles_per_chunk = (ntiles_total + best_c - 1) / best_c;
  const int64_t pairs_per_chunk = tiles_per_chunk * kTilePairs;
  const int64_t nchunks = (npairs + pairs_per_chunk - 1) / pairs_per_chunk;

  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t meta_b = al(sizeof(FilterMeta));
  const size_t pair_b = al(sizeof(UPair) * (size_t)npairs);
  const size_t fb_b = al(sizeof(int32_t) * (size_t)a.m);
  const size_t hist_b = al(sizeof(int) * kCells);
  const size_t shift_b = al(sizeof(float4) * (size_t)gx);
  const size_t part_b = nchunks > 1 ? al(sizeof(Top3) * (size_t)nchunks * (size_t)a.m) : 0;
  char* base = (char*)work.get(meta_b + pair_b + 2 * fb_b + hist_b + shift_b + part_b);
  FilterMeta* M = (FilterMeta*)base;
  UPair* U = (UPair*)(base + meta_b);
  int32_t* fb = (int32_t*)(base + meta_b + pair_b);
  int32_t* perm = (int32_t*)(base + meta_b + pair_b + fb_b);
  int* hist = (int*)(base + meta_b + pair_b + 2 * fb_b);
  float4* shift = (float4*)(base + meta_b + pair_b + 2 * fb_b + hist_b);
  Top3* part =
      nchunks > 1 ? (Top3*)(base + meta_b + pair_b + 2 * fb_b + hist_b + shift_b) : nullptr;

  const int prep_grid = (int)std::min<int64_t>(4LL * ctx.sm_count, (npairs + 255) / 256 + 1);
  const int sig_grid = (int)std::min<int64_t>(4LL * ctx.sm_count, (a.m + 255) / 256);
  k_filter_init<<<1, 1024, 0, stream>>>(M, hist);
  k_bbox<<<prep_grid, 256, 0, stream>>>(a, M);
  k_prep<<<prep_grid, 256, 0, stream>>>(a, M, U, npairs);
  k_sig_hist<<<sig_grid, 256, 0, stream>>>(a, M, hist);
  k_sig_scan<<<1, 1024, 0, stream>>>(hist);
  k_sig_scatter<<<sig_grid, 256, 0, stream>>>(a, M, hist, perm);
  dim3 grid((unsigned)gx, (unsigned)nchunks);
  k_filter<<<grid, kQT, 0, stream>>>(a, M, U, npairs, pairs_per_chunk, perm,
                                     nchunks > 1 ? shift : nullptr, part, fb);
  if (nchunks > 1)
    k_filter_merge<<<(unsigned)((a.m + 255) / 256), 256, 0, stream>>>(a, M, (int)nchunks, part,
                                                                        perm, shift, fb);
  k_fallback<<<ctx.sm_count * 8, kFbThreads, 0, stream>>>(a, M, U, npairs, fb);
  GS_CUDA(cudaGetLastError());
  g_launches += 8 + (nchunks > 1 ? 1 : 0);
  // fallback count for gs_find_last_fallbacks (device-to-device, stays async)
  if (!ctx.d_fallbacks) GS_CUDA(cudaMalloc(&ctx.d_fallbacks, sizeof(unsigned long long)));
  GS_CUDA(cudaMemcpyAsync(ctx.d_fallbacks, &M->nfb, 2 * sizeof(unsigned),
                          cudaMemcpyDeviceToDevice, stream));
  return true;
}

}  // namespace gs
