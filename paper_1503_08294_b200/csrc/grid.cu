// grid.cu -- exact uniform-grid find-winners (GS_FIND_GRID; AUTO for large
// scans), sm_100a.
//
// Same output as the exhaustive scan, bit for bit (reference:
// scan_best_two_into, pkg/src/growsurf/kernels/_scan.pyx:39-98): the rows
// of the lexicographic (d2, row) best two, d2 in binary64 with the
// reference rounding.  The reference's own HashGrid (grid.py:98-133) is
// approximate; this one is exact because it only stops searching when no
// unvisited unit can be as close as the current second best.
//
// Build (per call, all on the stream, no host synchronisation):
//   k_grid_init / k_grid_bbox   bounding box of the finite live rows
//   k_grid_setup               cell size h and grid dims (about one unit per
//                              cell, at most kGridMaxCells cells)
//   k_grid_count               cell of every row, per-cell counts
//   k_grid_scan_*              exclusive scan -> cell start offsets
//   k_grid_scatter             rows in cell order: double4 position + row
// Query (one thread per signal):
//   visit the cells of Chebyshev shells R = 0, 1, 2, ... around the signal's
//   cell; after shell R every unvisited unit lies outside the visited box,
//   at distance >= gap (the signal's distance to the box's inner faces that
//   still have cells beyond them).  Stop when the exact second-best d2 is
//   below (gap - slack)^2 with margin (slack covers the FP64 cell
//   assignment: a unit within a few ulps of a cell face may sit in the
//   neighbouring cell).  Signals that reach kMaxShell, non-finite signals
//   and degenerate builds go to an exhaustive FP64 scan (one CTA each).
//
// Rows with a non-finite coordinate are never selected by the reference
// (their d2 is inf or NaN for every signal) and are left out of the grid.

#include <algorithm>

#include "common.cuh"

namespace gs {

namespace {

constexpr int kGridMaxCells = 1 << 23;
constexpr int kMaxShell = 6;
constexpr int kScanItems = 4096;  // per scan block (1024 threads x 4)
constexpr int kGfThreads = 256;   // exhaustive fallback CTA

struct GridMeta {
  unsigned long long bbox[6];  // order-preserving encodings (min x,y,z; max x,y,z)
  double lo[3];
  double h, inv_h, slack;
  int dim[3];
  int ncell;
  unsigned nlive;
  unsigned nfb;   // signals scanned exhaustively
  unsigned nfb2;  // copy (gs_find_last_fallback_counts reads two words)
  unsigned nsig;  // finite signals (queried in cell order)
  int bad;        // no usable grid: every signal is scanned exhaustively
};

__device__ __forceinline__ unsigned long long ord_enc(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_dec(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ int64_t nrows_of(const FindArgs& a) {
  return a.n_dev ? (int64_t)*a.n_dev : a.n;
}

__device__ __forceinline__ bool grid_row(const FindArgs& a, int64_t r, double& x, double& y,
                                         double& z) {
  return load_row(a, r, x, y, z) && isfinite(x) && isfinite(y) && isfinite(z);
}

__global__ void k_grid_init(GridMeta* M) {
  if (threadIdx.x < 3) {
    M->bbox[threadIdx.x] = ~0ULL;
    M->bbox[3 + threadIdx.x] = 0ULL;
  }
  if (threadIdx.x == 0) {
    M->nlive = 0u;
    M->nfb = 0u;
    M->nfb2 = 0u;
    M->nsig = 0u;
    M->bad = 0;
  }
}

__global__ void k_grid_bbox(FindArgs a, GridMeta* M) {
  const int64_t n = nrows_of(a);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  unsigned live = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double p[3];
    if (!grid_row(a, r, p[0], p[1], p[2])) continue;
    ++live;
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
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
  if ((threadIdx.x & 31) == 0 && live) {
    atomicAdd(&M->nlive, live);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      atomicMin(&M->bbox[k], ord_enc(lo[k]));
      atomicMax(&M->bbox[3 + k], ord_enc(hi[k]));
    }
  }
}

// cell size: about one live unit per cell over the box's extent (lower
// dimensional clouds use their area / length), at most max_cells cells
__global__ void k_grid_setup(GridMeta* M, int max_cells) {
  if (threadIdx.x != 0) return;
  if (M->nlive == 0) {
    M->bad = 1;
    return;
  }
  double lo[3], ext[3];
  double emax = 0.0, amax = 0.0;
  for (int k = 0; k < 3; ++k) {
    lo[k] = ord_dec(M->bbox[k]);
    ext[k] = ord_dec(M->bbox[3 + k]) - lo[k];
    amax = fmax(amax, fabs(lo[k]) + ext[k]);
    emax = fmax(emax, ext[k]);
  }
  if (!(emax < 1e150) || !(amax < 1e150)) {  // cell arithmetic would overflow
    M->bad = 1;
    return;
  }
  const double target = fmin((double)M->nlive, (double)max_cells);
  double h;
  double e[3] = {ext[0], ext[1], ext[2]};  // ascending
  if (e[0] > e[1]) { const double t = e[0]; e[0] = e[1]; e[1] = t; }
  if (e[1] > e[2]) { const double t = e[1]; e[1] = e[2]; e[2] = t; }
  if (e[0] > e[1]) { const double t = e[0]; e[0] = e[1]; e[1] = t; }
  const double tiny = 1e-12 * fmax(emax, 1e-300);
  if (e[0] > tiny) {
    h = cbrt(e[0] * e[1] * e[2] / target);
  } else if (e[1] > tiny) {
    h = sqrt(e[1] * e[2] / target);
  } else if (e[2] > tiny) {
    h = e[2] / target;
  } else {
    h = 1.0;  // every unit at one point: one cell
  }
  if (!(h > 0.0) || !isfinite(h)) h = fmax(emax, 1.0);
  int dim[3];
  for (int it = 0; it < 64; ++it) {
    double cells = 1.0;
    for (int k = 0; k < 3; ++k) {
      const double d = floor(ext[k] / h) + 1.0;
      dim[k] = (int)fmin(d, (double)max_cells);
      cells *= (double)dim[k];
    }
    if (cells <= (double)max_cells) break;
    h *= 1.26;
  }
  M->h = h;
  M->inv_h = 1.0 / h;
  // a unit within this distance of a cell face may have been rounded into
  // the neighbouring cell (floor((p - lo) * inv_h) in binary64)
  M->slack = 1e-9 * (amax + h);
  M->ncell = dim[0] * dim[1] * dim[2];
  for (int k = 0; k < 3; ++k) {
    M->lo[k] = lo[k];
    M->dim[k] = dim[k];
  }
}

__device__ __forceinline__ int cell_coord(double p, double lo, double inv_h, int dim) {
  const double f = floor((p - lo) * inv_h);
  return (int)fmin(fmax(f, 0.0), (double)(dim - 1));
}

__global__ void k_grid_count(FindArgs a, const GridMeta* M, int64_t cap, int* cell_of_row,
                             int* count) {
  if (M->bad) return;
  const int64_t n = nrows_of(a);
  if (n > cap) {  // more rows than the arrays were sized for (stale estimate)
    if (blockIdx.x == 0 && threadIdx.x == 0) const_cast<GridMeta*>(M)->bad = 1;
    return;
  }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x, y, z;
    int c = -1;
    if (grid_row(a, r, x, y, z)) {
      const int cx = cell_coord(x, M->lo[0], M->inv_h, M->dim[0]);
      const int cy = cell_coord(y, M->lo[1], M->inv_h, M->dim[1]);
      const int cz = cell_coord(z, M->lo[2], M->inv_h, M->dim[2]);
      c = (cz * M->dim[1] + cy) * M->dim[0] + cx;
      atomicAdd(&count[c], 1);
    }
    cell_of_row[r] = c;
  }
}

// exclusive scan of count[0, ncell) into start[0, ncell]: block sums, one
// block over the sums, then the offsets (ncell <= kGridMaxCells)
__device__ int block_scan_1024(int v, int* sh) {  // inclusive, 1024 threads
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    int s = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    sh[lane] = s;
  }
  __syncthreads();
  const int r = v + (w ? sh[w - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_grid_scan_blocks(const GridMeta* M, const int* count,
                                                           int* start, int* bsum) {
  __shared__ int sh[32];
  if (M->bad) return;
  const int nc = M->ncell;
  const int base = blockIdx.x * kScanItems;
  if (base >= nc) return;
  int v[4], t = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = base + threadIdx.x * 4 + q;
    v[q] = i < nc ? count[i] : 0;
    t += v[q];
  }
  const int inc = block_scan_1024(t, sh);
  int run = inc - t;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = base + threadIdx.x * 4 + q;
    if (i < nc) start[i] = run;
    run += v[q];
  }
  if (threadIdx.x == 1023) bsum[blockIdx.x] = inc;
}

__global__ void __launch_bounds__(1024) k_grid_scan_top(const GridMeta* M, int* bsum) {
  __shared__ int sh[32];
  if (M->bad) return;
  const int nb = (M->ncell + kScanItems - 1) / kScanItems;  // <= 2048
  int v[2], t = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = threadIdx.x * 2 + q;
    v[q] = i < nb ? bsum[i] : 0;
    t += v[q];
  }
  const int inc = block_scan_1024(t, sh);
  int run = inc - t;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = threadIdx.x * 2 + q;
    if (i < nb) bsum[i] = run;  // exclusive block offsets
    run += v[q];
  }
}

__global__ void k_grid_scan_add(const GridMeta* M, int* start, int* cursor, const int* bsum,
                                const unsigned* total) {
  if (M->bad) return;
  const int nc = M->ncell;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nc; i += gridDim.x * blockDim.x) {
    int v;
    if (i < nc) {
      v = start[i] + bsum[i / kScanItems];
    } else {
      v = (int)*total;  // start[ncell] = total
    }
    start[i] = v;
    if (i < nc) cursor[i] = v;
  }
}

// signals in cell order: a warp's signals share cells (coherent shells,
// cached cell ranges and units); non-finite signals go straight to the
// exhaustive list
__global__ void k_grid_sig_count(FindArgs a, GridMeta* M, int* sig_cell, int* scount,
                                 int32_t* fb_list) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.m) return;
  const double qx = a.sig[3 * j], qy = a.sig[3 * j + 1], qz = a.sig[3 * j + 2];
  int c = -1;
  if (!M->bad && isfinite(qx) && isfinite(qy) && isfinite(qz)) {
    const int cx = cell_coord(qx, M->lo[0], M->inv_h, M->dim[0]);
    const int cy = cell_coord(qy, M->lo[1], M->inv_h, M->dim[1]);
    const int cz = cell_coord(qz, M->lo[2], M->inv_h, M->dim[2]);
    c = (cz * M->dim[1] + cy) * M->dim[0] + cx;
    atomicAdd(&scount[c], 1);
    atomicAdd(&M->nsig, 1u);
  } else {
    fb_list[atomicAdd(&M->nfb, 1u)] = (int32_t)j;
  }
  sig_cell[j] = c;
}

__global__ void k_grid_sig_scatter(FindArgs a, const GridMeta* M, const int* sig_cell, int* scur,
                                   int32_t* perm) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.m) return;
  const int c = sig_cell[j];
  if (c >= 0) perm[atomicAdd(&scur[c], 1)] = (int32_t)j;
}

__global__ void k_grid_scatter(FindArgs a, const GridMeta* M, const int* cell_of_row, int* cursor,
                               double4* gpos) {
  if (M->bad) return;
  const int64_t n = nrows_of(a);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int c = cell_of_row[r];
    if (c < 0) continue;
    double x, y, z;
    load_row(a, r, x, y, z);
    const int slot = atomicAdd(&cursor[c], 1);
    gpos[slot] = make_double4(x, y, z, __longlong_as_double((long long)r));
  }
}

__device__ __forceinline__ void scan_cell(const int* start, const double4* gpos, int c, double qx,
                                          double qy, double qz, Best2& b) {
  const int s0 = start[c], s1 = start[c + 1];
  for (int i = s0; i < s1; ++i) {
    const double4 p = gpos[i];
    best2_lex(b, dist2_exact(p.x, p.y, p.z, qx, qy, qz), (int32_t)__double_as_longlong(p.w));
  }
}

__global__ void __launch_bounds__(256) k_grid_query(FindArgs a, const GridMeta* M,
                                                    const int* start, const double4* gpos,
                                                    const int32_t* perm, int32_t* fb_list) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (M->bad || t >= (int64_t)M->nsig) return;
  const int64_t j = perm[t];
  const double qx = a.sig[3 * j], qy = a.sig[3 * j + 1], qz = a.sig[3 * j + 2];
  const int dx = M->dim[0], dy = M->dim[1], dz = M->dim[2];
  const double h = M->h, inv_h = M->inv_h, slack = M->slack;
  const double lx = M->lo[0], ly = M->lo[1], lz = M->lo[2];
  const int cx = cell_coord(qx, lx, inv_h, dx), cy = cell_coord(qy, ly, inv_h, dy),
            cz = cell_coord(qz, lz, inv_h, dz);
  Best2 b;
  b.init();
  for (int R = 0; R <= kMaxShell; ++R) {
    const int z0 = max(cz - R, 0), z1 = min(cz + R, dz - 1);
    const int y0 = max(cy - R, 0), y1 = min(cy + R, dy - 1);
    const int x0 = max(cx - R, 0), x1 = min(cx + R, dx - 1);
    for (int iz = z0; iz <= z1; ++iz) {
      const bool zf = iz == cz - R || iz == cz + R;
      for (int iy = y0; iy <= y1; ++iy) {
        const int row = (iz * dy + iy) * dx;
        if (zf || iy == cy - R || iy == cy + R) {  // a face row: every x
          for (int ix = x0; ix <= x1; ++ix) scan_cell(start, gpos, row + ix, qx, qy, qz, b);
        } else {  // interior row: the two x faces
          if (cx - R >= 0) scan_cell(start, gpos, row + cx - R, qx, qy, qz, b);
          if (R > 0 && cx + R < dx) scan_cell(start, gpos, row + cx + R, qx, qy, qz, b);
        }
      }
    }
    // distance from q to the visited box's faces that have cells beyond
    double gap = INFINITY;
    if (cx - R > 0) gap = fmin(gap, qx - (lx + (cx - R) * h));
    if (cx + R + 1 < dx) gap = fmin(gap, (lx + (cx + R + 1) * h) - qx);
    if (cy - R > 0) gap = fmin(gap, qy - (ly + (cy - R) * h));
    if (cy + R + 1 < dy) gap = fmin(gap, (ly + (cy + R + 1) * h) - qy);
    if (cz - R > 0) gap = fmin(gap, qz - (lz + (cz - R) * h));
    if (cz + R + 1 < dz) gap = fmin(gap, (lz + (cz + R + 1) * h) - qz);
    if (gap == INFINITY) {  // the visited box is the whole grid
      write_result(a, j, b);
      return;
    }
    const double g = gap - slack;
    if (b.i2 >= 0 && g > 0.0 && b.d2 < g * g * (1.0 - 1e-12)) {
      write_result(a, j, b);
      return;
    }
  }
  fb_list[atomicAdd(&((GridMeta*)M)->nfb, 1u)] = (int32_t)j;
}

// listed signals: exhaustive FP64 scan, one CTA per signal (persistent)
__global__ void __launch_bounds__(kGfThreads) k_grid_fallback(FindArgs a, const GridMeta* M,
                                                              const int32_t* fb_list) {
  __shared__ double s_d[2][kGfThreads / 32];
  __shared__ int32_t s_i[2][kGfThreads / 32];
  const int64_t n = nrows_of(a);
  const unsigned nfb = M->nfb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (unsigned f = blockIdx.x; f < nfb; f += gridDim.x) {
    const int64_t j = fb_list[f];
    const double qx = a.sig[3 * j], qy = a.sig[3 * j + 1], qz = a.sig[3 * j + 2];
    Best2 b;
    b.init();
    for (int64_t r = threadIdx.x; r < n; r += kGfThreads) {  // ascending per thread
      double x, y, z;
      if (load_row(a, r, x, y, z)) b.push(dist2_exact(x, y, z, qx, qy, qz), (int32_t)r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od1 = __shfl_xor_sync(0xffffffffu, b.d1, o);
      const double od2 = __shfl_xor_sync(0xffffffffu, b.d2, o);
      const int32_t oi1 = __shfl_xor_sync(0xffffffffu, b.i1, o);
      const int32_t oi2 = __shfl_xor_sync(0xffffffffu, b.i2, o);
      best2_lex(b, od1, oi1);
      best2_lex(b, od2, oi2);
    }
    if (lane == 0) {
      s_d[0][w] = b.d1;
      s_d[1][w] = b.d2;
      s_i[0][w] = b.i1;
      s_i[1][w] = b.i2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Best2 m;
      m.init();
      for (int k = 0; k < kGfThreads / 32; ++k) {
        best2_lex(m, s_d[0][k], s_i[0][k]);
        best2_lex(m, s_d[1][k], s_i[1][k]);
      }
      write_result(a, j, m);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ((GridMeta*)M)->nfb2 = nfb;
}

}  // namespace

void find_grid_launch(Ctx& ctx, const FindArgs& a, cudaStream_t stream, DevBuf& work) {
  if (a.m <= 0) return;
  // arrays sized for the host's row estimate plus headroom; a device count
  // past it marks the build bad (every signal is then scanned exhaustively)
  const int64_t cap = a.n + 1024;
  const int max_cells = (int)std::min<int64_t>(kGridMaxCells, std::max<int64_t>(2 * a.n, 1));
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t meta_b = al(sizeof(GridMeta));
  const size_t row_b = al(sizeof(int) * (size_t)cap);
  const size_t cnt_b = al(sizeof(int) * ((size_t)max_cells + 1));
  const size_t bsum_b = al(sizeof(int) * 2048);
  const size_t pos_b = al(sizeof(double4) * (size_t)cap);
  const size_t fb_b = al(sizeof(int32_t) * (size_t)a.m);
  char* base = (char*)work.get(meta_b + row_b + 3 * cnt_b + bsum_b + pos_b + 3 * fb_b);
  GridMeta* M = (GridMeta*)base;
  int* cell_of_row = (int*)(base + meta_b);
  int* count = (int*)(base + meta_b + row_b);
  int* start = (int*)(base + meta_b + row_b + cnt_b);
  int* cursor = (int*)(base + meta_b + row_b + 2 * cnt_b);
  int* bsum = (int*)(base + meta_b + row_b + 3 * cnt_b);
  double4* gpos = (double4*)(base + meta_b + row_b + 3 * cnt_b + bsum_b);
  int32_t* fb = (int32_t*)(base + meta_b + row_b + 3 * cnt_b + bsum_b + pos_b);
  int* sig_cell = (int*)(base + meta_b + row_b + 3 * cnt_b + bsum_b + pos_b + fb_b);
  int32_t* perm = (int32_t*)(base + meta_b + row_b + 3 * cnt_b + bsum_b + pos_b + 2 * fb_b);

  const int rgrid = (int)std::min<int64_t>(4LL * ctx.sm_count, (cap + 255) / 256);
  const int cgrid = (int)std::min<int64_t>(4LL * ctx.sm_count, (max_cells + 256) / 256);
  k_grid_init<<<1, 32, 0, stream>>>(M);
  GS_CUDA(cudaMemsetAsync(count, 0, sizeof(int) * (size_t)max_cells, stream));
  k_grid_bbox<<<rgrid, 256, 0, stream>>>(a, M);
  k_grid_setup<<<1, 32, 0, stream>>>(M, max_cells);
  k_grid_count<<<rgrid, 256, 0, stream>>>(a, M, cap, cell_of_row, count);
  k_grid_scan_blocks<<<(max_cells + kScanItems - 1) / kScanItems, 1024, 0, stream>>>(M, count,
                                                                                    start, bsum);
  k_grid_scan_top<<<1, 1024, 0, stream>>>(M, bsum);
  k_grid_scan_add<<<cgrid, 256, 0, stream>>>(M, start, cursor, bsum, &M->nlive);
  k_grid_scatter<<<rgrid, 256, 0, stream>>>(a, M, cell_of_row, cursor, gpos);
  // signals in cell order (count -> scan -> scatter, reusing count/cursor)
  const unsigned sgrid = (unsigned)((a.m + 255) / 256);
  GS_CUDA(cudaMemsetAsync(count, 0, sizeof(int) * (size_t)max_cells, stream));
  k_grid_sig_count<<<sgrid, 256, 0, stream>>>(a, M, sig_cell, count, fb);
  k_grid_scan_blocks<<<(max_cells + kScanItems - 1) / kScanItems, 1024, 0, stream>>>(M, count,
                                                                                    cursor, bsum);
  k_grid_scan_top<<<1, 1024, 0, stream>>>(M, bsum);
  k_grid_scan_add<<<cgrid, 256, 0, stream>>>(M, cursor, count, bsum, &M->nsig);
  k_grid_sig_scatter<<<sgrid, 256, 0, stream>>>(a, M, sig_cell, count, perm);
  k_grid_query<<<sgrid, 256, 0, stream>>>(a, M, start, gpos, perm, fb);
  k_grid_fallback<<<ctx.sm_count * 4, kGfThreads, 0, stream>>>(a, M, fb);
  GS_CUDA(cudaGetLastError());
  g_launches += 15;
  if (!ctx.d_fallbacks) GS_CUDA(cudaMalloc(&ctx.d_fallbacks, sizeof(unsigned long long)));
  GS_CUDA(cudaMemcpyAsync(ctx.d_fallbacks, &M->nfb, 2 * sizeof(unsigned), cudaMemcpyDeviceToDevice,
                          stream));
}

}  // namespace gs
