// common.cuh -- shared helpers for the growsurf B200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>

#include "growsurf_b200.h"

// ---------------------------------------------------------------------------
// error plumbing: every C entry point returns gs_status and records a
// thread-local message retrievable with gs_last_error().

namespace gs {

void set_error(const std::string& msg);

struct Fail {
  gs_status code;
};

#define GS_CUDA(expr)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      ::gs::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));               \
      throw ::gs::Fail{GS_CUDA_ERROR};                                                   \
    }                                                                                    \
  } while (0)

#define GS_CHECK(cond, code, msg)     \
  do {                                \
    if (!(cond)) {                    \
      ::gs::set_error(msg);           \
      throw ::gs::Fail{code};         \
    }                                 \
  } while (0)

// Run a body and translate exceptions into a gs_status.
template <class F>
gs_status guarded(F&& f) {
  try {
    f();
    return GS_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GS_CUDA_ERROR;
  }
}

// ---------------------------------------------------------------------------
// IEEE binary64 arithmetic with one rounding per written operation and no
// contraction: the reference compiles with -ffp-contract=off
// (pkg/setup.py:38-40) and numpy never fuses.  The explicit _rn intrinsics
// keep nvcc from forming DFMA regardless of -fmad.

__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// ((dx*dx + dy*dy) + dz*dz) with dx = p - s (_scan.pyx:82-85)
__device__ __forceinline__ double dist2_exact(double px, double py, double pz, double sx,
                                              double sy, double sz) {
  const double dx = dsub(px, sx), dy = dsub(py, sy), dz = dsub(pz, sz);
  return dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
}

// strict-< best-two update (_scan.pyx:86-93): the incumbent keeps ties, so
// feeding candidates in increasing row order yields lexicographic (d, row).
struct Best2 {
  double d1, d2;
  int32_t i1, i2;
  __device__ __forceinline__ void init() {
    d1 = d2 = __longlong_as_double(0x7ff0000000000000LL);
    i1 = i2 = -1;
  }
  __device__ __forceinline__ void push(double d, int32_t i) {
    if (d < d1) {
      d2 = d1;
      i2 = i1;
      d1 = d;
      i1 = i;
    } else if (d < d2) {
      d2 = d;
      i2 = i;
    }
  }
};

// ---------------------------------------------------------------------------
// growable device buffer (never shrinks; contents not preserved on growth)

// Stream-ordered allocations from a per-device caching pool (release
// threshold unbounded): engines and samplers are created and closed per run,
// and cudaMalloc/cudaFree of their arrays (a device-wide synchronisation and
// an unmap each) cost more than a short run. dfree is ordered after the work
// already queued on `st`; memory then returns to the pool, not the driver.
void* dmalloc(size_t bytes, cudaStream_t st);
void dfree(void* p, cudaStream_t st);
// pinned host staging, cached by size for the same reason
void* hmalloc(size_t bytes);
void hfree(void* p);

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr;  // set: pool allocations ordered on st; null: cudaMalloc
  void* get(size_t bytes) {
    if (bytes > cap) {
      release();
      const size_t want = bytes + bytes / 2 + 256;
      if (st) {
        p = dmalloc(want, st);
      } else {
        GS_CUDA(cudaMalloc(&p, want));
      }
      cap = want;
    }
    return p;
  }
  void release() {
    if (p) {
      if (st)
        dfree(p, st);
      else
        cudaFree(p);
    }
    p = nullptr;
    cap = 0;
  }
};

// ---------------------------------------------------------------------------
// context

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  // growable scratch for the host-buffer kernel-backend calls
  void* d_buf = nullptr;
  size_t d_cap = 0;
  void* h_buf = nullptr;  // pinned staging
  size_t h_cap = 0;
  DevBuf find_work;  // split-n partials / filter candidates
  // find-filter fallback counter (device int)
  unsigned long long* d_fallbacks = nullptr;
  void* ensure_device(size_t bytes);
  void* ensure_host(size_t bytes);
};

// kernel launch counter (evidence for bench.py's gpu_launches)
extern unsigned long long g_launches;

}  // namespace gs

struct gs_ctx : gs::Ctx {};

// ---------------------------------------------------------------------------
// find-winners entry points shared by the backend protocol and the engine

namespace gs {

// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier helpers (filter tiles, the update kernel's window staging)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// swizzled position of FP32 unit pair p (screened find staging, update
// snapshot): within each row of 32 pairs the column is XORed with the row, so
// a warp reading pairs l, l + 32, ... (one per lane) hits 32 distinct banks
__host__ __device__ __forceinline__ int sf_swz(int p) {
  return (p & ~31) | ((p ^ (p >> 5)) & 31);
}

// generic-proxy accesses of shared memory ordered before later async-proxy
// (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Rows are read through `rows` (row -> slot) when non-null; slots whose
// `alive` byte is 0 are skipped.  Output forms:
//   out_rows_d2: (m x 2) int64 rows + (m x 2) f64 squared distances
//   out_win:     per-signal {int32 id1, int32 id2, f64 sqrt(d2_1)}
struct WinRec {
  int32_t b, s;
  double dwin;
};
static_assert(sizeof(WinRec) == GS_WINREC_BYTES, "WinRec layout is part of the C ABI");

struct FindArgs {
  const double* pos = nullptr;   // plain rows: n x 3 f64
  const double4* pos4 = nullptr; // engine slots: double4 (x, y, z, -)
  const int32_t* rows = nullptr; // engine: row -> slot
  const uint8_t* alive = nullptr;
  int64_t n = 0;                 // rows to scan (host value / upper bound)
  const int* n_dev = nullptr;    // if set: exact row count read on the device
  // engine: row-ordered positions [3][stride] valid when *rowpos_n == rows
  const double* rowpos = nullptr;
  const int* rowpos_n = nullptr;
  int64_t rowpos_stride = 0;
  // engine: FP32 unit pairs of the same snapshot (valid with rowpos), their
  // centre and max-norm bound (the screened small find copies them)
  const float4* rowf = nullptr;
  int64_t rowf_stride = 0;
  const double* fcen = nullptr;
  const unsigned* fpm_bits = nullptr;
  const double* sig = nullptr;   // m x 3 f64
  // optional fused sampling: signal j is sig_pts[sig_idx[j]] and the find
  // writes it to sig (then non-const) for the update that follows
  const int64_t* sig_idx = nullptr;
  const double* sig_pts = nullptr;
  int64_t m = 0;
  int64_t* out_idx = nullptr;
  double* out_d2 = nullptr;
  WinRec* out_win = nullptr;
  int mode = GS_FIND_AUTO;
  int tl_batch = -1;             // timeline profiling builds: the update batch this feeds
  // the engine's own batches: the record epilogue also marks each winner's
  // first signal (atomicMin) for signals < fw_limit -- the update kernel's
  // first window then starts with its candidates resolved
  int32_t* firstwin = nullptr;
  int64_t fw_limit = 0;
  // non-null: each of the preceding update's snap_parts CTAs stores
  // 2 * snap_target + verdict in snap_token[part] once its part of the row
  // snapshot is complete (the screened find starts on them, not on the
  // grid's completion; it still waits for that before it exits)
  const int* snap_token = nullptr;
  int snap_target = 0;
  int snap_parts = 0;
  // speculative screen (the screened find, engine batches): the snapshot
  // before the preceding update (its FP32 pairs, centre, max-norm, rows) and
  // the row generations / largest displacements of both snapshots
  const float4* rowf_prev = nullptr;
  const double* fcen_prev = nullptr;
  const unsigned* fpm_prev = nullptr;
  const int* rowpos_n_prev = nullptr;
  const int* gen_prev = nullptr;
  const int* gen_cur = nullptr;
  const unsigned* disp_prev = nullptr;
  const unsigned* disp_cur = nullptr;
};

// row r of a find's unit set (false: a dead engine slot)
__device__ __forceinline__ bool load_row(const FindArgs& a, int64_t r, double& x, double& y,
                                         double& z) {
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

__device__ __forceinline__ void write_result(const FindArgs& a, int64_t j, const Best2& b) {
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
    w.dwin = __dsqrt_rn(b.d1);  // math.sqrt (correctly rounded): multi.py:72-78
    a.out_win[j] = w;
    if (a.firstwin && j < a.fw_limit && w.b >= 0 && w.s >= 0 && w.b != w.s)
      atomicMin(&a.firstwin[w.b], (int32_t)j);
  }
}

// lexicographic (d2, row) insertion, any visiting order
__device__ __forceinline__ void best2_lex(Best2& b, double d, int32_t i) {
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

void find_launch(Ctx& ctx, const FindArgs& a, cudaStream_t stream, DevBuf& work);
// face-list topology on the device (mesh.cu): out[6] = distinct face edges,
// edges with > 2 faces, boundary edges, vertices with boundary degree not in
// {0, 2}, connected components over the V vertices, bad-index flag
void mesh_topology_device(Ctx& ctx, const int64_t* d_faces, int64_t F, int64_t V, int64_t out[6],
                          cudaStream_t st);
// sig[j] = pts[idx[j]] for j < m (sampled batches materialised for every rank)
void gather_signals_launch(const int64_t* idx, const double* pts, double* sig, int64_t m,
                           cudaStream_t stream);

// device CloudSource sampler (sample.cu): m signals into d_out on `stream`
void sampler_draw(gs_sampler* s, int64_t m, double* d_out, cudaStream_t stream);
// ... or just their cloud indices (the find gathers them); the cloud
void sampler_indices(gs_sampler* s, int64_t m, int64_t* d_idx, cudaStream_t stream);
const double* sampler_points(const gs_sampler* s);

}  // namespace gs
