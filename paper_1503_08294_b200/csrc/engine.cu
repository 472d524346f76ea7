// engine.cu -- device-resident multi-signal growing network (sm_100a).
//
// One multi-signal iteration (reference run_multi, pkg/src/growsurf/multi.py:134-202):
//   find winners against the pre-batch snapshot (find.cu)
//   -> winner-lock resolution + batch-order update (multi.py:99-131,
//      engine.py:283-355)  [k_update_batch below]
//   -> convergence check (engine.py:358-365).
//
// State layout (HBM, indexed by unit id == slot; ids are never reused,
// network.py:10): double4 positions (32 B aligned), f64 habituation and
// threshold, byte alive/ring flags, a fixed-capacity adjacency of
// kMaxDeg (neighbour id, edge id) pairs per unit, and per-edge int32 ages.
// "Rows" (the id-ordered snapshot the find scans, network.py:47-59) are an
// append-only row->id list; dead rows are skipped by the find and compacted
// away once they exceed 1/8 of the list.
//
// Update = "windowed segmented replay".  The reference applies updates one
// signal at a time.  Within a window of up to 1024 signals, as long as the
// topology does not change, the sequential result is a pure function of
// per-unit event sequences: every unit wins at most once per batch (the
// winner lock), each update touches only the winner and its neighbours, and
// positions / habituation / edge ages evolve per unit (per edge) in batch
// order.  So one thread per signal:
//   A. marks candidates (alive winner and second, winner not yet claimed);
//      the first candidate per winner is the processed signal;
//   B. evaluates, against the window-start state, whether its update would
//      change the topology or the sweep clock: a new b-s edge, an insertion
//      (d_winner > theta_b and h_b(t) < h_t, with h_b(t) reconstructed from
//      the earlier same-window decays), an edge crossing max_age, a pending
//      sweep, or isolated units waiting for prune.  The first such signal j*
//      is the "event";
//   C. commits every processed signal before j* in parallel: for each
//      touched unit the owner thread replays that unit's (signal, rate)
//      sequence in batch order with the exact binary64 rounding sequence;
//      each touched edge's age is replayed by the later of its two touching
//      signals; threshold patience / shrink (engine.py:208-265) is evaluated
//      from the reconstructed per-unit habituation at time j;
//   D. executes j* exactly as update_single on one thread (block-parallel
//      sweep scan), then restarts the window at j*+1.
// Results are bit-identical to the reference's sequential loop (tests
// compare with the C oracle and the reference golden traces).

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>
#include <map>
#include <mutex>
#include <string>

#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <nccl.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gs {

constexpr int kMaxDeg = 64;  // adjacency slots per unit (overflow -> loud error)
constexpr int32_t kNone32 = 0x7f7f7f7f;
constexpr long long kNone64 = 0x7f7f7f7f7f7f7f7fLL;
constexpr int kRingDisk = 0, kRingHalf = 1, kRingInc = 2;
#ifndef GS_UPD_THREADS
#define GS_UPD_THREADS 256
#endif
constexpr int kUpdThreads = GS_UPD_THREADS;
constexpr long long kSweepEvery = 1024;  // engine.py:98
constexpr int kAffCap = kMaxDeg * (kMaxDeg + 2) + 64;
constexpr int kDeferCap = 16384;
constexpr int kDeferSm = 512;  // deferred ring recomputes held in shared memory (event path)

enum DevError {
  E_NONE = 0,
  E_DEGREE = 1,
  E_UNIT_CAP = 2,
  E_EDGE_CAP = 3,
  E_STALE = 4,
  E_UNKNOWN = 5,
  E_SELF = 6,
  E_NOEDGE = 7,
  E_AFF = 8,
  E_BADPOS = 9,
};

struct Counters {
  long long tick, next_sweep;
  long long processed, discarded, events, windows;
  int n_units, next_id, n_edges;
  int nrows, ndead_rows;
  int ring_counts[3];
  int untrained;
  int efree_top;
  int iso_count;
  int error;
  int max_degree;
  long long ev_create, ev_insert, ev_prune, ev_sweep;
  long long cyc_serial, cyc_total;
  long long cyc_phase[12];
  int inserted_start;
  int stale_n;
  int converged;
  int nwalk, defer_n, ev_fired, ev_b;
  // the row snapshot is double-buffered (slot = batch & 1: the next find
  // reads the newest, its speculative screen the one before)
  int rowpos_n[2];  // rows described by the slot (-1: stale, the find gathers through rows)
  int deaths;    // units removed so far (an event without deaths lets the window resume)
  long long ev_cutoff;
  // minimum last_active over live units at the end of a batch (the tail
  // computes it for the next one; slot batch_no & 1 is read, the other
  // written): the silent-sweep test's value for a first window the find
  // resolved
  long long minla_next[2];
  // (unused since the row snapshot hand-off moved to per-CTA flags in
  // S.snap_token; kept so the counters keep their cache-line layout)
  unsigned long long snap_word_unused;
  int halt_on_converge, halted;  // asynchronous runs: later batches become no-ops
  long long batches;             // update kernels that ran (not halted)
  // FP32 unit pairs of the row snapshot (the screened find's staging): centre
  // (row 0 rounded to FP32) and max-norm of P' = fl32(p - centre), float bits
  double fcen[2][3];
  unsigned fpm_bits[2];
  int row_gen;          // bumped by every change of the row list (insert, death, compaction)
  int snap_gen[2];      // row_gen when the slot's snapshot was taken
  unsigned snap_disp[2];  // float bits: max displacement of any row vs the other slot (inf: rows changed)
  unsigned prof_bmax[2];  // GS_PROF_B builds: slowest B / walk chain of the window (cycles)
  int pad_;
};

struct Params {
  double eps_b, eps_n, c_b, c_n, h_t, rho;
  long long max_age, ring_patience, stale_factor;
  int allow_boundary;
};

struct DevState {
  double4* pos;
  double* hab;
  double* theta;
  uint8_t* alive;
  uint8_t* ring;
  int32_t* deg;
  int2* adj;  // [U * kMaxDeg] (neighbour id, edge id)
  int32_t* patience;
  long long* la_val;    // last_active tick, -1 when absent (engine.py:117)
  long long* la_stamp;  // dict insertion order (3*tick + role), kNone64 when absent
  int32_t* claim;       // batch number that claimed the unit (multi.py:114-130)
  int32_t* firstwin;    // window scratch: first candidate signal per winner
  int32_t* touchfirst;  // window scratch: owner signal per touched unit
  int32_t* ttr;         // window scratch: signal after which the unit is trained (walk)
  int32_t* iso_pos;     // index in iso_list or -1
  int32_t* rows;        // row -> id (append-only, id order)
  double* rowpos;       // [3][U] row-ordered positions (dead rows +inf) for the find
  float4* rowf;         // [2][rowf_stride] FP32 unit pairs of the same rows (A0, A1)
  const double* rowpos_prev;  // the other slot's rowpos (the tail's displacement bound)
  int snap;             // snapshot slot this update writes
  int32_t* eage;        // [EC]
  int32_t* efree;       // [EC] free edge-id stack
  int32_t* iso_list;    // isolated units (network.py:93 _isolated)
  long long* scratch;   // [2U] sweep (stamp, id) pairs / lonely ids
  int32_t* aff;         // [kAffCap] ring-recompute set
  int32_t* defer_list;  // [kDeferCap] deferred ring recomputes (event path)
  int* defer_n;         // non-null: recompute_ring defers (set per launch)
  int* defer_sm;        // the event path's shared-memory part of the deferred list
  Counters* cnt;
  gs_batch_stats* stats;
  // row snapshot hand-off, own 128-byte line: update CTA q stores
  // 2 * batch + (its part keeps the speculative verdict) in snap_token[q]
  // once its part of the snapshot is written; the next find's CTAs poll the
  // kCluster flags and start when all carry the batch (before the update
  // grid has drained) -- no atomics, no reset, a halted launch stores too
  int* snap_token;
  int U, EC;
  int rowf_stride;  // unit pairs per half of rowf (multiple of 64)
};

// ---------------------------------------------------------------------------
// serial primitives (one thread).  Reference: network.py.

__device__ __forceinline__ void set_err(const DevState& S, int e) {
  if (S.cnt->error == 0) S.cnt->error = e;
}

__device__ __forceinline__ void set_hab(const DevState& S, const Params& P, int u, double h) {
  const double old = S.hab[u];
  if (old >= P.h_t && h < P.h_t) S.cnt->untrained--;
  else if (old < P.h_t && h >= P.h_t) S.cnt->untrained++;
  S.hab[u] = h;
}

__device__ void iso_add(const DevState& S, int u) {
  Counters* c = S.cnt;
  const int k = c->iso_count;
  S.iso_list[k] = u;
  S.iso_pos[u] = k;
  c->iso_count = k + 1;
}

__device__ void iso_del(const DevState& S, int u) {
  Counters* c = S.cnt;
  const int k = S.iso_pos[u];
  if (k < 0) return;
  const int last = --c->iso_count;
  const int w = S.iso_list[last];
  S.iso_list[k] = w;
  S.iso_pos[w] = k;
  S.iso_pos[u] = -1;
}

__device__ __forceinline__ int find_slot(const DevState& S, int a, int b) {
  const int d = S.deg[a];
  const int2* A = S.adj + (size_t)a * kMaxDeg;
  for (int k = 0; k < d; ++k)
    if (A[k].x == b) return k;
  return -1;
}

__device__ __forceinline__ int index_in(const int2* A, int k, int w) {
  for (int i = 0; i < k; ++i)
    if (A[i].x == w) return i;
  return -1;
}

// _classify_ring: network.py:379-414
__device__ int classify_ring(const DevState& S, int u) {
  const int k = S.deg[u];
  if (k < 2) return kRingInc;
  const int2* A = S.adj + (size_t)u * kMaxDeg;
  int deg1 = 0, deg2 = 0;
  for (int a = 0; a < k; ++a) {
    const int v = A[a].x;
    const int dv = S.deg[v];
    const int2* V = S.adj + (size_t)v * kMaxDeg;
    int d = 0;
    for (int c = 0; c < dv; ++c) {
      if (index_in(A, k, V[c].x) >= 0) {
        if (++d > 2) return kRingInc;
      }
    }
    if (d == 1) deg1++;
    else if (d == 2) deg2++;
    else return kRingInc;
  }
  int shape;
  if (deg1 == 0 && deg2 == k && k >= 3) shape = kRingDisk;
  else if (deg1 == 2 && deg1 + deg2 == k) shape = kRingHalf;
  else return kRingInc;
  unsigned long long seen = 1ull, todo = 1ull;
  while (todo) {
    const int a = __ffsll((long long)todo) - 1;
    todo &= ~(1ull << a);
    const int v = A[a].x;
    const int dv = S.deg[v];
    const int2* V = S.adj + (size_t)v * kMaxDeg;
    for (int c = 0; c < dv; ++c) {
      const int idx = index_in(A, k, V[c].x);
      if (idx >= 0 && !((seen >> idx) & 1ull)) {
        seen |= 1ull << idx;
        todo |= 1ull << idx;
      }
    }
  }
  return __popcll(seen) == k ? shape : kRingInc;
}

// deferred ring recompute (event path): the first kDeferSm entries in shared
// memory, the rest in S.defer_list; duplicates are dropped when the list is
// consumed (a ring is a pure function of the final adjacency)
__device__ __forceinline__ void defer_push(const DevState& S, int u) {
  const int k = atomicAdd(S.defer_n, 1);
  if (k < kDeferSm) S.defer_sm[k] = u;
  else if (k < kDeferSm + kDeferCap) S.defer_list[k - kDeferSm] = u;
  else set_err(S, E_AFF);
}
__device__ __forceinline__ int defer_at(const DevState& S, const int* sm, int k) {
  return k < kDeferSm ? sm[k] : S.defer_list[k - kDeferSm];
}

// _recompute_ring: network.py:416-422
__device__ void recompute_ring(const DevState& S, int u) {
  if (S.defer_n) {
    // batch-kernel event path: rings are a pure function of the final
    // adjacency and only read after the topology changes, so collect the
    // affected units and reclassify them in parallel afterwards
    defer_push(S, u);
    return;
  }
  const int nw = classify_ring(S, u);
  const int old = S.ring[u];
  if (nw != old) {
    S.ring[u] = (uint8_t)nw;
    S.cnt->ring_counts[old]--;
    S.cnt->ring_counts[nw]++;
  }
}

// _ring_neighborhood: network.py:424-433 -> appended to out; returns count
__device__ int ring_neighborhood(const DevState& S, int a, int b, int32_t* out, int room) {
  int n = 0;
  const int da = S.deg[a];
  const int2* A = S.adj + (size_t)a * kMaxDeg;
  if (room < da + 2) {
    set_err(S, E_AFF);
    return 0;
  }
  for (int k = 0; k < da; ++k) {
    const int v = A[k].x;
    if (v != b && find_slot(S, b, v) >= 0) out[n++] = v;
  }
  out[n++] = a;
  out[n++] = b;
  return n;
}

// add_unit: network.py:208-230
__device__ int add_unit(const DevState& S, const Params& P, double x, double y, double z,
                        double threshold) {
  Counters* c = S.cnt;
  if (!(isfinite(x) && isfinite(y) && isfinite(z)) || !(isfinite(threshold) && threshold > 0.0)) {
    set_err(S, E_BADPOS);
    return -1;
  }
  const int id = c->next_id;
  if (id >= S.U) {
    set_err(S, E_UNIT_CAP);
    return -1;
  }
  c->next_id = id + 1;
  S.pos[id] = make_double4(x, y, z, 0.0);
  S.hab[id] = 1.0;
  S.theta[id] = threshold;
  S.alive[id] = 1;
  S.ring[id] = kRingInc;
  c->ring_counts[kRingInc]++;
  S.deg[id] = 0;
  S.patience[id] = 0;
  S.la_val[id] = -1;
  S.la_stamp[id] = kNone64;
  S.claim[id] = -1;
  S.firstwin[id] = kNone32;
  S.touchfirst[id] = kNone32;
  iso_add(S, id);
  c->n_units++;
  if (1.0 >= P.h_t) c->untrained++;
  S.rows[c->nrows++] = id;
  c->row_gen++;
  return id;
}

// _remove_edge_raw: network.py:453-462
__device__ void remove_edge_raw(const DevState& S, int a, int b) {
  Counters* c = S.cnt;
  const int ka = find_slot(S, a, b);
  if (ka < 0) {
    set_err(S, E_NOEDGE);
    return;
  }
  int2* A = S.adj + (size_t)a * kMaxDeg;
  int2* B = S.adj + (size_t)b * kMaxDeg;
  const int e = A[ka].y;
  const int da = --S.deg[a];
  A[ka] = A[da];
  const int kb = find_slot(S, b, a);
  const int db = --S.deg[b];
  B[kb] = B[db];
  S.efree[c->efree_top++] = e;
  c->n_edges--;
  if (da == 0) iso_add(S, a);
  if (db == 0) iso_add(S, b);
}

// _remove_unit_raw: network.py:464-480 (precondition: no edges)
__device__ void remove_unit_raw(const DevState& S, const Params& P, int u) {
  Counters* c = S.cnt;
  S.alive[u] = 0;
  c->n_units--;
  c->ring_counts[S.ring[u]]--;
  iso_del(S, u);
  if (S.hab[u] >= P.h_t) c->untrained--;
  c->ndead_rows++;
  c->row_gen++;
  c->deaths++;
}

// remove_unit: network.py:232-240
__device__ void remove_unit(const DevState& S, const Params& P, int u) {
  int nb[kMaxDeg];
  const int k = S.deg[u];
  const int2* U_ = S.adj + (size_t)u * kMaxDeg;
  for (int i = 0; i < k; ++i) nb[i] = U_[i].x;
  for (int i = 0; i < k; ++i) remove_edge_raw(S, u, nb[i]);
  remove_unit_raw(S, P, u);
  for (int i = 0; i < k; ++i) recompute_ring(S, nb[i]);
}

// connect_or_reset: network.py:261-282.  1 created, 0 reset, -1 error.
__device__ int connect_or_reset(const DevState& S, int a, int b) {
  Counters* c = S.cnt;
  const int k = find_slot(S, a, b);
  if (k >= 0) {
    S.eage[S.adj[(size_t)a * kMaxDeg + k].y] = 0;
    return 0;
  }
  if (S.deg[a] >= kMaxDeg || S.deg[b] >= kMaxDeg) {
    set_err(S, E_DEGREE);
    return -1;
  }
  if (c->efree_top <= 0) {
    set_err(S, E_EDGE_CAP);
    return -1;
  }
  const int e = S.efree[--c->efree_top];
  S.eage[e] = 0;
  if (S.deg[a] == 0) iso_del(S, a);
  if (S.deg[b] == 0) iso_del(S, b);
  S.adj[(size_t)a * kMaxDeg + S.deg[a]++] = make_int2(b, e);
  S.adj[(size_t)b * kMaxDeg + S.deg[b]++] = make_int2(a, e);
  c->n_edges++;
  const int dm = max(S.deg[a], S.deg[b]);
  if (dm > c->max_degree) c->max_degree = dm;
  const int n = ring_neighborhood(S, a, b, S.aff, kAffCap);
  for (int i = 0; i < n; ++i) recompute_ring(S, S.aff[i]);
  return 1;
}

// remove_edge: network.py:284-292
__device__ void remove_edge(const DevState& S, int a, int b) {
  const int n = ring_neighborhood(S, a, b, S.aff, kAffCap);
  remove_edge_raw(S, a, b);
  for (int i = 0; i < n; ++i) recompute_ring(S, S.aff[i]);
}

// age_incident_edges(b, inc, exclude): network.py:294-319.  Records the
// neighbours whose shared edge crossed max_age (the over-age registry,
// network.py:315-316; it only ever holds edges of the current winner).
__device__ int age_incident(const DevState& S, const Params& P, int b, int exclude, int inc,
                            int32_t* over, int* nover) {
  const int d = S.deg[b];
  const int2* B = S.adj + (size_t)b * kMaxDeg;
  int top = 0;
  for (int k = 0; k < d; ++k) {
    const int v = B[k].x;
    if (v == exclude) continue;
    const int e = B[k].y;
    const int old = S.eage[e];
    const int nw = old + inc;
    S.eage[e] = nw;
    if (nw > top) top = nw;
    if (over && nw > P.max_age && old <= P.max_age) over[(*nover)++] = v;
  }
  return top;
}

__device__ void sort_ll(long long* a, int n) {  // insertion sort (small n)
  for (int i = 1; i < n; ++i) {
    const long long x = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = x;
  }
}

// removes isolated units in ascending id order down to a floor of 2 units
// (network.py:355-365); returns how many were removed
__device__ int remove_lonely(const DevState& S, const Params& P) {
  Counters* c = S.cnt;
  const int n = c->iso_count;
  if (n == 0) return 0;
  long long* ids = S.scratch;
  for (int i = 0; i < n; ++i) ids[i] = S.iso_list[i];
  sort_ll(ids, n);
  int removed = 0;
  for (int i = 0; i < n; ++i) {
    if (c->n_units <= 2) break;
    remove_unit_raw(S, P, (int)ids[i]);
    removed++;
  }
  return removed;
}

// prune on the winner's over-age edges: network.py:321-369.  The removal
// order of the over-age edges cannot change the result (ring classes are a
// function of the final adjacency and every ring that can change is in the
// union of the ring neighbourhoods); lonely units go in ascending id order.
__device__ void prune_winner(const DevState& S, const Params& P, int b, const int32_t* over,
                             int nover, int* pe, int* pu) {
  *pe = 0;
  *pu = 0;
  if (nover == 0 && S.cnt->iso_count == 0) return;
  int naff = 0;
  for (int i = 0; i < nover; ++i) {
    naff += ring_neighborhood(S, b, over[i], S.aff + naff, kAffCap - naff);
    remove_edge_raw(S, b, over[i]);
  }
  *pu = remove_lonely(S, P);
  for (int i = 0; i < naff; ++i)
    if (S.alive[S.aff[i]]) recompute_ring(S, S.aff[i]);
  *pe = nover;
}

// generic prune(max_age) for the Network API (scans every edge)
__device__ void prune_all(const DevState& S, const Params& P, long long max_age, int* pe,
                          int* pu) {
  Counters* c = S.cnt;
  int npe = 0;
  for (int a = 0; a < c->next_id; ++a) {
    if (!S.alive[a]) continue;
    for (int k = 0; k < S.deg[a];) {
      const int2 ent = S.adj[(size_t)a * kMaxDeg + k];
      if (a < ent.x && S.eage[ent.y] > max_age) {
        int nb[kMaxDeg + 2];
        // ring_neighborhood into a local list, then remove
        int n = 0;
        const int da = S.deg[a];
        for (int q = 0; q < da; ++q) {
          const int v = S.adj[(size_t)a * kMaxDeg + q].x;
          if (v != ent.x && find_slot(S, ent.x, v) >= 0 && n < kMaxDeg) nb[n++] = v;
        }
        nb[n++] = a;
        nb[n++] = ent.x;
        remove_edge_raw(S, a, ent.x);
        for (int q = 0; q < n; ++q)
          if (S.alive[nb[q]]) recompute_ring(S, nb[q]);
        npe++;
        continue;  // slot k now holds a different entry
      }
      ++k;
    }
  }
  *pu = remove_lonely(S, P);
  *pe = npe;
}

// last_active[u] = tick (engine.py:305-306,339) with dict order stamps
__device__ __forceinline__ void touch_active(const DevState& S, int u, long long tick, int role) {
  if (S.la_val[u] == -1) S.la_stamp[u] = 3 * tick + role;
  S.la_val[u] = tick;
}

// _sweep_stale body over a collected (stamp, id) list: engine.py:268-280
__device__ void sweep_apply(const DevState& S, const Params& P, long long* rec, int n) {
  // sort by stamp (dict iteration order)
  for (int i = 1; i < n; ++i) {
    const long long ks = rec[2 * i], kid = rec[2 * i + 1];
    int j = i - 1;
    while (j >= 0 && rec[2 * j] > ks) {
      rec[2 * (j + 1)] = rec[2 * j];
      rec[2 * (j + 1) + 1] = rec[2 * j + 1];
      --j;
    }
    rec[2 * (j + 1)] = ks;
    rec[2 * (j + 1) + 1] = kid;
  }
  for (int i = 0; i < n; ++i) {
    const int u = (int)rec[2 * i + 1];
    S.la_val[u] = -1;
    S.la_stamp[u] = kNone64;
    S.patience[u] = 0;
    if (S.alive[u] && S.cnt->n_units > 2) remove_unit(S, P, u);
  }
}

__device__ __forceinline__ long long sweep_cutoff(const DevState& S, const Params& P) {
  const long long v = S.cnt->n_units;
  return S.cnt->tick - P.stale_factor * (v > 100 ? v : 100);
}

// adapt_threshold: engine.py:208-238
__device__ void adapt_threshold(const DevState& S, const Params& P, int b) {
  const int ring = S.ring[b];
  if (ring == kRingDisk || (P.allow_boundary && ring == kRingHalf)) {
    S.patience[b] = 0;
    return;
  }
  if (S.hab[b] >= P.h_t) return;
  const int d = S.deg[b];
  const int2* B = S.adj + (size_t)b * kMaxDeg;
  for (int k = 0; k < d; ++k)
    if (S.hab[B[k].x] >= P.h_t) return;
  int count = S.patience[b] + 1;
  if (count >= P.ring_patience) {
    S.theta[b] = dmul(S.theta[b], P.rho);
    count = 0;
  }
  S.patience[b] = count;
}

__device__ __forceinline__ void move_toward(double4& p, double eps, double x, double y, double z) {
  p.x = dadd(p.x, dmul(eps, dsub(x, p.x)));
  p.y = dadd(p.y, dmul(eps, dsub(y, p.y)));
  p.z = dadd(p.z, dmul(eps, dsub(z, p.z)));
}

// update_single, everything up to and including prune (engine.py:297-344).
// Returns 1 if the sweep clock fired (engine.py:346).
__device__ int serial_update_part1(const DevState& S, const Params& P, int b, int s, double dw,
                                   double x, double y, double z) {
  Counters* c = S.cnt;
  const long long tick = ++c->tick;
  touch_active(S, b, tick, 0);
  touch_active(S, s, tick, 1);
  const int created = connect_or_reset(S, b, s);
  if (created < 0) return 0;
  if (created) c->ev_create++;
  int32_t over[kMaxDeg];
  int nover = 0;
  age_incident(S, P, b, s, 1, over, &nover);
  double4 wp = S.pos[b];
  move_toward(wp, P.eps_b, x, y, z);
  S.pos[b] = wp;
  set_hab(S, P, b, dmul(S.hab[b], P.c_b));
  {
    const int d = S.deg[b];
    const int2* B = S.adj + (size_t)b * kMaxDeg;
    for (int k = 0; k < d; ++k) {
      const int v = B[k].x;
      double4 pv = S.pos[v];
      move_toward(pv, P.eps_n, x, y, z);
      S.pos[v] = pv;
      set_hab(S, P, v, dmul(S.hab[v], P.c_n));
    }
  }
  // maybe_insert: engine.py:184-205 gated at :336
  if (dw > S.theta[b] && S.hab[b] < P.h_t) {
    const double theta_b = S.theta[b];
    const double mx = dmul(dadd(wp.x, x), 0.5);
    const double my = dmul(dadd(wp.y, y), 0.5);
    const double mz = dmul(dadd(wp.z, z), 0.5);
    const int r = add_unit(S, P, mx, my, mz, theta_b);
    if (r < 0) return 0;
    connect_or_reset(S, r, b);
    connect_or_reset(S, r, s);
    if (find_slot(S, b, s) >= 0) remove_edge(S, b, s);
    touch_active(S, r, tick, 2);
    c->ev_insert++;
  }
  int pe, pu;
  prune_winner(S, P, b, over, nover, &pe, &pu);
  if (pe || pu) c->ev_prune++;
  return tick >= c->next_sweep ? 1 : 0;
}

// sweep bookkeeping + adapt_threshold (engine.py:345-355)
__device__ void serial_update_part2(const DevState& S, const Params& P, int b, int swept_n,
                                    bool sweep_fired) {
  Counters* c = S.cnt;
  if (sweep_fired) {
    if (swept_n > 0) {
      const int before = c->n_units;
      sweep_apply(S, P, S.scratch, swept_n);
      if (c->n_units != before) c->ev_sweep++;
    }
    c->next_sweep = c->tick + kSweepEvery;
  }
  if (S.alive[b]) adapt_threshold(S, P, b);
}

// single-thread stale collection (API path)
__device__ int collect_stale_serial(const DevState& S, const Params& P) {
  const long long cutoff = sweep_cutoff(S, P);
  if (cutoff <= 0) return 0;
  int n = 0;
  for (int u = 0; u < S.cnt->next_id; ++u)
    if (S.la_val[u] != -1 && S.la_val[u] < cutoff) {
      S.scratch[2 * n] = S.la_stamp[u];
      S.scratch[2 * n + 1] = u;
      ++n;
    }
  return n;
}

// ---------------------------------------------------------------------------
// block primitives (1024 threads)

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive scan across the block; *total = block sum.  Contains __syncthreads.
__device__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  __syncthreads();
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int x = lane < nw ? s_warp[lane] : 0;
    const int xi = warp_incl_scan(x);
    if (lane < nw) s_warp[lane] = xi - x;
    if (lane == 31) s_warp[32] = xi;
  }
  __syncthreads();
  *total = s_warp[32];
  return s_warp[wid] + inc - v;
}

__device__ int block_min(int v, int* s_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) s_warp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int x = lane < nw ? s_warp[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) s_warp[32] = x;
  }
  __syncthreads();
  return s_warp[32];
}

__device__ int block_sum(int v, int* s_warp) {
  int total;
  block_excl_scan(v, s_warp, &total);
  return total;
}

#ifdef GS_PROF_TL
// timeline profiling builds: per batch, the update's lead thread stamps
// (resident, wait released, end) in globaltimer ns
__device__ unsigned long long g_tlu[8192][3];
extern "C" int gs_debug_tl_update(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_tlu, sizeof(unsigned long long) * 3 * (size_t)n);
}
// per batch, the latest CTA's: last cluster barrier passed, snapshot flag posted
__device__ unsigned long long g_tlu2[8192][2];
extern "C" int gs_debug_tl_update2(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_tlu2, sizeof(unsigned long long) * 2 * (size_t)n);
}
#endif
#include "update_kernel.cuh"

// ---------------------------------------------------------------------------
// Network API operations (single thread; not on the hot path)

enum OpCode {
  OP_ADD = 1,
  OP_CONNECT = 2,
  OP_REMOVE_UNIT = 3,
  OP_REMOVE_EDGE = 4,
  OP_AGE = 5,
  OP_PRUNE = 6,
  OP_SET = 7,
};

struct OpArgs {
  int op;
  int a, b;
  long long i0;
  double x, y, z, t, t2;
  int flags;  // OP_SET: 1 pos, 2 hab, 4 theta
};

__device__ bool valid_unit(const DevState& S, int u) {
  return u >= 0 && u < S.cnt->next_id && S.alive[u];
}

__global__ void k_op(DevState S, Params P, OpArgs a, long long* res) {
  Counters* c = S.cnt;
  c->rowpos_n[0] = c->rowpos_n[1] = -1;  // positions / rows may change: the find gathers
  res[0] = 0;
  res[1] = 0;
  res[2] = 0;
  switch (a.op) {
    case OP_ADD: {
      res[0] = add_unit(S, P, a.x, a.y, a.z, a.t);
      break;
    }
    case OP_CONNECT: {
      if (a.a == a.b) { res[2] = E_SELF; break; }
      if (!valid_unit(S, a.a) || !valid_unit(S, a.b)) { res[2] = E_UNKNOWN; break; }
      res[0] = connect_or_reset(S, a.a, a.b);
      break;
    }
    case OP_REMOVE_UNIT: {
      if (!valid_unit(S, a.a)) { res[2] = E_UNKNOWN; break; }
      remove_unit(S, P, a.a);
      break;
    }
    case OP_REMOVE_EDGE: {
      if (!valid_unit(S, a.a) || !valid_unit(S, a.b)) { res[2] = E_UNKNOWN; break; }
      if (find_slot(S, a.a, a.b) < 0) { res[2] = E_NOEDGE; break; }
      remove_edge(S, a.a, a.b);
      break;
    }
    case OP_AGE: {
      if (!valid_unit(S, a.a)) { res[2] = E_UNKNOWN; break; }
      res[0] = age_incident(S, P, a.a, a.b, (int)a.i0, nullptr, nullptr);
      break;
    }
    case OP_PRUNE: {
      int pe, pu;
      prune_all(S, P, a.i0, &pe, &pu);
      res[0] = pe;
      res[1] = pu;
      break;
    }
    case OP_SET: {
      if (!valid_unit(S, a.a)) { res[2] = E_UNKNOWN; break; }
      if (a.flags & 1) {
        double4 p = S.pos[a.a];
        p.x = a.x;
        p.y = a.y;
        p.z = a.z;
        S.pos[a.a] = p;
      }
      if (a.flags & 2) set_hab(S, P, a.a, a.t);
      if (a.flags & 4) S.theta[a.a] = a.t2;
      break;
    }
  }
  if (c->error && !res[2]) res[2] = 100 + c->error;
}

// audit (Network.audit, network.py:485-526): counts violations
__global__ void k_audit(DevState S, Params P, unsigned long long* bad) {
  const Counters* c = S.cnt;
  __shared__ int s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  // 0 units, 1 edge halves, 2 isolated, 3 disk, 4 half, 5 inc, 6 untrained
  for (int u = threadIdx.x; u < c->next_id; u += blockDim.x) {
    if (!S.alive[u]) continue;
    atomicAdd(&s_cnt[0], 1);
    const int d = S.deg[u];
    atomicAdd(&s_cnt[1], d);
    if (d == 0) atomicAdd(&s_cnt[2], 1);
    atomicAdd(&s_cnt[3 + S.ring[u]], 1);
    if (S.hab[u] >= P.h_t) atomicAdd(&s_cnt[6], 1);
    if (classify_ring(S, u) != S.ring[u]) atomicAdd(bad, 1ull);
    if (!(S.hab[u] >= 0.0 && S.hab[u] <= 1.0) || !(S.theta[u] > 0.0)) atomicAdd(bad, 1ull);
    for (int k = 0; k < d; ++k) {
      const int2 ent = S.adj[(size_t)u * kMaxDeg + k];
      const int v = ent.x;
      if (v == u || v < 0 || v >= c->next_id || !S.alive[v]) {
        atomicAdd(bad, 1ull);
        continue;
      }
      const int kv = find_slot(S, v, u);
      if (kv < 0 || S.adj[(size_t)v * kMaxDeg + kv].y != ent.y) atomicAdd(bad, 1ull);
      if (S.eage[ent.y] < 0) atomicAdd(bad, 1ull);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long e = 0;
    e += s_cnt[0] != c->n_units;
    e += s_cnt[1] != 2 * c->n_edges;
    e += s_cnt[2] != c->iso_count;
    e += s_cnt[3] != c->ring_counts[0];
    e += s_cnt[4] != c->ring_counts[1];
    e += s_cnt[5] != c->ring_counts[2];
    e += s_cnt[6] != c->untrained;
    atomicAdd(bad, e);
  }
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_fill_i64(long long* p, int64_t n, long long v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// push edge ids [lo, hi) onto the free stack, lowest id on top
__global__ void k_push_free(int32_t* efree, int top, int lo, int hi) {
  const int n = hi - lo;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    efree[top + i] = hi - 1 - i;
}

__global__ void k_set_top(Counters* c, int delta) { c->efree_top += delta; }

}  // namespace gs

using namespace gs;

// ---------------------------------------------------------------------------
// host side

struct gs_engine {
  gs_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  gs_params hp{};
  Params P{};
  DevState S{};
  int U = 0, EC = 0;
  DevBuf find_work;
  DevBuf sig_buf;
  DevBuf rec_buf;
  DevBuf idx_buf;  // sampled cloud indices (gs_engine_step_sampled)
  gs_batch_stats* h_stats = nullptr;  // pinned
  // per-batch stats copies (ring of pinned slots + completion events) so the
  // host can read batch i - lag while later batches are still queued
  gs_batch_stats* h_ring = nullptr;
  // the update kernel writes each batch's stats into a device ring slot (a
  // host-mapped write would sit on the kernel's completion, i.e. on the next
  // find's release); batches the host will read are copied to h_ring on a
  // copy stream behind their completion event
  gs_batch_stats* d_ring = nullptr;
  double* rowpos_b[2] = {nullptr, nullptr};  // the two row-snapshot slots
  bool spec_find = true;  // GS_SPEC_FIND=0 turns the speculative screen off
  float4* rowf_b[2] = {nullptr, nullptr};
  cudaStream_t cp = nullptr;
  cudaEvent_t cp_ev[64] = {};
  cudaEvent_t stat_ev[64] = {};
  int64_t issued = 0;
  int64_t reset_seq = 0;     // steps issued before the last reset (stale for lagged reads)
  bool ring_latest = false;  // h_ring holds the newest stats (device steps)
  double* h_sig = nullptr;            // pinned staging for host batches
  size_t h_sig_cap = 0;
  long long* d_res = nullptr;
  long long* h_res = nullptr;
  int batch_no = 0;
  long long launches = 0;
  // optional per-phase device timing: a ring of (start, find done, update
  // done) CUDA events on the engine stream, so every batch is timed even
  // with batches in flight; harvested at the next synchronisation
  static constexpr int kEvRing = 64;
  cudaEvent_t ev[kEvRing][4] = {};  // start, find done, update done, exchange done
  int ev_head = 0, ev_count = 0;
  bool timing = false;
  int timing_every = 1;      // time one batch in timing_every (weighted by it)
  long long timing_seq = 0;
  int ev_w[kEvRing] = {};
  bool ev_x[kEvRing] = {};  // entry has an exchange (all-gather) event
  int64_t ev_b[kEvRing] = {};  // batch (issue index) a timing entry belongs to
  // batch (issue index) whose completion event a stats-ring slot holds
  int64_t stat_batch[kEvRing];
  double find_ms = 0.0, update_ms = 0.0;
  // host mirror of the last known counters
  int next_id = 0, n_edges = 0, n_units = 0;
  // batches the host may enqueue ahead of its last stats read (gs_engine_set_async)
  int async_depth = 0;
  // asynchronous sampled runs draw the indices of async_depth batches per
  // sampler launch (fixed batch size)
  int64_t pf_m = 0, pf_next = 0, pf_left = 0;
  // ... on a side stream, one group ahead, into two halves of idx_buf, so a
  // group's draws overlap the previous group's update kernels (16 SMs busy)
  cudaStream_t side = nullptr;
  cudaEvent_t pf_done[2] = {}, use_done[2] = {};
  int64_t pf_issued = 0, pf_used = 0;
  int pf_half = 0;
  // signal sharding across GPUs: this rank finds winners for
  // signals [rank*m/world, (rank+1)*m/world) and one ncclAllGather of the
  // 16-byte records on the engine stream assembles the batch in rank order
  // == batch order; the update is replicated
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  double exchange_ms = 0.0;
};

namespace {
// drop prefetched groups (the side stream is drained first: its sampler
// launches advance the sampler state)
void drop_prefetch(gs_engine* e) {
  if (e->side) GS_CUDA(cudaStreamSynchronize(e->side));
  e->pf_left = e->pf_next = 0;
  e->pf_issued = e->pf_used = 0;
}
}  // namespace

namespace {

template <class T>
void grow_array(T*& p, size_t old_n, size_t new_n, cudaStream_t st) {
  T* q = (T*)dmalloc(sizeof(T) * new_n, st);
  if (p && old_n) GS_CUDA(cudaMemcpyAsync(q, p, sizeof(T) * old_n, cudaMemcpyDeviceToDevice, st));
  dfree(p, st);  // ordered after the copy
  p = q;
}

void fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return;
  k_fill_i32<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(p, n, v);
  GS_CUDA(cudaGetLastError());
}

void fill_i64(long long* p, int64_t n, long long v, cudaStream_t st) {
  if (n <= 0) return;
  k_fill_i64<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(p, n, v);
  GS_CUDA(cudaGetLastError());
}

void grow_units(gs_engine* e, int new_u) {
  if (new_u <= e->U) return;
  const int old = e->U;
  cudaStream_t st = e->stream;
  DevState& S = e->S;
  grow_array(S.pos, old, new_u, st);
  grow_array(S.hab, old, new_u, st);
  grow_array(S.theta, old, new_u, st);
  grow_array(S.alive, old, new_u, st);
  grow_array(S.ring, old, new_u, st);
  grow_array(S.deg, old, new_u, st);
  grow_array(S.adj, (size_t)old * kMaxDeg, (size_t)new_u * kMaxDeg, st);
  grow_array(S.patience, old, new_u, st);
  grow_array(S.la_val, old, new_u, st);
  grow_array(S.la_stamp, old, new_u, st);
  grow_array(S.claim, old, new_u, st);
  grow_array(S.firstwin, old, new_u, st);
  grow_array(S.touchfirst, old, new_u, st);
  grow_array(S.ttr, old, new_u, st);
  grow_array(S.iso_pos, old, new_u, st);
  grow_array(S.rows, old, new_u, st);
  S.rowf_stride = ((new_u + 1) / 2 + 63) / 64 * 64;
  for (int k = 0; k < 2; ++k) {  // regenerated by the next updates (stride U)
    dfree(e->rowpos_b[k], st);
    e->rowpos_b[k] = (double*)dmalloc(sizeof(double) * 3 * (size_t)new_u, st);
    dfree(e->rowf_b[k], st);
    e->rowf_b[k] = (float4*)dmalloc(sizeof(float4) * 2 * (size_t)S.rowf_stride, st);
  }
  S.rowpos = e->rowpos_b[0];
  S.rowf = e->rowf_b[0];
  S.rowpos_prev = e->rowpos_b[1];
  {
    const int stale2[2] = {-1, -1};
    GS_CUDA(cudaMemcpyAsync(&S.cnt->rowpos_n[0], stale2, sizeof(stale2), cudaMemcpyHostToDevice, st));
    GS_CUDA(cudaStreamSynchronize(st));
  }
  grow_array(S.iso_list, old, new_u, st);
  // scratch content is transient: plain reallocation
  dfree(S.scratch, st);
  S.scratch = (long long*)dmalloc(sizeof(long long) * 2 * (size_t)new_u + 64, st);
  const int64_t add = new_u - old;
  GS_CUDA(cudaMemsetAsync(S.alive + old, 0, add, st));
  GS_CUDA(cudaMemsetAsync(S.deg + old, 0, sizeof(int32_t) * add, st));
  fill_i32(S.firstwin + old, add, kNone32, st);
  fill_i32(S.touchfirst + old, add, kNone32, st);
  fill_i32(S.ttr + old, add, -1, st);
  fill_i32(S.claim + old, add, -1, st);
  fill_i32(S.iso_pos + old, add, -1, st);
  fill_i64(S.la_val + old, add, -1, st);
  fill_i64(S.la_stamp + old, add, kNone64, st);
  e->U = new_u;
  S.U = new_u;
}

void grow_edges(gs_engine* e, int new_ec) {
  if (new_ec <= e->EC) return;
  const int old = e->EC;
  cudaStream_t st = e->stream;
  DevState& S = e->S;
  grow_array(S.eage, old, new_ec, st);
  // the free stack keeps its first efree_top entries; new ids go on top of
  // them in descending order so the lowest new id pops first
  int32_t* nf = (int32_t*)dmalloc(sizeof(int32_t) * (size_t)new_ec, st);
  int top = 0;
  if (S.efree) {
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaStreamSynchronize(st));
    top = hc.efree_top;
    // existing free ids sit below; new ids above (popped first) - order of
    // edge ids is never observable
    if (top) GS_CUDA(cudaMemcpyAsync(nf, S.efree, sizeof(int32_t) * top, cudaMemcpyDeviceToDevice, st));
    dfree(S.efree, st);
  }
  S.efree = nf;
  k_push_free<<<64, 256, 0, st>>>(S.efree, top, old, new_ec);
  GS_CUDA(cudaGetLastError());
  k_set_top<<<1, 1, 0, st>>>(S.cnt, new_ec - old);
  GS_CUDA(cudaGetLastError());
  e->EC = new_ec;
  S.EC = new_ec;
}

void ensure_capacity(gs_engine* e, int64_t extra_units, int64_t extra_edges) {
  // with batches in flight the host's counters lag: leave room for them
  extra_units *= 1 + e->async_depth;
  extra_edges *= 1 + e->async_depth;
  const int64_t need_u = (int64_t)e->next_id + extra_units + 1;
  if (need_u > e->U) {
    int64_t nu = std::max<int64_t>(e->U, 1024);
    while (nu < need_u) nu *= 2;
    GS_CHECK(nu < (1LL << 30), GS_STATE_ERROR, "unit capacity exceeds 2^30 ids");
    grow_units(e, (int)nu);
  }
  const int64_t need_e = (int64_t)e->n_edges + extra_edges + 1;
  if (need_e > e->EC) {
    int64_t ne = std::max<int64_t>(e->EC, 4096);
    while (ne < need_e) ne *= 2;
    GS_CHECK(ne < (1LL << 30), GS_STATE_ERROR, "edge capacity exceeds 2^30");
    grow_edges(e, (int)ne);
  }
}

const char* dev_error_name(long long e) {
  switch (e) {
    case E_DEGREE: return "unit degree exceeded the device adjacency capacity (64)";
    case E_UNIT_CAP: return "unit capacity exhausted";
    case E_EDGE_CAP: return "edge capacity exhausted";
    case E_STALE: return "stale winner result";
    case E_UNKNOWN: return "unknown unit";
    case E_SELF: return "self loop";
    case E_NOEDGE: return "no such edge";
    case E_AFF: return "ring-recompute scratch overflow";
    case E_BADPOS: return "position / threshold must be finite (threshold > 0)";
    default: return "device error";
  }
}

void check_stats(gs_engine* e) {
  const gs_batch_stats& s = *e->h_stats;
  e->next_id = (int)s.next_id;
  e->n_edges = (int)s.edges;
  e->n_units = (int)s.units;
  if (s.error) {
    set_error(std::string("device engine error: ") + dev_error_name(s.error));
    throw Fail{GS_STATE_ERROR};
  }
}

long long run_op(gs_engine* e, const OpArgs& a, long long* res2 = nullptr) {
  ensure_capacity(e, 1, 1);
  k_op<<<1, 1, 0, e->stream>>>(e->S, e->P, a, e->d_res);
  GS_CUDA(cudaGetLastError());
  e->launches++;
  ++g_launches;
  GS_CUDA(cudaMemcpyAsync(e->h_res, e->d_res, 3 * sizeof(long long), cudaMemcpyDeviceToHost,
                          e->stream));
  Counters hc;
  GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
  GS_CUDA(cudaStreamSynchronize(e->stream));
  e->next_id = hc.next_id;
  e->n_edges = hc.n_edges;
  e->n_units = hc.n_units;
  const long long err = e->h_res[2];
  if (err == E_UNKNOWN) {
    set_error("unit is not alive");
    throw Fail{GS_UNKNOWN_UNIT};
  }
  if (err == E_SELF) {
    set_error("cannot connect a unit to itself");
    throw Fail{GS_VALUE_ERROR};
  }
  if (err == E_NOEDGE) {
    set_error("no edge between the units");
    throw Fail{GS_UNKNOWN_UNIT};
  }
  if (err > 100) {
    set_error(std::string("device engine error: ") + dev_error_name(err - 100));
    throw Fail{err - 100 == E_BADPOS ? GS_VALUE_ERROR : GS_STATE_ERROR};
  }
  if (res2) {
    res2[0] = e->h_res[0];
    res2[1] = e->h_res[1];
  }
  return e->h_res[0];
}

void launch_update(gs_engine* e, const double* d_sig, const WinRec* d_rec, int64_t m,
                   gs_batch_stats* st_out = nullptr, bool pre_fw = false) {
  static bool opted = false;
  if (!opted) {
    // clusters beyond the portable 8 CTAs need an opt-in; C1's staging in
    // shared memory is more than the default 48 KB
    if constexpr (kCluster > 8)
      GS_CUDA(cudaFuncSetAttribute(k_update_batch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    GS_CUDA(cudaFuncSetAttribute(k_update_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kUpdDynSmem));
    opted = true;
  }
  e->batch_no++;
  {  // this update's row-snapshot slot
    const int s = e->batch_no & 1;
    e->S.snap = s;
    e->S.rowpos = e->rowpos_b[s];
    e->S.rowf = e->rowf_b[s];
    e->S.rowpos_prev = e->rowpos_b[s ^ 1];
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCluster);
  cfg.blockDim = dim3(kUpdThreads);
  cfg.dynamicSmemBytes = kUpdDynSmem;
  cfg.stream = e->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GS_CUDA(cudaLaunchKernelEx(&cfg, k_update_batch, e->S, e->P, d_sig, d_rec, (int)m, e->batch_no,
                             pre_fw ? 1 : 0, st_out ? st_out : e->S.stats));
  GS_CUDA(cudaGetLastError());
  e->launches++;
  ++g_launches;
}

void launch_find(gs_engine* e, const double* d_sig, int64_t lo, int64_t hi, WinRec* d_rec,
                 const int64_t* sig_idx = nullptr, const double* sig_pts = nullptr,
                 bool pre_fw = false) {
  GS_CHECK(e->n_units >= 2, GS_STATE_ERROR, "need at least 2 units to find winners");
  FindArgs a;
  a.pos4 = e->S.pos;
  a.rows = e->S.rows;
  a.alive = e->S.alive;
  // host estimate of the row count (grid sizing, staging); with batches in
  // flight it can lag the device's count, which every find kernel reads
  // (n_dev) and handles past the estimate
  // rows hold the live units plus dead entries up to 1/8 of the rows (lazy
  // compaction in the update), and never more than next_id
  a.n = std::min<int64_t>(e->next_id, (int64_t)e->n_units + (e->n_units + 6) / 7 + 1);
  a.n_dev = &e->S.cnt->nrows;  // exact row count, read on the device
  a.rowpos = e->S.rowpos;
  a.rowpos_n = &e->S.cnt->rowpos_n[e->S.snap];
  a.rowpos_stride = e->U;
  a.rowf = e->S.rowf;
  a.rowf_stride = e->S.rowf_stride;
  a.fcen = e->S.cnt->fcen[e->S.snap];
  a.fpm_bits = &e->S.cnt->fpm_bits[e->S.snap];
  a.sig = d_sig + 3 * lo;
  a.sig_idx = sig_idx ? sig_idx + lo : nullptr;
  a.sig_pts = sig_pts;
  a.m = hi - lo;
  a.out_win = d_rec + lo;
  a.mode = e->hp.find_mode;
  a.tl_batch = e->batch_no + 1;  // the update this find feeds (timeline builds)
  if (pre_fw) {  // the whole batch on this engine: resolve the first window's candidates
    a.firstwin = e->S.firstwin;
    a.fw_limit = kWinC;
    // the previous kernel is this engine's update: start on its snapshot token
    if (e->batch_no > 0) {
      a.snap_token = e->S.snap_token;
      a.snap_target = e->batch_no;
      a.snap_parts = kCluster;
    }
    if (e->batch_no > 1 && e->spec_find) {  // two snapshots exist: screen speculatively
      const int cur = e->S.snap, prev = cur ^ 1;
      Counters* c = e->S.cnt;
      a.rowf_prev = e->rowf_b[prev];
      a.fcen_prev = c->fcen[prev];
      a.fpm_prev = &c->fpm_bits[prev];
      a.rowpos_n_prev = &c->rowpos_n[prev];
      a.gen_prev = &c->snap_gen[prev];
      a.gen_cur = &c->snap_gen[cur];
      a.disp_prev = &c->snap_disp[prev];
      a.disp_cur = &c->snap_disp[cur];
    }
  }
  const unsigned long long before = g_launches;
  find_launch(*e->ctx, a, e->stream, e->find_work);
  e->launches += (long long)(g_launches - before);
}

}  // namespace

namespace {
void set_params(gs_engine* e, const gs_params* p) {
  GS_CHECK(0.0 <= p->eps_n && p->eps_n < p->eps_b && p->eps_b <= 1.0, GS_VALUE_ERROR,
           "need 0 <= eps_n < eps_b <= 1");
  GS_CHECK(p->tau_b > 0 && p->tau_b < 1 && p->tau_n > 0 && p->tau_n < 1 && p->h_t > 0 &&
               p->h_t < 1 && p->rho > 0 && p->rho < 1,
           GS_VALUE_ERROR, "tau_b, tau_n, h_t, rho must lie in (0, 1)");
  GS_CHECK(p->max_age >= 0 && p->ring_patience >= 1 && p->stale_factor >= 1, GS_VALUE_ERROR,
           "bad max_age / ring_patience / stale_factor");
  GS_CHECK(p->find_mode >= 0 && p->find_mode <= 4, GS_VALUE_ERROR, "bad find mode");
  e->hp = *p;
  e->P.eps_b = p->eps_b;
  e->P.eps_n = p->eps_n;
  e->P.c_b = 1.0 - p->tau_b;  // engine.py:321
  e->P.c_n = 1.0 - p->tau_n;  // engine.py:329
  e->P.h_t = p->h_t;
  e->P.rho = p->rho;
  e->P.max_age = p->max_age;
  e->P.ring_patience = p->ring_patience;
  e->P.stale_factor = p->stale_factor;
  e->P.allow_boundary = p->allow_boundary ? 1 : 0;
}
}  // namespace

extern "C" gs_status gs_engine_set_params(gs_engine* e, const gs_params* p) {
  return guarded([&] {
    GS_CHECK(e && p, GS_VALUE_ERROR, "null argument");
    set_params(e, p);
  });
}

extern "C" gs_status gs_engine_create(gs_ctx* ctx, const gs_params* p, int64_t capacity_hint,
                                      gs_engine** out) {
  return guarded([&] {
    GS_CHECK(ctx && p && out, GS_VALUE_ERROR, "null argument");
    GS_CUDA(cudaSetDevice(ctx->device));
    gs_engine* e = new gs_engine();
    if (const char* sp = getenv("GS_SPEC_FIND")) e->spec_find = atoi(sp) != 0;
    e->ctx = ctx;
    try {
      set_params(e, p);
    } catch (...) {
      delete e;
      throw;
    }
    try {
      GS_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
      cudaStream_t st = e->stream;
      for (DevBuf* b : {&e->find_work, &e->sig_buf, &e->rec_buf, &e->idx_buf}) b->st = st;
      e->S.cnt = (Counters*)dmalloc(sizeof(Counters), st);
      GS_CUDA(cudaMemsetAsync(e->S.cnt, 0, sizeof(Counters), e->stream));
      Counters init{};
      init.next_sweep = kSweepEvery;
      GS_CUDA(cudaMemcpyAsync(e->S.cnt, &init, sizeof(Counters), cudaMemcpyHostToDevice, e->stream));
      GS_CUDA(cudaStreamSynchronize(e->stream));
      e->S.stats = (gs_batch_stats*)dmalloc(sizeof(gs_batch_stats), st);
      e->S.snap_token = (int*)dmalloc(128, st);
      GS_CUDA(cudaMemsetAsync(e->S.snap_token, 0, 128, st));
      GS_CUDA(cudaMemsetAsync(e->S.stats, 0, sizeof(gs_batch_stats), st));
      e->S.aff = (int32_t*)dmalloc(sizeof(int32_t) * kAffCap, st);
      e->S.defer_list = (int32_t*)dmalloc(sizeof(int32_t) * kDeferCap, st);
      e->h_stats = (gs_batch_stats*)hmalloc(sizeof(gs_batch_stats));
      memset(e->h_stats, 0, sizeof(gs_batch_stats));
      e->h_ring = (gs_batch_stats*)hmalloc(sizeof(gs_batch_stats) * gs_engine::kEvRing);
      memset(e->h_ring, 0, sizeof(gs_batch_stats) * gs_engine::kEvRing);
      for (auto& ev : e->stat_ev) GS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      for (auto& ev : e->cp_ev) GS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      e->d_ring = (gs_batch_stats*)dmalloc(sizeof(gs_batch_stats) * gs_engine::kEvRing, st);
      GS_CUDA(cudaMemsetAsync(e->d_ring, 0, sizeof(gs_batch_stats) * gs_engine::kEvRing, st));
      GS_CUDA(cudaStreamCreateWithFlags(&e->cp, cudaStreamNonBlocking));
      for (auto& b : e->stat_batch) b = -1;
      e->d_res = (long long*)dmalloc(4 * sizeof(long long), st);
      e->h_res = (long long*)hmalloc(4 * sizeof(long long));
      const int64_t cap = std::max<int64_t>(1024, std::min<int64_t>(capacity_hint, 1 << 28));
      grow_units(e, (int)cap);
      grow_edges(e, (int)std::min<int64_t>(4 * cap, 1 << 29));
      GS_CUDA(cudaStreamSynchronize(e->stream));
    } catch (...) {
      gs_engine_destroy(e);
      throw;
    }
    *out = e;
  });
}

extern "C" void gs_engine_destroy(gs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->ctx->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  DevState& S = e->S;
  void* ptrs[] = {S.pos, S.hab, S.theta, S.alive, S.ring, S.deg, S.adj, S.patience, S.la_val,
                  S.la_stamp, S.claim, S.firstwin, S.touchfirst, S.ttr, S.iso_pos, S.rows, S.eage,
                  S.efree, S.iso_list, S.scratch, S.aff, S.defer_list, S.cnt, S.stats, e->d_res,
                  S.snap_token,
                  e->rowpos_b[0], e->rowpos_b[1], e->rowf_b[0], e->rowf_b[1], e->d_ring};
  if (e->cp) {
    cudaStreamSynchronize(e->cp);
    cudaStreamDestroy(e->cp);
  }
  for (auto ev : e->cp_ev)
    if (ev) cudaEventDestroy(ev);
  for (void* q : ptrs) dfree(q, e->stream);  // stream is idle: back to the pool at once
  hfree(e->h_stats);
  hfree(e->h_ring);
  for (auto ev : e->stat_ev)
    if (ev) cudaEventDestroy(ev);
  hfree(e->h_res);
  hfree(e->h_sig);
  for (auto& trio : e->ev)
    for (auto ev : trio)
      if (ev) cudaEventDestroy(ev);
  e->find_work.release();
  e->sig_buf.release();
  e->rec_buf.release();
  e->idx_buf.release();
  if (e->side) {
    cudaStreamSynchronize(e->side);
    cudaStreamDestroy(e->side);
  }
  for (int h = 0; h < 2; ++h) {
    if (e->pf_done[h]) cudaEventDestroy(e->pf_done[h]);
    if (e->use_done[h]) cudaEventDestroy(e->use_done[h]);
  }
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

extern "C" gs_status gs_engine_add_unit(gs_engine* e, double x, double y, double z,
                                        double threshold, int64_t* id) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CHECK(std::isfinite(x) && std::isfinite(y) && std::isfinite(z), GS_VALUE_ERROR,
             "position must be finite");
    GS_CHECK(std::isfinite(threshold) && threshold > 0.0, GS_VALUE_ERROR,
             "threshold must be positive and finite");
    OpArgs a{};
    a.op = OP_ADD;
    a.x = x;
    a.y = y;
    a.z = z;
    a.t = threshold;
    const long long r = run_op(e, a);
    if (id) *id = r;
  });
}

extern "C" gs_status gs_engine_connect_or_reset(gs_engine* e, int64_t a_, int64_t b_,
                                                int32_t* created) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    OpArgs a{};
    a.op = OP_CONNECT;
    a.a = (int)a_;
    a.b = (int)b_;
    const long long r = run_op(e, a);
    if (created) *created = (int32_t)r;
  });
}

extern "C" gs_status gs_engine_remove_unit(gs_engine* e, int64_t id) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    OpArgs a{};
    a.op = OP_REMOVE_UNIT;
    a.a = (int)id;
    run_op(e, a);
  });
}

extern "C" gs_status gs_engine_remove_edge(gs_engine* e, int64_t a_, int64_t b_) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    OpArgs a{};
    a.op = OP_REMOVE_EDGE;
    a.a = (int)a_;
    a.b = (int)b_;
    run_op(e, a);
  });
}

extern "C" gs_status gs_engine_age_incident_edges(gs_engine* e, int64_t b, int64_t increment,
                                                  int64_t exclude, int64_t* top) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CHECK(increment >= 0, GS_VALUE_ERROR, "increment must be >= 0");
    OpArgs a{};
    a.op = OP_AGE;
    a.a = (int)b;
    a.b = (int)exclude;
    a.i0 = increment;
    const long long r = run_op(e, a);
    if (top) *top = r;
  });
}

extern "C" gs_status gs_engine_prune(gs_engine* e, int64_t max_age, int64_t* pruned_edges,
                                     int64_t* units_removed) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CHECK(max_age >= 0, GS_VALUE_ERROR, "max_age must be >= 0");
    OpArgs a{};
    a.op = OP_PRUNE;
    a.i0 = max_age;
    long long r[2];
    run_op(e, a, r);
    if (pruned_edges) *pruned_edges = r[0];
    if (units_removed) *units_removed = r[1];
  });
}

extern "C" gs_status gs_engine_set_unit(gs_engine* e, int64_t id, const double* xyz,
                                        const double* hab, const double* theta) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    OpArgs a{};
    a.op = OP_SET;
    a.a = (int)id;
    if (xyz) {
      a.flags |= 1;
      a.x = xyz[0];
      a.y = xyz[1];
      a.z = xyz[2];
    }
    if (hab) {
      a.flags |= 2;
      a.t = *hab;
    }
    if (theta) {
      a.flags |= 4;
      a.t2 = *theta;
    }
    run_op(e, a);
  });
}

namespace {
// fold the timing ring's oldest entries into find_ms / update_ms until at
// most `keep` remain (waits only for the batches it folds)
void harvest_timing(gs_engine* e, int keep = 0);

// find + update for one batch on the engine stream.  With sig_idx the find
// gathers the signals from the sampler's cloud into d_sig (fused sampling).
void step_device_impl(gs_engine* e, const double* d_sig, int64_t m, const int64_t* sig_idx,
                      const double* sig_pts, bool mark);
void step_device_impl(gs_engine* e, const double* d_sig, int64_t m, const int64_t* sig_idx,
                      const double* sig_pts, bool mark = true) {
  GS_CHECK(e && d_sig && m > 0, GS_VALUE_ERROR, "bad step arguments");
  GS_CHECK(m < (1LL << 30), GS_VALUE_ERROR, "batch too large");
  ensure_capacity(e, m, 3 * m);
  WinRec* rec = (WinRec*)e->rec_buf.get(sizeof(WinRec) * (size_t)m);
  // ring full: fold the older half, batches far behind the ones in flight
  // (no stall of an asynchronous run)
  if (e->timing && e->ev_count == gs_engine::kEvRing) harvest_timing(e, gs_engine::kEvRing / 2);
  const bool timed = e->timing && (e->timing_seq++ % e->timing_every) == 0;
  const int ev_slot = (e->ev_head + e->ev_count) % gs_engine::kEvRing;
  cudaEvent_t* evs = e->ev[ev_slot];
  if (timed) {
    e->ev_w[ev_slot] = e->timing_every;
    e->ev_b[ev_slot] = e->issued;
    e->ev_x[ev_slot] = e->comm != nullptr;
    GS_CUDA(cudaEventRecord(evs[0], e->stream));
  }
  if (e->comm) {
    // every rank holds the whole batch (replicated sampling): materialise it
    // for the update, find on this rank's slice, all-gather the records
    GS_CHECK(m % e->world == 0, GS_VALUE_ERROR,
             "sharded batches must divide evenly among the ranks (m % world == 0)");
    if (sig_idx) {
      const unsigned long long before = g_launches;
      gather_signals_launch(sig_idx, sig_pts, const_cast<double*>(d_sig), m, e->stream);
      e->launches += (long long)(g_launches - before);
    }
    const int64_t lo = (int64_t)e->rank * m / e->world, hi = (int64_t)(e->rank + 1) * m / e->world;
    launch_find(e, d_sig, lo, hi, rec);
    if (timed) GS_CUDA(cudaEventRecord(evs[1], e->stream));
    const ncclResult_t r = ncclAllGather(rec + lo, rec, sizeof(WinRec) * (size_t)(hi - lo),
                                         ncclUint8, e->comm, e->stream);
    GS_CHECK(r == ncclSuccess, GS_CUDA_ERROR, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    if (timed) GS_CUDA(cudaEventRecord(evs[3], e->stream));
  } else {
    launch_find(e, d_sig, 0, m, rec, sig_idx, sig_pts, true);
    if (timed) GS_CUDA(cudaEventRecord(evs[1], e->stream));
  }
  // the kernel writes its stats into the device ring slot; no copy between
  // this batch's kernels and the next
  const int slot = (int)(e->issued % gs_engine::kEvRing);
  launch_update(e, d_sig, rec, m, e->d_ring + slot, e->comm == nullptr);
  if (timed) {
    GS_CUDA(cudaEventRecord(evs[2], e->stream));
    e->ev_count++;
  }
  // completion events only where the caller wants them (each one sits
  // between two kernels and stops the programmatic overlap there)
  if (mark) {
    GS_CUDA(cudaEventRecord(e->stat_ev[slot], e->stream));
    GS_CUDA(cudaStreamWaitEvent(e->cp, e->stat_ev[slot], 0));
    GS_CUDA(cudaMemcpyAsync(e->h_ring + slot, e->d_ring + slot, sizeof(gs_batch_stats),
                            cudaMemcpyDeviceToHost, e->cp));
    GS_CUDA(cudaEventRecord(e->cp_ev[slot], e->cp));
    e->stat_batch[slot] = e->issued;
  }
  e->issued++;
  e->ring_latest = true;
}
}  // namespace

extern "C" gs_status gs_engine_step_device(gs_engine* e, const double* d_sig, int64_t m) {
  return guarded([&] { step_device_impl(e, d_sig, m, nullptr, nullptr); });
}

namespace {
// fold the oldest timing entry (complete) into find / exchange / update ms
void fold_timing_entry(gs_engine* e) {
  cudaEvent_t* evs = e->ev[e->ev_head];
  const double w = e->ev_w[e->ev_head];
  float a = 0.f, b = 0.f, x = 0.f;
  GS_CUDA(cudaEventElapsedTime(&a, evs[0], evs[1]));
  if (e->ev_x[e->ev_head]) {
    GS_CUDA(cudaEventElapsedTime(&x, evs[1], evs[3]));
    GS_CUDA(cudaEventElapsedTime(&b, evs[3], evs[2]));
  } else {
    GS_CUDA(cudaEventElapsedTime(&b, evs[1], evs[2]));
  }
  e->find_ms += a * w;
  e->exchange_ms += x * w;
  e->update_ms += b * w;
  e->ev_head = (e->ev_head + 1) % gs_engine::kEvRing;
}

void harvest_timing(gs_engine* e, int keep) {
  for (; e->ev_count > keep; --e->ev_count) {
    GS_CUDA(cudaEventSynchronize(e->ev[e->ev_head][2]));
    fold_timing_entry(e);
  }
}
}  // namespace

extern "C" gs_status gs_engine_phase_ms(gs_engine* e, int enable, double out[2]) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    if (enable >= 0 && !e->ev[0][0]) {
      for (auto& trio : e->ev)
        for (auto& ev : trio) GS_CUDA(cudaEventCreate(&ev));
    }
    // enable: 0 off, 1 every batch, k > 1 one batch in k (weighted by k: an
    // estimate that keeps the per-batch event records off the critical path)
    if (enable >= 0) {
      e->timing = enable != 0;
      e->timing_every = enable > 1 ? enable : 1;
      e->timing_seq = 0;
    }
    if (out) {
      out[0] = e->find_ms;
      out[1] = e->update_ms;
    }
  });
}

// newest device-step stats into h_stats (after the stream is idle)
void latest_stats(gs_engine* e) {
  if (e->ring_latest && e->issued > 0)
    GS_CUDA(cudaMemcpy(e->h_stats, e->d_ring + (e->issued - 1) % gs_engine::kEvRing,
                       sizeof(gs_batch_stats), cudaMemcpyDeviceToHost));
}

extern "C" gs_status gs_engine_stats(gs_engine* e, gs_batch_stats* out) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CUDA(cudaStreamSynchronize(e->stream));
    if (e->side) GS_CUDA(cudaStreamSynchronize(e->side));  // sampler state settled
    latest_stats(e);
    harvest_timing(e);
    check_stats(e);
    if (out) *out = *e->h_stats;
  });
}

// Stats of the batch issued `lag` batches before the newest, waiting only for
// that batch (later ones keep the GPU busy).  *seq receives its index among
// the device steps issued so far (-1: fewer than lag + 1 issued; out zeroed).
extern "C" gs_status gs_engine_stats_lagged(gs_engine* e, int64_t lag, gs_batch_stats* out,
                                            int64_t* seq) {
  return guarded([&] {
    GS_CHECK(e && out && lag >= 0 && lag < gs_engine::kEvRing - 1, GS_VALUE_ERROR,
             "lag must be in [0, 63)");
    int64_t target = e->issued - 1 - lag;
    // the nearest earlier batch that carries a completion event
    while (target >= e->reset_seq && target > e->issued - gs_engine::kEvRing &&
           e->stat_batch[target % gs_engine::kEvRing] != target)
      --target;
    if (target >= 0 && e->stat_batch[target % gs_engine::kEvRing] != target)
      target = e->reset_seq - 1;  // none in reach: report "not yet"
    if (seq) *seq = target < e->reset_seq ? -1 : target - e->reset_seq;
    if (target < e->reset_seq) {
      memset(out, 0, sizeof(*out));
      return;
    }
    GS_CUDA(cudaEventSynchronize(e->cp_ev[target % gs_engine::kEvRing]));
    // per-phase timings of the batches known complete (up to target)
    while (e->ev_count > 0 && e->ev_b[e->ev_head] <= target) {
      fold_timing_entry(e);
      e->ev_count--;
    }
    *e->h_stats = e->h_ring[target % gs_engine::kEvRing];
    check_stats(e);
    *out = *e->h_stats;
  });
}

// One iteration whose m signals are drawn on the device by a CloudSource
// sampler (sample.cu): the sampler kernel emits cloud indices, the find
// gathers the points into the engine's signal buffer as it loads them.
// out != NULL makes it synchronous (stats copied out), else it stays queued.
extern "C" gs_status gs_engine_step_sampled(gs_engine* e, gs_sampler* smp, int64_t m,
                                            gs_batch_stats* out) {
  return guarded([&] {
    GS_CHECK(e && smp && m > 0, GS_VALUE_ERROR, "bad step arguments");
    double* d_sig = (double*)e->sig_buf.get(sizeof(double) * 3 * (size_t)m);
    int64_t* d_idx;
    if (e->async_depth > 0) {
      // one sampler launch draws the next async_depth batches (same stream
      // order as one launch per batch); a batch-size change would reorder
      // draws already taken, so it is an error while some remain
      GS_CHECK(e->pf_issued == 0 || e->pf_m == m, GS_VALUE_ERROR,
               "asynchronous sampled runs need a fixed batch size");
      const int64_t k = e->async_depth;
      if (e->pf_left == 0) {
        if (!e->side) {
          GS_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
          for (int h = 0; h < 2; ++h) {
            GS_CUDA(cudaEventCreateWithFlags(&e->pf_done[h], cudaEventDisableTiming));
            GS_CUDA(cudaEventCreateWithFlags(&e->use_done[h], cudaEventDisableTiming));
          }
        }
        if (e->pf_issued == 0) {
          // first group: its buffers must be ready on the side stream too
          GS_CUDA(cudaStreamSynchronize(e->stream));
          e->idx_buf.get(sizeof(int64_t) * (size_t)(2 * k * m));
          GS_CUDA(cudaStreamSynchronize(e->stream));
        }
        int64_t* base = (int64_t*)e->idx_buf.p;
        auto issue = [&](int64_t grp) {
          const int h = (int)(grp & 1);
          if (grp >= 2) GS_CUDA(cudaStreamWaitEvent(e->side, e->use_done[h], 0));
          sampler_indices(smp, k * m, base + (size_t)h * k * m, e->side);
          GS_CUDA(cudaEventRecord(e->pf_done[h], e->side));
          e->launches++;
          e->pf_issued++;
        };
        if (e->pf_issued == 0) issue(0);
        const int64_t G = e->pf_used++;
        e->pf_half = (int)(G & 1);
        GS_CUDA(cudaStreamWaitEvent(e->stream, e->pf_done[e->pf_half], 0));
        issue(G + 1);  // next group's draws overlap this group's batches
        e->pf_m = m;
        e->pf_next = 0;
        e->pf_left = k;
      }
      d_idx = (int64_t*)e->idx_buf.p + ((size_t)e->pf_half * k + e->pf_next) * m;
      e->pf_next++;
      e->pf_left--;
    } else {
      d_idx = (int64_t*)e->idx_buf.get(sizeof(int64_t) * (size_t)m);
      sampler_indices(smp, m, d_idx, e->stream);
      e->launches++;
    }
    // asynchronous groups: one completion event per group, at its end (where
    // the next group's draws break the kernel chain anyway)
    step_device_impl(e, d_sig, m, d_idx, sampler_points(smp),
                     e->async_depth == 0 || e->pf_left == 0);
    if (e->async_depth > 0 && e->pf_left == 0)  // this half may be refilled now
      GS_CUDA(cudaEventRecord(e->use_done[e->pf_half], e->stream));
    if (out) {
      GS_CUDA(cudaStreamSynchronize(e->stream));
      latest_stats(e);
      harvest_timing(e);
      check_stats(e);
      *out = *e->h_stats;
    }
  });
}

extern "C" gs_status gs_engine_step(gs_engine* e, const double* signals, int64_t m,
                                    gs_batch_stats* out) {
  return guarded([&] {
    GS_CHECK(e && signals && m > 0, GS_VALUE_ERROR, "bad step arguments");
    const size_t bytes = sizeof(double) * 3 * (size_t)m;
    if (bytes > e->h_sig_cap) {
      GS_CUDA(cudaStreamSynchronize(e->stream));  // a queued copy may still read it
      hfree(e->h_sig);
      e->h_sig = nullptr;
      e->h_sig_cap = bytes + bytes / 2;
      e->h_sig = (double*)hmalloc(e->h_sig_cap);
    }
    memcpy(e->h_sig, signals, bytes);
    double* d_sig = (double*)e->sig_buf.get(bytes);
    GS_CUDA(cudaMemcpyAsync(d_sig, e->h_sig, bytes, cudaMemcpyHostToDevice, e->stream));
    gs_status st = gs_engine_step_device(e, d_sig, m);
    if (st != GS_OK) throw Fail{st};
    GS_CUDA(cudaStreamSynchronize(e->stream));
    latest_stats(e);
    harvest_timing(e);
    check_stats(e);
    if (out) *out = *e->h_stats;
  });
}

// ---------------------------------------------------------------------------
// mesh extraction on the device (metrics.py:148-163 extract_mesh): every
// 3-clique a < b < c of the unit graph once, as indices of the id-ordered
// live units, in the reference's order (a ascending, then b, then c)

namespace {
__global__ void k_alive_flags(const uint8_t* __restrict__ alive, int n, int* __restrict__ flags) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    flags[u] = alive[u] ? 1 : 0;
}

// one thread per unit a: its neighbours above a, sorted; a face per pair
// (b, c) of them that is an edge.  count pass: cnt[a]; write pass: faces
// at off[a]
__global__ void k_faces(DevState S, int n, const int* __restrict__ index,
                        long long* __restrict__ cnt, const long long* __restrict__ off,
                        int64_t* __restrict__ faces) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
    if (!S.alive[a]) {
      if (!off) cnt[a] = 0;
      continue;
    }
    const int d = S.deg[a];
    const int2* A = S.adj + (size_t)a * kMaxDeg;
    int up[kMaxDeg];
    int k = 0;
    for (int q = 0; q < d; ++q) {
      const int v = A[q].x;
      if (v > a) {
        int i = k++;
        while (i > 0 && up[i - 1] > v) {
          up[i] = up[i - 1];
          --i;
        }
        up[i] = v;
      }
    }
    long long f = 0;
    long long o = off ? off[a] : 0;
    for (int i = 0; i < k; ++i) {
      const int b = up[i];
      const int db = S.deg[b];
      const int2* B = S.adj + (size_t)b * kMaxDeg;
      for (int j = i + 1; j < k; ++j) {
        const int c = up[j];
        bool hit = false;
        for (int q = 0; q < db && !hit; ++q) hit = B[q].x == c;
        if (hit) {
          if (off) {
            faces[3 * o] = index[a];
            faces[3 * o + 1] = index[b];
            faces[3 * o + 2] = index[c];
            ++o;
          }
          ++f;
        }
      }
    }
    if (!off) cnt[a] = f;
  }
}
}  // namespace

extern "C" gs_status gs_engine_extract_mesh(gs_engine* e, int64_t cap, int64_t* faces,
                                            int64_t* n_faces, int64_t topo[6]) {
  return guarded([&] {
    GS_CHECK(e && n_faces, GS_VALUE_ERROR, "null argument");
    cudaStream_t st = e->stream;
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaStreamSynchronize(st));
    const int n = hc.next_id;
    const int grid = 4 * e->ctx->sm_count, threads = 256;
    size_t t1 = 0, t2 = 0;
    GS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, (int*)nullptr, (int*)nullptr, n + 1, st));
    GS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, (long long*)nullptr, (long long*)nullptr,
                                          n + 1, st));
    const size_t tb = std::max(t1, t2);
    const size_t bi = ((sizeof(int) * (size_t)(n + 1)) + 255) & ~(size_t)255;
    const size_t bl = ((sizeof(long long) * (size_t)(n + 1)) + 255) & ~(size_t)255;
    char* base = (char*)dmalloc(2 * bi + 2 * bl + tb, st);
    int* flags = (int*)base;
    int* index = (int*)(base + bi);
    long long* cnt = (long long*)(base + 2 * bi);
    long long* off = (long long*)(base + 2 * bi + bl);
    void* temp = base + 2 * bi + 2 * bl;
    int64_t* d_faces = nullptr;
    try {
      GS_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)(n + 1), st));
      GS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long) * (size_t)(n + 1), st));
      if (n) {
        k_alive_flags<<<grid, threads, 0, st>>>(e->S.alive, n, flags);
        k_faces<<<grid, threads, 0, st>>>(e->S, n, nullptr, cnt, nullptr, nullptr);
        e->launches += 2;
        g_launches += 2;
      }
      size_t ta = tb;
      GS_CUDA(cub::DeviceScan::ExclusiveSum(temp, ta, flags, index, n + 1, st));
      ta = tb;
      GS_CUDA(cub::DeviceScan::ExclusiveSum(temp, ta, cnt, off, n + 1, st));
      long long total = 0;
      GS_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
      GS_CUDA(cudaStreamSynchronize(st));
      *n_faces = total;
      d_faces = (int64_t*)dmalloc(sizeof(int64_t) * 3 * (size_t)std::max<long long>(total, 1), st);
      if (n && total) {
        k_faces<<<grid, threads, 0, st>>>(e->S, n, index, cnt, off, d_faces);
        e->launches++;
        g_launches++;
      }
      GS_CUDA(cudaGetLastError());
      if (topo) {
        const unsigned long long before = g_launches;
        mesh_topology_device(*e->ctx, d_faces, total, hc.n_units, topo, st);
        e->launches += (long long)(g_launches - before);
      }
      if (faces && cap >= total && total)
        GS_CUDA(cudaMemcpyAsync(faces, d_faces, sizeof(int64_t) * 3 * (size_t)total,
                                cudaMemcpyDeviceToHost, st));
      GS_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      dfree(d_faces, st);
      dfree(base, st);
      throw;
    }
    dfree(d_faces, st);
    dfree(base, st);
  });
}

// ---------------------------------------------------------------------------
// signal sharding across GPUs (one process per GPU)

extern "C" gs_status gs_shard_unique_id(uint8_t* out, int64_t len) {
  return guarded([&] {
    GS_CHECK(out && len == (int64_t)sizeof(ncclUniqueId), GS_VALUE_ERROR,
             "the shard id buffer must be GS_SHARD_ID_BYTES long");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    GS_CHECK(r == ncclSuccess, GS_CUDA_ERROR, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    memcpy(out, &id, sizeof(id));
  });
}

namespace {
// communicators by (id, world, rank): every engine joined with the same id
// shares one (a run's Network, the next run's Network ...), so only the
// first join pays ncclCommInitRank.  Kept for the life of the process;
// engines sharing one must not run sharded steps concurrently (the
// collectives of one communicator are issued in one order on every rank).
std::mutex g_comm_mu;
std::map<std::string, ncclComm_t> g_comms;
}  // namespace

extern "C" gs_status gs_engine_set_shards(gs_engine* e, int world, int rank, const uint8_t* id,
                                          int64_t len) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CHECK(world >= 0 && (world == 0 || (0 <= rank && rank < world)), GS_VALUE_ERROR,
             "bad world / rank");
    GS_CUDA(cudaStreamSynchronize(e->stream));
    e->comm = nullptr;
    e->world = 1;
    e->rank = 0;
    if (world == 0) return;
    GS_CHECK(id && len == (int64_t)sizeof(ncclUniqueId), GS_VALUE_ERROR,
             "the shard id must be GS_SHARD_ID_BYTES long");
    std::string key((const char*)id, (size_t)len);
    key += "/" + std::to_string(world) + "/" + std::to_string(rank) + "/" +
           std::to_string(e->ctx->device);
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comms.find(key);
    if (it == g_comms.end()) {
      ncclUniqueId uid;
      memcpy(&uid, id, sizeof(uid));
      GS_CUDA(cudaSetDevice(e->ctx->device));
      ncclComm_t comm = nullptr;
      const ncclResult_t r = ncclCommInitRank(&comm, world, uid, rank);
      GS_CHECK(r == ncclSuccess, GS_CUDA_ERROR,
               std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      it = g_comms.emplace(key, comm).first;
    }
    e->comm = it->second;
    e->world = world;
    e->rank = rank;
  });
}

extern "C" gs_status gs_engine_exchange_ms(gs_engine* e, double* out) {
  return guarded([&] {
    GS_CHECK(e && out, GS_VALUE_ERROR, "null argument");
    *out = e->exchange_ms;
  });
}

extern "C" gs_status gs_engine_find_device(gs_engine* e, const double* d_sig, int64_t lo,
                                           int64_t hi, void* d_records) {
  return guarded([&] {
    GS_CHECK(e && d_sig && d_records && 0 <= lo && lo <= hi, GS_VALUE_ERROR, "bad find range");
    if (hi == lo) return;
    launch_find(e, d_sig, lo, hi, (WinRec*)d_records);
  });
}

extern "C" gs_status gs_engine_update_device(gs_engine* e, const double* d_sig, int64_t m,
                                             const void* d_records) {
  return guarded([&] {
    GS_CHECK(e && d_sig && d_records && m > 0, GS_VALUE_ERROR, "bad update arguments");
    ensure_capacity(e, m, 3 * m);
    launch_update(e, d_sig, (const WinRec*)d_records, m);
    GS_CUDA(cudaMemcpyAsync(e->h_stats, e->S.stats, sizeof(gs_batch_stats),
                            cudaMemcpyDeviceToHost, e->stream));
    e->ring_latest = false;
  });
}

// resolve_and_update with host-given winners (multi.py:99-131): ids + d_winner
extern "C" gs_status gs_engine_resolve_host(gs_engine* e, const double* signals, int64_t m,
                                            const int64_t* win_b, const int64_t* win_s,
                                            const double* d_win, gs_batch_stats* out) {
  return guarded([&] {
    GS_CHECK(e && signals && win_b && win_s && d_win && m > 0, GS_VALUE_ERROR,
             "bad resolve arguments");
    std::vector<WinRec> recs((size_t)m);
    for (int64_t j = 0; j < m; ++j) {
      const bool ok = win_b[j] >= 0 && win_b[j] < (1LL << 31) && win_s[j] >= 0 &&
                      win_s[j] < (1LL << 31);
      recs[j].b = ok ? (int32_t)win_b[j] : -1;
      recs[j].s = ok ? (int32_t)win_s[j] : -1;
      recs[j].dwin = d_win[j];
    }
    const size_t sb = sizeof(double) * 3 * (size_t)m;
    double* d_sig = (double*)e->sig_buf.get(sb);
    WinRec* d_rec = (WinRec*)e->rec_buf.get(sizeof(WinRec) * (size_t)m);
    GS_CUDA(cudaMemcpyAsync(d_sig, signals, sb, cudaMemcpyHostToDevice, e->stream));
    GS_CUDA(cudaMemcpyAsync(d_rec, recs.data(), sizeof(WinRec) * m, cudaMemcpyHostToDevice,
                            e->stream));
    ensure_capacity(e, m, 3 * m);
    launch_update(e, d_sig, d_rec, m);
    GS_CUDA(cudaMemcpyAsync(e->h_stats, e->S.stats, sizeof(gs_batch_stats),
                            cudaMemcpyDeviceToHost, e->stream));
    e->ring_latest = false;
    GS_CUDA(cudaStreamSynchronize(e->stream));
    check_stats(e);
    if (out) *out = *e->h_stats;
  });
}

extern "C" void* gs_engine_stream(gs_engine* e) { return e ? (void*)e->stream : nullptr; }

extern "C" gs_status gs_engine_reserve(gs_engine* e, int64_t n) {
  return guarded([&] {
    GS_CHECK(e && n >= 0, GS_VALUE_ERROR, "bad reserve");
    ensure_capacity(e, n - e->next_id > 0 ? n - e->next_id : 0, 3 * n);
    GS_CUDA(cudaStreamSynchronize(e->stream));
  });
}

// Empty the network in place (no reallocation): a fresh Network() + RunState().
// Let the host enqueue up to `depth` batches ahead of its stats reads: the
// update kernel turns into a no-op once the network has converged (the
// device counts the batches it really ran), and capacity checks leave room
// for the batches in flight.  depth 0 restores the synchronous contract.
extern "C" gs_status gs_engine_set_async(gs_engine* e, int depth) {
  return guarded([&] {
    GS_CHECK(e && depth >= 0 && depth <= 1024, GS_VALUE_ERROR, "bad async depth");
    e->async_depth = depth;
    drop_prefetch(e);  // prefetched indices (if any) are dropped
    // {halt_on_converge, halted}: leaving async mode also clears the halt, so
    // the network can be stepped further like the reference's
    const int flags[2] = {depth > 0 ? 1 : 0, 0};
    GS_CUDA(cudaMemcpyAsync(&e->S.cnt->halt_on_converge, flags, (depth > 0 ? 1 : 2) * sizeof(int),
                            cudaMemcpyHostToDevice, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
  });
}

extern "C" gs_status gs_engine_reset(gs_engine* e) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    cudaStream_t st = e->stream;
    DevState& S = e->S;
    const int64_t U = e->U;
    GS_CUDA(cudaMemsetAsync(S.alive, 0, U, st));
    GS_CUDA(cudaMemsetAsync(S.deg, 0, sizeof(int32_t) * U, st));
    fill_i32(S.firstwin, U, kNone32, st);
    fill_i32(S.touchfirst, U, kNone32, st);
    fill_i32(S.ttr, U, -1, st);
    fill_i32(S.claim, U, -1, st);
    fill_i32(S.iso_pos, U, -1, st);
    fill_i64(S.la_val, U, -1, st);
    fill_i64(S.la_stamp, U, kNone64, st);
    k_push_free<<<64, 256, 0, st>>>(S.efree, 0, 0, e->EC);
    GS_CUDA(cudaGetLastError());
    Counters init{};
    init.next_sweep = kSweepEvery;
    init.efree_top = e->EC;
    init.halt_on_converge = e->async_depth > 0 ? 1 : 0;
    GS_CUDA(cudaMemcpyAsync(S.cnt, &init, sizeof(Counters), cudaMemcpyHostToDevice, st));
    GS_CUDA(cudaMemsetAsync(S.stats, 0, sizeof(gs_batch_stats), st));
    GS_CUDA(cudaStreamSynchronize(st));
    e->next_id = e->n_edges = e->n_units = 0;
    drop_prefetch(e);
    e->reset_seq = e->issued;
    memset(e->h_stats, 0, sizeof(gs_batch_stats));
    harvest_timing(e);
    e->find_ms = e->update_ms = e->exchange_ms = 0.0;
  });
}

extern "C" int64_t gs_engine_launch_count(const gs_engine* e) { return e ? e->launches : 0; }

extern "C" gs_status gs_engine_counts(gs_engine* e, int64_t out[11]) {
  return guarded([&] {
    GS_CHECK(e && out, GS_VALUE_ERROR, "null argument");
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    out[0] = hc.n_units;
    out[1] = hc.n_edges;
    out[2] = hc.next_id;
    out[3] = hc.tick;
    out[4] = hc.next_sweep;
    out[5] = hc.iso_count;
    out[6] = hc.ring_counts[0];
    out[7] = hc.ring_counts[1];
    out[8] = hc.ring_counts[2];
    out[9] = hc.untrained;
    out[10] = hc.nrows;
  });
}

namespace {
template <class T>
std::vector<T> d2h(const T* p, size_t n, cudaStream_t st) {
  std::vector<T> v(n);
  if (n) GS_CUDA(cudaMemcpyAsync(v.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
  return v;
}
}  // namespace

extern "C" gs_status gs_engine_export_units(gs_engine* e, int64_t cap, int64_t* ids, double* pos,
                                            double* hab, double* theta, int64_t* ring,
                                            int64_t* patience, int64_t* last_active,
                                            int64_t* n_out) {
  return guarded([&] {
    GS_CHECK(e && n_out, GS_VALUE_ERROR, "null argument");
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    const size_t n = (size_t)hc.next_id;
    cudaStream_t st = e->stream;
    auto alive = d2h(e->S.alive, n, st);
    auto p4 = d2h(e->S.pos, n, st);
    auto hb = d2h(e->S.hab, n, st);
    auto th = d2h(e->S.theta, n, st);
    auto rg = d2h(e->S.ring, n, st);
    auto pt = d2h(e->S.patience, n, st);
    auto la = d2h(e->S.la_val, n, st);
    GS_CUDA(cudaStreamSynchronize(st));
    int64_t k = 0;
    for (size_t u = 0; u < n; ++u) {
      if (!alive[u]) continue;
      if (k < cap) {
        if (ids) ids[k] = (int64_t)u;
        if (pos) {
          pos[3 * k] = p4[u].x;
          pos[3 * k + 1] = p4[u].y;
          pos[3 * k + 2] = p4[u].z;
        }
        if (hab) hab[k] = hb[u];
        if (theta) theta[k] = th[u];
        if (ring) ring[k] = rg[u];
        if (patience) patience[k] = pt[u];
        if (last_active) last_active[k] = la[u];
      }
      ++k;
    }
    *n_out = k;
  });
}

// RunState (engine.py:101-119) as arrays over ids [0, next_id): patience,
// last_active (-1 absent) and the dict-order stamp of each last_active entry.
extern "C" gs_status gs_engine_get_run_state(gs_engine* e, int64_t* tick, int64_t* next_sweep,
                                             int64_t cap, int64_t* patience,
                                             int64_t* last_active, int64_t* stamp,
                                             int64_t* n_ids) {
  return guarded([&] {
    GS_CHECK(e && tick && next_sweep && n_ids, GS_VALUE_ERROR, "null argument");
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    const size_t n = (size_t)hc.next_id;
    *tick = hc.tick;
    *next_sweep = hc.next_sweep;
    *n_ids = (int64_t)n;
    if (cap < (int64_t)n) return;
    cudaStream_t st = e->stream;
    auto pt = d2h(e->S.patience, n, st);
    auto la = d2h(e->S.la_val, n, st);
    auto sp = d2h(e->S.la_stamp, n, st);
    GS_CUDA(cudaStreamSynchronize(st));
    for (size_t u = 0; u < n; ++u) {
      if (patience) patience[u] = pt[u];
      if (last_active) last_active[u] = la[u];
      if (stamp) stamp[u] = la[u] == -1 ? -1 : sp[u];
    }
  });
}

// Load a RunState: ids [0, n) take the given values, ids [n, next_id) become
// absent.  Stamps order the last_active entries (dict insertion order) and
// must be < 3 * (tick + 1) so later entries sort after them.
extern "C" gs_status gs_engine_set_run_state(gs_engine* e, int64_t tick, int64_t next_sweep,
                                             int64_t n, const int64_t* patience,
                                             const int64_t* last_active, const int64_t* stamp) {
  return guarded([&] {
    GS_CHECK(e, GS_VALUE_ERROR, "null engine");
    GS_CHECK(tick >= 0 && n >= 0, GS_VALUE_ERROR, "bad run state");
    GS_CHECK(n == 0 || (patience && last_active && stamp), GS_VALUE_ERROR, "null argument");
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    GS_CHECK(n <= hc.next_id, GS_VALUE_ERROR, "run state names an id that was never created");
    const size_t N = (size_t)hc.next_id;
    std::vector<int32_t> pt(N, 0);
    std::vector<long long> la(N, -1), sp(N, kNone64);
    for (int64_t u = 0; u < n; ++u) {
      GS_CHECK(patience[u] >= 0 && patience[u] < (1LL << 31), GS_VALUE_ERROR, "bad patience");
      GS_CHECK(last_active[u] >= -1, GS_VALUE_ERROR, "bad last_active");
      pt[u] = (int32_t)patience[u];
      if (last_active[u] != -1) {
        GS_CHECK(stamp[u] < 3 * (tick + 1), GS_VALUE_ERROR, "bad last_active order stamp");
        la[u] = last_active[u];
        sp[u] = stamp[u];
      }
    }
    cudaStream_t st = e->stream;
    if (N) {
      GS_CUDA(cudaMemcpyAsync(e->S.patience, pt.data(), sizeof(int32_t) * N,
                              cudaMemcpyHostToDevice, st));
      GS_CUDA(cudaMemcpyAsync(e->S.la_val, la.data(), sizeof(long long) * N,
                              cudaMemcpyHostToDevice, st));
      GS_CUDA(cudaMemcpyAsync(e->S.la_stamp, sp.data(), sizeof(long long) * N,
                              cudaMemcpyHostToDevice, st));
    }
    const long long clocks[2] = {tick, next_sweep};
    GS_CUDA(cudaMemcpyAsync(&e->S.cnt->tick, clocks, sizeof(clocks), cudaMemcpyHostToDevice, st));
    GS_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" gs_status gs_engine_export_edges(gs_engine* e, int64_t cap, int64_t* abage,
                                            int64_t* n_out) {
  return guarded([&] {
    GS_CHECK(e && n_out, GS_VALUE_ERROR, "null argument");
    Counters hc;
    GS_CUDA(cudaMemcpyAsync(&hc, e->S.cnt, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    const size_t n = (size_t)hc.next_id;
    cudaStream_t st = e->stream;
    auto alive = d2h(e->S.alive, n, st);
    auto deg = d2h(e->S.deg, n, st);
    auto adj = d2h(e->S.adj, n * kMaxDeg, st);
    auto age = d2h(e->S.eage, (size_t)e->EC, st);
    GS_CUDA(cudaStreamSynchronize(st));
    std::vector<std::array<int64_t, 3>> out;
    for (size_t a = 0; a < n; ++a) {
      if (!alive[a]) continue;
      for (int k = 0; k < deg[a]; ++k) {
        const int2 ent = adj[a * kMaxDeg + k];
        if ((int64_t)a < ent.x) out.push_back({(int64_t)a, (int64_t)ent.x, (int64_t)age[ent.y]});
      }
    }
    std::sort(out.begin(), out.end());
    const int64_t ne = (int64_t)out.size();
    for (int64_t i = 0; i < ne && i < cap; ++i) {
      abage[3 * i] = out[i][0];
      abage[3 * i + 1] = out[i][1];
      abage[3 * i + 2] = out[i][2];
    }
    *n_out = ne;
  });
}

extern "C" gs_status gs_engine_audit(gs_engine* e, int64_t* violations) {
  return guarded([&] {
    GS_CHECK(e && violations, GS_VALUE_ERROR, "null argument");
    unsigned long long* d = (unsigned long long*)e->d_res;
    GS_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), e->stream));
    k_audit<<<1, 1024, 0, e->stream>>>(e->S, e->P, d);
    GS_CUDA(cudaGetLastError());
    GS_CUDA(cudaMemcpyAsync(e->h_res, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    *violations = (int64_t)e->h_res[0];
  });
}
