// update_kernel.cuh -- the batch update kernel (included by engine.cu).
//
// Windowed segmented replay of the reference's sequential update loop
// (multi.py:120-130 -> engine.py:283-355); see the engine.cu header for the
// argument.  One cluster of 8 CTAs x 1024 threads (8 SMs, cluster barriers
// between phases) processes windows of up to 8192 signals:
//
//   A  candidates: alive winner and second, winner not yet claimed this
//      batch; atomicMin(firstwin[b], j) -- the first candidate per winner is
//      the processed signal.  Processed signals are compacted, in batch
//      order, into a dense shared list (their rank is their tick offset).
//   B  one thread per processed signal evaluates, against the window-start
//      state, whether it changes the topology or needs the serial path:
//      a new b-s edge, an insertion, an edge crossing max_age, isolated units
//      awaiting prune, or a sweep that could remove a live unit.  Sweeps
//      that provably remove nothing (every live unit's last_active >= the
//      sweep cutoff) only move the sweep clock and stay on the fast path.
//      It also evaluates adapt_threshold (engine.py:208-265) at its time.
//   C  commits every processed signal before the first event: claims,
//      last_active (+ dict order stamps), patience / threshold, edge ages
//      (replayed by the later of the edge's two touching signals) and, for
//      every touched unit, its position / habituation sequence replayed in
//      batch order by one owner thread with the exact binary64 rounding.
//   D  the event signal runs exactly as update_single on thread 0 (the
//      sweep's stale scan is block-parallel); the next window starts after it.


// Neighbour lists up to kStage long are staged in registers so their loads
// (and the loads that depend on them) issue together instead of as a chain
// of dependent L2 round trips; longer lists take the plain loops.
#ifndef GS_PROF_B
#define GS_PROF_B 0
#endif
#ifndef GS_PROF_TAIL
#define GS_PROF_TAIL 0
#endif
#ifndef GS_PROF_EV
#define GS_PROF_EV 0
#endif
#ifndef GS_STATS_FENCE
#define GS_STATS_FENCE 0
#endif
#ifndef GS_STAGE
#define GS_STAGE 8
#endif
constexpr int kStage = GS_STAGE;

// 16-byte loads: two entries per load, so a row costs half the LSU
// wavefronts (these scattered loads are what bounds the window phases)
__device__ __forceinline__ void stage_adj(const int2* A, int d, int2 (&nb)[kStage]) {
  const int4* A4 = reinterpret_cast<const int4*>(A);
#pragma unroll
  for (int k = 0; k < kStage / 2; ++k) {
    const int4 v = 2 * k < d ? A4[k] : make_int4(-1, -1, -1, -1);
    nb[2 * k] = make_int2(v.x, v.y);
    nb[2 * k + 1] = 2 * k + 1 < d ? make_int2(v.z, v.w) : make_int2(-1, -1);
  }
}

// the event path's functions out of line (fewer spills in B / the walk, but
// measured slower: cfg3 395 vs 382 ms, the calls sit on the event's latency)
#ifndef GS_EV_NOINLINE
#define GS_EV_NOINLINE 0
#endif
#if GS_EV_NOINLINE
#define GS_EVNOINLINE __noinline__
#else
#define GS_EVNOINLINE
#endif
#ifndef GS_OPT_STAGEALL_B
#define GS_OPT_STAGEALL_B 1
#endif
#ifndef GS_OPT_STAGEALL_W
#define GS_OPT_STAGEALL_W 0
#endif
// the first kStage slots of a row regardless of the degree (rows hold kMaxDeg
// slots, so the loads never leave the row): they issue together with the
// degree load instead of after it; callers ignore slots past the degree
__device__ __forceinline__ void stage_adj_all(const int2* A, int2 (&nb)[kStage]) {
  const int4* A4 = reinterpret_cast<const int4*>(A);
#pragma unroll
  for (int k = 0; k < kStage / 2; ++k) {
    const int4 v = A4[k];
    nb[2 * k] = make_int2(v.x, v.y);
    nb[2 * k + 1] = make_int2(v.z, v.w);
  }
}

__device__ __forceinline__ void replay_event(double4& p, double& h, const Params& P,
                                             const double* sig, int key) {
  const size_t j = (size_t)(key >> 1);
  const double x = sig[3 * j], y = sig[3 * j + 1], z = sig[3 * j + 2];
  if (key & 1) {
    move_toward(p, P.eps_b, x, y, z);
    h = dmul(h, P.c_b);
  } else {
    move_toward(p, P.eps_n, x, y, z);
    h = dmul(h, P.c_n);
  }
}

// replay unit u's updates from the committed signals (< jstar) of this window
// in batch order: keys (j << 1) | self are unique (a signal has one winner),
// so "smallest key above the last one" walks them in order without sorting.
// Computes without storing: p / h are u's values after the replay, the
// return value the largest signal index replayed (-1: none, u unchanged).
// tt: the signal after whose update u's habituation first drops below h_t
// (-1: trained already, kNone: not within the replay) -- habituation only
// decays, so "u trained after the updates of signals <= j" is tt <= j.
__device__ int walk_compute(const DevState& S, const Params& P, const double* sig, int u,
                            int jstar, double4& p, double& h, int& tt) {
  const int2* A = S.adj + (size_t)u * kMaxDeg;
  const int d = S.deg[u];
  const int jself = S.firstwin[u];
  p = S.pos[u];
  h = S.hab[u];
  constexpr int kNone = 0x7fffffff;
  tt = h < P.h_t ? -1 : kNone;
  int last = -1;
  if (d <= 2 * kStage) {
    // up to 2*kStage neighbours: keys staged in registers, two chunks of loads
    constexpr int kK = 2 * kStage;
    int key[kK + 1];
    int2 nb[2][kStage];
#if GS_OPT_STAGEALL_W
    stage_adj_all(A, nb[0]);
    stage_adj_all(A + kStage, nb[1]);
#else
    stage_adj(A, min(kStage, d), nb[0]);
    stage_adj(A + kStage, d - kStage, nb[1]);
#endif
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int dc = min(kStage, d - c * kStage);
#pragma unroll
      for (int k = 0; k < kStage; ++k) {
        const int jw = k < dc ? S.firstwin[nb[c][k].x] : kNone;
        key[c * kStage + k] = jw < jstar ? (jw << 1) : kNone;
      }
    }
    key[kK] = jself < jstar ? ((jself << 1) | 1) : kNone;
    // four events per group: their signal loads issue together
#pragma unroll 1
    for (int grp = 0; grp < (kK + 4) / 4; ++grp) {
      int cur[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int cc = kNone;
#pragma unroll
        for (int k = 0; k <= kK; ++k) cc = (key[k] > last && key[k] < cc) ? key[k] : cc;
        cur[q] = cc;
        if (cc != kNone) last = cc;
      }
      double xs[4], ys[4], zs[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cur[q] != kNone) {
          const size_t j = (size_t)(cur[q] >> 1);
          xs[q] = sig[3 * j];
          ys[q] = sig[3 * j + 1];
          zs[q] = sig[3 * j + 2];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cur[q] == kNone) break;
        if (cur[q] & 1) {
          move_toward(p, P.eps_b, xs[q], ys[q], zs[q]);
          h = dmul(h, P.c_b);
        } else {
          move_toward(p, P.eps_n, xs[q], ys[q], zs[q]);
          h = dmul(h, P.c_n);
        }
        if (tt == kNone && h < P.h_t) tt = cur[q] >> 1;
      }
      if (cur[3] == kNone) break;
    }
  } else {
    while (true) {
      int cur = (jself < jstar && ((jself << 1) | 1) > last) ? ((jself << 1) | 1) : kNone;
      for (int k = 0; k < d; ++k) {
        const int jw = S.firstwin[A[k].x];
        const int kk = jw < jstar ? (jw << 1) : kNone;
        if (kk > last && kk < cur) cur = kk;
      }
      if (cur == kNone) break;
      replay_event(p, h, P, sig, cur);
      if (tt == kNone && h < P.h_t) tt = cur >> 1;
      last = cur;
    }
  }
  return last < 0 ? -1 : (last >> 1);
}

// store a walked unit (h0: its habituation before the replay)
__device__ __forceinline__ void walk_store(const DevState& S, const Params& P, int u,
                                           const double4& p, double h, double h0) {
  S.pos[u] = p;
  S.hab[u] = h;
  if (h0 >= P.h_t && h < P.h_t) atomicSub(&S.cnt->untrained, 1);
}

__device__ void walk_unit(const DevState& S, const Params& P, const double* sig, int u,
                          int jstar) {
  double4 p;
  double h;
  int tt;
  const double h0 = S.hab[u];
  if (walk_compute(S, P, sig, u, jstar, p, h, tt) >= 0) walk_store(S, P, u, p, h, h0);
}

// one chunk of the winner b's adjacency for B: the event tests (b-s edge
// exists, an edge crossing max_age) and, per entry, the C1 edge-age replay
// value (age after this signal) and the neighbour's first processed signal,
// all against the window-start state
struct BScan {
  bool found;
  bool ev;
  int kcn;
};
__device__ __forceinline__ void b_chunk(const DevState& S, const Params& P,
                                        const WinRec* __restrict__ rec, int b, int s, int jj,
                                        bool b_trained, const int2 (&nb)[kStage], int dc,
                                        int (&na)[kStage], int (&jvo)[kStage], BScan& acc) {
  int age[kStage], jv[kStage];
#pragma unroll
  for (int k = 0; k < kStage; ++k) {
    const bool valid = k < dc;
    age[k] = valid ? S.eage[nb[k].y] : 0;
    jv[k] = valid ? S.firstwin[nb[k].x] : kNone32;
  }
  int sv[kStage];
#pragma unroll
  for (int k = 0; k < kStage; ++k) sv[k] = (k < dc && jv[k] < jj) ? rec[jv[k]].s : -1;
#pragma unroll
  for (int k = 0; k < kStage; ++k) {
    jvo[k] = jv[k];
    na[k] = 0;
    if (k >= dc) continue;
    const bool is_s = nb[k].x == s;
    acc.found |= is_s;
    const bool age_risk = !is_s && age[k] + 2 > P.max_age;
    if (!b_trained || age_risk) {
      if (jv[k] < jj) acc.kcn++;
      if (age_risk) {
        const int a2 = jv[k] < jj ? ((sv[k] == b) ? 0 : age[k] + 1) : age[k];
        if (a2 + 1 > P.max_age) acc.ev = true;
      }
    }
    int a = age[k];
    if (jv[k] < jj) a = (sv[k] == b) ? 0 : a + 1;
    na[k] = is_s ? 0 : a + 1;
  }
}

__device__ __forceinline__ double pow_chain(double h, double c, int k) {
  for (int i = 0; i < k; ++i) h = dmul(h, c);
  return h;
}

__device__ long long block_min_ll(long long v, long long* s_ll32) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  __syncthreads();
  if (lane == 0) s_ll32[wid] = v;
  __syncthreads();
  if (wid == 0) {
    long long x = lane < (int)(blockDim.x >> 5) ? s_ll32[lane] : 0x7fffffffffffffffLL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long t = __shfl_xor_sync(0xffffffffu, x, o);
      x = t < x ? t : x;
    }
    if (lane == 0) s_ll32[32] = x;
  }
  __syncthreads();
  return s_ll32[32];
}


// _classify_ring (network.py:379-414), one warp: lane a owns neighbour a of u
// and counts its induced degree against N(u) staged in shared memory; the
// connectivity test expands a bitmask frontier with warp OR-reductions.
// All 32 lanes must call it with the same u.
// (k, v: u's degree and slot `lane` of its row, loaded by the caller)
__device__ int classify_ring_warp(const DevState& S, int u, int* sh, int k, int v) {
  const int lane = threadIdx.x & 31;
  if (k < 2) return kRingInc;
  if (k > 32) return classify_ring(S, u);
  if (lane < k) sh[lane] = v;
  __syncwarp();
  unsigned mask = 0;  // bit i: N(u)[i] is adjacent to this lane's neighbour
  if (lane < k) {
    const int2* V = S.adj + (size_t)v * kMaxDeg;
    const int dv = S.deg[v];
    int2 nb[kStage];
    stage_adj(V, kStage, nb);
    for (int c0 = 0;;) {
      for (int i = 0; i < k; ++i) {
        const int x = sh[i];
#pragma unroll
        for (int c = 0; c < kStage; ++c)
          if (c0 + c < dv && nb[c].x == x) mask |= 1u << i;
      }
      c0 += kStage;
      if (c0 >= dv) break;
      stage_adj(V + c0, min(kStage, dv - c0), nb);
    }
  }
  const int d = __popc(mask);
  const bool bad = lane < k && (d == 0 || d > 2);
  const unsigned bal_bad = __ballot_sync(0xffffffffu, bad);
  const int deg1 = __popc(__ballot_sync(0xffffffffu, lane < k && d == 1));
  const int deg2 = __popc(__ballot_sync(0xffffffffu, lane < k && d == 2));
  __syncwarp();  // sh is reused by the next call
  if (bal_bad) return kRingInc;
  int shape;
  if (deg1 == 0 && deg2 == k && k >= 3) shape = kRingDisk;
  else if (deg1 == 2 && deg1 + deg2 == k) shape = kRingHalf;
  else return kRingInc;
  unsigned seen = 1u;
  while (true) {
    const unsigned grow = __reduce_or_sync(0xffffffffu, (lane < k && ((seen >> lane) & 1u)) ? mask : 0u);
    const unsigned nxt = seen | grow;
    if (nxt == seen) break;
    seen = nxt;
  }
  return __popc(seen) == k ? shape : kRingInc;
}

// event path, part 1a (lane 0): update_single up to and including the edge
// aging (engine.py:303-308); over-age neighbours are recorded for prune
__device__ void event_part1a(const DevState& S, const Params& P, int b, int s, int* over,
                             int* nover) {
  Counters* c = S.cnt;
  const long long tick = ++c->tick;
  touch_active(S, b, tick, 0);
  touch_active(S, s, tick, 1);
  const int created = connect_or_reset(S, b, s);
  if (created > 0) c->ev_create++;
  *nover = 0;
  if (created >= 0) age_incident(S, P, b, s, 1, over, nover);
}

// part 1b (lane 0): maybe_insert, prune (engine.py:335-344); returns 1 when
// the sweep clock fired
__device__ int event_part1b(const DevState& S, const Params& P, int b, int s, double dw,
                            double x, double y, double z, const int* over, int nover) {
  Counters* c = S.cnt;
  const long long tick = c->tick;
  if (dw > S.theta[b] && S.hab[b] < P.h_t) {
    const double4 wp = S.pos[b];
    const double theta_b = S.theta[b];
    const int r = add_unit(S, P, dmul(dadd(wp.x, x), 0.5), dmul(dadd(wp.y, y), 0.5),
                           dmul(dadd(wp.z, z), 0.5), theta_b);
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

// ---------------------------------------------------------------------------
// Warp-cooperative event path.  The event signal runs update_single's
// topology work on one warp: every lane calls these with the same
// arguments, adjacency rows are scanned lane-parallel (one dependent load
// level instead of a per-entry chain), lane 0 performs the scalar updates
// in the reference's order, and __syncwarp orders them for the other lanes.
// Ring recomputes are deferred (S.defer_n set), exactly as in the serial
// primitives they replace (engine.cu: find_slot, connect_or_reset,
// remove_edge, age_incident, prune_winner; network.py:261-369).

// slot of b in a's adjacency, or -1 (uniform)
// deg(a) and slot `lane` of a's row issued together (one load level instead
// of two; slots past the degree are ignored by the callers)
__device__ __forceinline__ int2 row_lane(const DevState& S, int a, int& d) {
  d = S.deg[a];
  return S.adj[(size_t)a * kMaxDeg + (threadIdx.x & 31)];
}

__device__ int w_find_slot(const DevState& S, int a, int b) {
  const int lane = threadIdx.x & 31;
  int d;
  const int2 e0 = row_lane(S, a, d);
  unsigned bal = __ballot_sync(0xffffffffu, lane < d && e0.x == b);
  if (bal) return __ffs(bal) - 1;
  const int2* A = S.adj + (size_t)a * kMaxDeg;
  for (int k0 = 32; k0 < d; k0 += 32) {
    const int k = k0 + lane;
    bal = __ballot_sync(0xffffffffu, k < d && A[k].x == b);
    if (bal) return k0 + __ffs(bal) - 1;
  }
  return -1;
}

// deferred _recompute_ring for u (lanes may call it concurrently; the list
// is deduplicated when it is consumed)
__device__ __forceinline__ void w_defer(const DevState& S, int u) { defer_push(S, u); }

// defer the rings of _ring_neighborhood(a, b) (network.py:424-433): the
// common neighbours of a and b, then a and b.  stage: per-warp smem (64 ints)
__device__ void w_defer_ring_neighborhood(const DevState& S, int a, int b, int* stage) {
  const int lane = threadIdx.x & 31;
  int db, da;
  const int2 eb = row_lane(S, b, db);
  const int2 ea = row_lane(S, a, da);
  const int2* Bb = S.adj + (size_t)b * kMaxDeg;
  if (lane < db) stage[lane] = eb.x;
  for (int k = lane + 32; k < db; k += 32) stage[k] = Bb[k].x;
  __syncwarp();
  const int2* Aa = S.adj + (size_t)a * kMaxDeg;
  for (int k = lane; k < da; k += 32) {
    const int v = k < 32 ? ea.x : Aa[k].x;
    bool common = false;
    if (v != b)
      for (int q = 0; q < db; ++q) common |= stage[q] == v;
    if (common) w_defer(S, v);
  }
  if (lane == 0) {
    w_defer(S, a);
    w_defer(S, b);
  }
  __syncwarp();
}

// connect_or_reset (network.py:261-282): 1 created, 0 reset, -1 error (uniform)
__device__ int w_connect_or_reset(const DevState& S, int a, int b, int* stage) {
  const int lane = threadIdx.x & 31;
  const int k = w_find_slot(S, a, b);
  if (k >= 0) {
    if (lane == 0) S.eage[S.adj[(size_t)a * kMaxDeg + k].y] = 0;
    __syncwarp();
    return 0;
  }
  int ok = 0;
  if (lane == 0) {
    Counters* c = S.cnt;
    if (S.deg[a] >= kMaxDeg || S.deg[b] >= kMaxDeg) {
      set_err(S, E_DEGREE);
    } else if (c->efree_top <= 0) {
      set_err(S, E_EDGE_CAP);
    } else {
      const int e = S.efree[--c->efree_top];
      S.eage[e] = 0;
      if (S.deg[a] == 0) iso_del(S, a);
      if (S.deg[b] == 0) iso_del(S, b);
      S.adj[(size_t)a * kMaxDeg + S.deg[a]++] = make_int2(b, e);
      S.adj[(size_t)b * kMaxDeg + S.deg[b]++] = make_int2(a, e);
      c->n_edges++;
      const int dm = max(S.deg[a], S.deg[b]);
      if (dm > c->max_degree) c->max_degree = dm;
      ok = 1;
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  if (!ok) return -1;
  w_defer_ring_neighborhood(S, a, b, stage);
  return 1;
}

// _remove_edge_raw (network.py:453-462)
__device__ void w_remove_edge_raw(const DevState& S, int a, int b) {
  const int lane = threadIdx.x & 31;
  const int ka = w_find_slot(S, a, b);
  const int kb = w_find_slot(S, b, a);
  if (lane == 0) {
    if (ka < 0 || kb < 0) {
      set_err(S, E_NOEDGE);
    } else {
      Counters* c = S.cnt;
      int2* A = S.adj + (size_t)a * kMaxDeg;
      int2* B = S.adj + (size_t)b * kMaxDeg;
      const int e = A[ka].y;
      const int da = --S.deg[a];
      A[ka] = A[da];
      const int db = --S.deg[b];
      B[kb] = B[db];
      S.efree[c->efree_top++] = e;
      c->n_edges--;
      if (da == 0) iso_add(S, a);
      if (db == 0) iso_add(S, b);
    }
  }
  __syncwarp();
}

// age_incident_edges(b, inc, exclude) with the over-age registry
// (network.py:294-319); crossing neighbours land in over[] in adjacency order
__device__ void w_age_incident(const DevState& S, const Params& P, int b, int exclude, int inc,
                               int* over, int* nover) {
  const int lane = threadIdx.x & 31;
  int d;
  const int2 e0 = row_lane(S, b, d);
  const int2* B = S.adj + (size_t)b * kMaxDeg;
  int n = 0;
  for (int k0 = 0; k0 < d; k0 += 32) {
    const int k = k0 + lane;
    bool cross = false;
    int v = -1;
    if (k < d) {
      const int2 ent = k0 == 0 ? e0 : B[k];
      v = ent.x;
      if (v != exclude) {
        const int old = S.eage[ent.y];
        const int nw = old + inc;
        S.eage[ent.y] = nw;
        cross = nw > P.max_age && old <= P.max_age;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, cross);
    if (cross) over[n + __popc(bal & ((1u << lane) - 1u))] = v;
    n += __popc(bal);
  }
  if (lane == 0) *nover = n;
  __syncwarp();
}

// prune on the winner's over-age edges (network.py:321-369), as prune_winner
__device__ void w_prune_winner(const DevState& S, const Params& P, int b, const int* over,
                               int nover, int* stage, int* pe, int* pu) {
  const int lane = threadIdx.x & 31;
  *pe = 0;
  *pu = 0;
  if (nover == 0 && S.cnt->iso_count == 0) return;
  for (int i = 0; i < nover; ++i) {
    w_defer_ring_neighborhood(S, b, over[i], stage);
    w_remove_edge_raw(S, b, over[i]);
  }
  int removed = 0;
  if (lane == 0) removed = remove_lonely(S, P);
  *pu = __shfl_sync(0xffffffffu, removed, 0);
  *pe = nover;
  __syncwarp();
}

// sweep clock (no stale units to remove) + adapt_threshold (engine.py:208-238,
// 345-355), whole warp: the neighbours' habituation is checked lane-parallel
__device__ GS_EVNOINLINE void w_event_part2(const DevState& S, const Params& P, int b, bool sweep_fired) {
  const int lane = threadIdx.x & 31;
  Counters* c = S.cnt;
  if (lane == 0 && sweep_fired) c->next_sweep = c->tick + kSweepEvery;
  if (!S.alive[b]) return;
  const int ring = S.ring[b];
  if (ring == kRingDisk || (P.allow_boundary && ring == kRingHalf)) {
    if (lane == 0) S.patience[b] = 0;
    return;
  }
  if (S.hab[b] >= P.h_t) return;
  int d;
  const int2 e0 = row_lane(S, b, d);
  const int2* B = S.adj + (size_t)b * kMaxDeg;
  bool untrained = false;
  for (int k = lane; k < d; k += 32) untrained |= S.hab[(k < 32 ? e0 : B[k]).x] >= P.h_t;
  if (__any_sync(0xffffffffu, untrained)) return;
  if (lane == 0) {
    int count = S.patience[b] + 1;
    if (count >= P.ring_patience) {
      S.theta[b] = dmul(S.theta[b], P.rho);
      count = 0;
    }
    S.patience[b] = count;
  }
}

// update_single up to the edge aging (engine.py:303-308), whole warp
__device__ GS_EVNOINLINE void w_event_part1a(const DevState& S, const Params& P, int b, int s, int* over,
                               int* nover, int* stage) {
  const int lane = threadIdx.x & 31;
  Counters* c = S.cnt;
  if (lane == 0) {
    const long long tick = ++c->tick;
    touch_active(S, b, tick, 0);
    touch_active(S, s, tick, 1);
  }
  __syncwarp();
  const int created = w_connect_or_reset(S, b, s, stage);
  if (lane == 0) {
    if (created > 0) c->ev_create++;
    *nover = 0;
  }
  __syncwarp();
  if (created >= 0) w_age_incident(S, P, b, s, 1, over, nover);
}

// maybe_insert + prune (engine.py:335-344), whole warp; 1 when the sweep
// clock fired (uniform)
// (thb, hb, wp: the winner's threshold, habituation and position after its
// move, as the first part left them)
__device__ GS_EVNOINLINE int w_event_part1b(const DevState& S, const Params& P, int b, int s, double dw,
                              double x, double y, double z, const int* over, int nover,
                              int* stage, double thb, double hb, const double4& wp) {
  const int lane = threadIdx.x & 31;
  Counters* c = S.cnt;
  const long long tick = c->tick;
  if (dw > thb && hb < P.h_t) {
    int r = -1;
    if (lane == 0) {
      r = add_unit(S, P, dmul(dadd(wp.x, x), 0.5), dmul(dadd(wp.y, y), 0.5),
                   dmul(dadd(wp.z, z), 0.5), thb);
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    __syncwarp();
    if (r < 0) return 0;
    w_connect_or_reset(S, r, b, stage);
    w_connect_or_reset(S, r, s, stage);
    if (w_find_slot(S, b, s) >= 0) {
      w_defer_ring_neighborhood(S, b, s, stage);
      w_remove_edge_raw(S, b, s);
    }
    if (lane == 0) {
      touch_active(S, r, tick, 2);
      c->ev_insert++;
    }
    __syncwarp();
  }
  int pe, pu;
  w_prune_winner(S, P, b, over, nover, stage, &pe, &pu);
  int fired = 0;
  if (lane == 0) {
    if (pe || pu) c->ev_prune++;
    fired = tick >= c->next_sweep ? 1 : 0;
  }
  return __shfl_sync(0xffffffffu, fired, 0);
}

// update_single up to and including the moves (engine.py:297-333) for a
// winner and second of degree < 32, with every load issued up front: the two
// rows, the winner's / second's scalars and the top of the free-edge stack in
// one level, the winner's edge ages and neighbours' positions in the next;
// then connect_or_reset (network.py:261-282), the ring-neighbourhood defers
// (common neighbours from the two staged rows), age_incident_edges
// (network.py:294-319, over-age neighbours in row order) and the moves run on
// registers.  Whole warp, uniform arguments; lane 0's thb / hb / pb: the
// winner's threshold, habituation and position afterwards.
__device__ GS_EVNOINLINE void w_event_first(const DevState& S, const Params& P, int b, int s, double x,
                              double y, double z, int db, int2 eb, int ds, int2 es, int* over,
                              int* nover, int* stage, double& thb, double& hb, double4& pb) {
  const int lane = threadIdx.x & 31;
  Counters* c = S.cnt;
  // level 2 loads (the rows came with the caller's dispatch)
  long long la = 0;
  if (lane < 2) la = S.la_val[lane ? s : b];
  double4 ps = make_double4(0.0, 0.0, 0.0, 0.0);
  double hs = 0.0;
  int enext = -1;
  int top = 0;  // lane 0's (the only lane that uses or moves the free-edge stack)
  if (lane == 0) {
    top = c->efree_top;
    pb = S.pos[b];
    hb = S.hab[b];
    thb = S.theta[b];
    ps = S.pos[s];
    hs = S.hab[s];
    if (top > 0) enext = S.efree[top - 1];
  }
  // level 3: the winner's edge ages and neighbours
  int ag = 0;
  double4 pv = make_double4(0.0, 0.0, 0.0, 0.0);
  double hv = 0.0;
  if (lane < db) {
    ag = S.eage[eb.y];
    pv = S.pos[eb.x];
    hv = S.hab[eb.x];
  }
  // touch_active(b), touch_active(s) (engine.py:301-302): distinct units
  long long tick = 0;
  if (lane == 0) tick = ++c->tick;
  tick = __shfl_sync(0xffffffffu, tick, 0);
  if (lane < 2) {
    const int u = lane ? s : b;
    if (la == -1) S.la_stamp[u] = 3 * tick + lane;
    S.la_val[u] = tick;
  }
  // connect_or_reset(b, s)
  const unsigned fb = __ballot_sync(0xffffffffu, lane < db && eb.x == s);
  int created;
  if (fb) {
    const int k = __ffs(fb) - 1;
    if (lane == k) S.eage[eb.y] = 0;
    created = 0;
  } else {
    int ok = 0;
    if (lane == 0) {
      if (top <= 0) {
        set_err(S, E_EDGE_CAP);
      } else {
        c->efree_top = top - 1;
        const int e = enext;
        S.eage[e] = 0;
        if (db == 0) iso_del(S, b);
        if (ds == 0) iso_del(S, s);
        S.adj[(size_t)b * kMaxDeg + db] = make_int2(s, e);
        S.adj[(size_t)s * kMaxDeg + ds] = make_int2(b, e);
        S.deg[b] = db + 1;
        S.deg[s] = ds + 1;
        c->n_edges++;
        const int dm = max(db, ds) + 1;
        if (dm > c->max_degree) c->max_degree = dm;
        c->ev_create++;
        ok = 1;
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    created = ok ? 1 : -1;
    if (ok) {
      // _ring_neighborhood(b, s) (network.py:424-433): the common neighbours
      // of the rows before the new edge, then b and s
      if (lane < ds) stage[lane] = es.x;
      __syncwarp();
      bool common = false;
      if (lane < db && eb.x != s)
        for (int q = 0; q < ds; ++q) common |= stage[q] == eb.x;
      if (common) w_defer(S, eb.x);
      if (lane == 0) {
        w_defer(S, b);
        w_defer(S, s);
      }
      __syncwarp();  // stage is reused by the caller
    }
  }
  // age_incident_edges(b, +1, exclude s): the rows' entries other than s, in
  // row order (the new b-s entry, appended, is the excluded one)
  int n = 0;
  if (created >= 0) {
    bool cross = false;
    if (lane < db && eb.x != s) {
      const int nw = ag + 1;
      S.eage[eb.y] = nw;
      cross = nw > P.max_age && ag <= P.max_age;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, cross);
    if (cross) over[__popc(bal & ((1u << lane) - 1u))] = eb.x;
    n = __popc(bal);
  }
  if (lane == 0) *nover = n;
  // moves: the winner, its neighbours (the rows as they stand now: s joined
  // them if the edge was created)
  if (lane == 0) {
    move_toward(pb, P.eps_b, x, y, z);
    S.pos[b] = pb;
    const double h0 = hb;
    hb = dmul(h0, P.c_b);
    S.hab[b] = hb;
    if (h0 >= P.h_t && hb < P.h_t) atomicSub(&c->untrained, 1);
    if (created == 1) {
      move_toward(ps, P.eps_n, x, y, z);
      S.pos[s] = ps;
      const double h1 = dmul(hs, P.c_n);
      S.hab[s] = h1;
      if (hs >= P.h_t && h1 < P.h_t) atomicSub(&c->untrained, 1);
    }
  }
  if (lane < db) {
    move_toward(pv, P.eps_n, x, y, z);
    S.pos[eb.x] = pv;
    const double h1 = dmul(hv, P.c_n);
    S.hab[eb.x] = h1;
    if (hv >= P.h_t && h1 < P.h_t) atomicSub(&c->untrained, 1);
  }
  __syncwarp();
}

// habituation of neighbour v (untrained at the window start, hvT) at the
// time of signal jj: its decays from the window's signals before jj replayed
// (as a neighbour of their winners, and once as a winner itself)
__device__ __noinline__ double hab_at(const DevState& S, const Params& P, int v, double hvT,
                                      int jj) {
  const int jv = S.firstwin[v];
  const bool vwon = jv < jj;
  const int dv = S.deg[v];
  const int2* V = S.adj + (size_t)v * kMaxDeg;
  int k1 = 0, k2 = 0;
  for (int q0 = 0; q0 < dv; q0 += kStage) {
    const int dq = min(kStage, dv - q0);
    int2 wb[kStage];
    stage_adj(V + q0, dq, wb);
    int jw[kStage];
#pragma unroll
    for (int q = 0; q < kStage; ++q) jw[q] = q < dq ? S.firstwin[wb[q].x] : kNone32;
#pragma unroll
    for (int q = 0; q < kStage; ++q) {
      if (q < dq && jw[q] <= jj) {
        if (vwon && jw[q] > jv) k2++;
        else k1++;
      }
    }
  }
  double hv = pow_chain(hvT, P.c_n, k1);
  if (vwon) hv = dmul(hv, P.c_b);
  return pow_chain(hv, P.c_n, k2);
}

__device__ __forceinline__ bool adapt_ring_ok(const Params& P, int ringb) {
  return ringb == kRingDisk || (P.allow_boundary && ringb == kRingHalf);
}

// neighbours past the walked slots (networks above kWinC units): trained at
// time jj, from their decays replayed against the segment-start state (B)
__device__ bool far_nbrs_trained(const DevState& S, const Params& P, int jj, int db,
                                 const int2 (&nb0)[kStage], const int2 (&nb1)[kStage],
                                 int nwalked) {
#pragma unroll 1
  for (int k = 0; k < db; ++k) {
    int v = -1;
#pragma unroll
    for (int q = 0; q < kStage; ++q) {
      v = q == k ? nb0[q].x : v;
      v = kStage + q == k ? nb1[q].x : v;
    }
    if (v >= nwalked) {
      const double hv = S.hab[v];
      if (hv >= P.h_t && hab_at(S, P, v, hv, jj) >= P.h_t) return false;
    }
  }
  return true;
}

// adapt_threshold outcome (engine.py:208-265) of committed signal jj with
// winner b (degree db <= 2 * kStage, adjacency staged in nb0 / nb1), from
// the segment-start state: -2 none, else patience | shrink << 30.  Every
// neighbour must be trained at time jj (engine.py:225-231): the walk of this
// segment published each unit's time-to-trained (ttr, one load level for all
// neighbours); neighbours past the walked slots were checked in B (far_ok).
__device__ __forceinline__ int adapt_outcome_ttr(const DevState& S, const Params& P, int jj,
                                                 bool hb_low, int ringb, int patb, int db,
                                                 const int2 (&nb0)[kStage],
                                                 const int2 (&nb1)[kStage], int nwalked,
                                                 bool far_ok) {
  if (adapt_ring_ok(P, ringb)) return 0;
  if (!hb_low || !far_ok) return -2;
  int t[2 * kStage];
#pragma unroll
  for (int k = 0; k < kStage; ++k) {
    const int v0 = nb0[k].x, v1 = nb1[k].x;
    t[k] = (k < db && v0 < nwalked) ? S.ttr[v0] : -1;
    t[kStage + k] = (kStage + k < db && v1 < nwalked) ? S.ttr[v1] : -1;
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 2 * kStage; ++k) ok &= t[k] <= jj;
  if (!ok) return -2;
  int cnt = patb + 1;
  const int shrink = cnt >= P.ring_patience ? 1 : 0;
  if (shrink) cnt = 0;
  return cnt | (shrink << 30);
}

// ---------------------------------------------------------------------------
// cluster primitives: kCluster CTAs x 1024 threads cooperate on one window;
// cross-CTA values travel through distributed shared memory and every
// exchange is fenced by the hardware cluster barrier.

#ifndef GS_CLUSTER
#define GS_CLUSTER 16
#endif
constexpr int kCluster = GS_CLUSTER;

// cluster-wide barrier (a plain block barrier for a one-CTA "cluster")
__device__ __forceinline__ void csync() {
  if constexpr (kCluster == 1) {
    __syncthreads();
  } else {
    cg::this_cluster().sync();
  }
}
// split cluster barrier (no memory ordering on the arrive): the kernel's
// start-up barrier overlaps the first window's loads
__device__ __forceinline__ void carrive_relaxed() {
  if constexpr (kCluster > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void carrive_release() {
  if constexpr (kCluster > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cwait() {
  if constexpr (kCluster == 1) {
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
}
template <class T>
__device__ __forceinline__ T* cmap(T* p, int rank) {
  if constexpr (kCluster == 1) {
    return p;
  } else {
    return cg::this_cluster().map_shared_rank(p, rank);
  }
}
__device__ __forceinline__ int crank_of() {
  if constexpr (kCluster == 1) {
    return 0;
  } else {
    return (int)cg::this_cluster().block_rank();
  }
}
constexpr int kWinC = kCluster * kUpdThreads;  // one window signal per thread
// dynamic shared memory of the update kernel: B's per-rank results for C1,
// the walk's replay result
constexpr int kC1Smem = (int)((sizeof(int2) + 2 * sizeof(int)) * 2 * kStage * kUpdThreads +
                              sizeof(int) * kUpdThreads);
constexpr int kUpdDynSmem = kC1Smem + (int)((sizeof(double4) + sizeof(double2)) * kUpdThreads);

// exclusive scan over the whole cluster; s_cta is a [2][kCluster] buffer
// used with alternating parity so a CTA running one call ahead cannot
// overwrite values another CTA has not read yet.
// free: optional (start, total) of the whole warps left over per CTA, i.e.
// the exclusive scan of kUpdThreads - roundup32(CTA total) and its sum
__device__ int cl_excl_scan(int v, int* s_warp, int (*s_cta)[kCluster], int& parity, int* total,
                            int* blocal = nullptr, int* bcount = nullptr, int2* free = nullptr) {
  int btot;
  const int r = block_excl_scan(v, s_warp, &btot);
  if (blocal) *blocal = r;
  if (bcount) *bcount = btot;
  const int me = crank_of();
  if (threadIdx.x < kCluster) {
    int* dst = cmap(&s_cta[parity][0], threadIdx.x);
    dst[me] = btot;
  }
  csync();
  int off = 0, tot = 0, foff = 0, ftot = 0;
#pragma unroll
  for (int q = 0; q < kCluster; ++q) {
    const int t = s_cta[parity][q];
    const int f = kUpdThreads - ((t + 31) & ~31);
    off += q < me ? t : 0;
    tot += t;
    foff += q < me ? f : 0;
    ftot += f;
  }
  parity ^= 1;
  *total = tot;
  if (free) *free = make_int2(foff, ftot);
  return off + r;
}

__device__ int cl_min(int v, int* s_warp, int (*s_cta)[kCluster], int& parity) {
  const int bmin = block_min(v, s_warp);
  const int me = crank_of();
  if (threadIdx.x < kCluster) {
    int* dst = cmap(&s_cta[parity][0], threadIdx.x);
    dst[me] = bmin;
  }
  csync();
  int x = 0x7fffffff;
#pragma unroll
  for (int q = 0; q < kCluster; ++q) x = min(x, s_cta[parity][q]);
  parity ^= 1;
  return x;
}

__device__ long long cl_min_ll(long long v, long long* s_ll32, long long (*s_ctal)[kCluster],
                               int& parity) {
  const long long bmin = block_min_ll(v, s_ll32);
  const int me = crank_of();
  if (threadIdx.x < kCluster) {
    long long* dst = cmap(&s_ctal[parity][0], threadIdx.x);
    dst[me] = bmin;
  }
  csync();
  long long x = 0x7fffffffffffffffLL;
#pragma unroll
  for (int q = 0; q < kCluster; ++q) x = s_ctal[parity][q] < x ? s_ctal[parity][q] : x;
  parity ^= 1;
  return x;
}

// ---------------------------------------------------------------------------
// row-snapshot hand-off to the next find: each CTA arrives once per launch
// after its writes the find reads (snapshot rows, counters); the launch's last
// arrival publishes the batch number (release), see FindArgs::snap_token
// The token is 2 * batch + verdict: verdict 1 tells the next find that its
// speculative candidates (screened against the other slot, with the bound
// 2 x that slot's displacement, the find's own rule) stand -- no row changed
// and no row moved further.
// Each CTA's part of the verdict travels with its arrival (the count of
// failing parts in the arrival word's high half), so the last arrival
// publishes without reading anything else.
__device__ __forceinline__ void snapshot_arrive(const DevState& S, int batch_no, bool part_ok) {
  __syncthreads();
  if (threadIdx.x == 0) {  // (release: covers the CTA's snapshot stores, ordered by the barrier)
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(S.snap_token + crank_of()),
                 "r"(2 * batch_no + (part_ok ? 1 : 0))
                 : "memory");
#ifdef GS_PROF_TL
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&g_tlu2[batch_no & 8191][1], t);
#endif
  }
}

// the next batch's silent-sweep value: minimum last_active over live units
// (after the snapshot hand-off: only the next update reads it)
// (the loads and the warp's minimum before the hand-off, with the snapshot's;
// the fire-and-forget atomic after it)
// (la0 / al0: unit g's last_active and liveness, loaded with the snapshot)
__device__ __forceinline__ long long minla_part(const DevState& S, int g, long long la0, bool al0) {
  long long mla = (la0 != -1 && al0) ? la0 : 0x7fffffffffffffffLL;
  const int nid_e = S.cnt->next_id;
  for (int u = g + kWinC; u < nid_e; u += kWinC) {
    const long long t = S.la_val[u];
    if (t != -1 && S.alive[u] && t < mla) mla = t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long t = __shfl_xor_sync(0xffffffffu, mla, o);
    mla = t < mla ? t : mla;
  }
  return mla;
}
__device__ __forceinline__ void next_minla(const DevState& S, int batch_no, long long mla) {
  if ((threadIdx.x & 31) == 0 && mla != 0x7fffffffffffffffLL)
    atomicMin(&S.cnt->minla_next[(batch_no + 1) & 1], mla);
}

// ---------------------------------------------------------------------------
// the batch update kernel: one cluster of kCluster CTAs (8 SMs)

#if GS_CLUSTER > 1
#define GS_CLUSTER_DIMS __cluster_dims__(kCluster, 1, 1)
#else
#define GS_CLUSTER_DIMS
#endif
__global__ void GS_CLUSTER_DIMS __launch_bounds__(kUpdThreads, 1)
    k_update_batch(DevState S, Params P, const double* __restrict__ sig,
                   const WinRec* __restrict__ rec, int m, int batch_no, int pre_fw,
                   gs_batch_stats* st_out) {
  __shared__ int s_warp[33];
  __shared__ long long s_ll32[33];
  __shared__ int s_cta[2][kCluster];
  __shared__ long long s_ctal[2][kCluster];
  __shared__ int s_i[8];
  __shared__ int s_over[kMaxDeg];
  __shared__ int s_ring_sh[32][33];  // per-warp N(u) staging for classify_ring_warp
  __shared__ int s_stage[kMaxDeg];    // event warp: adjacency staging
  __shared__ int s_defer_n;
  // B's per-rank results for C1 ([entry][thread]: conflict-free), 64 KB
  extern __shared__ __align__(16) unsigned char s_c1dyn[];
  int2 (*s_c1nb)[kUpdThreads] = reinterpret_cast<int2 (*)[kUpdThreads]>(s_c1dyn);
  int (*s_c1a)[kUpdThreads] =
      reinterpret_cast<int (*)[kUpdThreads]>(s_c1dyn + sizeof(int2) * 2 * kStage * kUpdThreads);
  int (*s_c1j)[kUpdThreads] = reinterpret_cast<int (*)[kUpdThreads]>(
      s_c1dyn + (sizeof(int2) + sizeof(int)) * 2 * kStage * kUpdThreads);
  int* s_c1s = s_c1j[2 * kStage];  // C1's packed scalars (one int per thread)
  // the walk's replay result (position; habituation after / before)
  double4* s_wk = reinterpret_cast<double4*>(s_c1dyn + kC1Smem);
  double2* s_wkh = reinterpret_cast<double2*>(s_c1dyn + kC1Smem + sizeof(double4) * kUpdThreads);
  __shared__ bool s_dok[kUpdThreads / 32];  // the snapshot part's displacement within the bound
  __shared__ int s_defer_sm[kDeferSm];  // deferred ring recomputes (event path)
  __shared__ __align__(16) Counters s_cnt;  // event warp's working copy of the counters
  // this CTA's processed signals of the window, compacted in batch order:
  // processed signal k of the CTA is evaluated (B, C1) by thread k, while
  // the unit walks run on the CTA's top threads -- the two dependent-load
  // chains of a window run on different warps instead of one after the other
  __shared__ int4 s_pl[kUpdThreads];      // (signal, winner, second, rank)
  __shared__ double s_pdw[kUpdThreads];   // d_winner
  Counters* c = S.cnt;
  const int tid = threadIdx.x;
  const int crank = crank_of();
  const int g = crank * kUpdThreads + tid;  // cluster-wide thread index
  const bool lead = crank == 0 && tid == 0;
  const int warp = tid >> 5, lane = tid & 31;
  int parity = 0;
#ifdef GS_PROF_TL
  unsigned long long tl0, tl1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl0));
#endif
  // programmatic dependent launch after the find: wait for its records
  // here; the next batch's find may launch at once (its CTAs wait in turn)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef GS_PROF_TL
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl1));
#endif
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (S.cnt->halted) {  // converged earlier in an asynchronous run (uniform)
    // the batch's stats slot still gets the (unchanged) latest values
    if (st_out != S.stats && threadIdx.x == 0 && crank_of() == 0) *st_out = *S.stats;
    if (pre_fw) {  // undo the find's first-signal marks
      const int g0 = crank_of() * kUpdThreads + threadIdx.x;
      if (g0 < m) {
        const int b = rec[g0].b;
        if (b >= 0) S.firstwin[b] = kNone32;
      }
    }
    snapshot_arrive(S, batch_no, false);  // (no snapshot: no verdict)
    return;
  }
  const long long t_kernel = clock64();
  long long t_ph = t_kernel;
  // the lead thread's phase timers in shared memory until the kernel ends (a
  // global read-modify-write per phase would sit on its critical path, and
  // registers for them in every thread would add to the kernel's spills)
  __shared__ long long acc[13];
  if (tid < 13) acc[tid] = 0;
  if (lead) {
    c->minla_next[(batch_no + 1) & 1] = 0x7fffffffffffffffLL;  // the tail's atomicMin target
    c->processed = c->discarded = c->events = c->windows = 0;
    c->inserted_start = c->next_id;
    c->stale_n = 0;
    c->nwalk = 0;
    c->fpm_bits[S.snap] = 0u;
    c->snap_disp[S.snap] = 0u;
  }
  // every CTA of the cluster must have started before the first DSMEM
  // exchange; the lead's resets above are read only after later barriers
  carrive_relaxed();
  bool start_wait = true;
  int j0 = 0;
  // A window [j0, wend) is evaluated once (A: candidates, scan: processed
  // list by rank) and committed in segments of ranks [rbase, r*): after an
  // event that removed no unit the candidate set and ranks are unchanged, so
  // the window RESUMES at rank r*+1 (B re-evaluates the remaining ranks
  // against the post-event state); an event with deaths closes the window
  // and the next one starts at j*+1.
  bool resume = false;
  int rbase = 0, nproc = 0, wend = 0;
  long long tick0 = 0, minla = 0;
  bool cand = false;
  int cb = -1;
  int my_s = -1;      // this thread's window signal's record (second, d_winner)
  double my_dw = 0.0;
  bool my_proc = false;  // this thread's window signal is processed
  // the processed signal this thread evaluates (CTA-local batch order)
  bool p_valid = false;
  int p_j = 0, p_b = -1, p_s = -1, p_rank = 0;
  double p_dw = 0.0;
  int p_abs = 0;
  // the unit slot this thread walks (-1: none): the warps no processed
  // signal occupies take the units, contiguous ranges per CTA from its last
  // thread down; units past the free warps (nwalked) are walked after the
  // window's reduction
  int u_w = -1, nwalked = 0;
  while (j0 < m) {
    if (lead) t_ph = clock64();
    if (!resume) {
      wend = min(j0 + kWinC, m);
      const int next_id = c->next_id;
      tick0 = c->tick;
      const long long next_sweep0 = c->next_sweep;
      // ---- A: candidates; the first candidate per winner is processed.  In
      //      the batch's first window after the engine's own find, the find
      //      resolved them (its records are of live, distinct units, nothing
      //      is claimed yet, and it marked every winner's first signal).
      const bool pre = pre_fw && j0 == 0;
      const int j = j0 + g;
      cand = false;
      cb = -1;
      if (j < wend) {
        const WinRec r = rec[j];
        cb = r.b;
        my_s = r.s;
        my_dw = r.dwin;
        if (pre) {
          cand = r.b >= 0 && r.s >= 0 && r.b != r.s;
        } else {
          cand = r.b >= 0 && r.s >= 0 && r.b < next_id && r.s < next_id && r.b != r.s &&
                 S.alive[r.b] && S.alive[r.s] && S.claim[r.b] != batch_no;
          if (cand) atomicMin(&S.firstwin[r.b], j);
        }
      }
      if (start_wait) {
        cwait();
        start_wait = false;
      }
      if (pre) {
        // minimum last_active over live units (silent-sweep test) as the
        // previous batch left it
        minla = c->minla_next[batch_no & 1];
      } else {
        // window start; it only grows, so later segments may use this
        // (conservative) value
        long long mla = 0x7fffffffffffffffLL;
        if (tick0 + kWinC >= next_sweep0) {
          for (int u = g; u < next_id; u += kWinC) {
            const long long t = S.la_val[u];
            if (t != -1 && S.alive[u] && t < mla) mla = t;
          }
        }
        minla = cl_min_ll(mla, s_ll32, s_ctal, parity);  // cluster barrier: firstwin complete
      }
      if (lead) { const long long t_ = clock64(); acc[0] += t_ - t_ph; t_ph = t_; }
      // every thread keeps its own signal: its processing rank (batch
      // order among the processed signals) is all the later phases need
      my_proc = cand && S.firstwin[cb] == j;
      int bl, bcnt;
      int2 fr;
      const int my_rank =
          cl_excl_scan(my_proc ? 1 : 0, s_warp, s_cta, parity, &nproc, &bl, &bcnt, &fr);
      // whole warps: a warp that held both roles would run the two chains
      // one after the other
      u_w = tid >= ((bcnt + 31) & ~31) ? fr.x + (kUpdThreads - 1 - tid) : -1;
      nwalked = fr.y;
      if (my_proc) {
        s_pl[bl] = make_int4(j, cb, my_s, my_rank);
        s_pdw[bl] = my_dw;
      }
      __syncthreads();
      p_valid = tid < bcnt;
      if (p_valid) {
        const int4 q = s_pl[tid];
        p_j = q.x;
        p_b = q.y;
        p_s = q.z;
        p_rank = q.w;
        p_dw = s_pdw[tid];
      }
      rbase = 0;
      if (lead) { const long long t_ = clock64(); acc[0] += t_ - t_ph; t_ph = t_; }
    }
    const long long next_sweep = c->next_sweep;
    const int n_units = c->n_units;
    const bool iso = c->iso_count > 0;
    // ---- B: events, and everything C1 and the walk need, read once against
    //      the window-start state before the cluster reduction: each
    //      processed signal on the thread that found it in A computes its
    //      event tests, its adapt_threshold outcome and its edge-age replay
    //      values; every thread replays its own unit slot as if the whole
    //      segment commits.  After the reduction only stores remain (the
    //      reads of C1 and the walk no longer follow one another, so the
    //      barrier between them is gone).
    const long long horizon = P.stale_factor * (long long)(n_units > 100 ? n_units : 100);
    long long evkey = 0x7fffffffffffffffLL;  // (rank << 32) | signal of this thread's event
    int c1_ring = 0, c1_patb = 0;            // adapt_threshold inputs (evaluated in C1)
    bool c1_hblow = false, c1_far = true;
    int c1_d = 0;                            // winner degree (<= 2 * kStage)
    int2 c1_nb0[kStage], c1_nb1[kStage];     // its adjacency ...
    int c1_a0[kStage], c1_a1[kStage];        // ... edge ages after this signal ...
    int c1_j0[kStage], c1_j1[kStage];        // ... and the neighbours' first signals
    const int nid_b = c->next_id;
#if GS_PROF_B
    const long long tb0 = clock64();
#endif
    if (p_valid && p_rank >= rbase) {
      const int r = p_rank;
      const int jj = p_j;
      const int b = p_b, s = p_s;
      const long long tick_j = tick0 + r + 1;
      bool ev = iso;
      if (tick_j >= next_sweep && ((tick_j - next_sweep) % kSweepEvery) == 0) {
        const long long cutoff = tick_j - horizon;
        if (cutoff > 0 && (minla < cutoff || n_units <= 2)) ev = true;
      }
      // one load level for the winner's row, degree and scalars; the next
      // for its neighbours (edge ages, first signals, habituation)
      const int2* B = S.adj + (size_t)b * kMaxDeg;
      const int db = S.deg[b];
#if GS_OPT_STAGEALL_B
      stage_adj_all(B, c1_nb0);
      stage_adj_all(B + kStage, c1_nb1);
#else
      stage_adj(B, min(kStage, db), c1_nb0);
      stage_adj(B + kStage, db - kStage, c1_nb1);
#endif
      // habituation only decays, so a unit trained at the window start stays
      // trained: exact per-time values are replayed only for untrained units
      const double hbT = S.hab[b];
      const double thb = S.theta[b];
      const int ringb = S.ring[b], patb = S.patience[b];
      const long long la_b = S.la_val[b], la_s = S.la_val[s];
      const bool b_trained = hbT < P.h_t;
      BScan acc{false, false, 0};
      if (db <= 2 * kStage) {
        b_chunk(S, P, rec, b, s, jj, b_trained, c1_nb0, min(kStage, db), c1_a0, c1_j0, acc);
        b_chunk(S, P, rec, b, s, jj, b_trained, c1_nb1, db - kStage, c1_a1, c1_j1, acc);
        c1_d = db;
      } else {
        ev = true;  // a winner of degree > 2 * kStage takes the serial path (rare)
      }
      if (!acc.found) ev = true;  // connect_or_reset creates b-s
      if (acc.ev) ev = true;
      const bool hb_low = b_trained || dmul(pow_chain(hbT, P.c_n, acc.kcn), P.c_b) < P.h_t;
      if (hb_low && p_dw > thb) ev = true;  // maybe_insert fires
      // last_active presence at the window start (dict order stamps)
      p_abs = (la_b == -1 ? 1 : 0) | (la_s == -1 ? 2 : 0);
      if (ev) evkey = ((long long)r << 32) | (unsigned)jj;
      c1_ring = ringb;
      c1_patb = patb;
      c1_hblow = hb_low;
      // the walk stores of C1's phase race with replays of units past the
      // walked slots: those neighbours are checked here, against the
      // segment-start state (networks above kWinC units only)
      if (nid_b > nwalked && !ev && hb_low && !adapt_ring_ok(P, ringb))
        c1_far = far_nbrs_trained(S, P, jj, db, c1_nb0, c1_nb1, nwalked);
      // C1's inputs wait in shared memory (not in registers across the walk
      // and the reduction: the kernel is at its register limit)
      // (ring 2 bits, hb_low, far, degree 6 bits, patience the rest)
      s_c1s[tid] = c1_ring | (c1_hblow ? 4 : 0) | (c1_far ? 8 : 0) | (c1_d << 4) | (c1_patb << 10);
#pragma unroll
      for (int k = 0; k < kStage; ++k) {
        s_c1nb[k][tid] = c1_nb0[k];
        s_c1nb[kStage + k][tid] = c1_nb1[k];
        s_c1a[k][tid] = c1_a0[k];
        s_c1a[kStage + k][tid] = c1_a1[k];
        s_c1j[k][tid] = c1_j0[k];
        s_c1j[kStage + k][tid] = c1_j1[k];
      }
    }
    // this thread's unit slot replayed as if the whole window commits
    int wk_max = -1;
    if (u_w >= 0 && u_w < nid_b) {
      double4 wk_p;
      double wk_h;
      const double wk_h0 = S.hab[u_w];
      int tt;
      wk_max = walk_compute(S, P, sig, u_w, wend, wk_p, wk_h, tt);
      S.ttr[u_w] = tt;  // read by C1's adapt_threshold after the barrier below
      // the replay waits in shared memory across the reduction (registers
      // are the kernel's limit)
      s_wk[tid] = wk_p;
      s_wkh[tid] = make_double2(wk_h, wk_h0);
    }
#if GS_PROF_B
    {  // the slowest thread's B / walk work before the reduction (cycles)
      const long long tb2 = clock64() + (wk_max & 0) + (evkey & 0);
      const unsigned db_ = __reduce_max_sync(0xffffffffu, (unsigned)min(tb2 - tb0, 0x7fffffffLL));
      if (lane == 0) atomicMax(&c->prof_bmax[0], db_);
      if (lead) acc[3] += tb2 - tb0;  // the lead's own work
#ifdef GS_PROF_DUMP_BATCH
      if (batch_no == GS_PROF_DUMP_BATCH && j0 == 0 && rbase == 0) {
        const int du = u_w >= 0 && u_w < nid_b ? S.deg[u_w] : -1;
        const int db = p_valid ? S.deg[p_b] : -1;
        printf("D %d %d %lld %d %d %d %d %d\n", crank, tid, tb2 - tb0, p_valid ? 1 : 0, db,
               u_w >= 0 && u_w < nid_b ? 1 : 0, du, wk_max >= 0 ? 1 : 0);
      }
#endif
    }
    const long long tb3 = clock64();
#endif
    // the first event: smallest rank, and its signal, in one cluster reduction
    const long long kmin = cl_min_ll(evkey, s_ll32, s_ctal, parity);
    const bool has_ev = kmin != 0x7fffffffffffffffLL;
    const int rstar = has_ev ? (int)(kmin >> 32) : nproc;
    const int jstar = has_ev ? (int)(kmin & 0xffffffffLL) : wend;
    if (lead) { const long long t_ = clock64(); acc[2] += t_ - t_ph; t_ph = t_; }
#if GS_PROF_B
    if (lead) {
      acc[10] += c->prof_bmax[0];
      acc[11] += clock64() - tb3;  // the reduction (block + cluster barrier)
      c->prof_bmax[0] = 0u;
    }
#endif
    // ---- C1: claims, last_active (+ order stamps), patience/threshold and
    //      the edge ages each committed signal owns (the later toucher of an
    //      edge replays it), stored from the values B computed
    const bool com = p_valid && p_rank >= rbase && p_rank < rstar;
    int cb_com = -1;
    if (com) {
      {
        const int w = s_c1s[tid];
        c1_ring = w & 3;
        c1_hblow = (w & 4) != 0;
        c1_far = (w & 8) != 0;
        c1_d = (w >> 4) & 63;
        c1_patb = w >> 10;
      }
#pragma unroll
      for (int k = 0; k < kStage; ++k) {
        c1_nb0[k] = s_c1nb[k][tid];
        c1_nb1[k] = s_c1nb[kStage + k][tid];
        c1_a0[k] = s_c1a[k][tid];
        c1_a1[k] = s_c1a[kStage + k][tid];
        c1_j0[k] = s_c1j[k][tid];
        c1_j1[k] = s_c1j[kStage + k][tid];
      }
      const int cj = p_j;
      const int cb = p_b;
      cb_com = cb;
      const long long ctick = tick0 + p_rank + 1;
      const int absent = p_abs;
      S.claim[cb] = batch_no;
      if (absent & 1) atomicMin(&S.la_stamp[cb], 3 * ctick);
      if (absent & 2) atomicMin(&S.la_stamp[p_s], 3 * ctick + 1);
      atomicMax(&S.la_val[cb], ctick);
      atomicMax(&S.la_val[p_s], ctick);
      const int c1_pat = adapt_outcome_ttr(S, P, cj, c1_hblow, c1_ring, c1_patb, c1_d, c1_nb0,
                                           c1_nb1, min(nid_b, nwalked), c1_far);
      if (c1_pat != -2) {
        S.patience[cb] = c1_pat & 0x3fffffff;
        if (c1_pat >> 30) S.theta[cb] = dmul(S.theta[cb], P.rho);
      }
#pragma unroll
      for (int k = 0; k < kStage; ++k) {
        // v's own committed signal (later than cj) replays the edge instead
        if (k < c1_d && !(c1_j0[k] < jstar && c1_j0[k] > cj)) S.eage[c1_nb0[k].y] = c1_a0[k];
        if (kStage + k < c1_d && !(c1_j1[k] < jstar && c1_j1[k] > cj))
          S.eage[c1_nb1[k].y] = c1_a1[k];
      }
    }
    // ---- walk: each touched unit's position / habituation sequence in
    //      batch order; the precomputed replay holds unless it used a signal
    //      at or after the event (then this slot is replayed again)
    const bool fast = !has_ev && nid_b <= nwalked;
    if (wk_max >= 0) {
      if (wk_max < jstar) walk_store(S, P, u_w, s_wk[tid], s_wkh[tid].x, s_wkh[tid].y);
      else walk_unit(S, P, sig, u_w, jstar);
    }
    for (int u = nwalked + g; u < nid_b; u += kWinC) walk_unit(S, P, sig, u, jstar);
    const int deaths0 = c->deaths;  // stable until the event path
    if (fast) {
      // nothing reads firstwin after B here: clear the committed winners' now
      if (com) S.firstwin[cb_com] = kNone32;
    } else {
      csync();  // the walks above read firstwin; clear after them
    }
    if (lead) { const long long t_ = clock64(); acc[6] += t_ - t_ph; t_ph = t_; }
    // ---- counters, sweep clock, scratch reset
    // the window closes here unless an event without deaths lets it resume
    // (decided after the event; a closing window clears every candidate's
    // firstwin, a resuming one only the committed winners')
    if (lead) {
      c->tick = tick0 + rstar;
      c->processed += rstar - rbase;
      c->windows++;
      long long ns = next_sweep;  // silent sweeps among the committed ticks
      while (ns <= tick0 + rstar) ns += kSweepEvery;
      c->next_sweep = ns;
    }
    if (!fast && com) S.firstwin[cb_com] = kNone32;
    // the event path reads neither firstwin nor the walked units' marks, and
    // its own barrier publishes these clears; only a next window that starts
    // right away needs them first
    if (rstar == nproc && wend < m) csync();
    if (lead) {
      const long long t_ = clock64();
      acc[7] += t_ - t_ph;
      t_ph = t_;
    }
    // ---- D: the event signal, exactly as update_single, on CTA 0: warp 0
    //      runs the topology work lane-parallel, CTA 0's warps reclassify the
    //      deferred rings, the lead thread finishes (sweep, adapt_threshold);
    //      one cluster barrier publishes the result (two more only when a
    //      sweep must scan for stale units)
    if (rstar < nproc) {
      const long long t_ser = clock64();
      if (crank == 0) {
        if (tid == 0) s_defer_n = 0;
        __syncthreads();
        if (warp == 0) {
          // the event's counter traffic (tick, free-edge stack, unit / edge /
          // ring counts, isolated list length...) runs on a shared-memory copy
          // of the counters: warp 0 is the only user until the copy-back
          constexpr int kCntWords = (int)(sizeof(Counters) / sizeof(int));
          {
            const int* src = reinterpret_cast<const int*>(c);
            int* dst = reinterpret_cast<int*>(&s_cnt);
            for (int q = lane; q < kCntWords; q += 32) dst[q] = src[q];
          }
          __syncwarp();
          Counters* cc = &s_cnt;
          DevState SD = S;
          SD.defer_n = &s_defer_n;
          SD.defer_sm = s_defer_sm;
          SD.cnt = cc;
          const WinRec r = rec[jstar];
          const double x = sig[3 * (size_t)jstar], y = sig[3 * (size_t)jstar + 1],
                       z = sig[3 * (size_t)jstar + 2];
          if (lane == 0) {
            S.claim[r.b] = batch_no;
            S.firstwin[r.b] = kNone32;  // committed: later segments must not replay it
            cc->processed++;
            cc->events++;
            cc->stale_n = 0;
          }
#if GS_PROF_EV
          __syncwarp();
          const long long te0 = clock64() + (r.b & 0) + (long long)(x * 0.0);
          if (lead) acc[3] += te0 - t_ser;  // counters in + record / signal
#endif
          // the winner's and the second's rows (one load level) decide the path
          int rdb, rds;
          const int2 reb = row_lane(S, r.b, rdb);
          const int2 res = row_lane(S, r.s, rds);
          double thb = 0.0, hb = 0.0;
          double4 pb = make_double4(0.0, 0.0, 0.0, 0.0);
          if (rdb < 32 && rds < 32) {
            w_event_first(SD, P, r.b, r.s, x, y, z, rdb, reb, rds, res, s_over, &s_i[3], s_stage,
                          thb, hb, pb);
          } else {
            w_event_part1a(SD, P, r.b, r.s, s_over, &s_i[3], s_stage);
            // winner and neighbours move / decay: independent units, one lane each
            if (lane == 0) {
              pb = S.pos[r.b];
              move_toward(pb, P.eps_b, x, y, z);
              S.pos[r.b] = pb;
              const double h0 = S.hab[r.b];
              hb = dmul(h0, P.c_b);
              S.hab[r.b] = hb;
              thb = S.theta[r.b];
              if (h0 >= P.h_t && hb < P.h_t) atomicSub(&cc->untrained, 1);
            }
            int db;
            const int2 e0 = row_lane(S, r.b, db);
            const int2* B = S.adj + (size_t)r.b * kMaxDeg;
            for (int k = lane; k < db; k += 32) {
              const int v = k < 32 ? e0.x : B[k].x;
              double4 p = S.pos[v];
              move_toward(p, P.eps_n, x, y, z);
              S.pos[v] = p;
              const double h0 = S.hab[v], h = dmul(h0, P.c_n);
              S.hab[v] = h;
              if (h0 >= P.h_t && h < P.h_t) atomicSub(&cc->untrained, 1);
            }
            __syncwarp();
          }
#if GS_PROF_EV
          if (lead) acc[10] += clock64() - te0;  // touch + connect + age + moves
#endif
          thb = __shfl_sync(0xffffffffu, thb, 0);
          hb = __shfl_sync(0xffffffffu, hb, 0);
          const long long t_mid = clock64();
          const int fired = w_event_part1b(SD, P, r.b, r.s, r.dwin, x, y, z, s_over, s_i[3],
                                           s_stage, thb, hb, pb);
          if (lane == 0) {
            const long long t_end = clock64();
            acc[4] += t_mid - t_ser;  // event: connect/age + moves
            acc[5] += t_end - t_mid;  // event: insert + prune
            cc->ev_fired = fired;
            cc->ev_cutoff = fired ? sweep_cutoff(SD, P) : 0;
            cc->ev_b = r.b;
            cc->defer_n = s_defer_n;
          }
          __syncwarp();
          {
            const int* src = reinterpret_cast<const int*>(&s_cnt);
            int* dst = reinterpret_cast<int*>(c);
            for (int q = lane; q < kCntWords; q += 32) dst[q] = src[q];
          }
        }
        __syncthreads();
        const long long t_rc = clock64();
        // deferred ring reclassification, one warp per affected unit (an
        // entry repeated earlier in the list is skipped)
        const int nd = min(s_defer_n, kDeferSm + kDeferCap);
        for (int i = warp; i < nd; i += kUpdThreads / 32) {
          const int u = defer_at(S, s_defer_sm, i);
          bool dup = false;
          for (int q0 = 0; q0 < i; q0 += 32)
            dup |= q0 + lane < i && defer_at(S, s_defer_sm, q0 + lane) == u;
          if (__any_sync(0xffffffffu, dup)) continue;
          // one load level for the unit's state and row (slots past the degree
          // are ignored); the neighbours' rows are the second
          const uint8_t alive_u = S.alive[u];
          const int old = S.ring[u];
          const int ku = S.deg[u];
          const int vu = S.adj[(size_t)u * kMaxDeg + lane].x;
          if (alive_u) {
            const int nw = classify_ring_warp(S, u, s_ring_sh[warp], ku, vu);
            if (lane == 0) {
              if (nw != old) {
                S.ring[u] = (uint8_t)nw;
                atomicAdd(&c->ring_counts[old], -1);
                atomicAdd(&c->ring_counts[nw], 1);
              }
            }
          }
        }
        __syncthreads();
        if (tid == 0) acc[1] += clock64() - t_rc;  // event: ring reclassification
        if (warp == 0 && !(c->ev_fired && c->ev_cutoff > 0)) {
          const long long t_p2 = clock64();
          w_event_part2(S, P, c->ev_b, c->ev_fired != 0);
          if (lane == 0) {
            const long long t_ = clock64();
            acc[8] += t_ - t_p2;  // event: sweep clock + adapt_threshold
            acc[12] += t_ - t_ser;
          }
        }
      }
      const long long t_cs = clock64();
      csync();
      if (lead) acc[9] += clock64() - t_cs;  // event: publishing barrier
      const int fired = c->ev_fired;
      const long long cutoff = c->ev_cutoff;
      if (fired && cutoff > 0) {  // rare: the sweep collects stale units cluster-wide
        const int nid = c->next_id;
        for (int u = g; u < nid; u += kWinC) {
          const long long t = S.la_val[u];
          if (t != -1 && t < cutoff) {
            const int q = atomicAdd(&c->stale_n, 1);
            S.scratch[2 * q] = S.la_stamp[u];
            S.scratch[2 * q + 1] = u;
          }
        }
        csync();
        if (lead) {
          serial_update_part2(S, P, c->ev_b, c->stale_n, true);
          acc[12] += clock64() - t_ser;
        }
        csync();
      }
      // resume the window after an event that removed no unit
      resume = c->deaths == deaths0 && rstar + 1 < nproc;
      if (resume) {
        rbase = rstar + 1;
      } else {
        if (lead) c->discarded += (jstar + 1 - j0) - (rstar + 1);
        if (cand) S.firstwin[cb] = kNone32;
        j0 = jstar + 1;
      }
    } else {
      // no event: every candidate's winner had its first signal committed,
      // so reset (before its barrier) already cleared every firstwin entry
      // of this window -- the next window may start without another barrier
      if (lead) c->discarded += (wend - j0) - nproc;
      resume = false;
      j0 = wend;
      continue;
    }
    if (!resume) csync();  // firstwin cleared before the next window's candidates
  }
#if GS_PROF_TAIL
  const long long tt0 = clock64();
#endif
  if (start_wait) cwait();  // (no window ran: m == 0)
  if (lead) {  // the lead's phase timers (the stats thread reads them after the barrier)
#pragma unroll
    for (int q = 0; q < 12; ++q)
      if (acc[q]) atomicAdd((unsigned long long*)&c->cyc_phase[q], (unsigned long long)acc[q]);
    atomicAdd((unsigned long long*)&c->cyc_serial, (unsigned long long)acc[12]);
    atomicAdd((unsigned long long*)&c->cyc_total, (unsigned long long)(clock64() - t_kernel));
  }
  // The snapshot's row structure is stable by now: rows, their count, unit
  // liveness and next_id change only on the event path, which every window
  // ended with a cluster barrier after; the other slot's snapshot is the
  // previous launch's.  Their loads go between the barrier's arrive and its
  // wait (they overlap it), so only the positions (the walks' stores) and
  // last_active (C1's) are loaded after it.
  carrive_release();
  const int sn_n = c->nrows;
  const int sn_nid = c->next_id;
  const int sn_gen = c->row_gen;
  const int sn_dead = c->ndead_rows;
  const bool same_rows = c->snap_gen[S.snap ^ 1] == sn_gen && c->rowpos_n[S.snap ^ 1] == sn_n;
  const unsigned sn_disp = c->snap_disp[S.snap ^ 1];
  const int sn_u00 = sn_n > 0 ? S.rows[0] : -1;
  const bool sn_al0 = sn_u00 >= 0 && S.alive[sn_u00];
  int sn_u[2] = {-1, -1};  // this thread's first pair of rows: units (-1: dead / none) ...
  double sn_pv[2][3];      // ... and their previous snapshot positions
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = 2 * g + h;
    sn_pv[h][0] = sn_pv[h][1] = sn_pv[h][2] = 0.0;
    if (r < sn_n) {
      const int u = S.rows[r];
      sn_u[h] = S.alive[u] ? u : -1;
      if (same_rows) {
        sn_pv[h][0] = S.rowpos_prev[r];
        sn_pv[h][1] = S.rowpos_prev[(size_t)S.U + r];
        sn_pv[h][2] = S.rowpos_prev[2 * (size_t)S.U + r];
      }
    }
  }
  cwait();  // the last window's walk stores are visible to the snapshot below
#ifdef GS_PROF_TL
  if (tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&g_tlu2[batch_no & 8191][0], t);
  }
#endif
  // unit g's last_active / liveness for the next batch's silent-sweep value,
  // loaded with the snapshot's loads (reduced after it)
  long long la_g = -1;
  bool al_g = false;
  if (g < sn_nid) {
    la_g = S.la_val[g];
    al_g = S.alive[g] != 0;
  }
  if (g == kWinC - 1) {
    // the batch's stats, on a thread without a share of the row snapshot
    // (unless the rows fill every thread): off the hand-off's path and done
    // by the time a short next find waits for this grid.  is_converged:
    // engine.py:358-365 (max(h) < h_t <=> no untrained unit)
    const int ok = c->ring_counts[kRingDisk] + (P.allow_boundary ? c->ring_counts[kRingHalf] : 0);
    c->converged = (c->n_units >= 4 && ok == c->n_units && c->untrained == 0) ? 1 : 0;
    c->batches++;
    if (c->converged && c->halt_on_converge) c->halted = 1;
    gs_batch_stats* st = S.stats;
    st->processed = c->processed;
    st->discarded = c->discarded;
    st->inserted = c->next_id - c->inserted_start;
    st->units = c->n_units;
    st->edges = c->n_edges;
    st->next_id = c->next_id;
    st->converged = c->converged;
    st->tick = c->tick;
    st->events = c->events;
    st->windows = c->windows;
    st->error = c->error;
    st->max_degree = c->max_degree;
    st->ev_create = c->ev_create;
    st->ev_insert = c->ev_insert;
    st->ev_prune = c->ev_prune;
    st->ev_sweep = c->ev_sweep;
    st->cyc_serial = c->cyc_serial;
    st->cyc_total = c->cyc_total;
    st->batches = c->batches;
    st->halted = c->halted;
    for (int q = 0; q < 12; ++q) st->cyc_phase[q] = c->cyc_phase[q];
    if (st_out != st) *st_out = *st;  // the batch's device ring slot
  }
#if GS_PROF_TAIL
  const long long tt1 = clock64();
#endif
  {
    // row-ordered positions for the next find (its staging becomes coalesced
    // copies instead of a gather through rows), and the same rows as the
    // screened find's FP32 unit pairs {-2P'x, -2P'y, -2P'z, |P'|^2} relative
    // to row 0 rounded to FP32 (dead or non-finite rows: +inf, left out of
    // the max-norm bound); every CTA takes a slice of the pairs
    const int n = sn_n;
    const size_t U = (size_t)S.U;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    if (sn_al0) {
      const double4 p0 = S.pos[sn_u00];
      if (fabs(p0.x) < 1e30 && fabs(p0.y) < 1e30 && fabs(p0.z) < 1e30) {
        cx = (double)__double2float_rn(p0.x);
        cy = (double)__double2float_rn(p0.y);
        cz = (double)__double2float_rn(p0.z);
      }
    }
    if (lead) {
      c->fcen[S.snap][0] = cx;
      c->fcen[S.snap][1] = cy;
      c->fcen[S.snap][2] = cz;
      c->snap_gen[S.snap] = sn_gen;
    }
    // the rows' displacement since the other slot's snapshot (same rows only;
    // the next find's speculative screen checks it against its bound)
    double dmax = same_rows ? 0.0 : INFINITY;
    // the next find's bound (its rule: 2 x the previous update's displacement)
    const float dspec_part = __fadd_ru(__fmul_ru(2.f, __uint_as_float(sn_disp)), 1e-30f);
    const int np64 = (((n + 1) / 2) + 63) & ~63;
    float4* A0 = S.rowf;
    float4* A1 = S.rowf + S.rowf_stride;
    float pm = 0.f;
    for (int p = g; p < np64; p += kWinC) {
      float ax[2], ay[2], az[2], w[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * p + h;
        ax[h] = ay[h] = az[h] = 0.f;
        w[h] = INFINITY;
        if (r < n) {
          const bool first = p == g;  // (rows and liveness loaded before the barrier)
          const int u = first ? sn_u[h] : (S.alive[S.rows[r]] ? S.rows[r] : -1);
          double4 q = make_double4(INFINITY, INFINITY, INFINITY, 0.0);
          if (u >= 0) q = S.pos[u];
          S.rowpos[r] = q.x;
          S.rowpos[U + r] = q.y;
          S.rowpos[2 * U + r] = q.z;
          if (same_rows) {
            const double px0 = first ? sn_pv[h][0] : S.rowpos_prev[r];
            const double py0 = first ? sn_pv[h][1] : S.rowpos_prev[U + r];
            const double pz0 = first ? sn_pv[h][2] : S.rowpos_prev[2 * U + r];
            const double dx = q.x - px0, dy = q.y - py0, dz = q.z - pz0;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 == d2) dmax = fmax(dmax, d2);  // (dead rows: inf - inf)
          }
          if (isfinite(q.x) && isfinite(q.y) && isfinite(q.z)) {
            const float px = __double2float_rn(q.x - cx), py = __double2float_rn(q.y - cy),
                        pz = __double2float_rn(q.z - cz);
            ax[h] = -2.f * px;
            ay[h] = -2.f * py;
            az[h] = -2.f * pz;
            w[h] = __double2float_rn((double)px * px + (double)py * py + (double)pz * pz);
            const float mn = fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz)));
            pm = (mn == mn) ? fmaxf(pm, mn) : INFINITY;
          }
        }
      }
      A0[sf_swz(p)] = make_float4(ax[0], ax[1], ay[0], ay[1]);  // the find's swizzle
      A1[sf_swz(p)] = make_float4(az[0], az[1], w[0], w[1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
    if ((tid & 31) == 0 && pm > 0.f) atomicMax(&c->fpm_bits[S.snap], __float_as_uint(pm));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    float db = 0.f;
    if (dmax > 0.0) db = __double2float_ru(sqrt(dmax) * (1.0 + 1e-9));  // rounded up, FP64 room
    if ((tid & 31) == 0) {
      if (db > 0.f) atomicMax(&c->snap_disp[S.snap], __float_as_uint(db));
      s_dok[tid >> 5] = db <= dspec_part;
    }
  }
#if GS_PROF_TAIL
  const long long tt2 = clock64();
#endif
  const long long mla_w = minla_part(S, g, la_g, al_g);
  __syncthreads();
  bool part_ok = true;
#pragma unroll
  for (int q = 0; q < kUpdThreads / 32; ++q) part_ok = part_ok && s_dok[q];
  if (crank != 0) {
    snapshot_arrive(S, batch_no, part_ok);
    next_minla(S, batch_no, mla_w);
    return;
  }
  if (tid == 0) c->rowpos_n[S.snap] = sn_n;
  // compact rows when dead entries exceed 1/8 (keeps id order); CTA 0 only
  if (sn_dead * 8 > sn_n) {
    if (tid == 0) c->rowpos_n[S.snap] = -1;  // the rows move: the next find gathers
    const int n = c->nrows;
    int out = 0;
    for (int base = 0; base < n; base += kUpdThreads) {
      const int r = base + tid;
      const int id = r < n ? S.rows[r] : -1;
      const int keep = (id >= 0 && S.alive[id]) ? 1 : 0;
      int tot;
      const int rk = block_excl_scan(keep, s_warp, &tot);
      if (keep) S.rows[out + rk] = id;
      out += tot;
      __syncthreads();
    }
    if (tid == 0) {
      c->nrows = out;
      c->row_gen++;
      c->ndead_rows = 0;
    }
  }
  // (a compaction moves the rows: the candidates of the other slot are void)
  snapshot_arrive(S, batch_no, part_ok && c->rowpos_n[S.snap] >= 0);
  next_minla(S, batch_no, mla_w);
#if GS_PROF_TAIL
  if (tid == 0) {  // (reach the stats one batch late)
    const long long tt3 = clock64();
    atomicAdd((unsigned long long*)&c->cyc_phase[3], (unsigned long long)(tt1 - tt0));
    atomicAdd((unsigned long long*)&c->cyc_phase[10], (unsigned long long)(tt2 - tt1));
    atomicAdd((unsigned long long*)&c->cyc_phase[11], (unsigned long long)(tt3 - tt2));
  }
#endif
#ifdef GS_PROF_TL
  if (tid == 0) {
    unsigned long long tl2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl2));
    unsigned long long* gt = g_tlu[batch_no & 8191];
    gt[0] = tl0;
    gt[1] = tl1;
    gt[2] = tl2;
  }
#endif
}
