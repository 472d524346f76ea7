// update_kernel.cuh -- the batch update kernel (included by engine.cu).
//
// Windowed segmented replay of the reference's sequential update loop
// (multi.py:120-130 -> engine.py:283-355); see the engine.cu header for the
// argument.  One CTA of 1024 threads processes windows of up to kWin
// signals:
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

constexpr int kSigPerThread = 4;
constexpr int kWin = kUpdThreads * kSigPerThread;

// replay unit u's updates from the committed signals (< jstar) of this window
__device__ void walk_unit(const DevState& S, const Params& P, const double* sig, int u,
                          int jstar) {
  const int2* A = S.adj + (size_t)u * kMaxDeg;
  const int d = S.deg[u];
  int t[kMaxDeg + 1];  // (j << 1) | self
  int n = 0;
  const int jself = S.firstwin[u];
  if (jself < jstar) t[n++] = (jself << 1) | 1;
  for (int k = 0; k < d; ++k) {
    const int jw = S.firstwin[A[k].x];
    if (jw < jstar) t[n++] = jw << 1;
  }
  for (int i = 1; i < n; ++i) {  // insertion sort: n is a handful
    const int x = t[i];
    int q = i - 1;
    while (q >= 0 && t[q] > x) {
      t[q + 1] = t[q];
      --q;
    }
    t[q + 1] = x;
  }
  double4 p = S.pos[u];
  const double h0 = S.hab[u];
  double h = h0;
  for (int i = 0; i < n; ++i) {
    const size_t j = (size_t)(t[i] >> 1);
    const double x = sig[3 * j], y = sig[3 * j + 1], z = sig[3 * j + 2];
    if (t[i] & 1) {
      move_toward(p, P.eps_b, x, y, z);
      h = dmul(h, P.c_b);
    } else {
      move_toward(p, P.eps_n, x, y, z);
      h = dmul(h, P.c_n);
    }
  }
  S.pos[u] = p;
  S.hab[u] = h;
  if (h0 >= P.h_t && h < P.h_t) atomicSub(&S.cnt->untrained, 1);
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
__device__ int classify_ring_warp(const DevState& S, int u, int* sh) {
  const int lane = threadIdx.x & 31;
  const int k = S.deg[u];
  if (k < 2) return kRingInc;
  if (k > 32) return classify_ring(S, u);
  const int2* A = S.adj + (size_t)u * kMaxDeg;
  if (lane < k) sh[lane] = A[lane].x;
  __syncwarp();
  int d = 0;
  unsigned mask = 0;
  if (lane < k) {
    const int v = sh[lane];
    const int dv = S.deg[v];
    const int2* V = S.adj + (size_t)v * kMaxDeg;
    for (int c = 0; c < dv && d <= 2; ++c) {
      const int w = V[c].x;
      for (int i = 0; i < k; ++i)
        if (sh[i] == w) {
          ++d;
          mask |= 1u << i;
          break;
        }
    }
  }
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

__global__ void __launch_bounds__(kUpdThreads, 1)
    k_update_batch(DevState S, Params P, const double* __restrict__ sig,
                   const WinRec* __restrict__ rec, int m, int batch_no) {
  __shared__ int s_warp[33];
  __shared__ long long s_ll32[33];
  __shared__ int s_plist[kWin];  // processed signals of the window, batch order
  __shared__ int s_pat[kWin];    // adapt_threshold outcome: -2 none, else patience | shrink<<30
  __shared__ int s_i[8];
  __shared__ long long s_l[4];
  __shared__ int s_over[kMaxDeg];
  __shared__ int s_ring_sh[32][33];  // per-warp N(u) staging for classify_ring_warp
  __shared__ int s_defer_n;
  Counters* c = S.cnt;
  const int tid = threadIdx.x;
  const long long t_kernel = clock64();
  if (tid == 0) {
    c->processed = c->discarded = c->events = c->windows = 0;
    c->inserted_start = c->next_id;
    c->stale_n = 0;
  }
  __syncthreads();
  int j0 = 0;
  long long t_ph = clock64();
  while (j0 < m) {
    if (tid == 0) t_ph = clock64();
    const int wend = min(j0 + kWin, m);
    const int next_id = c->next_id;
    const long long tick0 = c->tick;
    const long long next_sweep = c->next_sweep;
    const int n_units = c->n_units;
    const bool iso = c->iso_count > 0;
    // ---- A: candidates (thread owns a contiguous chunk: order-preserving compaction)
    const int cj0 = j0 + tid * kSigPerThread;
    unsigned cmask = 0;
#pragma unroll
    for (int q = 0; q < kSigPerThread; ++q) {
      const int j = cj0 + q;
      if (j < wend) {
        const WinRec r = rec[j];
        const bool cand = r.b >= 0 && r.s >= 0 && r.b < next_id && r.s < next_id && r.b != r.s &&
                          S.alive[r.b] && S.alive[r.s] && S.claim[r.b] != batch_no;
        if (cand) {
          cmask |= 1u << q;
          atomicMin(&S.firstwin[r.b], j);
        }
      }
    }
    // minimum last_active over live units (silent-sweep test), window-start state
    long long minla = 0x7fffffffffffffffLL;
    if (tick0 + kWin >= next_sweep) {
      for (int u = tid; u < next_id; u += kUpdThreads) {
        const long long t = S.la_val[u];
        if (t != -1 && S.alive[u] && t < minla) minla = t;
      }
    }
    minla = block_min_ll(minla, s_ll32);  // contains __syncthreads
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[0] += t_ - t_ph; t_ph = t_; }
    unsigned pmask = 0;
#pragma unroll
    for (int q = 0; q < kSigPerThread; ++q)
      if ((cmask >> q) & 1u) {
        const int j = cj0 + q;
        if (S.firstwin[rec[j].b] == j) pmask |= 1u << q;
      }
    int nproc;
    int rank = block_excl_scan(__popc(pmask), s_warp, &nproc);
#pragma unroll
    for (int q = 0; q < kSigPerThread; ++q)
      if ((pmask >> q) & 1u) s_plist[rank++] = cj0 + q;
    __syncthreads();
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[1] += t_ - t_ph; t_ph = t_; }
    // ---- B: events and adapt_threshold outcomes, one processed signal per thread
    // sweep schedule inside the window: fires at ticks next_sweep + 1024 k; the
    // k-th is silent iff cutoff_k <= 0 or every live unit's last_active >= cutoff_k
    const long long horizon = P.stale_factor * (long long)(n_units > 100 ? n_units : 100);
    int evr = 0x7fffffff;
    for (int r = tid; r < nproc; r += kUpdThreads) {
      const int j = s_plist[r];
      const WinRec w = rec[j];
      const int b = w.b, s = w.s;
      const long long tick_j = tick0 + r + 1;
      bool ev = iso;
      if (tick_j >= next_sweep && ((tick_j - next_sweep) % kSweepEvery) == 0) {
        const long long cutoff = tick_j - horizon;
        if (cutoff > 0 && (minla < cutoff || n_units <= 2)) ev = true;
      }
      const int db = S.deg[b];
      const int2* B = S.adj + (size_t)b * kMaxDeg;
      // habituation only decays (x c_b, x c_n < 1), so a unit trained at the
      // window start is trained at any later time: the exact per-time value is
      // reconstructed only for units still at or above h_t
      const double hbT = S.hab[b];
      const bool b_trained = hbT < P.h_t;
      bool found = false;
      int kcn = 0;
      for (int k = 0; k < db; ++k) {
        const int2 ent = B[k];
        const int v = ent.x;
        const bool is_s = v == s;
        found |= is_s;
        const int age = is_s ? 0 : S.eage[ent.y];
        const bool age_risk = !is_s && age + 2 > P.max_age;  // may exceed max_age at j
        if (!b_trained || age_risk) {
          const int jv = S.firstwin[v];
          if (jv < j) kcn++;
          if (age_risk) {
            const int a2 = jv < j ? ((rec[jv].s == b) ? 0 : age + 1) : age;
            if (a2 + 1 > P.max_age) ev = true;
          }
        }
      }
      if (!found) ev = true;  // connect_or_reset creates b-s
      const bool hb_low = b_trained || dmul(pow_chain(hbT, P.c_n, kcn), P.c_b) < P.h_t;
      if (hb_low && w.dwin > S.theta[b]) ev = true;  // maybe_insert fires
      int pat = -2;
      if (!ev) {
        const int ring = S.ring[b];
        if (ring == kRingDisk || (P.allow_boundary && ring == kRingHalf)) {
          pat = 0;
        } else if (hb_low) {
          bool ok = true;
          for (int k = 0; k < db && ok; ++k) {
            const int v = B[k].x;
            const double hvT = S.hab[v];
            if (hvT < P.h_t) continue;  // trained neighbour stays trained
            const int jv = S.firstwin[v];
            const bool vwon = jv < j;
            const int dv = S.deg[v];
            const int2* V = S.adj + (size_t)v * kMaxDeg;
            int k1 = 0, k2 = 0;
            for (int q = 0; q < dv; ++q) {
              const int jw = S.firstwin[V[q].x];
              if (jw <= j) {
                if (vwon && jw > jv) k2++;
                else k1++;
              }
            }
            double hv = pow_chain(hvT, P.c_n, k1);
            if (vwon) hv = dmul(hv, P.c_b);
            hv = pow_chain(hv, P.c_n, k2);
            if (hv >= P.h_t) ok = false;
          }
          if (ok) {
            int cnt = S.patience[b] + 1;
            const int shrink = cnt >= P.ring_patience ? 1 : 0;
            if (shrink) cnt = 0;
            pat = cnt | (shrink << 30);
          }
        }
      }
      s_pat[r] = pat;
      if (ev && r < evr) evr = r;
    }
    const int rstar = min(block_min(evr, s_warp), nproc);  // first event (rank)
    const int jstar = rstar < nproc ? s_plist[rstar] : wend;
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[2] += t_ - t_ph; t_ph = t_; }
    // ---- C: commit ranks [0, rstar)
    for (int r = tid; r < rstar; r += kUpdThreads) {
      const int j = s_plist[r];
      const WinRec w = rec[j];
      const long long tick_j = tick0 + r + 1;
      S.claim[w.b] = batch_no;
      if (S.la_val[w.b] == -1) atomicMin(&S.la_stamp[w.b], 3 * tick_j);
      if (S.la_val[w.s] == -1) atomicMin(&S.la_stamp[w.s], 3 * tick_j + 1);
      const int p = s_pat[r];
      if (p != -2) {
        S.patience[w.b] = p & 0x3fffffff;
        if (p >> 30) S.theta[w.b] = dmul(S.theta[w.b], P.rho);
      }
      atomicMin(&S.touchfirst[w.b], j);
      const int db = S.deg[w.b];
      const int2* B = S.adj + (size_t)w.b * kMaxDeg;
      for (int k = 0; k < db; ++k) atomicMin(&S.touchfirst[B[k].x], j);
    }
    if (tid == 0) s_i[0] = 0;
    __syncthreads();
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[3] += t_ - t_ph; t_ph = t_; }
    // last_active values after the stamps were taken from the window-start state
    for (int r = tid; r < rstar; r += kUpdThreads) {
      const WinRec w = rec[s_plist[r]];
      const long long tick_j = tick0 + r + 1;
      atomicMax(&S.la_val[w.b], tick_j);
      atomicMax(&S.la_val[w.s], tick_j);
    }
    // owner list of touched units + edge-age replay
    for (int r = tid; r < rstar; r += kUpdThreads) {
      const int j = s_plist[r];
      const WinRec w = rec[j];
      const int b = w.b, s = w.s;
      if (S.touchfirst[b] == j) S.scratch[atomicAdd(&s_i[0], 1)] = b;
      const int db = S.deg[b];
      const int2* B = S.adj + (size_t)b * kMaxDeg;
      for (int k = 0; k < db; ++k) {
        const int2 ent = B[k];
        const int v = ent.x;
        if (S.touchfirst[v] == j) S.scratch[atomicAdd(&s_i[0], 1)] = v;
        const int jv = S.firstwin[v];
        if (jv < jstar && jv > j) continue;  // v's own signal replays this edge
        int age = S.eage[ent.y];
        if (jv < j) age = (rec[jv].s == b) ? 0 : age + 1;
        age = (v == s) ? 0 : age + 1;
        S.eage[ent.y] = age;
      }
    }
    __syncthreads();
    const int nwalk = s_i[0];
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[4] += t_ - t_ph; t_ph = t_; }
    for (int i = tid; i < nwalk; i += kUpdThreads) walk_unit(S, P, sig, (int)S.scratch[i], jstar);
    __syncthreads();
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[6] += t_ - t_ph; t_ph = t_; }
    // ---- counters, sweep clock, scratch reset
    if (tid == 0) {
      c->tick = tick0 + rstar;
      c->processed += rstar;
      c->discarded += (jstar - j0) - rstar;
      c->windows++;
      // silent sweeps that fired among the committed ticks move the clock
      long long ns = next_sweep;
      while (ns <= tick0 + rstar) ns += kSweepEvery;
      c->next_sweep = ns;
    }
    for (int q = 0; q < kSigPerThread; ++q)
      if ((cmask >> q) & 1u) S.firstwin[rec[cj0 + q].b] = kNone32;
    for (int i = tid; i < nwalk; i += kUpdThreads) S.touchfirst[(int)S.scratch[i]] = kNone32;
    __syncthreads();
    // ---- D: the event signal, exactly as update_single
    if (tid == 0) { const long long t_ = clock64(); c->cyc_phase[7] += t_ - t_ph; t_ph = t_; }
    if (rstar < nproc) {
      const long long t_ser = clock64();
      const int warp = tid >> 5, lane = tid & 31;
      if (tid == 0) s_defer_n = 0;
      __syncthreads();
      if (warp == 0) {
        DevState SD = S;
        SD.defer_n = &s_defer_n;
        const WinRec r = rec[jstar];
        const double x = sig[3 * (size_t)jstar], y = sig[3 * (size_t)jstar + 1],
                     z = sig[3 * (size_t)jstar + 2];
        if (lane == 0) {
          S.claim[r.b] = batch_no;
          event_part1a(SD, P, r.b, r.s, s_over, &s_i[3]);
          c->processed++;
          c->events++;
          c->stale_n = 0;
        }
        __syncwarp();
        // winner and its neighbours move / decay: independent units, one lane each
        // (engine.py:316-329)
        if (lane == 0) {
          double4 p = S.pos[r.b];
          move_toward(p, P.eps_b, x, y, z);
          S.pos[r.b] = p;
          const double h0 = S.hab[r.b], h = dmul(h0, P.c_b);
          S.hab[r.b] = h;
          if (h0 >= P.h_t && h < P.h_t) atomicSub(&c->untrained, 1);
        }
        const int db = S.deg[r.b];
        const int2* B = S.adj + (size_t)r.b * kMaxDeg;
        for (int k = lane; k < db; k += 32) {
          const int v = B[k].x;
          double4 p = S.pos[v];
          move_toward(p, P.eps_n, x, y, z);
          S.pos[v] = p;
          const double h0 = S.hab[v], h = dmul(h0, P.c_n);
          S.hab[v] = h;
          if (h0 >= P.h_t && h < P.h_t) atomicSub(&c->untrained, 1);
        }
        __syncwarp();
        if (lane == 0) {
          const int fired = event_part1b(SD, P, r.b, r.s, r.dwin, x, y, z, s_over, s_i[3]);
          s_i[1] = fired;
          s_l[0] = fired ? sweep_cutoff(S, P) : 0;
          s_i[2] = r.b;
        }
      }
      __syncthreads();
      // deferred ring reclassification, one warp per affected unit
      {
        const int nd = min(s_defer_n, kDeferCap);
        for (int i = warp; i < nd; i += 32) {
          const int u = S.defer_list[i];
          if (S.alive[u]) {
            const int nw = classify_ring_warp(S, u, s_ring_sh[warp]);
            if (lane == 0) {
              const int old = S.ring[u];
              if (nw != old) {
                S.ring[u] = (uint8_t)nw;
                atomicAdd(&c->ring_counts[old], -1);
                atomicAdd(&c->ring_counts[nw], 1);
              }
            }
          }
          if (lane == 0) S.touchfirst[u] = kNone32;
        }
      }
      __syncthreads();
      const int fired = s_i[1];
      const long long cutoff = s_l[0];
      if (fired && cutoff > 0) {
        const int nid = c->next_id;
        for (int u = tid; u < nid; u += kUpdThreads) {
          const long long t = S.la_val[u];
          if (t != -1 && t < cutoff) {
            const int q = atomicAdd(&c->stale_n, 1);
            S.scratch[2 * q] = S.la_stamp[u];
            S.scratch[2 * q + 1] = u;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        serial_update_part2(S, P, s_i[2], c->stale_n, fired != 0);
        c->cyc_serial += clock64() - t_ser;
      }
      __syncthreads();
      j0 = jstar + 1;
    } else {
      j0 = wend;
    }
    __syncthreads();
  }
  // compact rows when dead entries exceed 1/8 (keeps id order)
  if (c->ndead_rows * 8 > c->nrows) {
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
      c->ndead_rows = 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    // is_converged: engine.py:358-365 (max(h) < h_t <=> no untrained unit)
    const int ok = c->ring_counts[kRingDisk] + (P.allow_boundary ? c->ring_counts[kRingHalf] : 0);
    c->converged = (c->n_units >= 4 && ok == c->n_units && c->untrained == 0) ? 1 : 0;
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
    c->cyc_total += clock64() - t_kernel;
    st->cyc_serial = c->cyc_serial;
    st->cyc_total = c->cyc_total;
    for (int q = 0; q < 8; ++q) st->cyc_phase[q] = c->cyc_phase[q];
  }
}
