/*
 * growsurf_oracle.c -- CPU restatement of the reference's multi-signal hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product in paper_1503_08294_b200/: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls it (and fails loudly when its own CUDA library is
 * missing).
 *
 * It restates, in plain C with IEEE binary64 and no FP contraction
 * (compile with -ffp-contract=off), the reference package `growsurf`:
 *   - scan_best_two_into / best_two_single  pkg/src/growsurf/kernels/_scan.pyx:14-98
 *   - Network mutation + ring bookkeeping   pkg/src/growsurf/network.py:208-480
 *   - update_single and its helpers         pkg/src/growsurf/engine.py:184-355
 *   - resolve_and_update (winner lock)      pkg/src/growsurf/multi.py:99-131
 *   - is_converged                          pkg/src/growsurf/engine.py:358-365
 * The per-batch driver (sampling, batch_size) stays in Python
 * (oracle/oracle.py) so both paths consume the same numpy signal stream.
 *
 * Pinned against the reference itself: tests/golden/*.npz were produced by
 * running the reference (tests/golden/make_golden.py) and tests/test_oracle.py
 * checks this file reproduces them bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RING_DISK 0
#define RING_HALF 1
#define RING_INCONSISTENT 2

typedef struct {
  double eps_b, eps_n, theta0;
  int64_t max_age;
  double tau_b, tau_n, h_t, rho;
  int64_t ring_patience;
  int32_t allow_boundary;
  int32_t pad_;
  int64_t stale_factor;
} go_params;

typedef struct {
  int64_t nbr;
  int64_t age;
} adj_entry;

typedef struct {
  adj_entry *e;
  int32_t n, cap;
} adj_list;

typedef struct {
  go_params p;
  double c_b, c_n; /* fl(1 - tau_b), fl(1 - tau_n): engine.py:321,329 */
  /* id-indexed unit state (ids are never reused: network.py:10) */
  int64_t cap;
  double *pos; /* 3 per id */
  double *hab, *theta;
  uint8_t *alive, *ring;
  adj_list *adj;
  int64_t *patience;               /* absent == 0 (dict.get(w, 0)) */
  int64_t *la_val, *la_stamp;      /* last_active value + dict insertion order */
  uint8_t *la_present;
  /* rows: alive ids in increasing order (network.py:47-53, 464-480) */
  int64_t *rows;
  int64_t n_units, next_id, n_edges, isolated;
  int64_t ring_counts[3];
  /* over-age registry (network.py:242-256), kept as a small unsorted list */
  int64_t *over_a, *over_b;
  int64_t n_over, cap_over;
  /* RunState (engine.py:101-119) */
  int64_t tick, next_sweep, la_seq;
  /* per-batch claim marks (multi.py:114-130) */
  int64_t *claim_mark;
  int64_t batch_no;
  /* scratch */
  int64_t *scratch;
  int64_t scratch_cap;
  int32_t error;
} go_net;

#define SWEEP_EVERY 1024 /* engine.py:98 */

/* ------------------------------------------------------------------ */
/* find winners: _scan.pyx:39-98 (single-signal variant :14-36)         */

void go_scan_best_two(const double *pos, int64_t n, const double *sig, int64_t m,
                      int64_t *out_idx, double *out_d2) {
  for (int64_t j = 0; j < m; ++j) {
    const double x = sig[3 * j], y = sig[3 * j + 1], z = sig[3 * j + 2];
    int64_t i1 = -1, i2 = -1;
    double d1 = INFINITY, d2 = INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      const double dx = pos[3 * i] - x;
      const double dy = pos[3 * i + 1] - y;
      const double dz = pos[3 * i + 2] - z;
      const double d = dx * dx + dy * dy + dz * dz; /* ((dx*dx+dy*dy)+dz*dz) */
      if (d < d1) {
        d2 = d1; i2 = i1; d1 = d; i1 = i;
      } else if (d < d2) {
        d2 = d; i2 = i;
      }
    }
    out_idx[2 * j] = i1;
    out_idx[2 * j + 1] = i2;
    out_d2[2 * j] = d1;
    out_d2[2 * j + 1] = d2;
  }
}

/* ------------------------------------------------------------------ */
/* network storage                                                     */

static void grow(go_net *g, int64_t need) {
  if (need <= g->cap) return;
  int64_t nc = g->cap ? g->cap : 64;
  while (nc < need) nc *= 2;
#define RE(ptr, T, k)                                                    \
  do {                                                                   \
    g->ptr = (T *)realloc(g->ptr, sizeof(T) * (size_t)(k) * (size_t)nc); \
    memset(g->ptr + (size_t)(k) * (size_t)g->cap, 0,                     \
           sizeof(T) * (size_t)(k) * (size_t)(nc - g->cap));             \
  } while (0)
  RE(pos, double, 3);
  RE(hab, double, 1);
  RE(theta, double, 1);
  RE(alive, uint8_t, 1);
  RE(ring, uint8_t, 1);
  RE(adj, adj_list, 1);
  RE(patience, int64_t, 1);
  RE(la_val, int64_t, 1);
  RE(la_stamp, int64_t, 1);
  RE(la_present, uint8_t, 1);
  RE(rows, int64_t, 1);
  RE(claim_mark, int64_t, 1);
#undef RE
  for (int64_t i = g->cap; i < nc; ++i) g->claim_mark[i] = -1;
  g->cap = nc;
}

go_net *go_new(const go_params *p) {
  go_net *g = (go_net *)calloc(1, sizeof(go_net));
  g->p = *p;
  g->c_b = 1.0 - p->tau_b;
  g->c_n = 1.0 - p->tau_n;
  g->next_sweep = SWEEP_EVERY;
  g->batch_no = 0;
  grow(g, 64);
  return g;
}

void go_free(go_net *g) {
  if (!g) return;
  for (int64_t i = 0; i < g->next_id; ++i) free(g->adj[i].e);
  free(g->pos); free(g->hab); free(g->theta); free(g->alive); free(g->ring);
  free(g->adj); free(g->patience); free(g->la_val); free(g->la_stamp);
  free(g->la_present); free(g->rows); free(g->claim_mark);
  free(g->over_a); free(g->over_b); free(g->scratch);
  free(g);
}

static int64_t *scratch(go_net *g, int64_t n) {
  if (n > g->scratch_cap) {
    g->scratch_cap = n * 2 + 16;
    g->scratch = (int64_t *)realloc(g->scratch, sizeof(int64_t) * (size_t)g->scratch_cap);
  }
  return g->scratch;
}

static int find_nbr(const adj_list *l, int64_t v) {
  for (int32_t k = 0; k < l->n; ++k)
    if (l->e[k].nbr == v) return k;
  return -1;
}

static void adj_push(adj_list *l, int64_t v, int64_t age) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 8;
    l->e = (adj_entry *)realloc(l->e, sizeof(adj_entry) * (size_t)l->cap);
  }
  l->e[l->n].nbr = v;
  l->e[l->n].age = age;
  l->n++;
}

static void adj_del(adj_list *l, int64_t v) {
  int k = find_nbr(l, v);
  if (k < 0) return;
  l->e[k] = l->e[l->n - 1]; /* neighbour order is never observable */
  l->n--;
}

static int has_edge(const go_net *g, int64_t a, int64_t b) {
  return find_nbr(&g->adj[a], b) >= 0;
}

/* over-age registry helpers: network.py:258-259, 268-269, 315-316, 454-455 */
static void over_add(go_net *g, int64_t a, int64_t b) {
  if (a > b) { int64_t t = a; a = b; b = t; }
  for (int64_t i = 0; i < g->n_over; ++i)
    if (g->over_a[i] == a && g->over_b[i] == b) return;
  if (g->n_over == g->cap_over) {
    g->cap_over = g->cap_over ? 2 * g->cap_over : 16;
    g->over_a = (int64_t *)realloc(g->over_a, sizeof(int64_t) * (size_t)g->cap_over);
    g->over_b = (int64_t *)realloc(g->over_b, sizeof(int64_t) * (size_t)g->cap_over);
  }
  g->over_a[g->n_over] = a;
  g->over_b[g->n_over] = b;
  g->n_over++;
}

static void over_discard(go_net *g, int64_t a, int64_t b) {
  if (a > b) { int64_t t = a; a = b; b = t; }
  for (int64_t i = 0; i < g->n_over; ++i)
    if (g->over_a[i] == a && g->over_b[i] == b) {
      g->over_a[i] = g->over_a[g->n_over - 1];
      g->over_b[i] = g->over_b[g->n_over - 1];
      g->n_over--;
      return;
    }
}

/* _classify_ring: network.py:379-414 */
static int classify_ring(const go_net *g, int64_t u) {
  const adj_list *nu = &g->adj[u];
  const int32_t k = nu->n;
  if (k < 2) return RING_INCONSISTENT;
  int deg1 = 0, deg2 = 0;
  for (int32_t a = 0; a < k; ++a) {
    const int64_t v = nu->e[a].nbr;
    const adj_list *nv = &g->adj[v];
    int d = 0;
    for (int32_t c = 0; c < nv->n; ++c) {
      if (find_nbr(nu, nv->e[c].nbr) >= 0) {
        if (++d > 2) return RING_INCONSISTENT;
      }
    }
    if (d == 1) deg1++;
    else if (d == 2) deg2++;
    else return RING_INCONSISTENT;
  }
  int shape;
  if (deg1 == 0 && deg2 == k && k >= 3) shape = RING_DISK;
  else if (deg1 == 2 && deg1 + deg2 == k) shape = RING_HALF;
  else return RING_INCONSISTENT;
  /* connectivity of the induced subgraph (any start vertex) */
  int64_t *seen = (int64_t *)calloc((size_t)k, sizeof(int64_t));
  int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  int32_t top = 0, nseen = 1;
  stack[top++] = 0;
  seen[0] = 1;
  while (top) {
    const int32_t ia = (int32_t)stack[--top];
    const adj_list *nv = &g->adj[nu->e[ia].nbr];
    for (int32_t c = 0; c < nv->n; ++c) {
      const int kk = find_nbr(nu, nv->e[c].nbr);
      if (kk >= 0 && !seen[kk]) {
        seen[kk] = 1;
        nseen++;
        stack[top++] = kk;
      }
    }
  }
  free(seen);
  free(stack);
  return nseen == k ? shape : RING_INCONSISTENT;
}

/* _recompute_ring: network.py:416-422 */
static void recompute_ring(go_net *g, int64_t u) {
  const int nw = classify_ring(g, u);
  const int old = g->ring[u];
  if (nw != old) {
    g->ring[u] = (uint8_t)nw;
    g->ring_counts[old]--;
    g->ring_counts[nw]++;
  }
}

/* _ring_neighborhood: network.py:424-433.  Writes {a,b} U (N(a) & N(b)). */
static int64_t ring_neighborhood(const go_net *g, int64_t a, int64_t b, int64_t *out) {
  int64_t n = 0;
  const adj_list *na = &g->adj[a];
  for (int32_t k = 0; k < na->n; ++k) {
    const int64_t v = na->e[k].nbr;
    if (v != b && find_nbr(&g->adj[b], v) >= 0) out[n++] = v;
  }
  out[n++] = a;
  out[n++] = b;
  return n;
}

/* add_unit: network.py:208-230 */
int64_t go_add_unit(go_net *g, double x, double y, double z, double threshold) {
  if (!(isfinite(x) && isfinite(y) && isfinite(z))) return -1;
  if (!(isfinite(threshold) && threshold > 0.0)) return -1;
  const int64_t uid = g->next_id++;
  grow(g, g->next_id);
  g->pos[3 * uid] = x;
  g->pos[3 * uid + 1] = y;
  g->pos[3 * uid + 2] = z;
  g->hab[uid] = 1.0;
  g->theta[uid] = threshold;
  g->alive[uid] = 1;
  g->ring[uid] = RING_INCONSISTENT;
  g->ring_counts[RING_INCONSISTENT]++;
  g->adj[uid].n = 0;
  g->rows[g->n_units++] = uid;
  g->isolated++;
  return uid;
}

/* _remove_edge_raw: network.py:453-462 */
static void remove_edge_raw(go_net *g, int64_t a, int64_t b) {
  const int k = find_nbr(&g->adj[a], b);
  if (g->adj[a].e[k].age > g->p.max_age) over_discard(g, a, b);
  adj_del(&g->adj[a], b);
  adj_del(&g->adj[b], a);
  g->n_edges--;
  if (g->adj[a].n == 0) g->isolated++;
  if (g->adj[b].n == 0) g->isolated++;
}

/* _remove_unit_raw: network.py:464-480 (rows stay id-sorted) */
static void remove_unit_raw(go_net *g, int64_t u) {
  int64_t r = 0;
  while (g->rows[r] != u) ++r;
  memmove(g->rows + r, g->rows + r + 1, sizeof(int64_t) * (size_t)(g->n_units - r - 1));
  g->n_units--;
  g->alive[u] = 0;
  g->ring_counts[g->ring[u]]--;
  g->isolated--;
}

/* remove_unit: network.py:232-240 */
static void remove_unit(go_net *g, int64_t u) {
  const int32_t k = g->adj[u].n;
  int64_t *aff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k + 1));
  for (int32_t i = 0; i < k; ++i) aff[i] = g->adj[u].e[i].nbr;
  for (int32_t i = 0; i < k; ++i) remove_edge_raw(g, u, aff[i]);
  remove_unit_raw(g, u);
  for (int32_t i = 0; i < k; ++i) recompute_ring(g, aff[i]);
  free(aff);
}

/* connect_or_reset: network.py:261-282.  Returns 1 when created. */
static int connect_or_reset(go_net *g, int64_t a, int64_t b) {
  const int k = find_nbr(&g->adj[a], b);
  if (k >= 0) {
    if (g->adj[a].e[k].age > g->p.max_age) over_discard(g, a, b);
    g->adj[a].e[k].age = 0;
    g->adj[b].e[find_nbr(&g->adj[b], a)].age = 0;
    return 0;
  }
  if (g->adj[a].n == 0) g->isolated--;
  if (g->adj[b].n == 0) g->isolated--;
  adj_push(&g->adj[a], b, 0);
  adj_push(&g->adj[b], a, 0);
  g->n_edges++;
  int64_t *aff = scratch(g, g->adj[a].n + 2);
  const int64_t na = ring_neighborhood(g, a, b, aff);
  for (int64_t i = 0; i < na; ++i) recompute_ring(g, aff[i]);
  return 1;
}

/* remove_edge: network.py:284-292 */
static void remove_edge(go_net *g, int64_t a, int64_t b) {
  int64_t *aff = scratch(g, g->adj[a].n + 2);
  const int64_t na = ring_neighborhood(g, a, b, aff);
  int64_t *copy = (int64_t *)malloc(sizeof(int64_t) * (size_t)na);
  memcpy(copy, aff, sizeof(int64_t) * (size_t)na);
  remove_edge_raw(g, a, b);
  for (int64_t i = 0; i < na; ++i) recompute_ring(g, copy[i]);
  free(copy);
}

/* age_incident_edges(b, 1, exclude): network.py:294-319 */
static void age_incident_edges(go_net *g, int64_t b, int64_t exclude) {
  adj_list *nb = &g->adj[b];
  for (int32_t k = 0; k < nb->n; ++k) {
    const int64_t v = nb->e[k].nbr;
    if (v == exclude) continue;
    const int64_t age = nb->e[k].age;
    const int64_t nw = age + 1;
    nb->e[k].age = nw;
    g->adj[v].e[find_nbr(&g->adj[v], b)].age = nw;
    if (nw > g->p.max_age && age <= g->p.max_age) over_add(g, b, v);
  }
}

static int cmp_pair(const void *x, const void *y) {
  const int64_t *a = (const int64_t *)x, *b = (const int64_t *)y;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
  return 0;
}

/* prune(max_age) on the watched limit: network.py:321-369.
 * Returns pruned_edges in out[0], units_removed in out[1]. */
static void prune(go_net *g, int64_t out[2]) {
  out[0] = out[1] = 0;
  if (g->n_over == 0 && g->isolated == 0) return;
  const int64_t no = g->n_over;
  int64_t *ov = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * no + 2));
  for (int64_t i = 0; i < no; ++i) {
    ov[2 * i] = g->over_a[i];
    ov[2 * i + 1] = g->over_b[i];
  }
  qsort(ov, (size_t)no, 2 * sizeof(int64_t), cmp_pair);
  /* affected set as a growable list (duplicates harmless: recompute is idempotent) */
  int64_t acap = 64, an = 0;
  int64_t *aff = (int64_t *)malloc(sizeof(int64_t) * (size_t)acap);
  for (int64_t i = 0; i < no; ++i) {
    const int64_t a = ov[2 * i], b = ov[2 * i + 1];
    const int64_t need = an + g->adj[a].n + 2;
    if (need > acap) {
      while (acap < need) acap *= 2;
      aff = (int64_t *)realloc(aff, sizeof(int64_t) * (size_t)acap);
    }
    an += ring_neighborhood(g, a, b, aff + an);
    remove_edge_raw(g, a, b);
  }
  int64_t removed = 0;
  if (g->isolated) {
    int64_t nl = 0;
    int64_t *lonely = (int64_t *)malloc(sizeof(int64_t) * (size_t)(g->n_units + 1));
    for (int64_t r = 0; r < g->n_units; ++r)
      if (g->adj[g->rows[r]].n == 0) lonely[nl++] = g->rows[r]; /* rows are id-sorted */
    for (int64_t i = 0; i < nl; ++i) {
      if (g->n_units <= 2) break;
      remove_unit_raw(g, lonely[i]);
      removed++;
    }
    free(lonely);
  }
  for (int64_t i = 0; i < an; ++i)
    if (g->alive[aff[i]]) recompute_ring(g, aff[i]);
  free(aff);
  free(ov);
  out[0] = no;
  out[1] = removed;
}

/* last_active[u] = t with dict insertion-order bookkeeping (engine.py:305-306,339) */
static void touch_active(go_net *g, int64_t u, int64_t t) {
  if (!g->la_present[u]) {
    g->la_present[u] = 1;
    g->la_stamp[u] = g->la_seq++;
  }
  g->la_val[u] = t;
}

typedef struct {
  int64_t stamp, id;
} stale_rec;

static int cmp_stale(const void *x, const void *y) {
  const stale_rec *a = (const stale_rec *)x, *b = (const stale_rec *)y;
  return a->stamp < b->stamp ? -1 : (a->stamp > b->stamp);
}

/* _sweep_stale: engine.py:268-280 (dict iteration order == insertion order) */
static void sweep_stale(go_net *g) {
  const int64_t horizon = g->p.stale_factor * (g->n_units > 100 ? g->n_units : 100);
  const int64_t cutoff = g->tick - horizon;
  if (cutoff <= 0) return;
  int64_t ns = 0;
  stale_rec *st = (stale_rec *)malloc(sizeof(stale_rec) * (size_t)(g->next_id + 1));
  for (int64_t u = 0; u < g->next_id; ++u)
    if (g->la_present[u] && g->la_val[u] < cutoff) {
      st[ns].stamp = g->la_stamp[u];
      st[ns].id = u;
      ns++;
    }
  qsort(st, (size_t)ns, sizeof(stale_rec), cmp_stale);
  for (int64_t i = 0; i < ns; ++i) {
    const int64_t u = st[i].id;
    g->la_present[u] = 0;
    g->patience[u] = 0;
    if (g->alive[u] && g->n_units > 2) remove_unit(g, u);
  }
  free(st);
}

/* adapt_threshold: engine.py:208-238 (== _adapt_threshold_fast :241-265) */
static void adapt_threshold(go_net *g, int64_t b) {
  const int ring = g->ring[b];
  if (ring == RING_DISK || (g->p.allow_boundary && ring == RING_HALF)) {
    g->patience[b] = 0;
    return;
  }
  if (g->hab[b] >= g->p.h_t) return;
  const adj_list *nb = &g->adj[b];
  for (int32_t k = 0; k < nb->n; ++k)
    if (g->hab[nb->e[k].nbr] >= g->p.h_t) return;
  int64_t count = g->patience[b] + 1;
  if (count >= g->p.ring_patience) {
    g->theta[b] = g->theta[b] * g->p.rho;
    count = 0;
  }
  g->patience[b] = count;
}

/* update_single: engine.py:283-355.  Returns 1 when a unit was inserted,
 * -1 on a stale winner result (StateError in the reference). */
int go_update_single(go_net *g, const double *xi, int64_t b, int64_t s, double d_winner) {
  if (b < 0 || s < 0 || b >= g->next_id || s >= g->next_id || !g->alive[b] || !g->alive[s])
    return -1;
  const int64_t tick = ++g->tick;
  touch_active(g, b, tick);
  touch_active(g, s, tick);
  connect_or_reset(g, b, s);
  age_incident_edges(g, b, s);
  double *wp = g->pos + 3 * b;
  const double eps_b = g->p.eps_b, eps_n = g->p.eps_n;
  wp[0] = wp[0] + eps_b * (xi[0] - wp[0]);
  wp[1] = wp[1] + eps_b * (xi[1] - wp[1]);
  wp[2] = wp[2] + eps_b * (xi[2] - wp[2]);
  g->hab[b] = g->hab[b] * g->c_b;
  const adj_list *nb = &g->adj[b];
  for (int32_t k = 0; k < nb->n; ++k) {
    const int64_t v = nb->e[k].nbr;
    double *pv = g->pos + 3 * v;
    pv[0] = pv[0] + eps_n * (xi[0] - pv[0]);
    pv[1] = pv[1] + eps_n * (xi[1] - pv[1]);
    pv[2] = pv[2] + eps_n * (xi[2] - pv[2]);
    g->hab[v] = g->hab[v] * g->c_n;
  }
  int inserted = 0;
  /* maybe_insert: engine.py:184-205, gated at engine.py:336 */
  if (d_winner > g->theta[b] && g->hab[b] < g->p.h_t) {
    const double theta_b = g->theta[b];
    const double mx = (wp[0] + xi[0]) * 0.5;
    const double my = (wp[1] + xi[1]) * 0.5;
    const double mz = (wp[2] + xi[2]) * 0.5;
    const int64_t r = go_add_unit(g, mx, my, mz, theta_b);
    if (r < 0) {
      g->error = 1;
      return -2;
    }
    connect_or_reset(g, r, b);
    connect_or_reset(g, r, s);
    if (has_edge(g, b, s)) remove_edge(g, b, s);
    touch_active(g, r, tick);
    inserted = 1;
  }
  int64_t pr[2];
  prune(g, pr);
  if (tick >= g->next_sweep) {
    sweep_stale(g);
    g->next_sweep = tick + SWEEP_EVERY;
  }
  if (g->alive[b]) adapt_threshold(g, b);
  return inserted;
}

/* resolve_and_update: multi.py:99-131.  winners: (m) b, s ids and d_winner.
 * out[0..2] = processed, discarded, inserted_units. */
int go_resolve_and_update(go_net *g, const double *batch, int64_t m, const int64_t *win_b,
                          const int64_t *win_s, const double *d_win, int64_t out[3]) {
  const int64_t created_before = g->next_id;
  const int64_t mark = g->batch_no++;
  int64_t processed = 0, discarded = 0;
  for (int64_t j = 0; j < m; ++j) {
    const int64_t w = win_b[j], s = win_s[j];
    if (w >= 0 && w < g->next_id && g->claim_mark[w] == mark) {
      discarded++;
      continue;
    }
    if (!(w >= 0 && w < g->next_id && g->alive[w] && s >= 0 && s < g->next_id && g->alive[s])) {
      discarded++;
      continue;
    }
    g->claim_mark[w] = mark;
    if (go_update_single(g, batch + 3 * j, w, s, d_win[j]) < -1) return -2;
    processed++;
  }
  out[0] = processed;
  out[1] = discarded;
  out[2] = g->next_id - created_before;
  return 0;
}

/* snapshot (network.py:191-203): ids and id-ordered positions of live units */
int64_t go_snapshot(const go_net *g, int64_t *ids, double *pos) {
  for (int64_t r = 0; r < g->n_units; ++r) {
    const int64_t u = g->rows[r];
    if (ids) ids[r] = u;
    if (pos) {
      pos[3 * r] = g->pos[3 * u];
      pos[3 * r + 1] = g->pos[3 * u + 1];
      pos[3 * r + 2] = g->pos[3 * u + 2];
    }
  }
  return g->n_units;
}

/* One multi-signal batch: snapshot -> exhaustive find (sequential_executor,
 * multi.py:58-96) -> resolve_and_update.  out as go_resolve_and_update.
 * Optionally returns the winners (ids + squared distances) for tracing. */
int go_step(go_net *g, const double *batch, int64_t m, int64_t out[3], int64_t *w_ids,
            double *w_d2) {
  const int64_t n = g->n_units;
  if (n < 2) return -1; /* StateError: multi.py:60-61 */
  double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)n);
  int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  go_snapshot(g, ids, pos);
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)m);
  double *d2 = (double *)malloc(sizeof(double) * 2 * (size_t)m);
  go_scan_best_two(pos, n, batch, m, idx, d2);
  int64_t *wb = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
  int64_t *ws = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
  double *dw = (double *)malloc(sizeof(double) * (size_t)m);
  for (int64_t j = 0; j < m; ++j) {
    wb[j] = ids[idx[2 * j]];
    ws[j] = ids[idx[2 * j + 1]];
    dw[j] = sqrt(d2[2 * j]); /* _to_results: multi.py:72-78 */
    if (w_ids) {
      w_ids[2 * j] = wb[j];
      w_ids[2 * j + 1] = ws[j];
    }
    if (w_d2) {
      w_d2[2 * j] = d2[2 * j];
      w_d2[2 * j + 1] = d2[2 * j + 1];
    }
  }
  const int rc = go_resolve_and_update(g, batch, m, wb, ws, dw, out);
  free(pos); free(ids); free(idx); free(d2); free(wb); free(ws); free(dw);
  return rc;
}

/* is_converged: engine.py:358-365 */
int go_is_converged(const go_net *g) {
  if (g->n_units < 4) return 0;
  int64_t ok = g->ring_counts[RING_DISK];
  if (g->p.allow_boundary) ok += g->ring_counts[RING_HALF];
  if (ok != g->n_units) return 0;
  double mx = -INFINITY;
  for (int64_t r = 0; r < g->n_units; ++r)
    if (g->hab[g->rows[r]] > mx) mx = g->hab[g->rows[r]];
  return mx < g->p.h_t;
}

/* counters: V, E, next_id, tick, next_sweep, isolated, disk, half, inconsistent, n_over */
void go_counts(const go_net *g, int64_t out[10]) {
  out[0] = g->n_units;
  out[1] = g->n_edges;
  out[2] = g->next_id;
  out[3] = g->tick;
  out[4] = g->next_sweep;
  out[5] = g->isolated;
  out[6] = g->ring_counts[RING_DISK];
  out[7] = g->ring_counts[RING_HALF];
  out[8] = g->ring_counts[RING_INCONSISTENT];
  out[9] = g->n_over;
}

/* Per-live-unit export in row (id) order. */
void go_export_units(const go_net *g, int64_t *ids, double *pos, double *hab, double *theta,
                     int64_t *ring, int64_t *patience, int64_t *last_active) {
  for (int64_t r = 0; r < g->n_units; ++r) {
    const int64_t u = g->rows[r];
    ids[r] = u;
    pos[3 * r] = g->pos[3 * u];
    pos[3 * r + 1] = g->pos[3 * u + 1];
    pos[3 * r + 2] = g->pos[3 * u + 2];
    hab[r] = g->hab[u];
    theta[r] = g->theta[u];
    ring[r] = g->ring[u];
    patience[r] = g->patience[u];
    last_active[r] = g->la_present[u] ? g->la_val[u] : -1;
  }
}

/* All edges as (a, b, age) with a < b, sorted (network.py:152-161). */
int64_t go_export_edges(const go_net *g, int64_t *out) {
  int64_t n = 0;
  for (int64_t r = 0; r < g->n_units; ++r) {
    const int64_t a = g->rows[r];
    const adj_list *na = &g->adj[a];
    for (int32_t k = 0; k < na->n; ++k)
      if (a < na->e[k].nbr) {
        out[3 * n] = a;
        out[3 * n + 1] = na->e[k].nbr;
        out[3 * n + 2] = na->e[k].age;
        n++;
      }
  }
  qsort(out, (size_t)n, 3 * sizeof(int64_t), cmp_pair); /* (a,b) unique */
  return n;
}

/* Recompute every ring from scratch and compare with the cached classes
 * (the ring part of Network.audit, network.py:521-526).  Returns #mismatches. */
int64_t go_audit_rings(go_net *g) {
  int64_t bad = 0;
  for (int64_t r = 0; r < g->n_units; ++r) {
    const int64_t u = g->rows[r];
    if (classify_ring(g, u) != g->ring[u]) bad++;
  }
  return bad;
}

/* Exposed for fine-grained tests of the network primitives. */
int go_connect_or_reset(go_net *g, int64_t a, int64_t b) { return connect_or_reset(g, a, b); }
int go_classify_ring(const go_net *g, int64_t u) { return classify_ring(g, u); }
void go_set_hab(go_net *g, int64_t u, double h) { g->hab[u] = h; }
