/*
 * growsurf_b200.h -- C ABI of the B200-native multi-signal growing network.
 *
 * Plain C types only (no torch, no CUDA runtime types): pointers, sizes and
 * an opaque `void *stream` (a cudaStream_t, NULL = the context's own stream).
 * Every entry point returns a gs_status; gs_last_error() returns a
 * thread-local message for the last failure on the calling thread.
 *
 * Reference interfaces each group replaces (paths under the reference's
 * pkg/src/growsurf/):
 *
 *   Kernel-backend protocol (kernels/__init__.py:6-7, 26-44)
 *     gs_best_two_single      <- _scan.pyx:14-36   best_two_single
 *     gs_scan_best_two_into   <- _scan.pyx:39-98   scan_best_two_into
 *   Batched find on device data (multi.py:58-69 _scan_batch,
 *   parallel.py:63-88 _parallel_scan): gs_find_device
 *   Device-resident multi-signal engine (multi.py:99-202 resolve_and_update /
 *   run_multi, engine.py:283-365 update_single / is_converged, network.py
 *   Network accessors): gs_engine_*
 *
 * Threading: a gs_ctx owns one CUDA stream and scratch buffers and
 * serialises its own calls with an internal mutex, so the reference's
 * "disjoint output slices may be filled from parallel threads" contract
 * (_scan.pyx:49-50, parallel.py:78-87) holds.  A gs_engine is
 * single-threaded, like the reference Network (network.py:74).
 */
#ifndef GROWSURF_B200_H
#define GROWSURF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GS_OK = 0,
  GS_VALUE_ERROR = 1, /* ValueError in the reference (_scan.pyx:56-61, engine.py:71-91) */
  GS_STATE_ERROR = 2, /* StateError (network.py:30, multi.py:60-61, engine.py:299-300) */
  GS_CUDA_ERROR = 3,  /* no device, launch or copy failure */
  GS_UNKNOWN_UNIT = 4 /* UnknownUnitError (network.py:26, 438-442) */
} gs_status;

const char *gs_last_error(void);
const char *gs_version(void);

/* ------------------------------------------------------------------ */
/* context                                                              */

typedef struct gs_ctx gs_ctx;

gs_status gs_ctx_create(int device, gs_ctx **out);
void gs_ctx_destroy(gs_ctx *ctx);
/* Face-edge counts of a triangle list (metrics.py:165-240 _edge_face_counts /
 * manifold_check / _is_connected / genus, on the device): faces n_faces x 3
 * int64 (host) indexing [0, n_vertices); out[0] distinct face edges, out[1]
 * edges bordering > 2 faces, out[2] boundary edges (1 face), out[3] vertices
 * whose boundary degree is neither 0 nor 2, out[4] connected components of
 * the face-edge graph over all n_vertices vertices, out[5] 0.
 * GS_VALUE_ERROR for an index outside [0, n_vertices). */
gs_status gs_mesh_topology(gs_ctx *ctx, const int64_t *faces, int64_t n_faces, int64_t n_vertices,
                           int64_t out[6]);
/* Number of SMs of the context's device (grid sizing, roofline). */
int gs_ctx_sm_count(const gs_ctx *ctx);
/* Measured FP32 peak of the device: packed FFMA2 chains on every SM, best of
 * 5 timed launches (TFLOP/s; *ms = that launch's time, may be NULL). */
gs_status gs_fp32_peak(gs_ctx *ctx, double *tflops, double *ms);

/* ------------------------------------------------------------------ */
/* kernel-backend protocol: host buffers, synchronous                   */

/* best_two_single(pos, n, x, y, z) -> (r1, r2, d2_1, d2_2); rows are -1 and
 * distances +inf where fewer than two units exist (fallback.py:21-30).
 * pos: n_rows x 3 float64, C-contiguous; requires n <= n_rows. */
gs_status gs_best_two_single(gs_ctx *ctx, const double *pos, int64_t n_rows, int64_t n, double x,
                             double y, double z, int64_t *r1, int64_t *r2, double *d2_1,
                             double *d2_2);

/* scan_best_two_into(pos, n, signals, out_idx, out_d2, tile): for each of the
 * m signals, the ROWS of the nearest and second-nearest of the first n rows
 * of pos and their squared distances, lexicographic on (d^2, row) with
 * d^2 = ((dx*dx + dy*dy) + dz*dz) in IEEE binary64 (no contraction).
 * out_idx: out_rows x 2 int64, out_d2: out_d2_rows x 2 float64, written for
 * [0, m).  GS_VALUE_ERROR when n > n_rows, an output is shorter than m, or
 * tile < 1; tile never changes the result. */
gs_status gs_scan_best_two_into(gs_ctx *ctx, const double *pos, int64_t n_rows, int64_t n,
                                const double *signals, int64_t m, int64_t *out_idx,
                                int64_t out_rows, double *out_d2, int64_t out_d2_rows,
                                int64_t tile);

/* ------------------------------------------------------------------ */
/* batched find on device buffers (asynchronous on `stream`)            */

typedef enum {
  GS_FIND_EXACT = 0,  /* FP64 scan, the reference arithmetic */
  GS_FIND_FILTER = 1, /* FP32 top-3 filter + certified FP64 re-check (bit-identical output) */
  GS_FIND_AUTO = 2,
  GS_FIND_SMALL = 3,  /* n <= 4096: one kernel, FP32 screen + exact FP64 re-evaluation (bit-identical) */
  GS_FIND_GRID = 4    /* exact uniform grid rebuilt per call: shells until certified (bit-identical) */
} gs_find_mode;

/* d_pos: n x 3 float64 (device), d_sig: m x 3 float64 (device);
 * d_idx: m x 2 int64 rows, d_d2: m x 2 float64 (device).  Returns without
 * synchronising.  *fallbacks (optional, host) receives, after the next
 * synchronisation of `stream`, the number of signals the filter could not
 * certify and re-scanned exactly. */
gs_status gs_find_device(gs_ctx *ctx, const double *d_pos, int64_t n, const double *d_sig,
                         int64_t m, int64_t *d_idx, double *d_d2, int mode, void *stream);
/* Signals the last GS_FIND_FILTER call on this ctx could not certify and
 * re-scanned (syncs). */
gs_status gs_find_last_fallbacks(gs_ctx *ctx, int64_t *count);
/* out[0]: signals re-scanned by the FP32 direct-form tier; out[1]: of those,
 * signals that also needed the exact FP64 scan (syncs). */
gs_status gs_find_last_fallback_counts(gs_ctx *ctx, int64_t out[2]);

/* ------------------------------------------------------------------ */
/* device-resident multi-signal engine                                  */

typedef struct {
  double eps_b, eps_n, theta0;
  int64_t max_age;
  double tau_b, tau_n, h_t, rho;
  int64_t ring_patience;
  int32_t allow_boundary;
  int32_t find_mode; /* gs_find_mode */
  int64_t stale_factor;
} gs_params;

typedef struct {
  int64_t processed, discarded, inserted; /* BatchOutcome (multi.py:35-41) */
  int64_t units, edges, next_id;          /* Network.unit_count / edge_count / next_id */
  int64_t converged;                      /* is_converged after the batch (engine.py:358-365) */
  int64_t tick;                           /* RunState.tick */
  int64_t events;                         /* signals executed on the serial event path */
  int64_t windows;                        /* parallel windows used by the batch */
  int64_t error;                          /* device error code (0 = none) */
  int64_t max_degree;                     /* largest unit degree seen (capacity check) */
  int64_t ev_create, ev_insert, ev_prune, ev_sweep; /* serial-path causes (cumulative) */
  int64_t cyc_serial, cyc_total;          /* update-kernel SM cycles: serial path / all (cumulative) */
  int64_t cyc_phase[12];                  /* update-kernel SM cycles (cumulative): window phases
                                           * 0 A+scan, 2 B, 3 C1, 6 walk, 7 reset; event path
                                           * 4 connect/age+moves, 5 insert+prune, 1 ring
                                           * reclassification, 8 adapt_threshold, 9 barrier;
                                           * 10, 11 spare */
  int64_t batches;                        /* update kernels run so far (cumulative) */
  int64_t halted;                         /* 1: converged, later batches are no-ops (async runs) */
} gs_batch_stats;

typedef struct gs_engine gs_engine;

gs_status gs_engine_create(gs_ctx *ctx, const gs_params *params, int64_t capacity_hint,
                           gs_engine **out);
void gs_engine_destroy(gs_engine *eng);

/* Network.add_unit (network.py:208-230): hab 1, no edges; returns the id. */
gs_status gs_engine_add_unit(gs_engine *eng, double x, double y, double z, double threshold,
                             int64_t *id);
/* Network.connect_or_reset (network.py:261-282); *created = 1 if new. */
gs_status gs_engine_connect_or_reset(gs_engine *eng, int64_t a, int64_t b, int32_t *created);
/* Network.remove_unit (network.py:232-240). */
gs_status gs_engine_remove_unit(gs_engine *eng, int64_t id);
/* Network.remove_edge (network.py:284-292). */
gs_status gs_engine_remove_edge(gs_engine *eng, int64_t a, int64_t b);
/* Network.age_incident_edges(b, increment, exclude or -1) (network.py:294-319). */
gs_status gs_engine_age_incident_edges(gs_engine *eng, int64_t b, int64_t increment,
                                       int64_t exclude, int64_t *top);
/* Network.prune(max_age) (network.py:321-369). */
gs_status gs_engine_prune(gs_engine *eng, int64_t max_age, int64_t *pruned_edges,
                          int64_t *units_removed);
/* Overwrite one unit's habituation / position (tests set net._hab directly). */
gs_status gs_engine_set_unit(gs_engine *eng, int64_t id, const double *xyz, const double *hab,
                             const double *theta);

/* One multi-signal iteration on a HOST batch (m x 3 float64): H2D, find
 * winners against the pre-batch snapshot, winner-lock resolution, batch-order
 * update, convergence check, stats D2H.  Synchronous. */
gs_status gs_engine_step(gs_engine *eng, const double *signals, int64_t m, gs_batch_stats *out);
/* Same on a DEVICE batch; asynchronous on the engine stream.  Stats land in
 * the engine's pinned stats block; read them with gs_engine_stats. */
gs_status gs_engine_step_device(gs_engine *eng, const double *d_signals, int64_t m);
/* Find only: writes device winner records for signals [lo, hi) of a device
 * batch (a multi-GPU shard) at record index lo.., then gs_engine_update_device
 * applies the full batch's records (after an all-gather).  Records are
 * GS_WINREC_BYTES = 16 bytes per signal: int32 winner ID, int32 second ID
 * (ids, not rows: snapshot.ids[row], multi.py:72-78), float64 d_winner =
 * sqrt(d2_1) correctly rounded. */
#define GS_WINREC_BYTES 16
gs_status gs_engine_find_device(gs_engine *eng, const double *d_signals, int64_t lo, int64_t hi,
                                void *d_records);
gs_status gs_engine_update_device(gs_engine *eng, const double *d_signals, int64_t m,
                                  const void *d_records);
/* resolve_and_update with caller-supplied winners (multi.py:99-131): winner /
 * second ids and d_winner per signal (e.g. from an external executor).
 * Synchronous; out receives the batch stats. */
gs_status gs_engine_resolve_host(gs_engine *eng, const double *signals, int64_t m,
                                 const int64_t *win_b, const int64_t *win_s,
                                 const double *d_win, gs_batch_stats *out);
/* ---- signal sharding across GPUs (one process per GPU) ----
 * The reference's static split of each batch over workers (parallel.py:78)
 * across ranks: with shards set, every step on this engine (host, device or
 * sampled batch) finds winners only for signals [rank*m/world,
 * (rank+1)*m/world), one ncclAllGather of the GS_WINREC_BYTES records on the
 * engine stream assembles the batch in rank order == batch order, and every
 * rank runs the identical update (replicas stay bit-identical).  Every rank
 * must draw the same batches (same seed) and m % world == 0. */
#define GS_SHARD_ID_BYTES 128
/* A fresh communicator id (rank 0 makes it, the caller broadcasts it). */
gs_status gs_shard_unique_id(uint8_t *out, int64_t len);
/* Join the world (blocks until every rank joined); world = 0 detaches.
 * Engines joined with the same id share one communicator (initialised by
 * the first join, kept for the process); they must not run sharded steps
 * concurrently. */
gs_status gs_engine_set_shards(gs_engine *eng, int world, int rank, const uint8_t *id,
                               int64_t len);
/* Device time of the record all-gathers (with phase timing on), ms. */
gs_status gs_engine_exchange_ms(gs_engine *eng, double *out);

/* Per-phase device time (CUDA events on the engine stream) accumulated over
 * steps: out[0] find ms, out[1] update ms.  enable: 1 every batch, k > 1 one
 * batch in k weighted by k (an estimate with the event records off the
 * critical path), 0 off, -1 leave unchanged. */
gs_status gs_engine_phase_ms(gs_engine *eng, int enable, double out[2]);
/* Replace the run parameters used by subsequent updates (EngineParams). */
gs_status gs_engine_set_params(gs_engine *eng, const gs_params *params);
/* Synchronise the engine stream and copy out the last batch's stats. */
gs_status gs_engine_stats(gs_engine *eng, gs_batch_stats *out);
/* Stats of a device step at least `lag` steps before the newest one (0 <= lag
 * < 63; the nearest earlier step that carries a completion event: every
 * step, or in asynchronous sampled runs the last of each group), waiting only
 * for that step so later ones keep the GPU busy; *seq receives its index
 * (-1 and zeroed stats when none is available yet). */
gs_status gs_engine_stats_lagged(gs_engine *eng, int64_t lag, gs_batch_stats *out, int64_t *seq);
/* The engine's CUDA stream (cudaStream_t) for callers sharing it. */
void *gs_engine_stream(gs_engine *eng);
/* Allow up to `depth` batches to be enqueued ahead of the host's stats reads:
 * once converged, later batches leave the network untouched (stats.halted),
 * and stats.batches counts the batches that ran.  0 = synchronous contract.
 * While async, gs_engine_step_sampled draws `depth` batches of indices per
 * sampler launch (the batch size must stay fixed), so the sampler's state
 * may run up to depth-1 batches ahead of the batches executed. */
gs_status gs_engine_set_async(gs_engine *eng, int depth);
/* Pre-size device storage for ids [0, n) (avoids growth inside timed loops). */
gs_status gs_engine_reserve(gs_engine *eng, int64_t n);
/* Empty the network in place, keeping device allocations (a fresh
 * Network() + RunState(), network.py:79-96, engine.py:115-119). */
gs_status gs_engine_reset(gs_engine *eng);
/* Device launches issued by the engine so far (kernel count evidence). */
int64_t gs_engine_launch_count(const gs_engine *eng);

/* Counters: units, edges, next_id, tick, next_sweep, isolated, disk, half,
 * inconsistent, untrained (hab >= h_t), rows (find rows incl. dead). */
gs_status gs_engine_counts(gs_engine *eng, int64_t out[11]);
/* Live units in id order: ids, positions (n x 3), hab, theta, ring class
 * (0 disk, 1 half-disk, 2 inconsistent), patience, last_active (-1 absent). */
gs_status gs_engine_export_units(gs_engine *eng, int64_t cap, int64_t *ids, double *pos,
                                 double *hab, double *theta, int64_t *ring, int64_t *patience,
                                 int64_t *last_active, int64_t *n_out);
/* RunState (engine.py:101-119) over ids [0, next_id): *n_ids = next_id; when
 * cap >= next_id, patience[u], last_active[u] (-1 = no entry) and stamp[u]
 * (dict insertion order of the last_active entries; -1 = no entry) are
 * written (any array may be NULL).  Replaces reading state.tick /
 * state.next_sweep / state.patience / state.last_active. */
gs_status gs_engine_get_run_state(gs_engine *eng, int64_t *tick, int64_t *next_sweep, int64_t cap,
                                  int64_t *patience, int64_t *last_active, int64_t *stamp,
                                  int64_t *n_ids);
/* Load a RunState for the following updates (a fresh RunState() is tick 0,
 * next_sweep 1024, n 0).  Ids [0, n) take patience / last_active (-1 = no
 * entry) / stamp; stamps order the entries like dict insertion and must be
 * < 3 * (tick + 1).  Ids [n, next_id) get no entry; n <= next_id. */
gs_status gs_engine_set_run_state(gs_engine *eng, int64_t tick, int64_t next_sweep, int64_t n,
                                  const int64_t *patience, const int64_t *last_active,
                                  const int64_t *stamp);
/* All edges (a, b, age), a < b, sorted (network.py:152-161). */
gs_status gs_engine_export_edges(gs_engine *eng, int64_t cap, int64_t *abage, int64_t *n_out);
/* extract_mesh (metrics.py:148-163) on the device: every 3-clique a < b < c
 * of the unit graph once, as indices of the id-ordered live units, in the
 * reference's order.  *n_faces = the face count; faces (n x 3 int64) is
 * written when cap >= it; topo (may be NULL) = gs_mesh_topology's counts of
 * the same faces. */
gs_status gs_engine_extract_mesh(gs_engine *eng, int64_t cap, int64_t *faces, int64_t *n_faces,
                                 int64_t topo[6]);
/* Device audit (Network.audit, network.py:485-526): recomputes rings, degree
 * symmetry, counters; returns the number of violations found. */
gs_status gs_engine_audit(gs_engine *eng, int64_t *violations);

/* ------------------------------------------------------------------ */
/* device-side CloudSource sampler (sampling.py:175-177)               */

/* CloudSource.sample(rng, m) == points[rng.integers(0, N, size=m)] with
 * rng = Generator(Philox(seed)); the generator state lives on the device and
 * every draw is bit-identical to numpy's (Philox4x64-10, Lemire bounded
 * 32-bit draws).  points: N x 3 float64, host (copied once) or device
 * (points_on_device = 1, borrowed; must outlive the sampler), or NULL for
 * an index-only sampler; 1 <= N < 2^32. */
typedef struct gs_sampler gs_sampler;
gs_status gs_sampler_create(gs_ctx *ctx, const double *points, int64_t npts, int points_on_device,
                            gs_sampler **out);
void gs_sampler_destroy(gs_sampler *s);
/* numpy Philox bit_generator.state as uint64[15]: counter[4], key[2],
 * buffer[4], buffer_pos, has_uint32, uinteger, 0, 0 */
gs_status gs_sampler_set_state(gs_sampler *s, const uint64_t *state);
gs_status gs_sampler_get_state(gs_sampler *s, uint64_t *state);
/* m signals into d_out (m x 3 float64, device); asynchronous on `stream`
 * (NULL = the context stream); advances the device state. */
gs_status gs_sampler_draw(gs_sampler *s, int64_t m, double *d_out, void *stream);
/* rng.integers(0, npts, size=m) into d_idx (int64, device); a sampler made
 * with points == NULL only draws indices. */
gs_status gs_sampler_draw_indices(gs_sampler *s, int64_t m, int64_t *d_idx, void *stream);
/* gs_engine_step with the batch drawn on the device by `smp`; out == NULL
 * leaves the iteration queued (read stats later with gs_engine_stats). */
gs_status gs_engine_step_sampled(gs_engine *eng, gs_sampler *smp, int64_t m, gs_batch_stats *out);

#ifdef __cplusplus
}
#endif
#endif /* GROWSURF_B200_H */
