"""ctypes wrapper + Python driver for the C oracle (growsurf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker.  The product package
(paper_1503_08294_b200) never imports this module.

``run_multi_oracle`` mirrors the reference driver run_multi
(pkg/src/growsurf/multi.py:134-202): it seeds two units from the first two
samples, then per batch computes m = batch_size(V) (multi.py:44-55), samples
on the host, and calls the C step (find + winner lock + update_single).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class _Params(C.Structure):
    _fields_ = [
        ("eps_b", C.c_double), ("eps_n", C.c_double), ("theta0", C.c_double),
        ("max_age", C.c_int64), ("tau_b", C.c_double), ("tau_n", C.c_double),
        ("h_t", C.c_double), ("rho", C.c_double), ("ring_patience", C.c_int64),
        ("allow_boundary", C.c_int32), ("pad_", C.c_int32), ("stale_factor", C.c_int64),
    ]


def build() -> str:
    """Compile liboracle.so with the repo's Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "growsurf_oracle.c"))
        ):
            build()
        L = C.CDLL(LIB_PATH)
        L.go_new.restype = C.c_void_p
        L.go_new.argtypes = [C.POINTER(_Params)]
        L.go_free.argtypes = [C.c_void_p]
        L.go_add_unit.restype = C.c_int64
        L.go_add_unit.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double]
        L.go_scan_best_two.argtypes = [_f64p, C.c_int64, _f64p, C.c_int64, _i64p, _f64p]
        L.go_step.restype = C.c_int
        L.go_step.argtypes = [C.c_void_p, _f64p, C.c_int64, _i64p, C.c_void_p, C.c_void_p]
        L.go_resolve_and_update.restype = C.c_int
        L.go_resolve_and_update.argtypes = [C.c_void_p, _f64p, C.c_int64, _i64p, _i64p, _f64p, _i64p]
        L.go_is_converged.restype = C.c_int
        L.go_is_converged.argtypes = [C.c_void_p]
        L.go_counts.argtypes = [C.c_void_p, _i64p]
        L.go_export_units.argtypes = [C.c_void_p, _i64p, _f64p, _f64p, _f64p, _i64p, _i64p, _i64p]
        L.go_export_edges.restype = C.c_int64
        L.go_export_edges.argtypes = [C.c_void_p, _i64p]
        L.go_audit_rings.restype = C.c_int64
        L.go_audit_rings.argtypes = [C.c_void_p]
        L.go_connect_or_reset.restype = C.c_int
        L.go_connect_or_reset.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.go_classify_ring.restype = C.c_int
        L.go_classify_ring.argtypes = [C.c_void_p, C.c_int64]
        L.go_set_hab.argtypes = [C.c_void_p, C.c_int64, C.c_double]
        _lib = L
    return _lib


def scan_best_two(pos, signals):
    """Exact FP64 best-two scan (_scan.pyx:39-98): (m,2) int64 rows, (m,2) f64 d^2."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    sig = np.ascontiguousarray(signals, dtype=np.float64).reshape(-1, 3)
    m = sig.shape[0]
    idx = np.empty((m, 2), np.int64)
    d2 = np.empty((m, 2), np.float64)
    lib().go_scan_best_two(pos, pos.shape[0], sig, m, idx, d2)
    return idx, d2


@dataclass
class OracleParams:
    """Field-for-field EngineParams (engine.py:38-95)."""

    eps_b: float = 0.1
    eps_n: float = 0.01
    theta0: float = 0.2
    max_age: int = 200
    tau_b: float = 0.05
    tau_n: float = 0.005
    h_t: float = 0.3
    rho: float = 0.8
    ring_patience: int = 500
    max_signals: int = 5_000_000
    allow_boundary: bool = False
    batch_cap: int = 8192
    batch_floor: int = 64
    stale_factor: int = 30

    @classmethod
    def of(cls, params):
        names = [f for f in cls.__dataclass_fields__]
        return cls(**{k: getattr(params, k) for k in names})


def batch_size(units: int, cap: int = 8192, floor: int = 64) -> int:
    """multi.py:44-55."""
    m = 1 << int(units).bit_length()
    return min(max(m, floor), cap)


class OracleNet:
    """A C-oracle network + RunState."""

    def __init__(self, params):
        p = OracleParams.of(params)
        self.params = p
        cp = _Params(p.eps_b, p.eps_n, p.theta0, p.max_age, p.tau_b, p.tau_n, p.h_t, p.rho,
                     p.ring_patience, int(bool(p.allow_boundary)), 0, p.stale_factor)
        self._h = lib().go_new(C.byref(cp))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.go_free(h)
            self._h = None

    def add_unit(self, pos, theta):
        uid = lib().go_add_unit(self._h, float(pos[0]), float(pos[1]), float(pos[2]), float(theta))
        if uid < 0:
            raise ValueError("bad unit")
        return uid

    def connect_or_reset(self, a, b):
        return lib().go_connect_or_reset(self._h, a, b)

    def set_hab(self, u, h):
        lib().go_set_hab(self._h, u, h)

    def classify_ring(self, u):
        return lib().go_classify_ring(self._h, u)

    def step(self, batch, trace=False):
        batch = np.ascontiguousarray(batch, dtype=np.float64).reshape(-1, 3)
        m = batch.shape[0]
        out = np.zeros(3, np.int64)
        wid = np.empty((m, 2), np.int64) if trace else None
        wd2 = np.empty((m, 2), np.float64) if trace else None
        rc = lib().go_step(self._h, batch, m, out,
                           wid.ctypes.data if trace else None, wd2.ctypes.data if trace else None)
        if rc != 0:
            raise RuntimeError(f"oracle step failed rc={rc}")
        if trace:
            return out, wid, wd2
        return out

    def resolve_and_update(self, batch, win_b, win_s, d_win):
        batch = np.ascontiguousarray(batch, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(3, np.int64)
        rc = lib().go_resolve_and_update(
            self._h, batch, batch.shape[0], np.ascontiguousarray(win_b, np.int64),
            np.ascontiguousarray(win_s, np.int64), np.ascontiguousarray(d_win, np.float64), out)
        if rc != 0:
            raise RuntimeError(f"oracle resolve failed rc={rc}")
        return out

    def converged(self) -> bool:
        return bool(lib().go_is_converged(self._h))

    def counts(self):
        c = np.zeros(10, np.int64)
        lib().go_counts(self._h, c)
        keys = ("units", "edges", "next_id", "tick", "next_sweep", "isolated",
                "disk", "half", "inconsistent", "n_over")
        return dict(zip(keys, (int(x) for x in c)))

    def export(self):
        c = self.counts()
        n = c["units"]
        ids = np.empty(n, np.int64)
        pos = np.empty((n, 3), np.float64)
        hab = np.empty(n, np.float64)
        theta = np.empty(n, np.float64)
        ring = np.empty(n, np.int64)
        patience = np.empty(n, np.int64)
        last_active = np.empty(n, np.int64)
        lib().go_export_units(self._h, ids, pos, hab, theta, ring, patience, last_active)
        edges = np.empty((max(c["edges"], 1), 3), np.int64)
        ne = lib().go_export_edges(self._h, edges)
        return dict(ids=ids, pos=pos, hab=hab, theta=theta, ring=ring, patience=patience,
                    last_active=last_active, edges=edges[:ne].copy(), tick=c["tick"],
                    next_sweep=c["next_sweep"], next_id=c["next_id"])

    def audit_rings(self) -> int:
        return int(lib().go_audit_rings(self._h))


def run_multi_oracle(source, params, seed, *, trace=False):
    """run_multi (multi.py:134-202) driven by the C oracle.

    Returns (OracleNet, stats dict, per_batch (k,4) int64, signal sha256).
    """
    p = OracleParams.of(params)
    rng = np.random.Generator(np.random.Philox(seed))
    net = OracleNet(p)
    seeds = source.sample(rng, 2)
    digest = hashlib.sha256()
    digest.update(np.ascontiguousarray(seeds).tobytes())
    for k in range(2):
        net.add_unit(seeds[k], p.theta0)
    per_batch = []
    signals = discarded = iterations = 0
    converged = False
    t0 = time.perf_counter()
    while signals < p.max_signals:
        m = batch_size(net.counts()["units"], p.batch_cap, p.batch_floor)
        batch = source.sample(rng, m)
        digest.update(np.ascontiguousarray(batch).tobytes())
        out = net.step(batch)
        per_batch.append((m, int(out[0]), int(out[1]), int(out[2])))
        signals += m
        discarded += int(out[1])
        iterations += 1
        if net.converged():
            converged = True
            break
    c = net.counts()
    stats = dict(iterations=iterations, signals=signals, discarded=discarded, units=c["units"],
                 connections=c["edges"], converged=converged,
                 total_s=time.perf_counter() - t0)
    return net, stats, np.array(per_batch, np.int64).reshape(-1, 4), digest.hexdigest()
