"""Device-resident Network with the reference's accessor/mutator API.

The reference Network (pkg/src/growsurf/network.py:71-546) keeps dense
id-ordered numpy arrays plus dict adjacency on the host.  Here the whole
network lives in B200 HBM inside a gs_engine (csrc/engine.cu): unit state
indexed by id, fixed-capacity adjacency with per-edge ages, incrementally
maintained ring classes.  Readers below copy a snapshot of the device state
to the host (cached until the next mutation); mutators run the serial
device primitives.  The training loop itself (run_multi /
resolve_and_update in multi.py) never leaves the device.

``state_arrays()`` returns host copies whose element writes go through to
the device (``hab[:] = 0.05``, ``pos[rows] = moved``, ``theta[k] *= rho``,
the in-place edits the reference's tests make on its live views,
network.py:178-186); a write that cannot be intercepted (a slice of a view,
``np.copyto``) fails loudly on a read-only array instead of being lost.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .params import (
    RING_FROM_CODE,
    EngineParams,
    RingClass,
    StateError,
    UnknownUnitError,
)

__all__ = ["Network", "Snapshot", "RingClass", "StateError", "UnknownUnitError"]


class Snapshot:
    """Dense id-ordered positions (network.py:47-59)."""

    __slots__ = ("ids", "positions")

    def __init__(self, ids: np.ndarray, positions: np.ndarray):
        self.ids = ids
        self.positions = positions

    def __len__(self) -> int:
        return self.ids.shape[0]


def to_gs_params(params: EngineParams, find_mode: int = _lib.FIND_AUTO) -> _lib.GsParams:
    return _lib.GsParams(
        params.eps_b, params.eps_n, params.theta0, int(params.max_age), params.tau_b,
        params.tau_n, params.h_t, params.rho, int(params.ring_patience),
        int(bool(params.allow_boundary)), int(find_mode), int(params.stale_factor))


class _WriteThrough(np.ndarray):
    """Host copy of one device unit array (positions, habituation or
    thresholds, id order) that writes changed rows back to the device.

    The buffer is read-only: ``__setitem__`` and the in-place operators
    (``+=``, ``*=`` ... via ``__array_ufunc__`` with ``out=self``) are the
    only writers, and both push every changed row with ``set_unit``.
    Slices and ufunc results are plain ndarrays (slices stay read-only).
    """

    def __new__(cls, data, net, field):
        obj = np.array(data, copy=True).view(cls)
        obj._gs = (net, field)
        obj.flags.writeable = False
        return obj

    def __array_finalize__(self, obj):
        self._gs = None

    def __getitem__(self, key):
        return np.ndarray.__getitem__(self.view(np.ndarray), key)

    def _commit(self, before):
        net, field = self._gs
        now = self.view(np.ndarray)
        diff = now.view(np.uint64) != before.view(np.uint64)
        if diff.ndim == 2:
            diff = diff.any(axis=1)
        ids = net._mirror()["ids"].copy()
        for r in np.flatnonzero(diff).tolist():
            kw = {"position": now[r]} if field == "pos" else {field: float(now[r])}
            net.set_unit(int(ids[r]), **kw)

    def _write(self, fn):
        if self._gs is None:
            raise ValueError("assignment destination is read-only")
        before = self.view(np.ndarray).copy()
        self.flags.writeable = True
        try:
            fn(self.view(np.ndarray))
        finally:
            self.flags.writeable = False
        self._commit(before)

    def __setitem__(self, key, value):
        self._write(lambda a: a.__setitem__(key, value))

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kw):
        plain = tuple(x.view(np.ndarray) if isinstance(x, _WriteThrough) else x for x in inputs)
        if out is None:
            return getattr(ufunc, method)(*plain, **kw)
        targets = [o for o in out if isinstance(o, _WriteThrough)]
        if len(targets) != 1 or len(out) != 1 or method != "__call__":
            raise ValueError("assignment destination is read-only")
        result = getattr(ufunc, method)(*plain, **kw)
        targets[0]._write(lambda a: a.__setitem__(Ellipsis, result))
        return targets[0]


class Network:
    """Growable undirected unit graph, resident on the GPU."""

    def __init__(self, params: EngineParams | None = None, *, capacity: int = 4096,
                 find_mode: int = _lib.FIND_AUTO, context: _lib.Context | None = None):
        self._lib = _lib.load_library()
        self._ctx = context or _lib.default_context()
        self._params = params or EngineParams()
        self._find_mode = find_mode
        gp = to_gs_params(self._params, find_mode)
        h = C.c_void_p()
        _lib.check(self._lib.gs_engine_create(self._ctx.handle, C.byref(gp), int(capacity),
                                              C.byref(h)))
        self._h = h
        self._version = 0
        self._cache = None
        self._watch_limit = None

    # -- lifetime -----------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.gs_engine_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def stream_handle(self) -> int:
        """The engine's cudaStream_t as an integer (for torch.cuda.ExternalStream)."""
        return int(self._lib.gs_engine_stream(self._h) or 0)

    def reset(self) -> None:
        """Empty the network in place (a fresh Network + RunState), keeping allocations."""
        _lib.check(self._lib.gs_engine_reset(self._h))
        self._touch()

    def set_async(self, depth: int) -> None:
        """Allow `depth` batches in flight ahead of stats reads (gs_engine_set_async)."""
        _lib.check(self._lib.gs_engine_set_async(self._h, int(depth)))

    def set_shards(self, world: int, rank: int, uid: bytes | None = None) -> None:
        """Shard every later step's find over ``world`` ranks (this is
        ``rank``; ``uid`` is the communicator id all ranks share, see
        distributed.attach); world = 0 detaches."""
        buf = None
        if world:
            if uid is None or len(uid) != _lib.SHARD_ID_BYTES:
                raise ValueError("a shard id of SHARD_ID_BYTES bytes is required")
            buf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
        _lib.check(self._lib.gs_engine_set_shards(self._h, int(world), int(rank), buf,
                                                  _lib.SHARD_ID_BYTES))

    def exchange_ms(self) -> float:
        """Device time of the sharded record all-gathers so far (phase timing on)."""
        out = C.c_double()
        _lib.check(self._lib.gs_engine_exchange_ms(self._h, C.byref(out)))
        return out.value

    def reserve(self, n_ids: int) -> None:
        _lib.check(self._lib.gs_engine_reserve(self._h, int(n_ids)))

    def launch_count(self) -> int:
        return int(self._lib.gs_engine_launch_count(self._h))

    def set_params(self, params: EngineParams) -> None:
        if params is self._params:
            return
        gp = to_gs_params(params, self._find_mode)
        _lib.check(self._lib.gs_engine_set_params(self._h, C.byref(gp)))
        self._params = params

    def _touch(self):
        self._version += 1
        self._cache = None

    # -- device mirror --------------------------------------------------------
    def counts(self) -> dict:
        out = np.zeros(11, np.int64)
        _lib.check(self._lib.gs_engine_counts(self._h, out))
        keys = ("units", "edges", "next_id", "tick", "next_sweep", "isolated", "disk", "half",
                "inconsistent", "untrained", "rows")
        return dict(zip(keys, (int(v) for v in out)))

    def _mirror(self):
        if self._cache is not None:
            return self._cache
        cnt = self.counts()
        n = cnt["units"]
        ids = np.empty(n, np.int64)
        pos = np.empty((n, 3), np.float64)
        hab = np.empty(n, np.float64)
        theta = np.empty(n, np.float64)
        ring = np.empty(n, np.int64)
        patience = np.empty(n, np.int64)
        last_active = np.empty(n, np.int64)
        got = C.c_int64()
        _lib.check(self._lib.gs_engine_export_units(
            self._h, n, ids.ctypes.data, pos.ctypes.data, hab.ctypes.data, theta.ctypes.data,
            ring.ctypes.data, patience.ctypes.data, last_active.ctypes.data, C.byref(got)))
        ne = cnt["edges"]
        edges = np.empty((max(ne, 1), 3), np.int64)
        gote = C.c_int64()
        _lib.check(self._lib.gs_engine_export_edges(self._h, ne, edges.ctypes.data, C.byref(gote)))
        edges = edges[: gote.value]
        row = {int(u): i for i, u in enumerate(ids)}
        adj = {int(u): {} for u in ids}
        for a, b, age in edges.tolist():
            adj[a][b] = age
            adj[b][a] = age
        self._cache = dict(counts=cnt, ids=ids, pos=pos, hab=hab, theta=theta, ring=ring,
                           patience=patience, last_active=last_active, edges=edges, row=row,
                           adj=adj)
        return self._cache

    def export(self) -> dict:
        """Full state dump (ids, pos, hab, theta, ring, patience, last_active, edges, ...)."""
        m = self._mirror()
        c = m["counts"]
        return dict(ids=m["ids"], pos=m["pos"], hab=m["hab"], theta=m["theta"], ring=m["ring"],
                    patience=m["patience"], last_active=m["last_active"], edges=m["edges"],
                    tick=c["tick"], next_sweep=c["next_sweep"], next_id=c["next_id"])

    def _require(self, unit_id) -> int:
        try:
            return self._mirror()["row"][int(unit_id)]
        except (KeyError, TypeError, ValueError):
            raise UnknownUnitError(f"unit {unit_id!r} is not alive") from None

    # -- introspection (network.py:101-203) -----------------------------------
    @property
    def unit_count(self) -> int:
        return self.counts()["units"]

    @property
    def edge_count(self) -> int:
        return self.counts()["edges"]

    @property
    def next_id(self) -> int:
        return self.counts()["next_id"]

    @property
    def version(self) -> int:
        return self._version

    def is_alive(self, unit_id: int) -> bool:
        try:
            return int(unit_id) in self._mirror()["row"]
        except (TypeError, ValueError):
            return False

    def unit_ids(self) -> list[int]:
        return [int(u) for u in self._mirror()["ids"]]

    def position(self, unit_id: int) -> np.ndarray:
        return self._mirror()["pos"][self._require(unit_id)].copy()

    def habituation(self, unit_id: int) -> float:
        return float(self._mirror()["hab"][self._require(unit_id)])

    def local_threshold(self, unit_id: int) -> float:
        return float(self._mirror()["theta"][self._require(unit_id)])

    def neighbors(self, unit_id: int) -> set[int]:
        self._require(unit_id)
        return set(self._mirror()["adj"][int(unit_id)])

    def degree(self, unit_id: int) -> int:
        self._require(unit_id)
        return len(self._mirror()["adj"][int(unit_id)])

    def has_edge(self, a: int, b: int) -> bool:
        adj = self._mirror()["adj"]
        return a in adj and b in adj[a]

    def edge_age(self, a: int, b: int) -> int:
        self._require(a)
        self._require(b)
        try:
            return self._mirror()["adj"][a][b]
        except KeyError:
            raise KeyError(f"no edge between {a} and {b}") from None

    def edges(self) -> list[tuple[int, int, int]]:
        return [tuple(e) for e in self._mirror()["edges"].tolist()]

    def ring_class_counts(self) -> dict:
        c = self.counts()
        return {RingClass.DISK: c["disk"], RingClass.HALF_DISK: c["half"],
                RingClass.INCONSISTENT: c["inconsistent"]}

    def all_rings_surface(self, allow_half_disks: bool = False) -> bool:
        c = self.counts()
        ok = c["disk"] + (c["half"] if allow_half_disks else 0)
        return ok == c["units"]

    def max_habituation(self) -> float:
        hab = self._mirror()["hab"]
        if hab.size == 0:
            raise StateError("empty network has no habituation")
        return float(np.max(hab))

    def state_arrays(self):
        """(ids, positions, habituation, thresholds) in id order
        (network.py:178-186).  ids is read-only; the other three write
        element edits through to the device (see _WriteThrough)."""
        m = self._mirror()
        ids = m["ids"].copy()
        ids.flags.writeable = False
        return (ids, _WriteThrough(m["pos"], self, "pos"),
                _WriteThrough(m["hab"], self, "habituation"),
                _WriteThrough(m["theta"], self, "threshold"))

    def row_of(self, unit_id: int) -> int:
        return self._require(unit_id)

    def snapshot(self, copy: bool = True) -> Snapshot:
        m = self._mirror()
        return Snapshot(m["ids"].copy(), np.ascontiguousarray(m["pos"].copy()))

    def link_ring(self, unit_id: int) -> RingClass:
        return RING_FROM_CODE[int(self._mirror()["ring"][self._require(unit_id)])]

    def audit(self) -> None:
        """Device-side invariant check (network.py:485-526); AssertionError on damage."""
        v = C.c_int64()
        _lib.check(self._lib.gs_engine_audit(self._h, C.byref(v)))
        assert v.value == 0, f"device audit found {v.value} violations"
        ids = self._mirror()["ids"]
        assert np.all(np.diff(ids) > 0), "ids must be strictly increasing"

    # -- mutation (network.py:208-369) ----------------------------------------
    def add_unit(self, position, threshold: float) -> int:
        pos = np.asarray(position, dtype=np.float64).reshape(-1)
        if pos.shape != (3,):
            raise ValueError(f"position must have 3 components, got shape {pos.shape}")
        uid = C.c_int64()
        _lib.check(self._lib.gs_engine_add_unit(self._h, float(pos[0]), float(pos[1]),
                                                float(pos[2]), float(threshold), C.byref(uid)))
        self._touch()
        return uid.value

    def remove_unit(self, unit_id: int) -> None:
        _lib.check(self._lib.gs_engine_remove_unit(self._h, int(unit_id)))
        self._touch()

    def watch_age_limit(self, max_age: int) -> None:
        if max_age < 0:
            raise ValueError("max_age must be >= 0")
        self._watch_limit = max_age

    def connect_or_reset(self, a: int, b: int) -> str:
        if a == b:
            raise ValueError(f"cannot connect unit {a} to itself")
        created = C.c_int32()
        _lib.check(self._lib.gs_engine_connect_or_reset(self._h, int(a), int(b),
                                                        C.byref(created)))
        self._touch()
        return "created" if created.value == 1 else "reset"

    def remove_edge(self, a: int, b: int) -> None:
        self._require(a)
        self._require(b)
        if not self.has_edge(a, b):
            raise KeyError(f"no edge between {a} and {b}")
        _lib.check(self._lib.gs_engine_remove_edge(self._h, int(a), int(b)))
        self._touch()

    def age_incident_edges(self, b: int, increment: int, exclude: int | None = None) -> int:
        top = C.c_int64()
        _lib.check(self._lib.gs_engine_age_incident_edges(
            self._h, int(b), int(increment), -1 if exclude is None else int(exclude),
            C.byref(top)))
        self._touch()
        return top.value

    def prune(self, max_age: int, removed_units: list | None = None) -> tuple[int, int]:
        before = set(self.unit_ids()) if removed_units is not None else None
        pe, pu = C.c_int64(), C.c_int64()
        _lib.check(self._lib.gs_engine_prune(self._h, int(max_age), C.byref(pe), C.byref(pu)))
        self._touch()
        if removed_units is not None:
            removed_units.extend(sorted(before - set(self.unit_ids())))
        return pe.value, pu.value

    def set_unit(self, unit_id: int, position=None, habituation=None, threshold=None) -> None:
        """Overwrite one unit's position / habituation / threshold on the device."""
        xyz = None if position is None else np.ascontiguousarray(position, dtype=np.float64)
        h = None if habituation is None else C.c_double(float(habituation))
        t = None if threshold is None else C.c_double(float(threshold))
        _lib.check(self._lib.gs_engine_set_unit(
            self._h, int(unit_id), None if xyz is None else xyz.ctypes.data,
            None if h is None else C.addressof(h), None if t is None else C.addressof(t)))
        self._touch()
