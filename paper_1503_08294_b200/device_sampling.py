"""Device-side CloudSource sampling, bit-identical to numpy.

The reference samples every batch on the host: ``CloudSource.sample(rng, m)
= points[rng.integers(0, N, size=m)]`` with ``rng =
Generator(Philox(seed))`` (pkg/src/growsurf/sampling.py:175-177,
multi.py:151).  ``DeviceCloudSampler`` keeps the cloud and the Philox state
on the GPU (csrc/sample.cu) and produces the identical stream, so a run
never returns to the host for signals: the cloud crosses PCIe once.

The state is read from (and can be written back to) a numpy Generator, so
host and device sampling can be interleaved freely without changing a
single draw.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

__all__ = ["DeviceCloudSampler", "philox_state_words", "set_philox_state"]


def philox_state_words(rng: np.random.Generator) -> np.ndarray:
    """numpy Philox state as the C ABI's uint64[15] layout."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "Philox":
        raise ValueError("device sampling needs a Philox generator (multi.py:151)")
    w = np.zeros(15, np.uint64)
    w[0:4] = np.asarray(st["state"]["counter"], np.uint64)
    w[4:6] = np.asarray(st["state"]["key"], np.uint64)
    w[6:10] = np.asarray(st["buffer"], np.uint64)
    w[10] = st["buffer_pos"]
    w[11] = st["has_uint32"]
    w[12] = st["uinteger"]
    return w


def set_philox_state(rng: np.random.Generator, w: np.ndarray) -> None:
    """Write a uint64[15] device state back into a numpy Philox Generator."""
    st = rng.bit_generator.state
    st["state"]["counter"] = np.asarray(w[0:4], np.uint64).copy()
    st["state"]["key"] = np.asarray(w[4:6], np.uint64).copy()
    st["buffer"] = np.asarray(w[6:10], np.uint64).copy()
    st["buffer_pos"] = int(w[10])
    st["has_uint32"] = int(w[11])
    st["uinteger"] = int(w[12])
    rng.bit_generator.state = st


class DeviceCloudSampler:
    """CloudSource.sample on the GPU (gs_sampler_* in include/growsurf_b200.h)."""

    def __init__(self, points, rng: np.random.Generator | None = None, *, device_ptr: int = 0,
                 npts: int | None = None, context: _lib.Context | None = None):
        self._lib = _lib.load_library()
        self._ctx = context or _lib.default_context()
        h = C.c_void_p()
        if device_ptr:
            n = int(npts)
            _lib.check(self._lib.gs_sampler_create(self._ctx.handle, C.c_void_p(device_ptr), n, 1,
                                                   C.byref(h)))
            self._host = None
        elif points is None:
            n = int(npts)
            _lib.check(self._lib.gs_sampler_create(self._ctx.handle, None, n, 0, C.byref(h)))
            self._host = None
        else:
            self._host = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
            n = self._host.shape[0]
            _lib.check(self._lib.gs_sampler_create(self._ctx.handle,
                                                   self._host.ctypes.data_as(C.c_void_p), n, 0,
                                                   C.byref(h)))
        self._h = h
        self.npts = n
        if rng is not None:
            self.load_state(rng)

    @property
    def handle(self):
        return self._h

    def load_state(self, rng: np.random.Generator) -> None:
        _lib.check(self._lib.gs_sampler_set_state(self._h, philox_state_words(rng)))

    def state_words(self) -> np.ndarray:
        w = np.zeros(15, np.uint64)
        _lib.check(self._lib.gs_sampler_get_state(self._h, w))
        return w

    def store_state(self, rng: np.random.Generator) -> None:
        """Continue ``rng`` where the device stream stopped."""
        set_philox_state(rng, self.state_words())

    def draw(self, m: int, d_out: int, stream: int = 0) -> None:
        """m signals into the device buffer at d_out (m x 3 float64)."""
        _lib.check(self._lib.gs_sampler_draw(self._h, int(m), C.c_void_p(d_out),
                                             C.c_void_p(stream) if stream else None))

    def draw_indices(self, m: int, d_idx: int, stream: int = 0) -> None:
        _lib.check(self._lib.gs_sampler_draw_indices(self._h, int(m), C.c_void_p(d_idx),
                                                     C.c_void_p(stream) if stream else None))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gs_sampler_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
