"""CPU-only checks of the C ABI and host logic (no device calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "growsurf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1503_08294_b200 import _lib

    lib = _lib.load_library()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table covers the header exactly
    assert sorted(_lib.EXPORTED) == syms


def test_library_is_sm100a():
    from paper_1503_08294_b200 import _lib

    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1503_08294_b200 import DeviceUnavailable, Network, kernels

    with pytest.raises(DeviceUnavailable):
        Network()
    with pytest.raises(DeviceUnavailable):
        kernels.best_two_single(np.zeros((2, 3)), 2, 0.0, 0.0, 0.0)


def test_version_string():
    from paper_1503_08294_b200 import _lib

    assert b"sm_100a" in _lib.load_library().gs_version()


def test_engine_params_validation():
    from paper_1503_08294_b200 import EngineParams

    EngineParams()
    for bad in (dict(eps_n=0.2), dict(theta0=0.0), dict(max_age=-1), dict(tau_b=1.0),
                dict(ring_patience=0), dict(max_signals=0), dict(batch_floor=100, batch_cap=64),
                dict(stale_factor=0)):
        with pytest.raises(ValueError):
            EngineParams(**bad)


def test_batch_size_rule():
    # pkg/tests/test_multi.py:25-55
    from paper_1503_08294_b200 import batch_size

    assert batch_size(330) == 512 and batch_size(512) == 1024
    assert batch_size(9000) == 8192 and batch_size(0) == 64 and batch_size(63) == 64
    for v in range(0, 20001, 7):
        m = batch_size(v)
        assert m & (m - 1) == 0 and 64 <= m <= 8192
        if m < 8192:
            assert m > v
    with pytest.raises(ValueError):
        batch_size(-1)


def test_cloud_stream_concatenates():
    """Consecutive CloudSource batches == one big draw (device-resident stream)."""
    from paper_1503_08294_b200 import CloudSource

    pts = np.random.default_rng(0).random((1000, 3))
    src = CloudSource(pts)
    r1 = np.random.Generator(np.random.Philox(7))
    a = np.concatenate([src.sample(r1, k) for k in (2, 64, 64, 128, 1024, 3)])
    r2 = np.random.Generator(np.random.Philox(7))
    b = src.sample(r2, 2 + 64 + 64 + 128 + 1024 + 3)
    assert np.array_equal(a, b)


def test_mesh_metrics_euler_anchors():
    # pkg/tests/test_metrics.py:126-137
    from paper_1503_08294_b200.metrics import euler_genus

    assert euler_genus(347, 1035, 690) == 0
    assert euler_genus(658, 1980, 1320) == 2


def test_library_then_torch_import_order():
    """Loading the library before torch must not break torch: the library
    links libnccl.so.2 by soname and _lib preloads the NCCL torch ships."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r); from paper_1503_08294_b200 import _lib; "
            "_lib.load_library(); import torch; print('ok')" % REPO)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
