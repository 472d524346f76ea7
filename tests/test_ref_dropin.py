"""Drop-in proof from the reference's side (SURVEY.md 8(b) boundaries 1-2).

1. The reference's OWN test suite (copied next to the built reference into
   oracle/_ref/ref_tests by oracle/build_ref.sh; the reference sources stay
   unmodified) runs with the B200 kernels registered in its backend registry
   as the default (tests/ref_dropin_plugin.py, the registration
   INTEGRATION.md section 1 describes): every test must pass and the B200
   kernels must have served the scans.
2. The reference's own ``run_multi`` driver (multi.py:134-202) with the find
   done by this package -- ``sequential_executor(backend=<b200 module>)``
   from the reference and ``b200_executor()`` from this package -- must
   reproduce the golden runs bit for bit.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from cases import CASES, load_golden, make_source, same_numpy

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import growsurf
    except ImportError:
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    return growsurf


def test_reference_test_suite_on_b200_backend(tmp_path):
    _ref()
    suite = os.path.join(REF, "ref_tests")
    if not os.path.isdir(suite):
        pytest.skip("reference tests not copied (oracle/build_ref.sh)")
    report = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO, os.path.join(REPO, "tests")])
    env["GS_DROPIN_REPORT"] = str(report)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "ref_dropin_plugin", suite],
                       cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    calls = json.loads(report.read_text())
    assert calls["exitstatus"] == 0
    # the scans really ran on the B200 (single-signal runs, batches, kernels)
    assert calls["scan_best_two_into"] > 1000 and calls["best_two_single"] > 1000, calls
    assert " passed" in tail and "failed" not in tail


def _assert_net_equals_golden(rnet, gold):
    ids, pos, hab, theta = rnet.state_arrays()
    assert np.array_equal(ids, gold["ids"])
    assert np.array_equal(np.array(rnet.edges(), np.int64).reshape(-1, 3), gold["edges"])
    for a, k in ((pos, "pos"), (hab, "hab"), (theta, "theta")):
        assert np.array_equal(np.ascontiguousarray(a).view(np.int64), gold[k].view(np.int64)), k


@pytest.mark.parametrize("how", ["ref_sequential_b200_backend", "b200_executor"])
@pytest.mark.parametrize("name", ["sphere_exec", "cfg1"])
def test_reference_run_multi_with_b200_find(name, how):
    R = _ref()
    from growsurf.multi import sequential_executor as ref_sequential_executor

    from paper_1503_08294_b200 import b200_executor
    from paper_1503_08294_b200 import kernels as b200

    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    case = CASES[name]
    params = R.EngineParams(**case["params"])
    src = make_source(case["source"])
    before = b200.calls["scan_best_two_into"]
    if how == "b200_executor":
        ex = b200_executor()
    else:
        ex = ref_sequential_executor(backend=b200)
    rnet, st = R.run_multi(src, params, case["seed"], ex)
    assert b200.calls["scan_best_two_into"] - before == st.iterations
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k
    _assert_net_equals_golden(rnet, gold)
