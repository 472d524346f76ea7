"""pytest plugin: run the reference's OWN test suite on the B200 backend.

Loaded by tests/test_ref_dropin.py (``pytest -p ref_dropin_plugin
oracle/_ref/ref_tests``).  It does exactly what INTEGRATION.md section 1 tells
a maintainer to add to growsurf/kernels/__init__.py:26-44: register
``paper_1503_08294_b200.kernels`` as ``_BACKENDS["b200"]`` and make it the
default backend, so every reference test that scans (kernels, parallel
executor, batch finds, run_multi, single-signal run, quantization error)
goes through the sm_100a kernels, and the backend-parametrised kernel tests
also run on "b200" by name.  The reference package itself is unmodified.
"""

import json
import os


def pytest_configure(config):
    import growsurf.kernels as K

    from paper_1503_08294_b200 import kernels as b200

    K._BACKENDS["b200"] = b200
    K.DEFAULT_BACKEND_NAME = "b200"


def pytest_sessionfinish(session, exitstatus):
    from paper_1503_08294_b200 import kernels as b200

    out = os.environ.get("GS_DROPIN_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump(dict(b200.calls, exitstatus=int(exitstatus)), fh)
