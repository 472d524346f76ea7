#!/usr/bin/env bash
# Build the UNMODIFIED reference package (growsurf, Python + Cython scan kernel)
# into oracle/_ref/ so tests, smoke() and bench.py's reference arm can import it.
# Test infrastructure only: the product never imports oracle/_ref.
# /root/reference is read-only, so the build runs on a scratch copy under /tmp.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
if [ ! -d "$src" ]; then
  echo "build_ref: $src not present; skipping (the GPU box uses the prebuilt oracle/_ref)" >&2
  exit 0
fi
tmp="$(mktemp -d /tmp/growsurf_ref.XXXXXX)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$here/_ref" "$tmp/pkg"
# the reference's own test suite travels with it (tests/test_ref_dropin.py runs
# it with the B200 kernels registered as the default backend)
cp -r "$src/tests" "$here/_ref/ref_tests"
python - "$here/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from growsurf import kernels
assert kernels.HAVE_COMPILED, "reference Cython kernel did not build"
print("oracle/_ref: growsurf built, backends", kernels.available_backends())
PY
