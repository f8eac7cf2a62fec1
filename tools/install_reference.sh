#!/bin/bash
# Install the unmodified reference (kvlab, with its compiled Cython matcher)
# into baseline/_ref (git-ignored; travels to the GPU box with gpurun), plus
# its own test files under baseline/_ref/kvlab_tests so that the reference's
# matcher suite can run against the GPU _matchcore (tests/test_gpu_reference_suite.py).
# The build writes into its source tree, so it runs from a copy under /tmp.
set -euo pipefail
cd "$(dirname "$0")/.."
SRC=${KVLAB_SRC:-/root/reference/pkg}
TMP=$(mktemp -d /tmp/kvlab_src.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target baseline/_ref "$TMP" > /dev/null
mkdir -p baseline/_ref/kvlab_tests
cp "$TMP"/tests/*.py baseline/_ref/kvlab_tests/
rm -rf "$TMP"
python - <<'PY'
import sys
sys.path.insert(0, "baseline/_ref")
import kvlab.matching as m
print("kvlab installed in baseline/_ref; matcher backend:", m.BACKEND)
PY
