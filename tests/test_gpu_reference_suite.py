"""The reference's own matcher tests against the GPU matcher (SURVEY.md 7's
minimum-slice check): pkg/tests/test_matching.py and acceptance criteria C5
(matcher/oracle equivalence on 1000 pairs + adversarial + 200 forced
collisions) and C6 (adaptive >= fixed), run unchanged from the reference
install in baseline/_ref (tools/install_reference.sh) with this repo's
CUDA-backed _matchcore selected as kvlab's compiled backend."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "kvlab_tests")


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not installed "
                    "(tools/install_reference.sh)")
def test_reference_matcher_suite_on_gpu_matchcore():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [os.path.join(ROOT, "tests"), os.path.join(ROOT, "baseline", "_ref"), ROOT]))
    cmd = [sys.executable, "-m", "pytest", "-p", "_gpu_matchcore_plugin",
           "-p", "no:cacheprovider", os.path.join(REF_TESTS, "test_matching.py"),
           os.path.join(REF_TESTS, "test_acceptance.py"), "-k",
           "not test_acceptance or criterion_05 or criterion_06"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS,
                         timeout=1200)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    import re
    m = re.search(r"(\d+) passed", out.stdout)
    assert m and int(m.group(1)) >= 30 and "failed" not in out.stdout, tail
    assert "GPU drop-in" in out.stdout, tail          # the plugin's report header
    print(out.stdout.strip().splitlines()[-1])
