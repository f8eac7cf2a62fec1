"""pytest plugin (tests/test_gpu_reference_suite.py): before the reference's
own test files import kvlab, install this repo's GPU drop-in as
``kvlab._matchcore`` - exactly what placing the module in the reference
package does - so kvlab.matching selects it as its
compiled backend.  Runs at plugin import (-p), ahead of the reference's
conftest, which imports kvlab."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

import paper_2503_16525_b200._matchcore as gpu_matchcore  # noqa: E402

sys.modules["kvlab._matchcore"] = gpu_matchcore

import kvlab.matching as _m  # noqa: E402

assert _m.BACKEND == "compiled" and _m._matchcore is gpu_matchcore, "GPU matcher not selected"


def pytest_report_header(config):
    return f"kvlab._matchcore -> {gpu_matchcore.__file__} (GPU drop-in)"
