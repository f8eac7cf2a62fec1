"""pytest plugin (tests/test_gpu_reference_suite.py): before the reference's
own test files import kvlab, install this repo's GPU drop-in as
``kvlab._matchcore`` - exactly what placing the module in the reference
package does - so kvlab.matching selects it as its
compiled backend."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    sys.path.insert(0, ROOT)
    import paper_2503_16525_b200._matchcore as gpu_matchcore
    sys.modules["kvlab._matchcore"] = gpu_matchcore
    import kvlab.matching as m
    assert m.BACKEND == "compiled" and m._matchcore is gpu_matchcore, "GPU matcher not selected"
