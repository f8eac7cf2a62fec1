"""Phase timeline of the fused D3 kernel (build with -DKVS_D3_TRACE, load
through KVS_LIB): per-CTA globaltimer stamps, median over CTAs."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_16525_b200 import _native as N  # noqa: E402

if __name__ == "__main__":
    for n in [int(x) for x in sys.argv[1:]] or [64, 256]:
        r = bench.decode_select_batch_leg(n, iters=1)
        lib = N.load()
        buf = (ctypes.c_ulonglong * (148 * 8))()
        lib.kvs_d3_trace(buf)
        t = np.array(buf, dtype=np.float64).reshape(148, 8)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        names = ["p1_end", "barrier", "stats", "list0", "list", "scored", "merge0", "end"]
        print(n, r["ms"] * 1000, "us;", " ".join(
            f"{nm}: med {np.median(rel[:, i][t[:, i] > 0]):.1f} max {rel[:, i][t[:, i] > 0].max():.1f}"
            if (t[:, i] > 0).any() else f"{nm}: -" for i, nm in enumerate(names)))
