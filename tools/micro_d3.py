"""D3 fused decode-stage DHD on decode batches of 8-256 Llama-shape requests
(bench.decode_select_batch_leg): achieved algorithmic GB/s vs measured HBM."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    hbm = bench.peaks()[0]
    sizes = [int(x) for x in sys.argv[1:]] or [8, 64, 128, 256]
    for n in sizes:
        r = bench.decode_select_batch_leg(n)
        r["frac"] = r["achieved"] / hbm
        print(json.dumps(r))
