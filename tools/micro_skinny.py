"""P1 (kvs_proj_skinny) against the library GEMM at decode row counts for
the benched projection shapes: time per call (CUDA events, 50 calls after
warm-up, weights larger in total than L2 so each call streams from HBM)
and the fraction of measured HBM bandwidth the weight stream reaches.

    python tools/micro_skinny.py [--rows 8,32,64]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_16525_b200 import _native as N  # noqa: E402
from paper_2503_16525_b200.engine import Engine  # noqa: E402

SHAPES = {"llama_qkv": (4096, 6144), "llama_o": (4096, 4096), "qwen_qkv": (3584, 4608),
          "qwen_o": (3584, 3584)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="8,32,64")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs_burst") or peaks.get("hbm_gbs") or 6551.4)
    reps = 50
    for name, (k, n) in SHAPES.items():
        # 40 distinct weight copies (> L2 in total) cycled through
        ws = [(torch.randn(k, n, device="cuda") / k ** 0.5).to(torch.bfloat16) for _ in range(40)]
        wts = [Engine.pack_skinny(w) for w in ws]
        for m in [int(v) for v in a.rows.split(",")]:
            x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
            def p1(i):
                wt = wts[i % 40]
                N.call("kvs_proj_skinny", x.data_ptr(), m, wt.data_ptr(), n, k, 0, out.data_ptr(),
                       None, N.stream_ptr())
            def lib(i):
                torch.matmul(x, ws[i % 40], out=out)
            res = {}
            for label, fn in (("p1", p1), ("cublas", lib)):
                for i in range(10):
                    fn(i)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for i in range(reps):
                    fn(i)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / reps
                res[label] = {"us": round(us, 2),
                              "hbm_frac": round(k * n * 2 / (us * 1e-6) / 1e9 / hbm, 3)}
            print(json.dumps({"shape": name, "m": m, "k": k, "n": n, **res}), flush=True)
        del ws, wts


if __name__ == "__main__":
    main()
