"""D2 phase timeline inside a real bench step (diagnostic; run under gpurun).
Builds the library with -DKVS_SEL_TRACE, runs bench steps and prints the
per-CTA phase stamps of the step's dhd_select_fused launch.

    python tools/select_trace_step.py [bench args...]
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = "/tmp/libkvshare_seltrace.so"
subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), LIB,
                       "-DKVS_SEL_TRACE", *os.environ.get("KVS_DEFS", "").split()],
                      stdout=subprocess.DEVNULL)
os.environ["KVS_LIB"] = LIB

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_16525_b200 import _native as N  # noqa: E402
from paper_2503_16525_b200.workload import request_batches  # noqa: E402


def main():
    sys.argv = [sys.argv[0]] + sys.argv[1:]
    args = bench.parse()
    if args.layers is None:
        args.layers = 32
    dev = torch.device("cuda", 0)
    cfg, model, pool, eng, sources = bench.build_engine(args, dev)
    batches = request_batches(sources, 4, args.batch, args.seq, args.hit, cfg.vocab_size, seed=1)
    lib = N.load()
    lib.kvs_sel_trace_dump.restype = ctypes.c_int32
    buf = np.zeros(1024 * 8, dtype=np.uint64)
    for i in range(3):
        lib.kvs_sel_trace_dump(buf.ctypes.data, buf.size)          # clear
        st = eng.prefill_batch(batches[i], ratio=args.ratio)
        torch.cuda.synchronize()
        # the top-B's candidate counts on this step's scores: rows in the
        # threshold exponent (c0) and within the 17-bit prefix (c1)
        sc = st.score.cpu().numpy()
        slot = st.src_slot.cpu().numpy()
        bud = st._bud.cpu().numpy()
        offs = np.asarray(st.req_off_host)
        for r in range(min(3, len(offs) - 1)):
            s_r, l_r = sc[offs[r]:offs[r + 1]], slot[offs[r]:offs[r + 1]]
            keys = ~np.maximum(s_r[l_r >= 0], 0).astype(np.float32).view(np.uint32)
            kk = np.sort(keys)
            B = int(bud[r])
            if B <= 0 or B > len(kk):
                continue
            thr = kk[B - 1]
            c0 = int(((kk >> 23) == (thr >> 23)).sum())
            c1 = int(((kk >> 15) == (thr >> 15)).sum())
            print(f"step {i} req {r}: reused {len(kk)} B {B} c0 {c0} c1 {c1} "
                  f"score range {s_r[l_r >= 0].min():.3g}..{s_r[l_r >= 0].max():.3g}")
        eng.release(st)
    lib.kvs_sel_trace_dump(buf.ctypes.data, buf.size)
    tr = buf.reshape(1024, 8)[:148].astype(np.int64)
    t0 = tr[:, 0].min()
    names = ["start", "meta", "streamed", "sel_start", "sel_end", "keys", "radix", "pass0"]
    print(f"start spread {((tr[:, 0] - t0).max()) / 1e3:.2f} us")
    for ph in (1, 2, 3, 5, 7, 6, 4):
        v = tr[:, ph]
        v = v[v > 0] - t0
        if len(v):
            print(f"  {names[ph]:>9}: min {v.min() / 1e3:6.2f} med {np.median(v) / 1e3:6.2f} "
                  f"max {v.max() / 1e3:6.2f} us (n={len(v)})")


if __name__ == "__main__":
    main()
