"""Diagnostic: item-boundary timeline of the persistent A1 kernel (fwdp).
Builds libkvshare with KVS_ATTN_TRACE, runs one launch of equal-length items
(n_kb key blocks each, tools/micro_attn_overhead.py's case) and prints CTA
0's events in microseconds (clock64 / SM clock).

    python tools/attn_trace_p.py [n_kb]
"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
LIB = "/tmp/libkvshare_trace.so"
from paper_2503_16525_b200 import build as B  # noqa: E402

objs = []
for src in B.SOURCES:
    o = f"/tmp/trace_{src}.o"
    subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, "-DKVS_ATTN_TRACE", "-c",
                           os.path.join(B.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static"])
from paper_2503_16525_b200 import _native as N  # noqa: E402
N.LIB_PATH = LIB
lib = N.load()
lib.kvs_attn_trace_dump.restype = ctypes.c_int32
lib.kvs_attn_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_int32]
from attn_case import build_case  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "4"
H, G = 32, 8
if arg == "real":
    # the bench's DHD row set shape: 8 x 4096 tokens, 60% of positions
    n_kb = 0
    eng, st, rows, q, layer = build_case(8, 4096, H, G, 0.6, seed=1, rope_theta=5e5)
else:
    n_kb = int(arg)
    reqs = 74
    eng, st, rows, q, layer = build_case(reqs, 128 * n_kb, H, G, 1.0, seed=1, rope_theta=5e5)
    last0 = torch.tensor([int(rows.row_off[r + 1]) - 128 for r in range(reqs)],
                         dtype=torch.int32, device="cuda")
    rows.tiles = torch.stack([torch.arange(reqs, dtype=torch.int32, device="cuda"), last0,
                              torch.full((reqs,), 128, dtype=torch.int32,
                                         device="cuda")]).contiguous()
    rows.n_tiles = reqs
qkv = torch.randn(rows.n_rows, (H + 2 * G) * 128, device="cuda").to(torch.bfloat16)
o = torch.empty(rows.n_rows, H, 128, dtype=torch.bfloat16, device="cuda")
fused = os.environ.get("FUSED", "0") == "1"
run = (lambda: eng._attention_qkv(qkv, rows, layer, eng.arena.c, st.batch_c, o)) if fused else \
      (lambda: eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o))
buf = np.zeros(2 * 16384, dtype=np.int64)
run()
torch.cuda.synchronize()
lib.kvs_attn_trace_dump(buf.ctypes.data, 16384)
run()
torch.cuda.synchronize()
k = lib.kvs_attn_trace_dump(buf.ctypes.data, 16384)
ev = buf[:2 * k].reshape(-1, 2)
ev = ev[np.argsort(ev[:, 0], kind="stable")]
mhz = 1.0e3 * float(os.environ.get("SM_GHZ", "1.9"))
t0 = ev[0, 0]
names = {1: "prod: Q_a issue (item)", 2: "prod: Q_b issue (item)", 3: "mma: item start, K ready",
         4: "mma: Q_a ready -> QK_a(0)", 5: "mma: Q_b ready -> QK_b(0)",
         6: "mma: PV_a issue (blk)", 7: "mma: PV_b issue (blk)",
         20: "smx a: S ready (blk)", 22: "smx a: P done (blk)", 25: "smx a: epi start (item)",
         26: "smx a: pv_done (item)", 27: "smx a: epi end (item)",
         30: "smx b: S ready (blk)", 32: "smx b: P done (blk)", 35: "smx b: epi start (item)",
         36: "smx b: pv_done (item)", 37: "smx b: epi end (item)"}
print(f"n_kb={n_kb} fused={fused}: CTA 0 events, us from its first event (SM clock {mhz:.0f} MHz)")
for t, tag in ev:
    tg, idx = int(tag) >> 32, int(tag) & 0xffffffff
    print(f"{(t - t0) / mhz:9.3f}  {names.get(tg, tg)} #{idx}")
