"""Diagnostic: build libkvshare with KVS_ATTN_TRACE, run one Llama-shape
session-layer attention launch and print the first CTA's pipeline timeline."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
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

import paper_2503_16525_b200 as K  # noqa: E402
from paper_2503_16525_b200.engine import Engine, RowSet  # noqa: E402
from paper_2503_16525_b200.pool import CachePool, KVArena  # noqa: E402

cfg = K.ModelConfig(num_layers=1, num_heads=32, num_kv_heads=8, d_model=4096, vocab_size=1000,
                    rope_theta=500000.0, max_positions=8192)
model = K.ToyModel(cfg, init="device")
arena = KVArena(cfg, 80)
eng = Engine(model, CachePool(cfg, arena=arena))
n = 4096
st = eng.new_batch([np.arange(n) % 1000])
arena.data.normal_()
rows = eng._rows_all(st)
q = torch.randn(n, 32, 128, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
eng._attention(q, rows, 0, arena.c, st.batch_c, o)
torch.cuda.synchronize()
lib.kvs_attn_trace_dump(None, 0) if False else None
buf = np.zeros(2 * 4096, dtype=np.int64)
lib.kvs_attn_trace_dump(buf.ctypes.data, 4096)                  # clear the warm-up run
eng._attention(q, rows, 0, arena.c, st.batch_c, o)
torch.cuda.synchronize()
k = lib.kvs_attn_trace_dump(buf.ctypes.data, 4096)
ev = buf[:2 * k].reshape(-1, 2)
ev = ev[np.argsort(ev[:, 0])]
t0 = ev[0, 0]
names = {10: "mma:V ready", 11: "mma:p_full a -> PV_a", 12: "mma:p_full b -> PV_b",
         13: "mma:QK_a issue", 14: "mma:QK_b issue", 20: "smx a: S ready", 21: "smx a: S loaded",
         22: "smx a: P stored", 30: "smx b: S ready", 31: "smx b: S loaded", 32: "smx b: P stored"}
print("longest tile (n_kb = 32), head pair 0; clock64 cycles")
T = {}
for t, tag in ev:
    T.setdefault((int(tag >> 32), int(tag & 0xffffffff)), int(t - t0))
for t, tag in ev[:60]:
    print(f"{t - t0:8d}  kb={tag & 0xffffffff:3d}  {names.get(int(tag >> 32), tag >> 32)}")
kbs = sorted({kb for (_, kb) in T})
mid = [kb for kb in kbs if 4 <= kb <= kbs[-1] - 4]
def avg(f):
    v = [f(kb) for kb in mid]
    v = [x for x in v if x is not None]
    return sum(v) / max(len(v), 1)
g = lambda a, kb: T.get((a, kb))
def d(a, ka, b, kb_):
    return lambda kb: (g(b, kb + kb_) - g(a, kb + ka)) if g(b, kb + kb_) is not None and g(a, kb + ka) is not None else None
print(f"period per kb (S ready a -> next S ready a): {avg(d(20, 0, 20, 1)):.0f}")
print(f"softmax a: S ready -> S loaded {avg(d(20, 0, 21, 0)):.0f}, S loaded -> P stored {avg(d(21, 0, 22, 0)):.0f}, P stored -> next S ready {avg(d(22, 0, 20, 1)):.0f}")
print(f"softmax b: S ready -> S loaded {avg(d(30, 0, 31, 0)):.0f}, S loaded -> P stored {avg(d(31, 0, 32, 0)):.0f}, P stored -> next S ready {avg(d(32, 0, 30, 1)):.0f}")
print(f"P stored a -> mma sees p_full a {avg(d(22, 0, 11, 0)):.0f}; p_full a -> QK_a issue {avg(d(11, 0, 13, 0)):.0f}; QK_a issue -> S ready a(kb+1) {avg(d(13, 0, 20, 1)):.0f}")
print(f"P stored b -> mma sees p_full b {avg(d(32, 0, 12, 0)):.0f}; p_full b -> QK_b issue {avg(d(12, 0, 14, 0)):.0f}; QK_b issue -> S ready b(kb+1) {avg(d(14, 0, 30, 1)):.0f}")
print(f"softmax a start vs b start offset: {avg(d(20, 0, 30, 0)):.0f}")
for t, base in (("a", 20), ("b", 30)):
    print(f"softmax {t}: loaded->max done {avg(d(base + 1, 0, base + 3, 0)):.0f}, "
          f"max->exp start {avg(d(base + 3, 0, base + 4, 0)):.0f}, "
          f"exp phase {avg(d(base + 4, 0, base + 5, 0)):.0f}, "
          f"exp end->P stored(wait st) {avg(d(base + 5, 0, base + 2, 0)):.0f}")
