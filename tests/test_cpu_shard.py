"""World-size-2 gloo tests of the multi-GPU host logic: remote-row planning
and the three-phase row exchange (counts, request lists, packed rows)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_16525_b200.shard import exchange_rows, plan_remote_rows

ROW = 6


def _row_value(owner, slot, cand):
    return np.array([owner, slot, cand, owner * 1000 + slot * 10 + cand, -1, 7], np.float32)


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    n_slots = 6
    slot_owner = np.array([0, 1, 0, 1, -1, 1], dtype=np.int32)   # -1: local to everyone
    n = 50
    src_slot = rng.integers(-1, n_slots, n).astype(np.int32)
    src_cand = rng.integers(0, 40, n).astype(np.int32)
    need = plan_remote_rows(src_slot, slot_owner, rank, world)
    received = {}

    def pack(slots, cands):
        rows = [_row_value(rank, int(s), int(c)) for s, c in zip(slots.tolist(), cands.tolist())]
        return torch.from_numpy(np.stack(rows)) if rows else torch.zeros((0, ROW))

    def unpack(flat_t, cands, buf):
        for t, c, row in zip(flat_t.tolist(), cands.tolist(), buf.numpy()):
            received[t] = row.copy()

    got = exchange_rows(need, src_slot, src_cand, pack, unpack, rank, world, ROW,
                        torch.float32, torch.device("cpu"))
    expect = {}
    for t in range(n):
        s = src_slot[t]
        if s >= 0 and slot_owner[s] >= 0 and slot_owner[s] != rank:
            expect[t] = _row_value(slot_owner[s], s, src_cand[t])
    ok = got == len(expect) and set(received) == set(expect) and \
        all(np.array_equal(received[t], expect[t]) for t in expect)
    results[rank] = bool(ok)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_remote_rows():
    src = np.array([-1, 0, 1, 2, 3, -1, 1], dtype=np.int32)
    owner = np.array([0, 1, -1, 2], dtype=np.int32)
    need = plan_remote_rows(src, owner, rank=0, world=3)
    assert need[0].tolist() == [] and need[1].tolist() == [2, 6] and need[2].tolist() == [4]
    need = plan_remote_rows(src, owner, rank=1, world=3)
    assert need[0].tolist() == [1] and need[1].tolist() == [] and need[2].tolist() == [4]


def test_exchange_rows_world2_gloo():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert results[0] and results[1]
