"""World-size-2 gloo tests of the multi-GPU host logic: the
device-side remote-row planning (run here on CPU tensors), the grouped
exchange (counts, request lists, packed rows) through RemoteFetch with the
kernels replaced by host fakes, and the scheduler's partition of a batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_16525_b200.shard import RemoteFetch, RemoteFetcher, plan_remote

ROW = 6


def _row_value(owner, slot, cand):
    return np.array([owner, slot, cand, owner * 1000 + slot * 10 + cand, -1, 7], np.float32)


class _FakeEngine:
    class cfg:
        num_layers = 1
        kv_heads = 1


class _FakeFetcher(RemoteFetcher):
    """RemoteFetcher with the pack kernel replaced by a host function that
    encodes (owner rank, owner slot, cached position) into the row."""

    def __init__(self):
        super().__init__(_FakeEngine())
        self.row_elems = ROW

    def pack(self, slots, cands, idx):
        rows = [_row_value(self.rank, int(s), int(c))
                for s, c in zip(slots.tolist(), cands.tolist())]
        return torch.from_numpy(np.stack(rows)).to(torch.bfloat16) if rows else \
            torch.zeros((0, ROW), dtype=torch.bfloat16)


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    n_slots = 6
    slot_owner = torch.tensor([0, 1, 0, 1, -1, 1], dtype=torch.int32)   # -1: every rank holds it
    on_owner = torch.tensor([10, 11, 12, 13, 14, 15], dtype=torch.int32)  # owners' numbering
    n = 50
    src_slot = torch.from_numpy(rng.integers(-1, n_slots, n).astype(np.int32))
    src_cand = torch.from_numpy(rng.integers(0, 40, n).astype(np.int32))
    idx = {"slot_owner_dev": slot_owner, "slot_on_owner_dev": on_owner}
    rf = RemoteFetch(_FakeFetcher(), src_slot, src_cand, idx).start().finish()
    expect = {}
    for t in range(n):
        s = int(src_slot[t])
        if s >= 0 and int(slot_owner[s]) >= 0 and int(slot_owner[s]) != rank:
            expect[t] = torch.from_numpy(_row_value(int(slot_owner[s]), int(on_owner[s]),
                                                    int(src_cand[t]))).to(torch.bfloat16).float().numpy()
    got = {int(t): row.float().numpy() for t, row in zip(rf.flat_t, rf.rows)}
    ok = rf.n_rows == len(expect) and set(got) == set(expect) and \
        all(np.array_equal(got[t], expect[t]) for t in expect) and \
        rf.cand.tolist() == [int(src_cand[t]) for t in rf.flat_t.tolist()]
    results[rank] = bool(ok)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_remote_groups_by_owner():
    src = torch.tensor([-1, 0, 1, 2, 3, -1, 1, 3], dtype=torch.int32)
    owner = torch.tensor([0, 1, -1, 2], dtype=torch.int32)
    order, counts = plan_remote(src, owner, rank=0, world=3)
    assert counts.tolist() == [0, 2, 2]
    assert order[:4].tolist() == [2, 6, 4, 7]            # owner 1 first, ascending positions
    order, counts = plan_remote(src, owner, rank=1, world=3)
    assert counts.tolist() == [1, 0, 2] and order[:3].tolist() == [1, 4, 7]


def test_exchange_world2_gloo():
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


def test_partition_batch_prefers_owner_and_balances():
    from paper_2503_16525_b200.scheduling import Batch, Request, partition_batch
    reqs = [Request(f"r{i}", 0.0, [1] * 100, 0, 0.5) for i in range(8)]
    owner = [[90, 0], [90, 0], [90, 0], [90, 0], [0, 90], [0, 90], [0, 90], [0, 90]]
    parts = partition_batch(Batch(reqs), 2, owner)
    assert parts == [[0, 1, 2, 3], [4, 5, 6, 7]]
    skew = [[90, 0]] * 8                                  # every hit on rank 0: balance wins
    parts = partition_batch(Batch(reqs), 2, skew)
    assert sorted(len(p) for p in parts) == [3, 5] or sorted(len(p) for p in parts) == [4, 4]
    assert sorted(parts[0] + parts[1]) == list(range(8))
