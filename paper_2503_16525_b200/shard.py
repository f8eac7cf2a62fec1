"""Multi-GPU: sharded KV pool and the remote-row fetch.

One process per GPU.  The token side of the pool is replicated (every rank
inserts every entry's tokens, ``CachePool.insert_remote`` for entries it does
not own), so every rank computes the same hit maps as the single-pool
reference (pool.py:125-161).  K/V payload stays on the GPU that wrote it.
After the lookup a rank splits its hit rows into local ones (G1 gather) and
remote ones, and fetches the latter in one grouped exchange:

  1. all_to_all of per-peer row counts;
  2. send (slot, cand) request lists to the owners;
  3. owners pack the rows (kvs_pack_rows: all layers, K and V) and send
     them back; receivers unpack into their pages with RoPE re-alignment
     (kvs_unpack_rows).

Point-to-point ops go through torch.distributed (NCCL over NVLink on the
GPU box; gloo for the CPU tests of the planning and the exchange pattern).
Nothing else on the path communicates.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N


def plan_remote_rows(src_slot: np.ndarray, slot_owner: np.ndarray, rank: int, world: int):
    """Flat positions whose hit lives on another rank, grouped by owner.
    ``slot_owner[s]`` is the owning rank (or -1 for this rank)."""
    need = [np.zeros(0, dtype=np.int64) for _ in range(world)]
    hit = np.nonzero(src_slot >= 0)[0]
    if hit.size == 0:
        return need
    own = slot_owner[src_slot[hit]]
    own = np.where(own < 0, rank, own)
    for q in range(world):
        if q != rank:
            need[q] = hit[own == q].astype(np.int64)
    return need


def exchange_rows(need, src_slot, src_cand, pack_fn, unpack_fn, rank: int, world: int,
                  row_elems: int, dtype, device, group=None) -> int:
    """Run the three-phase exchange; returns the number of rows received.
    ``src_slot`` must already be in the owners' slot numbering.  With the gloo
    backend the payloads are staged through host memory (CPU tests and the
    single-GPU functional run); with NCCL they move GPU to GPU."""
    staged = dist.get_backend(group) == "gloo"
    comm = torch.device("cpu") if staged else device
    send_counts = torch.tensor([len(need[q]) for q in range(world)], dtype=torch.int64,
                               device=comm)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    recv_counts = recv_counts.cpu().numpy()
    # phase 2: request lists (slot, cand) to the owners
    ops, req_in = [], {}
    for q in range(world):
        if q == rank:
            continue
        if len(need[q]):
            t = need[q]
            lst = torch.from_numpy(np.stack([src_slot[t], src_cand[t]], 1).astype(np.int32))
            ops.append(dist.P2POp(dist.isend, lst.to(comm).contiguous(), q, group))
        if recv_counts[q]:
            req_in[q] = torch.empty((int(recv_counts[q]), 2), dtype=torch.int32, device=comm)
            ops.append(dist.P2POp(dist.irecv, req_in[q], q, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    # phase 3: owners pack and send rows back; requesters receive and unpack
    ops, rows_in = [], {}
    for q, lst in req_in.items():
        lst = lst.to(device)
        packed = pack_fn(lst[:, 0].contiguous(), lst[:, 1].contiguous())
        ops.append(dist.P2POp(dist.isend, packed.to(comm), q, group))
    for q in range(world):
        if q != rank and len(need[q]):
            rows_in[q] = torch.empty((len(need[q]), row_elems), dtype=dtype, device=comm)
            ops.append(dist.P2POp(dist.irecv, rows_in[q], q, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    got = 0
    for q, buf in rows_in.items():
        t = need[q]
        unpack_fn(torch.from_numpy(t).to(device), torch.from_numpy(src_cand[t].astype(np.int32))
                  .to(device), buf.to(device))
        got += len(t)
    return got


class RemoteFetcher:
    """Engine hook: local rows via G1, remote rows via exchange_rows."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        cfg = engine.cfg
        self.row_elems = cfg.num_layers * 2 * cfg.kv_heads * 128

    def local_mask(self, src_slot: torch.Tensor, idx) -> torch.Tensor:
        owner = idx["slot_owner_dev"]
        s = src_slot.clamp(min=0).long()
        local = (src_slot >= 0) & ((owner[s] < 0) | (owner[s] == self.rank))
        return torch.where(local, src_slot, torch.full_like(src_slot, -1))

    def fetch(self, st, idx) -> int:
        eng = self.engine
        src = st.src_slot.cpu().numpy()
        cand = st.src_cand.cpu().numpy()
        need = plan_remote_rows(src, idx["slot_owner"], self.rank, self.world)
        on_owner = np.where(src >= 0, idx["slot_on_owner"][np.maximum(src, 0)], -1)
        arena = eng.arena

        def pack(slots, cands):
            out = torch.empty((slots.numel(), self.row_elems), dtype=torch.bfloat16,
                              device=eng.device)
            N.call("kvs_pack_rows", arena.c, slots.data_ptr(), cands.data_ptr(), slots.numel(),
                   idx["slot_pages"].data_ptr(), idx["slot_max_pages"], out.data_ptr(),
                   N.stream_ptr())
            return out

        def unpack(flat_t, cands, buf):
            N.call("kvs_unpack_rows", arena.c, st.batch_c, flat_t.data_ptr(), cands.data_ptr(),
                   flat_t.numel(), buf.data_ptr(), eng._rope(), N.stream_ptr())

        return exchange_rows(need, on_owner, cand, pack, unpack, self.rank, self.world,
                             self.row_elems, torch.bfloat16, eng.device, self.group)
