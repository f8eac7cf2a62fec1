"""Multi-GPU: sharded KV pool and the remote-row fetch.

One process per GPU.  The token side of the pool is replicated (every rank
inserts every entry's tokens, ``CachePool.insert_remote`` for entries it does
not own), so every rank computes the same hit maps as the single-pool
reference (pool.py:125-161).  K/V payload stays on the GPU that wrote it.
After the lookup a rank splits its hit rows into local ones (G1 gather) and
remote ones, and fetches the latter in one grouped exchange:

  1. plan on the device: owner of every hit row, remote rows grouped by owner
     (a stable sort), per-peer counts; all_to_all of the counts;
  2. the only host round trip: the 2 x world counts, to size the transfers;
  3. all_to_all of the (owner slot, cached position) request lists;
  4. owners pack the rows (kvs_pack_rows: all layers, K and V); all_to_all
     of the packed rows; requesters unpack them into their pages with RoPE
     re-alignment (kvs_unpack_rows, a layer range at a time).

Steps 1-2 run on a fetch stream right after the lookup, so the host waits
only for the count exchange while the probe's layer 0 is already queued on
the main stream; steps 3-4 overlap the probe as well (engine.prefill_batch).
Collectives go through torch.distributed: NCCL over NVLink on a multi-GPU
box, gloo (staged through host memory) for the CPU tests and for the
two-ranks-on-one-GPU functional test.  Nothing else on the path
communicates.

PeerArenas is the peer-memory transport: every rank's KV arena is mapped into
every other rank's process once (CUDA IPC handles swapped through
torch.distributed), the token index carries each remote entry's page ids in
its owner's arena, and G1 (kvs_gather_kv_peer) reads remote rows straight from
the owner's memory - NVLink loads between GPUs - in the same launch that
gathers the local ones, with the RoPE re-alignment fused: no plan, count
exchange, pack, all-to-all or unpack, and no host round trip.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as N
from .errors import DeviceError


def plan_remote(src_slot: torch.Tensor, slot_owner: torch.Tensor, rank: int, world: int):
    """Flat positions whose hit lives on another rank, grouped by owner rank
    (ascending position within an owner), and the per-owner counts.
    ``slot_owner[s]`` is the owning rank of slot s (-1 = every rank holds it).
    Returns (order int64 [n] - the first counts.sum() entries are the remote
    rows -, counts int64 [world]).  Runs where the tensors live; no sync."""
    hit = src_slot >= 0
    own = torch.where(hit, slot_owner[src_slot.clamp(min=0).long()].to(torch.int64),
                      torch.full_like(src_slot, -1, dtype=torch.int64))
    remote = hit & (own >= 0) & (own != rank)
    key = torch.where(remote, own, torch.full_like(own, world))
    order = torch.sort(key, stable=True).indices
    counts = torch.bincount(key, minlength=world + 1)[:world]
    return order, counts


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group, staged: bool):
    """all_to_all_single; with gloo the payload is staged through host memory."""
    if not staged:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
        return out
    host_out = torch.empty(out.shape, dtype=out.dtype)
    dist.all_to_all_single(host_out, inp.cpu(), out_splits, in_splits, group=group)
    out.copy_(host_out)
    return out


class RemoteFetch:
    """One exchange in flight: start() plans and swaps the counts, finish()
    moves the rows and returns what unpack() needs."""

    def __init__(self, fetcher: "RemoteFetcher", src_slot, src_cand, idx):
        self.f, self.src_slot, self.src_cand, self.idx = fetcher, src_slot, src_cand, idx
        self.rows = self.flat_t = self.cand = None
        self.n_rows = 0

    def start(self):
        f = self.f
        self.order, send = plan_remote(self.src_slot, self.idx["slot_owner_dev"], f.rank, f.world)
        recv = torch.empty_like(send)
        _a2a(recv, send, None, None, f.group, f.staged)
        pair = torch.stack([send, recv])
        self._counts = torch.empty(pair.shape, dtype=pair.dtype, pin_memory=not f.staged)
        self._counts.copy_(pair, non_blocking=not f.staged)
        if not f.staged:
            self._ev = torch.cuda.Event()
            self._ev.record()
        return self

    def finish(self):
        f = self.f
        if not f.staged:
            self._ev.synchronize()                       # the one host round trip
        send, recv = (self._counts[0].tolist(), self._counts[1].tolist())
        n_need, n_give = int(sum(send)), int(sum(recv))
        dev = self.src_slot.device
        need = self.order[:n_need]
        on_owner = self.idx["slot_on_owner_dev"][self.src_slot[need].long()]
        req = torch.stack([on_owner, self.src_cand[need]], dim=1).to(torch.int32).contiguous()
        got = torch.empty((n_give, 2), dtype=torch.int32, device=dev)
        _a2a(got, req, recv, send, f.group, f.staged)
        packed = f.pack(got[:, 0].contiguous(), got[:, 1].contiguous(), self.idx)
        rows = torch.empty((n_need, f.row_elems), dtype=torch.bfloat16, device=dev)
        _a2a(rows, packed, send, recv, f.group, f.staged)
        self.rows, self.flat_t, self.cand = rows, need.contiguous(), self.src_cand[need].contiguous()
        self.n_rows = n_need
        return self

    def unpack(self, st, layers, skip=None):
        """Remote rows' layers [begin, end) into the request pages; rows with
        skip[flat_t] set (e.g. DHD-selected positions) are left alone."""
        if self.n_rows == 0:
            return
        eng = self.f.engine
        N.call("kvs_unpack_rows", eng.arena.c, st.batch_c, self.flat_t.data_ptr(),
               self.cand.data_ptr(), self.n_rows, self.rows.data_ptr(), eng._rope(), layers[0],
               layers[1], N.ptr(skip), N.stream_ptr())


class RemoteFetcher:
    """Engine hook: local rows via G1, remote rows via RemoteFetch."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) == "gloo"
        cfg = engine.cfg
        self.row_elems = cfg.num_layers * 2 * cfg.kv_heads * 128

    def local_mask(self, src_slot: torch.Tensor, idx) -> torch.Tensor:
        owner = idx["slot_owner_dev"]
        s = src_slot.clamp(min=0).long()
        local = (src_slot >= 0) & ((owner[s] < 0) | (owner[s] == self.rank))
        return torch.where(local, src_slot, torch.full_like(src_slot, -1))

    def pack(self, slots: torch.Tensor, cands: torch.Tensor, idx) -> torch.Tensor:
        eng = self.engine
        out = torch.empty((slots.numel(), self.row_elems), dtype=torch.bfloat16,
                          device=eng.device)
        N.call("kvs_pack_rows", eng.arena.c, slots.data_ptr(), cands.data_ptr(), slots.numel(),
               idx["slot_pages"].data_ptr(), idx["slot_max_pages"], out.data_ptr(),
               N.stream_ptr())
        return out

    def begin(self, st, idx) -> RemoteFetch:
        return RemoteFetch(self, st.src_slot, st.src_cand, idx).start()

    def fetch(self, st, idx, layers=None) -> int:
        """Whole exchange and unpack of layers [begin, end) on the current
        stream (the plain, non-overlapped path)."""
        rf = self.begin(st, idx).finish()
        rf.unpack(st, layers or (0, self.engine.cfg.num_layers))
        return rf.n_rows


class PeerArenas:
    """Peer-memory transport (see the module docstring).  Construct on every
    rank (collective); keeps the mapped peer storages alive."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        data = engine.arena.data
        stor = data.untyped_storage()
        share = stor._share_cuda_()           # (device, handle, size, offset, refcount..., event...)
        off = data.data_ptr() - stor.data_ptr()
        infos = [None] * self.world
        dist.all_gather_object(infos, (share, off), group=group)
        self._mapped = []
        bases = []
        for r, (sh, o) in enumerate(infos):
            if r == self.rank:
                bases.append(data.data_ptr())
                continue
            s = torch.UntypedStorage._new_shared_cuda(*sh)
            self._mapped.append(s)
            bases.append(s.data_ptr() + o)
        # uint64 addresses carried in an int64 tensor (the kernel reads the bits)
        self.peer_base = torch.tensor([b if b < (1 << 63) else b - (1 << 64) for b in bases],
                                      dtype=torch.int64, device=engine.device)

    def close(self):
        """Drop the peer mappings (before the owners' processes exit)."""
        self._mapped.clear()
        self.peer_base = None

    def gather(self, st, idx, slot, layers):
        """G1 for layers [begin, end) over local and remote slots in one launch."""
        if self.peer_base is None:
            raise DeviceError("PeerArenas.gather after close()")
        eng = self.engine
        owner = idx["slot_owner_dev"]              # int32 per slot (-1: local), rebuilt with idx
        N.call("kvs_gather_kv_peer", eng.arena.c, st.batch_c, slot.data_ptr(),
               st.src_cand.data_ptr(), idx["slot_pages"].data_ptr(), idx["slot_max_pages"],
               owner.data_ptr(), self.peer_base.data_ptr(), layers[0], layers[1], eng._rope(),
               N.stream_ptr())


def share_entry_pages(pool, ids_pages: dict, group=None) -> dict:
    """All-gather {request_id: page ids} of the entries each rank owns, so
    every rank can register the others' entries with their pages."""
    world = dist.get_world_size(group)
    got = [None] * world
    dist.all_gather_object(got, dict(ids_pages), group=group)
    out = {}
    for r, d in enumerate(got):
        for rid, pages in d.items():
            out[rid] = (r, list(pages))
    return out
