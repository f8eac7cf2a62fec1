"""Per-GPU shared KV pool: paged bf16 KV arena + replicated token index.

Mirrors reference pkg/src/kvlab/pool.py: ``KVEntry`` (:35-55), ``ReuseMap``
(:58-75) and ``CachePool`` (:78-172) keep their names, arguments and error
behaviour.  What changes is where things live:

* K/V rows live in one paged bf16 arena on the GPU (``KVArena``); an entry is
  a list of pages (64 tokens each, layout in include/kvshare.h).  Request
  caches use the same arena, so writing a finished request back to the pool
  is zero-copy (``insert_pages``).
* The token side (entry tokens, window hashes, a hash-sorted window list and
  the recency ranks) is a device index queried by the R2 lookup kernel
  (``kvs_pool_lookup``) for a whole scheduled batch at once.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import CacheError, FormatError, InputError, ParameterError
from .matching import HashParams, window_hashes_device
from .model import HEAD_DIM, ModelConfig

PAGE_SIZE = 64
MAX_SEQ = 1 << 21          # R2 packs positions into 21-bit fields (csrc/retriever.cu)
_MAGIC = b"KVSH"          # pool file format of reference pool.py:8-17
_VERSION = 1


class KVArena:
    """Paged KV storage [pages][L][2][64][kv_heads][128] bf16 with a free list."""

    def __init__(self, config: ModelConfig, num_pages: int, device="cuda",
                 page_size: int = PAGE_SIZE):
        self.config = config
        self.page_size = page_size
        self.device = torch.device(device)
        self.data = torch.zeros(num_pages, config.num_layers, 2, page_size, config.kv_heads,
                                HEAD_DIM, dtype=torch.bfloat16, device=self.device)
        self._free = list(range(num_pages - 1, -1, -1))
        self.c = N.KVArena(self.data.data_ptr(), num_pages, config.num_layers, config.kv_heads,
                           HEAD_DIM, page_size)

    @property
    def num_pages(self) -> int:
        return self.data.shape[0]

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def pages_for(self, n_tokens: int) -> int:
        return (n_tokens + self.page_size - 1) // self.page_size

    def alloc(self, n: int) -> list[int]:
        if n > len(self._free):
            raise CacheError(f"KV arena exhausted: need {n} pages, {len(self._free)} free")
        return [self._free.pop() for _ in range(n)]

    def release(self, pages) -> None:
        self._free.extend(int(p) for p in pages)

    @staticmethod
    def bytes_per_page(config: ModelConfig, page_size: int = PAGE_SIZE) -> int:
        return config.num_layers * 2 * page_size * config.kv_heads * HEAD_DIM * 2

    def rows(self, pages, n: int, layer: int, kv: int) -> torch.Tensor:
        """Gather rows [0, n) of a page list at (layer, kv): [n, kv_heads, 128]."""
        p = torch.as_tensor(list(pages), device=self.device, dtype=torch.long)
        x = self.data[p, layer, kv]  # [pages, 64, G, 128]
        return x.reshape(-1, self.config.kv_heads, HEAD_DIM)[:n]


@dataclass
class KVEntry:
    """One cached request (pool.py:35-55): tokens plus its arena pages."""

    request_id: str
    tokens: np.ndarray
    pages: list
    pool: "CachePool" = field(repr=False)
    slot: int = -1
    last_access: int = 0
    insert_seq: int = 0
    owner: int = -1          # GPU rank holding the K/V pages (-1 = this GPU)
    owner_slot: int = -1     # the entry's slot id on its owner (remote entries)
    remote_pages: list = field(default_factory=list)   # the owner's page ids (peer memory)

    @property
    def n_tokens(self) -> int:
        return int(self.tokens.size)

    @property
    def size_bytes(self) -> int:
        """Serialized (KVSH) size, pool.py:51-55."""
        cfg = self.pool.config
        return (4 + len(self.request_id.encode()) + 4 + 4 * self.n_tokens + 12
                + 2 * 4 * cfg.num_layers * cfg.kv_heads * self.n_tokens * cfg.d_k)

    @property
    def live(self) -> bool:
        """Still in its pool: its slot and pages have not been handed on."""
        s = self.pool._slots
        return 0 <= self.slot < len(s) and s[self.slot] is self

    def check_live(self) -> None:
        """Raise CacheError for an evicted or replaced entry, whose slot and
        arena pages may already belong to another entry (a stale ReuseMap)."""
        if not self.live:
            raise CacheError(f"entry {self.request_id!r} is no longer in the pool "
                             "(evicted or replaced)")

    def export_f32(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Device fp32 K and V in KVSH order [L][n][kv_heads][d_k] (F3 kernel)."""
        self.check_live()
        if self.owner >= 0:
            raise CacheError(f"entry {self.request_id!r} lives on GPU {self.owner}")
        cfg, dev = self.pool.config, self.pool.device
        shape = (cfg.num_layers, self.n_tokens, cfg.kv_heads, cfg.d_k)
        k = torch.empty(shape, dtype=torch.float32, device=dev)
        v = torch.empty(shape, dtype=torch.float32, device=dev)
        pages = torch.as_tensor(np.asarray(self.pages, dtype=np.int32), device=dev)
        N.call("kvs_entry_export", self.pool.arena.c, pages.data_ptr(), self.n_tokens, cfg.d_k,
               k.data_ptr(), v.data_ptr(), N.stream_ptr())
        return k, v

    def _kv(self, kv: int) -> np.ndarray:
        x = self.export_f32()[kv]                                     # L, n, G, d_k
        return x.permute(0, 2, 1, 3).double().cpu().numpy()          # (L, G, n, d_k)

    @property
    def k(self) -> np.ndarray:
        return self._kv(0)

    @property
    def v(self) -> np.ndarray:
        return self._kv(1)

    @property
    def window_hash_set(self) -> frozenset:
        h = self.pool._slot_hash[self.slot]
        return frozenset(int(x) for x in h.cpu().numpy()) if h is not None else frozenset()


@dataclass
class ReuseMap:
    """Alignment of a request's positions onto cached K/V rows (pool.py:58-75).

    ``sources`` is the reference's ``{pos: (KVEntry, cand_pos)}``; the device
    form (``src_slot``/``src_cand``, int32 per position) is what the engine
    consumes without leaving the GPU."""

    length: int
    sources: dict = field(default_factory=dict)
    src_slot: torch.Tensor | None = None
    src_cand: torch.Tensor | None = None

    @property
    def hit_rate(self) -> float:
        return len(self.sources) / self.length if self.length else 0.0

    def validate(self, tokens) -> None:
        tokens = np.asarray(tokens, dtype=np.int64)
        for pos, (entry, cand_pos) in self.sources.items():
            if tokens[pos] != entry.tokens[cand_pos]:
                raise CacheError(f"reuse map position {pos} maps to a different token")


@dataclass
class AdmittedHits:
    """A request's admission-time device hit map (CachePool.admit); its
    source slots stay pinned in the pool until release()."""

    pool: "CachePool" = field(repr=False)
    length: int
    n_hit: int
    src_slot: torch.Tensor         # int32 [length], -1 = miss
    src_cand: torch.Tensor         # int32 [length]
    slots: list

    @property
    def hit_rate(self) -> float:
        return self.n_hit / self.length if self.length else 0.0

    def release(self) -> None:
        if self.slots is not None:
            self.pool.unpin(self.slots)
            self.slots = None


@dataclass
class BatchLookup:
    """Device hit maps of a batched lookup (flat over the batch)."""

    req_off: torch.Tensor          # int64 [R+1]
    tokens: torch.Tensor           # int64 [n_total]
    src_slot: torch.Tensor         # int32 [n_total]
    src_cand: torch.Tensor         # int32 [n_total]
    n_hit: torch.Tensor            # int32 [R] (device)
    contributed: torch.Tensor      # uint8 [R, n_slots]


class CachePool:
    """KV entries indexed by content; most-recent insertion wins (pool.py:78-172)."""

    def __init__(self, config: ModelConfig, params: HashParams | None = None,
                 capacity_bytes: int | None = None, *, arena: KVArena | None = None,
                 arena_pages: int | None = None, device="cuda"):
        self.config = config
        self.params = params or HashParams()
        self.capacity_bytes = capacity_bytes
        self.device = torch.device(device)
        if arena is None:
            arena = KVArena(config, arena_pages or 256, device)
        self.arena = arena
        from .model import _pad_index
        self.pad_index = _pad_index(config.d_k)
        self.entries: dict[str, KVEntry] = {}
        self._counter = 0
        self._slots: list[KVEntry | None] = []
        self._slot_tokens: list[torch.Tensor | None] = []
        self._slot_hash: list[torch.Tensor | None] = []
        self._dirty = True
        self._index = None
        self._tidx = None
        self._ws = N.Workspace()
        self._pins: dict[int, int] = {}           # slot -> holders of a device hit map
        self._retired: dict[int, KVEntry] = {}    # dropped while pinned: pages kept

    # ------------------------------------------------------------------ basics
    def __len__(self) -> int:
        return len(self.entries)

    @property
    def total_bytes(self) -> int:
        return sum(e.size_bytes for e in self.entries.values())

    def _tick(self) -> int:
        self._counter += 1
        return self._counter

    def _validate_tokens(self, tokens) -> np.ndarray:
        tokens = np.asarray(tokens, dtype=np.int64)
        if tokens.ndim != 1 or tokens.size == 0:
            raise CacheError("entry tokens must be a non-empty 1-D sequence")
        if tokens.min() < 0 or tokens.max() >= 2**32:
            raise CacheError("token ids must fit an unsigned 32-bit integer")
        if tokens.size >= MAX_SEQ:
            raise ParameterError(f"entries of {MAX_SEQ} tokens or more are not supported")
        return tokens

    # ------------------------------------------------------------------ insert
    def _new_slot(self) -> int:
        """Slots are append-only (a freed slot is never handed out again), so
        the device index only ever appends; _compact() reclaims them."""
        self._slots.append(None)
        self._slot_tokens.append(None)
        self._slot_hash.append(None)
        return len(self._slots) - 1

    def _drop(self, entry: KVEntry, release: bool = True) -> None:
        self.entries.pop(entry.request_id, None)
        self._slots[entry.slot] = None
        self._slot_tokens[entry.slot] = None
        self._slot_hash[entry.slot] = None
        if self._pins.get(entry.slot):
            # a held hit map still gathers from this slot (the reference's
            # ReuseMap keeps a dropped entry's arrays alive): lookups no longer
            # see it, its slot id and pages stay reserved until unpin()
            self._retired[entry.slot] = entry
            entry._release_pages = release
        elif release and entry.owner < 0:
            self.arena.release(entry.pages)
        self._dirty = True

    def pin(self, slots) -> None:
        """Hold slots referenced by a device hit map (admission-time lookup,
        simulate.py:180-186) so that eviction or replacement before the batch
        runs (simulate.py:165-171) cannot hand their ids or pages on."""
        for s in slots:
            s = int(s)
            self._pins[s] = self._pins.get(s, 0) + 1

    def unpin(self, slots) -> None:
        for s in slots:
            s = int(s)
            c = self._pins.get(s, 0) - 1
            if c > 0:
                self._pins[s] = c
                continue
            self._pins.pop(s, None)
            entry = self._retired.pop(s, None)
            if entry is not None:
                if entry._release_pages and entry.owner < 0:
                    self.arena.release(entry.pages)
                self._dirty = True
        if not self._pins:
            self._maybe_renumber()

    def insert_remote(self, request_id: str, tokens, owner: int,
                      owner_slot: int | None = None, pages=None) -> KVEntry:
        """Replicate the token side of an entry whose K/V pages live on GPU
        ``owner`` in its slot ``owner_slot`` (sharded pool).
        Lookups see it like any other entry; its rows are fetched from the
        owner by shard.RemoteFetcher.  ``owner_slot`` defaults to this pool's
        slot, which is the owner's too when every rank inserts in one order
        (slot ids are append-only and sharded pools never evict or renumber).
        ``pages``: the entry's page ids in the owner's arena, for G1 reading
        them through peer memory (shard.PeerArenas)."""
        if self.capacity_bytes is not None:
            # every rank evicts on its own LRU: victims (and slot ids) would
            # diverge between the ranks that share this entry's owner slot
            raise ParameterError("a sharded pool cannot use capacity_bytes")
        entry = self.insert_pages(request_id, tokens, [])
        entry.owner = int(owner)
        entry.owner_slot = entry.slot if owner_slot is None else int(owner_slot)
        entry.remote_pages = [] if pages is None else [int(x) for x in pages]
        self._dirty = True
        return entry

    def insert_pages(self, request_id: str, tokens, pages) -> KVEntry:
        """Register K/V already resident in arena pages (zero-copy write-back
        of a finished request, simulate.py:207-210)."""
        tokens = self._validate_tokens(tokens)
        old = self.entries.get(request_id)
        if old is not None:
            self._drop(old, release=set(old.pages) != set(pages))
        seq = self._tick()
        slot = self._new_slot()
        entry = KVEntry(request_id, tokens.copy(), list(pages), self, slot, seq, seq)
        tok_dev = torch.from_numpy(tokens).to(self.device)
        self._slots[slot] = entry
        self._slot_tokens[slot] = tok_dev
        self._slot_hash[slot] = window_hashes_device(tok_dev, self.params)
        self.entries[request_id] = entry
        self._dirty = True
        if self.capacity_bytes is not None:
            self.evict_to_capacity(self.capacity_bytes)
        self._maybe_renumber()
        return entry

    def insert(self, request_id: str, tokens, k, v) -> None:
        """pool.py:100-123: store host K/V (L, kv_heads, n, d_k); replaces any
        entry with the same id."""
        cfg = self.config
        tokens = self._validate_tokens(tokens)
        k = k if torch.is_tensor(k) else torch.from_numpy(np.ascontiguousarray(k, dtype=float))
        v = v if torch.is_tensor(v) else torch.from_numpy(np.ascontiguousarray(v, dtype=float))
        expected = (cfg.num_layers, cfg.kv_heads, tokens.size, cfg.d_k)
        if tuple(k.shape) != expected or tuple(v.shape) != expected:
            raise CacheError(f"K/V shape {tuple(k.shape)} does not match pool config {expected}")
        pages = self.arena.alloc(self.arena.pages_for(tokens.size))
        self.write_rows(pages, k, v)
        self.insert_pages(request_id, tokens, pages)

    def write_rows(self, pages, k: torch.Tensor, v: torch.Tensor) -> None:
        """Copy (L, G, n, d_k) K/V into pages (bf16, padded lanes) with the F3
        import kernel."""
        dev = self.device
        kf = k.to(dev, torch.float32).permute(0, 2, 1, 3).contiguous()     # L, n, G, d_k
        vf = v.to(dev, torch.float32).permute(0, 2, 1, 3).contiguous()
        self._import(pages, kf, vf)

    def _import(self, pages, k_lnhd: torch.Tensor, v_lnhd: torch.Tensor) -> None:
        pg = torch.as_tensor(np.asarray(list(pages), dtype=np.int32), device=self.device)
        N.call("kvs_entry_import", self.arena.c, pg.data_ptr(), k_lnhd.shape[1],
               self.config.d_k, k_lnhd.data_ptr(), v_lnhd.data_ptr(), N.stream_ptr())

    # ------------------------------------------------------------------ KVSH file
    def save(self, path) -> None:
        """pool.py:174-189: entries in insertion order, K/V as little-endian
        f32 [layer][token][head][dim].  Heads are the pool's kv_heads (the
        reference's num_heads for a multi-head model).  Each entry's rows
        leave the arena through the export kernel, one D2H copy per entry."""
        cfg = self.config
        with open(path, "wb") as fh:
            fh.write(_MAGIC)
            fh.write(struct.pack("<I", _VERSION))
            fh.write(struct.pack("<Q", len(self.entries)))
            for entry in self.entries.values():
                ident = entry.request_id.encode()
                fh.write(struct.pack("<I", len(ident)))
                fh.write(ident)
                fh.write(struct.pack("<I", entry.n_tokens))
                fh.write(entry.tokens.astype("<u4").tobytes())
                fh.write(struct.pack("<III", cfg.num_layers, cfg.kv_heads, cfg.d_k))
                if entry.owner >= 0:
                    raise CacheError(f"entry {entry.request_id!r} lives on GPU {entry.owner}")
                k, v = entry.export_f32()
                fh.write(k.cpu().numpy().astype("<f4").tobytes())
                fh.write(v.cpu().numpy().astype("<f4").tobytes())

    def load(self, path) -> "CachePool":
        """pool.py:191-241: replace the pool contents from a KVSH file.  The
        header is validated on the host with the reference's errors and byte
        offsets; each entry's f32 block goes to the device once and the import
        kernel writes it into fresh arena pages (bf16)."""
        with open(path, "rb") as fh:
            data = fh.read()
        off = 0

        def take(n: int, what: str) -> bytes:
            nonlocal off
            if off + n > len(data):
                raise FormatError(f"truncated while reading {what}", off)
            chunk = data[off:off + n]
            off += n
            return chunk

        if take(4, "magic") != _MAGIC:
            raise FormatError("bad magic bytes", 0)
        (version,) = struct.unpack("<I", take(4, "version"))
        if version != _VERSION:
            raise FormatError(f"unsupported version {version}", 4)
        (count,) = struct.unpack("<Q", take(8, "entry count"))
        cfg = self.config
        parsed = []
        for _ in range(count):
            (id_len,) = struct.unpack("<I", take(4, "id length"))
            ident = take(id_len, "id").decode()
            (n_tok,) = struct.unpack("<I", take(4, "token count"))
            tokens = np.frombuffer(take(4 * n_tok, "tokens"), dtype="<u4").astype(np.int64)
            layers, heads, d_k = struct.unpack("<III", take(12, "dimensions"))
            if (layers, heads, d_k) != (cfg.num_layers, cfg.kv_heads, cfg.d_k):
                raise CacheError(
                    f"entry {ident!r} dims ({layers}, {heads}, {d_k}) do not match "
                    f"pool config ({cfg.num_layers}, {cfg.kv_heads}, {cfg.d_k})")
            if n_tok == 0:
                raise CacheError(f"entry {ident!r} has no tokens")
            size = layers * n_tok * heads * d_k
            k_off = off
            take(4 * size, "K")
            v_off = off
            take(4 * size, "V")
            parsed.append((ident, tokens, k_off, v_off, size))
        if off != len(data):
            raise FormatError("trailing data after final entry", off)
        for entry in list(self.entries.values()):
            self._drop(entry)
        shape = (cfg.num_layers, -1, cfg.kv_heads, cfg.d_k)
        cap, self.capacity_bytes = self.capacity_bytes, None     # load never evicts
        for ident, tokens, k_off, v_off, size in parsed:
            k = torch.from_numpy(np.frombuffer(data, "<f4", size, k_off).reshape(shape).copy())
            v = torch.from_numpy(np.frombuffer(data, "<f4", size, v_off).reshape(shape).copy())
            pages = self.arena.alloc(self.arena.pages_for(tokens.size))
            self._import(pages, k.to(self.device), v.to(self.device))
            self.insert_pages(ident, tokens, pages)
        self.capacity_bytes = cap
        return self

    # ------------------------------------------------------------------ index
    def _build_index(self):
        """The device token index, maintained incrementally:

        * entry tokens, window hashes and window slots live in append-only
          flat device buffers (capacity doubling); a new entry appends its
          rows and its windows are merged into the hash-sorted window list
          (sort of the new windows + a searchsorted merge: O(new log new +
          total) device work, no re-sort and no host rebuild of the index);
        * a dropped entry only loses its recency rank (-1): the lookup
          kernels skip its windows;
        * when dead windows outnumber live ones the buffers are compacted
          (live slots keep their ids), and when freed slot ids dominate, live
          entries are renumbered (single-GPU pools only: a sharded pool's
          slot ids are shared with the owners).
        Recency ranks, slot page tables and owners are small per-slot host
        arrays re-uploaded after any change."""
        if not self._dirty and self._index is not None:
            return self._index
        dev = self.device
        n_slots = len(self._slots)
        live = [i for i, e in enumerate(self._slots) if e is not None]
        ti = self._tidx
        if ti is None:
            ti = self._tidx = _TokenIndexBuffers(dev)
        # append the slots that are new since the last build
        for sl in range(ti.n_slots, n_slots):
            ti.append(self._slot_tokens[sl], self._slot_hash[sl])
        ti.set_live(self._slots)
        if ti.dead_windows() > max(ti.live_windows(), 1 << 16):
            ti.compact(self._slots, self._slot_tokens, self._slot_hash)
        order = sorted(live, key=lambda sl: -self._slots[sl].insert_seq)
        rank = np.full(max(n_slots, 1), -1, dtype=np.int32)
        r2s = np.zeros(max(n_slots, 1), dtype=np.int32)
        for r, sl in enumerate(order):
            rank[sl] = r
            r2s[r] = sl
        idx = dict(tokens=ti.tokens, tok_off=ti.tok_off_dev(), win_off=ti.win_off_dev(),
                   win_hash=ti.win_hash, win_slot=ti.win_slot, sorted_hash=ti.sorted_hash,
                   sorted_widx=ti.sorted_widx, slot_rank=torch.from_numpy(rank).to(dev),
                   rank2slot=torch.from_numpy(r2s).to(dev))
        p = self.params
        c = N.TokenIndex(n_slots, ti.n_sorted, p.window_size, p.base, p.modulus,
                         *(idx[k].data_ptr() for k in ("tokens", "tok_off", "win_off", "win_hash",
                                                        "win_slot", "sorted_hash", "sorted_widx",
                                                        "slot_rank", "rank2slot")))
        def _pg(e):                  # remote entries: the owner's pages (peer memory)
            return e.remote_pages if e.owner >= 0 else e.pages
        max_pages = max([len(_pg(e)) for e in self._slots if e is not None]
                        + [len(_pg(e)) for e in self._retired.values()] + [1])
        sp = np.zeros((max(n_slots, 1), max_pages), dtype=np.int32)
        owner = np.full(max(n_slots, 1), -1, dtype=np.int32)
        oslot = np.arange(max(n_slots, 1), dtype=np.int32)
        for sl in live + list(self._retired):
            e = self._slots[sl] if self._slots[sl] is not None else self._retired[sl]
            sp[sl, :len(_pg(e))] = _pg(e)
            owner[sl] = e.owner
            if e.owner >= 0:
                oslot[sl] = e.owner_slot
        idx["slot_pages"] = torch.from_numpy(sp).to(dev)
        idx["slot_max_pages"] = max_pages
        idx["slot_owner"] = owner
        idx["slot_on_owner"] = oslot
        idx["slot_owner_dev"] = torch.from_numpy(owner).to(dev)
        idx["slot_on_owner_dev"] = torch.from_numpy(oslot).to(dev)
        idx["c"] = c
        self._index = idx
        self._dirty = False
        return idx

    def _maybe_renumber(self) -> None:
        """Reclaim freed slot ids once they dominate (single-GPU pools)."""
        n_live = len(self.entries)
        if len(self._slots) <= 2 * n_live + 64 or self._pins or \
                any(e.owner >= 0 for e in self.entries.values()):
            return
        live = [e for e in self._slots if e is not None]
        toks = [self._slot_tokens[e.slot] for e in live]
        hashes = [self._slot_hash[e.slot] for e in live]
        self._slots, self._slot_tokens, self._slot_hash = list(live), toks, hashes
        for i, e in enumerate(live):
            e.slot = i
        self._tidx = None                       # rebuilt from the renumbered slots
        self._dirty = True

    # ------------------------------------------------------------------ lookup
    def lookup_device(self, tokens_flat: torch.Tensor, req_off: torch.Tensor,
                      req_off_host: np.ndarray) -> BatchLookup:
        """Batched R2 lookup of a scheduled batch (flat device tokens)."""
        n_req = len(req_off_host) - 1
        n_total = int(req_off_host[-1])
        if n_req and int(np.diff(req_off_host).max()) >= MAX_SEQ:
            raise ParameterError(f"requests of {MAX_SEQ} tokens or more are not supported")
        dev = self.device
        src_slot = torch.empty(max(n_total, 1), dtype=torch.int32, device=dev)
        src_cand = torch.empty(max(n_total, 1), dtype=torch.int32, device=dev)
        n_hit = torch.zeros(n_req, dtype=torch.int32, device=dev)
        n_slots = max(len(self._slots), 1)
        contributed = torch.zeros((n_req, n_slots), dtype=torch.uint8, device=dev)
        if self.entries:
            idx = self._build_index()
            ws = self._ws.get(N.ws_bytes("kvs_pool_lookup_workspace", n_total), dev)
            N.call("kvs_pool_lookup", idx["c"], tokens_flat.data_ptr(), req_off.data_ptr(),
                   n_req, n_total, src_slot.data_ptr(), src_cand.data_ptr(), n_hit.data_ptr(),
                   contributed.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr())
        else:
            src_slot.fill_(-1)
            src_cand.fill_(-1)
        return BatchLookup(req_off, tokens_flat, src_slot[:n_total], src_cand[:n_total], n_hit,
                           contributed)

    def admit(self, token_lists, fixed_chunk: int | None = None) -> list["AdmittedHits"]:
        """Admission-time lookups of several requests at once (simulate.py:
        180-186): one device lookup over all of them, LRU refreshed request by
        request in order (identical to sequential pool.lookup calls, since a
        lookup reads insertion order, not recency).  Each result holds the
        request's device hit map and pins the slots it reads until
        ``release()``, like the reference's ReuseMap holding its entries."""
        toks = [np.asarray(t, dtype=np.int64) for t in token_lists]
        if not toks:
            return []
        for t in toks:
            if t.ndim != 1 or t.size == 0:
                raise InputError("token sequence must be a non-empty 1-D array")
        dev = self.device
        off = np.zeros(len(toks) + 1, dtype=np.int64)
        off[1:] = np.cumsum([t.size for t in toks])
        flat = torch.from_numpy(np.concatenate(toks)).to(dev)
        off_dev = torch.from_numpy(off).to(dev)
        n_total = int(off[-1])
        if fixed_chunk is None or not self.entries:
            res = self.lookup_device(flat, off_dev, off)
            slot, cand, n_hit, contributed = res.src_slot, res.src_cand, res.n_hit, res.contributed
        else:
            if fixed_chunk < 1:
                raise ParameterError(f"chunk_size must be >= 1, got {fixed_chunk}")
            idx = self._build_index()
            slot = torch.empty(n_total, dtype=torch.int32, device=dev)
            cand = torch.empty(n_total, dtype=torch.int32, device=dev)
            n_hit = torch.zeros(len(toks), dtype=torch.int32, device=dev)
            contributed = torch.zeros((len(toks), max(len(self._slots), 1)), dtype=torch.uint8,
                                      device=dev)
            N.call("kvs_fixed_chunk_lookup", idx["c"], flat.data_ptr(), off_dev.data_ptr(),
                   len(toks), int(np.diff(off).max()), int(fixed_chunk), slot.data_ptr(),
                   cand.data_ptr(), n_hit.data_ptr(), contributed.data_ptr(), n_total,
                   N.stream_ptr())
        contrib = contributed.cpu().numpy()
        hits = n_hit.cpu().numpy()
        out = []
        for r, t in enumerate(toks):
            self.refresh_lru(contrib[r])
            slots = np.nonzero(contrib[r])[0].tolist()
            self.pin(slots)
            a, b = int(off[r]), int(off[r + 1])
            out.append(AdmittedHits(self, t.size, int(hits[r]), slot[a:b], cand[a:b], slots))
        return out

    def refresh_lru(self, contributed_row: np.ndarray) -> None:
        """pool.py:157-159: contributors get new ticks in old last_access order."""
        contributors = [self._slots[s] for s in np.nonzero(contributed_row)[0]
                        if s < len(self._slots) and self._slots[s] is not None]
        for entry in sorted(contributors, key=lambda e: e.last_access):
            entry.last_access = self._tick()

    def lookup(self, tokens, fixed_chunk: int | None = None) -> ReuseMap:
        """pool.py:125-161 for one request."""
        tokens = np.asarray(tokens, dtype=np.int64)
        reuse = ReuseMap(length=int(tokens.size))
        if tokens.size == 0 or not self.entries:
            return reuse
        if fixed_chunk is not None:
            return self._lookup_fixed(tokens, fixed_chunk)
        dev = self.device
        tok = torch.from_numpy(tokens).to(dev)
        off = np.array([0, tokens.size], dtype=np.int64)
        res = self.lookup_device(tok, torch.from_numpy(off).to(dev), off)
        slot = res.src_slot.cpu().numpy()
        cand = res.src_cand.cpu().numpy()
        self.refresh_lru(res.contributed[0].cpu().numpy())
        for pos in np.nonzero(slot >= 0)[0]:
            reuse.sources[int(pos)] = (self._slots[slot[pos]], int(cand[pos]))
        reuse.src_slot, reuse.src_cand = res.src_slot, res.src_cand
        return reuse

    def _lookup_fixed(self, tokens: np.ndarray, chunk: int) -> ReuseMap:
        """Fixed-chunk baseline (pool.py:148-149 -> matching.fixed_chunk_match)
        on the device: the F5 kernel claims each chunk-aligned block for the
        newest entry holding it at an aligned offset."""
        if chunk < 1:
            raise ParameterError(f"chunk_size must be >= 1, got {chunk}")
        reuse = ReuseMap(length=int(tokens.size))
        dev, n = self.device, int(tokens.size)
        idx = self._build_index()
        tok = torch.from_numpy(tokens).to(dev)
        off = torch.tensor([0, n], dtype=torch.int64, device=dev)
        slot = torch.empty(n, dtype=torch.int32, device=dev)
        cand = torch.empty(n, dtype=torch.int32, device=dev)
        n_hit = torch.zeros(1, dtype=torch.int32, device=dev)
        contributed = torch.zeros((1, max(len(self._slots), 1)), dtype=torch.uint8, device=dev)
        N.call("kvs_fixed_chunk_lookup", idx["c"], tok.data_ptr(), off.data_ptr(), 1, n, int(chunk),
               slot.data_ptr(), cand.data_ptr(), n_hit.data_ptr(), contributed.data_ptr(), n,
               N.stream_ptr())
        self.refresh_lru(contributed[0].cpu().numpy())
        sl, cd = slot.cpu().numpy(), cand.cpu().numpy()
        for pos in np.nonzero(sl >= 0)[0]:
            reuse.sources[int(pos)] = (self._slots[sl[pos]], int(cd[pos]))
        reuse.src_slot, reuse.src_cand = slot, cand
        return reuse

    # ------------------------------------------------------------------ eviction
    def evict_to_capacity(self, max_bytes: int) -> list[str]:
        """pool.py:163-172: drop least-recently-accessed entries until it fits."""
        if max_bytes < 0:
            raise ParameterError(f"max_bytes must be >= 0, got {max_bytes}")
        evicted = []
        while self.entries and self.total_bytes > max_bytes:
            victim = min(self.entries.values(), key=lambda e: e.last_access)
            self._drop(victim)
            evicted.append(victim.request_id)
        return evicted

    def slot_entry(self, slot: int) -> KVEntry | None:
        return self._slots[slot] if 0 <= slot < len(self._slots) else None


class _TokenIndexBuffers:
    """Append-only device buffers behind CachePool's token index (see
    CachePool._build_index).  Hashes are < 2^63, so int64 order is the
    uint64 order the lookup kernels search."""

    def __init__(self, device):
        self.device = device
        z64 = lambda: torch.zeros(1, dtype=torch.int64, device=device)   # noqa: E731
        self.tokens, self.win_hash = z64(), z64()
        self.win_slot = torch.zeros(1, dtype=torch.int32, device=device)
        self.sorted_hash, self.sorted_widx = z64(), torch.zeros(1, dtype=torch.int32, device=device)
        self.n_tok = self.n_win = self.n_sorted = 0
        self.tok_off, self.win_off = [0], [0]
        self.live = []                              # per slot: still in the pool
        self._off_dev = None

    @property
    def n_slots(self) -> int:
        return len(self.tok_off) - 1

    @staticmethod
    def _grow(buf: torch.Tensor, need: int) -> torch.Tensor:
        if buf.numel() >= need:
            return buf
        out = torch.empty(max(need, 2 * buf.numel()), dtype=buf.dtype, device=buf.device)
        out[:buf.numel()].copy_(buf)
        return out

    def append(self, tok: torch.Tensor | None, hashes: torch.Tensor | None) -> None:
        n = 0 if tok is None else tok.numel()
        m = 0 if hashes is None else hashes.numel()
        slot = self.n_slots
        self.tokens = self._grow(self.tokens, self.n_tok + n)
        self.win_hash = self._grow(self.win_hash, self.n_win + m)
        self.win_slot = self._grow(self.win_slot, self.n_win + m)
        if n:
            self.tokens[self.n_tok:self.n_tok + n].copy_(tok)
        if m:
            self.win_hash[self.n_win:self.n_win + m].copy_(hashes)
            self.win_slot[self.n_win:self.n_win + m].fill_(slot)
            self._merge(hashes, self.n_win)
        self.n_tok += n
        self.n_win += m
        self.tok_off.append(self.n_tok)
        self.win_off.append(self.n_win)
        self.live.append(tok is not None)
        self._off_dev = None

    def _merge(self, hashes: torch.Tensor, first_widx: int) -> None:
        """Merge new windows (widx first_widx + k) into the sorted list."""
        h_new, perm = torch.sort(hashes)
        w_new = (perm + first_widx).to(torch.int32)
        N0, M = self.n_sorted, h_new.numel()
        out_h = torch.empty(N0 + M, dtype=torch.int64, device=self.device)
        out_w = torch.empty(N0 + M, dtype=torch.int32, device=self.device)
        if N0:
            old_h, old_w = self.sorted_hash[:N0], self.sorted_widx[:N0]
            pos_new = torch.searchsorted(old_h, h_new, right=True) + \
                torch.arange(M, device=self.device)
            pos_old = torch.searchsorted(h_new, old_h, right=False) + \
                torch.arange(N0, device=self.device)
            out_h[pos_old] = old_h
            out_w[pos_old] = old_w
            out_h[pos_new] = h_new
            out_w[pos_new] = w_new
        else:
            out_h.copy_(h_new)
            out_w.copy_(w_new)
        self.sorted_hash, self.sorted_widx, self.n_sorted = out_h, out_w, N0 + M

    def set_live(self, slots) -> None:
        self.live = [slots[i] is not None for i in range(self.n_slots)]

    def live_windows(self) -> int:
        return sum(self.win_off[i + 1] - self.win_off[i] for i in range(self.n_slots)
                   if self.live[i])

    def dead_windows(self) -> int:
        return self.n_sorted - self.live_windows()

    def compact(self, slots, slot_tokens, slot_hash) -> None:
        """Rebuild the buffers from the live slots only (slot ids kept; a dead
        slot keeps an empty range)."""
        fresh = _TokenIndexBuffers(self.device)
        for i in range(self.n_slots):
            alive = slots[i] is not None
            fresh.append(slot_tokens[i] if alive else None, slot_hash[i] if alive else None)
        fresh.set_live(slots)
        self.__dict__.update(fresh.__dict__)

    def tok_off_dev(self) -> torch.Tensor:
        self._offsets()
        return self._off_dev[0]

    def win_off_dev(self) -> torch.Tensor:
        self._offsets()
        return self._off_dev[1]

    def _offsets(self) -> None:
        if self._off_dev is None:
            self._off_dev = (torch.tensor(self.tok_off, dtype=torch.int64, device=self.device),
                             torch.tensor(self.win_off, dtype=torch.int64, device=self.device))
