"""F2: the serving loop of the reference simulator with measured GPU batch times.

Reference: pkg/src/kvlab/simulate.py:140-215 (run_simulation's event loop),
trace.py:20-42 / 93-119 (TraceRecord, generate_trace), scheduling.py:54-94
(LatencyModel, batch_latency).  One prefill server drains the queue batch by
batch: arrivals are admitted whenever the server frees up, each admitted
request gets its hit rate from a pool lookup (R2 on the device), the
cache-aware (or FCFS) scheduler forms the next batch, and the batch is
charged a prefill latency.  Decode runs off the server, one tick per token;
completed requests write their K/V back to the pool.

What changes: the batch actually runs on the GPU (Engine.prefill_batch: G1,
probe, D1, D2, partial prefill over the scheduled requests together), and
with ``latency=None`` the charged latency is that batch's measured device
time (CUDA events) instead of f(mean hit rate).  With a LatencyModel the
loop reproduces the reference's logical clock exactly (TTFT, completion and
hit rates match run_simulation's, tests/test_gpu_serving.py), which pins the
event loop; the measured run then turns the logical TTFT into real TTFT and
records (mean hit rate, measured ms) per batch for the paper's concave
latency premise.  Write-back is zero-copy: the request's
arena pages become the pool entry (reference copies K/V, simulate.py:207-210).
After each prefill batch the decode stage runs on the device (decode-stage
DHD, simulate.py:268-276), so write-back stores the decode-corrected K/V of
the prefill rows like the reference (simulate.py:298-301).  With metrics=True the
per-request deviation metrics of _process_request (simulate.py:250-296) are
measured too; decode ticks cost 1 ms plus per_token_ms per recomputed row as in
the reference (simulate.py:278-279).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import ConfigError, ParameterError
from .scheduling import LatencyModel, Request, batch_latency, fcfs_schedule, schedule


@dataclass
class TraceRecord:
    """trace.py:20-42."""

    id: str
    arrival_ms: float
    tokens: list
    decode_steps: int = 0

    def validate(self) -> None:
        if not self.id:
            raise ConfigError("record id is empty")
        if self.arrival_ms < 0:
            raise ConfigError(f"arrival_ms {self.arrival_ms} is negative")
        if not self.tokens:
            raise ConfigError("token list is empty")
        if self.decode_steps < 0:
            raise ConfigError(f"decode_steps {self.decode_steps} is negative")


def generate_trace(num_requests: int = 16, seed: int = 0, vocab_size: int = 4096,
                   chunk_len: int = 16, library_size: int = 8, segments: int = 3,
                   overlap: float = 0.5, decode_steps: int = 8,
                   arrival_gap_ms: float = 50.0) -> list[TraceRecord]:
    """trace.py:93-119: requests assembled from a shared chunk library (drawn
    with probability ``overlap``) plus fresh random chunks; same RNG stream."""
    rng = np.random.default_rng(seed)
    library = [rng.integers(0, vocab_size, chunk_len).tolist() for _ in range(library_size)]
    records = []
    for i in range(num_requests):
        tokens: list = []
        for _ in range(segments):
            if rng.uniform() < overlap:
                tokens += library[int(rng.integers(library_size))]
            else:
                tokens += rng.integers(0, vocab_size, chunk_len).tolist()
        records.append(TraceRecord(f"r{i:04d}", round(i * arrival_gap_ms, 6), tokens,
                                   decode_steps))
    return records


@dataclass
class RequestMetrics:
    """simulate.py:80-95.  ``delta_h_before``/``delta_h_after`` (per-layer
    ||H' - H||_F of the heads' attention outputs against a fresh forward,
    simulate.py:129-131, 251-267) and ``decode_cum_deviation`` (run_generation's
    sum of ||h - h_ref||, engine.py:325-327) are measured only when
    run_serving(metrics=True); otherwise they are None."""

    id: str
    arrival_ms: float
    ttft_ms: float
    completion_ms: float
    hit_rate: float
    n_tokens: int
    decode_steps: int
    tokens_recomputed: int = 0
    tokens_reused_uncorrected: int = 0
    tokens_fresh: int = 0
    delta_h_before: list | None = None
    delta_h_after: list | None = None
    decode_cum_deviation: float | None = None
    mean_tpot_ms: float = 0.0


ServedRequest = RequestMetrics


@dataclass
class ServingReport:
    requests: list
    batches: list = field(default_factory=list)   # (mean hit rate, charged ms, measured ms)
    aggregate: dict = field(default_factory=dict)


def measure_prefill(engine, token_lists, ratio: float, mode: str = "selective",
                    decode_capacity: int = 0, hits=None):
    """Run one scheduled batch through Engine.prefill_batch; returns (state,
    device milliseconds between CUDA events around it)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = engine.prefill_batch(token_lists, ratio=ratio, mode=mode,
                              decode_capacity=decode_capacity, hits=hits)
    e1.record()
    torch.cuda.synchronize()
    return st, float(e0.elapsed_time(e1))


def decode_token_stream(seed: int, request_index: int, steps: int, vocab_size: int) -> list:
    """simulate.py:134-137: Philox over SeedSequence((seed, request index))."""
    seq = np.random.SeedSequence(entropy=(seed, request_index))
    gen = np.random.Generator(np.random.Philox(seq))
    return gen.integers(0, vocab_size, steps).tolist()


def decode_batch(engine, st, streams, n_extra: int, ref_st=None):
    """The decode stage of a served batch on the device (simulate.py:268-276
    -> engine.py:298-328): every step, D3 picks up to n_extra still-stale
    rows per request and recomputes them in the same pass as the new token,
    so the request's pages end up holding the decode-corrected K/V that the
    reference writes back (simulate.py:298-301).  A request whose own decode
    steps are done stops recomputing (its eligibility is cleared); its extra
    appended rows lie beyond the written-back prefix.

    Returns the per-step recompute counts [steps, R] (device int32) and, with
    ref_st (a fresh full-recompute state of the same requests decoding the
    same tokens - run_generation's ref_session), ||h - h_ref|| per step
    [steps, R] (device fp32)."""
    R = len(streams)
    steps = max((len(s) for s in streams), default=0)
    dev = engine.device
    if steps == 0:
        return (torch.zeros((0, R), dtype=torch.int32, device=dev),
                None if ref_st is None else torch.zeros((0, R), device=dev))
    if st.eligible is None:
        n_extra = 0
    toks = np.zeros((steps, R), dtype=np.int64)
    for r, s in enumerate(streams):
        toks[:len(s), r] = s
    tok_dev = torch.from_numpy(toks).to(dev)
    counts, devs = [], []
    g = g_ref = None
    for t in range(steps):
        for r, s in enumerate(streams):
            if len(s) == t and n_extra > 0:        # request r has no step t: no more recompute
                a, b = int(st.req_off_host[r]), int(st.req_off_host[r + 1])
                st.eligible[a:b] = 0
        if t == 1 and steps > 2:
            # after one eager step, the rest replay one CUDA graph per token
            g = engine.decode_graph(st, n_extra)
            g_ref = engine.decode_graph(ref_st, 0) if ref_st is not None else None
        if g is not None:
            h, _, nch = g.replay(tok_dev[t])
            h, nch = h.clone(), nch.clone()
        else:
            h, _, nch = engine.decode_step_device(st, tok_dev[t], n_extra)
        counts.append(nch)
        if ref_st is not None:
            h_ref = g_ref.replay(tok_dev[t])[0] if g_ref is not None else \
                engine.decode_step_device(ref_st, tok_dev[t], 0)[0]
            devs.append(torch.linalg.vector_norm(h - h_ref, dim=1))
    return torch.stack(counts), (torch.stack(devs) if ref_st is not None else None)


class _DeviationSink:
    """forward_rows capture target: keeps the reference pass's head outputs
    (mode "keep") or accumulates, per layer and request, the squared
    Frobenius distance of a pass's head outputs from them (delta_h_exact's
    norm_exact summed over heads, deviation.py:59-66, simulate.py:129-131)."""

    def __init__(self, row_req: torch.Tensor, n_req: int, ref=None):
        self.row_req = row_req.long()
        self.n_req = n_req
        self.ref = ref
        self.o = {}
        self.sq = {}

    def append(self, item) -> None:
        layer, what = item[0], item[1]
        if isinstance(what, str):
            return
        o = item[2]
        if self.ref is None:
            self.o[layer] = o
            return
        d = (o.float() - self.ref.o[layer].float()).pow(2).sum(dim=(1, 2))
        acc = torch.zeros(self.n_req, dtype=torch.float32, device=o.device)
        self.sq[layer] = acc.index_add_(0, self.row_req, d)

    def norms(self, L: int) -> torch.Tensor:
        return torch.stack([self.sq[l] for l in range(L)]).sqrt()          # [L, R]


def _batch_metrics(engine, token_lists, hits, selected, mode: str, decode_steps: int):
    """Per-layer ||dH|| before (naive reuse) and after (the PRACTICAL
    session's prefill: selected rows recomputed at every layer) against a
    fresh forward, for each request (simulate.py:250-267).  The passes cover
    every row like the reference's LayerStates; the served batch itself only
    computed rows S.  Returns (before [L, R], after [L, R], ref_state): the
    fresh forward's state is kept for the decode reference."""
    L = engine.cfg.num_layers
    dev = engine.device
    st_ref = engine.new_batch(token_lists, max(1, decode_steps))
    R = len(token_lists)
    n = int(st_ref.req_off_host[-1])
    rows_req = torch.from_numpy(np.repeat(np.arange(R), st_ref.lengths)).to(dev)
    ref = _DeviationSink(rows_req, R)
    engine.forward_all_rows(st_ref, torch.ones(n, dtype=torch.uint8, device=dev), ref)
    passes = {}
    src = torch.cat([h.src_slot for h in hits])
    reused = src >= 0
    masks = {"before": (~reused).to(torch.uint8)}
    if mode == "selective" and selected is not None:
        masks["after"] = (~reused | selected.bool()).to(torch.uint8)
    for name, mask in masks.items():
        st = engine.new_batch(token_lists, 0)
        engine.set_hits(st, hits)
        engine.gather(st)
        sink = _DeviationSink(rows_req, R, ref)
        engine.forward_all_rows(st, mask, sink)
        passes[name] = sink.norms(L)
        engine.release(st)
    ref.o = {}
    before = passes["before"]
    after = passes.get("after", before)
    return before, after, st_ref


def run_serving(trace, engine, *, batch_size: int = 4, ratio: float = 0.2,
                scheduler: str = "cache_aware", mode: str = "selective",
                latency: LatencyModel | None = None, matcher: str = "adaptive",
                chunk_size: int | None = None, n_extra: int = 3,
                seed: int = 0, metrics: bool = False) -> ServingReport:
    """simulate.py:140-215 over the GPU engine.  ``latency=None`` charges each
    batch its measured device time; a LatencyModel charges f(mean hit) +
    per-token term exactly like the reference (the batch still runs).  Each
    request's reuse map is the one looked up at admission (CachePool.admit;
    its source entries stay pinned until the request's batch has run, like
    the reference's ReuseMap holding them).  The decode stage runs on the
    device after each prefill batch (decode-stage DHD with n_extra, decode
    tokens from the reference's stream for ``seed``) so completed requests
    write back decode-corrected K/V; its recompute counts give TPOT
    (simulate.py:278-279).  metrics=True adds _process_request's deviation
    metrics (simulate.py:250-296): three extra all-row forwards and a fresh
    reference decode per batch."""
    if batch_size < 1:
        raise ConfigError(f"batch_size must be >= 1, got {batch_size}")
    if mode not in ("selective", "fr", "naive"):
        raise ParameterError(f"unknown mode {mode!r}")
    pool = engine.pool
    L = engine.cfg.num_layers
    per_token_ms = latency.per_token_ms if latency is not None else 0.0
    seen = set()
    for rec in trace:
        rec.validate()
        if rec.id in seen:
            raise ConfigError(f"duplicate request id in trace: {rec.id!r}")
        seen.add(rec.id)
    chunk = chunk_size or pool.params.window_size
    pending = sorted(trace, key=lambda r: (r.arrival_ms, r.id))
    records = {r.id: r for r in pending}
    index = {r.id: i for i, r in enumerate(pending)}     # simulate.py:159 request index
    queue: list = []
    admitted: dict = {}              # id -> AdmittedHits (pinned admission-time hit map)
    writebacks: list = []            # heap of (completion_ms, seq, id, tokens, pages)
    wb_seq = 0
    out, batches = [], []
    now = 0.0

    def flush(upto: float) -> None:
        while writebacks and writebacks[0][0] <= upto:
            _, _, rid, tokens, pages = heapq.heappop(writebacks)
            pool.insert_pages(rid, tokens, pages)

    while pending or queue:
        if not queue:
            now = max(now, pending[0].arrival_ms)
        flush(now)
        arrivals = []
        while pending and pending[0].arrival_ms <= now:
            arrivals.append(pending.pop(0))
        if arrivals and mode != "fr":
            for rec, h in zip(arrivals, pool.admit(
                    [r.tokens for r in arrivals],
                    fixed_chunk=chunk if matcher == "fixed" else None)):
                admitted[rec.id] = h
        for rec in arrivals:
            hit = admitted[rec.id].hit_rate if mode != "fr" else 0.0
            queue.append(Request(rec.id, rec.arrival_ms, rec.tokens, rec.decode_steps, hit))
        if not queue:
            continue
        batch = (schedule(queue, batch_size) if scheduler == "cache_aware"
                 else fcfs_schedule(queue, batch_size))[0]
        chosen = {r.id for r in batch.requests}
        queue = [r for r in queue if r.id not in chosen]
        toks = [np.asarray(records[r.id].tokens, dtype=np.int64) for r in batch.requests]
        steps = max(records[r.id].decode_steps for r in batch.requests)
        hits = [admitted.pop(r.id) for r in batch.requests] if mode != "fr" else None
        run_mode = "full" if mode == "fr" else ("naive" if mode == "naive" else "selective")
        st, measured = measure_prefill(engine, toks, ratio, run_mode,
                                       decode_capacity=steps if mode != "fr" else 0, hits=hits)
        R = len(batch.requests)
        n_hit = np.array([h.n_hit for h in hits], dtype=np.int64) if hits else np.zeros(R, np.int64)
        n_sel = np.zeros(R, dtype=np.int64)
        if st.selected is not None:
            seg = torch.from_numpy(np.repeat(np.arange(R), st.lengths)).to(engine.device)
            n_sel = torch.zeros(R, dtype=torch.int64, device=engine.device).index_add_(
                0, seg, st.selected.long()).cpu().numpy()
        before = after = ref_st = None
        if metrics and mode != "fr" and int(n_hit.sum()):
            before, after, ref_st = _batch_metrics(engine, toks, hits, st.selected, run_mode,
                                                   steps)
        counts = devs = None
        if mode != "fr":
            # FR writes back fresh K/V (simulate.py:232-248); the other modes
            # write back what decode leaves in the cache
            streams = [decode_token_stream(seed, index[r.id], records[r.id].decode_steps,
                                           engine.cfg.vocab_size) for r in batch.requests]
            counts, devs = decode_batch(engine, st, streams, 0 if mode == "naive" else n_extra,
                                        ref_st=ref_st)
        if hits:
            for h in hits:
                h.release()
        counts = counts.cpu().numpy() if counts is not None else np.zeros((steps, R), np.int64)
        devs = devs.cpu().numpy() if devs is not None else None
        before = before.cpu().numpy() if before is not None else None
        after = after.cpu().numpy() if after is not None else None
        if ref_st is not None:
            engine.release(ref_st)
        charged = batch_latency(batch, latency) if latency is not None else measured
        batches.append((batch.mean_hit_rate, charged, measured))
        prefill_done = now + charged
        for i, req in enumerate(batch.requests):
            rec = records[req.id]
            s = rec.decode_steps
            tpot = [1.0 + per_token_ms * int(c) for c in counts[:s, i]]
            completion = prefill_done + sum(tpot)
            n = len(rec.tokens)
            m = RequestMetrics(rec.id, rec.arrival_ms, round(prefill_done - rec.arrival_ms, 9),
                               round(completion, 9), req.hit_rate, n, s,
                               mean_tpot_ms=float(np.mean(tpot)) if tpot else 0.0)
            if mode == "fr":
                m.tokens_fresh = n * L
                if metrics:
                    m.delta_h_before = m.delta_h_after = [0.0] * L
                    m.decode_cum_deviation = 0.0
            else:
                reused = int(n_hit[i])
                rec_per_layer = int(n_sel[i]) + int(counts[:s, i].sum())
                m.tokens_recomputed = L * rec_per_layer
                m.tokens_reused_uncorrected = L * (reused - rec_per_layer)
                m.tokens_fresh = (n - reused) * L
                if metrics:
                    if before is None:                   # no reuse in this batch
                        m.delta_h_before = m.delta_h_after = [0.0] * L
                    else:
                        m.delta_h_before = [float(x) for x in before[:, i]]
                        m.delta_h_after = [float(x) for x in after[:, i]]
                    m.decode_cum_deviation = float(devs[:s, i].sum()) if devs is not None else 0.0
            out.append(m)
            n_pages = engine.arena.pages_for(len(rec.tokens))
            wb_seq += 1
            heapq.heappush(writebacks, (m.completion_ms, wb_seq, rec.id, rec.tokens,
                                        st.pages[i][:n_pages]))
            engine.arena.release(st.pages[i][n_pages:])
        st.pages = []
        now = prefill_done
    flush(float("inf"))
    out.sort(key=lambda m: (m.arrival_ms, m.id))
    return ServingReport(out, batches, _aggregate(out))


def _aggregate(reqs) -> dict:
    """simulate.py:313-345."""
    if not reqs:
        return {"requests": 0}
    ttft = np.array([m.ttft_ms for m in reqs])
    arrivals = np.array([m.arrival_ms for m in reqs])
    completions = np.array([m.completion_ms for m in reqs])
    total_tokens = sum(m.n_tokens + m.decode_steps for m in reqs)
    makespan = float(completions.max() - arrivals.min())
    tpots = [m.mean_tpot_ms for m in reqs if m.decode_steps > 0]
    out = {
        "requests": len(reqs),
        "mean_ttft_ms": float(ttft.mean()),
        "p50_ttft_ms": float(np.percentile(ttft, 50)),
        "p95_ttft_ms": float(np.percentile(ttft, 95)),
        "mean_tpot_ms": float(np.mean(tpots)) if tpots else 0.0,
        "mean_hit_rate": float(np.mean([m.hit_rate for m in reqs])),
        "makespan_ms": makespan,
        "throughput_tokens_per_s": total_tokens / (makespan / 1000.0) if makespan > 0 else 0.0,
        "throughput_requests_per_s": len(reqs) / (makespan / 1000.0) if makespan > 0 else 0.0,
        "tokens_recomputed_total": sum(m.tokens_recomputed for m in reqs),
        "tokens_reused_uncorrected_total": sum(m.tokens_reused_uncorrected for m in reqs),
        "tokens_fresh_total": sum(m.tokens_fresh for m in reqs),
    }
    if all(m.decode_cum_deviation is not None for m in reqs):
        out["mean_decode_cum_deviation"] = float(np.mean([m.decode_cum_deviation for m in reqs]))
    return out
