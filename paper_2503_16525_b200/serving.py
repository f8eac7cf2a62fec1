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
the prefill rows like the reference (simulate.py:298-301).  The per-request
deviation metrics of _process_request (simulate.py:250-296) are not carried;
decode ticks cost 1 ms per token on the logical clock as in the reference
with LatencyModel.per_token_ms = 0.
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
class ServedRequest:
    id: str
    arrival_ms: float
    ttft_ms: float
    completion_ms: float
    hit_rate: float
    n_tokens: int
    decode_steps: int


@dataclass
class ServingReport:
    requests: list
    batches: list = field(default_factory=list)   # (mean hit rate, charged ms, measured ms)
    aggregate: dict = field(default_factory=dict)


def measure_prefill(engine, token_lists, ratio: float, mode: str = "selective",
                    decode_capacity: int = 0):
    """Run one scheduled batch through Engine.prefill_batch; returns (state,
    device milliseconds between CUDA events around it)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = engine.prefill_batch(token_lists, ratio=ratio, mode=mode,
                              decode_capacity=decode_capacity)
    e1.record()
    torch.cuda.synchronize()
    return st, float(e0.elapsed_time(e1))


def decode_token_stream(seed: int, request_index: int, steps: int, vocab_size: int) -> list:
    """simulate.py:134-137: Philox over SeedSequence((seed, request index))."""
    seq = np.random.SeedSequence(entropy=(seed, request_index))
    gen = np.random.Generator(np.random.Philox(seq))
    return gen.integers(0, vocab_size, steps).tolist()


def decode_batch(engine, st, streams, n_extra: int) -> None:
    """The decode stage of a served batch on the device (simulate.py:268-276
    -> engine.py:298-328): every step, D3 picks up to n_extra still-stale
    rows per request and recomputes them in the same pass as the new token,
    so the request's pages end up holding the decode-corrected K/V that the
    reference writes back (simulate.py:298-301).  A request whose own decode
    steps are done stops recomputing (its eligibility is cleared); its extra
    appended rows lie beyond the written-back prefix."""
    R = len(streams)
    steps = max((len(s) for s in streams), default=0)
    if steps == 0:
        return
    if st.eligible is None:
        n_extra = 0
    toks = np.zeros((steps, R), dtype=np.int64)
    for r, s in enumerate(streams):
        toks[:len(s), r] = s
    dev = engine.device
    tok_dev = torch.from_numpy(toks).to(dev)
    for t in range(steps):
        for r, s in enumerate(streams):
            if len(s) == t and n_extra > 0:        # request r has no step t: no more recompute
                a, b = int(st.req_off_host[r]), int(st.req_off_host[r + 1])
                st.eligible[a:b] = 0
        engine.decode_step_device(st, tok_dev[t], n_extra)


def run_serving(trace, engine, *, batch_size: int = 4, ratio: float = 0.2,
                scheduler: str = "cache_aware", mode: str = "selective",
                latency: LatencyModel | None = None, matcher: str = "adaptive",
                chunk_size: int | None = None, n_extra: int = 3,
                seed: int = 0) -> ServingReport:
    """simulate.py:140-215 over the GPU engine.  ``latency=None`` charges each
    batch its measured device time; a LatencyModel charges f(mean hit) +
    per-token term exactly like the reference (the batch still runs).  The
    decode stage runs on the device after each prefill batch (decode-stage
    DHD with n_extra, decode tokens from the reference's stream for ``seed``)
    so completed requests write back decode-corrected K/V."""
    if batch_size < 1:
        raise ConfigError(f"batch_size must be >= 1, got {batch_size}")
    if mode not in ("selective", "fr", "naive"):
        raise ParameterError(f"unknown mode {mode!r}")
    pool = engine.pool
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
        while pending and pending[0].arrival_ms <= now:
            rec = pending.pop(0)
            if mode == "fr":
                hit = 0.0
            else:
                reuse = pool.lookup(rec.tokens,
                                    fixed_chunk=chunk if matcher == "fixed" else None)
                hit = reuse.hit_rate
            queue.append(Request(rec.id, rec.arrival_ms, rec.tokens, rec.decode_steps, hit))
        if not queue:
            continue
        batch = (schedule(queue, batch_size) if scheduler == "cache_aware"
                 else fcfs_schedule(queue, batch_size))[0]
        chosen = {r.id for r in batch.requests}
        queue = [r for r in queue if r.id not in chosen]
        toks = [np.asarray(records[r.id].tokens, dtype=np.int64) for r in batch.requests]
        steps = max(records[r.id].decode_steps for r in batch.requests)
        st, measured = measure_prefill(engine, toks, ratio,
                                       "full" if mode == "fr" else
                                       ("naive" if mode == "naive" else "selective"),
                                       decode_capacity=steps if mode != "fr" else 0)
        if mode != "fr":
            # FR writes back fresh K/V (simulate.py:232-248); the other modes
            # write back what decode leaves in the cache
            streams = [decode_token_stream(seed, index[r.id], records[r.id].decode_steps,
                                           engine.cfg.vocab_size) for r in batch.requests]
            decode_batch(engine, st, streams, 0 if mode == "naive" else n_extra)
        charged = batch_latency(batch, latency) if latency is not None else measured
        batches.append((batch.mean_hit_rate, charged, measured))
        prefill_done = now + charged
        for i, req in enumerate(batch.requests):
            rec = records[req.id]
            completion = prefill_done + float(rec.decode_steps)      # 1 ms per decode tick
            out.append(ServedRequest(rec.id, rec.arrival_ms,
                                     round(prefill_done - rec.arrival_ms, 9),
                                     round(completion, 9), req.hit_rate, len(rec.tokens),
                                     rec.decode_steps))
            n_pages = engine.arena.pages_for(len(rec.tokens))
            wb_seq += 1
            heapq.heappush(writebacks, (round(completion, 9), wb_seq, rec.id, rec.tokens,
                                        st.pages[i][:n_pages]))
            engine.arena.release(st.pages[i][n_pages:])
        st.pages = []
        now = prefill_done
    flush(float("inf"))
    out.sort(key=lambda m: (m.arrival_ms, m.id))
    return ServingReport(out, batches, _aggregate(out))


def _aggregate(reqs) -> dict:
    """simulate.py:313-345 (timing part)."""
    if not reqs:
        return {"requests": 0}
    ttft = np.array([m.ttft_ms for m in reqs])
    arrivals = np.array([m.arrival_ms for m in reqs])
    completions = np.array([m.completion_ms for m in reqs])
    total_tokens = sum(m.n_tokens + m.decode_steps for m in reqs)
    makespan = float(completions.max() - arrivals.min())
    return {
        "requests": len(reqs),
        "mean_ttft_ms": float(ttft.mean()),
        "p50_ttft_ms": float(np.percentile(ttft, 50)),
        "p95_ttft_ms": float(np.percentile(ttft, 95)),
        "mean_hit_rate": float(np.mean([m.hit_rate for m in reqs])),
        "makespan_ms": makespan,
        "throughput_tokens_per_s": total_tokens / (makespan / 1000.0) if makespan > 0 else 0.0,
    }
