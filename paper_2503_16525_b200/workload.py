"""Seeded synthetic multi-tenant request streams with a controlled hit rate.

Follows SURVEY.md 8(d) (the pattern of reference studies._reuse_scenario,
pkg/src/kvlab/studies.py:133-152, and trace.generate_trace, trace.py:85-112):
P source requests are pre-inserted into the pool; each target request is
assembled from spans copied out of random sources at random offsets (span
length uniform in [span_min, span_max], always >= the hash window),
interleaved with fresh random tokens until the copied fraction reaches the
requested hit rate.  Copied spans are claimed in full by the retriever;
accidental 8-token matches of random tokens are negligible at vocab >= 64k.
"""
from __future__ import annotations

import numpy as np


def source_requests(n_sources: int, length: int, vocab: int, seed: int = 0) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    return [rng.integers(0, vocab, length, dtype=np.int64) for _ in range(n_sources)]


def target_request(sources, length: int, hit: float, vocab: int, rng, span_min: int = 64,
                   span_max: int = 1024) -> np.ndarray:
    out = np.empty(length, dtype=np.int64)
    want = int(round(hit * length))
    copied, pos = 0, 0
    while pos < length:
        remaining_copy = want - copied
        remaining = length - pos
        if remaining_copy > 0 and (remaining <= remaining_copy or rng.uniform() < 0.5):
            span = int(min(rng.integers(span_min, span_max + 1), remaining_copy, remaining))
            src = sources[int(rng.integers(len(sources)))]
            span = min(span, src.size)
            a = int(rng.integers(0, src.size - span + 1))
            out[pos:pos + span] = src[a:a + span]
            copied += span
            pos += span
        else:
            gap = remaining - remaining_copy
            k = int(min(rng.integers(span_min // 2, span_max // 2 + 1), gap)) if gap > 0 else 0
            if k <= 0:
                k = remaining
            out[pos:pos + k] = rng.integers(0, vocab, k)
            pos += k
    return out


def request_batches(sources, n_batches: int, batch: int, length: int, hit: float, vocab: int,
                    seed: int = 1) -> list[list[np.ndarray]]:
    rng = np.random.default_rng(seed)
    return [[target_request(sources, length, hit, vocab, rng) for _ in range(batch)]
            for _ in range(n_batches)]
