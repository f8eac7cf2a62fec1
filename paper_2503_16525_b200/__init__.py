"""B200-native KVShare DHD hot path (arXiv 2503.16525), drop-in for the
reference ``kvlab`` names on that path.

Public names follow reference pkg/src/kvlab/__init__.py:71-86 for everything
on the hot path: KV Retriever (HashParams, match_sequences, CachePool.lookup),
DHD selection (v_impact_scores, select_prefill, select_decode_step),
sessions and generation (ReuseSession, prefill_with_selection,
run_generation) and the cache-aware batch hand-off (schedule).  Compute runs
in libkvshare.so (CUDA, sm_100a); importing does not require a GPU, calling
does.
"""
from .errors import (CacheError, ConfigError, DeviceError, FormatError, InputError, KVLabError,
                     NumericError, ParameterError, ShapeError)
from .matching import (HashParams, MatchResult, build_hash_index, fixed_chunk_match, hit_rate,
                       match_sequences, rolling_hash, window_hashes)
from .model import LLAMA31_8B, QWEN25_7B, YI15_9B, ModelConfig, ToyModel, init_model
from .scheduling import (Batch, LatencyModel, Request, batch_latency, fcfs_schedule,
                         partition_batch, schedule)

__version__ = "0.1.0"

_LAZY = {
    "CachePool": "pool", "KVEntry": "pool", "ReuseMap": "pool", "KVArena": "pool",
    "v_impact_scores": "deviation", "top_indices": "deviation",
    "SelectionConfig": "selection", "SelectionMode": "selection",
    "SelectionResult": "selection", "Strategy": "selection", "select_baseline": "selection",
    "select_decode_step": "selection", "select_prefill": "selection",
    "Engine": "engine", "LayerStates": "session", "ReuseSession": "session",
    "PrefillResult": "session", "GenerationResult": "session", "model_forward": "session",
    "model_forward_with_reuse": "session", "prefill_with_selection": "session",
    "run_generation": "session",
    "TraceRecord": "serving", "generate_trace": "serving", "run_serving": "serving",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(set(_LAZY) | {
    "Batch", "CacheError", "ConfigError", "DeviceError", "FormatError", "HashParams",
    "InputError", "KVLabError", "LatencyModel", "MatchResult", "ModelConfig", "NumericError",
    "ParameterError", "Request", "ShapeError", "ToyModel", "batch_latency", "build_hash_index",
    "fcfs_schedule", "fixed_chunk_match", "hit_rate", "init_model", "match_sequences",
    "partition_batch", "rolling_hash", "schedule", "window_hashes", "LLAMA31_8B", "QWEN25_7B", "YI15_9B"})
