"""ctypes boundary to libkvshare.so (the C ABI declared in include/kvshare.h).

The library is the product path: there is no CPU fallback.  If it is missing
or no CUDA device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

from .errors import STATUS_ERRORS, DeviceError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVS_LIB") or os.path.join(_PKG, "libkvshare.so")   # KVS_LIB: experiment builds

c_i32, c_i64, c_u64, c_f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
c_size, c_vp = ctypes.c_size_t, ctypes.c_void_p


class TokenIndex(ctypes.Structure):
    _fields_ = [("n_slots", c_i32), ("n_windows", c_i64), ("w", c_i32), ("b", c_u64),
                ("m", c_u64), ("tokens", c_vp), ("tok_off", c_vp), ("win_off", c_vp),
                ("win_hash", c_vp), ("win_slot", c_vp), ("sorted_hash", c_vp),
                ("sorted_widx", c_vp), ("slot_rank", c_vp), ("rank2slot", c_vp)]


class KVArena(ctypes.Structure):
    _fields_ = [("base", c_vp), ("num_pages", c_i64), ("num_layers", c_i32),
                ("kv_heads", c_i32), ("head_dim", c_i32), ("page_size", c_i32)]


class Batch(ctypes.Structure):
    _fields_ = [("n_req", c_i32), ("n_total", c_i64), ("req_off", c_vp),
                ("block_table", c_vp), ("max_pages", c_i32)]


class Rope(ctypes.Structure):
    _fields_ = [("cos", c_vp), ("sin", c_vp), ("max_pos", c_i32)]


P = ctypes.POINTER
_SIGS = {
    "kvs_window_hashes": [c_vp, c_i64, c_i32, c_u64, c_u64, c_vp, c_vp],
    "kvs_match_pairs": [c_vp, c_i64, c_vp, c_i64, c_i32, c_u64, c_u64, c_vp, c_vp, c_vp, c_vp,
                        c_size, c_vp],
    "kvs_index_sort": [c_vp, c_i64, c_vp, c_vp, c_vp, c_size, c_vp],
    "kvs_pool_lookup": [P(TokenIndex), c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                        c_size, c_vp],
    "kvs_gather_kv": [P(KVArena), P(Batch), c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, P(Rope), c_vp],
    "kvs_gather_kv_peer": [P(KVArena), P(Batch), c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32,
                           P(Rope), c_vp],
    "kvs_qkv_rope_scatter": [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, P(KVArena), P(Batch),
                             P(Rope), c_vp, c_vp, c_vp, c_vp],
    "kvs_qkv_rope_scatter_rows": [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, P(KVArena),
                                  P(Batch), P(Rope), c_vp, c_vp, c_vp, c_vp],
    "kvs_fixed_chunk_lookup": [P(TokenIndex), c_vp, c_vp, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp,
                               c_vp, c_i64, c_vp],
    "kvs_topk_select": [c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp],
    "kvs_proj_skinny": [c_vp, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp],
    "kvs_ideal_scores": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_f32,
                         c_vp, c_vp, c_size, c_vp],
    "kvs_entry_import": [P(KVArena), c_vp, c_i64, c_i32, c_vp, c_vp, c_vp],
    "kvs_entry_export": [P(KVArena), c_vp, c_i64, c_i32, c_vp, c_vp, c_vp],
    "kvs_embed_rows": [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "kvs_pack_rows": [P(KVArena), c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_vp],
    "kvs_unpack_rows": [P(KVArena), P(Batch), c_vp, c_vp, c_i64, c_vp, P(Rope), c_i32, c_i32,
                        c_vp, c_vp],
    "kvs_build_rows": [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "kvs_attention_fwd": [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_i32, c_i32,
                          P(KVArena), P(Batch), c_f32, c_vp, c_vp, c_vp],
    "kvs_attention_fwd_qkv": [c_vp, c_i64, P(Rope), c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32,
                              c_vp, c_i32, c_i32, P(KVArena), P(Batch), c_f32, c_vp, c_vp],
    "kvs_decode_attention": [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, P(KVArena),
                             P(Batch), c_f32, c_vp, c_vp, c_size, c_vp],
    "kvs_dhd_alpha": [c_vp, c_i32, c_i32, c_i32, P(KVArena), P(Batch), c_vp, c_vp, c_vp, c_vp,
                      c_i32, c_vp, c_f32, c_vp, c_vp, c_size, c_vp],
    "kvs_dhd_select": [c_vp, c_vp, c_vp, c_i32, P(KVArena), P(Batch), c_vp, c_vp, c_vp, c_vp,
                       c_vp, c_size, c_vp],
    "kvs_dhd_decode_select": [c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_i32, P(KVArena), P(Batch),
                              c_i32, c_f32, c_vp, c_vp, c_vp, c_vp, c_size, c_vp],
}
_WS_SIGS = {
    "kvs_match_pairs_workspace": [c_i64, c_i64],
    "kvs_index_sort_workspace": [c_i64],
    "kvs_pool_lookup_workspace": [c_i64],
    "kvs_decode_attention_workspace": [c_i64, c_i32, c_i32, c_i32, c_i32],
    "kvs_dhd_alpha_workspace": [c_i64, c_i32, c_i32],
    "kvs_ideal_scores_workspace": [c_i32, c_i32, c_i32],
    "kvs_dhd_select_workspace": [c_i64, c_i32],
    "kvs_dhd_decode_select_workspace": [c_i32, c_i32, c_i32],
}

_lib = None

# kernels launched per entry point (for the bench's gpu_launches claim)
KERNELS_PER_CALL = {
    "kvs_window_hashes": 1, "kvs_match_pairs": 9, "kvs_index_sort": 5, "kvs_pool_lookup": 4,
    "kvs_gather_kv": 1, "kvs_gather_kv_peer": 1, "kvs_qkv_rope_scatter": 1, "kvs_qkv_rope_scatter_rows": 1, "kvs_embed_rows": 1, "kvs_build_rows": 1,
    "kvs_proj_skinny": 1,
    "kvs_attention_fwd": 1, "kvs_attention_fwd_qkv": 1, "kvs_decode_attention": 2, "kvs_dhd_alpha": 3,
    "kvs_dhd_select": 1, "kvs_ideal_scores": 3, "kvs_dhd_decode_select": 1, "kvs_pack_rows": 1, "kvs_unpack_rows": 1,
}
launch_count = {"kernels": 0}


def exported_symbols():
    return sorted(set(_SIGS) | set(_WS_SIGS) | {"kvs_last_error", "kvs_abi_version"})


def load(require_gpu: bool = True):
    """Load libkvshare.so (raises if it is missing - no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = c_i32
        for name, args in _WS_SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = c_size
        lib.kvs_last_error.restype = ctypes.c_char_p
        lib.kvs_abi_version.restype = c_i32
        _lib = lib
    if require_gpu and not torch.cuda.is_available():
        raise DeviceError("libkvshare needs a CUDA device (B200, sm_100a); none is visible")
    return _lib


def call(name: str, *args):
    lib = load()
    launch_count["kernels"] += KERNELS_PER_CALL.get(name, 1)
    st = getattr(lib, name)(*args)
    if st != 0:
        msg = lib.kvs_last_error().decode(errors="replace")
        raise STATUS_ERRORS.get(st, DeviceError)(f"{name}: {msg}")


def ws_bytes(name: str, *args) -> int:
    return int(getattr(load(require_gpu=False), name)(*args))


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Workspace:
    """Grow-only device scratch buffer (hot calls never allocate)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device, zero: bool = False) -> torch.Tensor:
        """zero=True: a newly allocated buffer starts zeroed (kernels that keep
        self-resetting counters in their workspace rely on it)."""
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = (torch.zeros if zero else torch.empty)(nbytes, dtype=torch.uint8,
                                                             device=device)
        return self.buf
