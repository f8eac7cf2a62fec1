"""Loaders for the committed golden vectors (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

from oracle import kvshare_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODEL_CASES = ("small", "default", "wide")


def match_doc():
    with open(os.path.join(GOLDEN, "golden_match.json")) as fh:
        return json.load(fh)


def model_case(name):
    z = np.load(os.path.join(GOLDEN, f"golden_model_{name}.npz"), allow_pickle=True)
    c = z["config"]
    cfg = O.OracleConfig(num_layers=int(c[0]), num_heads=int(c[1]), d_model=int(c[2]),
                         vocab_size=int(c[3]), seed=int(c[4]))
    return cfg, z


def weights_digest(W):
    h = hashlib.sha256(np.ascontiguousarray(W["embedding"]).tobytes())
    for layer in W["layers"]:
        for w in layer:
            h.update(np.ascontiguousarray(w).tobytes())
    return h.hexdigest()


def reuse_of(z):
    return O.Reuse(z["src_entry"], z["src_cand"], list(z["entry_k"]), list(z["entry_v"]))
