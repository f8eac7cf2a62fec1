"""Generate the cfg1 serving-metrics goldens by running the REFERENCE here.

    python tests/golden/make_golden_serving.py [/root/reference/pkg/src]

golden_serving_metrics.json: the reference's run_simulation
(simulate.py:140-215) with every per-request metric of _process_request
(simulate.py:218-310: token accounting, per-layer ||dH|| before/after the
prefill correction, decode cumulative deviation, mean TPOT) and the full
aggregate (simulate.py:313-345), on BASELINE configs[0]: the reference's
default trace (generate_trace(num_requests=8)) through the default SimConfig
at L=4 (the default model) and L=2, plus the overlap=0.8 / 500 ms-gap run,
FR and NAIVE modes, a per-token decode latency and a byte-capacity pool that
evicts while admitted requests still hold their admission-time reuse maps.
"""
from __future__ import annotations

import json
import os
import sys
from dataclasses import asdict

HERE = os.path.dirname(os.path.abspath(__file__))
REF = next((a for a in sys.argv[1:] if not a.startswith("--")), "/root/reference/pkg/src")
sys.path.insert(0, REF)

from kvlab.model import ModelConfig  # noqa: E402
from kvlab.scheduling import LatencyModel  # noqa: E402
from kvlab.simulate import SimConfig, SimMode, run_simulation  # noqa: E402
from kvlab.trace import generate_trace  # noqa: E402

CASES = [
    # name, trace kwargs, SimConfig kwargs
    ("default_L4", {}, {}),
    ("default_L2", {}, {"model": ModelConfig(num_layers=2)}),
    ("overlap08_gap500_L2", {"overlap": 0.8, "arrival_gap_ms": 500.0},
     {"model": ModelConfig(num_layers=2)}),
    ("fr_L2", {}, {"mode": SimMode.FR, "model": ModelConfig(num_layers=2)}),
    ("naive_L2", {}, {"mode": SimMode.NAIVE, "model": ModelConfig(num_layers=2)}),
    ("ratio0_L2", {"overlap": 0.8}, {"ratio": 0.0, "model": ModelConfig(num_layers=2)}),
    ("per_token_L2", {"overlap": 0.8, "arrival_gap_ms": 60.0},
     {"model": ModelConfig(num_layers=2), "latency": LatencyModel(per_token_ms=0.5),
      "batch_size": 3}),
    # entry size_bytes (pool.py:51-55) at L=2, n=48, id "r00xx": 49369 - room for 3
    ("capacity_L2", {"num_requests": 12, "overlap": 0.8, "arrival_gap_ms": 20.0},
     {"model": ModelConfig(num_layers=2), "capacity_bytes": 3 * 49369, "batch_size": 2}),
]


def main():
    out = []
    for name, tkw, skw in CASES:
        trace = generate_trace(num_requests=tkw.pop("num_requests", 8), **tkw)
        cfg = SimConfig(**skw)
        rep = run_simulation(trace, cfg)
        out.append({
            "name": name,
            "config": cfg.to_dict(),
            "trace": [{"id": r.id, "arrival_ms": r.arrival_ms, "tokens": r.tokens,
                       "decode_steps": r.decode_steps} for r in trace],
            "requests": [asdict(m) for m in rep.requests],
            "aggregate": rep.aggregate,
        })
        print(name, {k: rep.aggregate[k] for k in ("mean_ttft_ms", "tokens_recomputed_total",
                                                   "mean_decode_cum_deviation")})
    with open(os.path.join(HERE, "golden_serving_metrics.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
