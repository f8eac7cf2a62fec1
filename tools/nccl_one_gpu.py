"""Probe: can two NCCL ranks share one GPU on this box (the gpurun pods give
one GPU per call)?  Two spawned ranks on cuda:0 run one send/recv; prints
one JSON line with the outcome (NCCL normally refuses duplicate devices).

    timeout 120 python tools/nccl_one_gpu.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _rank(rank, world, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29531")
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", 0))
        t = torch.full((1 << 20,), float(rank + 1), device="cuda")
        if rank == 0:
            dist.send(t, 1)
        else:
            dist.recv(t, 0)
        torch.cuda.synchronize()
        q.put((rank, "ok", float(t[0])))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001 - reported, not hidden
        q.put((rank, "error", repr(e)[:300]))


def main():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, 2, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = []
    for _ in ps:
        try:
            out.append(q.get(timeout=90))
        except Exception:  # noqa: BLE001
            out.append((None, "timeout", ""))
    for p in ps:
        p.join(5)
        if p.is_alive():
            p.kill()
    print(json.dumps({"nccl_two_ranks_one_gpu": sorted(out, key=lambda x: str(x[0])),
                      "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
