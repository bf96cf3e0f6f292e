"""Host-side logic of the N > 1 path, world_size 2 over gloo on CPU.

Covers what does not need a GPU: the rank-ordered IPC-blob exchange used by
``hvd.init``, cross-rank agreement of the Tensor Fusion plan (every rank must
enqueue the same collectives), and bench.py's max-over-ranks timing and
agreed pre-load step count.
"""
import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_1802_05799_b200 as hvd
        import workloads
        out = {}
        blob = bytes([rank]) * 96 + b"HVDB"
        out["blobs"] = hvd.exchange_blobs(blob)
        counts = [c for _, c in workloads.gradient_set("resnet101")]
        p = hvd.plan(counts, ["f32"] * len(counts))
        out["plan_hash"] = hashlib.sha256(repr(p).encode()).hexdigest()
        out["plan_hashes"] = hvd.exchange_blobs(out["plan_hash"])
        out["max"] = bench._max_over_ranks(float(rank + 1) * 1.5, world)
        bench._dist_env()
        q.put((rank, out))
        dist.barrier()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
        assert res[r]["blobs"] == [bytes([i]) * 96 + b"HVDB" for i in range(world)]  # rank order
        assert len(set(res[r]["plan_hashes"])) == 1                                   # same plan everywhere
        assert res[r]["max"] == 1.5 * world                                          # max over ranks
