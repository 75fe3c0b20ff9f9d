"""N>1 host logic on CPU with the gloo backend (world size 2, 127.0.0.1 rendezvous).

The hot path shards by independent scene replicas (BASELINE.json configs[4]; DESIGN.md
§6): every rank owns a disjoint block of replica ids, there is no data-path collective,
and the benchmark's whole-job number is (sum of particles) / (max over ranks of the
device-timed region).  These tests run the same functions bench.py uses."""
import os
import socket
import sys
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import backends
    from paper_2502_18437_b200 import scenes
    R = 3
    ids = bench.shard_replicas(rank, R)
    specs = bench.workload_specs("c5", rank, R)
    seeds = [s["particle_objects"][0]["seed"] for s in specs]
    # per-rank particle count of the shard, from the restatement's spawn
    n_local = sum(backends.make_scene("oracle", sp).particle_count() for sp in specs[:1]) * len(specs)
    ms = 10.0 + 5.0 * rank  # stand-in for the per-rank CUDA-event time
    ms_max, e2e_max, n_total = bench.reduce_over_ranks(ms, 2 * ms, n_local, world, "cpu")
    all_ids = [None] * world
    dist.all_gather_object(all_ids, ids)
    ref_line = None
    if rank != 0:  # the reference arm runs on rank 0 only; other ranks produce nothing
        class A:
            workload = "c5"; steps = 1; warmup = 0; cpu_seconds = 0.1; gpus = world; replicas = R
        ref_line = bench.run_reference(A(), rank)
    q.put((rank, ids, seeds, ms_max, e2e_max, n_total, all_ids, ref_line, n_local))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_sharding_and_reductions_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ids0, seeds0, m0, e0, n0, all0, ref0, nl0), (r1, ids1, seeds1, m1, e1, n1, all1, ref1, nl1) = out
    assert ids0 == [0, 1, 2] and ids1 == [3, 4, 5]              # disjoint, contiguous blocks
    assert sorted(ids0 + ids1) == list(range(6))
    assert seeds0 == [4242, 4243, 4244] and seeds1 == [4245, 4246, 4247]
    assert m0 == m1 == 15.0 and e0 == e1 == 30.0                # max over ranks
    assert n0 == n1 == nl0 + nl1 == 6 * 64800                   # sum over ranks
    assert all0 == all1 == [[0, 1, 2], [3, 4, 5]]
    assert ref1 is None                                          # reference arm: rank 0 only
