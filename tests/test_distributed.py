"""Multi-process (world_size 2, gloo, CPU) checks of the element sharding and
the max-over-ranks timing used by bench.py (contiguous even
element ranges, no collective on the data path)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle
    from paper_1711_00984_b200.inputs import WORKLOADS

    wl = WORKLOADS["c2_h1_p5_general"]
    E = 6
    lo, hi = bench.shard(E * world, world, rank)
    assert hi - lo == E
    b = wl.batch(E * world).slice(lo, hi)
    # each rank integrates its own shard (CPU oracle stands in for the device here)
    packed = oracle.gram_batched(wl.space, wl.path, (2, 2, 2), 3, b.kind, b.params, b.coef)
    local = torch.tensor([packed.sum(), float(rank + 1)], dtype=torch.float64)
    gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, local)  # optional checksum gather (no data-path collective)
    t = bench.max_over_ranks(0.5 + rank, world)
    out[rank] = (lo, hi, float(sum(g[0] for g in gathered)), t)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_and_timing():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert (r0[0], r0[1], r1[0], r1[1]) == (0, 6, 6, 12)  # contiguous, disjoint, covering
    assert r0[3] == r1[3] == 1.5  # max over ranks
    assert abs(r0[2] - r1[2]) < 1e-9  # every rank sees the same global checksum
    # shard checksums equal the single-process result over the full batch
    from oracle import oracle
    from paper_1711_00984_b200.inputs import WORKLOADS

    wl = WORKLOADS["c2_h1_p5_general"]
    b = wl.batch(12)
    full = oracle.gram_batched(wl.space, wl.path, (2, 2, 2), 3, b.kind, b.params, b.coef)
    assert abs(full.sum() - r0[2]) <= 1e-9 * abs(full.sum())


def _ck_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    shard = torch.arange(12, dtype=torch.float64).reshape(3, 4) + 100.0 * rank
    out[rank] = (bench.gather_checksums(shard, world), bench.gather_objects({"r": rank}, world))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_checksum_gather_two_ranks():
    """bench.gather_checksums / gather_objects over a 2-rank gloo group: every rank
    holds every shard's (sum, sum of squares, first / last element norm, count)."""
    import numpy as np

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ck_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        ck, objs = out[r]
        assert objs == [{"r": 0}, {"r": 1}]
        for q in range(world):
            a = np.arange(12, dtype=np.float64).reshape(3, 4) + 100.0 * q
            want = [a.sum(), (a * a).sum(), np.linalg.norm(a[0]), np.linalg.norm(a[2]), 3.0]
            np.testing.assert_allclose(ck[q], want, rtol=1e-14)


@pytest.mark.timeout(600)
def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); rank 0 alone prints the JSON line.  The
    reference arm runs here (host CPU), so the launcher is exercised without a GPU."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "1", "--warmup", "0", "--workload",
                        "c1_h1_p3_affine"], capture_output=True, text=True, env=env, timeout=560)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["one_core_value"] > 0
