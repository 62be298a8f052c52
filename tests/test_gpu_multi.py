"""Element sharding over several GPUs, one process per GPU over
NCCL: every rank integrates its contiguous shard of a seeded global batch on
its own device; the first and last element of every shard are checked against
the CPU oracle (the parity sample spreads over every shard)
and the NCCL-gathered shard checksums equal a single-device run of the whole
batch.  Skipped unless >= 2 GPUs are visible."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    import bench
    from oracle import oracle
    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import WORKLOADS, dim

    wl = WORKLOADS["c2_h1_p5_general"]
    Eg = 600
    lo, hi = bench.shard(Eg, world, rank)
    b = wl.batch(Eg).slice(lo, hi)
    packed, status = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef,
                                  rule_order=wl.L, device=torch.device("cuda", rank))
    N = dim(wl.space, wl.orders)
    pick = [0, hi - lo - 1]
    ref = oracle.gram_batched(wl.space, wl.path, wl.orders, wl.L, b.kind[pick], b.params[pick],
                              b.coef[pick])
    got = packed[pick].cpu().numpy()
    worst = 0.0
    for k in range(2):
        G, R = oracle.unpack(got[k], N), oracle.unpack(ref[k], N)
        worst = max(worst, float(np.linalg.norm(G - R) / np.linalg.norm(R)))
    out[rank] = (lo, hi, worst, int(status.abs().sum()), bench.gather_checksums(packed, world))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_gpu_shards_parity_and_checksums():
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    import bench
    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import WORKLOADS

    for r in range(world):
        lo, hi, worst, bad, _ = out[r]
        assert worst <= 1e-12 and bad == 0
    wl = WORKLOADS["c2_h1_p5_general"]
    b = wl.batch(600)
    full, _ = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef, rule_order=wl.L)
    for r in range(world):
        lo, hi = out[r][0], out[r][1]
        want = bench.gather_checksums(full[lo:hi], 1)[0]
        np.testing.assert_allclose(out[0][4][r], want, rtol=1e-12)
