"""Benchmark of the batched Gram integration (BASELINE.json metric: Gram
elements/s per space & test order, achieved fraction of the FP64/HBM
roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step is one pass of the hot path over one synthetic batch of the
workload (default: BASELINE configs[1], H1 Gram, trilinear maps, p_test=5,
4096 elements per GPU).  Elements are sharded across ranks (weak scaling:
each rank integrates its own slice of a seeded global batch; no collective on
the data path).  Rank 0 prints one JSON line.

--impl reference times the reference's CPU algorithm on the host cores (the
C restatement in oracle/, pinned bit-exact to the reference package) on the
same workload, metric and unit.
"""

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1711_00984_b200.inputs import ALL_WORKLOADS, WORKLOADS, dim  # noqa: E402

METRIC = "Gram elements/sec per space & test order; achieved % of FP64/HBM roofline"
UNIT = "elements/s"
L2_BYTES = 126 * 2 ** 20
PEAK_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "peaks_r01.jsonl")
NCU_TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
PATH_CODES = {"general": 0, "affine": 1, "extrusion": 2}


def algorithmic(space, orders, path, L):
    """Per element: F = 2 x reference accumulations, B = packed fp64 output
    bytes."""
    from paper_1711_00984_b200.gram import counters

    N = dim(space, orders)
    P = N * (N + 1) // 2
    c = counters(space, orders, "tensorized" if path == "general" else "simplified",
                 L if path == "general" else None)
    return 2.0 * c.accumulations, 8.0 * P, P


def peaks():
    hbm = 6650.0
    src_hbm = "fallback (B200_PROFILING.md)"
    if os.path.exists(PEAK_FILE):
        with open(PEAK_FILE) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
        src_hbm = "MEASURED_PEAKS.json hbm_gbs"
    fp64 = 37.0
    src_fp64 = "profiles/peaks_r01.jsonl dmma_m8n8k4 (measured on this pool's B200)"
    if os.path.exists(FP64_PEAK_FILE):
        with open(FP64_PEAK_FILE) as fh:
            vals = [json.loads(l) for l in fh if l.strip()]
        dm = [v["tflops"] for v in vals if v.get("test", "").startswith("dmma")]
        if dm:
            fp64 = max(dm)
    return hbm, src_hbm, fp64, src_fp64


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = None

    def __enter__(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.tmp, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.tmp.flush()
        with open(self.tmp.name) as fh:
            rows = [r.strip().split(",") for r in fh if r.strip()]
        os.unlink(self.tmp.name)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def maybe_spawn(args, argv):
    """`--gpus N` (N > 1) outside a torchrun environment: re-launch this script
    as N ranks under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1) and return its exit code; None when already inside a launcher
    or N == 1.  Only rank 0 prints, so the parent's stdout is the one JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using the launcher's "
              f"world size", file=sys.stderr)
    if world > 1 and not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            if torch.cuda.device_count() <= local:
                raise RuntimeError(f"rank {rank}: LOCAL_RANK {local} but only "
                                   f"{torch.cuda.device_count()} visible GPU(s)")
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def gather_checksums(out, world, device=None):
    """Per-shard checksums of the packed output (sum, sum of squares, Frobenius
    norm of the shard's first and last element), all-gathered over the
    process group -- the only collective of the multi-GPU run."""
    import torch

    E = out.shape[0]
    # reductions only, in row blocks (no output-sized temporaries, no 2^31 BLAS limit: 100 GB sweeps)
    rows = max(1, (1 << 28) // max(1, out.shape[1]))
    s1 = torch.zeros((), dtype=torch.float64, device=out.device)
    s2 = torch.zeros((), dtype=torch.float64, device=out.device)
    for r0 in range(0, E, rows):
        blk = out[r0:r0 + rows].reshape(-1)
        s1 += blk.sum()
        s2 += torch.dot(blk, blk)
    loc = torch.stack([s1, s2, torch.linalg.norm(out[0]), torch.linalg.norm(out[E - 1]),
                       torch.tensor(float(E), dtype=torch.float64, device=out.device)])
    if world == 1:
        return [loc.tolist()]
    import torch.distributed as dist

    allv = [torch.zeros_like(loc) for _ in range(world)]
    dist.all_gather(allv, loc)
    return [v.tolist() for v in allv]


def gather_objects(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist

    allv = [None] * world
    dist.all_gather_object(allv, obj)
    return allv


def max_over_ranks(x, world, device=None):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard(E, world, rank):
    """Contiguous even element ranges [r E / n, (r+1) E / n)."""
    lo = (rank * E) // world
    hi = ((rank + 1) * E) // world
    return lo, hi


# ---------------------------------------------------------------------------
# CPU legs (oracle = C restatement of the reference, test infrastructure)
# ---------------------------------------------------------------------------
def cpu_rate(wl, seconds, nthreads=0):
    """Elements/s of the reference algorithm on the host cores over a bounded
    sample (>= `seconds` of work, starting at 64 elements and doubling)."""
    from oracle import oracle

    threads = nthreads or oracle.num_cpus()
    b = wl.batch(64)
    L = wl.L if wl.path != "affine" else 1
    oracle.gram_batched(wl.space, wl.path, wl.orders, L, b.kind[:threads], b.params[:threads],
                        b.coef[:threads], nthreads=threads)  # warm
    n = max(threads, 8)
    while True:
        bb = wl.batch(n)
        t0 = time.perf_counter()
        oracle.gram_batched(wl.space, wl.path, wl.orders, L, bb.kind, bb.params, bb.coef,
                            nthreads=threads)
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= 1 << 20:
            return n / dt, n, dt, threads
        n = int(n * min(8.0, max(2.0, 1.2 * seconds / max(dt, 1e-3))))


def cpu_host_info():
    """CPU model, os.cpu_count() and the affinity-mask size."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        aff = None
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff}


def run_reference(args, wl, world, rank):
    if rank != 0:
        return
    from oracle import oracle

    threads = oracle.num_cpus()
    # size one step to ~2 s of host work
    rate, _, _, _ = cpu_rate(wl, 1.0, threads)
    per_step = max(threads, int(rate * 2.0))
    b = wl.batch(per_step)
    L = wl.L if wl.path != "affine" else 1
    for _ in range(args.warmup):
        oracle.gram_batched(wl.space, wl.path, wl.orders, L, b.kind, b.params, b.coef,
                            nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.gram_batched(wl.space, wl.path, wl.orders, L, b.kind, b.params, b.coef,
                            nthreads=threads)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    F, B, P = algorithmic(wl.space, wl.orders, wl.path, wl.L)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY 8(d))",
        "config": {"workload": wl.name, "space": wl.space, "p_test": wl.p, "L": wl.L,
                   "path": wl.path, "maps": wl.maps, "elements_per_step": per_step},
        "gram_entries_per_s": value * P,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} elements per step of {wl.name}, "
                                   f"oracle/hexgram_oracle.c (alternative loop order, "
                                   f"pthreads over elements)",
                         "one_core_value": cpu_rate(wl, 2.0, 1)[0], **cpu_host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
class DeviceStep:
    """One batch resident in HBM; step() launches the hot path on `stream`."""

    def __init__(self, wl, E, lo, device):
        import torch

        from paper_1711_00984_b200 import _native
        from paper_1711_00984_b200.engine import get_engine

        self.wl = wl
        self.E = E
        self.torch = torch
        self.eng = get_engine(device)
        self.lib = _native.lib()
        b = wl.batch(lo + E).slice(lo, lo + E)
        self.host = b
        dev = self.eng.device
        self.kind = torch.as_tensor(b.kind).to(dev)
        self.params = torch.as_tensor(b.params).to(dev)
        self.coef = torch.as_tensor(b.coef).to(dev)
        self.sc = _native.SPACE_CODES[wl.space]
        self.L = wl.L if wl.path != "affine" else 1
        self.pc = PATH_CODES[wl.path]
        N = dim(wl.space, wl.orders)
        self.P = N * (N + 1) // 2
        self.out = torch.empty((E, self.P), dtype=torch.float64, device=dev)
        self.status = torch.zeros(E, dtype=torch.int32, device=dev)
        self.tab = self.eng.tables(self.L)
        # low orders (p <= hxg_fused_order_max()) run one kernel (geometry evaluated in the contraction kernel): time the
        # whole hxg_gram_batched call; otherwise time metric and contraction separately,
        # with a workspace holding the metric fields of the whole batch
        # (hxg_workspace_size is capped at one 512 MB launch chunk)
        self.fused = wl.path == "general" and wl.p <= self.lib.hxg_fused_order_max()
        ws = self.lib.hxg_workspace_size(self.sc, self.pc,
                                         *wl.orders, self.L, E)
        per = self.lib.hxg_workspace_size(self.sc, 0, *wl.orders, self.L, 1) if wl.path == "general" else 0
        self.full_metric = wl.path == "general" and not self.fused and E * per <= (16 << 30)
        if self.full_metric:
            ws = E * per
        self.ws_bytes = ws
        self.ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
        self.chunks = -(-E // max(1, ws // per)) if per else 1
        self.flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
        self.launches_per_step = 0

    def _p(self, t):
        return ctypes.c_void_p(t.data_ptr())

    def flush(self):
        self.flush_buf.fill_(1)

    def step(self, stream, ev_mid=None):
        wl, lib, s = self.wl, self.lib, ctypes.c_void_p(stream.cuda_stream)
        if wl.path == "general" and ev_mid is not None and self.full_metric:
            rc = lib.hxg_metric_batched(self.sc, *wl.orders, self.L, self.E, self._p(self.kind),
                                        self._p(self.params), self._p(self.coef), None,
                                        self._p(self.tab), self._p(self.ws), self._p(self.status), s)
            assert rc == 0, rc
            ev_mid.record(stream)
            rc = lib.hxg_contract_batched(self.sc, *wl.orders, self.L, self.E, self._p(self.tab),
                                          self._p(self.ws), self._p(self.out), s)
            assert rc == 0, rc
            self.launches_per_step = 2
            return
        if ev_mid is not None and wl.path != "general":
            ev_mid.record(stream)
        rc = lib.hxg_gram_batched(self.sc, self.pc, *wl.orders, self.L,
                                  self.E, self._p(self.kind), self._p(self.params),
                                  self._p(self.coef), None, self._p(self.tab), self._p(self.out),
                                  self._p(self.status), self._p(self.ws), self.ws_bytes, s)
        assert rc == 0, rc
        if ev_mid is not None and wl.path == "general":
            ev_mid.record(stream)
        self.launches_per_step = 1 if wl.path != "general" else (1 if self.fused else 2 * self.chunks)


def measure_device(wl, E, lo, steps, warmup, world, device, with_clocks=True):
    import torch

    ds = DeviceStep(wl, E, lo, device)
    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        ds.flush()
        ds.step(stream)
    torch.cuda.synchronize(device)
    assert int(ds.status.abs().sum()) == 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize(device)
    sampler = ClockSampler(device.index if device.index is not None else 0) if with_clocks else None

    def keep_busy(seconds):
        # untimed steps around the timed region so the ~20 ms nvidia-smi samples
        # see the clocks of the loaded GPU even when the timed region is short
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            ds.step(stream)
            torch.cuda.synchronize(device)

    if sampler:
        sampler.__enter__()
        keep_busy(0.3)
    for k in range(steps):
        ds.flush()  # L2 flush between timed iterations (outside the timed events)
        ev[k][0].record(stream)
        ds.step(stream, ev[k][1])
        ev[k][2].record(stream)
    torch.cuda.synchronize(device)
    if sampler:
        keep_busy(0.3)
        sampler.__exit__(None, None, None)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    kern_ms = [b.elapsed_time(c) for a, b, c in ev]
    total_ms = sum(step_ms)
    return ds, total_ms, kern_ms, (sampler.summary() if sampler else None)


def measure_e2e(ds, steps, world, device):
    """Through the C ABI with HOST buffers: inputs from host memory, packed
    triangles back into pinned host memory, every step (hxg_gram_batched_host)."""
    import torch

    wl = ds.wl
    out = torch.empty((ds.E, ds.P), dtype=torch.float64).pin_memory()
    b = ds.host
    kind = np.ascontiguousarray(b.kind)
    params = np.ascontiguousarray(b.params)
    coef = np.ascontiguousarray(b.coef)
    ds.eng.integrate_host(wl.space, wl.path, wl.orders, ds.L, kind, params, coef, out)  # warm
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        ds.eng.integrate_host(wl.space, wl.path, wl.orders, ds.L, kind, params, coef, out)
    dt = time.perf_counter() - t0
    dt = max_over_ranks(dt, world, device)
    h2d = kind.nbytes + params.nbytes + coef.nbytes
    d2h = ds.E * ds.P * 8
    del out
    return dt, h2d, d2h


def dpg_suite(device, fp64, hbm, reps=3):
    """SURVEY 8(f) rows 2-3 on seeded batches: the adjoint-graph Gram of the
    ultraweak acoustics problem (dpg.py:179-231, packed real block form) and
    batched static condensation (dpg.py:348-357).  Condensation FLOPs are the
    reference algorithm's (cho_factor m^3/3, cho_solve 2 m^2 (n+1), B^T X
    2 m n (n+1)); the graph Gram is reported against the HBM bytes of its
    outputs (two packed Grams + the packed 2m x 2m block matrix)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.dpg import adjoint_graph_gram_batched, condense_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    def timed(fn):
        fn()
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize(device)
        return e0.elapsed_time(e1) / 1e3 / reps

    out = []
    # adjoint-graph Gram, p_r = 4, trilinear maps
    pr, E = 4, 512
    b = trilinear_batch(E, 21)
    kind = torch.as_tensor(b.kind).to(device)
    params = torch.as_tensor(b.params).to(device)
    t = timed(lambda: adjoint_graph_gram_batched(pr, 2.0, 0.5, kind, params))
    mw, mv = (pr + 1) ** 3, 3 * pr * pr * (pr + 1)
    m2 = 2 * (mw + mv)
    byt = 8.0 * (mw * (mw + 1) // 2 + mv * (mv + 1) // 2 + m2 * (m2 + 1) // 2)
    out.append({"workload": f"dpg_graph_acoustics_p{pr}_general", "elements_per_s": E / t,
                "ms_per_step": t * 1e3, "bound": "hbm", "hbm_write_gbs": E * byt / t / 1e9,
                "roofline_frac": E * byt / t / 1e9 / hbm, "N": m2})
    # condensation: Poisson primal (H1 Gram p_r = 5 from the Gram kernel, trial p0 = 4) and
    # acoustics real block form (p_r = 4, 2m = 850, trial 2 x 4 x 27)
    rng = np.random.default_rng(8)
    pa = 3  # acoustics: test order p_r = 3, trial p0 = 2 (real block form 2m = 416, 2 x 4 x 8)
    m2a = 2 * ((pa + 1) ** 3 + 3 * pa * pa * (pa + 1))
    for name, m, n, E in (("dpg_condense_poisson_p5", 216, 125, 1024),
                          (f"dpg_condense_acoustics_p{pa}", m2a, 2 * 4 * 8, 1024)):
        if name.startswith("dpg_condense_poisson"):
            bb = trilinear_batch(E, 22, variable_coef=True)
            G, _ = gram_batched("H1", (5, 5, 5), bb.kind, bb.params, bb.coef)
        else:
            ba = trilinear_batch(E, 24)
            G = adjoint_graph_gram_batched(pa, 2.0, 0.5, ba.kind, ba.params)
        B = torch.as_tensor(rng.standard_normal((E, m, n))).to(device)
        l = torch.as_tensor(rng.standard_normal((E, m))).to(device)
        t = timed(lambda: condense_batched(G, B, l, check=False))
        F = m ** 3 / 3 + 2.0 * m * m * (n + 1) + 2.0 * m * n * (n + 1)
        out.append({"workload": name, "elements_per_s": E / t, "ms_per_step": t * 1e3,
                    "bound": "fp64", "fp64_tflops_alg": E * F / t / 1e12,
                    "roofline_frac": E * F / t / 1e12 / fp64, "m": m, "n": n})
        del G, B, l
        torch.cuda.empty_cache()
    # ultraweak acoustics stiffness B + load l (dpg.py:234-302), p0 = 3, p_r = 5, trilinear;
    # FLOPs = 2 x the multiply-adds of the reference's 22 mixed_tens_term calls
    # (_kernels.py:1908-1930: stage A L^3 n3 p0, stage B L^2 n2 p0 n3 p0, stage C L nt ny)
    from paper_1711_00984_b200.dpg import acoustics_batched

    p0, pq, E = 3, 5, 2048
    L = pq + 1
    bb = trilinear_batch(E, 23)
    kind2 = torch.as_tensor(bb.kind).to(device)
    params2 = torch.as_tensor(bb.params).to(device)
    fg = torch.as_tensor(np.random.default_rng(9).uniform(0.5, 1.5, (E, L ** 3))).to(device)
    t = timed(lambda: acoustics_batched(p0, pq, 1.5, kind2, params2, fg, parts=False))
    q = pq + 1
    terms = [(0, 0, 0)] + [(0, 0, 0)] * 9 + [(a != 0, a != 1, a != 2) for a in range(3)] * 4
    F = 0.0
    for sh in terms:
        n1, n2, n3 = (q - x for x in sh)
        F += 2.0 * (L ** 3 * n3 * p0 + L * L * n2 * p0 * n3 * p0 + L * n1 * n2 * n3 * p0 ** 3)
    m_, n_ = q ** 3 + 3 * pq * pq * q, 4 * p0 ** 3
    byt = 8.0 * (4 * m_ * n_ + 2 * m_)  # B2 (real block form) and l
    tf, tb = E * F / (fp64 * 1e12), E * byt / (hbm * 1e9)
    out.append({"workload": f"dpg_acoustics_B_p0{p0}_pr{pq}_general", "elements_per_s": E / t,
                "ms_per_step": t * 1e3, "bound": "fp64" if tf >= tb else "hbm",
                "fp64_tflops_alg": E * F / t / 1e12, "hbm_write_gbs": E * byt / t / 1e9,
                "roofline_frac": max(tf, tb) / t})
    return out


def run_ours(args, wl, world, rank, local):
    import torch

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    E = args.elements or wl.E
    lo, _ = shard(E * world, world, rank)
    F, B, P = algorithmic(wl.space, wl.orders, wl.path, wl.L)
    hbm, src_hbm, fp64, src_fp64 = peaks()

    ds, total_ms, kern_ms, clocks = measure_device(wl, E, lo, args.steps, args.warmup, world,
                                                   device)
    total_ms = max_over_ranks(total_ms, world, device)
    sec = total_ms / 1e3
    value = E * world * args.steps / sec
    # dominant kernel: the contraction kernel (general) / the affine kernel
    kmean_s = statistics.mean(kern_ms) / 1e3
    if wl.path == "general" and not ds.full_metric:
        kmean_s = sec / args.steps  # chunked launches: whole step
    t_f, t_b = E * F / (fp64 * 1e12), E * B / (hbm * 1e9)
    bound = "tensor" if t_f >= t_b else "hbm"
    traffic = None
    if os.path.exists(NCU_TRAFFIC_FILE):
        with open(NCU_TRAFFIC_FILE) as fh:
            traffic = json.load(fh).get(wl.name)
    if bound == "tensor":
        achieved = E * F / kmean_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64, "traffic": traffic,
                "peak_source": src_fp64 + " (FP64 DMMA; no fp64 entry in MEASURED_PEAKS.json)"}
    else:
        achieved = E * B / kmean_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_source": src_hbm}
    roof.update({
        "kernel": {"general": "general_kernel (hxg_contract_batched)", "affine": "affine_v2_kernel",
                   "extrusion": "ext_v2_kernel"}[wl.path],
        "kernel_ms_per_launch": kmean_s * 1e3,
        "algorithmic_flops_per_launch": E * F, "algorithmic_bytes_per_launch": E * B,
        "flops_per_element": F, "bytes_per_element": B,
        "roofline_model_frac": max(t_f, t_b) / (sec / args.steps),
        "hbm_write_gbs": E * B / kmean_s / 1e9,
        "fp64_tflops_alg": E * F / kmean_s / 1e12,
    })
    e2e_steps = args.e2e_steps or args.steps
    if e2e_steps > 0:
        e2e_dt, h2d, d2h = measure_e2e(ds, e2e_steps, world, device)
    else:  # development runs only (--e2e-steps -1): no end-to-end leg
        e2e_dt, h2d, d2h, e2e_steps = float("nan"), 0, 0, 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY 8(d)); random-init element maps",
        "config": {"workload": wl.name, "space": wl.space, "p_test": wl.p, "L": wl.L,
                   "path": wl.path, "maps": wl.maps, "elements_per_gpu": E,
                   "global_elements": E * world, "N": dim(wl.space, wl.orders),
                   "parallelism": f"element-shard x{world}",
                   "l2": "flushed (256 MB write) between timed steps; output per step "
                         f"{E * B / 2**20:.0f} MB"},
        "gram_entries_per_s": value * P,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": ds.launches_per_step * args.steps,
        "e2e": {"value": E * world * e2e_steps / e2e_dt if e2e_steps else None, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "hxg_gram_batched_host (C ABI, host buffers, pinned output)"},
    }
    line["shard_checksums"] = gather_checksums(ds.out, world, device)
    line["clocks_per_rank"] = gather_objects(clocks, world)
    if world > 1:
        # strong scaling on the same run: the config's global batch split over the ranks
        Eg = wl.E
        slo, shi = shard(Eg, world, rank)
        del ds
        torch.cuda.empty_cache()
        ds2, tms2, _, _ = measure_device(wl, shi - slo, slo, args.steps, args.warmup, world,
                                         device, with_clocks=False)
        tms2 = max_over_ranks(tms2, world, device)
        line["strong_scaling"] = {"global_elements": Eg, "elements_per_gpu": shi - slo,
                                  "value": Eg * args.steps / (tms2 / 1e3),
                                  "ms_per_step": tms2 / args.steps, "unit": UNIT}
        del ds2
    if args.suite and rank == 0 and world == 1:
        suite = []
        for name, w2 in WORKLOADS.items():
            d2, tms, kms, _ = measure_device(w2, w2.E, 0, max(3, args.steps // 2), 2, 1, device,
                                             with_clocks=False)
            F2, B2, P2 = algorithmic(w2.space, w2.orders, w2.path, w2.L)
            st = tms / 1e3 / max(3, args.steps // 2)
            km = statistics.mean(kms) / 1e3 if d2.full_metric else st
            tf2, tb2 = w2.E * F2 / (fp64 * 1e12), w2.E * B2 / (hbm * 1e9)
            suite.append({"workload": name, "elements_per_s": w2.E / st,
                          "gram_entries_per_s": w2.E * P2 / st, "ms_per_step": st * 1e3,
                          "kernel_ms": km * 1e3, "roofline_frac": max(tf2, tb2) / st,
                          "bound": "fp64" if tf2 >= tb2 else "hbm",
                          "fp64_tflops_alg": w2.E * F2 / km / 1e12,
                          "hbm_write_gbs": w2.E * B2 / km / 1e9})
            del d2
            torch.cuda.empty_cache()
        line["suite"] = suite
        line["dpg_suite"] = dpg_suite(device, fp64, hbm)
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, n, dt, threads = cpu_rate(wl, args.cpu_seconds)
        rate1, n1, dt1, _ = cpu_rate(wl, 3.0, 1)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{n} elements of {wl.name} in {dt:.1f} s "
                                          f"(oracle/hexgram_oracle.c, {threads} threads)",
                                "one_core_value": rate1,
                                "one_core_sample": f"{n1} elements in {dt1:.1f} s, 1 thread",
                                **cpu_host_info()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sweep(args, world, rank, local):
    """BASELINE config 5: H1/H(curl)/H(div), p_test = 2..10 (L = p + 1), affine and
    trilinear maps, E_p = floor(budget / B(p)) elements (<= 100 GB of packed fp64
    output), strong scaling over ranks (each rank integrates E_p / N elements).
    Reports elements/s, Gram-entries/s, roofline fraction per point and the
    fitted exponent of time-per-element vs p (p^7 general, p^6 affine expected
    for the FP64-bound points; HBM-bound points scale with the output, ~p^6)."""
    import torch

    from paper_1711_00984_b200 import _native
    from paper_1711_00984_b200.engine import get_engine
    from paper_1711_00984_b200.inputs import (affine_batch, extrusion_batch, packed_size,
                                              trilinear_batch)

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    eng = get_engine(device)
    lib = _native.lib()
    hbm, _, fp64, _ = peaks()
    budget = args.sweep_gb * 1e9
    pmax_out = max(packed_size(sp, (pp, pp, pp)) for sp in ("H1", "Hcurl", "Hdiv")
                   for pp in range(2, args.sweep_pmax + 1))
    out_all = torch.empty(int(budget // 8) + pmax_out, dtype=torch.float64, device=device)
    base_n = 4096
    results = []
    stream = torch.cuda.current_stream(device)
    for path, maps in (("general", "trilinear"), ("affine", "affine"), ("extrusion", "extrusion")):
        gen = {"trilinear": trilinear_batch, "affine": affine_batch, "extrusion": extrusion_batch}[maps]
        base = gen(base_n, 4)  # seed 4 (config 5)
        for space in ("H1", "Hcurl", "Hdiv"):
            for p in range(2, args.sweep_pmax + 1):
                orders = (p, p, p)
                L = p + 1 if path != "affine" else 1
                Pk = packed_size(space, orders)
                Eg = int(budget // (8 * Pk))
                lo, hi = shard(Eg, world, rank)
                E = hi - lo
                # the seeded base batch tiled on the device to E elements (timing only;
                # parity of these orders is covered by tests/test_gpu_parity.py)
                reps = (E + base_n - 1) // base_n
                kind = torch.as_tensor(base.kind).to(device).repeat(reps)[:E].contiguous()
                params = torch.as_tensor(base.params).to(device).repeat(reps, 1)[:E].contiguous()
                coef = torch.as_tensor(base.coef).to(device).repeat(reps)[:E].contiguous()
                status = torch.zeros(E, dtype=torch.int32, device=device)
                tab = eng.tables(L)
                sc, pc = _native.SPACE_CODES[space], _native.PATH_CODES[path]
                ws_bytes = lib.hxg_workspace_size(sc, pc, *orders, L, E)
                ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
                out = out_all[: E * Pk]
                ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

                def step():
                    rc = lib.hxg_gram_batched(sc, pc, *orders, L, E, ptr(kind), ptr(params), ptr(coef),
                                              None, ptr(tab), ptr(out), ptr(status), ptr(ws), ws_bytes,
                                              ctypes.c_void_p(stream.cuda_stream))
                    assert rc == 0, rc

                step()
                torch.cuda.synchronize(device)
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if world > 1:
                    import torch.distributed as dist

                    dist.barrier()
                ev0.record(stream)
                for _ in range(args.sweep_reps):
                    step()
                ev1.record(stream)
                torch.cuda.synchronize(device)
                sec = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / args.sweep_reps, world, device)
                F, B, _ = algorithmic(space, orders, path, L)
                t_roof = Eg / world * max(F / (fp64 * 1e12), B / (hbm * 1e9))
                results.append({"space": space, "path": path, "p_test": p, "L": L, "elements": Eg,
                                "elements_per_s": Eg / sec, "gram_entries_per_s": Eg * Pk / sec,
                                "ms": sec * 1e3, "roofline_frac": t_roof / sec,
                                "bound": "fp64" if F / fp64 / 1e3 > B / hbm else "hbm"})
                del kind, params, coef, status, ws
    fits = {}
    for path in ("general", "affine", "extrusion"):
        for space in ("H1", "Hcurl", "Hdiv"):
            for pmin in (2, 5):
                pts = [r for r in results if r["path"] == path and r["space"] == space
                       and r["p_test"] >= pmin]
                x = np.log([r["p_test"] for r in pts])
                y = np.log([1.0 / r["elements_per_s"] for r in pts])
                fits[f"{space}/{path}/p>={pmin}"] = float(np.polyfit(x, y, 1)[0]) if len(pts) > 1 else None
    if rank == 0:
        print(json.dumps({"metric": METRIC, "mode": "sweep (BASELINE config 5)", "n_gpus": world,
                          "scaling": "strong", "budget_gb_per_job": args.sweep_gb,
                          "fitted_time_exponent_vs_p": fits, "points": results}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2_h1_p5_general", choices=sorted(ALL_WORKLOADS))
    ap.add_argument("--elements", type=int, default=0, help="elements per GPU (default: config)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--suite", action=argparse.BooleanOptionalAction, default=True)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sweep", action="store_true", help="BASELINE config 5 order sweep")
    ap.add_argument("--sweep-gb", type=float, default=100.0)
    ap.add_argument("--sweep-pmax", type=int, default=10)
    ap.add_argument("--sweep-reps", type=int, default=2)
    args = ap.parse_args()
    rc = maybe_spawn(args, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference" and not args.sweep:
        # the reference arm is a host-CPU measurement: rank 0 runs it on the box's
        # cores and prints; the other ranks exit without work (no process group)
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if int(os.environ.get("RANK", "0")) == 0:
            run_reference(args, ALL_WORKLOADS[args.workload], world, 0)
        return
    world, rank, local = dist_setup(args)
    wl = ALL_WORKLOADS[args.workload]
    if args.sweep:
        run_sweep(args, world, rank, local)
    else:
        run_ours(args, wl, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
