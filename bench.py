"""ECC benchmark -- BASELINE.json metric: GVoxels/s for 512^3 3D ECC.

Workload (config 2 of BASELINE.json, the one the metric is quoted on): each
rank owns a 512^3 u8 z-slab (axis-0 planes [512 r, 512 r + 512)) of a
(512 N) x 512 x 512 synthetic volume (v = counter_hash(1,
i) >> 56), plus one halo plane from each neighbouring slab.  One step at
N = 1 is ONE fused launch (ecc_curve_device: stencil + histogram + the last
CTA's compaction + prefix sum); at N > 1 it is also ONE launch per rank
(ecc_curve_sharded): K1+K2 over the slab, then the last CTA stores the rank's
2 x 256 int64 histogram into every peer's exchange buffer over NVLink (CUDA
IPC), waits for all ranks and runs K3 on the sum -- the all-reduce fused into
the kernel; NCCL all-reduce + K3 is the fallback (--no-p2p, or when the peer
mappings cannot be opened).  Per-GPU work is fixed as N grows ("scaling":
"weak").

* value     -- device-resident voxels/s (inputs already in HBM), CUDA events
               on the compute stream, max over ranks, L2 flushed (256 MiB
               write) between timed steps.
* e2e       -- the same metric through the public C ABI with a pinned HOST
               buffer (ecc_curve for N = 1: the H2D is split into plane chunks
               on a copy stream and each chunk's kernel runs as soon as it
               and its halo plane have landed; per-rank H2D + slab +
               exchange + K3 + D2H for N > 1), host<->device copies inside the
               timed region.
* roofline  -- the dominant kernel (k_u8_3d: K1+K2, with K3 fused at N = 1):
               algorithmic bytes (1 B/voxel read) / its CUDA-event time vs
               MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline -- the reference engine (oracle/_ref, compiled from the
               reference sources) on this host's cores, rank 0 at N = 1.
* legs      -- the other sharded configs north_star names, at the same N:
               C4 (1024^3 f32, 65536 levels, z-slab over the N GPUs, ONE
               all-reduce of the 1 MiB histogram, device time max over ranks)
               and C5 (4096^3 u8 streamed from each rank's own pinned host
               slab, GPU-local CPU affinity, ONE all-reduce).  Each is
               golden-checked (format-independent digest of the curve against
               tests/golden/golden.json, written by the reference engine)
               before its time is reported.

`--gpus N` without torchrun re-launches itself through torch.distributed.run
(one process per GPU).  When the box has fewer GPUs than ranks, the ranks
share devices over gloo (the line says so; such a time is not a scaling
number).  `--impl reference` times the reference CPU engine alone (rank 0;
other ranks exit) on the same config and metric.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIDE = 512
METRIC = "GVoxels/s for 512^3 3D ECC at 1/2/4/8 B200; % HBM roofline; vs CPU ref"
UNIT = "GVoxels/s"
WORKLOAD = "C2: 512^3 u8 3D ECC per GPU (z-slab of a (512N)x512x512 volume)"
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def base_config(n: int) -> dict:
    """The `config` both arms print (the driver compares them verbatim)."""
    return {"workload": WORKLOAD, "voxels_per_gpu": SIDE ** 3, "bins": 256,
            "parallelism": f"zslab{n}", "l2": "flushed between timed steps (256 MiB write)"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def curve_digest(thresholds, chi) -> str:
    """Format-independent SHA-256 of a curve (thresholds as float64 LE, then
    chi as int64 LE) -- the `digest` field of tests/golden/golden.json."""
    import numpy as np
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(thresholds, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(chi, dtype="<i8").tobytes())
    return h.hexdigest()


def golden(name):
    try:
        with open(GOLDEN) as f:
            return json.load(f)["configs"].get(name)
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every 5 ms while
    the timed region runs (the recipe's nvidia-smi clocks line, in-process)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self.reasons = set()
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: reported as no samples
            self.nv = None
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for name, b in bits.items():
                    if r & b:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        s = self.samples
        return {"sm_mhz": statistics.median(s) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def cpu_reference_run(steps: int, warmup: int, budget_s: float):
    """Times the reference engine on a bounded sample of the workload: the
    full 512^3 u8 volume per repetition, all host threads, CLI-default plan
    (workers = hardware_concurrency, chunks = max(2, workers))."""
    import oracle
    vol = oracle.synth("u8", (SIDE, SIDE, SIDE), seed=1)
    R = oracle.ref()
    cores = int(R.ref_hardware_concurrency()) or os.cpu_count() or 1
    for _ in range(max(0, warmup)):
        oracle.ref_vcec(vol, chunks=max(2, cores), workers=cores)
    times = []
    t_start = time.perf_counter()
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        v, c = oracle.ref_vcec(vol, chunks=max(2, cores), workers=cores)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    assert int(c.sum()) == 1
    best = min(times)
    mean = sum(times) / len(times)
    return {"value": SIDE ** 3 / mean / 1e9, "best": SIDE ** 3 / best / 1e9, "unit": UNIT,
            "cores": cores, "kind": "reference",
            "sample": f"full 512^3 u8 volume x {len(times)} reps (reference process_image + "
                      f"vcec_to_ecc, workers={cores}, chunks={max(2, cores)})",
            "ms_per_step": mean * 1e3, "reps": len(times)}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` (N > 1) without torchrun: one process per
    GPU through torch.distributed.run, exactly as the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Ranks:
    """The process group plumbing of one rank (torch.distributed)."""

    def __init__(self, backend_pref: str):
        import torch
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        ndev = max(1, torch.cuda.device_count())
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % ndev
        self.shared = self.world > ndev  # ranks time-slice devices
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.dist = None
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist
            self.backend = "gloo" if (self.shared or backend_pref == "gloo") else "nccl"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, *vals):
        import torch
        if self.dist is None:
            return vals
        t = torch.tensor(list(vals), dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return tuple(float(x) for x in t.tolist())

    def all_true(self, ok: bool) -> bool:
        import torch
        if self.dist is None:
            return ok
        t = torch.tensor([1 if ok else 0], device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return int(t.item()) == 1

    def all_reduce(self, t):
        if self.dist is not None:
            self.dist.all_reduce(t)


def check_curve(bins, chi, cnt, nbins: int, scale: float = 1.0, gold=None):
    """(ok, digest_ok): the curve is complete (count within range, final
    chi 1) and -- when a golden entry exists -- equals the reference's."""
    m = int(cnt.item())
    if not 0 < m <= nbins:
        return False, False
    c = chi[:m].cpu().numpy()
    ok = int(c[-1]) == 1
    if gold is None:
        return ok, None
    t = bins[:m].cpu().numpy().astype("float64") * scale
    return ok, curve_digest(t, c) == gold["digest"]


def leg_c4(R, ctx, reps: int):
    """BASELINE config 4: 1024^3 f32 quantised to 65536 levels, z-slab
    sharded over the N ranks, each rank's slab (+ halo planes) resident on its
    GPU; one step = the rank's K1+K2 (affine key pass + 16-bit kernel), ONE
    all-reduce of the 2 x 65536 int64 histogram, K3."""
    import torch
    import paper_2203_09087_b200 as eb
    from paper_2203_09087_b200.shard import shard_bounds
    S, nb = 1024, 65536
    dims = eb.Dims(S, S, S)
    sh = shard_bounds(S, R.world, R.rank)
    slab = torch.empty((sh.planes, S, S), dtype=torch.float32, device=R.dev)
    ctx.fill_synthetic(slab, seed=1, base=sh.plane0 * S * S)
    bm = eb.quantised_binmap(nb)
    hist = torch.zeros(2 * nb, dtype=torch.int64, device=R.dev)
    bins = torch.empty(nb, dtype=torch.int32, device=R.dev)
    chg = torch.empty(nb, dtype=torch.int64, device=R.dev)
    chi = torch.empty(nb, dtype=torch.int64, device=R.dev)
    cnt = torch.empty(1, dtype=torch.int64, device=R.dev)

    def step():
        hist.zero_()
        if sh.own1 > sh.own0:
            ctx.accumulate_slab(slab, dims, sh.plane0, sh.own0, sh.own1, hist, binmap=bm)
        R.all_reduce(hist)
        ctx.finalize(hist, nb, bins, chg, chi, cnt)

    step()
    torch.cuda.synchronize()
    ok, gok = check_curve(bins, chi, cnt, nb, 2.0 ** -16, golden("C4"))
    ms = []
    for _ in range(reps):
        R.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ok2, gok2 = check_curve(bins, chi, cnt, nb, 2.0 ** -16, golden("C4"))
    t = statistics.median(ms)
    (t,) = R.max(t)
    good = R.all_true(bool(ok and ok2 and gok and gok2))
    del slab
    torch.cuda.empty_cache()
    return {"workload": "C4: 1024^3 f32, 65536 levels, z-slab over N GPUs + one all-reduce",
            "value": S ** 3 / (t * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": t, "reps": reps,
            "golden_ok": good, "timing": "device (CUDA events), median of reps, max over ranks",
            "bytes_per_gpu": sh.planes * S * S * 4}


def pinned_host(shape):
    """An exactly-sized page-locked host array (anonymous mmap, pages
    first-touched by this thread, then cudaHostRegister) -- torch's pinned
    allocator rounds large requests up to a power of two, which would double a
    C5 rank's 8-32 GiB slab."""
    import mmap

    import numpy as np
    import torch
    n = 1
    for d in shape:
        n *= d
    mm = mmap.mmap(-1, max(n, 1), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    arr = np.frombuffer(mm, dtype=np.uint8, count=n).reshape(shape)
    t = torch.from_numpy(arr)
    rt = torch.cuda.cudart()
    err = rt.cudaHostRegister(t.data_ptr(), n, 0)
    if int(err) != 0:
        raise RuntimeError(f"cudaHostRegister of {n} bytes failed ({err})")

    def unpin():
        rt.cudaHostUnregister(t.data_ptr())
    return t, unpin


def _gpu_local_affinity(local: int) -> str:
    """Pins this rank's threads to the CPUs nearest its GPU (NVML), so the
    pinned host slab it allocates next is first-touched on that NUMA node."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        nv.nvmlDeviceSetCpuAffinity(nv.nvmlDeviceGetHandleByIndex(local))
        return f"gpu-local ({len(os.sched_getaffinity(0))} cpus)"
    except Exception as e:
        return f"default ({str(e)[:40]})"


def leg_c5(R, ctx, reps: int, side: int):
    """BASELINE config 5: 4096^3 u8 streamed from pinned host memory.  Rank r
    holds only its z-slab + halo planes in its own pinned buffer (allocated
    after pinning the rank to its GPU's CPUs) and streams it in 64-plane
    chunks over its own PCIe link (ecc_accumulate_host: copy stream || K1+K2),
    then ONE all-reduce of the 2 x 256 histogram and K3.  The timed region
    includes every H2D copy."""
    import torch
    import paper_2203_09087_b200 as eb
    from paper_2203_09087_b200.shard import shard_bounds
    S = side
    dims = eb.Dims(S, S, S)
    plane = S * S
    sh = shard_bounds(S, R.world, R.rank)
    need = sh.planes * plane
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = None
    # every rank of this node allocates its share: skip if the node cannot hold it
    share_ok = avail is None or avail > 1.25 * need * R.world
    if not R.all_true(share_ok):
        return {"workload": f"C5: {S}^3 u8 streamed", "skipped":
                f"host memory: {need * R.world / 2**30:.0f} GiB pinned needed, "
                f"{(avail or 0) / 2**30:.0f} GiB free"}
    affinity = _gpu_local_affinity(R.local) if R.world > 1 else "default (one rank)"
    host, unpin = pinned_host((sh.planes, S, S))
    step = max(1, (1 << 30) // plane)
    buf = torch.empty((min(step, sh.planes), S, S), dtype=torch.uint8, device=R.dev)
    for p in range(sh.plane0, sh.plane1, step):
        q = min(p + step, sh.plane1)
        ctx.fill_synthetic(buf[: q - p], seed=1, base=p * plane)
        host[p - sh.plane0: q - sh.plane0].copy_(buf[: q - p])
    del buf
    torch.cuda.synchronize()
    bounds = list(range(sh.own0, sh.own1, 64)) + [sh.own1]
    hist = torch.zeros(512, dtype=torch.int64, device=R.dev)
    bins = torch.empty(256, dtype=torch.int32, device=R.dev)
    chg = torch.empty(256, dtype=torch.int64, device=R.dev)
    chi = torch.empty(256, dtype=torch.int64, device=R.dev)
    cnt = torch.empty(1, dtype=torch.int64, device=R.dev)
    cs = torch.cuda.ExternalStream(ctx.stream, device=R.dev)
    ms = []
    for _ in range(reps):
        hist.zero_()
        R.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)  # the context's streams carry every copy and kernel
        if sh.own1 > sh.own0:
            ctx.accumulate_host(host, sh.plane0, dims, bounds, hist)
        with torch.cuda.stream(cs):
            R.all_reduce(hist)
            ctx.finalize(hist, 256, bins, chg, chi, cnt, stream=ctx.stream)
        b.record(cs)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    gold = golden("C5_full") if S == 4096 else None
    ok, gok = check_curve(bins, chi, cnt, 256, 1.0, gold)
    t = statistics.median(ms)
    (t,) = R.max(t)
    good = R.all_true(bool(ok and (gok is not False)))
    unpin()
    del host
    return {"workload": f"C5: {S}^3 u8 streamed from per-rank pinned host slabs (64-plane chunks)",
            "value": S ** 3 / (t * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": t, "reps": reps,
            "golden_ok": good if gold is not None else None, "chi_end_is_1": ok,
            "h2d_gbs_per_gpu": sh.planes * plane / (t * 1e-3) / 1e9, "host_affinity": affinity,
            "timing": "device (CUDA events on the context stream, H2D inside), median, max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-p2p", action="store_true",
                    help="N > 1: NCCL all-reduce instead of the exchange fused into the launch")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--legs", default="c4,c5",
                    help="extra sharded configs to time after C2 (comma list of c4, c5; 'none')")
    ap.add_argument("--c5-side", type=int, default=4096)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the N > 1 path on a box with fewer GPUs "
                         "(chosen automatically when ranks must share devices)")
    args = ap.parse_args()
    warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n = world

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference_run(args.steps, warmup, budget_s=240.0)
        out = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": n,
               "steps": cb["reps"], "warmup": warmup, "ms_per_step": cb["ms_per_step"],
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
               "data": "synthetic (counter_hash seed 1, SURVEY.md 8(d))", "impl": "reference",
               "config": base_config(n),
               "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
               "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    import paper_2203_09087_b200 as eb

    R = Ranks(args.dist_backend)
    dist, local, dev = R.dist, R.local, R.dev
    ctx = eb.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    # ---------------- data: this rank's slab + halo planes
    from paper_2203_09087_b200.shard import shard_bounds, sharded_histogram
    W0 = SIDE * n
    sh = shard_bounds(W0, n, rank)  # weak scaling: 512 planes per rank
    own0, own1, p0, p1 = sh.own0, sh.own1, sh.plane0, sh.plane1
    dims = eb.Dims(W0, SIDE, SIDE)
    plane = SIDE * SIDE
    slab = torch.empty(((p1 - p0), SIDE, SIDE), dtype=torch.uint8, device=dev)
    # every device call below reads planes [p0, p1) of the (512N)-plane image:
    # the slab must hold exactly those (owned planes + halo planes)
    assert own1 - own0 == SIDE and p0 <= max(own0 - 1, 0) and p1 >= min(own1 + 1, W0)
    assert slab.shape[0] == p1 - p0
    ctx.fill_synthetic(slab, seed=1, base=p0 * plane)
    hist = torch.zeros(512, dtype=torch.int64, device=dev)
    bins = torch.empty(256, dtype=torch.int32, device=dev)
    chg = torch.empty(256, dtype=torch.int64, device=dev)
    chi = torch.empty(256, dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    # N > 1: the histogram exchange fused into the stencil launch over peer
    # memory (ecc_curve_sharded, CUDA IPC + NVLink stores); NCCL all-reduce
    # if the peer mappings cannot be set up or disagree with it
    xchg = None
    exchange = "none" if dist is None else f"{R.backend}_allreduce"
    if dist is not None and not args.no_p2p:
        # every collective below is reached by every rank whatever fails
        # locally, so a rank whose peer mappings fail cannot strand the others
        x, why = None, ""
        try:
            x = eb.Exchange(ctx, rank, world)
            h = x.handle
        except Exception as e:
            h, why = None, str(e)[:80]
        handles = [None] * world
        dist.all_gather_object(handles, h)
        ok = all(hh is not None for hh in handles)  # the same on every rank
        if ok:
            try:
                x.open(handles)
            except Exception as e:
                ok, why = False, str(e)[:80]
            ok = R.all_true(ok)
        if ok:
            ref = []
            try:
                for use in (None, x):  # one all-reduce step, one fused step: same curve?
                    with torch.cuda.stream(stream):
                        if use is None:
                            hist.zero_()
                            sharded_histogram(sh, lambda shd, h: ctx.accumulate_slab(
                                slab, dims, shd.plane0, shd.own0, shd.own1, h, stream=ctx.stream),
                                hist, dist.all_reduce)
                            ctx.finalize(hist, 256, bins, chg, chi, cnt, stream=ctx.stream)
                        else:
                            ctx.curve_sharded(x, slab, dims, p0, own0, own1, bins, chg, chi, cnt,
                                              stream=ctx.stream)
                    torch.cuda.synchronize()
                    if use is not None:
                        x.status()
                    ref.append((cnt.clone(), chi.clone(), bins.clone()))
                same = all(torch.equal(a, b) for a, b in zip(ref[0], ref[1]))
            except Exception as e:  # fall back to the all-reduce, reported in the JSON
                same, why = False, str(e)[:80]
            ok = R.all_true(same)
        if ok:
            xchg, exchange = x, "p2p_fused_exchange"
        else:
            if x is not None:
                try:
                    x.close()
                except Exception:
                    pass
            exchange = f"{R.backend}_allreduce" + (f" (p2p setup failed: {why})" if why else "")

    def step(ev_k0=None, ev_k1=None):
        with torch.cuda.stream(stream):
            if xchg is not None:
                # K1+K2 + exchange over peer memory + K3: ONE launch
                if ev_k0 is not None:
                    ev_k0.record(stream)
                ctx.curve_sharded(xchg, slab, dims, p0, own0, own1, bins, chg, chi, cnt,
                                  stream=ctx.stream)
                if ev_k1 is not None:
                    ev_k1.record(stream)
                return
            if dist is None:
                # whole volume on one GPU: ONE fused launch (K1+K2+K3)
                if ev_k0 is not None:
                    ev_k0.record(stream)
                ctx.curve_device(slab, dims, bins, chg, chi, cnt, stream=ctx.stream)
                if ev_k1 is not None:
                    ev_k1.record(stream)
                return
            hist.zero_()

            def accumulate(shard, h):
                if ev_k0 is not None:
                    ev_k0.record(stream)
                ctx.accumulate_slab(slab, dims, shard.plane0, shard.own0, shard.own1, h,
                                    stream=ctx.stream)
                if ev_k1 is not None:
                    ev_k1.record(stream)

            sharded_histogram(sh, accumulate, hist, dist.all_reduce)  # ONE all-reduce
            ctx.finalize(hist, 256, bins, chg, chi, cnt, stream=ctx.stream)

    # correctness of what we time: the global curve equals the reference's
    # (N = 1: the C2 golden digest) and ends at chi == 1
    gold_c2 = golden("C2") if n == 1 else None
    step()
    torch.cuda.synchronize()
    ok0, g0 = check_curve(bins, chi, cnt, 256, 1.0, gold_c2)
    assert ok0 and g0 is not False, "bench volume failed the curve check before timing"

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    # K steps enqueued back to back (the host runs ahead, so launch latency is
    # hidden behind the previous step's L2 flush); each step is bracketed by
    # CUDA events on the compute stream, the whole region by barrier + sync.
    # A fused step is ONE kernel launch, so its bracket is the kernel's time
    # too; the NCCL fallback step (accumulate, all-reduce, finalize) also
    # brackets its accumulate kernel for the roofline.
    single_launch = xchg is not None or dist is None
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    R.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            a, b, k0, k1 = evs[i]
            with torch.cuda.stream(stream):
                flush.fill_(1)  # evict L2 (126 MB) between timed steps
            a.record(stream)
            if single_launch:
                step()
            else:
                step(k0, k1)
            b.record(stream)
        torch.cuda.synchronize()
        R.barrier()
    launches = ctx.launch_count() - l0
    # the last timed step's curve must still be the whole, exact one (a peer
    # that timed out in the fused exchange poisons the count and the status)
    if xchg is not None:
        xchg.status()
    ok1, g1 = check_curve(bins, chi, cnt, 256, 1.0, gold_c2)
    assert R.all_true(ok1 and g1 is not False), "curve check failed after the timed steps"
    step_ms = [a.elapsed_time(b) for a, b, _, _ in evs]
    kern_ms = step_ms if single_launch else [k0.elapsed_time(k1) for _, _, k0, k1 in evs]
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kern_ms) / len(kern_ms)
    t_step, t_kern = R.max(t_step, t_kern)
    voxels_total = SIDE ** 3 * n
    value = voxels_total / (t_step * 1e-3) / 1e9

    # ---------------- e2e through the public API, host pinned input
    host = torch.empty(((p1 - p0), SIDE, SIDE), dtype=torch.uint8, pin_memory=True)
    host.copy_(slab.cpu())
    h2d = host.numel()
    e2e_ms = []
    if n == 1:
        arr = host.numpy()
        for i in range(warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cur = ctx.curve(arr)
            dt = time.perf_counter() - t0
            if i >= warmup:
                e2e_ms.append(dt * 1e3)
        assert int(cur.chi[-1]) == 1
        d2h = cur.size() * (1 + 8) + 8
    else:
        buf = torch.empty_like(slab)
        hcur = torch.empty((3, 256), dtype=torch.int64, pin_memory=True)
        for i in range(warmup + args.steps):
            R.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                buf.copy_(host, non_blocking=True)
                if xchg is not None:
                    ctx.curve_sharded(xchg, buf, dims, p0, own0, own1, bins, chg, chi, cnt,
                                      stream=ctx.stream)
                else:
                    hist.zero_()
                    ctx.accumulate_slab(buf, dims, p0, own0, own1, hist, stream=ctx.stream)
                    dist.all_reduce(hist)
                    ctx.finalize(hist, 256, bins, chg, chi, cnt, stream=ctx.stream)
                hcur[0].copy_(bins.to(torch.int64), non_blocking=True)
                hcur[1].copy_(chi, non_blocking=True)
            stream.synchronize()
            dt = time.perf_counter() - t0
            if i >= warmup:
                e2e_ms.append(dt * 1e3)
        if xchg is not None:
            xchg.status()
        d2h = 256 * 8 * 2
    t_e2e = sum(e2e_ms) / len(e2e_ms)
    (t_e2e,) = R.max(t_e2e)
    e2e_value = voxels_total / (t_e2e * 1e-3) / 1e9

    # ---------------- roofline of K1+K2
    peak, peak_kind = _peaks()
    alg_bytes = SIDE ** 3  # 1 B/voxel read once; the 4 KB histogram is negligible
    achieved = alg_bytes / (t_kern * 1e-3) / 1e9
    traffic = None
    pipes = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            nt = json.load(f)
        traffic = nt.get("k1k2_dram_bytes_per_launch")
        if "alu_pipe_busy_pct" in nt:
            # what bounds the kernel instead of HBM (ncu --set full of the same kernel)
            pipes = {"bound": nt.get("bound", "integer ALU pipe"),
                     "alu_busy_pct": nt["alu_pipe_busy_pct"],
                     "fma_busy_pct": nt.get("fma_pipe_busy_pct"),
                     "issue_active_pct": nt.get("issue_active_pct"),
                     "warp_instr_per_step": nt.get("warp_instr_per_step"),
                     "source": nt.get("source")}
    except Exception:
        pass

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
           "warmup": warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (counter_hash seed 1, SURVEY.md 8(d)); device-generated",
           "config": base_config(n),
           "checks": {"exchange": exchange if n > 1 else None,
                      "golden_c2": bool(g1) if n == 1 else None,
                      "chi_end_is_1": bool(ok1), "devices_shared": R.shared},
           "kernel_ms": t_kern,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind},
           "compute_limit": pipes,
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e},
           "gpu_launches": launches,
           "clocks": clocks.summary()}
    if R.shared:
        out["checks"]["note"] = ("ranks share GPUs over gloo: a functional run of the N-rank "
                                 "path, not a scaling number")

    # ---------------- the other sharded configs north_star names (same N)
    del host
    legs = {}
    want = [s.strip() for s in args.legs.split(",") if s.strip() and s.strip() != "none"]
    for name in want:
        try:
            if name == "c4":
                legs["C4"] = leg_c4(R, ctx, reps=5)
            elif name == "c5":
                legs["C5"] = leg_c5(R, ctx, reps=2, side=args.c5_side)
        except Exception as e:  # reported; the C2 line stands on its own
            legs[name.upper()] = {"error": str(e)[:200]}
    if legs:
        out["legs"] = legs

    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_run(3, 1, budget_s=args.cpu_budget)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # reported, never fatal for the GPU number
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if xchg is not None:
        xchg.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
