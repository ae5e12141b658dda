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
mappings cannot be opened).  Per-GPU work is fixed as
N grows ("scaling": "weak").

* value     -- device-resident voxels/s (inputs already in HBM), CUDA events
               on the compute stream, max over ranks, L2 flushed (256 MiB
               write) between timed steps.
* e2e       -- the same metric through the public C ABI with a pinned HOST
               buffer (ecc_curve for N = 1: the H2D is split into plane chunks
               on a copy stream and each chunk's kernel runs as soon as it
               and its halo plane have landed; per-rank H2D + slab +
               all-reduce + finalize + D2H for N > 1), host<->device copies
               inside the timed region.
* roofline  -- the dominant kernel (k_u8_3d: K1+K2, with K3 fused at N = 1):
               algorithmic bytes (1 B/voxel read) / its CUDA-event time vs
               MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline -- the reference engine (oracle/_ref, compiled from the
               reference sources) on this host's cores, rank 0 at N = 1.

`--impl reference` times the reference CPU engine alone (rank 0; other ranks
exit) on the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
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


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
            self._stop.wait(0.005)

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
    import numpy as np
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
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the N > 1 path on a box with fewer GPUs "
                         "(ranks then share devices; the timing is not a scaling number)")
    args = ap.parse_args()
    warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = world if world > 1 else args.gpus

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference_run(args.steps, min(args.warmup, 1), budget_s=240.0)
        out = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": n,
               "steps": cb["reps"], "warmup": min(args.warmup, 1), "ms_per_step": cb["ms_per_step"],
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
               "data": "synthetic (counter_hash seed 1, SURVEY.md 8(d))", "impl": "reference",
               "config": {"workload": "C2: 512^3 u8 3D ECC (reference CPU engine, one volume per step)",
                          "voxels_per_step": SIDE ** 3},
               "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
               "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import numpy as np
    import torch
    import paper_2203_09087_b200 as eb

    local = local % max(1, torch.cuda.device_count())  # gloo test runs may share a GPU
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    ctx = eb.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # ---------------- data: this rank's slab + halo planes
    from paper_2203_09087_b200.shard import shard_bounds, sharded_histogram
    W0 = SIDE * n
    sh = shard_bounds(W0, n, rank)  # weak scaling: 512 planes per rank
    own0, own1, p0, p1 = sh.own0, sh.own1, sh.plane0, sh.plane1
    dims = eb.Dims(W0, SIDE, SIDE)
    plane = SIDE * SIDE
    slab = torch.empty(((p1 - p0), SIDE, SIDE), dtype=torch.uint8, device=dev)
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
    exchange = "none" if dist is None else "nccl_allreduce"
    if dist is not None and not args.no_p2p:
        try:
            x = eb.Exchange(ctx, rank, world)
            handles = [None] * world
            dist.all_gather_object(handles, x.handle)
            x.open(handles)
            ref = []
            for use in (None, x):  # one NCCL step, one fused step: same curve?
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
            agree = torch.tensor([1 if same else 0], device=dev)
            dist.all_reduce(agree, op=dist.ReduceOp.MIN)
            if int(agree.item()) == 1:
                xchg, exchange = x, "p2p_fused_exchange"
            else:
                x.close()
        except Exception as e:  # fall back to NCCL, reported in the JSON
            exchange = f"nccl_allreduce (p2p setup failed: {str(e)[:80]})"
        flag = torch.tensor([1 if xchg is not None else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0 and xchg is not None:  # every rank must agree
            xchg.close()
            xchg, exchange = None, "nccl_allreduce"

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

    # correctness of what we time: final chi of a complete volume is 1
    step()
    torch.cuda.synchronize()
    m = int(cnt.item())
    assert int(chi[m - 1].item()) == 1, "bench volume failed the chi == 1 check"

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    step_ms, kern_ms = [], []
    # K steps enqueued back to back (the host runs ahead, so launch latency is
    # hidden behind the previous step's L2 flush); each step is bracketed by
    # CUDA events on the compute stream, the whole region by barrier + sync.
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            a, b, k0, k1 = evs[i]
            with torch.cuda.stream(stream):
                flush.fill_(1)  # evict L2 (126 MB) between timed steps
            a.record(stream)
            step(k0, k1)
            b.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b, _, _ in evs]
    kern_ms = [k0.elapsed_time(k1) for _, _, k0, k1 in evs]
    launches = ctx.launch_count() - l0
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kern_ms) / len(kern_ms)
    if dist is not None:
        t = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, t_kern = float(t[0]), float(t[1])
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
            dist.barrier()
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
        d2h = 256 * 8 * 2
    t_e2e = sum(e2e_ms) / len(e2e_ms)
    if dist is not None:
        t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t[0])
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
            pipes = {"bound": "integer ALU pipe", "alu_busy_pct": nt["alu_pipe_busy_pct"],
                     "fma_busy_pct": nt.get("fma_pipe_busy_pct"),
                     "issue_active_pct": nt.get("issue_active_pct"), "source": nt.get("source")}
    except Exception:
        pass

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
           "warmup": warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (counter_hash seed 1, SURVEY.md 8(d)); device-generated",
           "config": {"workload": "C2: 512^3 u8 3D ECC per GPU (z-slab of a (512N)x512x512 volume)",
                      "voxels_per_gpu": SIDE ** 3, "bins": 256,
                      "parallelism": f"zslab{n}" + (f"+{exchange}" if n > 1 else ""),
                      "l2": "flushed between timed steps (256 MiB write)"},
           "kernel_ms": t_kern,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind},
           "compute_limit": pipes,
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e},
           "gpu_launches": launches,
           "clocks": clocks.summary()}
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
