"""C5 (4096^3 u8 streamed from pinned host memory) sharded over GPUs
(SURVEY.md 8(e)): one process per GPU (torchrun), rank r holds only its
z-slab + halo planes of the volume in its own pinned host buffer, streams it
chunk by chunk through ecc_accumulate_host (pipelined DMA, each GPU on its own
PCIe link), then ONE all-reduce of the 2 x 256 int64 histogram and K3.  The
curve is checked (chi ends at 1; with --golden, the digest of the first 64
planes case is not applicable) and the time is the max over ranks.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/c5_sharded.py [--side 4096]
  python tools/c5_sharded.py --side 1024          # one GPU
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402
from paper_2203_09087_b200.shard import shard_bounds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=4096)
    ap.add_argument("--chunk-planes", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    S = args.side
    dims = eb.Dims(S, S, S)
    plane = S * S
    sh = shard_bounds(S, world, rank)
    ctx = eb.Context(local)
    # this rank's planes (+ halos) of the synthetic volume, generated on the
    # GPU piecewise and copied into pinned host memory (untimed)
    host = torch.empty((sh.planes, S, S), dtype=torch.uint8, pin_memory=True)
    step = max(1, (1 << 30) // plane)
    buf = torch.empty((min(step, sh.planes), S, S), dtype=torch.uint8, device="cuda")
    for p in range(sh.plane0, sh.plane1, step):
        q = min(p + step, sh.plane1)
        ctx.fill_synthetic(buf[: q - p], seed=1, base=p * plane)
        host[p - sh.plane0: q - sh.plane0].copy_(buf[: q - p])
    del buf
    torch.cuda.synchronize()
    n = sh.own1 - sh.own0
    bounds = list(range(sh.own0, sh.own1, args.chunk_planes)) + [sh.own1]
    hist = torch.zeros(512, dtype=torch.int64, device="cuda")
    bins = torch.empty(256, dtype=torch.int32, device="cuda")
    chg = torch.empty(256, dtype=torch.int64, device="cuda")
    chi = torch.empty(256, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    times = []
    for rep in range(args.reps):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hist.zero_()
        torch.cuda.synchronize()
        if n > 0:
            ctx.accumulate_host(host, sh.plane0, dims, bounds, hist)
        if dist is not None:
            dist.all_reduce(hist)
        ctx.finalize(hist, 256, bins, chg, chi, cnt)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = min(times)
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    m = int(cnt.item())
    ok = int(chi[m - 1].item()) == 1
    # the full 4096^3 curve against the reference engine's digest (golden.json C5_full)
    golden_ok = None
    if S == 4096:
        import hashlib
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"].get("C5_full")
        if gold is not None:
            h = hashlib.sha256()
            h.update(bins[:m].cpu().numpy().astype("<f8").tobytes())
            h.update(chi[:m].cpu().numpy().astype("<i8").tobytes())
            golden_ok = h.hexdigest() == gold["digest"]
    if rank == 0:
        print(json.dumps({"config": f"C5 {S}^3 u8 streamed from pinned host, {world} GPU(s)",
                          "seconds": t, "gvox_s": S ** 3 / t / 1e9,
                          "h2d_gbs_per_gpu": (sh.planes * plane) / t / 1e9, "chi_end_is_1": ok,
                          "golden_ok": golden_ok,
                          "points": m, "chunk_planes": args.chunk_planes,
                          "backend": args.dist_backend if world > 1 else None}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
