"""C4 (1024^3 f32 quantised to 65536 levels) z-slab sharded over GPUs
(BASELINE config 4): one process per GPU (torchrun); rank r
generates its slab + halo planes on its GPU (v = (H >> 48) * 2^-16), runs
ecc_accumulate_slab with the affine bin map (k_affine_keys + the 16-bit
kernel), then ONE all-reduce of the 2 x 65536 int64 histogram (1 MiB) and K3.
Device time, max over ranks; the curve is checked against the Appendix-B
golden digest.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/c4_sharded.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402
from paper_2203_09087_b200.shard import shard_bounds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=5)
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
    sh = shard_bounds(S, world, rank)
    ctx = eb.Context(local)
    slab = torch.empty((sh.planes, S, S), dtype=torch.float32, device="cuda")
    ctx.fill_synthetic(slab, seed=1, base=sh.plane0 * S * S)
    bm = eb.quantised_binmap(65536)
    nb = 65536
    hist = torch.zeros(2 * nb, dtype=torch.int64, device="cuda")
    bins = torch.empty(nb, dtype=torch.int32, device="cuda")
    chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")

    def step():
        hist.zero_()
        ctx.accumulate_slab(slab, dims, sh.plane0, sh.own0, sh.own1, hist, binmap=bm)
        if dist is not None:
            dist.all_reduce(hist)
        ctx.finalize(hist, nb, bins, chg, chi, cnt)

    step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.reps):
        if dist is not None:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = min(ms)
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    m = int(cnt.item())
    ok = None
    if S == 1024:
        import json as _j
        gold = _j.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"]["C4"]
        vals = bins[:m].cpu().numpy().astype("float64") * 2.0 ** -16
        ok = oracle.curve_digest(vals, chi[:m].cpu().numpy()) == gold["digest"]
    if rank == 0:
        print(json.dumps({"config": f"C4 {S}^3 f32 65536 levels, {world} GPU(s)", "device_ms": t,
                          "gvox_s": S ** 3 / (t * 1e-3) / 1e9, "golden": ok, "points": m,
                          "backend": args.dist_backend if world > 1 else None}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
