"""Multi-process check of the fused rank exchange (ecc_curve_sharded): every
rank holds a z-slab of the same synthetic volume, one fused launch per step
gives every rank the global curve; compared with the oracle (rank 0) for
several consecutive steps (both exchange parities).  Runs with any number of
ranks on one GPU (CUDA IPC between processes) or one rank per GPU.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/xchg_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402
from paper_2203_09087_b200.shard import shard_bounds  # noqa: E402


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ctx = eb.Context(local)
    x = eb.Exchange(ctx, rank, world)
    handles = [None] * world
    dist.all_gather_object(handles, x.handle)
    x.open(handles)
    ok = True
    for shape, seed in [((70, 48, 64), 3), ((33, 40, 32), 4), ((129, 30, 48), 5)]:
        vol = oracle.synth("u8", shape, seed=seed)
        dims = eb.Dims.of(shape)
        sh = shard_bounds(shape[0], world, rank)
        slab = torch.from_numpy(np.ascontiguousarray(vol[sh.plane0:sh.plane1])).cuda()
        bins = torch.empty(256, dtype=torch.int32, device="cuda")
        chg = torch.empty(256, dtype=torch.int64, device="cuda")
        chi = torch.empty(256, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        v, c = oracle.vcec(vol)
        for step in range(3):
            ctx.curve_sharded(x, slab, dims, sh.plane0, sh.own0, sh.own1, bins, chg, chi, cnt,
                              stream=ctx.stream)
            x.status()
            m = int(cnt.item())
            good = (np.array_equal(bins[:m].cpu().numpy(), v.astype(np.int32)) and
                    np.array_equal(chg[:m].cpu().numpy(), c) and
                    np.array_equal(chi[:m].cpu().numpy(), np.cumsum(c)))
            ok &= good
            if not good:
                print(f"rank {rank}: MISMATCH shape {shape} step {step}", flush=True)
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("XCHG OK" if int(flag) == 1 else "XCHG FAILED", world, "ranks", flush=True)
    x.close()
    dist.destroy_process_group()
    sys.exit(0 if int(flag) == 1 else 1)


if __name__ == "__main__":
    main()
