"""Failure path of the fused rank exchange (ecc_curve_sharded): rank 1 dies
(never launches) on the second step, so rank 0's launch times out waiting
for its histogram.  Rank 0 must then get no partial curve: the count is
poisoned, ecc_xchg_status fails with ECC_ECUDA, and every later
ecc_curve_sharded call on that exchange fails too (its step count is out of
step with its peers).  Runs as 2 processes on one GPU (CUDA IPC).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/xchg_timeout_check.py [--kill]

--kill: rank 1's PROCESS is killed (SIGKILL) before the second step instead
of merely skipping it; rank 0 must still get ECC_ECUDA, a poisoned count and
no hang (no collective runs after the kill).
"""
import os
import signal
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
    assert world == 2
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ctx = eb.Context(local)
    x = eb.Exchange(ctx, rank, world)
    handles = [None] * world
    dist.all_gather_object(handles, x.handle)
    x.open(handles)
    shape = (40, 48, 64)
    vol = oracle.synth("u8", shape, seed=7)
    dims = eb.Dims.of(shape)
    sh = shard_bounds(shape[0], world, rank)
    slab = torch.from_numpy(np.ascontiguousarray(vol[sh.plane0:sh.plane1])).cuda()
    bins = torch.empty(256, dtype=torch.int32, device="cuda")
    chg = torch.empty(256, dtype=torch.int64, device="cuda")
    chi = torch.empty(256, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")

    def launch():
        ctx.curve_sharded(x, slab, dims, sh.plane0, sh.own0, sh.own1, bins, chg, chi, cnt,
                          stream=ctx.stream)

    launch()  # step 1: both ranks
    x.status()
    v, c = oracle.vcec(vol)
    m = int(cnt.item())
    ok = np.array_equal(chg[:m].cpu().numpy(), c)
    dist.barrier()
    kill = "--kill" in sys.argv
    if kill and rank == 1:
        torch.cuda.synchronize()
        os.kill(os.getpid(), signal.SIGKILL)  # a rank dies mid-run
    result = "ok"
    if rank == 0:
        if kill:
            import time
            time.sleep(2.0)  # the peer is gone before this step starts
        launch()  # step 2: rank 1 is dead -> times out after 10 s
        try:
            x.status()
            result = "status did not fail"
        except eb.EccError as e:
            if "timed out" not in str(e):
                result = f"wrong error: {e}"
            elif e.code != -2:  # ECC_ECUDA
                result = f"wrong error code {e.code}"
        if result == "ok" and int(cnt.item()) != -1:  # ~0ull read as int64
            result = f"count not poisoned: {int(cnt.item())}"
        if result == "ok":
            try:
                launch()
                result = "next call did not fail"
            except eb.EccError as e:
                if "timed out" not in str(e):
                    result = f"wrong error on the next call: {e}"
    if kill:  # no collectives with a dead peer
        tag = "KILL"
        print(f"{tag} OK" if (ok and result == "ok") else f"{tag} FAILED: {result} step1={ok}",
              flush=True)
        x.close()
        os._exit(0)
    dist.barrier()
    if rank == 0:
        print("TIMEOUT OK" if (ok and result == "ok") else f"TIMEOUT FAILED: {result} step1={ok}",
              flush=True)
    x.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
