"""GPU checks added in round 2: context state across a rejected call, the
fused exchange's failure path, and `bench.py --gpus 2` on a one-GPU box."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_rejected_nan_call_leaves_no_stale_flags(ctx):
    """A call rejected for a NaN must not fail the next call on the same
    context: here the next call is a >= 32 MB host u8 volume, which takes the
    overlapped path (its result block carries the context's error flags)."""
    bad = np.zeros((8, 8, 8), np.float32)
    bad[3, 3, 3] = np.nan
    with pytest.raises(eb.EccError, match="NaN"):
        ctx.vcec(bad)
    img = oracle.synth("u8", (128, 512, 512), seed=2)
    got = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(got.changes, c)
    # and the affine-grid rejection likewise
    off = np.full((4, 4, 4), 0.3, np.float32)
    with pytest.raises(eb.EccError, match="affine bin grid"):
        ctx.vcec(off, binmap=eb.quantised_binmap(16))
    assert np.array_equal(ctx.vcec(img).changes, c)


def test_fused_exchange_timeout_fails_loudly():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "tools", "xchg_timeout_check.py")],
                       capture_output=True, text=True, timeout=300)
    assert "TIMEOUT OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_fused_exchange_peer_process_killed():
    """A rank's process is SIGKILLed mid-run: the surviving rank's next fused
    launch must fail with ECC_ECUDA (timed out), a poisoned count, and not
    hang.  The two ranks are started directly (torchrun would tear the
    survivor down as soon as a worker dies)."""
    port = _port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tools",
                                                                    "xchg_timeout_check.py"),
                                       "--kill"], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    assert procs[1].returncode == -9, outs[1][1][-2000:]  # the killed rank
    assert procs[0].returncode == 0 and "KILL OK" in outs[0][0], outs[0][0][-2000:] + outs[0][1][-2000:]


def test_bench_two_ranks_self_launch():
    """`python bench.py --gpus 2` without torchrun re-launches itself with one
    process per rank; on a one-GPU box the ranks share the device over gloo.
    One valid JSON line, n_gpus 2, the C4 leg golden-exact, a C5 leg."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--legs", "c4,c5", "--c5-side", "512"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["value"] > 0 and out["e2e"]["value"] > 0
    assert out["legs"]["C4"]["golden_ok"] is True, out["legs"]
    assert out["legs"]["C5"].get("chi_end_is_1") is True, out["legs"]
