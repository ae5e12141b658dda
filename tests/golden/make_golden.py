"""Generates tests/golden/golden.json with the UNMODIFIED reference engine.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

For each BASELINE config input (seed 1) it runs the
reference's process_image + vcec_to_ecc (compiled in place by
``make -C oracle ref``), formats the curve with the reference's own
write_curve, and records:
  * csv_sha256  -- SHA-256 of the reference CSV bytes (must equal SURVEY.md
                   Appendix B, asserted below),
  * digest      -- oracle.curve_digest (float64 thresholds + int64 chi), the
                   format-independent hash the GPU tests compare against on
                   the GPU box, where the reference is absent,
  * points / first / final / min / max.
Small hand fixtures (acceptance.cpp:169-200, test_kernel.cpp:85-116,
test_oracle.cpp:100-119, test_streaming.cpp:84-120) are recorded with their
full expected curves from the reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

APPENDIX_B = {
    "C1": "83ee98223e5e1e49f5ff79581f2f1907e14ba9ef3f59ab9b093c3c732c10fd41",
    "C2": "94c004b9334de29b436dc8923f84b07e8a3ae8c3e14662a36c0a0daf57eeddca",
    "C3_0": "190e7c093b33689f433ea9b7235a8f2229840b369361d28430a22d9df7574836",
    "C3_4095": "bb3f52565af1b4d6faed6ea727862f3e5cf45e3f81eeb09840ea483899368842",
    "C4": "dd3b90fa2b5a0dfb7b49a098a675f621d23c7ac96cd88aa562323fcc65749384",
    "C5_64": "411d82ae28a1b305cbf5ad381e947a77b3a1a4c6e32bab372545328bc9fd9b75",
}


def record(name, img, workers):
    t0 = time.time()
    t, chi = oracle.ref_curve(img, chunks=max(2, workers), workers=workers)
    dt = time.time() - t0
    csv = oracle.ref_csv(t, chi)
    sha = hashlib.sha256(csv).hexdigest()
    rec = {
        "shape": list(img.shape), "dtype": str(img.dtype),
        "points": int(len(t)), "first": [float(t[0]), int(chi[0])],
        "final": int(chi[-1]), "min": int(chi.min()), "max": int(chi.max()),
        "csv_sha256": sha, "digest": oracle.curve_digest(t, chi),
        "ref_seconds": round(dt, 3),
    }
    ok = APPENDIX_B.get(name) == sha
    print(f"{name}: {rec['points']} points, sha {'OK' if ok else 'MISMATCH'} ({dt:.1f}s)", flush=True)
    assert ok, (name, sha)
    return rec


def hand_fixtures():
    fx = {
        "ring_3x3": (np.array([[0, 0, 0], [0, 9, 0], [0, 0, 0]], np.float32), None),
        "staircase_2x2": (np.array([[1, 2], [3, 4]], np.float32), None),
        "checkerboard_2x2": (np.array([[0, 1], [1, 0]], np.float32), None),
        "single_voxel_2d": (np.array([[3.5]], np.float32), None),
        "single_value_3d": (np.full((1, 1, 2), 3.5, np.float32), None),
        "constant_cube_2x2x2": (np.ones((2, 2, 2), np.float32), None),
        "u8_ring_keeps_zero_change": (np.array([[0, 0, 0], [0, 9, 0], [0, 0, 0]], np.uint8), None),
        "negzero_2x2": (np.array([[-0.0, 0.0], [1.0, -0.0]], np.float32), None),
        "posinf_1x1": (np.array([[np.inf]], np.float32), None),
        "posinf_corner_2x2": (np.array([[1.0, 2.0], [3.0, np.inf]], np.float32), None),
        "posinf_first_2x2": (np.array([[np.inf, 2.0], [3.0, 4.0]], np.float32), None),
        "neginf_3d": (np.array([[[-np.inf, 1.0], [2.0, 3.0]]], np.float32), None),
    }
    out = {}
    for name, (img, _) in fx.items():
        v, c = oracle.ref_vcec(img)
        out[name] = {"image": img.tolist(), "shape": list(img.shape), "dtype": str(img.dtype),
                     "values": [float(x) for x in v], "changes": [int(x) for x in c]}
    return out


def random_fixtures():
    """A handful of small random images with the reference's full VCEC."""
    rng = np.random.default_rng(20260101)
    out = []
    for t in range(24):
        d = (int(rng.integers(1, 9)), int(rng.integers(1, 9))) if t % 2 == 0 else \
            tuple(int(x) for x in rng.integers(1, 7, 3))
        kind = ("u8", "f32", "u16")[t % 3]
        if kind == "u8":
            img = rng.integers(0, 8, d).astype(np.uint8)
        elif kind == "u16":
            img = rng.integers(0, 6, d).astype(np.uint16)
        else:
            pool = rng.random(5).astype(np.float32)
            img = pool[rng.integers(0, 5, d)]
        v, c = oracle.ref_vcec(img, chunks=1 + t % 3)
        out.append({"image": img.ravel().tolist(), "shape": list(img.shape), "dtype": str(img.dtype),
                    "values": [float(x) for x in v], "changes": [int(x) for x in c]})
    return out


def main():
    oracle.build(ref=True)
    workers = max(1, os.cpu_count() or 1)
    g = {"_about": __doc__.strip().splitlines()[0], "configs": {}}
    g["hand"] = hand_fixtures()
    g["random"] = random_fixtures()
    cfg = g["configs"]
    cfg["C1"] = record("C1", oracle.synth("u8", (256, 256)), 1)
    cfg["C2"] = record("C2", oracle.synth("u8", (512, 512, 512)), workers)
    for b in (0, 4095):
        img = oracle.synth("u16", (512, 512), seed=1, base=b * 512 * 512)
        cfg[f"C3_{b}"] = record(f"C3_{b}", img, 1)
    cfg["C5_64"] = record("C5_64", oracle.synth("u8", (64, 4096, 4096)), workers)
    if "--skip-c4" not in sys.argv:
        cfg["C4"] = record("C4", oracle.synth("f32q", (1024, 1024, 1024)), workers)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
