"""CPU tests of the drop-in boundary and the host logic (no GPU compute)."""
import os
import re

import numpy as np
import pytest

import paper_2203_09087_b200 as eb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "ecc_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^ECC_API [^;]*?\b(ecc_\w+)\(", src, flags=re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = eb.lib()
    syms = _declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert L.ecc_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(eb.EccError) as ei:
        eb.Context(0)
    assert ei.value.code == eb.ECC_ECUDA


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2203_09087_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "_ref/" not in txt, fn


def test_bin_count():
    import ctypes as C
    n = C.c_uint64()
    assert eb.lib().ecc_bin_count(eb.ECC_U8, None, C.byref(n)) == 0 and n.value == 256
    assert eb.lib().ecc_bin_count(eb.ECC_U16, None, C.byref(n)) == 0 and n.value == 65536
    bm = eb._BinMap(eb.ECC_BIN_AFFINE, 65536, 0.0, 2.0 ** -16)
    assert eb.lib().ecc_bin_count(eb.ECC_F32, C.byref(bm), C.byref(n)) == 0 and n.value == 65536
    bad = eb._BinMap(eb.ECC_BIN_AFFINE, 0, 0.0, 1.0)
    assert eb.lib().ecc_bin_count(eb.ECC_F32, C.byref(bad), C.byref(n)) == eb.ECC_EINVAL


# ---- plan_chunks, mirroring test_streaming.cpp:13-66
def test_plan_ceiling_lengths():
    p = eb.plan_chunks(eb.Dims(10, 1, 1), eb.ChunkTarget.count(3))
    assert [(r.begin, r.end) for r in p.ranges] == [(0, 4), (4, 8), (8, 10)]


def test_plan_one_chunk_identity():
    p = eb.plan_chunks(eb.Dims(5, 1, 1), eb.ChunkTarget.count(1))
    assert [(r.begin, r.end) for r in p.ranges] == [(0, 5)]


def test_plan_invariants():
    for w0 in (1, 2, 3, 7, 10, 64, 100):
        for c in (1, 2, 3, 5, 8, 200):
            p = eb.plan_chunks(eb.Dims(w0, 4, 4), eb.ChunkTarget.count(c))
            eff = min(max(c, 1), w0)
            mx = (w0 + eff - 1) // eff
            b = 0
            for r in p.ranges:
                assert r.begin == b and r.end > r.begin and r.len() <= mx
                b = r.end
            assert b == w0


def test_budget_plan_within_budget():
    d = eb.Dims(4096, 512, 512)
    budget = 64 << 20
    p = eb.plan_chunks(d, eb.ChunkTarget.memory_budget(budget))
    assert eb.padded_chunk_bytes(d, max(r.len() for r in p.ranges)) <= budget


def test_infeasible_budget_names_minimum():
    d = eb.Dims(8, 1024, 1024)
    with pytest.raises(eb.EccError) as ei:
        eb.plan_chunks(d, eb.ChunkTarget.memory_budget(1024))
    assert str(2 * eb.padded_chunk_bytes(d, 1)) in str(ei.value)


def test_vcec_to_ecc_prefix_sum_and_empty():
    v = eb.GlobalVcec(np.array([1, 2, 3], np.uint8), np.array([1, -1, 1], np.int64))
    c = eb.vcec_to_ecc(v)
    assert list(c.chi) == [1, 0, 1]
    with pytest.raises(eb.EccError):
        eb.vcec_to_ecc(eb.GlobalVcec(np.array([], np.uint8), np.array([], np.int64)))
