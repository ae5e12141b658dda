"""CPU tests of the oracle (test infrastructure): the C restatement is pinned
against the reference's known answers and golden fixtures, and -- where the
reference compiled here (oracle/_ref) -- against the reference engine and its
brute-force naive_ecc."""
import hashlib

import numpy as np
import pytest

import oracle

ref_only = pytest.mark.skipif(not oracle.ref_available(), reason="reference not compiled here")


def test_counter_hash_pinned():
    # test_datagen.cpp:48-53
    L = oracle.lib()
    assert L.ecc_oracle_counter_hash(0, 0) == 0xE220A8397B1DCDAF
    assert L.ecc_oracle_counter_hash(0, 1) == 0x6E789E6AA1B965F4
    assert L.ecc_oracle_counter_hash(42, 0) == 0xBDD732262FEB6E95


def test_float_order_key_monotone_and_invertible():
    # test_value_index.cpp:111-125
    L = oracle.lib()
    samples = np.array([-1e30, -2.5, -1e-40, 0.0, 1e-40, 0.5, 2.5, 1e30], np.float32)
    keys = [L.ecc_oracle_float_order_key(float(s)) for s in samples]
    for i, s in enumerate(samples):
        assert np.float32(L.ecc_oracle_float_from_order_key(keys[i])) == s
        for j in range(i + 1, len(samples)):
            assert keys[i] < keys[j]
    assert L.ecc_oracle_float_order_key(-0.0) == L.ecc_oracle_float_order_key(0.0)
    assert not np.signbit(L.ecc_oracle_float_from_order_key(L.ecc_oracle_float_order_key(-0.0)))


def _img(rec):
    return np.array(rec["image"], dtype=rec["dtype"]).reshape(rec["shape"])


def test_hand_fixtures(golden):
    for name, rec in golden["hand"].items():
        v, c = oracle.vcec(_img(rec))
        assert [float(x) for x in v] == rec["values"], name
        assert [int(x) for x in c] == rec["changes"], name


def test_hand_fixture_curves_from_reference_tests():
    # acceptance.cpp:182-198 (curves), test_streaming.cpp:115-120 (u8 ring)
    cases = [
        (np.array([[0, 0, 0], [0, 9, 0], [0, 0, 0]], np.float32), [0, 9], [0, 1]),
        (np.array([[1, 2], [3, 4]], np.float32), [1, 2, 3, 4], [1, 1, 1, 1]),
        (np.array([[0, 1], [1, 0]], np.float32), [0, 1], [1, 1]),
        (np.array([[3.5]], np.float32), [3.5], [1]),
        (np.full((1, 1, 2), 3.5, np.float32), [3.5], [1]),
        (np.ones((2, 2, 2), np.float32), [1.0], [1]),
    ]
    for img, t, chi in cases:
        tt, cc = oracle.curve(img)
        assert list(tt) == t and list(cc) == chi
    v, c = oracle.vcec(np.array([[0, 0, 0], [0, 9, 0], [0, 0, 0]], np.uint8))
    assert list(v) == [0, 9] and list(c) == [0, 1]


def test_random_fixtures(golden):
    for rec in golden["random"]:
        v, c = oracle.vcec(_img(rec))
        assert [float(x) for x in v] == rec["values"]
        assert [int(x) for x in c] == rec["changes"]


def test_appendix_b_small_configs(golden):
    # C1 and one C3 image are cheap enough for the C restatement here.
    t, chi = oracle.curve(oracle.synth("u8", (256, 256)))
    assert oracle.curve_digest(t, chi) == golden["configs"]["C1"]["digest"]
    img = oracle.synth("u16", (512, 512), seed=1, base=0)
    t, chi = oracle.curve(img)
    assert oracle.curve_digest(t, chi) == golden["configs"]["C3_0"]["digest"]
    assert len(t) == golden["configs"]["C3_0"]["points"]


@ref_only
def test_appendix_b_csv_hash_c1():
    t, chi = oracle.curve(oracle.synth("u8", (256, 256)))
    assert hashlib.sha256(oracle.ref_csv(t, chi)).hexdigest() == \
        "83ee98223e5e1e49f5ff79581f2f1907e14ba9ef3f59ab9b093c3c732c10fd41"


@ref_only
def test_restatement_matches_reference_engine():
    # the oracle-equivalence sweep of acceptance.cpp:95-142, against the engine
    rng = np.random.default_rng(7)
    for t in range(200):
        d = (int(rng.integers(1, 9)), int(rng.integers(1, 9))) if t % 2 == 0 else \
            tuple(int(x) for x in rng.integers(1, 7, 3))
        k = t % 3
        if k == 0:
            img = rng.integers(0, 8, d).astype(np.uint8)
        elif k == 1:
            img = rng.random(5).astype(np.float32)[rng.integers(0, 5, d)]
        else:
            img = rng.integers(0, 6, d).astype(np.uint16)
        a = oracle.vcec(img)
        b = oracle.ref_vcec(img, chunks=int(rng.integers(1, 4)), workers=int(rng.integers(1, 3)))
        assert np.array_equal(np.asarray(a[0], np.float64), np.asarray(b[0], np.float64))
        assert np.array_equal(a[1], b[1])


@ref_only
def test_restatement_matches_naive_ecc():
    # test_oracle.cpp:132-145: engine == naive cell counting (finite values)
    rng = np.random.default_rng(11)
    for t in range(60):
        d = (int(rng.integers(1, 7)), int(rng.integers(1, 7))) if t % 2 == 0 else \
            tuple(int(x) for x in rng.integers(1, 5, 3))
        img = rng.random(4).astype(np.float32)[rng.integers(0, 4, d)]
        t1, c1 = oracle.curve(img)
        t2, c2 = oracle.ref_naive(img)
        assert np.array_equal(t1, t2) and np.array_equal(c1, c2)


@ref_only
def test_restatement_matches_reference_on_edge_values():
    # +inf collar tie quirk, -0/+0 folding
    cases = [np.array([[np.inf]], np.float32),
             np.array([[np.inf, 2.0], [3.0, 4.0]], np.float32),
             np.array([[1.0, 2.0], [3.0, np.inf]], np.float32),
             np.array([[-0.0, 0.0], [1.0, -0.0]], np.float32),
             np.array([[[np.inf, np.inf], [np.inf, 1.0]]], np.float32),
             np.array([[[-np.inf, 5.0], [np.inf, -0.0]]], np.float32)]
    for img in cases:
        a = oracle.vcec(img)
        b = oracle.ref_vcec(img)
        assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
        assert np.array_equal(a[1], b[1])
