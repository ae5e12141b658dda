"""The C++ side of the drop-in (include/ecc/*.hpp over the C ABI) and the
bit-sliced helpers, exercised through the compiled C++ test programs in
tests/cpp (built by __graft_entry__.build() / `make -C tests/cpp`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin")


def _bin(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return path


def _run(args, timeout=600):
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    return p.stdout


def test_bit_sliced_sum_and_code_transpose():
    out = _run([_bin("test_bits")])
    for name in ("sum_code", "transpose_codes", "sum_blocks9", "hist16 encoding", "cols layout"):
        assert f"{name} ok" in out, out


def test_cpp_api_host_cases():
    out = _run([_bin("test_api"), "cpu"])
    assert "0 failures" in out


def test_cpp_headers_compile_standalone(tmp_path):
    # every drop-in header is self-contained (includes what it uses)
    for h in sorted(os.listdir(os.path.join(ROOT, "include", "ecc"))):
        src = tmp_path / f"t_{h}.cpp"
        src.write_text(f'#include "ecc/{h}"\nint main() {{ return 0; }}\n')
        subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        str(src)], check=True)


@pytest.mark.gpu
def test_cpp_api_gpu_cases():
    out = _run([_bin("test_api"), "gpu"])
    assert "0 failures" in out, out


def test_cpp_curve_csv_matches_reference_writer(tmp_path):
    """include/ecc/curve.hpp write_curve vs the reference's own write_curve
    (compiled in oracle/_ref): byte-identical CSV for float thresholds,
    including the shortest round-trip formatting of awkward values."""
    import numpy as np
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference not compiled here")
    rng = np.random.default_rng(3)
    t = np.unique(np.concatenate([
        rng.random(500).astype(np.float32),
        (rng.integers(0, 65536, 300) * 2.0 ** -16).astype(np.float32),
        np.array([0.0, 1e-38, 3.4e38, 1e10, 123456.7, 2.0 ** -149, 0.1, 1.0 / 3], np.float32),
        -rng.random(50).astype(np.float32) * 1e6]))
    chi = rng.integers(-10 ** 12, 10 ** 12, t.size).astype(np.int64)
    f = tmp_path / "c.bin"
    with open(f, "wb") as fh:
        fh.write(np.uint64(t.size).tobytes())
        fh.write(t.astype(np.float32).tobytes())
        fh.write(chi.tobytes())
    mine = subprocess.run([_bin("test_api"), "csv", str(f)], capture_output=True, check=True).stdout
    assert mine == oracle.ref_csv(t, chi)


def test_reference_tests_compile_against_the_drop_in():
    """The reference's own test programs (proj/tests/test_streaming.cpp,
    test_kernel.cpp, test_value_index.cpp, test_curve.cpp, acceptance.cpp)
    compile UNMODIFIED with include/ first on the include path -- the
    drop-in's headers provide every symbol they use.  (They run on the GPU
    in tests/test_gpu_reference_suite.py.)"""
    if not os.path.isdir("/root/reference/proj/tests"):
        pytest.skip("the reference sources exist only in the build container")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    for t in ["test_streaming", "test_kernel", "test_value_index", "test_curve", "acceptance"]:
        assert os.path.exists(os.path.join(BIN, "ref_" + t)), t


def test_f2s_matches_to_chars():
    """csrc/f2s.cuh (the GPU's float formatter) == std::to_chars(float) on
    special values, every exponent's extremes, 4 M random bit patterns and
    decimal-looking values (`tests/cpp/bin/test_f2s all` checks all 2^32
    floats: profiles/r02v_f2s_all_floats.log)."""
    out = _run([_bin("test_f2s")])
    assert "f2s ok" in out
