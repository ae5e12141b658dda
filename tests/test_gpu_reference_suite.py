"""The reference's OWN tests -- proj/tests/test_streaming.cpp, test_kernel.cpp,
test_value_index.cpp, test_curve.cpp and acceptance.cpp -- compiled
unmodified against the drop-in headers in include/ (tests/cpp/Makefile: the
Catch2 stand-in and the reference's test-only oracle come from
tests/cpp/shim), every voxel evaluated on the GPU through the C ABI.

The binaries are built where /root/reference exists (build(), this
container) and travel to the GPU box with the snapshot; without them the
tests skip with that reason."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin")


def _binary(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} is built only where /root/reference exists (make -C tests/cpp)")
    return path


@pytest.mark.parametrize("suite", ["test_streaming", "test_kernel", "test_value_index",
                                   "test_curve"])
def test_reference_unit_suite(suite):
    r = subprocess.run([_binary("ref_" + suite)], capture_output=True, text=True, timeout=900)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    m = re.search(r"(\d+) cases, (\d+) checks, (\d+) failed", r.stdout)
    assert m, tail
    assert r.returncode == 0 and int(m.group(3)) == 0, tail
    assert int(m.group(1)) > 0 and int(m.group(2)) > 0


def test_reference_acceptance_criteria_1_to_9():
    """acceptance.cpp:486-527 prints one PASS/FAIL line per criterion.
    Criteria 1-9 must pass.  Criterion 10 runs the reference's CLI
    (ECC_CLI_PATH), which is out of scope and fails
    for the reference itself in this image (CLI11 is absent), so its line is
    only reported."""
    r = subprocess.run([_binary("ref_acceptance")], capture_output=True, text=True, timeout=1500,
                       cwd="/tmp")
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    got = {}
    for ln in lines:
        m = re.match(r"(PASS|FAIL)\s+criterion (\d+)", ln)
        if m:
            got[int(m.group(2))] = (m.group(1), ln)
    assert sorted(got) == list(range(1, 11)), r.stdout[-3000:] + r.stderr[-2000:]
    bad = [got[c][1] for c in range(1, 10) if got[c][0] != "PASS"]
    assert not bad, "\n".join(bad)
    print("\n".join(lines))
