"""Drop-in proof: the reference's OWN acceptance suite (tests/acceptance.cpp,
unmodified, 9 criteria) linked against the reference library with
integration/fusegraph_b200_shim.cpp in front, so index build, search,
batch_query, NN-Descent, the refinery and brute-force truth run on the B200
through libfgb200.so.  Built by `make -C integration` where /root/reference
exists; the binary travels with the snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_on_b200():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 9
