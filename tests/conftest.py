import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_built():
    """Build the product library and the restatement oracle if missing (the
    GPU box has the same toolchain; the reference checker is only rebuilt
    where /root/reference exists)."""
    lib = os.path.join(ROOT, "paper_2511_00855_b200", "libfgb200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2511_00855_b200", "csrc"), "-j8"],
                       check=True, stdout=subprocess.DEVNULL)
    if (os.path.exists(os.path.join(ROOT, "oracle", "fg_oracle.cpp"))
            and not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so"))):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


_ensure_built()


@pytest.fixture(scope="session")
def ref():
    from oracle.refpy import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libfgref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def oracle():
    from oracle.refpy import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def has_gpu():
    from paper_2511_00855_b200 import device_count
    return device_count() > 0


def pytest_collection_modifyitems(config, items):
    from paper_2511_00855_b200 import device_count
    if device_count() > 0:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if item.get_closest_marker("gpu"):
            item.add_marker(skip)
