import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """The oracle (test infrastructure) and the product library must exist before any test."""
    # make rebuilds the C restatement when tlb_oracle.c is newer than the library (a one-second compile)
    subprocess.check_call(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"])
    # the product library: mtime-incremental (a no-op when libtlb.so is newer than every source), so tests can never
    # pass against a binary that is older than csrc/. Without nvcc (never the case in this image) a prebuilt library
    # is used as is.
    import shutil
    lib = ROOT / "paper_2603_02298_b200" / "libtlb.so"
    if shutil.which("nvcc") or Path("/usr/local/cuda/bin/nvcc").exists() or not lib.exists():
        from paper_2603_02298_b200 import build as _b
        _b.build()
    yield


@pytest.fixture
def tlb_config():
    """Set library knobs for one test (tlb_config_set: the TLB_* environment is read only once per process); every knob
    the test touched goes back to its default afterwards."""
    from paper_2603_02298_b200 import host
    touched = []

    def set_knob(name, value):
        touched.append(name)
        host.config(name, value)

    yield set_knob
    for name in touched:
        host.config(name, None)


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
