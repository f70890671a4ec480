import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (run with `-m gpu` on a B200)")


@pytest.fixture(scope="session", autouse=True)
def _native_libs():
    """The native libraries are built in-tree once; tests never JIT-compile."""
    from paper_1805_08995_b200 import build
    import oracle_lib

    if not (build.PKG / "libchgpu.so").exists() or not (build.PKG / "libchsynth.so").exists():
        build.build_all()
    if not oracle_lib.RESTATEMENT.exists() or (
            Path("/root/reference/proj/src/matcher.cpp").exists() and not oracle_lib.REFERENCE.exists()):
        oracle_lib.build_oracle()


@pytest.fixture(scope="session")
def restatement():
    import oracle_lib
    return oracle_lib.restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle_lib
    ref = oracle_lib.reference()
    if ref is None:
        pytest.skip("oracle/_ref not built here (needs /root/reference)")
    return ref


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    g = ROOT / "tests" / "golden"
    return {name: np.load(g / f"{name}.npz") for name in ("family", "small_dataset", "plans", "plans_guided", "cache")}


@pytest.fixture(scope="session")
def matcher():
    from paper_1805_08995_b200 import Matcher
    m = Matcher(int(os.environ.get("LOCAL_RANK", "0")))
    yield m
    m.close()
