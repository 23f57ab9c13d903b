import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libps CUDA kernels)")
    config.addinivalue_line("markers", "slow: minutes of CPU (large configs)")


@pytest.hookimpl(trylast=True)
def pytest_collection_modifyitems(config, items):
    """GPU session: test_gpu_c5.py last, its 7-minute input generation started now in a child
    process (tests/_prefetch.py) so that it overlaps the other configs' GPU tests."""
    c5 = [it for it in items if os.path.basename(str(it.fspath)) == "test_gpu_c5.py" and it.get_closest_marker("gpu")]
    if not c5:
        return
    rest = [it for it in items if it not in c5]
    items[:] = rest + c5
    if rest and os.path.exists("/dev/nvidia0"):
        from tests import _prefetch
        _prefetch.start("C5")


def pytest_sessionfinish(session, exitstatus):
    from tests import _prefetch
    _prefetch.stop()


@pytest.fixture(scope="session")
def cfgdata():
    """Generated physical configs (cached under data/ or $PS_DATA_DIR)."""
    from hmgen.build import load_or_generate
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_or_generate(name)
        return cache[name]
    return get


@pytest.fixture(scope="session")
def synthfile(tmp_path_factory):
    """Write a seeded synthetic H-matrix to a .hm file; returns (path, HData)."""
    from hmgen.build import write_hm
    from hmgen.synth import synthetic
    cache = {}
    d = tmp_path_factory.mktemp("synth")

    def get(**kw):
        key = tuple(sorted(kw.items()))
        if key not in cache:
            hd = synthetic(**kw)
            p = str(d / f"s{len(cache)}.hm")
            write_hm(p, hd)
            cache[key] = (p, hd)
        return cache[key]
    return get


def rel_l2_cols(a, b):
    a = np.asarray(a).reshape(a.shape[0], -1)
    b = np.asarray(b).reshape(b.shape[0], -1)
    return np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)
