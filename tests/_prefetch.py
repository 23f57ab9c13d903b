"""Background generation of the C5 input for the GPU test session.

C5's seeded generator runs ~7 minutes on the GPU box's host cores; the GPU tests of the
other configs spend much of their time waiting on the GPU. tests/conftest.py therefore
orders test_gpu_c5.py last and starts the generator (a separate process calling
hmgen.build.load_or_generate, the same call the test makes) when the session begins; the C5
tests wait for that process and then load the cached files. No arithmetic here: the file
is the one load_or_generate would have written in-process (its section checksums are
compared with the golden's by the test).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_state = {"proc": None, "log": None}


def _cached(name: str) -> bool:
    from hmgen.build import _src_digest, cache_dir
    js = os.path.join(cache_dir(), f"{name}.json")
    if not (os.path.exists(js) and os.path.exists(os.path.join(cache_dir(), f"{name}.hm"))):
        return False
    try:
        with open(js) as f:
            return json.load(f).get("digest") == _src_digest()
    except Exception:
        return False


def start(name: str = "C5") -> bool:
    """Start generating `name` in a child process unless it is cached or already running."""
    if _state["proc"] is not None or os.environ.get("PS_C5_PREFETCH", "1") == "0" or _cached(name):
        return False
    from hmgen.build import cache_dir
    log = open(os.path.join(cache_dir(), f"{name}.prefetch.log"), "w")
    env = dict(os.environ, OMP_WAIT_POLICY="passive")      # share the cores with the running tests
    _state["proc"] = subprocess.Popen(
        [sys.executable, "-c", f"from hmgen.build import load_or_generate; load_or_generate({name!r})"],
        cwd=ROOT, env=env, stdout=log, stderr=subprocess.STDOUT)
    _state["log"] = log
    return True


def wait() -> None:
    """Block until the child (if any) has exited; the caller then calls load_or_generate,
    which regenerates in-process should the child have failed."""
    p = _state["proc"]
    if p is not None:
        p.wait()
        _state["proc"] = None
        if _state["log"]:
            _state["log"].close()


def stop() -> None:
    p = _state["proc"]
    if p is not None and p.poll() is None:
        p.kill()
        p.wait()
    _state["proc"] = None
