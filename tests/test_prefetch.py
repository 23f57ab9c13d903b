"""The background input generation of the GPU test session (tests/_prefetch.py): the child
process writes the same cached files load_or_generate() would, and is skipped when cached."""
import os


def test_prefetch_generates_and_caches(tmp_path, monkeypatch):
    from hmgen.build import load_or_generate
    from tests import _prefetch
    monkeypatch.setenv("PS_DATA_DIR", str(tmp_path))
    monkeypatch.setitem(_prefetch._state, "proc", None)
    assert _prefetch.start("T2")
    _prefetch.wait()
    assert _prefetch._cached("T2") and not _prefetch.start("T2")
    t0 = os.path.getmtime(tmp_path / "T2.hm")
    meta = load_or_generate("T2")                      # served from the child's files
    assert os.path.getmtime(tmp_path / "T2.hm") == t0 and meta["N"] == 1152
    monkeypatch.setenv("PS_C5_PREFETCH", "0")
    os.remove(tmp_path / "T2.json")
    assert not _prefetch.start("T2")                   # switched off
