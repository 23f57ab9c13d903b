"""GPU parity of the alternative execution paths selected by environment knobs
(each read once per process, so every variant runs in a subprocess):

  PS_CHAINS=0      sweeps as one dependent hop per elimination-tree level
                   (no chain matrices T_c, DESIGN.md §6 / R23)
  PS_MMA=dmma      every wide table on the FP64 tensor-core consumer
  PS_MMA=dfma      every wide table on the DFMA consumer (far field included)
  PS_SOLVE=stages  one launch per operator instead of the single-launch program
  PS_SLOT_BUDGET_MB=-1 partial-slot budget exceeded: the program falls back to task-keyed
                   ticket order (the path C5 takes)
  PS_KSPLIT=0      wide DFMA tiles in the one-column-per-lane layout (no k-split)
  PS_DEFER_FIN=0   narrow split-K combine in line (no finisher warp)
  PS_SLOT_REUSE=0  one partial slot per split chunk (no recycling)

Each must match the oracle to the north-star bar (relative L2 <= 1e-11 per RHS).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, warnings
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2109_04129_b200 import PsHandle
from hmgen.synth import random_rhs
warnings.simplefilter("ignore")
h = PsHandle({path!r}); h.setup()
B = random_rhs(h.N, {nrhs}, 4)
Bd = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(B).T)).cuda().T
Xd = torch.empty_like(Bd)
st, rep = h.solve(Bd, Xd)
np.save({out!r}, Xd.T.cpu().numpy().T)
np.save({out!r} + ".it.npy", np.stack([rep["it0"], rep["it1"]]))
"""


def _run(path, nrhs, env, out):
    e = dict(os.environ)
    e.update(env)
    code = _SCRIPT.format(root=ROOT, path=path, nrhs=nrhs, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out), np.load(out + ".it.npy")


@pytest.mark.parametrize("env", [{"PS_CHAINS": "0"}, {"PS_MMA": "dmma"},
                                 {"PS_MMA": "dfma"}, {"PS_SOLVE": "stages"},
                                 {"PS_SLOT_BUDGET_MB": "-1"}, {"PS_KSPLIT": "0"}, {"PS_DEFER_FIN": "0"},
                                 {"PS_SLOT_REUSE": "0"}, {"PS_INV_CLUSTER_MIN": "1"}, {}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("nrhs", [1, 70])
def test_variant_matches_oracle(cfgdata, tmp_path, env, nrhs):
    from hmgen.synth import random_rhs
    from oracle import compute_scaling, read_hm, solve
    from tests.conftest import rel_l2_cols
    path = cfgdata("C1")["hm"]
    x, it = _run(path, nrhs, env, str(tmp_path / "x.npy"))
    H = read_hm(path)
    ref = solve(H, compute_scaling(H), random_rhs(H.N, nrhs, 4))
    assert rel_l2_cols(x, ref.x).max() <= 1e-11
    assert np.allclose(it[0], ref.it0, rtol=1e-11)
    assert np.allclose(it[1], ref.it1, rtol=1e-10)


# The one-pass far apply of narrow solves (far1p): taken by default for nrhs <= 8
# where the far field is large (C4, C5); PS_FAR1P=1 forces it, 0 keeps the two-stage far field
# inside one program launch; PS_F1P_CHUNK cuts
# the items smaller than the 2048-element default, so most blocks of the small configs take
# the big-block path (alpha / gamma / beta chunks, dense chunks with a last-arriver sum) with
# many chunks per block and many waits.
@pytest.mark.parametrize("env", [{"PS_FAR1P": "1"}, {"PS_FAR1P": "0"}, {"PS_FAR1P": "1", "PS_F1P_CHUNK": "64"},
                                 {"PS_FAR1P": "1", "PS_F1P_CHUNK": "300"}, {"PS_FAR1P": "1", "PS_F1P_CHUNK": "128"},
                                 {}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("nrhs", [1, 3, 8])
@pytest.mark.parametrize("cfg", ["C1", "T2"])
def test_far1p_matches_oracle(cfgdata, tmp_path, env, nrhs, cfg):
    from hmgen.synth import random_rhs
    from oracle import compute_scaling, read_hm, solve
    from tests.conftest import rel_l2_cols
    path = cfgdata(cfg)["hm"]
    x, it = _run(path, nrhs, env, str(tmp_path / "x.npy"))
    H = read_hm(path)
    ref = solve(H, compute_scaling(H), random_rhs(H.N, nrhs, 4))
    assert rel_l2_cols(x, ref.x).max() <= 1e-11
    assert np.allclose(it[0], ref.it0, rtol=1e-11)
    assert np.allclose(it[1], ref.it1, rtol=1e-10)


# ps_solve on HOST buffers with many columns runs as two pipelined column halves on copy streams
# (default from 256 columns). PS_HOST_PIPE_MIN=2 takes that path on C1: an odd
# block (second half padded by one column), an even one, and pageable as well as pinned buffers.
_HOST_SCRIPT = r"""
import sys, warnings
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2109_04129_b200 import PsHandle
from hmgen.synth import random_rhs
warnings.simplefilter("ignore")
h = PsHandle({path!r}); h.setup()
B = np.asfortranarray(random_rhs(h.N, {nrhs}, 4))
X = np.zeros_like(B)
st, rep = h.solve(B, X)
Bp = torch.from_numpy(np.ascontiguousarray(B.T)).pin_memory().T
Xp = torch.empty_like(Bp.T).pin_memory().T
for _ in range(2):
    h.solve(Bp, Xp)
assert np.array_equal(Xp.numpy(), X), "pinned and pageable host buffers differ"
np.save({out!r}, X)
np.save({out!r} + ".it.npy", np.stack([rep["it0"], rep["it1"]]))
"""


@pytest.mark.parametrize("nrhs", [2, 7, 70])
def test_host_pipelined_halves_match_oracle(cfgdata, tmp_path, nrhs):
    from hmgen.synth import random_rhs
    from oracle import compute_scaling, read_hm, solve
    from tests.conftest import rel_l2_cols
    path = cfgdata("C1")["hm"]
    out = str(tmp_path / "xh.npy")
    e = dict(os.environ, PS_HOST_PIPE_MIN="2")
    r = subprocess.run([sys.executable, "-c", _HOST_SCRIPT.format(root=ROOT, path=path, nrhs=nrhs, out=out)],
                       env=e, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    x, it = np.load(out), np.load(out + ".it.npy")
    H = read_hm(path)
    ref = solve(H, compute_scaling(H), random_rhs(H.N, nrhs, 4))
    assert x.shape == ref.x.shape and rel_l2_cols(x, ref.x).max() <= 1e-11
    assert np.allclose(it[0], ref.it0, rtol=1e-11)
    assert np.allclose(it[1], ref.it1, rtol=1e-10)
