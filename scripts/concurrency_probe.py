"""Probe: the RHS block split into G groups solved concurrently on G streams
(one handle per group, persistent grid = PS_GRID), vs one solve of the block."""
import os
import sys
import threading
import time
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    warnings.simplefilter("ignore")
    import torch
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    meta = load_or_generate(cfg)
    B, _ = read_rhs(meta["rhs"])
    cols = np.array_split(np.arange(B.shape[1]), G)
    hs = [PsHandle(meta["hm"]) for _ in range(G)]
    for h in hs:
        h.setup()
    streams = [torch.cuda.Stream() for _ in range(G)]
    Bd = [torch.from_numpy(np.ascontiguousarray(B[:, c].T)).cuda().T for c in cols]
    Xd = [torch.empty_like(b) for b in Bd]

    def run(i, n):
        for _ in range(n):
            hs[i].solve(Bd[i], Xd[i], stream=streams[i], want_norms=False)

    for i in range(G):
        run(i, 2)
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(i, n)) for i in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{cfg} G={G} grid={os.environ.get('PS_GRID', 'default')}: {dt * 1e3:.3f} ms per full block "
          f"({meta['N'] * B.shape[1] / dt:.3e} N*nrhs/s)")


if __name__ == "__main__":
    main()
