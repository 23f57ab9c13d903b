"""Oracle golden for BASELINE config 4 (C5: PEC sphere r = 3 m, icosphere sub-7, N = 491520).

Calls only the oracle (oracle/: file reader, sequential scaling Eqs. 14-23, two-term solve
Eqs. 24-36) and the shared input generator (hmgen: the .hm file and the plane-wave RHS).
The oracle's alpha panels (67 GB) are spilled to a memory-mapped file and the .hm file is
memory-mapped (storage only; tests/test_oracle.py pins both as value-identical).

Writes tests/golden/C5_x.npz: the oracle's x for 2 RHS columns (RWG order), ||it_0||,
||it_1||, the column indices, and the .hm file's stored section checksums (the GPU test
regenerates C5 and requires identical checksums before comparing).

  python scripts/c5_golden.py [--spill /path/alpha.bin]
"""
import argparse
import json
import os
import struct
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

COLS = [0, 127]          # theta = 0 and 89.6 degrees of the 256-column monostatic sweep (R19)


def hm_checksums(path):
    with open(path, "rb") as f:
        hdr = f.read(128)
        N, nl, nn, nf, _ = struct.unpack_from("<5q", hdr, 8)
        nna, nfa = struct.unpack_from("<2q", hdr, 112)
        sums = [struct.unpack("<Q", f.read(8))[0]]
        for nbytes in (8 * N, 8 * (nl + 1), 12 * nl, 4 * nl, 24 * nn, 16 * nna, 56 * nf, 16 * nfa):
            f.seek(nbytes + (-nbytes) % 8, 1)
            sums.append(struct.unpack("<Q", f.read(8))[0])
    return ["%016x" % s for s in sums]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spill", default=os.path.join(ROOT, "data", "C5_alpha.bin"))
    args = ap.parse_args()
    from hmgen.build import load_or_generate, read_rhs
    from oracle import compute_scaling, read_hm, solve
    t0 = time.time()
    meta = load_or_generate("C5", verbose=True)
    print("generated", time.time() - t0, flush=True)
    B, ang = read_rhs(meta["rhs"])
    B = np.asfortranarray(B[:, COLS])
    H = read_hm(meta["hm"], mmap=True)
    print("read", time.time() - t0, flush=True)
    S = compute_scaling(H, spill=args.spill)
    print("scaling", time.time() - t0, flush=True)
    res = solve(H, S, B)
    print("solve", time.time() - t0, "ratio", res.ratio, flush=True)
    out = os.path.join(ROOT, "tests", "golden", "C5_x.npz")
    np.savez_compressed(out, x=res.x, cols=np.array(COLS), angles=ang[COLS], it0=res.it0, it1=res.it1,
                        hm_checksums=np.array(hm_checksums(meta["hm"])), N=H.N)
    print(json.dumps({"out": out, "seconds": time.time() - t0, "it0": res.it0.tolist(),
                      "it1": res.it1.tolist()}), flush=True)


if __name__ == "__main__":
    main()
