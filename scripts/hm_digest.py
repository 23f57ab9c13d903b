"""Print the stored section checksums of .hm files (header + 8 sections): a cheap
content digest to compare files generated on different hosts."""
import json
import struct
import sys

import numpy as np

out = {}
for path in sys.argv[1:]:
    try:
        with open(path, "rb") as f:
            hdr = f.read(128)
            N, nl, nn, nf, _ = struct.unpack_from("<5q", hdr, 8)
            nna, nfa = struct.unpack_from("<2q", hdr, 112)
            sums = [struct.unpack("<Q", f.read(8))[0]]
            for nbytes in (8 * N, 8 * (nl + 1), 12 * nl, 4 * nl, 24 * nn, 16 * nna, 56 * nf, 16 * nfa):
                f.seek(nbytes + (-nbytes) % 8, 1)
                sums.append(struct.unpack("<Q", f.read(8))[0])
        out[path] = ["%016x" % s for s in sums]
    except Exception as e:  # noqa: BLE001
        out[path] = str(e)
print(json.dumps(out, indent=1))
