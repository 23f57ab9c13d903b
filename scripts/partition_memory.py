"""Per-rank device memory of the row partition (host-only ps_analyze_rank), written to
profiles/r2/partition_memory_<cfg>.json:  python scripts/partition_memory.py C5 8"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from hmgen.build import load_or_generate                       # noqa: E402
from paper_2109_04129_b200.binding import analyze              # noqa: E402

name = sys.argv[1]
Ps = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
path = load_or_generate(name)["hm"]
one = analyze(path)
out = {"config": name, "single": {k: one[k] for k in ("N", "op_bytes", "setup_bytes")}, "partitions": {}}
for P in Ps:
    ranks = [analyze(path, g, P) for g in range(P)]
    out["partitions"][P] = {
        "sep_rows": ranks[0]["sep_rows"], "own_rows": [r["own_rows"] for r in ranks],
        "op_bytes": [r["op_bytes"] for r in ranks], "setup_bytes": [r["setup_bytes"] for r in ranks],
        "max_op_share": max(r["op_bytes"] for r in ranks) / one["op_bytes"],
        "max_setup_share": max(r["setup_bytes"] for r in ranks) / one["setup_bytes"]}
    print(P, json.dumps({k: v for k, v in out["partitions"][P].items() if "share" in k or k == "sep_rows"}), flush=True)
os.makedirs(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2"), exist_ok=True)
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2",
                       f"partition_memory_{name}.json"), "w") as f:
    json.dump(out, f, indent=1)
