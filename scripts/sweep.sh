#!/bin/bash
# Run bench.py (C2 by default) under several tuning environments; one summary line each.
# usage: scripts/sweep.sh CONFIG NRHS "ENV1" "ENV2" ...
cfg=$1; nrhs=$2; shift 2
for e in "$@"; do
  env $e timeout 150 python bench.py --config $cfg --nrhs $nrhs --steps 20 --warmup 3 --no-cpu-baseline > /tmp/sw.log 2>&1
  python - "$e" <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/sw.log').read().strip().splitlines()[-1])
    pc = {k: round(v['ms_per_step'], 3) for k, v in d['roofline']['per_class'].items() if v['ms_per_step'] > 0}
    print(f"{sys.argv[1]:40s} ms={d['ms_per_step']:.3f} frac={d['roofline']['frac']:.3f} {pc}")
except Exception as ex:
    print(sys.argv[1], "FAILED", ex, open('/tmp/sw.log').read()[-500:])
PY
done
