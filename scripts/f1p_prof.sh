#!/bin/bash
# far1p profiling on one GPU: per-class device times of C4-1 under a few knobs, then an ncu
# --set full capture (with source) of the far1p kernel of one C4-1 solve.  outputs: gpurun_out/TAG/
set -u
TAG=${1:-f1pp}
O=gpurun_out/$TAG
mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['C1','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
timeout 600 python -m pytest tests/test_gpu_variants.py -k "far1p and C1" -x -q > $O/pytest_f1p.log 2>&1; echo "pytest_f1p=$?"; tail -n 1 $O/pytest_f1p.log
for v in "" "PS_F1P_CHUNK=1024"; do
  env $v timeout 300 python scripts/class_times.py --config C4 --nrhs 1 --reps 5 > $O/ct.json 2> $O/ct.err
  echo "[$v] $(python -c "import json; d=json.load(open('$O/ct.json'))['classes']; print({k: round(v['ms'],3) for k, v in d.items()})")"
done
python scripts/ncu_solve.py --config C4 --nrhs 1 > $O/plain.log 2>&1 && \
timeout 900 ncu -f --profile-from-start off --set full --import-source on --clock-control none -k "regex:far1p" \
   -o /tmp/f1p python scripts/ncu_solve.py --config C4 --nrhs 1 > $O/ncu.log 2>&1; echo "ncu=$?"
python scripts/ncu_summary.py /tmp/f1p.ncu-rep --config C4 --nrhs 1 > $O/ncu_far1p_C4_1.json 2>/dev/null
ncu -i /tmp/f1p.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/ncu_source_far1p.csv.gz
ncu -i /tmp/f1p.ncu-rep --page details --csv 2>/dev/null > $O/ncu_details_far1p.csv
