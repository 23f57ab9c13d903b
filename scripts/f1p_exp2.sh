#!/bin/bash
set -u
O=gpurun_out/${1:-f1pn}; mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['C3','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
for c in C4 C3; do
for v in "PS_F1P_GRID=0" "PS_F1P_GRID=148" "PS_F1P_GRID=74" "PS_F1P_SKIP=3 PS_F1P_GRID=148" "PS_F1P_SKIP=3 PS_F1P_GRID=296" "PS_F1P_PACKS_PER_UNIT=2"; do
  env $v timeout 300 python scripts/class_times.py --config $c --nrhs 1 --reps 5 > $O/ct.json 2> $O/ct.err
  echo "$c [$v] $(python -c "import json; d=json.load(open('$O/ct.json'))['classes']; print({k: round(v['ms'],3) for k, v in d.items()})")"
done
done
