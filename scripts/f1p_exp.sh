#!/bin/bash
# far1p timing experiments (one GPU): class times of C4-1 / C3-1 / C2-1 with compute skipped
# for packs (1), big units (2) or both (3).  outputs: gpurun_out/TAG/
set -u
TAG=${1:-f1px}
O=gpurun_out/$TAG
mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['C2','C3','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
for c in C4 C3 C2; do
for v in "PS_F1P_SKIP=0" "PS_F1P_SKIP=1" "PS_F1P_SKIP=2" "PS_F1P_SKIP=3" ${EXTRA:-}; do
  env $v timeout 300 python scripts/class_times.py --config $c --nrhs 1 --reps 5 > $O/ct.json 2> $O/ct.err
  echo "$c [$v] $(python -c "import json; d=json.load(open('$O/ct.json'))['classes']; print({k: round(v['ms'],3) for k, v in d.items()})")"
done
done
