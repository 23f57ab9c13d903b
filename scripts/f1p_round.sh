#!/bin/bash
# far1p check on one GPU: oracle parity of the narrow paths, then per-class device times of
# C4 / C3 / C2 at 1 RHS with and without the one-pass far apply.  outputs: gpurun_out/TAG/
set -u
TAG=${1:-f1p}
O=gpurun_out/$TAG
mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['T2','C1','C2','C3','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py -k far1p -x -q > $O/pytest_f1p.log 2>&1; echo "pytest_f1p=$?"; tail -n 2 $O/pytest_f1p.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1; echo "pytest_parity=$?"; tail -n 2 $O/pytest_parity.log
for c in C4 C3 C2; do
  for f in 1 0; do
    PS_FAR1P=$f timeout 300 python scripts/class_times.py --config $c --nrhs 1 --reps 5 > $O/ct_${c}_f$f.json 2> $O/ct_${c}_f$f.err
    echo "$c far1p=$f: $(cat $O/ct_${c}_f$f.json | head -c 600)"
  done
done
