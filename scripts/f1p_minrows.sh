#!/bin/bash
# far1p: rows per consumer warp on big chunks (PS_F1P_MINROWS), class times of C4-1
O=gpurun_out/${1:-f1pr}; mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
g('C4', verbose=False)
" > /dev/null 2>&1
for v in 0 8 16 32; do
  PS_F1P_MINROWS=$v timeout 300 python scripts/class_times.py --config C4 --nrhs 1 --reps 5 > $O/ct.json 2> $O/ct.err
  echo "minrows=$v $(python -c "import json; d=json.load(open('$O/ct.json'))['classes']; print({k: round(v['ms'],3) for k, v in d.items()})")"
done
