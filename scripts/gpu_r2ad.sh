#!/bin/bash
set -u
O=gpurun_out/r2ad; mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['T2','C1','C2','C3','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_variants.py -m gpu -x -q -k "INV_CLUSTER or default" ) > $O/pytest_var.log 2>&1; echo "var=$?"; tail -n 2 $O/pytest_var.log
( time timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dinv or c3 or singular or synthetic or c1" ) > $O/pytest_par.log 2>&1; echo "par=$?"; tail -n 2 $O/pytest_par.log
for c in C3 C4; do
  PS_VERBOSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-nrhs1 --steps 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?"
done
bash scripts/setup_ncu.sh r2ad > /dev/null 2>&1; echo "setup_ncu=$?"
ls -la $O
