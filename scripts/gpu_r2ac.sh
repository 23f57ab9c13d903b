#!/bin/bash
# inverse-kernel change: parity + setup times; RCS call overhead diagnosis
set -u
O=gpurun_out/r2ac; mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
for n in ['T2','C1','C2','C3','C4']: g(n, verbose=False)
" > $O/gen.log 2>&1
timeout 300 python scripts/rcs_diag.py > $O/rcs_diag.log 2>&1; echo "diag=$?"
timeout 600 python scripts/rcs_bench.py --config C4 --bistatic 181 > $O/rcs_C4.json 2> $O/rcs_C4.err; echo "rcs=$?"
for c in C3 C4 C2; do
  PS_VERBOSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-nrhs1 --steps 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?"
done
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_series.py -m gpu -x -q --durations=10 ) > $O/pytest.log 2>&1; echo "pytest=$?"
tail -n 3 $O/pytest.log
ls -la $O
