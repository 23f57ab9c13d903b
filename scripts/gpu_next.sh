#!/bin/bash
# GPU session for the NEXT-3 / NEXT-4 rows: their parity tests, timing scripts, and an ncu
# capture of the far-field kernel. Usage: scripts/gpu_next.sh TAG  (outputs under gpurun_out/TAG/)
set -u
TAG=${1:-r2next}
O=gpurun_out/$TAG
mkdir -p $O
( time python -c "
from hmgen.build import load_or_generate as g
for n in ['T2','C1','C2','C3','C4']: g(n, verbose=False)
" ) > $O/gen.log 2>&1
( time timeout 1500 python -m pytest tests/test_gpu_series.py tests/test_gpu_rcs.py -m gpu -q --durations=15 ) > $O/pytest_next.log 2>&1; echo "pytest=$?"
tail -n 3 $O/pytest_next.log
timeout 600 python scripts/series_bench.py --config C4 --nrhs 1 360 --terms 6 > $O/series_C4.jsonl 2> $O/series_C4.err; echo "series=$?"
timeout 300 python scripts/series_bench.py --config C3 --nrhs 1 181 --terms 6 > $O/series_C3.jsonl 2> $O/series_C3.err; echo "series3=$?"
timeout 600 python scripts/rcs_bench.py --config C4 --bistatic 181 > $O/rcs_C4.json 2> $O/rcs_C4.err; echo "rcs=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:farfield_kernel" -c 2 \
   -o /tmp/ff_C4 python scripts/rcs_bench.py --config C4 --bistatic 181 --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu_ff=$?"
ncu -i /tmp/ff_C4.ncu-rep --page raw --csv > $O/ncu_ff_C4_raw.csv 2>/dev/null
ncu -i /tmp/ff_C4.ncu-rep --page details --csv > $O/ncu_ff_C4_details.csv 2>/dev/null
ls -la $O
