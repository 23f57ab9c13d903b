#!/bin/bash
# C5 at 1 RHS with the one-pass far apply forced on (the default leaves it off for C5), from the
# box's C5 cache if a previous call left it; then the far1p rows-per-warp experiment on C4.
set -u
CACHE=/root/.cache/ps_c5
mkdir -p data gpurun_out
if [ -f $CACHE/C5.json ]; then cp $CACHE/C5.* data/; echo "restored C5 from cache"; fi
python -c "from hmgen.build import load_or_generate as g; g('C5')" > gpurun_out/c5f_gen.log 2>&1
PS_FAR1P=1 timeout 900 python bench.py --config C5 --nrhs 1 --no-cpu-baseline --steps 5 > gpurun_out/bench_C5_1_far1p.json 2> gpurun_out/bench_C5_1_far1p.err; echo "bench=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_C5_1_far1p.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernel_parts_ms'))"
bash scripts/f1p_minrows.sh f1pr
