#!/bin/bash
# BASELINE config 4 (sphere r = 3 m, N = 491520) on one GPU: generate, residual pins, bench lines
# (1 and 256 RHS, BASELINE configs[4]). The generated files are cached under /root/.cache/ps_c5
# (a reused box keeps them; a fresh one regenerates, ~8 min on 16 cores).
set -u
TAG=${1:-r1}
CACHE=/root/.cache/ps_c5
nproc > gpurun_out/c5_host_$TAG.txt; free -g >> gpurun_out/c5_host_$TAG.txt
mkdir -p data
if [ -f $CACHE/C5.json ]; then cp $CACHE/C5.* data/; echo "restored C5 from cache"; fi
( time python -c "from hmgen.build import load_or_generate as g; m = g('C5', verbose=True); print({k: m[k] for k in m if k != 'desc'})" ) > gpurun_out/c5_gen_$TAG.log 2>&1
echo "gen=$?"
if [ ! -f $CACHE/C5.json ]; then mkdir -p $CACHE && cp data/C5.* $CACHE/; fi
python - <<'PY' >> gpurun_out/c5_gen_$TAG.log 2>&1
import ctypes, json
from paper_2109_04129_b200.binding import INFO_KEYS, load_library
L = load_library()
out = (ctypes.c_double * len(INFO_KEYS))()
n = L.ps_analyze(b"data/C5.hm", out, len(INFO_KEYS))
print(json.dumps({k: out[i] for i, k in enumerate(INFO_KEYS[:n])}))
PY
PS_VERBOSE=1 PS_C5=1 timeout 1800 python -m pytest tests/test_gpu_c5.py -x -q -s -k residual > gpurun_out/c5_pytest_$TAG.log 2>&1; echo "pytest=$?"
PS_VERBOSE=1 timeout 900 python bench.py --config C5 --nrhs 1 --no-cpu-baseline --steps 5 > gpurun_out/bench_C5_1_$TAG.json 2> gpurun_out/bench_C5_1_$TAG.err; echo "bench1=$?"
PS_VERBOSE=1 timeout 900 python bench.py --config C5 --nrhs 256 --no-cpu-baseline --steps 3 > gpurun_out/bench_C5_256_$TAG.json 2> gpurun_out/bench_C5_256_$TAG.err; echo "bench256=$?"
tail -n 3 gpurun_out/c5_gen_$TAG.log gpurun_out/c5_pytest_$TAG.log
