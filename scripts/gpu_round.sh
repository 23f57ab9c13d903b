#!/bin/bash
# One GPU session: tests, smoke, bench lines, ncu launch list + full capture summaries.
# Outputs under gpurun_out/ (kept small: ncu reports are exported to CSV on the box).
set -u
TAG=${1:-r1}
python -c "from hmgen.build import load_or_generate as g; g('C2'); g('C3'); g('C4')" > gpurun_out/gen_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
tail -n 2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?"; tail -n 1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_C2_$TAG.json 2> gpurun_out/bench_C2_$TAG.err; echo "bench=$?"
timeout 300 python bench.py --config C3 --nrhs 1 --no-cpu-baseline > gpurun_out/bench_C3_1_$TAG.json 2>/dev/null; echo "bench3=$?"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3_181_$TAG.json 2>/dev/null; echo "bench3b=$?"
timeout 300 python bench.py --config C2 --nrhs 1 --no-cpu-baseline > gpurun_out/bench_C2_1_$TAG.json 2>/dev/null; echo "bench2a=$?"
timeout 300 python bench.py --config C1 --nrhs 1 --no-cpu-baseline > gpurun_out/bench_C1_1_$TAG.json 2>/dev/null; echo "bench1=$?"
timeout 300 python bench.py --config C4 --nrhs 1 --no-cpu-baseline > gpurun_out/bench_C4_1_$TAG.json 2>/dev/null; echo "bench4a=$?"
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_C4_360_$TAG.json 2>/dev/null; echo "bench4b=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C2_$TAG.json 2>/dev/null; echo "ref=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_C2_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu_list=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:flow_kernel -o /tmp/full_$TAG python scripts/ncu_solve.py --config C2 > /dev/null 2>&1; echo "ncu_full=$?"
ncu -i /tmp/full_$TAG.ncu-rep --page raw --csv > /tmp/full_raw.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/full_$TAG.ncu-rep > gpurun_out/ncu_full_C2_181_$TAG.json 2>/dev/null
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:flow_kernel -o /tmp/full3_$TAG python scripts/ncu_solve.py --config C3 --nrhs 1 > /dev/null 2>&1; echo "ncu_full3=$?"
python scripts/ncu_summary.py /tmp/full3_$TAG.ncu-rep > gpurun_out/ncu_full_C3_1_$TAG.json 2>/dev/null
python scripts/launch_summary.py gpurun_out/ncu_launches_C2_$TAG.csv > gpurun_out/ncu_launches_C2_${TAG}_summary.json 2>/dev/null
ls -la gpurun_out | tail -20
