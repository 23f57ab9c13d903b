#!/bin/bash
# Driver-like GPU session on a clean tree: pytest -m gpu with NO pre-generated data (the test
# session generates C1-C5 itself; C5 in the background, tests/_prefetch.py), smoke, bench lines,
# ncu launch list + full captures of C4-360 / C4-1.   Usage: scripts/gpu_r2af.sh TAG
set -u
TAG=${1:-r2af}
O=gpurun_out/$TAG
mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $O/host.txt
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 ) > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -n 5 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke=$?"; tail -n 1 $O/smoke.log
python scripts/hm_digest.py data/T2.hm data/C1.hm data/C2.hm data/C3.hm data/C4.hm > $O/hm_digest.json 2>&1
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench=$?"
for c in C2 C3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?"
done
timeout 300 python bench.py --config C1 --nrhs 1 --no-cpu-baseline > $O/bench_C1_1.json 2> $O/bench_C1_1.err; echo "bench_C1=$?"
if [ -f data/C5.hm ]; then
  PS_VERBOSE=1 timeout 900 python bench.py --config C5 --steps 3 --no-cpu-baseline --no-next > $O/bench_C5.json 2> $O/bench_C5.err; echo "bench_C5=$?"
fi
for v in ${AB_VARIANTS:-base 1824_2 2240_2 768_4}; do   # far1p tiling A/B (scripts/f1p_variants.sh), C4 at 1 RHS
  L=ab_libs/libps_$v.so; [ $v = base ] && L=paper_2109_04129_b200/libps.so
  [ -f $L ] && PS_LIB=$L timeout 300 python bench.py --config C4 --nrhs 1 --no-cpu-baseline --no-next > $O/ab_f1p_$v.json 2> $O/ab_f1p_$v.err
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/ncu_launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu_list=$?"
python scripts/launch_summary.py $O/ncu_launches_C4.csv > $O/ncu_launches_C4_summary.json 2>/dev/null
for NR in 360 1; do
  python scripts/ncu_solve.py --config C4 --nrhs $NR > $O/plain_solve_$NR.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:flow_kernel|far1p|far_reduce" \
     -o /tmp/full_C4_$NR python scripts/ncu_solve.py --config C4 --nrhs $NR > /dev/null 2>&1; echo "ncu_full_$NR=$?"
  python scripts/ncu_summary.py /tmp/full_C4_$NR.ncu-rep --config C4 --nrhs $NR > $O/ncu_full_C4_${NR}.json 2>/dev/null
  ncu -i /tmp/full_C4_$NR.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/ncu_source_C4_${NR}.csv.gz
done
[ "${SKIP_REF:-0}" = 1 ] || { timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_C4.json 2> $O/bench_ref_C4.err; echo "ref=$?"; }
ls -la $O
