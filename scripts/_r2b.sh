set -u
O=gpurun_out/r2b; mkdir -p $O
python -c "from hmgen.build import load_or_generate as g; [g(n) for n in ['C2','C3','C4']]" > $O/gen.log 2>&1
for c in "C4 360" "C2 181" "C3 181"; do set -- $c;
  for ks in 0 1; do PS_KSPLIT=$ks timeout 300 python scripts/class_times.py --config $1 --nrhs $2 --both >> $O/class_times_ks$ks.jsonl 2>>$O/class_times.err; done; done
for c in "C4 1" "C2 1" "C3 1"; do set -- $c; timeout 300 python scripts/class_times.py --config $1 --nrhs $2 --both >> $O/class_times_ks1.jsonl 2>>$O/class_times.err; done
timeout 300 python scripts/trace_prog.py --config C4 --nrhs 1 --out /tmp/trace_C4_1.npz > $O/trace.log 2>&1
python scripts/trace_stats.py /tmp/trace_C4_1.npz --bin-us 100 > $O/trace_C4_1.txt 2>&1
ls -la $O
