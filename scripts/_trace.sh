set -u
O=gpurun_out/$1; shift; mkdir -p $O
python -c "from hmgen.build import load_or_generate as g; [g(n) for n in ['C2','C3','C4']]" > $O/gen.log 2>&1
for e in "$@"; do
for c in "C4 1" "C2 1"; do set -- $c;
env $e timeout 300 python scripts/trace_prog.py --config $1 --nrhs $2 --out /tmp/trace_$1_$2.npz >> $O/trace.log 2>&1
python scripts/trace_stats.py /tmp/trace_$1_$2.npz --bin-us 100 > $O/trace_$1_$2_$e.txt 2>&1
done; done
