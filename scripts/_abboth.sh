# A/B of env knobs on narrow and wide programs: bash scripts/_abboth.sh TAG "ENV1" "ENV2" ...
set -u
O=gpurun_out/$1; shift; mkdir -p $O
python -c "from hmgen.build import load_or_generate as g; [g(n) for n in ['C2','C3','C4']]" > $O/gen.log 2>&1
for e in "$@"; do
  for c in "C4 1" "C2 1" "C3 1" "C4 360" "C2 181" "C3 181"; do set -- $c; env $e timeout 300 python scripts/class_times.py --config $1 --nrhs $2 | sed "s/^/$e /" >> $O/ab.txt 2>>$O/ab.err; done
done
