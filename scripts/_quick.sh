set -u
O=gpurun_out/${1:-q}; mkdir -p $O
python -c "from hmgen.build import load_or_generate as g; [g(n) for n in ['C2','C3','C4']]" > $O/gen.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest=$?"; tail -2 $O/pytest.log
for c in "C4 1" "C2 1" "C3 1"; do set -- $c; timeout 300 python scripts/class_times.py --config $1 --nrhs $2 --both >> $O/class_times.jsonl 2>>$O/class_times.err; done
for c in "C4 360" "C2 181"; do set -- $c; timeout 300 python scripts/class_times.py --config $1 --nrhs $2 >> $O/class_times.jsonl 2>>$O/class_times.err; done
ls $O
