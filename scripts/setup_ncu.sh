#!/bin/bash
# ncu launch list of one ps_setup (C3): per-kernel device time of the setup levels
O=gpurun_out/${1:-stn}; mkdir -p $O
python -c "
from hmgen.build import load_or_generate as g
g('C3', verbose=False)
" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/setup_launches_C3.csv python scripts/setup_only.py C3 > $O/setup_ncu.log 2>&1; echo "ncu=$?"
python scripts/launch_summary.py $O/setup_launches_C3.csv > $O/setup_launches_C3_summary.json 2>/dev/null; cat $O/setup_launches_C3_summary.json
