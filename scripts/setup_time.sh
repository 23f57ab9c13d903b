python -c "
from hmgen.build import load_or_generate as g
for n in ['C2','C3','C4']: g(n, verbose=False)
" > /dev/null 2>&1
for c in C2 C3 C4; do PS_VERBOSE=1 python -c "
import time, warnings; warnings.simplefilter('ignore')
from hmgen.build import load_or_generate
from paper_2109_04129_b200 import PsHandle
m = load_or_generate('$c'); h = PsHandle(m['hm']); t = time.time(); h.setup(); print('$c setup', round(time.time()-t, 3), 's')
" 2>&1 | grep -E "setup"; done
