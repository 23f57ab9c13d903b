"""One ps_setup of a config (ncu launch lists of the setup kernels): python scripts/setup_only.py C3"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.simplefilter("ignore")
from hmgen.build import load_or_generate  # noqa: E402
from paper_2109_04129_b200 import PsHandle  # noqa: E402

m = load_or_generate(sys.argv[1] if len(sys.argv) > 1 else "C3")
h = PsHandle(m["hm"])
h.setup()
print("ok")
