"""tools/par_debug.py against an experiment build (EXP_FLAGS, built by tools/exp_bench.py BUILD_ONLY=1)."""
import os, sys, runpy
sys.path.insert(0, ".")
from paper_2505_02922_b200 import _lib
FL = os.environ.get("EXP_FLAGS", "").split()
tag = "_".join(f.lower() for f in FL) or "none"
_lib.LIB_PATH = os.path.join("paper_2505_02922_b200", "build_exp_" + tag, "libwavekv_exp.so")
runpy.run_path("tools/par_debug.py", run_name="__main__")
