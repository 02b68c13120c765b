"""pytest against an experiment build (EXP_FLAGS, built by tools/exp_bench.py BUILD_ONLY=1): regression tests must fail on it."""
import os, sys
sys.path.insert(0, ".")
from paper_2505_02922_b200 import _lib
FL = os.environ.get("EXP_FLAGS", "").split()
_lib.LIB_PATH = os.path.join("paper_2505_02922_b200", "build_exp_" + ("_".join(f.lower() for f in FL) or "none"),
                             "libwavekv_exp.so")
import pytest
sys.exit(pytest.main(sys.argv[1:]))
