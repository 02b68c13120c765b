"""A/B experiments: build libwavekv with extra -D flags into its own directory
(EXP_FLAGS="A B" -> -DA -DB, build_exp_<tag>/; the product library is
untouched) and run bench.py's main() against it with the remaining argv.
Build here (BUILD_ONLY=1) so the library travels with the gpurun snapshot."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_02922_b200 import _build
FL = os.environ.get("EXP_FLAGS", "").split()
tag = "_".join(f.lower() for f in FL) or "none"
HERE = os.path.dirname(os.path.abspath(_build.__file__))
_build.OBJ = os.path.join(HERE, "build_exp_" + tag)
_build.LIB = os.path.join(_build.OBJ, "libwavekv_exp.so")
os.environ["WK_EXTRA_NVCC_FLAGS"] = " ".join("-D" + f for f in FL)
os.makedirs(_build.OBJ, exist_ok=True)
if os.environ.get("BUILD_ONLY") == "1":
    _build.build(force=True)
    print(_build.LIB)
    sys.exit(0)
assert os.path.exists(_build.LIB), "build it here first (BUILD_ONLY=1)"
from paper_2505_02922_b200 import _lib
_lib.LIB_PATH = _build.LIB
import bench
sys.argv = ["bench.py"] + sys.argv[1:]
bench.main()
