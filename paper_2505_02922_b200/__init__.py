"""B200-native wave-index decode attention (RetroInfer, arXiv 2505.02922).

Drop-in for the decode-attention path of the reference package ``tierkv``:
the same public names (``HeadEngine``, ``EngineConfig``, ``IndexConfig``,
``spherical_kmeans``, ``rank_clusters``, ``plan_zones``, ...) backed by
hand-written sm_100a kernels in ``libwavekv.so`` (include/wavekv.h).  The
batched multi-request / GQA engine is ``WaveLayer``.
"""

from .config import EngineConfig, IndexConfig, round_half_up
from .errors import ConfigError, IntegrityError, TierKVError, TraceFormatError
from .clustering import spherical_kmeans
from .engine import HeadEngine, StepMetrics, relative_l2
from .runner import TraceEngine, oracle_trace, run_trace
from .tracefile import TraceFile, read_trace, write_trace
from .wave import WaveLayer

__version__ = "0.1.0"
