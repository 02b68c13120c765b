"""B200-native wave-index decode attention (RetroInfer, arXiv 2505.02922).

Drop-in for the decode-attention path of the reference package ``tierkv``:
the same public names (tierkv __init__.py:10-22) backed by hand-written
sm_100a kernels in ``libwavekv.so`` (include/wavekv.h).  The batched
multi-request / GQA engine is ``WaveLayer``; ``HeadEngine`` and the
function-level API (attention / index / block cache / store / metrics) are
the per-head forms tierkv's callers and tests use.
"""

from .config import EngineConfig, IndexConfig, round_half_up
from .errors import ConfigError, IntegrityError, TierKVError, TraceFormatError
from .attention import (AttentionOutput, PartialAttention, estimate_partial, exact_partial, merge,
                        merged_sums, oracle_attention, tail_denominator_partial)
from .store import Block, SlowTierStore, TokenKV, block_capacity
from .block_cache import BlockCache, ClusterDescriptor, ExecutionBuffer
from .clustering import spherical_kmeans
from .index import ClusterIndex, MetaIndexEntry, ZonePlan, finalize_cluster, plan_zones, rank_clusters
from .metrics import recall_at_k, relative_l2, top_k_token_ids
from .engine import HeadEngine, StepMetrics
from .runner import TraceEngine, oracle_trace, run_trace
from .tracefile import TraceFile, read_trace, write_trace
from .wave import WaveLayer

__version__ = "0.1.0"
