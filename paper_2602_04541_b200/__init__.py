"""B200-native LycheeDecode hybrid-head decode attention (sm_100a).

The hot path -- retrieval-head split-KV decode attention with fused pooled
selection scores, cluster radix top-k into the per-head index cache,
sparse-head gather attention and the split-KV merge -- lives in the in-tree
CUDA library ``liblyc.so`` behind the C-ABI ``include/lyc.h``.  This package
is the Python mirror of the reference operator interface
(/root/reference/proj/include/hh: kernel_sim.hpp, attention.hpp, policy.hpp,
decode_engine.hpp).  There is no CPU fallback: importing the package without
the built library raises ImportError.
"""
from ._lib import (CudaError, InvalidArgument, LogicError, LycError, NotSupported, lib)
from .decode import HybridDecoder, SparsityPolicy, args_top_k, fraction_budget
from .kvcache import KvCache, correction_attention
from .model import DecodeModel, ModelConfig
from .kernel import (BlockIndexSet, CostReport, RunResult, SplitSchedule, WorkUnit, Workload,
                     latency_model, plan_splits, run)

lib()  # fail loudly at import when the native library is missing

__all__ = [
    "BlockIndexSet", "CostReport", "CudaError", "DecodeModel", "HybridDecoder", "InvalidArgument",
    "KvCache", "ModelConfig",
    "LogicError",
    "LycError", "NotSupported", "RunResult", "SparsityPolicy", "SplitSchedule", "WorkUnit",
    "Workload", "args_top_k", "correction_attention", "fraction_budget", "latency_model",
    "plan_splits", "run",
]
