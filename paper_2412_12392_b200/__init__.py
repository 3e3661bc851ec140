"""B200-native hot paths of MASt3R-SLAM (arXiv 2412.12392).

Drop-in for the matching / tracking / backend-optimiser API of the CPU
reference "pmslam" (/root/reference/proj).  The compute is libpmx_cuda.so
(sm_100a CUDA, C ABI in include/pmx.h); this package is its host-side mirror.
"""
from . import abi
from .api import (Context, FeatureMap, Graph, MatchSet, OptimizeResult, PmxDomainError, PmxError,
                  PmxInvalidArgument, Pointmap, TrackResult, sim3)

__all__ = ["abi", "Context", "FeatureMap", "Graph", "MatchSet", "OptimizeResult", "PmxDomainError", "PmxError",
           "PmxInvalidArgument", "Pointmap", "TrackResult", "sim3"]
