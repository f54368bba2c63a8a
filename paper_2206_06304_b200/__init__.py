"""B200-native solver engine for the offloading/scheduling hot path of
arXiv 2206.06304 (IP-SSA, same-sub-task aggregation, OG grouping, online
slot driver).  See DESIGN.md.

Layers:
  include/coinfer_b200.h      C ABI (plain pointers, SoA fp64, status codes)
  include/coinfer/*.hpp       C++ drop-in for the reference's API (Scenario,
                              ip_ssa, og, baseline, ...) on top of the ABI
  csrc/*.cu                   sm_100a kernels + the ABI implementation
  engine.Engine               batch API over numpy (host) or CUDA torch tensors
  shard                       weak-scaling instance shards for multi-GPU runs
"""
from ._abi import load_library  # noqa: F401
from .engine import Engine, ProfileArrays, SolverError  # noqa: F401
from .scenarios import profile_heavy, profile_light, sample_batch, sub_seed, synth_profile  # noqa: F401
