"""B200-native encoder<->LLM data path of arXiv 2605.08962 (reference package `muxsim`).

Modules mirror the reference's API names:
  workload   pkg/src/muxsim/workload.py (hybrid_pack on the GPU)
  costs      pkg/src/muxsim/costs.py    (cost formulas; byte accounting)
  balance    SPEC.md:377-446            (kk_partition / LPT / grouped_reorder on the GPU)
  reshard    SPEC.md:448-508            (plan_reshard UlyssesUniform on the GPU)
and the tensor-level hot path:
  planner    one device plan per step
  dataplane  pack+dispatch / return+scatter kernels over NVLink peer pointers
The compute lives in libmuxb200.so (csrc/, C ABI in include/mux_b200.h).
"""

__version__ = "0.1.0"
