"""paper_2203_14685_b200 -- the HetuMoE (arXiv 2203.14685) token-routing hot
path, B200-native: a thin Python binding over libmoe_b200.so (include/moe.h).

Importing this package loads the CUDA library; if it is not built the import
fails (there is no CPU fallback).
"""
from ._lib import MoeError, lib as _lib

_lib()  # fail loudly now if libmoe_b200.so is missing

from .api import (ALGOS, KINDS, MODES, PRIOS, Comm, Gate, Routing, SimWorld, alltoall_plan, alltoallv_plan,  # noqa: E402
                  capacity, expert_offsets, expert_scale, gate, gate_backward, layout,
                  layout_backward, layout_packed, layout_packed_backward, reverse_layout,
                  reverse_layout_backward, reverse_layout_packed, reverse_layout_packed_backward,
                  get_tuning, set_tuning, tuned, version)
from . import autograd  # noqa: E402
from .route import RoutePipeline  # noqa: E402

__all__ = ["MoeError", "Comm", "SimWorld", "Gate", "Routing", "RoutePipeline", "alltoall_plan", "alltoallv_plan",
           "capacity",
           "expert_scale", "gate", "gate_backward", "layout", "layout_backward", "reverse_layout",
           "reverse_layout_backward", "autograd", "version", "expert_offsets", "layout_packed",
           "reverse_layout_packed", "layout_packed_backward", "reverse_layout_packed_backward", "KINDS", "MODES",
           "PRIOS", "ALGOS", "get_tuning", "set_tuning", "tuned"]
