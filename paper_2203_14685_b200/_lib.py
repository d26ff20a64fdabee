"""ctypes declarations of libmoe_b200.so (include/moe.h).  Argument
marshalling only: every step of the routing path runs in the library's CUDA
kernels or NCCL.  There is no fallback: if the shared library is missing the
import of the binding fails loudly."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libmoe_b200.so")

i32, i64, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
vp = ctypes.c_void_p


class GateDesc(ctypes.Structure):
    """moe_gate_desc_t"""
    _fields_ = [("S", i32), ("E", i32), ("k", i32), ("capacity", i32), ("kind", i32),
                ("weight_mode", i32), ("priority", i32)]


class RoutingC(ctypes.Structure):
    """moe_routing_t"""
    _fields_ = [("expert_idx", vp), ("slot_idx", vp), ("weight", vp), ("load", vp),
                ("slot_src", vp)]


class GateInputs(ctypes.Structure):
    """moe_gate_inputs_t"""
    _fields_ = [("logits", vp), ("token_ids", vp), ("table", vp), ("vocab", i32),
                ("group_logits", vp), ("n_groups", i32), ("uniforms", vp),
                ("tau", ctypes.c_double), ("eps", ctypes.c_double)]


class A2AOp(ctypes.Structure):
    """moe_a2a_op_t"""
    _fields_ = [("phase", i32), ("op", i32), ("peer", i32), ("src_buf", i32), ("dst_buf", i32),
                ("src_off", i64), ("dst_off", i64), ("chunks", i64)]


TUNING_FIELDS = ("gate_tiles", "gate_max_tile", "gate_two_maxw", "layout_u",
                 "layout_pads_first", "reverse_ku", "reverse_tpw", "reverse_kspec",
                 "reverse_backwards", "reverse_y_ef", "row_ctas_per_sm", "reverse_ctas_per_sm",
                 "combine_ctas_per_sm", "combine_bwd_kspec",
                 "gate_bwd_lanes", "p2p_dedupe", "p2p_local_pad", "a2a_ctas_per_sm",
                 "barrier_timeout_ms", "barrier_pdl", "disable_p2p", "nccl_alltoall", "nccl_max_ctas",
                 "nccl_min_ctas", "nccl_cta_policy", "layout_tokens_per_warp",
                 "p2p_precombine")


class Tuning(ctypes.Structure):
    """moe_tuning_t"""
    _fields_ = [(f, i32) for f in TUNING_FIELDS]


# (name, restype, argtypes) for every symbol include/moe.h declares
SIGNATURES = [
    ("moe_capacity", i32, [i32, i32, i32, ctypes.c_double]),
    ("moe_gate_workspace_bytes", sz, [ctypes.POINTER(GateDesc)]),
    ("moe_gate_kernel_count", i32, [ctypes.POINTER(GateDesc), i32]),
    ("moe_gate", ctypes.c_int, [ctypes.POINTER(GateDesc), vp, vp, vp, i32,
                                ctypes.POINTER(RoutingC), vp, sz, vp]),
    ("moe_gate_ex", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(GateInputs),
                                   ctypes.POINTER(RoutingC), vp, sz, vp]),
    ("moe_gate_layout", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(GateInputs),
                                       ctypes.POINTER(RoutingC), vp, sz, vp, i32, i32, vp, vp]),
    ("moe_gate_check", ctypes.c_int, [vp, vp, ctypes.POINTER(i32)]),
    ("moe_layout", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp, i32,
                                  i32, vp, vp]),
    ("moe_reverse_layout", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                          i32, i32, vp, vp]),
    ("moe_expert_scale", ctypes.c_int, [vp, vp, i32, i32, i32, i32, i32, i32, vp]),
    ("moe_expert_offsets", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                          vp]),
    ("moe_layout_packed", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                         vp, i32, i32, vp, vp]),
    ("moe_reverse_layout_packed", ctypes.c_int, [ctypes.POINTER(GateDesc),
                                                 ctypes.POINTER(RoutingC), vp, vp, i32, i32, vp,
                                                 vp]),
    ("moe_alltoallv", ctypes.c_int, [vp, vp, ctypes.POINTER(i64), vp, ctypes.POINTER(i64), sz, vp]),
    ("moe_dispatch_packed_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                               ctypes.POINTER(RoutingC), vp, vp, vp, vp, vp, i32,
                                               i32, vp, i64, i32, vp]),
    ("moe_combine_packed_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                              ctypes.POINTER(RoutingC), vp, vp, vp, i32, i32, i64,
                                              vp, i32, vp]),
    ("moe_reverse_layout_backward", ctypes.c_int, [ctypes.POINTER(GateDesc),
                                                   ctypes.POINTER(RoutingC), vp, vp, i32, i32,
                                                   vp, vp, vp]),
    ("moe_layout_backward", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                           i32, i32, vp, vp]),
    ("moe_gate_backward", ctypes.c_int, [ctypes.POINTER(GateDesc), vp, ctypes.POINTER(RoutingC),
                                         vp, vp, vp]),
    ("moe_reverse_layout_packed_backward", ctypes.c_int, [ctypes.POINTER(GateDesc),
                                                          ctypes.POINTER(RoutingC), vp, vp, vp,
                                                          i32, i32, vp, vp, vp]),
    ("moe_layout_packed_backward", ctypes.c_int, [ctypes.POINTER(GateDesc),
                                                  ctypes.POINTER(RoutingC), vp, vp, i32, i32, vp,
                                                  vp]),
    ("moe_gate_backward_ex", ctypes.c_int, [ctypes.POINTER(GateDesc), ctypes.POINTER(GateInputs),
                                            ctypes.POINTER(RoutingC), vp, vp, vp, vp]),
    ("moe_gate_dispatch_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                             ctypes.POINTER(GateInputs), ctypes.POINTER(RoutingC),
                                             vp, sz, vp, i32, i32, vp, i32, vp]),
    ("moe_combine_backward_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                                ctypes.POINTER(RoutingC), vp, vp, i32, i32, vp,
                                                vp, i32, vp]),
    ("moe_combine_backward_push_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                                     ctypes.POINTER(RoutingC), vp, vp, i32, i32,
                                                     vp, vp, vp, vp, i32, vp]),
    ("moe_combine_packed_backward_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                                       ctypes.POINTER(RoutingC), vp, vp, vp, vp,
                                                       i32, i32, i64, vp, vp, i32, vp]),
    ("moe_dispatch_packed_backward_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                                        ctypes.POINTER(RoutingC), vp, vp, vp, i32,
                                                        i32, i64, vp, i32, vp]),
    ("moe_dispatch_backward_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc),
                                                 ctypes.POINTER(RoutingC), vp, i32, i32, vp, i32,
                                                 vp]),
    ("moe_comm_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("moe_comm_init", ctypes.c_int, [ctypes.c_char_p, i32, i32, ctypes.POINTER(vp)]),
    ("moe_comm_destroy", ctypes.c_int, [vp]),
    ("moe_comm_size", ctypes.c_int, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
    ("moe_alltoall_workspace_bytes", sz, [i32, i32, i32, sz]),
    ("moe_alltoall", ctypes.c_int, [vp, i32, i32, vp, vp, sz, vp, sz, vp]),
    ("moe_alltoall_plan", ctypes.c_int, [i32, i32, i32, i32, ctypes.POINTER(A2AOp), i32,
                                         ctypes.POINTER(i32)]),
    ("moe_comm_symm_alloc", ctypes.c_int, [vp, sz, ctypes.POINTER(vp)]),
    ("moe_comm_symm_free", ctypes.c_int, [vp, vp]),
    ("moe_comm_barrier", ctypes.c_int, [vp, vp]),
    ("moe_dispatch_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                        i32, i32, vp, i32, vp]),
    ("moe_combine_p2p", ctypes.c_int, [vp, ctypes.POINTER(GateDesc), ctypes.POINTER(RoutingC), vp,
                                       i32, i32, vp, i32, vp]),
    ("moe_comm_check", ctypes.c_int, [vp, vp]),
    ("moe_comm_mem_alloc", ctypes.c_int, [vp, sz, ctypes.POINTER(vp)]),
    ("moe_comm_mem_free", ctypes.c_int, [vp, vp]),
    ("moe_comm_abort", ctypes.c_int, [vp]),
    ("moe_alltoallv_plan", ctypes.c_int, [i32, i32, vp, vp, vp, vp, vp]),
    ("moe_sim_world_create", ctypes.c_int, [i32, ctypes.POINTER(vp)]),
    ("moe_sim_world_comm", ctypes.c_int, [vp, i32, ctypes.POINTER(vp)]),
    ("moe_sim_world_run", ctypes.c_int, [vp, vp]),
    ("moe_sim_live_barrier", ctypes.c_int, [vp, i32, vp]),
    ("moe_sim_world_destroy", ctypes.c_int, [vp]),
    ("moe_set_trace", ctypes.c_int, [vp, sz]),
    ("moe_get_tuning", ctypes.c_int, [ctypes.POINTER(Tuning)]),
    ("moe_set_tuning", ctypes.c_int, [ctypes.POINTER(Tuning)]),
    ("moe_status_str", ctypes.c_char_p, [ctypes.c_int]),
    ("moe_last_error", ctypes.c_char_p, []),
    ("moe_version", ctypes.c_char_p, []),
]


class MoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError("libmoe_b200.so is not built (run `python "
                              "paper_2203_14685_b200/csrc/build.py`); there is no CPU fallback")
        L = ctypes.CDLL(SO_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        L = lib()
        raise MoeError(status, "%s%s: %s" % (what + ": " if what else "",
                                             L.moe_status_str(status).decode(),
                                             L.moe_last_error().decode()))
