"""C-ABI checks that need no GPU: libmoe_b200.so loads, exports every symbol
include/moe.h declares, and rejects bad arguments on the host BEFORE
enqueuing anything (include/moe.h "Arguments are validated on the host")."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

import paper_2203_14685_b200 as moe
from paper_2203_14685_b200._lib import SIGNATURES, SO_PATH, GateDesc, RoutingC, lib

HEADER = os.path.join(ROOT, "include", "moe.h")

OK, INVALID, UNSUPPORTED, ALIGN, WS, CUDA = 0, 1, 2, 3, 4, 5


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+[\s\*]+(moe_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_four_calls():
    fns = declared_functions()
    for f in ("moe_gate", "moe_layout", "moe_alltoall", "moe_reverse_layout"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    fns = declared_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", SO_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [f for f in fns if f not in exported]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert sorted(n for n, _, _ in SIGNATURES) == fns
    L = lib()
    for f in fns:
        assert getattr(L, f) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", SO_PATH], capture_output=True, text=True,
                         check=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_links_torch_nccl():
    out = subprocess.run(["ldd", SO_PATH], capture_output=True, text=True, check=True).stdout
    line = [l for l in out.splitlines() if "libnccl" in l][0]
    assert "nvidia/nccl/lib" in line  # the 2.28 torch loads, not /usr/lib's 2.27
    assert moe.version().startswith("libmoe_b200 sm_100a nccl-2.28")


def test_capacity_matches_oracle(orc):
    for S in (1, 3, 4, 100, 1024, 32768, 65536):
        for E in (1, 2, 3, 8, 32, 64):
            for k in (1, 2, 3):
                for C in (0.5, 1.0, 1.25, 2.0):
                    assert moe.capacity(S, E, k, C) == orc.capacity(S, E, k, C)
    with pytest.raises(ValueError):
        moe.capacity(0, 8, 1, 1.0)


FAKE = 0x7f0000001000  # 4 KiB aligned, never dereferenced: validation fails first


def _gate(desc, logits=FAKE, ids=None, table=None, vocab=0, routing="ok", ws=FAKE, ws_bytes=1 << 30):
    r = RoutingC(FAKE, FAKE, FAKE, FAKE, None) if routing == "ok" else routing
    return lib().moe_gate(ctypes.byref(desc), logits, ids, table, vocab,
                          None if r is None else ctypes.byref(r), ws, ws_bytes, None)


@pytest.mark.parametrize("fields,status", [
    (dict(S=0), INVALID), (dict(E=0), INVALID), (dict(k=0), INVALID), (dict(k=9), INVALID),
    (dict(capacity=0), INVALID), (dict(kind=5), INVALID), (dict(weight_mode=2), INVALID),
    (dict(kind=4, k=2), INVALID),                                # Dense-to-Sparse needs k == E
    (dict(priority=5), INVALID), (dict(kind=1, k=3), INVALID),   # E % k != 0
    (dict(kind=2, k=2), INVALID),                                # hash needs k == 1
    (dict(E=257, k=1), UNSUPPORTED),
    (dict(E=256, k=9, priority=1), UNSUPPORTED),                 # k*E > 2048 columns
])
def test_gate_rejects_invalid_desc(fields, status):
    base = dict(S=64, E=8, k=2, capacity=16, kind=0, weight_mode=0, priority=0)
    base.update(fields)
    d = GateDesc(**base)
    ws_need = lib().moe_gate_workspace_bytes(ctypes.byref(d))
    if status == INVALID:
        assert ws_need == 0
    assert _gate(d) == status
    assert lib().moe_last_error().decode().startswith("moe_gate")


def test_gate_ex_kinds_need_their_inputs():
    """SAM / D2S go through moe_gate_ex; their extra inputs are checked on the
    host before anything is enqueued."""
    from paper_2203_14685_b200._lib import GateInputs
    L = lib()
    r = RoutingC(FAKE, FAKE, FAKE, FAKE, None)
    sam = GateDesc(64, 8, 2, 16, 3, 0, 0)
    assert _gate(sam) == INVALID and "moe_gate_ex" in L.moe_last_error().decode()
    need = L.moe_gate_workspace_bytes(ctypes.byref(sam))
    assert need > 0

    def ex(d, **kw):
        base = dict(logits=FAKE, token_ids=None, table=None, vocab=0, group_logits=FAKE,
                    n_groups=2, uniforms=None, tau=1.0, eps=1e-3)
        base.update(kw)
        return L.moe_gate_ex(ctypes.byref(d), ctypes.byref(GateInputs(**base)), ctypes.byref(r),
                             FAKE, need, None)
    assert ex(sam, group_logits=None) == INVALID
    assert ex(sam, n_groups=3) == INVALID                # 3 does not divide E = 8
    assert ex(sam, n_groups=8) == INVALID                # k = 2 > E/n_groups = 1
    assert ex(GateDesc(64, 64, 9, 16, 3, 0, 0), n_groups=4) == UNSUPPORTED  # k > 8
    d2s = GateDesc(64, 8, 8, 16, 4, 0, 0)
    assert ex(d2s, tau=0.0) == INVALID
    assert ex(d2s, eps=-1.0) == INVALID


def test_gate_rejects_missing_buffers():
    d = GateDesc(64, 8, 2, 16, 0, 0, 0)
    assert _gate(d, logits=None) == INVALID
    assert _gate(d, routing=None) == INVALID
    assert _gate(d, routing=RoutingC(FAKE, None, FAKE, FAKE, None)) == INVALID
    assert _gate(d, ws=None) == WS
    need = lib().moe_gate_workspace_bytes(ctypes.byref(d))
    assert need > 0
    assert _gate(d, ws_bytes=need - 1) == WS
    assert "workspace" in lib().moe_last_error().decode()
    assert _gate(d, logits=FAKE + 2) == ALIGN
    h = GateDesc(64, 8, 1, 16, 2, 0, 0)
    assert _gate(h, logits=None, ids=FAKE, table=None, vocab=10) == INVALID
    assert _gate(h, logits=None, ids=FAKE, table=FAKE, vocab=0) == INVALID


def test_gate_without_gpu_fails_loudly():
    """Valid arguments on a box with no GPU: the launch fails with MOE_ERR_CUDA
    (there is no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    d = GateDesc(64, 8, 2, 16, 0, 0, 0)
    assert _gate(d) == CUDA


def _rows(fn, d, x=FAKE, out=FAKE, dcols=1024, dtype=1, r="ok"):
    rr = RoutingC(FAKE, FAKE, FAKE, FAKE, None) if r == "ok" else r
    return getattr(lib(), fn)(ctypes.byref(d), None if rr is None else ctypes.byref(rr), x, dcols,
                              dtype, out, None)


@pytest.mark.parametrize("fn", ["moe_layout", "moe_reverse_layout"])
def test_rows_validation(fn):
    d = GateDesc(64, 8, 2, 16, 0, 0, 0)
    assert _rows(fn, d, dtype=7) == INVALID
    assert _rows(fn, d, dcols=0) == INVALID
    assert _rows(fn, d, x=None) == INVALID
    assert _rows(fn, d, r=None) == INVALID
    assert _rows(fn, d, dcols=4, dtype=1) == ALIGN       # 8-byte rows
    assert _rows(fn, d, dcols=6, dtype=0) == ALIGN       # 24-byte rows
    assert _rows(fn, d, x=FAKE + 8) == ALIGN
    bad = GateDesc(64, 8, 9, 16, 0, 0, 0)
    assert _rows(fn, bad) == INVALID


def test_alltoall_and_plan_validation():
    L = lib()
    assert L.moe_alltoall(None, 0, 1, FAKE, FAKE, 64, None, 0, None) == INVALID
    n = ctypes.c_int32(0)
    assert L.moe_alltoall_plan(8, 0, 1, 3, None, 0, ctypes.byref(n)) == INVALID  # 8 % 3
    assert L.moe_alltoall_plan(8, 8, 0, 1, None, 0, ctypes.byref(n)) == INVALID  # rank range
    assert L.moe_alltoall_plan(8, 0, 0, 1, None, 0, ctypes.byref(n)) == INVALID  # no room
    assert n.value == 16
    assert L.moe_alltoall_workspace_bytes(8, 0, 4, 1 << 20) == 0
    assert L.moe_alltoall_workspace_bytes(8, 1, 4, 1 << 20) == 2 * 4 * 8 * (1 << 20)
    assert L.moe_expert_scale(FAKE, FAKE, 0, 1, 0, 1, 8, 1, None) == INVALID
    for s in range(7):
        assert L.moe_status_str(s).decode().startswith("MOE_")


def test_backward_and_packed_entry_points_validate_on_host():
    """The NEXT-1 / NEXT-4 entry points reject bad arguments before anything
    is enqueued (no GPU needed: validation fails first)."""
    from paper_2203_14685_b200._lib import i64
    L = lib()
    d = GateDesc(64, 8, 2, 16, 0, 0, 0)
    r = RoutingC(FAKE, FAKE, FAKE, FAKE, None)
    rd, dr = ctypes.byref(d), ctypes.byref(r)
    # combine adjoint: d_back / d_weight required, alignment, dtype
    assert L.moe_reverse_layout_backward(rd, dr, FAKE, FAKE, 64, 1, None, FAKE, None) == INVALID
    assert L.moe_reverse_layout_backward(rd, dr, FAKE, FAKE, 64, 1, FAKE + 8, FAKE, None) == ALIGN
    assert L.moe_reverse_layout_backward(rd, dr, FAKE, FAKE, 64, 7, FAKE, FAKE, None) == INVALID
    assert L.moe_reverse_layout_backward(rd, dr, FAKE, FAKE, 3, 1, FAKE, FAKE, None) == ALIGN
    # layout adjoint
    assert L.moe_layout_backward(rd, dr, None, 64, 1, FAKE, None) == INVALID
    assert L.moe_layout_backward(rd, dr, FAKE, 64, 1, FAKE + 4, None) == ALIGN
    # gate adjoint: the hash gate has no logits
    h = GateDesc(64, 8, 1, 16, 2, 0, 0)
    assert L.moe_gate_backward(ctypes.byref(h), FAKE, dr, FAKE, FAKE, None) == INVALID
    assert "hash" in L.moe_last_error().decode()
    assert L.moe_gate_backward(rd, FAKE, dr, None, FAKE, None) == INVALID
    # packed form
    assert L.moe_expert_offsets(rd, dr, None, None) == INVALID
    assert L.moe_layout_packed(rd, dr, None, FAKE, 64, 1, FAKE, None) == INVALID
    assert L.moe_reverse_layout_packed(rd, dr, None, FAKE, 64, 1, FAKE, None) == INVALID
    assert L.moe_layout_packed(rd, dr, FAKE, FAKE, 3, 1, FAKE, None) == ALIGN
    # alltoallv and the device-side exchanges need a communicator
    rows = (i64 * 1)(0)
    assert L.moe_alltoallv(None, FAKE, rows, FAKE, rows, 64, None) == INVALID
    assert L.moe_dispatch_packed_p2p(None, rd, dr, FAKE, FAKE, FAKE, FAKE, FAKE, 64, 1, FAKE,
                                     1 << 20, 0, None) == INVALID
    assert L.moe_combine_packed_p2p(None, rd, dr, FAKE, FAKE, FAKE, 64, 1, 1 << 20, FAKE, 0,
                                    None) == INVALID
    assert L.moe_combine_backward_p2p(None, rd, dr, FAKE, FAKE, 64, 1, FAKE, FAKE, 0, None) == INVALID
    assert L.moe_dispatch_backward_p2p(None, rd, dr, FAKE, 64, 1, FAKE, 0, None) == INVALID


def test_tuning_table_roundtrip_and_validation():
    """moe_get/set_tuning: the process-wide kernel-variant table (read once
    from the environment, include/moe.h "tuning"); out-of-range values are
    rejected without changing it."""
    before = moe.get_tuning()
    assert before["gate_tiles"] >= 1 and before["p2p_dedupe"] in (0, 1)
    with moe.tuned(gate_tiles=17, reverse_ku=2):
        t = moe.get_tuning()
        assert t["gate_tiles"] == 17 and t["reverse_ku"] == 2
    assert moe.get_tuning() == before
    for bad in ({"layout_u": 3}, {"reverse_ku": 1}, {"gate_bwd_lanes": 6},
                {"barrier_timeout_ms": -1}, {"nccl_cta_policy": 7},
                {"layout_tokens_per_warp": -1}, {"p2p_precombine": 2}):
        with pytest.raises(moe.MoeError) as ei:
            moe.set_tuning(**bad)
        assert ei.value.status == INVALID
        assert moe.get_tuning() == before
    with pytest.raises(KeyError):
        moe.set_tuning(no_such_field=1)


def test_alltoallv_plan_in_c():
    """moe_alltoallv_plan (host, C): send rows per destination rank from the
    expert offsets, receive rows and offsets from the received counts."""
    offsets = [0, 3, 3, 7, 9]           # E = 4, P = 2: rank 0 owns experts 0-1
    recv_counts = [1, 2, 5, 0]          # from rank 0: (1, 2), from rank 1: (5, 0)
    sr, rr, ro = moe.alltoallv_plan(offsets, recv_counts, 2)
    assert sr == [3, 6] and rr == [3, 5] and ro == [0, 1, 3, 8, 8]


def test_tuning_fields_match_the_header():
    """The binding's moe_tuning_t mirror lists the header's fields in order."""
    from paper_2203_14685_b200._lib import TUNING_FIELDS
    src = open(HEADER).read()
    body = src[src.index("typedef struct {\n  int32_t gate_tiles;"):src.index("} moe_tuning_t;")]
    assert re.findall(r"int32_t\s+(\w+);", body) == list(TUNING_FIELDS)
