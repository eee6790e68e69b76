"""ctypes binding of libmuxb200.so (include/mux_b200.h).

There is no fallback: if the library is missing or a call fails, the caller
gets an exception.  Status codes become the reference's exception types
(pkg/src/muxsim/workload.py:29-34).
"""

from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("MUX_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libmuxb200.so")  # env: A/B of two builds

MUX_OK, MUX_ERR_CONFIG, MUX_ERR_PACKING, MUX_ERR_VALUE, MUX_ERR_CUDA, MUX_ERR_RUNTIME = range(6)
MODE_PACK, MODE_STEP = 0, 1
LPT, KK, LPT_LOCAL, LPT_LOCAL_RW = 0, 1, 2, 3
N_GROUPS = 2

H_STATUS, H_ERR_INDEX, H_N_SEQ, H_N_DISPATCH, H_N_RETURN = 0, 1, 2, 3, 4
H_DISPATCH_CHUNKS, H_RETURN_CHUNKS, H_DISPATCH_BYTES, H_RETURN_BYTES = 5, 6, 7, 8
H_N_BATCH, H_DISPATCH_REMOTE, H_RETURN_REMOTE, H_RECV_ROWS0, H_RECV_ROWS1 = 9, 10, 11, 12, 13
H_STAGE_ROWS0, H_STAGE_ROWS1 = 14, 15
H_N_GRAD, H_GRAD_CHUNKS, H_GRAD_BYTES, H_GRAD_REMOTE, H_STAMP0 = 16, 17, 18, 19, 20
H_N_TEXT, H_TEXT_ROWS = 30, 31
RET_FINAL, RET_STAGED = 0, 1
H_SLOTS = 32


class PlanCfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "S", "n_carry", "n_carry_seqs", "n_chunks", "capacity", "gbs", "dp", "sp", "world",
        "mbs", "method", "pooled", "me", "mode")] + [
        ("row_bytes_in", C.c_int32 * N_GROUPS), ("row_bytes_ret", C.c_int32 * N_GROUPS),
        ("chunk_bytes", C.c_int32), ("ret_mode", C.c_int32),
        ("row_bytes_grad", C.c_int32 * N_GROUPS), ("lssp_sp", C.c_int32),
        ("lssp_eta", C.c_int32), ("reshard", C.c_int32), ("cp_threshold", C.c_int32),
        ("text_embed", C.c_int32), ("reorder_group", C.c_int32), ("cost_model", C.c_int32),
        ("reserved0", C.c_int32), ("cost_lin", C.c_double * N_GROUPS),
        ("cost_quad", C.c_double * N_GROUPS)]


LAYOUT_FIELDS = (
    "header", "sync", "seq", "off", "span", "origin", "origin_pos", "group", "enc", "arena_off",
    "enc_off", "stage_off", "llm_rank", "llm_row", "bin_fill", "bin_nspan", "bin_of", "chunk_nbins",
    "chunk_err", "fills", "nspans", "cu", "shard_len", "shard_start", "row_base", "arena_rows",
    "recv_rows", "stage_rows", "llm_rows", "order", "scratch_a", "scratch_b", "dseg_src_row", "dseg_dst_row",
    "dseg_rows", "dseg_group", "dseg_dst_rank", "dseg_chunk0", "rseg_src_row", "rseg_dst_row",
    "rseg_rows", "rseg_group", "rseg_dst_rank", "rseg_chunk0", "gseg_src_row", "gseg_dst_row",
    "gseg_rows", "gseg_group", "gseg_dst_rank", "gseg_chunk0", "lssp_state", "lssp_row",
    "lp_n", "lp_k", "lp_t0", "lp_len", "lp_row", "text_off", "tseg_src", "tseg_dst",
    "tseg_rows", "tseg_row0", "total")
RESHARD = {"ulysses": 0, "cp_hybrid": 1}
COST_TOKENS, COST_FLOPS = 0, 1
LSSP_MAX = 8


class PlanLayout(C.Structure):
    _fields_ = [(n, C.c_int64) for n in LAYOUT_FIELDS]


class ProjGroup(C.Structure):
    """mux_proj_group: one problem of a grouped projector launch."""
    _fields_ = [("X", C.c_void_p), ("W", C.c_void_p), ("bias", C.c_void_p),
                ("M_max", C.c_int64), ("M_dev", C.c_void_p), ("K", C.c_int32),
                ("reserved", C.c_int32), ("row_dst", C.c_void_p)]


# (name, restype, argtypes) for every exported symbol of include/mux_b200.h
_P = C.c_void_p
_SIGS = [
    ("mux_version", C.c_int, []),
    ("mux_abi_sizes", None, [_P]),
    ("mux_last_error", C.c_char_p, []),
    ("mux_plan_layout_of", C.c_int, [C.POINTER(PlanCfg), C.POINTER(PlanLayout)]),
    ("mux_plan_step", C.c_int, [C.POINTER(PlanCfg), _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    ("mux_plan_check", C.c_int, [C.POINTER(PlanCfg), _P, _P, _P]),
    ("mux_assign_scratch_bytes", C.c_size_t, [C.c_int32, C.c_int32]),
    ("mux_assign", C.c_int, [C.c_int32, _P, _P, C.c_int32, C.c_int32, _P, _P, _P]),
    ("mux_segcopy", C.c_int, [C.POINTER(PlanCfg), _P, C.c_int32, _P, _P, C.c_int32, _P, _P]),
    ("mux_segcopy_signal", C.c_int, [C.POINTER(PlanCfg), _P, C.c_int32, _P, _P, C.c_int32, _P,
                                     _P, _P, _P]),
    ("mux_segcopy_ex", C.c_int, [C.POINTER(PlanCfg), _P, C.c_int32, _P, _P, C.c_int32,
                                 C.c_int32, _P, _P, _P, _P, _P]),
    ("mux_copy_bytes", C.c_int, [_P, _P, C.c_int64, C.c_int32, _P]),
    ("mux_memcpy_async", C.c_int, [_P, _P, C.c_int64, _P]),
    ("mux_copy_ranges", C.c_int, [C.c_int32, _P, _P, _P, C.c_int64, C.c_int32, C.c_int32, _P]),
    ("mux_signal", C.c_int, [C.c_int32, C.c_int32, _P, _P, _P]),
    ("mux_wait", C.c_int, [C.c_int32, _P, _P, C.c_int32, _P, _P]),
    ("mux_signal_ex", C.c_int, [C.c_int32, C.c_int32, _P, _P, C.c_int32, _P]),
    ("mux_wait_value", C.c_int, [C.c_int32, _P, C.c_uint64, C.c_int32, _P, _P]),
    ("mux_encoder_standin", C.c_int, [C.POINTER(PlanCfg), _P, _P, _P, C.c_int32, C.c_int32, _P,
                                      _P]),
    ("mux_return_rows", C.c_int, [C.POINTER(PlanCfg), _P, C.c_int32, _P, C.c_int64, _P]),
    ("mux_stage_rows", C.c_int, [C.POINTER(PlanCfg), _P, _P, C.c_int32, _P, C.c_int64, _P]),
    ("mux_text_embed", C.c_int, [C.POINTER(PlanCfg), _P, _P, _P, C.c_int64, C.c_int32, _P, _P,
                                 _P]),
    ("mux_proj_scatter", C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P,
                                   C.c_int32, _P]),
    ("mux_proj_scatter_dev", C.c_int, [_P, _P, _P, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P,
                                       C.c_int32, _P]),
    ("mux_proj_scatter_grouped", C.c_int, [C.POINTER(ProjGroup), C.c_int32, C.c_int32, _P,
                                           C.c_int32, _P]),
    ("mux_proj_scatter_grouped_signal", C.c_int, [C.POINTER(ProjGroup), C.c_int32, C.c_int32,
                                                  _P, C.c_int32, C.c_int32, C.c_int32, _P, _P,
                                                  _P, _P, _P, _P, _P]),
    ("mux_meta_record_words", C.c_int64, [C.c_int32, C.c_int32]),
    ("mux_assemble_table", C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64, _P,
                                     _P]),
    ("mux_proj_backward_workspace", C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    ("mux_proj_backward", C.c_int, [_P, _P, _P, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P, _P,
                                    _P, C.c_size_t, C.c_int32, _P]),
]
EXPORTS = tuple(n for n, _, _ in _SIGS)

_lib = None


def lib():
    """Load libmuxb200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2605_08962_b200.build`")
        h = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            if os.environ.get("MUX_LIB_PATH") and not hasattr(h, name):
                continue  # an older build under A/B: bind what it has
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def last_error() -> str:
    return lib().mux_last_error().decode(errors="replace")


def raise_for(status: int, what: str = "") -> None:
    """Map a MUX_* status onto the reference's exception types."""
    if status == MUX_OK:
        return
    from .workload import ConfigError, PackingError
    msg = last_error()
    if status == MUX_ERR_CONFIG:
        raise ConfigError(msg)
    if status == MUX_ERR_PACKING:
        raise PackingError(msg)
    if status == MUX_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def check(status: int, what: str = "") -> None:
    raise_for(status, what)
