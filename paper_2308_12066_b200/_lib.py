"""ctypes binding of libpgmoe.so (include/pgmoe.h).

The library is built in-tree by ``paper_2308_12066_b200.build`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or the device is not a B200, calls fail loudly.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libpgmoe.so")

OK, E_CONFIG, E_SHAPE, E_GATE_OVERFLOW, E_GATE_UNDERFLOW, E_ROUTING, E_OOM, E_CUDA, E_NCCL, \
    E_WEIGHT_FILE, E_INVARIANT = range(11)
F32, BF16, F64 = 0, 1, 2
RESIDENT, OFFLOADED = 0, 1
KERNEL_AUTO, KERNEL_SIMT, KERNEL_TCGEN05 = 0, 1, 2

_EXC = {
    E_CONFIG: errors.ConfigError,
    E_SHAPE: errors.ShapeError,
    E_GATE_OVERFLOW: errors.GateOverflowError,
    E_GATE_UNDERFLOW: errors.GateOverflowError,
    E_ROUTING: errors.RoutingError,
    E_OOM: errors.OomError,
    E_CUDA: errors.DeviceError,
    E_NCCL: errors.DeviceError,
    E_WEIGHT_FILE: errors.WeightFileError,
    E_INVARIANT: errors.InvariantError,
}


class Config(ctypes.Structure):
    _fields_ = [("d_model", ctypes.c_int32), ("d_ff", ctypes.c_int32), ("num_blocks", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("activation_level", ctypes.c_int32), ("seed", ctypes.c_uint64)]


class Routing(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("ids", "w", "hist", "off", "perm", "w_perm", "act", "n_act", "status", "inv")]


class IterationIO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("ids_trace", "w_trace", "x_trace", "ids_supplied", "w_supplied")]


class Stats(ctypes.Structure):
    _fields_ = [("pinned_hbm_bytes", ctypes.c_int64), ("slot_capacity_bytes", ctypes.c_int64),
                ("eq1_peak_bytes", ctypes.c_int64), ("ledger_peak_bytes", ctypes.c_int64),
                ("h2d_bytes", ctypes.c_int64), ("h2d_copies", ctypes.c_int64),
                ("route_fallbacks", ctypes.c_int64), ("reserved0", ctypes.c_int64),
                ("h2d_seconds", ctypes.c_double), ("last_step_seconds", ctypes.c_double),
                ("cache_bytes", ctypes.c_int64), ("cache_hits", ctypes.c_int64), ("cache_misses", ctypes.c_int64),
                ("d2d_bytes", ctypes.c_int64), ("fused_blocks", ctypes.c_int64),
                ("fused_routes", ctypes.c_int64)]


EXPORTS = (
    "pgmoe_route_workspace_bytes", "pgmoe_gate_forward", "pgmoe_expert_forward", "pgmoe_dense_forward",
    "pgmoe_check_routing", "pgmoe_fill_weights", "pgmoe_model_create", "pgmoe_model_destroy",
    "pgmoe_model_init_weights", "pgmoe_model_set_matrix", "pgmoe_model_get_matrix",
    "pgmoe_model_set_kernel", "pgmoe_decoder_iteration", "pgmoe_decoder_iteration_host",
    "pgmoe_moe_block_forward", "pgmoe_model_matrix_ptr", "pgmoe_model_stats", "pgmoe_model_reset_stats",
    "pgmoe_model_timeline_jsonl", "pgmoe_model_set_timeline", "pgmoe_last_error", "pgmoe_version",
    "pgmoe_launch_count", "pgmoe_model_create_ex", "pgmoe_model_expert_records", "pgmoe_gather_rows",
    "pgmoe_unpermute_combine", "pgmoe_ep_local_routing", "pgmoe_model_config", "pgmoe_weight_file_config",
    "pgmoe_model_load_pgmoe1", "pgmoe_model_save_pgmoe1", "pgmoe_model_set_strategy", "pgmoe_model_set_cache",
    "pgmoe_cache_replay", "pgmoe_debug_set_probe", "pgmoe_model_set_fused_route",
    "pgmoe_ep_pack_send", "pgmoe_ep_local_routing_padded", "pgmoe_ep_pack_recv", "pgmoe_ep_recv_route_pack",
    "pgmoe_expert_forward_packed",
    "pgmoe_ep_unpermute_padded", "pgmoe_ep_unpermute_padded_bf16", "pgmoe_dense_forward_packed", "pgmoe_ep_slot_rows", "pgmoe_route_from_decisions", "pgmoe_decoder_iteration_ex",
    "pgmoe_model_check_routing", "pgmoe_gate_forward_f64", "pgmoe_debug_green_context",
    "pgmoe_model_set_decode", "pgmoe_model_decode_iterations",
    "pgmoe_model_set_ll_decode", "pgmoe_model_ll_decode_iterations", "pgmoe_model_block_stamps",
)

_lib = None


def load():
    """Load libpgmoe.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PGMOE_LIB_PATH", LIB_PATH)  # A/B of library builds (tools/)
    if not os.path.exists(path):
        raise errors.DeviceError(
            f"{path} is missing: build it with `python -m paper_2308_12066_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "pgmoe_route_workspace_bytes": (sz, [i32, i32]),
        "pgmoe_gate_forward": (i32, [vp, i32, i32, vp, i32, i32, i32, P(Routing), vp, vp]),
        "pgmoe_expert_forward": (i32, [vp, i32, i32, i32, i32, vp, sz, i32, i32, P(Routing), vp, vp, i32, vp]),
        "pgmoe_dense_forward": (i32, [vp, i32, i32, i32, vp, i32, vp, i32, vp]),
        "pgmoe_check_routing": (i32, [P(Routing), P(i32)]),
        "pgmoe_route_from_decisions": (i32, [vp, vp, i32, i32, i32, P(Routing), vp]),
        "pgmoe_model_check_routing": (i32, [vp]),
        "pgmoe_debug_green_context": (i32, [i32, P(i32)]),
        "pgmoe_gate_forward_f64": (i32, [vp, i32, i32, vp, i32, i32, P(Routing), vp, vp]),
        "pgmoe_decoder_iteration_ex": (i32, [vp, vp, i32, vp, P(IterationIO), vp]),
        "pgmoe_fill_weights": (i32, [vp, i32, ctypes.c_uint64, i32, i32, i32, i64, i64, vp]),
        "pgmoe_model_create": (i32, [P(Config), i32, i32, i32, P(vp)]),
        "pgmoe_model_destroy": (i32, [vp]),
        "pgmoe_model_init_weights": (i32, [vp]),
        "pgmoe_model_set_matrix": (i32, [vp, ctypes.c_char_p, i32, i32, vp, sz]),
        "pgmoe_model_get_matrix": (i32, [vp, ctypes.c_char_p, i32, i32, vp, sz]),
        "pgmoe_model_set_kernel": (i32, [vp, i32]),
        "pgmoe_decoder_iteration": (i32, [vp, vp, i32, vp, vp, vp, vp]),
        "pgmoe_decoder_iteration_host": (i32, [vp, vp, i32, vp, vp, vp]),
        "pgmoe_moe_block_forward": (i32, [vp, i32, vp, i32, P(Routing), vp, P(Routing), vp]),
        "pgmoe_model_matrix_ptr": (vp, [vp, ctypes.c_char_p, i32, i32]),
        "pgmoe_model_stats": (i32, [vp, P(Stats)]),
        "pgmoe_model_reset_stats": (i32, [vp]),
        "pgmoe_model_timeline_jsonl": (i64, [vp, ctypes.c_char_p, i64]),
        "pgmoe_model_set_timeline": (i32, [vp, i32]),
        "pgmoe_last_error": (ctypes.c_char_p, []),
        "pgmoe_version": (ctypes.c_char_p, []),
        "pgmoe_launch_count": (i64, []),
        "pgmoe_model_create_ex": (i32, [P(Config), i32, i32, i32, i32, i32, P(vp)]),
        "pgmoe_model_expert_records": (i32, [vp, i32, P(vp), P(sz), P(i32), P(i32)]),
        "pgmoe_gather_rows": (i32, [vp, vp, i32, i32, i32, vp, vp]),
        "pgmoe_unpermute_combine": (i32, [vp, vp, vp, i32, i32, vp, vp]),
        "pgmoe_ep_local_routing": (i32, [vp, i32, i32, P(Routing), vp]),
        "pgmoe_model_config": (i32, [vp, P(Config), P(i32)]),
        "pgmoe_model_set_strategy": (i32, [vp, i32]),
        "pgmoe_model_set_cache": (i32, [vp, i32, ctypes.c_double]),
        "pgmoe_cache_replay": (i32, [i32, i32, vp, vp, i32, vp, vp]),
        "pgmoe_weight_file_config": (i32, [ctypes.c_char_p, P(Config)]),
        "pgmoe_model_load_pgmoe1": (i32, [vp, ctypes.c_char_p]),
        "pgmoe_model_save_pgmoe1": (i32, [vp, ctypes.c_char_p]),
        "pgmoe_debug_set_probe": (i32, [i32, vp, i64]),
        "pgmoe_model_set_fused_route": (i32, [vp, i32]),
        "pgmoe_model_set_decode": (i32, [vp, i32, i32]),
        "pgmoe_model_decode_iterations": (i64, [vp]),
        "pgmoe_model_set_ll_decode": (i32, [vp, i32, i32]),
        "pgmoe_model_ll_decode_iterations": (i64, [vp]),
        "pgmoe_model_block_stamps": (i32, [vp, vp, i32]),
        "pgmoe_ep_pack_send": (i32, [vp, P(Routing), i32, i32, i32, i32, i32, i32, vp, vp]),
        "pgmoe_ep_local_routing_padded": (i32, [vp, i32, i32, i32, i32, P(Routing), vp]),
        "pgmoe_ep_slot_rows": (i32, [i32, i32, i32]),
        "pgmoe_ep_pack_recv": (i32, [vp, P(Routing), i32, i32, i32, vp, vp]),
        "pgmoe_ep_recv_route_pack": (i32, [vp, i32, i32, i32, i32, P(Routing), vp, vp]),
        "pgmoe_expert_forward_packed": (i32, [vp, i32, i32, i32, vp, sz, P(Routing), vp, vp, vp]),
        "pgmoe_ep_unpermute_padded": (i32, [vp, P(Routing), i32, i32, i32, i32, i32, i32, vp, vp]),
        "pgmoe_ep_unpermute_padded_bf16": (i32, [vp, P(Routing), i32, i32, i32, i32, i32, vp, vp]),
        "pgmoe_dense_forward_packed": (i32, [vp, i32, i32, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return load().pgmoe_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map a pgmoe_status onto the reference exception tree."""
    if status == OK:
        return
    msg = last_error() or what
    if status == E_GATE_OVERFLOW:
        msg = "numerical overflow in gate"            # core.py:298
    elif status == E_GATE_UNDERFLOW:
        msg = "gate routing weight underflowed to zero"  # core.py:304
    raise _EXC.get(status, errors.MoESimError)(msg)
