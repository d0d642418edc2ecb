"""ctypes binding of the C-ABI in include/bittrain_b200.h.

This is the "reference-side binding" of INTEGRATION.md: plain pointers and
sizes, status codes mapped 1:1 onto errors.py.  There is no fallback: if the
library is missing or no CUDA device is present, device entry points raise.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["BT_LIB_PATH"]) if os.environ.get("BT_LIB_PATH") else PKG / "libbittrain_b200.so"

_u64, _i64, _i32, _dbl, _vp = C.c_uint64, C.c_int64, C.c_int32, C.c_double, C.c_void_p
_u64p, _i64p, _i32p, _dp = C.POINTER(C.c_uint64), C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double)

BT_P = 161
BT_MAX_TABLE = 64
BT_MAX_REPLICA_OUT = 8
BT_MAX_XDEV, BT_XSP = 8, 162
DTYPE_F64, DTYPE_F32 = 0, 1
REDUCE_UPDATE, REDUCE_MEAN_ONLY, REDUCE_SUM_ONLY, REDUCE_ADAM, REDUCE_MEAN_CHECK = 0, 1, 2, 3, 4
REDUCE_APPLY_SGD, REDUCE_APPLY_ADAM = 5, 6

STATUS_TO_ERROR = {
    1: errors.InputError,
    2: errors.ConfigError,
    3: errors.StateError,
    4: errors.ProgressError,
    5: errors.NumericError,
    6: errors.CorruptionError,
    8: errors.VersionError,
}


class MlpArgs(C.Structure):
    """bt_mlp_args (paper_2208_14228_b200/csrc/bt_mlp.cuh)."""

    _fields_ = [
        ("E", _i32), ("est_base", _i32), ("E_total", _i32), ("B", _i32), ("X", _i32), ("K", _i32),
        ("fuse_reduce", _i32), ("est_per_cta", _i32), ("comm_fanin", _i32), ("est_fanin_uniform", _i32),
        ("rank_override", _i64), ("rate", _dbl), ("lr", _dbl), ("mu", _dbl), ("jitter", _dbl),
        ("replicas", _vp), ("est_fanin", _vp), ("rng", _vp), ("stat_mean", _vp), ("stat_count", _vp),
        ("grads", _vp), ("losses", _vp), ("rot", _vp), ("rows", _vp), ("dataset", _vp), ("lists", _vp),
        ("seed", _u64), ("step0", _i64), ("spe", _i64), ("epoch_base", _i64),
        ("flags", _vp), ("bar", _vp), ("param_trace", _vp), ("dataset_rows", _i64),
        ("n_dev", _i32), ("dev_index", _i32), ("xin", _vp * 8), ("xrep", _vp * 8),
    ]


class ReduceArgs(C.Structure):
    """bt_reduce_args (paper_2208_14228_b200/csrc/bt_reduce.cuh)."""

    _fields_ = [
        ("dtype", _i32), ("mode", _i32), ("E", _i32), ("fanin", _i32), ("nout", _i32), ("divisor", _i32),
        ("n", _i64), ("grads_ld", _i64), ("grads", _vp * BT_MAX_TABLE), ("rot", _vp),
        ("param", _vp), ("vel", _vp), ("param_out", _vp), ("vel_out", _vp),
        ("extra_param_out", _vp * BT_MAX_REPLICA_OUT), ("extra_vel_out", _vp * BT_MAX_REPLICA_OUT),
        ("lr", _dbl), ("mu", _dbl), ("flags", _vp),
        ("vel2", _vp), ("vel2_out", _vp), ("extra_vel2_out", _vp * BT_MAX_REPLICA_OUT),
        ("beta2", _dbl), ("eps", _dbl), ("bc1", _dbl), ("bc2", _dbl),
        ("stage", _vp), ("gate", _vp), ("ngate", _i32), ("pad_", _i32),
    ]


EXPORTS = {
    # name: (restype, argtypes)
    "bt_abi_version": (C.c_int, []),
    "bt_last_error": (C.c_char_p, []),
    "bt_device_count": (C.c_int, []),
    "bt_host_mix64": (_u64, [_u64]),
    "bt_host_derive_stream": (_u64, [_u64p, _i32]),
    "bt_host_fnv1a64": (_u64, [_vp, _i64]),
    "bt_host_shuffled_range": (C.c_int, [_i64, _u64, _i32p]),
    "bt_host_epoch_indices": (C.c_int, [_u64, _u64, _i64, _i32, _i32, _i32, _i32p]),
    "bt_host_layout_arrival_perm": (C.c_int, [_i64, _i32, _u64p, _i64p, _i32p]),
    "bt_host_rotation_table": (C.c_int, [_i32, _i32p, _i32p, _i32, _i64, _i32p]),
    "bt_splitmix64_draws": (C.c_int, [_u64, _u64, _i64, _vp, _vp, _vp]),
    "bt_reduce_sum_f64": (C.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "bt_init_random": (C.c_int, [_u64, _dbl, _i64, _vp, _vp]),
    "bt_tanh_f64": (C.c_int, [_vp, _i64, _vp, _vp]),
    "bt_fwd_bwd_mlp_f64": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _dbl, _i64, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _vp]),
    "bt_mlp_step": (C.c_int, [C.POINTER(MlpArgs), _vp]),
    "bt_mlp_run": (C.c_int, [C.POINTER(MlpArgs), _vp, _vp, _vp]),
    "bt_l2_flush": (C.c_int, [_vp, _i64, C.c_uint32, _vp]),
    "bt_mlp_run_sampled": (C.c_int, [C.POINTER(MlpArgs), _u64, _i64, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "bt_stage_wait": (C.c_int, [_vp]),
    "bt_mlp_run_group": (C.c_int, [C.POINTER(C.POINTER(MlpArgs)), _i32p, C.POINTER(_vp), _i32, C.POINTER(_vp),
                                   C.POINTER(_vp)]),
    "bt_mlp_step_profiled": (C.c_int, [C.POINTER(MlpArgs), _vp, _vp]),
    "bt_mlp_fused_fits": (C.c_int, [C.POINTER(MlpArgs)]),
    "bt_mlp_pick_est_per_cta": (C.c_int, [_i32, _i32]),
    "bt_reduce_update": (C.c_int, [C.POINTER(ReduceArgs), _vp]),
    "bt_gemm_bf16_tn": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "bt_gemm_bf16_tn_batched": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i64, _i64, _i32, _i32, _vp]),
    "bt_gemm_bf16_ffn": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _u64, _i64, _i32, _i32,
                                   C.c_float, _i32, _vp]),
    "bt_gemm_bf16_ffn_cs": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _u64, _i64, _i32,
                                      _i32, C.c_float, _i32, _vp]),
    "bt_colsum_fold": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _i64, _vp]),
    "bt_ffn_data": (C.c_int, [_u64, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "bt_ffn_fwd_act": (C.c_int, [_vp, _vp, _u64, _i64, _i32, _i32, _i32, _i32, C.c_float, _vp, _vp, _vp]),
    "bt_ffn_out": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "bt_ffn_bwd_act": (C.c_int, [_vp, _vp, _u64, _i64, _i32, _i32, _i32, _i32, C.c_float, _vp, _vp]),
    "bt_colsum_bf16": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "bt_transpose_to_bf16": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bt_cast_f32_bf16": (C.c_int, [_vp, _i64, _vp, _vp]),
    "bt_gemm_bf16_tn_ex": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _i32, _vp, _i32,
                                     _vp]),
    "bt_gemm_bf16_ex": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _i32, _vp, _i32, _i32,
                                  _vp]),
    "bt_gemm_conv": (C.c_int, [_i32, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp,
                               _i32, _i32, _i32, _i64, _i32, _vp]),
    "bt_colsum_bf16_strided": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp]),
    "bt_bert_data": (C.c_int, [_u64, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "bt_bert_tokens": (C.c_int, [_u64, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "bt_bert_embed_fwd": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "bt_rows_gather": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "bt_rows_scatter": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bt_bert_mlm_ce": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "bt_bert_embed_grad_scratch": (C.c_int, [_i32, _i32, _i32, _i64p, _i64p]),
    "bt_bert_embed_grad": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i64, _vp]),
    "bt_bert_attn": (C.c_int, [_i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _u64, _i64,
                               C.c_float, _vp, _vp]),
    "bt_bert_attn_ex": (C.c_int, [_i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _u64, _i64,
                                  C.c_float, _vp, _vp, _vp]),
    "bt_bert_attn_ex2": (C.c_int, [_i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _u64, _i64,
                                  C.c_float, _vp, _vp, _vp, _vp]),
    "bt_bert_ln_fwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                 _i32, _u64, _i64, C.c_float, C.c_float, _vp, _vp]),
    "bt_bert_ln_fwd_rc": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32,
                                    _i32, _i32, _i32, _i32, _u64, _i64, C.c_float, C.c_float, _vp, _vp]),
    "bt_bert_ln_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                 _u64, _i64, C.c_float, _vp, _vp]),
    "bt_bert_ln_fold": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp]),
    "bt_bert_mse": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "bt_cnn_data": (C.c_int, [_u64, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "bt_cnn_im2col": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp]),
    "bt_cnn_bn_stats": (C.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64,
                                  _i32, _i32, _i32, C.c_float, _vp]),
    "bt_cnn_bn_apply": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bt_cnn_bn_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "bt_cnn_add": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "bt_cnn_upsample": (C.c_int, [_vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bt_cnn_filter_taps": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "bt_cnn_add_s2": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp]),
    "bt_cnn_head": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _vp]),
    "bt_fold_splits": (C.c_int, [_vp, _i32, _i32, _i64, _vp, _i64, _vp]),
    "bt_cnn_conv_weights": (C.c_int, [C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i32p, _i32p, _i32p, _i32p,
                                      _i32, _vp]),
    "bt_cast_weights_bf16": (C.c_int, [C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i32p, _i32p, _i32, _vp]),
    "bt_sgd_step_f64": (C.c_int, [_vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _vp, _vp, _vp]),
    "bt_make_dataset": (C.c_int, [_u64, _i64, _i32, _vp, _vp]),
    "bt_jitter_gather": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i64, _u64, _i64, _i64, _dbl, _vp, _vp]),
    "bt_dropout_mask": (C.c_int, [_u64, _i64, _i32, _dbl, _vp, _vp]),
    "bt_replica_check": (C.c_int, [C.POINTER(_vp), _i32, _i64, _vp, _vp]),
    "bt_est_slot_copy": (C.c_int, [C.POINTER(_vp), C.POINTER(_vp), _i64p, _i32, _vp]),
    "bt_allgather_params": (C.c_int, [_i32, _vp, C.POINTER(_vp), _i32, _i64, _vp]),
    "bt_memcpy_async": (C.c_int, [_vp, _vp, _i64, _vp]),
    "bt_fnv1a64_chunks": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "bt_flags_reset": (C.c_int, [_vp, _vp]),
    "bt_step_status": (C.c_int, [_vp, _i32p, _i32p, _vp]),
    "bt_ipc_handle_size": (C.c_int, []),
    "bt_ipc_get_handle": (C.c_int, [_vp, _vp, _i64p]),
    "bt_stream_write_u32": (C.c_int, [_vp, C.c_uint32, _vp]),
    "bt_stream_wait_u32_geq": (C.c_int, [_vp, C.c_uint32, _vp]),
    "bt_ipc_open_handle": (C.c_int, [_vp, C.POINTER(_vp)]),
    "bt_ipc_close": (C.c_int, [_vp]),
    "bt_enable_peer_access": (C.c_int, [_i32]),
}

_lib = None


def lib():
    """Load libbittrain_b200.so (built by __graft_entry__.build / build.py)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            if os.environ.get("BT_AUTOBUILD", "1") == "1":
                from .build import build

                build()
            else:
                raise ImportError(f"{LIB_PATH} is missing; run `python paper_2208_14228_b200/build.py`")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.bt_abi_version() != 1:
            raise errors.VersionError(f"C-ABI version {L.bt_abi_version()} != 1")
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().bt_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Raise the errors.py class mapped from a C-ABI status."""
    if status == 0:
        return
    msg = last_error() or what
    exc = STATUS_TO_ERROR.get(status)
    if exc is None:
        raise RuntimeError(f"bittrain_b200 CUDA failure ({status}): {msg}")
    raise exc(msg)


def host_derive_stream(*words: int) -> int:
    arr = (C.c_uint64 * max(1, len(words)))(*[w & (2**64 - 1) for w in words])
    return lib().bt_host_derive_stream(arr, len(words))


def host_fnv1a64(data: bytes) -> int:
    return lib().bt_host_fnv1a64(data, len(data))
