"""ctypes binding of the in-tree C-ABI library (include/edpc_b200.h).

The library is the only compute path: if it is missing, or no CUDA device is
visible, every compute call raises ``EdpcNativeError`` -- there is no CPU
fallback in the product (the CPU oracle under ``oracle/`` is test
infrastructure only).
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_edpc_b200.so")

OK, ERR_INVALID, ERR_CUDA, ERR_CODER, ERR_STATE, ERR_NOMEM = range(6)
# numerics flags (include/edpc_b200.h EDPC_NUM_*), recorded in the container
NUM_TCGEN05, NUM_FP16, NUM_LTE_FUSED, NUM_RND_TF32 = 1, 2, 4, 8
NUMERICS_MASK = 15
REGIONS = ["gemm", "fdm_fwd", "fdm_bwd_adam", "adam_shared", "softmax_quant", "encode",
           "decode", "colsum", "elementwise", "embed_grad"]


class EdpcNativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[edpc status {code}] {msg}")
        self.code = code


class EdpcConfig(ctypes.Structure):
    _fields_ = [("context_len", ctypes.c_int32), ("embed_dim", ctypes.c_int32),
                ("hidden_local", ctypes.c_int32), ("hidden_global", ctypes.c_int32),
                ("lte_ratio", ctypes.c_int32), ("branches", ctypes.c_int32),
                ("lanes", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("adam_eps", ctypes.c_double), ("seed", ctypes.c_uint64)]

    @classmethod
    def from_model_config(cls, cfg) -> "EdpcConfig":
        return cls(cfg.context_len, cfg.embed_dim, cfg.hidden_local, cfg.hidden_global,
                   cfg.lte_ratio, cfg.branches, cfg.lanes, 0, cfg.lr, cfg.beta1, cfg.beta2,
                   cfg.adam_eps, cfg.seed)


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SIGS = {
    "edpc_last_error": ([], ctypes.c_char_p),
    "edpc_abi_version": ([], ctypes.c_int),
    "edpc_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "edpc_has_tcgen05": ([], ctypes.c_int),
    "edpc_quantize_rows": ([ctypes.c_int, _P, _I64, ctypes.c_int, _P], ctypes.c_int),
    "edpc_encode_rows": ([ctypes.c_int, _P, _P, _I64, _P, _P, _I64], ctypes.c_int),
    "edpc_encode_finish": ([ctypes.c_int, _P, _P, _I64, _P], ctypes.c_int),
    "edpc_decoder_init": ([ctypes.c_int, _P, _P, _I64, _I64], ctypes.c_int),
    "edpc_decode_rows": ([ctypes.c_int, _P, _P, _I64, _I64, _P, _I64, _P, _P], ctypes.c_int),
    "edpc_ctx_create": ([ctypes.POINTER(EdpcConfig), _I32, _I64, _I32, _I32, _I32,
                         ctypes.POINTER(_P)], ctypes.c_int),
    "edpc_ctx_create_ex": ([ctypes.POINTER(EdpcConfig), _I32, _I64, _I32, _I32, _I32, _I32,
                            ctypes.POINTER(_P)], ctypes.c_int),
    "edpc_ctx_destroy": ([_P], ctypes.c_int),
    "edpc_ctx_info": ([_P, _P, _P, _P], ctypes.c_int),
    "edpc_load_params": ([_P, _P, _I64], ctypes.c_int),
    "edpc_get_params": ([_P, _P, _I64], ctypes.c_int),
    "edpc_set_input": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "edpc_set_input_columns": ([_P, _P, _I64, _I64, _I64], ctypes.c_int),
    "edpc_set_input_local": ([_P, _P, _I64], ctypes.c_int),
    "edpc_get_intervals": ([_P, _I64, _I64, _P], ctypes.c_int),
    "edpc_get_columns": ([_P, _I64, _I64, _P], ctypes.c_int),
    "edpc_compress_steps": ([_P, _I64, _I64], ctypes.c_int),
    "edpc_compress_finish": ([_P, _P, _P], ctypes.c_int),
    "edpc_get_payloads": ([_P, _P, _I64], ctypes.c_int),
    "edpc_set_payloads": ([_P, _P, _P], ctypes.c_int),
    "edpc_decompress_steps": ([_P, _I64, _I64], ctypes.c_int),
    "edpc_get_output": ([_P, _P, _I64], ctypes.c_int),
    "edpc_predict": ([_P, _P, _P], ctypes.c_int),
    "edpc_train_step": ([_P, _P, _P], ctypes.c_int),
    "edpc_last_probs": ([_P, _P], ctypes.c_int),
    "edpc_step_phase": ([_P, _I64, _I32, _I32], ctypes.c_int),
    "edpc_grad_partials": ([_P, _P, _P], ctypes.c_int),
    "edpc_ctx_groups": ([_P, _P, _P], ctypes.c_int),
    "edpc_partials_copy": ([_P, _I32, _I32, _P, _I32], ctypes.c_int),
    "edpc_encode_pending": ([_P, _I64], ctypes.c_int),
    "edpc_partials_pull": ([_P, _P], ctypes.c_int),
    "edpc_weights_pull": ([_P, _P], ctypes.c_int),
    "edpc_shard_range": ([_P, _P, _P], ctypes.c_int),
    "edpc_nccl_unique_id": ([_P, _I32], ctypes.c_int),
    "edpc_ctx_set_comm": ([_P, _P, _I32, _I32], ctypes.c_int),
    "edpc_sync": ([_P], ctypes.c_int),
    "edpc_trim_pool": ([ctypes.c_int32], ctypes.c_int),
    "edpc_debug_read": ([_P, _I32, _P, _I64], ctypes.c_int),
    "edpc_ctx_numerics": ([_P, _P], ctypes.c_int),
    "edpc_ksg_counts": ([_P, _I32, _P, _I32, _I64, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "edpc_debug_keep_grads": ([_P, _I32], ctypes.c_int),
    "edpc_debug_adam": ([_P, _P, _I64, _I32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                         ctypes.c_double, _P, _P, _P], ctypes.c_int),
    "edpc_debug_gemm": ([_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _I32], ctypes.c_int),
    "edpc_debug_gemm_h": ([_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _I32, _I32], ctypes.c_int),
    "edpc_bench_gemm": ([_I32, _I32, _I32, _I32, _I32, _I32, _I32, _P], ctypes.c_int),
    "edpc_prof": ([_P, ctypes.c_int], ctypes.c_int),
    "edpc_timer": ([_P, _I32, _P], ctypes.c_int),
    "edpc_prof_read": ([_P, _I32, _P, _P], ctypes.c_int),
}


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load(path: str | None = None):
    """Load (once) and return the library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise EdpcNativeError(ERR_CUDA, f"native library missing: {p} (run "
                                  "`python -m paper_2507_18969_b200.build`); there is no CPU fallback")
        lib = ctypes.CDLL(p)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(status: int) -> None:
    if status != OK:
        msg = load().edpc_last_error()
        raise EdpcNativeError(status, msg.decode() if msg else "unknown error")


def device_count() -> int:
    n = ctypes.c_int(0)
    st = load().edpc_device_count(ctypes.byref(n))
    return n.value if st == OK else 0


def require_device(device: int = 0) -> None:
    n = device_count()
    if n <= device:
        raise EdpcNativeError(ERR_CUDA, f"no CUDA device {device} visible ({n} found); the B200 "
                              "path has no CPU fallback")


def ptr(a) -> int:
    """Address of a numpy array / bytes-like for ctypes."""
    import numpy as np
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    raise TypeError(type(a))
