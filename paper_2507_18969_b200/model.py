"""GPU ``EdpcModel``: the model-level operator seam (`pkg/src/edpc/model.py:184-300`).

``predict(contexts) -> (probs, cache)`` and ``train_step(cache, targets) ->
loss`` keep the reference's contract (shape checks, stale-cache ValueError,
mean NLL in nats) while the forward pass, backward pass and fused Adam run
in the sm_100a kernels of the context (``edpc_predict`` / ``edpc_train_step``).
Parameters live on the device in fp32; ``parameters_flat`` / ``load_flat``
move them in the reference's ``parameters()`` order.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import ModelConfig, VOCAB, model_param_count, param_offsets
from .init import init_params_f32


@dataclass
class StepCache:
    version: int
    contexts: np.ndarray


class DeviceContext:
    """Owns one ``edpc_ctx`` (one container on one device)."""

    def __init__(self, cfg: ModelConfig, segments: int, original_len: int, device: int = 0,
                 lane_begin: int = 0, lane_count: int | None = None,
                 numerics: int | None = None):
        lib = _lib.load()
        self.cfg = cfg
        self.device = device
        self.lane_begin = lane_begin
        self.lane_count = cfg.lanes if lane_count is None else lane_count
        self.segments = segments
        c = _lib.EdpcConfig.from_model_config(cfg)
        h = ctypes.c_void_p()
        _lib.check(lib.edpc_ctx_create_ex(ctypes.byref(c), segments, original_len, device,
                                          lane_begin, self.lane_count,
                                          -1 if numerics is None else int(numerics),
                                          ctypes.byref(h)))
        self.h = h
        L, npar, nsh = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.edpc_ctx_info(h, ctypes.addressof(L), ctypes.addressof(npar),
                                     ctypes.addressof(nsh)))
        self.lane_len, self.n_params, self.n_shared = L.value, npar.value, nsh.value

    def close(self):
        if getattr(self, "h", None):
            _lib.load().edpc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_flat(self, params: np.ndarray) -> None:
        p = np.ascontiguousarray(params, dtype=np.float32)
        _lib.check(_lib.load().edpc_load_params(self.h, p.ctypes.data, p.size))

    def params_flat(self) -> np.ndarray:
        out = np.empty(self.n_params, dtype=np.float32)
        _lib.check(_lib.load().edpc_get_params(self.h, out.ctypes.data, out.size))
        return out

    def numerics_flags(self) -> int:
        """EDPC_NUM_* flags of this context (recorded in the container)."""
        f = ctypes.c_int32()
        _lib.check(_lib.load().edpc_ctx_numerics(self.h, ctypes.byref(f)))
        return int(f.value)

    def numerics(self) -> dict:
        """GEMM numerics of this context (policy: a function of the config):
        tensor cores (tf32), fp16 operands for the MBRB branch / out-projection
        GEMMs, the fused LTE forward, tf32 operands rounded to nearest."""
        f = self.numerics_flags()
        return {"tcgen05": bool(f & _lib.NUM_TCGEN05), "fp16_mbrb": bool(f & _lib.NUM_FP16),
                "lte_fused": bool(f & _lib.NUM_LTE_FUSED), "rnd_tf32": bool(f & _lib.NUM_RND_TF32)}

    def state_checksum(self) -> str:
        """sha256 over the fp32 parameter bytes (the lockstep probe, `model.py:294-300`)."""
        return hashlib.sha256(self.params_flat().tobytes()).hexdigest()

    def last_probs(self) -> np.ndarray:
        out = np.empty((self.lane_count, VOCAB), dtype=np.float32)
        _lib.check(_lib.load().edpc_last_probs(self.h, out.ctypes.data))
        return out


class EdpcModel:
    """The full predictor on one device; construction order fixes the init stream."""

    def __init__(self, cfg: ModelConfig, *, device: int = 0, params: np.ndarray | None = None,
                 numerics: int | None = None):
        cfg.validate()
        self.cfg = cfg
        self._ctx = DeviceContext(cfg, 1, 0, device, numerics=numerics)
        self._ctx.load_flat(init_params_f32(cfg) if params is None else params)
        self._version = 0

    def predict(self, contexts: np.ndarray):
        cfg = self.cfg
        ctx = np.ascontiguousarray(contexts)
        if ctx.shape != (cfg.lanes, cfg.context_len):
            raise ValueError(f"contexts shape {ctx.shape} != ({cfg.lanes}, {cfg.context_len})")
        if ctx.size and (ctx.min() < 0 or ctx.max() >= VOCAB):
            raise ValueError("context byte out of range")
        c8 = np.ascontiguousarray(ctx, dtype=np.uint8)
        probs = np.empty((cfg.lanes, VOCAB), dtype=np.float32)
        _lib.check(_lib.load().edpc_predict(self._ctx.h, c8.ctypes.data, probs.ctypes.data))
        return probs.astype(np.float64), StepCache(self._version, c8)

    def train_step(self, cache: StepCache, targets: np.ndarray) -> float:
        if cache.version != self._version:
            raise ValueError("stale cache: model was updated since this predict")
        t = np.asarray(targets)
        if t.shape != (self.cfg.lanes,):
            raise ValueError(f"targets shape {t.shape} mismatches batch {self.cfg.lanes}")
        if t.size and (t.min() < 0 or t.max() >= VOCAB):
            raise ValueError("target symbol out of range")
        t8 = np.ascontiguousarray(t, dtype=np.uint8)
        loss = ctypes.c_float(0.0)
        _lib.check(_lib.load().edpc_train_step(self._ctx.h, t8.ctypes.data, ctypes.addressof(loss)))
        self._version += 1
        return float(loss.value)

    def parameters_flat(self) -> np.ndarray:
        return self._ctx.params_flat()

    def parameters(self) -> dict[str, np.ndarray]:
        flat = self.parameters_flat()
        return {n: flat[o: o + int(np.prod(s))].reshape(s) for n, (o, s) in param_offsets(self.cfg).items()}

    def load_flat(self, params: np.ndarray) -> None:
        self._ctx.load_flat(params)

    def state_checksum(self) -> str:
        return self._ctx.state_checksum()

    def numerics(self) -> dict:
        return self._ctx.numerics()

    def param_count(self) -> dict[str, int]:
        total = model_param_count(self.cfg)
        return {"total": total}
