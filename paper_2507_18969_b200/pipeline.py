"""compress / decompress on the B200: the drop-in for `pkg/src/edpc/pipeline.py:109-298`.

Same signatures, same container, same geometry errors.  What moves:

* the DPCA segment scheduler becomes the lane geometry of the device
  context -- all B lanes are the M dimension of every per-step GEMM, and the
  S segments are S independent coders (one device thread/warp each);
* stage A (predict + train) and stage B (quantize + encode) are device
  streams: the quantizer runs in the softmax kernel, the encoder kernel
  consumes the interval ring on a second stream (``edpc_compress_steps``);
* decode runs on the critical path between predict(i) and train(i), on the
  device, with no host round trip per step.

``serial``, ``threads`` and ``queue_capacity`` are accepted for API
compatibility and never change bytes (as in the reference).  ``step_hook``
and ``param_probe`` still fire (they force a per-step host sync; debug
only).  Multi-GPU: pass ``devices=[...]`` (see dist.py).
"""

from __future__ import annotations

import ctypes
import time
from typing import Callable

import numpy as np

from . import _lib
from .config import ModelConfig
from .container import EdpcContainer, Header
from .coder import CoderError
from .init import init_params_f32
from .lanes import lane_len_for, validate_geometry
from .model import DeviceContext

StepHook = Callable[[int, np.ndarray, np.ndarray], None]
ParamProbe = Callable[[int, object], None]
DEFAULT_CHUNK = 512


def _stats(stats, **kw):
    if stats is not None:
        stats.update(kw)


def _devices(device: int, devices) -> tuple[int, list[int] | None]:
    """Normalise ``device`` / ``devices``: one entry means that device; more
    than one means the lane-sharded multi-GPU path (dist.py)."""
    if devices is None:
        return int(device), None
    devs = [int(d) for d in devices]
    if not devs:
        raise ValueError("devices must not be empty")
    if len(devs) == 1:
        return devs[0], None
    return devs[0], devs


def compress(data: bytes, cfg: ModelConfig, segments: int = 4, *,
             serial: bool = False, threads: int | None = None,
             queue_capacity: int = 8, stats: dict | None = None,
             step_hook: StepHook | None = None,
             param_probe: ParamProbe | None = None,
             probe_every: int = 0, device: int = 0, devices=None,
             chunk: int = DEFAULT_CHUNK) -> EdpcContainer:
    """Compress ``data`` into a self-describing container (bytes are a pure
    function of (data, cfg, segments))."""
    validate_geometry(cfg, segments)
    device, devs = _devices(device, devices)
    if devs is not None:
        from .dist import compress_multi
        return compress_multi(data, cfg, segments, devs, stats=stats)
    t0 = time.perf_counter()
    n = len(data)
    if n == 0:
        _stats(stats, steps=0, predict_s=0.0, train_s=0.0, encode_s=0.0,
               wall_s=time.perf_counter() - t0, peak_queue_depth=0)
        return EdpcContainer(header=Header.from_config(cfg, 0, []), segments=[])
    _lib.require_device(device)
    ctx = DeviceContext(cfg, segments, n, device)
    try:
        ctx.load_flat(init_params_f32(cfg))
        numerics = ctx.numerics_flags()
        setup_s = time.perf_counter() - t0
        buf = np.frombuffer(bytes(data), dtype=np.uint8)
        L = ctx.lane_len
        T = cfg.context_len
        lib = _lib.load()
        tl = time.perf_counter()
        if step_hook is None and (param_probe is None or not probe_every):
            # streaming ingest: each block of lane columns
            # goes H2D on the context's copy stream while the previous block's
            # model steps run; the steps wait only for their own columns
            for i0 in range(0, L, chunk):
                i1 = min(L, i0 + chunk)
                _lib.check(lib.edpc_set_input_columns(ctx.h, buf.ctypes.data, n, i0, i1))
                _lib.check(lib.edpc_compress_steps(ctx.h, i0, i1))
        else:
            _lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, n, 0))
            _lib.check(lib.edpc_compress_steps(ctx.h, 0, min(T, L)))
            mat = None
            if step_hook is not None:
                mat = np.zeros((cfg.lanes, L), dtype=np.uint8)
                mat.reshape(-1)[:n] = buf
            for i in range(T, L):
                _lib.check(lib.edpc_compress_steps(ctx.h, i, i + 1))
                if step_hook is not None:
                    step_hook(i, ctx.last_probs().astype(np.float64), mat[:, i].copy())
                if probe_every and param_probe is not None and (i - T + 1) % probe_every == 0:
                    param_probe(i, ctx)
        _lib.check(lib.edpc_sync(ctx.h))
        loop_s = time.perf_counter() - tl
        te = time.perf_counter()
        bits = np.zeros(segments, dtype=np.int64)
        total = ctypes.c_int64(0)
        _lib.check(lib.edpc_compress_finish(ctx.h, bits.ctypes.data, ctypes.addressof(total)))
        finish_s = time.perf_counter() - te
        pay = np.zeros(max(total.value, 1), dtype=np.uint8)
        _lib.check(lib.edpc_get_payloads(ctx.h, pay.ctypes.data, pay.size))
        d2h_s = time.perf_counter() - te - finish_s
    finally:
        tc = time.perf_counter()
        ctx.close()
        close_s = time.perf_counter() - tc
    payloads, pos = [], 0
    for b in bits.tolist():
        nb = (b + 7) // 8
        payloads.append(pay[pos: pos + nb].tobytes())
        pos += nb
    _stats(stats, steps=max(0, L - T), predict_s=loop_s, train_s=0.0,
           encode_s=time.perf_counter() - te, wall_s=time.perf_counter() - t0,
           peak_queue_depth=0, setup_s=setup_s, device_loop_s=loop_s, finish_s=finish_s,
           payload_d2h_s=d2h_s, close_s=close_s,
           note="predict, quantize, encode and train run as one device schedule: "
                "predict_s is the whole device loop, train_s is inside it")
    return EdpcContainer(header=Header.from_config(cfg, n, bits.tolist(), numerics),
                         segments=payloads)


def decompress(container: EdpcContainer, *, threads: int = 1, stats: dict | None = None,
               step_hook: StepHook | None = None, param_probe: ParamProbe | None = None,
               probe_every: int = 0, device: int = 0, devices=None,
               chunk: int = DEFAULT_CHUNK) -> bytes:
    """Reconstruct the original bytes by replaying the encoder's schedule."""
    t0 = time.perf_counter()
    header = container.header
    header.validate()
    n = header.original_len
    if n == 0:
        _stats(stats, steps=0, wall_s=time.perf_counter() - t0)
        return b""
    cfg = header.model_config()
    segments = header.segment_count
    validate_geometry(cfg, segments)
    if len(container.segments) != segments:
        raise ValueError("segment payload count mismatch")
    for s, (p, b) in enumerate(zip(container.segments, header.bit_lengths)):
        if b > len(p) * 8:
            raise CoderError(f"segment {s}: bit length {b} exceeds payload of {len(p)} bytes")
    device, devs = _devices(device, devices)
    if devs is not None:
        from .dist import decompress_multi
        return decompress_multi(container, devs, stats=stats)
    _lib.require_device(device)
    lib = _lib.load()
    # replay the encoder's numerics (recorded in the version byte)
    ctx = DeviceContext(cfg, segments, n, device, numerics=header.numerics)
    try:
        ctx.load_flat(init_params_f32(cfg))
        pay = np.frombuffer(b"".join(container.segments) or b"\0", dtype=np.uint8)
        bits = np.ascontiguousarray(header.bit_lengths, dtype=np.int64)
        _lib.check(lib.edpc_set_payloads(ctx.h, pay.ctypes.data, bits.ctypes.data))
        L = ctx.lane_len
        T = cfg.context_len
        if step_hook is None and (param_probe is None or not probe_every):
            for i0 in range(0, L, chunk):
                _lib.check(lib.edpc_decompress_steps(ctx.h, i0, min(L, i0 + chunk)))
        else:
            _lib.check(lib.edpc_decompress_steps(ctx.h, 0, min(T, L)))
            for i in range(T, L):
                _lib.check(lib.edpc_decompress_steps(ctx.h, i, i + 1))
                if step_hook is not None:
                    out = np.empty(cfg.lanes * L, dtype=np.uint8)
                    _lib.check(lib.edpc_get_output(ctx.h, out.ctypes.data, out.size))
                    step_hook(i, ctx.last_probs().astype(np.float64),
                              out.reshape(cfg.lanes, L)[:, i].copy())
                if probe_every and param_probe is not None and (i - T + 1) % probe_every == 0:
                    param_probe(i, ctx)
        out = np.empty(n, dtype=np.uint8)
        st = lib.edpc_get_output(ctx.h, out.ctypes.data, n)
        if st == _lib.ERR_CODER:
            raise CoderError(lib.edpc_last_error().decode())
        _lib.check(st)
    finally:
        ctx.close()
    _stats(stats, steps=max(0, L - T), wall_s=time.perf_counter() - t0)
    return out.tobytes()
