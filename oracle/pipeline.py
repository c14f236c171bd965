"""Serial CPU compress/decompress over the oracle model + C coder (oracle only).

Restates `pkg/src/edpc/pipeline.py:109-298` in its serial form (the
reference's bytes are schedule-invariant, `pipeline.py:117-118`): lane split
(`:44-56`), segment spans (`:66-68`), uniform bootstrap of the first
min(t, L) columns (`:84-102`), then per step predict -> quantize+code per
segment -> train.  Returns / consumes (payloads, bit_lengths) so tests can
compare against either the reference's or the B200 container.
"""

from __future__ import annotations

import numpy as np

from . import coder as oc
from .model import OracleModel


def _spans(lanes, segments):
    c = lanes // segments
    return [(s * c, (s + 1) * c) for s in range(segments)]


def _split(data: bytes, lanes: int):
    n = len(data)
    L = -(-n // lanes) if n else 0
    mat = np.zeros((lanes, L), dtype=np.uint8)
    if n:
        mat.reshape(-1)[:n] = np.frombuffer(data, dtype=np.uint8)
    return L, mat


def compress(data: bytes, cfg, segments: int, *, step_hook=None, max_steps=None,
             model: OracleModel | None = None):
    """-> (payloads list[bytes], bit_lengths list[int]).  ``max_steps`` truncates
    the model loop (used only for step-sampled CPU timing; output then invalid)."""
    n = len(data)
    if n == 0:
        return [], []
    L, mat = _split(data, cfg.lanes)
    t = cfg.context_len
    spans = _spans(cfg.lanes, segments)
    encs = [oc.ArithmeticEncoder() for _ in spans]
    model = model or OracleModel(cfg)
    uni = oc.uniform_cums(spans[0][1] - spans[0][0])
    for (lo, hi), e in zip(spans, encs):
        for i in range(min(t, L)):
            e.encode_rows(uni, mat[lo:hi, i])
    end = L if max_steps is None else min(L, t + max_steps)
    for i in range(t, end):
        probs, cache = model.predict(mat[:, i - t: i])
        tg = mat[:, i]
        if step_hook is not None:
            step_hook(i, probs, tg)
        _, cums = oc.quantize_rows(probs)
        for (lo, hi), e in zip(spans, encs):
            e.encode_rows(cums[lo:hi], tg[lo:hi])
        model.train_step(cache, tg)
    outs = [e.finish() for e in encs]
    return [p for p, _ in outs], [b for _, b in outs]


def decompress(payloads, bit_lengths, cfg, n: int) -> bytes:
    if n == 0:
        return b""
    segments = len(payloads)
    L = -(-n // cfg.lanes)
    mat = np.zeros((cfg.lanes, L), dtype=np.uint8)
    t = cfg.context_len
    spans = _spans(cfg.lanes, segments)
    decs = [oc.ArithmeticDecoder(p, b) for p, b in zip(payloads, bit_lengths)]
    model = OracleModel(cfg)
    chunk = spans[0][1] - spans[0][0]
    uni = oc.uniform_cums(chunk)
    out = np.empty(chunk, dtype=np.int64)
    for (lo, hi), d in zip(spans, decs):
        for i in range(min(t, L)):
            d.decode_rows(uni, out)
            mat[lo:hi, i] = out
    for i in range(t, L):
        probs, cache = model.predict(mat[:, i - t: i])
        _, cums = oc.quantize_rows(probs)
        for (lo, hi), d in zip(spans, decs):
            d.decode_rows(cums[lo:hi], out)
            mat[lo:hi, i] = out
        model.train_step(cache, mat[:, i])
    return mat.reshape(-1)[:n].tobytes()
