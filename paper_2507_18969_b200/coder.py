"""Quantizer and arithmetic coder API, computed on the GPU.

Same surface as the reference coder (`pkg/src/edpc/coder.py:35-353`):
``quantize_rows``, ``quantize``, ``QuantizedDistribution``,
``uniform_distribution``, ``ArithmeticEncoder`` and ``ArithmeticDecoder``,
with the same validation and error types.  Every computation runs in the
sm_100a kernels behind the C ABI (``edpc_quantize_rows``,
``edpc_encode_rows``/``edpc_encode_finish``, ``edpc_decoder_init``/
``edpc_decode_rows``); the Python objects only hold the coder registers
between calls, exactly like the reference's ``_reg``/``_bitpos`` arrays.
These are the parity entry points; the compress/decompress hot path keeps
all coder state on the device (see pipeline.py).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

TOTAL_BITS = 16
TOTAL = 1 << TOTAL_BITS
STATE_BITS = 32
_MASK = (1 << STATE_BITS) - 1


class CoderError(Exception):
    pass


class QuantizedDistribution:
    """256 integer frequencies summing to TOTAL, with a cumulative table."""

    __slots__ = ("freqs", "cumulative")

    def __init__(self, freqs: np.ndarray):
        freqs = np.asarray(freqs, dtype=np.uint32)
        if freqs.shape != (256,):
            raise ValueError("need exactly 256 frequencies")
        if freqs.min() < 1:
            raise ValueError("every symbol needs frequency >= 1")
        cum = np.zeros(257, dtype=np.uint64)
        np.cumsum(freqs, out=cum[1:])
        if int(cum[-1]) != TOTAL:
            raise ValueError(f"frequencies sum to {int(cum[-1])}, expected {TOTAL}")
        self.freqs = freqs
        self.cumulative = cum


def _validate_probs(probs: np.ndarray) -> None:
    if probs.ndim != 2 or probs.shape[1] != 256:
        raise ValueError(f"expected (n, 256) probabilities, got {probs.shape}")
    if not np.isfinite(probs).all():
        raise ValueError("probability contains NaN or Inf")
    if probs.size and probs.min() < 0.0:
        raise ValueError("negative probability")
    if probs.shape[0]:
        sums = probs.astype(np.float64).sum(axis=1)
        if np.abs(sums - 1.0).max() > 1e-6:
            raise ValueError("probability row does not sum to 1")


def quantize_cums(probs: np.ndarray, device: int = 0) -> np.ndarray:
    """Device quantizer -> cumulative tables uint32 (n, 257).  float32 rows
    take the fp32 fast path (the one the predictor uses); float64 rows the
    general one."""
    p = np.asarray(probs)
    dtype = 0 if p.dtype == np.float32 else 1
    p = np.ascontiguousarray(p, dtype=np.float32 if dtype == 0 else np.float64)
    _validate_probs(p)
    n = p.shape[0]
    cums = np.empty((n, 257), dtype=np.uint32)
    if n:
        _lib.check(_lib.load().edpc_quantize_rows(device, p.ctypes.data, n, dtype, cums.ctypes.data))
    return cums


def quantize_rows(probs: np.ndarray, device: int = 0):
    """(freqs int64 (n,256), cumulative uint64 (n,257)); `coder.py:83-106`."""
    cums = quantize_cums(probs, device)
    freqs = np.diff(cums.astype(np.int64), axis=1)
    return freqs, cums.astype(np.uint64)


def quantize(prob_row: np.ndarray, device: int = 0) -> QuantizedDistribution:
    freqs, _ = quantize_rows(np.asarray(prob_row).reshape(1, 256), device)
    return QuantizedDistribution(freqs[0])


_UNIFORM = None


def uniform_distribution() -> QuantizedDistribution:
    """The bootstrap table: every byte at frequency TOTAL/256 (`coder.py:118-123`)."""
    global _UNIFORM
    if _UNIFORM is None:
        _UNIFORM = QuantizedDistribution(np.full(256, TOTAL // 256, dtype=np.uint32))
    return _UNIFORM


def _as_cums32(cums: np.ndarray) -> np.ndarray:
    c = np.asarray(cums)
    if c.ndim != 2 or c.shape[1] != 257:
        raise ValueError(f"expected (n, 257) cumulative rows, got {c.shape}")
    return np.ascontiguousarray(c, dtype=np.uint32)


class ArithmeticEncoder:
    """Streaming encoder on the GPU; `coder.py:241-306`."""

    def __init__(self, device: int = 0):
        self._device = device
        self._state = np.array([0, _MASK, 0, 0], dtype=np.int64)
        self._buf = np.zeros(4096, dtype=np.uint8)
        self._finished = False

    @property
    def pending_bits(self) -> int:
        return int(self._state[2])

    def _ensure_capacity(self, extra_bits: int) -> None:
        need = int(self._state[3]) + extra_bits
        if need > self._buf.size * 8:
            grown = np.zeros(max(self._buf.size * 2, (need + 7) // 8 + 4096), dtype=np.uint8)
            grown[: self._buf.size] = self._buf
            self._buf = grown

    def encode_rows(self, cums: np.ndarray, symbols: np.ndarray) -> None:
        if self._finished:
            raise CoderError("encoder already finished")
        c = _as_cums32(cums)
        s = np.ascontiguousarray(symbols, dtype=np.int32)
        if s.shape != (c.shape[0],):
            raise ValueError("one symbol per cumulative row")
        self._ensure_capacity(18 * s.size + self.pending_bits + 64)
        if s.size:
            _lib.check(_lib.load().edpc_encode_rows(
                self._device, self._state.ctypes.data, self._buf.ctypes.data, self._buf.size,
                c.ctypes.data, s.ctypes.data, s.size))

    def encode_prob_rows(self, probs: np.ndarray, symbols: np.ndarray) -> None:
        self.encode_rows(quantize_cums(probs, self._device), symbols)

    def encode_symbol(self, dist: QuantizedDistribution, symbol: int) -> None:
        self.encode_rows(dist.cumulative.reshape(1, 257), np.array([symbol]))

    def finish(self) -> tuple[bytes, int]:
        if self._finished:
            raise CoderError("encoder already finished")
        self._finished = True
        self._ensure_capacity(self.pending_bits + 8)
        bits = ctypes.c_int64(0)
        _lib.check(_lib.load().edpc_encode_finish(self._device, self._state.ctypes.data,
                                                  self._buf.ctypes.data, self._buf.size,
                                                  ctypes.addressof(bits)))
        nbytes = (bits.value + 7) // 8
        return self._buf[:nbytes].tobytes(), bits.value


class ArithmeticDecoder:
    """Mirror of ArithmeticEncoder (`coder.py:309-353`); zeros past bit_length,
    CoderError when the stream cannot supply the requested symbols."""

    def __init__(self, data: bytes, bit_length: int, device: int = 0):
        if bit_length > len(data) * 8:
            raise CoderError(f"bit length {bit_length} exceeds payload of {len(data)} bytes")
        self._device = device
        self._data = np.frombuffer(bytes(data), dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
        self._nbytes = len(data)
        self._bit_length = bit_length
        self._state = np.zeros(4, dtype=np.int64)
        _lib.check(_lib.load().edpc_decoder_init(device, self._state.ctypes.data,
                                                 self._data.ctypes.data, self._nbytes, bit_length))

    def decode_rows(self, cums: np.ndarray, out: np.ndarray) -> None:
        c = _as_cums32(cums)
        n = c.shape[0]
        res = np.empty(n, dtype=np.int32)
        done = ctypes.c_int64(0)
        st = _lib.load().edpc_decode_rows(self._device, self._state.ctypes.data,
                                          self._data.ctypes.data, self._nbytes, self._bit_length,
                                          c.ctypes.data, n, res.ctypes.data, ctypes.addressof(done))
        out[: done.value] = res[: done.value]
        if st == _lib.ERR_CODER:
            raise CoderError(f"bitstream exhausted at symbol {done.value} of this batch")
        _lib.check(st)

    def decode_prob_rows(self, probs: np.ndarray, out: np.ndarray) -> None:
        self.decode_rows(quantize_cums(probs, self._device), out)

    def decode_symbol(self, dist: QuantizedDistribution) -> int:
        out = np.empty(1, dtype=np.int64)
        self.decode_rows(dist.cumulative.reshape(1, 257), out)
        return int(out[0])
