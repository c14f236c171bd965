"""ctypes wrapper around the C oracle coder (test infrastructure only).

API mirrors the reference coder (`pkg/src/edpc/coder.py:83-353`):
``quantize_rows``, ``ArithmeticEncoder`` (``encode_rows``, ``finish``),
``ArithmeticDecoder`` (``decode_rows``) and ``uniform_cums``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libedpc_oracle.so")
TOTAL = 1 << 16

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_lib = None


class OracleCoderError(Exception):
    pass


def build() -> str:
    subprocess.run(["bash", os.path.join(_HERE, "build.sh")], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        L.oracle_quantize.argtypes = [_f64p, i64, _i64p, _u64p]
        L.oracle_encode.argtypes = [_i64p, _u8p, _u64p, _i64p, i64]
        L.oracle_finish.argtypes = [_i64p, _u8p]
        L.oracle_finish.restype = i64
        L.oracle_decoder_init.argtypes = [_i64p, _u8p, i64]
        L.oracle_decode.argtypes = [_i64p, _u8p, i64, _u64p, _i64p, i64]
        L.oracle_decode.restype = i64
        L.oracle_adam.argtypes = [_f64p, _f64p, _f64p, _f64p, i64, i64, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.oracle_gelu_fwd.argtypes = [_f64p, _f64p, _f64p, i64]
        L.oracle_gelu_bwd.argtypes = [_f64p, _f64p, _f64p, _f64p, i64]
        _lib = L
    return _lib


def quantize_rows(probs: np.ndarray):
    """(freqs int64 (n,256), cums uint64 (n,257)); restates coder.py:83-106."""
    p = np.ascontiguousarray(probs, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 256:
        raise ValueError(f"expected (n, 256) probabilities, got {p.shape}")
    n = p.shape[0]
    freqs = np.empty((n, 256), dtype=np.int64)
    cums = np.empty((n, 257), dtype=np.uint64)
    if n:
        lib().oracle_quantize(p, n, freqs, cums)
    return freqs, cums


def uniform_cums(rows: int) -> np.ndarray:
    """The bootstrap table (`coder.py:118-123`) tiled over ``rows``."""
    c = (np.arange(257, dtype=np.uint64) * 256)
    return np.ascontiguousarray(np.broadcast_to(c, (rows, 257)))


class ArithmeticEncoder:
    def __init__(self):
        self._state = np.array([0, (1 << 32) - 1, 0, 0], dtype=np.int64)
        self._buf = np.zeros(4096, dtype=np.uint8)
        self._done = False

    def _grow(self, extra_bits: int) -> None:
        need = int(self._state[3]) + extra_bits
        if need > self._buf.size * 8:
            nb = max(self._buf.size * 2, (need + 7) // 8 + 4096)
            g = np.zeros(nb, dtype=np.uint8)
            g[: self._buf.size] = self._buf
            self._buf = g

    def encode_rows(self, cums: np.ndarray, symbols: np.ndarray) -> None:
        if self._done:
            raise OracleCoderError("encoder already finished")
        sym = np.ascontiguousarray(symbols, dtype=np.int64)
        c = np.ascontiguousarray(cums, dtype=np.uint64)
        self._grow(18 * sym.size + int(self._state[2]) + 64)
        if sym.size:
            lib().oracle_encode(self._state, self._buf, c, sym, sym.size)

    def finish(self) -> tuple[bytes, int]:
        if self._done:
            raise OracleCoderError("encoder already finished")
        self._done = True
        self._grow(int(self._state[2]) + 8)
        bits = int(lib().oracle_finish(self._state, self._buf))
        return self._buf[: (bits + 7) // 8].tobytes(), bits


class ArithmeticDecoder:
    def __init__(self, data: bytes, bit_length: int):
        if bit_length > len(data) * 8:
            raise OracleCoderError(f"bit length {bit_length} exceeds payload")
        self._data = np.frombuffer(data, dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
        self._bits = bit_length
        self._state = np.zeros(4, dtype=np.int64)
        lib().oracle_decoder_init(self._state, self._data, bit_length)

    def decode_rows(self, cums: np.ndarray, out: np.ndarray) -> None:
        c = np.ascontiguousarray(cums, dtype=np.uint64)
        n = c.shape[0]
        tmp = np.empty(n, dtype=np.int64)
        done = lib().oracle_decode(self._state, self._data, self._bits, c, tmp, n)
        out[:done] = tmp[:done]
        if done != n:
            raise OracleCoderError(f"bitstream exhausted at symbol {done} of this batch")
