"""Lane split/join and the segment plan (the DPCA segment scheduler's geometry).

Restates `pkg/src/edpc/pipeline.py:36-76`: the stream is cut into ``lanes``
contiguous rows of ``ceil(n/lanes)`` bytes (zero padded), and segment ``s``
owns lanes ``[s*B/S, (s+1)*B/S)``.  On the device the same (B, L) matrix is
the M dimension of every per-step GEMM; see DESIGN.md "Data layout".
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import ModelConfig


@dataclass
class LaneSplit:
    lane_count: int
    lane_len: int
    original_len: int
    pad_value: int = 0


def lane_len_for(n: int, lanes: int) -> int:
    return -(-n // lanes) if n else 0


def split_lanes(data: bytes, lanes: int):
    """(LaneSplit, uint8[lanes, lane_len]) with zero padding (`pipeline.py:44-56`)."""
    if lanes < 1:
        raise ValueError("lane count must be >= 1")
    n = len(data)
    L = lane_len_for(n, lanes)
    mat = np.zeros((lanes, L), dtype=np.uint8)
    if n:
        mat.reshape(-1)[:n] = np.frombuffer(data, dtype=np.uint8)
    return LaneSplit(lane_count=lanes, lane_len=L, original_len=n), mat


def join_lanes(split: LaneSplit, mat: np.ndarray) -> bytes:
    """Inverse of split_lanes, dropping the padding (`pipeline.py:59-63`)."""
    if mat.shape != (split.lane_count, split.lane_len):
        raise ValueError("lane matrix shape mismatch")
    return np.ascontiguousarray(mat).reshape(-1)[: split.original_len].tobytes()


def segment_spans(lanes: int, segments: int) -> list[tuple[int, int]]:
    chunk = lanes // segments
    return [(s * chunk, (s + 1) * chunk) for s in range(segments)]


def validate_geometry(cfg: ModelConfig, segments: int) -> None:
    """`pipeline.py:71-76`: config validity and S | B, raised as ValueError."""
    cfg.validate()
    if segments < 1:
        raise ValueError("segment count must be >= 1")
    if cfg.lanes % segments != 0:
        raise ValueError(f"segments ({segments}) must divide lanes ({cfg.lanes})")
