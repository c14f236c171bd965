"""Chunked multi-container framing.

The reference format holds one container per stream (`container.py:3-28`):
one model, one set of lanes, L = ceil(n / B) serial steps.  An *archive*
splits a stream into fixed-size chunks and stores one independent container
per chunk (each with its own model, trained from the same seed), so that

* very large inputs are bounded in per-container state and can be produced
  and consumed chunk by chunk (resumable: a damaged chunk does not take the
  others with it);
* chunks compress in parallel on several GPUs with no communication at all
  ("replicas" mode, SURVEY.md §8e last row) -- the bytes of each chunk depend
  only on (chunk data, cfg, S), never on which or how many GPUs ran it.

Layout (little-endian)::

    magic "EDPA" | u8 version (1) | u32 chunk count C | u64 chunk_bytes |
    u64 total length | C x u64 container lengths | u32 CRC32 of the above |
    C containers (the EDPC byte format of container.py), back to back

Every chunk but the last holds exactly ``chunk_bytes`` input bytes.
"""

from __future__ import annotations

import struct
import threading
import time
import zlib
from dataclasses import dataclass

from .config import ModelConfig
from .container import (BadMagicError, BadVersionError, ChecksumError, ContainerError,
                        InvalidHeaderError, TruncatedError, read_container, write_container)

ARCHIVE_MAGIC = b"EDPA"
ARCHIVE_VERSION = 1
_FIXED = struct.Struct("<4sBIQQ")  # magic, version, chunk count, chunk_bytes, total length
_MAX_CHUNKS = 1 << 24


@dataclass
class ArchiveHeader:
    chunk_bytes: int
    total_len: int
    container_lengths: list[int]

    @property
    def chunk_count(self) -> int:
        return len(self.container_lengths)

    def chunk_span(self, k: int) -> tuple[int, int]:
        """[start, end) of chunk k in the original stream."""
        a = k * self.chunk_bytes
        return a, min(self.total_len, a + self.chunk_bytes)


def archive_header_size(chunks: int) -> int:
    return _FIXED.size + 8 * chunks + 4


def write_archive(chunk_bytes: int, total_len: int, containers: list[bytes]) -> bytes:
    if chunk_bytes < 1:
        raise InvalidHeaderError("chunk_bytes must be >= 1")
    expect = -(-total_len // chunk_bytes) if total_len else 0
    if len(containers) != expect:
        raise InvalidHeaderError(f"{len(containers)} containers for {expect} chunks")
    head = bytearray(_FIXED.pack(ARCHIVE_MAGIC, ARCHIVE_VERSION, len(containers), chunk_bytes,
                                 total_len))
    head += struct.pack(f"<{len(containers)}Q", *[len(c) for c in containers])
    head += struct.pack("<I", zlib.crc32(head))
    return bytes(head) + b"".join(containers)


def is_archive(buf: bytes) -> bool:
    return bytes(buf[:4]) == ARCHIVE_MAGIC


def read_archive(buf: bytes) -> tuple[ArchiveHeader, list[bytes]]:
    """Parses and validates the index (bounds-checked before any sizing from
    untrusted fields); returns the header and the raw container blobs."""
    buf = bytes(buf)
    if len(buf) < 5:
        raise TruncatedError("shorter than magic + version")
    if buf[:4] != ARCHIVE_MAGIC:
        raise BadMagicError("bad archive magic")
    if buf[4] != ARCHIVE_VERSION:
        raise BadVersionError(f"unsupported archive version {buf[4]}")
    if len(buf) < _FIXED.size:
        raise TruncatedError("truncated archive header")
    _, _, count, chunk_bytes, total = _FIXED.unpack_from(buf, 0)
    if count > _MAX_CHUNKS:
        raise InvalidHeaderError(f"implausible chunk count {count}")
    hs = archive_header_size(count)
    if len(buf) < hs:
        raise TruncatedError("truncated archive index")
    lens = list(struct.unpack_from(f"<{count}Q", buf, _FIXED.size))
    (crc,) = struct.unpack_from("<I", buf, hs - 4)
    if crc != zlib.crc32(buf[: hs - 4]):
        raise ChecksumError("archive index checksum mismatch")
    if chunk_bytes < 1 or count != (-(-total // chunk_bytes) if total else 0):
        raise InvalidHeaderError("chunk count does not match total length / chunk_bytes")
    out, pos = [], hs
    for k, n in enumerate(lens):
        if pos + n > len(buf):
            raise TruncatedError(f"chunk {k}: container truncated")
        out.append(buf[pos: pos + n])
        pos += n
    if pos != len(buf):
        raise InvalidHeaderError("trailing bytes after the last container")
    return ArchiveHeader(chunk_bytes, total, lens), out


def _run_parallel(jobs: list, devices: list[int], fn) -> list:
    """fn(job, device) for every job; job k goes to devices[k % G], one host
    thread per device (each thread drives its own contexts; the C ABI
    releases the GIL, so the devices run concurrently)."""
    results: list = [None] * len(jobs)
    errors: list = []

    def worker(w: int):
        try:
            for k in range(w, len(jobs), len(devices)):
                results[k] = fn(jobs[k], devices[w])
        except BaseException as exc:  # re-raised on the calling thread
            errors.append(exc)

    if len(devices) == 1:
        worker(0)
    else:
        ts = [threading.Thread(target=worker, args=(w,)) for w in range(len(devices))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    if errors:
        raise errors[0]
    return results


def compress_chunked(data: bytes, cfg: ModelConfig, segments: int = 4, *, chunk_bytes: int,
                     devices=None, stats: dict | None = None) -> bytes:
    """Archive of one container per ``chunk_bytes`` of ``data``; chunks are
    spread over ``devices`` (replicas: no communication, bytes independent of
    the device count)."""
    from .pipeline import compress
    if chunk_bytes < 1:
        raise ValueError("chunk_bytes must be >= 1")
    devs = [0] if devices is None else [int(d) for d in devices]
    if not devs:
        raise ValueError("devices must not be empty")
    t0 = time.perf_counter()
    n = len(data)
    spans = [(a, min(n, a + chunk_bytes)) for a in range(0, n, chunk_bytes)]
    mv = memoryview(bytes(data))
    blobs = _run_parallel(spans, devs, lambda sp, d: write_container(
        compress(mv[sp[0]:sp[1]].tobytes(), cfg, segments, device=d)))
    out = write_archive(chunk_bytes, n, blobs)
    if stats is not None:
        stats.update(chunks=len(spans), devices=devs, wall_s=time.perf_counter() - t0)
    return out


def decompress_chunked(blob: bytes, *, devices=None, stats: dict | None = None) -> bytes:
    from .pipeline import decompress
    devs = [0] if devices is None else [int(d) for d in devices]
    if not devs:
        raise ValueError("devices must not be empty")
    t0 = time.perf_counter()
    head, blobs = read_archive(blob)
    parts = _run_parallel(list(range(head.chunk_count)), devs,
                          lambda k, d: decompress(read_container(blobs[k]), device=d))
    for k, p in enumerate(parts):
        a, b = head.chunk_span(k)
        if len(p) != b - a:
            raise ContainerError(f"chunk {k}: {len(p)} bytes decoded, {b - a} expected")
    if stats is not None:
        stats.update(chunks=head.chunk_count, devices=devs, wall_s=time.perf_counter() - t0)
    return b"".join(parts)
