"""Seeded synthetic byte streams for the benchmark configs.

There is no network for corpora, so every benchmark input is generated from a
``numpy.random.Generator(PCG64(seed))`` and identified by its sha256:

* ``text_like``  -- phrase-level Zipf text over a fixed pseudo-English
  vocabulary, with punctuation and newlines (order-0 entropy ~4.3-4.6 bpb,
  like prose);
* ``image_like`` -- smooth 2-D fields (low-frequency sinusoids + Gaussian
  noise) quantised to uint8 and emitted as raster tiles (gray and RGB);
* ``mixed``      -- alternating 1 MiB blocks of the two.

All generators are vectorised so 1 GiB streams take seconds, not minutes.
"""

from __future__ import annotations

import hashlib

import numpy as np

_CONS = np.frombuffer(b"tnshrdlcmwfgypbvkjxqz", dtype=np.uint8)
_CONS_P = np.array([9.1, 6.7, 6.3, 6.1, 6.0, 4.3, 4.0, 2.8, 2.4, 2.4, 2.2, 2.0, 2.0,
                    1.9, 1.5, 1.0, 0.8, 0.15, 0.15, 0.1, 0.07])
_VOWS = np.frombuffer(b"eaoiu", dtype=np.uint8)
_VOWS_P = np.array([12.7, 8.2, 7.5, 7.0, 2.8])


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _vocabulary(rng: np.random.Generator, n_words: int) -> list[bytes]:
    cons_p = _CONS_P / _CONS_P.sum()
    vow_p = _VOWS_P / _VOWS_P.sum()
    words = []
    for i in range(n_words):
        syll = 1 + min(int(rng.geometric(0.45)), 5)
        out = bytearray()
        for _ in range(syll):
            if rng.random() < 0.8:
                out.append(int(rng.choice(_CONS, p=cons_p)))
            out.append(int(rng.choice(_VOWS, p=vow_p)))
            if rng.random() < 0.35:
                out.append(int(rng.choice(_CONS, p=cons_p)))
        words.append(bytes(out))
    return words


def _zipf_indices(rng: np.random.Generator, n: int, size: int, s: float = 1.1) -> np.ndarray:
    ranks = np.arange(1, size + 1, dtype=np.float64)
    p = ranks ** (-s)
    cdf = np.cumsum(p / p.sum())
    return np.minimum(np.searchsorted(cdf, rng.random(n)), size - 1)


def _gather_tokens(tok_bytes: list[bytes], seq: np.ndarray) -> np.ndarray:
    lens = np.array([len(t) for t in tok_bytes], dtype=np.int64)
    blob = np.frombuffer(b"".join(tok_bytes), dtype=np.uint8)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    pl = lens[seq]
    ends = np.cumsum(pl)
    pos = np.arange(int(ends[-1]), dtype=np.int64)
    owner = np.searchsorted(ends, pos, side="right")
    return blob[starts[seq][owner] + (pos - (ends[owner] - pl[owner]))]


def text_like(n: int, seed: int = 0) -> bytes:
    """Pseudo-English prose from a word-level order-1 Markov chain.

    Tokens are words (with a trailing space, some capitalised) and
    punctuation.  Each token owns a Zipf-ranked table of 16 successors; a step
    follows that table with probability 0.55 and otherwise draws from the
    global Zipf marginal.  4096 independent chains advance in lock step so the
    generator is vectorised; their outputs are concatenated.
    """
    if n <= 0:
        return b""
    rng = _rng(seed)
    words = _vocabulary(rng, 4000)
    toks = [w + b" " for w in words]
    toks += [w[:1].upper() + w[1:] + b" " for w in words[:600]]
    punct = [b", ", b". ", b".\n", b"; ", b"? ", b"\n\n", b": ", b"(", b") ", b"\"", b"-"]
    toks += punct
    V = len(toks)
    succ = _zipf_indices(rng, V * 16, V, 1.0).reshape(V, 16)
    mean_len = float(np.mean([len(t) for t in toks[:2000]])) * 0.8
    chains = 4096
    steps = int(n / mean_len / chains) + 8
    seq = np.empty((steps, chains), dtype=np.int64)
    seq[0] = _zipf_indices(rng, chains, V, 1.0)
    for i in range(1, steps):
        follow = rng.random(chains) < 0.55
        pick = _zipf_indices(rng, chains, 16, 1.2)
        glob = _zipf_indices(rng, chains, V, 1.0)
        seq[i] = np.where(follow, succ[seq[i - 1], pick], glob)
    out = _gather_tokens(toks, seq.T.reshape(-1))
    while out.size < n:  # extremely unlikely: top up with another pass
        out = np.concatenate([out, np.frombuffer(text_like(n - out.size, seed + 7919), np.uint8)])
    return out[:n].tobytes()


def image_like(n: int, seed: int = 0, tile: int = 512) -> bytes:
    """Raster tiles of smooth 2-D fields plus noise, gray and RGB alternating."""
    if n <= 0:
        return b""
    rng = _rng(seed)
    out = []
    total = 0
    yy, xx = np.mgrid[0:tile, 0:tile].astype(np.float32) / tile
    t = 0
    while total < n:
        chans = 1 if t % 2 == 0 else 3
        planes = []
        for _ in range(chans):
            f = np.zeros((tile, tile), dtype=np.float32)
            for _ in range(4):
                fx, fy = rng.uniform(0.5, 6.0, size=2)
                ph = rng.uniform(0, 2 * np.pi)
                amp = rng.uniform(10, 50)
                f += amp * np.sin(2 * np.pi * (fx * xx + fy * yy) + ph).astype(np.float32)
            f += 128.0 + rng.normal(0.0, 3.0, size=(tile, tile)).astype(np.float32)
            planes.append(np.clip(np.rint(f), 0, 255).astype(np.uint8))
        img = planes[0] if chans == 1 else np.stack(planes, axis=-1)
        out.append(img.reshape(-1))
        total += img.size
        t += 1
    return np.concatenate(out)[:n].tobytes()


def mixed(n: int, seed: int = 0, block: int = 1 << 20) -> bytes:
    """Alternating ``block``-byte text and image blocks."""
    if n <= 0:
        return b""
    nb = -(-n // block)
    n_text = -(-nb // 2) * block
    n_img = (nb // 2) * block
    text = text_like(n_text, seed)
    img = image_like(max(n_img, 1), seed + 1)
    parts = []
    for b in range(nb):
        src, k = (text, b // 2) if b % 2 == 0 else (img, b // 2)
        parts.append(src[k * block: (k + 1) * block])
    return b"".join(parts)[:n]


GENERATORS = {"text": text_like, "image": image_like, "mixed": mixed}


def generate(kind: str, n: int, seed: int = 0) -> bytes:
    return GENERATORS[kind](n, seed)


def sha256(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()


def order0_bpb(data: bytes) -> float:
    if not data:
        return 0.0
    c = np.bincount(np.frombuffer(data, dtype=np.uint8), minlength=256).astype(np.float64)
    p = c[c > 0] / len(data)
    return float(-(p * np.log2(p)).sum())
