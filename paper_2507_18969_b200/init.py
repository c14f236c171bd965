"""Deterministic parameter init in the reference's RNG draw order.

`EdpcModel.__init__` (`pkg/src/edpc/model.py:187-199`) draws every weight from
one ``Generator(PCG64(seed))`` (`nn.py:142-144`) as ``uniform(-1/sqrt(fan_in),
+1/sqrt(fan_in))`` (`nn.py:147-150`) in construction order: embedding, local
branch weights then out_w, lte down_w, lane_mats, up_w, global branch weights
then out_w, head_w.  Biases are zeros and LN gains ones; they draw nothing.

We reproduce those float64 draws bit for bit with numpy's PCG64 and hand the
device an fp32 copy in the flat ``parameters()`` order; the device computes in
fp32/tf32 from there on.
"""

from __future__ import annotations

import dataclasses
import functools
import math

import numpy as np

from .config import ModelConfig, VOCAB, param_offsets


def init_params_f64(cfg: ModelConfig) -> np.ndarray:
    """Flat float64 parameters in ``parameters()`` order, as the reference inits them."""
    cfg.validate()
    offs = param_offsets(cfg)
    total = sum(int(np.prod(s)) for _, s in offs.values())
    flat = np.zeros(total, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    f, fp = cfg.feature_dim, cfg.latent_dim

    def draw(name: str, fan_in: int) -> None:
        off, shape = offs[name]
        bound = 1.0 / math.sqrt(fan_in)
        vals = rng.uniform(-bound, bound, size=shape)
        flat[off: off + vals.size] = vals.reshape(-1)

    def ones(name: str) -> None:
        off, shape = offs[name]
        flat[off: off + int(np.prod(shape))] = 1.0

    draw("embedding", cfg.embed_dim)
    for blk, h in (("local", cfg.hidden_local),):
        ones(f"{blk}.ln_gain")
        for i in range(cfg.branches):
            draw(f"{blk}.branch{i}_w", f)
        draw(f"{blk}.out_w", h)
    draw("lte.down_w", f)
    draw("lte.lane_mats", fp)
    draw("lte.up_w", fp)
    ones("global.ln_gain")
    for i in range(cfg.branches):
        draw(f"global.branch{i}_w", f)
    draw("global.out_w", cfg.hidden_global)
    draw("head_w", f)
    assert VOCAB == 256
    return flat


@functools.lru_cache(maxsize=4)
def _init_f32_cached(key) -> np.ndarray:
    cfg = ModelConfig(**dict(key))
    a = init_params_f64(cfg).astype(np.float32)
    a.flags.writeable = False  # shared between calls
    return a


def init_params_f32(cfg: ModelConfig) -> np.ndarray:
    """fp32 init (read-only, cached per config: compress and decompress of
    the same container draw the identical 21.6M-parameter PCG64 stream)."""
    return _init_f32_cached(tuple(sorted(dataclasses.asdict(cfg).items())))
