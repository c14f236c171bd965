"""Regenerates tests/golden/*.npz from the UNMODIFIED reference (dev container only).

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src:. python oracle/make_goldens.py

The reference ships no golden vectors, so these are produced
by calling the reference's own public functions on seeded inputs:

* quantize.npz  -- ``edpc.coder.quantize_rows`` on fp32-representable rows of
  several families (uniform, one-hot, Dirichlet, peaked, tiny-mass tails)
  plus a block of genuine float64 Dirichlet rows;
* coder.npz     -- ``ArithmeticEncoder.encode_rows`` + ``finish`` payloads and
  bit lengths for seeded (CDF, symbol) streams, including the reference
  test-suite's adversarial cases (certain symbol, empty message);
* model.npz     -- init parameters for several configs/seeds, the per-step
  probabilities of the first steps of a tiny-config compress (``step_hook``)
  and the lockstep checksums (``param_probe``);
* pipeline.npz  -- whole v1 containers written by ``edpc.compress`` for the
  reference test-suite's tiny configuration on assorted inputs;
* adam.npz      -- the fused Adam kernel's trajectory on a random buffer;
* ifr.npz       -- ``edpc.ifr.ksg_mi`` estimates on seeded sample matrices
  (correlated, scalar, duplicate-heavy and degenerate cases) and
  ``edpc.ifr.digamma`` values.

Files are small (< 1 MB total) and committed; their sha256s are in
tests/golden/MANIFEST.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

import edpc  # noqa: E402
from edpc import _kernels  # noqa: E402
from edpc.coder import ArithmeticEncoder, quantize_rows  # noqa: E402
from edpc.container import write_container  # noqa: E402
from edpc.model import EdpcModel, ModelConfig  # noqa: E402

TINY = dict(context_len=8, embed_dim=4, hidden_local=16, hidden_global=32, lte_ratio=4,
            branches=2, lanes=8, seed=5)


def f32_rows(rng, n, kind):
    if kind == "dirichlet":
        alpha = rng.uniform(0.05, 3.0)
        p = rng.dirichlet(np.full(256, alpha), size=n)
    elif kind == "peaked":
        logits = rng.normal(0, 1, size=(n, 256)) * rng.uniform(2, 12, size=(n, 1))
        p = np.exp(logits - logits.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
    elif kind == "tail":  # tiny-mass symbols down to fp32 denormal range
        p = rng.random((n, 256)) ** 20 * 1e-30
        p[:, rng.integers(0, 256, size=n)] = 1.0
        p /= p.sum(1, keepdims=True)
    elif kind == "uniform":
        p = np.full((n, 256), 1.0 / 256)
    elif kind == "onehot":
        p = np.zeros((n, 256))
        p[np.arange(n), rng.integers(0, 256, size=n)] = 1.0
    else:
        raise ValueError(kind)
    p32 = p.astype(np.float32)
    # renormalise in fp32 the way a GPU softmax would, then keep fp32 values
    p32 = (p32 / p32.sum(1, keepdims=True, dtype=np.float32)).astype(np.float32)
    return p32


def gen_quantize(rng):
    rows = [f32_rows(rng, 120, "dirichlet"), f32_rows(rng, 120, "peaked"),
            f32_rows(rng, 24, "tail"), f32_rows(rng, 4, "uniform"), f32_rows(rng, 12, "onehot")]
    p32 = np.concatenate(rows)
    freqs32, _ = quantize_rows(p32.astype(np.float64))
    p64 = rng.dirichlet(np.full(256, 0.4), size=40)
    freqs64, _ = quantize_rows(p64)
    return dict(probs_f32=p32, freqs_f32=freqs32.astype(np.uint16),
                probs_f64=p64, freqs_f64=freqs64.astype(np.uint16))


def gen_coder(rng):
    pool_p = np.concatenate([f32_rows(rng, 48, "dirichlet"), f32_rows(rng, 16, "peaked")])
    pool_f, pool_c = quantize_rows(pool_p.astype(np.float64))
    onehot = np.zeros((1, 256))
    onehot[0, 7] = 1.0
    f1, c1 = quantize_rows(onehot)
    pool_f = np.concatenate([pool_f, f1])
    pool_c = np.concatenate([pool_c, c1])
    streams = []
    lengths = [0, 1, 2, 37, 500, 3000, 3000, 12000]
    for k, n in enumerate(lengths):
        if k == 6:  # certain-symbol stream: mass on 7, min freq elsewhere
            rows = np.full(n, pool_f.shape[0] - 1)
            syms = np.full(n, 7)
            syms[n // 2] = 255
        else:
            rows = rng.integers(0, pool_f.shape[0] - 1, size=n)
            syms = rng.integers(0, 256, size=n)
            # bias half the symbols toward likely ones so pending-bit runs occur
            likely = np.argmax(pool_f[rows], axis=1)
            pick = rng.random(n) < 0.5
            syms = np.where(pick, likely, syms)
        enc = ArithmeticEncoder()
        enc.encode_rows(np.ascontiguousarray(pool_c[rows]), syms.astype(np.int64))
        payload, bits = enc.finish()
        streams.append((rows, syms, payload, bits))
    row_off = np.cumsum([0] + [len(s[0]) for s in streams])
    pay_off = np.cumsum([0] + [len(s[2]) for s in streams])
    return dict(pool_freqs=pool_f.astype(np.uint16),
                rows=np.concatenate([s[0] for s in streams]).astype(np.int32),
                symbols=np.concatenate([s[1] for s in streams]).astype(np.uint8),
                row_off=row_off.astype(np.int64),
                payload=np.frombuffer(b"".join(s[2] for s in streams), dtype=np.uint8),
                pay_off=pay_off.astype(np.int64),
                bits=np.array([s[3] for s in streams], dtype=np.int64))


def gen_model(rng):
    out = {}
    cfgs = [TINY, dict(TINY, seed=0), dict(TINY, seed=1), dict(TINY, seed=42),
            dict(context_len=4, embed_dim=4, hidden_local=8, hidden_global=8, lte_ratio=2,
                 branches=3, lanes=2, seed=7)]
    for i, c in enumerate(cfgs):
        m = EdpcModel(ModelConfig(**c))
        out[f"init_{i}"] = np.concatenate([p.value.reshape(-1) for p in m.parameters()])
        out[f"init_cfg_{i}"] = np.array(json.dumps(c))
    # per-step probs + checksums of a tiny compress
    data = (b"lockstep parameter trajectories must match exactly. " * 30)
    cfg = ModelConfig(**TINY)
    probs_log, tg_log, sums = [], [], []
    edpc.compress(data, cfg, 2, serial=True,
                  step_hook=lambda i, p, t: (probs_log.append(p.copy()), tg_log.append(t.copy())),
                  param_probe=lambda i, m: sums.append(m.state_checksum()), probe_every=25)
    out["step_data"] = np.frombuffer(data, dtype=np.uint8)
    out["step_probs"] = np.stack(probs_log[:16])
    out["step_targets"] = np.stack(tg_log[:16])
    out["step_checksums"] = np.array(sums)
    return out


def gen_pipeline(rng):
    cases = [
        ("text4", b"the quick brown fox jumps over the lazy dog. " * 70, TINY, 4),
        ("zeros1", b"\x00" * 3000, TINY, 1),
        ("ramp2", bytes(range(256)) * 12, TINY, 2),
        ("rand8", rng.integers(0, 256, size=2000, dtype=np.uint8).tobytes(), TINY, 8),
        ("short", b"abcdef", TINY, 4),
        ("one", b"\x7f", TINY, 4),
        ("empty", b"", TINY, 4),
        ("l16", b"schedule invariance probe " * 120, dict(TINY, lanes=16), 8),
        ("k1", b"single branch block " * 90, dict(TINY, branches=1, seed=9), 2),
        ("k3", b"three branch block " * 90, dict(TINY, branches=3, seed=11), 2),
    ]
    out = {}
    for name, data, c, s in cases:
        blob = write_container(edpc.compress(data, ModelConfig(**c), s, serial=True))
        out[f"{name}_data"] = np.frombuffer(data, dtype=np.uint8)
        out[f"{name}_blob"] = np.frombuffer(blob, dtype=np.uint8)
        out[f"{name}_cfg"] = np.array(json.dumps(dict(c, segments=s)))
    return out


def gen_adam(rng):
    n = 1024
    value = rng.normal(size=n)
    m = np.zeros(n)
    v = np.zeros(n)
    v0 = value.copy()
    grads = rng.normal(size=(30, n)) * np.logspace(-6, 1, n)
    for t in range(1, 31):
        g = grads[t - 1].copy()
        _kernels.adam_update(value, g, m, v, t, 1e-3, 0.9, 0.999, 1e-8)
    return dict(value0=v0, grads=grads, value=value, m=m, v=v)


def gen_ifr(_rng):
    from edpc.ifr import digamma, ksg_mi
    rng = np.random.Generator(np.random.PCG64(7))
    out = {}
    cases = []
    z = rng.standard_normal((700, 2))
    cases.append((z, np.concatenate([0.8 * z[:, :1] + 0.6 * rng.standard_normal((700, 1)),
                                     rng.standard_normal((700, 2))], 1), 5, 0))
    z = rng.standard_normal((500, 1))
    cases.append((z, 0.5 * z + rng.standard_normal((500, 1)), 1, 3))
    z = np.round(rng.standard_normal((400, 1)), 1)
    cases.append((z, np.round(z + 0.1 * rng.standard_normal((400, 1)), 1), 4, 0))
    z = rng.standard_normal((300, 2))
    cases.append((z, z.copy(), 5, 0))
    z = rng.standard_normal((1200, 8))
    cases.append((z, z[:, :8] * 0.3 + rng.standard_normal((1200, 8)), 5, 11))
    for i, (a, b, k, js) in enumerate(cases):
        est = ksg_mi(a, b, k, jitter_seed=js)
        out[f"z{i}"], out[f"y{i}"] = a, b
        out[f"meta{i}"] = np.array([k, js], np.int64)
        out[f"value{i}"] = np.array(est.value)
        out[f"flagged{i}"] = np.array(est.flagged)
    xs = np.concatenate([rng.uniform(1e-3, 1.0, 40), rng.uniform(1.0, 100.0, 40),
                         np.arange(1, 2001, dtype=np.float64)])
    out["digamma_x"] = xs
    out["digamma"] = digamma(xs)
    return out


def main():
    os.makedirs(GOLD, exist_ok=True)
    rng = np.random.Generator(np.random.PCG64(20250718))
    manifest = {}
    for name, fn in (("quantize", gen_quantize), ("coder", gen_coder), ("model", gen_model),
                     ("pipeline", gen_pipeline), ("adam", gen_adam), ("ifr", gen_ifr)):
        arrs = fn(rng)
        path = os.path.join(GOLD, f"{name}.npz")
        np.savez_compressed(path, **arrs)
        manifest[f"{name}.npz"] = hashlib.sha256(open(path, "rb").read()).hexdigest()
        print(name, os.path.getsize(path))
    manifest["generator"] = "oracle/make_goldens.py"
    manifest["reference"] = "/root/reference/pkg/src/edpc (edpc 0.1.0), numpy " + np.__version__
    with open(os.path.join(GOLD, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
