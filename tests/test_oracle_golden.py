"""Pins the CPU oracle against golden vectors the reference itself produced.

The goldens (tests/golden/*.npz) were written by oracle/make_goldens.py by
calling the unmodified reference (`pkg/src/edpc`); this file checks that the
oracle restatement reproduces them bit for bit, so that the oracle can stand
in for the reference as the parity checker on the GPU box (where
/root/reference does not exist).
"""

import json

import numpy as np

from oracle import coder as oc
from oracle.model import OracleModel, init_flat
from oracle import pipeline as op
from paper_2507_18969_b200.config import ModelConfig
from paper_2507_18969_b200.container import read_container
from paper_2507_18969_b200.init import init_params_f64


def test_quantize_matches_reference(golden):
    g = golden("quantize")
    f32, _ = oc.quantize_rows(g["probs_f32"].astype(np.float64))
    assert np.array_equal(f32, g["freqs_f32"].astype(np.int64))
    f64, _ = oc.quantize_rows(g["probs_f64"])
    assert np.array_equal(f64, g["freqs_f64"].astype(np.int64))


def _cums(freqs):
    c = np.zeros((freqs.shape[0], 257), dtype=np.uint64)
    np.cumsum(freqs.astype(np.uint64), axis=1, out=c[:, 1:])
    return c


def test_coder_matches_reference(golden):
    g = golden("coder")
    pool = _cums(g["pool_freqs"])
    for k in range(len(g["bits"])):
        r0, r1 = g["row_off"][k], g["row_off"][k + 1]
        rows, syms = g["rows"][r0:r1], g["symbols"][r0:r1].astype(np.int64)
        enc = oc.ArithmeticEncoder()
        enc.encode_rows(pool[rows], syms)
        payload, bits = enc.finish()
        p0, p1 = g["pay_off"][k], g["pay_off"][k + 1]
        assert bits == g["bits"][k]
        assert payload == g["payload"][p0:p1].tobytes()
        dec = oc.ArithmeticDecoder(payload, bits)
        out = np.empty(len(syms), dtype=np.int64)
        dec.decode_rows(pool[rows], out)
        assert np.array_equal(out, syms)


def test_init_matches_reference(golden):
    g = golden("model")
    i = 0
    while f"init_{i}" in g:
        cfg = ModelConfig(**json.loads(str(g[f"init_cfg_{i}"])))
        assert np.array_equal(init_flat(cfg), g[f"init_{i}"])
        assert np.array_equal(init_params_f64(cfg), g[f"init_{i}"])
        i += 1


def test_step_probs_and_checksums_match_reference(golden):
    g = golden("model")
    cfg = ModelConfig(context_len=8, embed_dim=4, hidden_local=16, hidden_global=32,
                      lte_ratio=4, branches=2, lanes=8, seed=5)
    data = g["step_data"].tobytes()
    probs, sums = [], []
    m = OracleModel(cfg)
    L = -(-len(data) // cfg.lanes)
    mat = np.zeros((cfg.lanes, L), np.uint8)
    mat.reshape(-1)[: len(data)] = np.frombuffer(data, np.uint8)
    for i in range(cfg.context_len, L):
        p, c = m.predict(mat[:, i - cfg.context_len: i])
        probs.append(p)
        m.train_step(c, mat[:, i])
        if (i - cfg.context_len + 1) % 25 == 0:
            sums.append(m.state_checksum())
    n = g["step_probs"].shape[0]
    assert np.array_equal(np.stack(probs[:n]), g["step_probs"])
    assert sums == list(g["step_checksums"])


def test_pipeline_containers_match_reference(golden):
    g = golden("pipeline")
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    for name in names:
        meta = json.loads(str(g[f"{name}_cfg"]))
        segs = meta.pop("segments")
        cfg = ModelConfig(**meta)
        data = g[f"{name}_data"].tobytes()
        blob = g[f"{name}_blob"].tobytes()
        ref = read_container(blob, version=1)
        payloads, bits = op.compress(data, cfg, segs)
        if not data:
            assert ref.header.segment_count == 0 and payloads == []
            continue
        assert bits == ref.header.bit_lengths, name
        assert payloads == ref.segments, name
        assert op.decompress(payloads, bits, cfg, len(data)) == data


def test_adam_matches_reference(golden):
    g = golden("adam")
    n = g["value0"].size
    value = g["value0"].copy()
    m, v = np.zeros(n), np.zeros(n)
    for t in range(1, g["grads"].shape[0] + 1):
        grad = g["grads"][t - 1].copy()
        oc.lib().oracle_adam(value, grad, m, v, n, t, 1e-3, 0.9, 0.999, 1e-8)
        assert not grad.any()
    assert np.array_equal(value, g["value"])
    assert np.array_equal(m, g["m"]) and np.array_equal(v, g["v"])


def test_ksg_oracle_matches_reference(golden):
    """oracle/ifr.py (KSG restatement) reproduces the reference's estimates
    bit for bit; the product's host digamma equals the reference's."""
    from oracle import ifr as oi
    from paper_2507_18969_b200.ifr import digamma
    g = golden("ifr")
    i = 0
    while f"z{i}" in g:
        k, js = (int(v) for v in g[f"meta{i}"])
        value, flagged = oi.ksg_mi(g[f"z{i}"], g[f"y{i}"], k, js)
        assert value == float(g[f"value{i}"]), i
        assert flagged == bool(g[f"flagged{i}"]), i
        i += 1
    assert i == 5
    assert np.array_equal(digamma(g["digamma_x"]), g["digamma"])
    assert np.array_equal(oi.digamma(g["digamma_x"]), g["digamma"])
