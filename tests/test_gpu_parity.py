"""Parity at the numerics the benchmark runs (tcgen05 + fp16 MBRB + fused LTE
forward at paper dims, B >= 1024), against the fp64 CPU oracle that is pinned
bit-for-bit to the reference (tests/test_oracle_golden.py).

* trained weights: the GPU model is trained online for a few hundred steps on
  the benchmark's own stream (compress loop), its weights are read back and
  loaded into the oracle, and the next step's probabilities are compared --
  max |dp| <= 1e-3 (the north star's example tolerance; the measured bound is
  printed).  Near-uniform probabilities at init would hide operand-precision
  errors (bf16 passed at init, failed after 300 steps).
* gradients: every shared-parameter gradient (the 8 lane-group partials,
  tree-summed in the canonical order) and the per-lane FDM gradient against
  the oracle's accumulated .grad, per tensor, relative Frobenius error.
* Adam: the device Adam kernel against the reference-generated 30-step
  trajectory (tests/golden/adam.npz).
"""
import ctypes

import numpy as np
import pytest

from oracle.model import OracleModel
from paper_2507_18969_b200 import EdpcModel, ModelConfig, _lib, synth
from paper_2507_18969_b200.config import param_offsets
from paper_2507_18969_b200.dist import tree_sum
from paper_2507_18969_b200.init import init_params_f32
from paper_2507_18969_b200.model import DeviceContext
from helpers import PAPER, TINY, DESK

pytestmark = pytest.mark.gpu
PROB_TOL = 1e-3
ORACLE_LANES = 256  # probability check on an evenly spread lane sample (lanes are independent)

# (name, model dims, lanes, segments, stream kind, stream bytes, training steps,
#  expected numerics flags)
TRAINED = [
    ("c2", PAPER, 4096, 256, "text", 4 << 20, 300, 15),
    ("c4a", dict(PAPER, branches=1), 4096, 256, "text", 4 << 20, 300, 13),
    ("c4b", dict(PAPER, lte_ratio=1), 4096, 256, "text", 4 << 20, 300, 11),
    ("c3", PAPER, 32768, 1024, "mixed", 8 << 20, 200, 15),
]


def _read(ctx, which, n):
    out = np.empty(n, dtype=np.float32)
    _lib.check(_lib.load().edpc_debug_read(ctx.h, which, out.ctypes.data, n))
    return out


def _lane_subset(cfg, params, lanes):
    """(cfg, params) of a model restricted to `lanes` (the per-lane FDM rows)."""
    offs = param_offsets(cfg)
    o, shape = offs["lte.lane_mats"]
    fdm = shape[1] * shape[2]
    mats = params[o: o + cfg.lanes * fdm].reshape(cfg.lanes, fdm)[lanes]
    sub = np.concatenate([params[:o], mats.reshape(-1), params[o + cfg.lanes * fdm:]])
    return cfg.with_overrides(lanes=len(lanes)), sub


@pytest.mark.parametrize("name,dims,lanes,segs,kind,nbytes,steps,flags", TRAINED,
                         ids=[t[0] for t in TRAINED])
def test_trained_probs_match_oracle(name, dims, lanes, segs, kind, nbytes, steps, flags):
    cfg = ModelConfig(**dims, lanes=lanes)
    data = synth.generate(kind, nbytes, 0)
    lib = _lib.load()
    ctx = DeviceContext(cfg, segs, len(data), 0)
    assert ctx.numerics_flags() == flags, ctx.numerics()
    ctx.load_flat(init_params_f32(cfg))
    buf = np.frombuffer(data, np.uint8)
    _lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, len(data), 0))
    T = cfg.context_len
    i = T + steps
    _lib.check(lib.edpc_compress_steps(ctx.h, 0, i))
    params = ctx.params_flat()
    numerics = ctx.numerics()
    ctx.close()
    L = -(-len(data) // lanes)
    mat = np.zeros((lanes, L), np.uint8)
    mat.reshape(-1)[: len(data)] = buf
    contexts = np.ascontiguousarray(mat[:, i - T: i])
    g = EdpcModel(cfg, params=params)
    assert g.numerics() == numerics
    pg, _ = g.predict(contexts)
    sel = np.linspace(0, lanes - 1, ORACLE_LANES).astype(np.int64)
    scfg, sparams = _lane_subset(cfg, params.astype(np.float64), sel)
    po, _ = OracleModel(scfg, params=sparams).predict(contexts[sel])
    err = float(np.abs(pg[sel] - po).max())
    mean = float(np.abs(pg[sel] - po).mean())
    print(f"{name}: trained {steps} steps, max p {po.max():.3f}, max|dp| {err:.2e}, "
          f"mean|dp| {mean:.2e}")
    assert po.max() > 0.5, "model did not train (probabilities still near uniform)"
    assert err <= PROB_TOL, (name, err)


GRAD_CASES = [
    # (cfg, relative Frobenius tolerance per tensor): fp32 SIMT path (measured
    # <= 2.3e-6) / tcgen05 + fp16 MBRB + tf32 path at paper dims (measured <= 1.6e-3)
    (TINY, 1e-5),
    (ModelConfig(**DESK, lanes=16), 1e-5),
    (ModelConfig(**PAPER, lanes=64), 1e-5),
    (ModelConfig(**PAPER, lanes=4096), 5e-3),
]


@pytest.mark.parametrize("cfg,tol", GRAD_CASES, ids=["tiny", "desk", "paper64", "paper4096"])
def test_gradients_match_oracle(cfg, tol):
    """One predict + train_step on trained-ish inputs (a text stream's
    contexts): every gradient tensor against the oracle's .grad."""
    params = init_params_f32(cfg)
    g = EdpcModel(cfg, params=params)
    # fused weight-gradient/Adam kernels never materialise the partials: keep
    # the reduced gradient readable through edpc_debug_read(0)
    _lib.check(_lib.load().edpc_debug_keep_grads(g._ctx.h, 1))
    o = OracleModel(cfg, params=params.astype(np.float64))
    o._adam = lambda: None  # keep the accumulated gradients (the oracle zeroes them in Adam)
    data = np.frombuffer(synth.generate("text", cfg.lanes * (cfg.context_len + 1), 7), np.uint8)
    rows = data.reshape(cfg.lanes, cfg.context_len + 1)
    ctx, tg = rows[:, :-1], rows[:, -1]
    _, cg = g.predict(ctx)
    g.train_step(cg, tg)
    _, co = o.predict(ctx)
    o.train_step(co, tg)
    n_sh = g._ctx.n_shared
    parts = _read(g._ctx, 0, 8 * n_sh).reshape(8, n_sh)
    grad = tree_sum([p for p in parts])
    offs = param_offsets(cfg)
    lm, lshape = offs["lte.lane_mats"]
    fdm = int(np.prod(lshape))
    worst = {}
    for nm, (off, shape) in offs.items():
        ref = o.G[nm].reshape(-1)
        if nm == "lte.lane_mats":
            # fused FDM backward + Adam: after the first step m = (1 - beta1) * g
            got = _read(g._ctx, 9, fdm).astype(np.float64) / (1.0 - cfg.beta1)
        else:
            so = off if off < lm else off - fdm
            got = grad[so: so + ref.size].astype(np.float64)
        den = max(np.linalg.norm(ref), 1e-30)
        worst[nm] = float(np.linalg.norm(got - ref) / den)
    print({k: f"{v:.1e}" for k, v in worst.items()})
    bad = {k: v for k, v in worst.items() if v > tol}
    assert not bad, bad


def test_shared_adam_state_after_one_step_matches_oracle():
    """m and v of the shared parameters after one update equal the oracle's
    (1 - beta1) g and (1 - beta2) g^2: checks the gradient scale removal and
    the moment updates of the fused Adam path end to end (fp32 SIMT path)."""
    cfg = ModelConfig(**DESK, lanes=16)
    params = init_params_f32(cfg)
    g = EdpcModel(cfg, params=params)
    o = OracleModel(cfg, params=params.astype(np.float64))
    rng = np.random.default_rng(3)
    ctx = rng.integers(0, 256, size=(cfg.lanes, cfg.context_len))
    tg = rng.integers(0, 256, size=cfg.lanes)
    _, cg = g.predict(ctx)
    g.train_step(cg, tg)
    _, co = o.predict(ctx)
    o.train_step(co, tg)
    offs = param_offsets(cfg)
    lm, lshape = offs["lte.lane_mats"]
    fdm = int(np.prod(lshape))
    keep = np.ones(o.m.size, bool)
    keep[lm: lm + fdm] = False
    m_ref, v_ref = o.m[keep], o.v[keep]
    n_sh = g._ctx.n_shared
    m = _read(g._ctx, 10, n_sh).astype(np.float64)
    v = _read(g._ctx, 11, n_sh).astype(np.float64)
    assert np.linalg.norm(m - m_ref) / np.linalg.norm(m_ref) < 1e-4
    assert np.linalg.norm(v - v_ref) / np.linalg.norm(v_ref) < 2e-4
    pg = g.parameters_flat().astype(np.float64)
    # first Adam step: w -= lr * g / (|g| + eps'), so the step is sign-driven;
    # compare where the gradient is not negligible
    big = np.abs(o.m) > 1e-3 * np.abs(o.m).max()
    d_gpu, d_ref = (pg - params)[big], (o.value - params)[big]
    assert np.abs(d_gpu - d_ref).max() <= 1e-3 * cfg.lr * 10


def test_device_adam_matches_reference_trajectory(golden):
    """k_adam_shared (fp32) over the reference's 30-step Adam trajectory."""
    gd = golden("adam")
    n = gd["value0"].size
    steps = gd["grads"].shape[0]
    w0 = gd["value0"].astype(np.float32)
    grads = np.ascontiguousarray(gd["grads"].astype(np.float32))
    w, m, v = (np.empty(n, np.float32) for _ in range(3))
    _lib.check(_lib.load().edpc_debug_adam(w0.ctypes.data, grads.ctypes.data, n, steps, 1e-3, 0.9,
                                           0.999, 1e-8, w.ctypes.data, m.ctypes.data,
                                           v.ctypes.data))
    # fp32 state vs the fp64 reference: a few ulp of drift per step
    assert np.abs(w - gd["value"]).max() <= 1e-6 + 1e-6 * np.abs(gd["value"]).max()
    # moments: relative to their scale (m cancels through zero for some entries)
    assert np.abs(m - gd["m"]).max() <= 1e-5 * np.abs(gd["m"]).max()
    assert np.abs(v - gd["v"]).max() <= 1e-5 * np.abs(gd["v"]).max()
