"""numpy restatement of the EDPC predictor and its online update (oracle only).

Follows the reference's float64 algorithm step by step so that, with the same
OpenBLAS and the C oracle kernels, it reproduces the reference bit for bit
(pinned by tests/test_oracle_golden.py):

* embedding gather            model.py:252-255
* MBRB forward / backward     model.py:95-121  (LN nn.py:103-125, linear nn.py:78-96,
                              GeLU _kernels.py:35-51, product rule model.py:109-119)
* LTE forward / backward      model.py:150-162 (per-row matmul nn.py:168-179)
* head + softmax              model.py:259-260, nn.py:186-190
* cross-entropy gradient      nn.py:193-210
* embedding scatter-add       model.py:276-278
* fused Adam over flat bufs   model.py:223-235 -> _kernels.py:18-32

``dtype=np.float32`` gives an fp32 variant of the same math (used to size
tolerances); the default float64 is the reference's.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from . import coder as _oc

VOCAB = 256


def _layout(cfg):
    f, fp, k = cfg.context_len * cfg.embed_dim, (cfg.context_len * cfg.embed_dim) // cfg.lte_ratio, cfg.branches
    names = [("embedding", (VOCAB, cfg.embed_dim))]

    def mbrb(blk, h):
        names.extend([(f"{blk}.ln_gain", (1, f)), (f"{blk}.ln_bias", (1, f))])
        for i in range(k):
            names.extend([(f"{blk}.branch{i}_w", (f, h)), (f"{blk}.branch{i}_b", (1, h))])
        names.extend([(f"{blk}.out_w", (h, f)), (f"{blk}.out_b", (1, f))])

    mbrb("local", cfg.hidden_local)
    names.extend([("lte.down_w", (f, fp)), ("lte.down_b", (1, fp)),
                  ("lte.lane_mats", (cfg.lanes, fp, fp)), ("lte.up_w", (fp, f)),
                  ("lte.up_b", (1, f))])
    mbrb("global", cfg.hidden_global)
    names.extend([("head_w", (f, VOCAB)), ("head_b", (1, VOCAB))])
    return names


def init_flat(cfg) -> np.ndarray:
    """Reference init (model.py:187-199, nn.py:50-58) as one float64 vector."""
    lay = _layout(cfg)
    sizes = [int(np.prod(s)) for _, s in lay]
    flat = np.zeros(sum(sizes))
    offs = dict(zip([n for n, _ in lay], np.cumsum([0] + sizes[:-1])))
    shapes = dict(lay)
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    f = cfg.context_len * cfg.embed_dim

    def u(name, fan_in):
        b = 1.0 / math.sqrt(fan_in)
        v = rng.uniform(-b, b, size=shapes[name]).reshape(-1)
        flat[offs[name]: offs[name] + v.size] = v

    u("embedding", cfg.embed_dim)
    for i in range(cfg.branches):
        u(f"local.branch{i}_w", f)
    u("local.out_w", cfg.hidden_local)
    u("lte.down_w", f)
    u("lte.lane_mats", f // cfg.lte_ratio)
    u("lte.up_w", f // cfg.lte_ratio)
    for i in range(cfg.branches):
        u(f"global.branch{i}_w", f)
    u("global.out_w", cfg.hidden_global)
    u("head_w", f)
    for blk in ("local", "global"):
        flat[offs[f"{blk}.ln_gain"]: offs[f"{blk}.ln_gain"] + f] = 1.0
    return flat


class OracleModel:
    """CPU oracle of ``EdpcModel`` (predict / train_step / state_checksum)."""

    def __init__(self, cfg, params: np.ndarray | None = None, dtype=np.float64):
        cfg.validate()
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        lay = _layout(cfg)
        init = init_flat(cfg) if params is None else np.asarray(params, dtype=np.float64)
        self.value = init.astype(self.dtype)
        self.grad = np.zeros_like(self.value)
        self.m = np.zeros_like(self.value)
        self.v = np.zeros_like(self.value)
        self.t = 0
        self.version = 0
        self.P, self.G = {}, {}
        off = 0
        for name, shape in lay:
            n = int(np.prod(shape))
            self.P[name] = self.value[off: off + n].reshape(shape)
            self.G[name] = self.grad[off: off + n].reshape(shape)
            off += n
        self.names = [n for n, _ in lay]

    # ------------------------------------------------------------ primitives
    def _lin(self, x, w, b):
        y = x @ self.P[w]
        y += self.P[b]
        return y

    def _lin_bwd(self, x, w, b, up):
        self.G[w] += x.T @ up
        self.G[b] += up.sum(axis=0, keepdims=True)
        return up @ self.P[w].T

    def _gelu(self, x):
        x = np.ascontiguousarray(x)
        if self.dtype == np.float64:
            out, cdf = np.empty_like(x), np.empty_like(x)
            _oc.lib().oracle_gelu_fwd(x.reshape(-1), out.reshape(-1), cdf.reshape(-1), x.size)
            return out, cdf
        from scipy.special import erf
        cdf = (0.5 * (1.0 + erf(x / np.sqrt(2.0).astype(x.dtype)))).astype(x.dtype)
        return x * cdf, cdf

    def _gelu_bwd(self, x, cdf, up):
        up = np.ascontiguousarray(up)
        if self.dtype == np.float64:
            out = np.empty_like(x)
            _oc.lib().oracle_gelu_bwd(np.ascontiguousarray(x).reshape(-1), cdf.reshape(-1),
                                      up.reshape(-1), out.reshape(-1), x.size)
            return out
        pdf = (np.exp(-0.5 * x * x) / np.sqrt(2.0 * np.pi)).astype(x.dtype)
        return up * (cdf + x * pdf)

    def _mbrb(self, blk, x):
        mean = x.mean(axis=1, keepdims=True)
        var = x.var(axis=1, keepdims=True)
        inv_std = 1.0 / np.sqrt(var + 1e-5)
        x_hat = (x - mean) * inv_std
        x0 = x_hat * self.P[f"{blk}.ln_gain"] + self.P[f"{blk}.ln_bias"]
        hs = [self._lin(x0, f"{blk}.branch{i}_w", f"{blk}.branch{i}_b")
              for i in range(self.cfg.branches)]
        prod = hs[0]
        for h in hs[1:]:
            prod = prod * h
        ff, cdf = self._gelu(prod)
        out = self._lin(ff, f"{blk}.out_w", f"{blk}.out_b") + x
        return out, (x0, x_hat, inv_std, hs, prod, cdf, ff)

    def _mbrb_bwd(self, blk, cache, up):
        x0, x_hat, inv_std, hs, prod, cdf, ff = cache
        g_ff = self._lin_bwd(ff, f"{blk}.out_w", f"{blk}.out_b", up)
        g_prod = self._gelu_bwd(prod, cdf, g_ff)
        g_x0 = None
        for i in range(len(hs)):
            g_h = g_prod
            for j in range(len(hs)):
                if j != i:
                    g_h = g_h * hs[j]
            gi = self._lin_bwd(x0, f"{blk}.branch{i}_w", f"{blk}.branch{i}_b", g_h)
            g_x0 = gi if g_x0 is None else g_x0 + gi
        gain = self.P[f"{blk}.ln_gain"]
        self.G[f"{blk}.ln_gain"] += (g_x0 * x_hat).sum(axis=0, keepdims=True)
        self.G[f"{blk}.ln_bias"] += g_x0.sum(axis=0, keepdims=True)
        g = g_x0 * gain
        gm = g.mean(axis=1, keepdims=True)
        gxm = (g * x_hat).mean(axis=1, keepdims=True)
        return (g - gm - x_hat * gxm) * inv_std + up

    # ------------------------------------------------------------- API
    def predict(self, contexts):
        cfg = self.cfg
        ctx = np.ascontiguousarray(contexts).astype(np.intp)
        if ctx.shape != (cfg.lanes, cfg.context_len):
            raise ValueError(f"contexts shape {ctx.shape} != ({cfg.lanes}, {cfg.context_len})")
        x = self.P["embedding"][ctx].reshape(cfg.lanes, -1)
        xl, c_local = self._mbrb("local", x)
        down = self._lin(xl, "lte.down_w", "lte.down_b")
        mixed = np.matmul(down[:, None, :], self.P["lte.lane_mats"])[:, 0, :]
        xt = self._lin(mixed, "lte.up_w", "lte.up_b")
        xg, c_global = self._mbrb("global", xt)
        logits = self._lin(xg, "head_w", "head_b")
        z = logits - logits.max(axis=1, keepdims=True)
        e = np.exp(z)
        probs = e / e.sum(axis=1, keepdims=True)
        cache = dict(version=self.version, ctx=ctx, c_local=c_local, xl=xl, down=down,
                     mixed=mixed, c_global=c_global, xg=xg, probs=probs)
        return probs, cache

    def train_step(self, cache, targets) -> float:
        if cache["version"] != self.version:
            raise ValueError("stale cache: model was updated since this predict")
        cfg = self.cfg
        tg = np.asarray(targets).astype(np.intp)
        probs = cache["probs"]
        rows = np.arange(cfg.lanes)
        loss = float(-np.log(probs[rows, tg]).mean())
        g = probs.copy()
        g[rows, tg] -= 1.0
        g /= cfg.lanes
        g = self._lin_bwd(cache["xg"], "head_w", "head_b", g)
        g = self._mbrb_bwd("global", cache["c_global"], g)
        g_mixed = self._lin_bwd(cache["mixed"], "lte.up_w", "lte.up_b", g)
        down = cache["down"]
        U = self.P["lte.lane_mats"]
        self.G["lte.lane_mats"] += down[:, :, None] * g_mixed[:, None, :]
        g_down = np.matmul(g_mixed[:, None, :], np.swapaxes(U, 1, 2))[:, 0, :]
        g = self._lin_bwd(cache["xl"], "lte.down_w", "lte.down_b", g_down)
        g = self._mbrb_bwd("local", cache["c_local"], g)
        np.add.at(self.G["embedding"], cache["ctx"].reshape(-1),
                  g.reshape(-1, cfg.embed_dim))
        self._adam()
        self.version += 1
        return loss

    def _adam(self):
        cfg = self.cfg
        self.t += 1
        if self.dtype == np.float64:
            _oc.lib().oracle_adam(self.value, self.grad, self.m, self.v, self.value.size, self.t,
                                  cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
            return
        b1, b2 = self.dtype.type(cfg.beta1), self.dtype.type(cfg.beta2)
        bc1 = self.dtype.type(1.0 - cfg.beta1 ** self.t)
        bc2 = self.dtype.type(1.0 - cfg.beta2 ** self.t)
        g = self.grad
        self.m[:] = b1 * self.m + (1 - b1) * g
        self.v[:] = b2 * self.v + (1 - b2) * (g * g)
        self.value -= (self.dtype.type(cfg.lr) * (self.m / bc1)) / (
            np.sqrt(self.v / bc2) + self.dtype.type(cfg.adam_eps))
        self.grad[:] = 0

    def parameters_flat(self) -> np.ndarray:
        return self.value

    def state_checksum(self) -> str:
        return hashlib.sha256(self.value.astype(np.float64).tobytes()).hexdigest()
