"""Model hyperparameters and closed-form parameter counts.

Mirrors the reference's ``ModelConfig`` (`pkg/src/edpc/model.py:23-63`) field
for field, default for default, so a reference caller can construct the same
object and hand it to :func:`paper_2507_18969_b200.compress`.  The parameter
count helpers restate `pkg/src/edpc/model.py:303-332`.

The parameter *layout* (``param_layout``) is the reference's flat parameter
order (`model.py:237-239`, `MbrbBlock.parameters` `:88-93`,
`LteBlock.parameters` `:147-148`); the device keeps its fp32 master copy,
Adam moments and gradient partials in exactly this order, which is what makes
``state_checksum`` and the host init comparable with the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

VOCAB = 256


@dataclass
class ModelConfig:
    context_len: int = 16
    embed_dim: int = 16
    hidden_local: int = 2048
    hidden_global: int = 4096
    lte_ratio: int = 4
    branches: int = 2
    lanes: int = 64
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 0

    @property
    def feature_dim(self) -> int:
        return self.context_len * self.embed_dim

    @property
    def latent_dim(self) -> int:
        return self.feature_dim // self.lte_ratio

    def validate(self) -> None:
        """Same checks and messages class as `model.py:46-60` (ValueError)."""
        if self.context_len < 1:
            raise ValueError("context_len must be >= 1")
        if self.embed_dim < 1:
            raise ValueError("embed_dim must be >= 1")
        if self.branches < 1:
            raise ValueError("branches must be >= 1")
        if self.lanes < 1:
            raise ValueError("lanes must be >= 1")
        if self.hidden_local < 1 or self.hidden_global < 1:
            raise ValueError("hidden dims must be >= 1")
        if self.lte_ratio < 1 or self.feature_dim % self.lte_ratio != 0:
            raise ValueError("lte_ratio must divide context_len * embed_dim")
        if self.feature_dim // self.lte_ratio < 1:
            raise ValueError("latent dim must be >= 1")

    def with_overrides(self, **kwargs) -> "ModelConfig":
        return replace(self, **kwargs)


def lte_param_count(feature_dim: int, lte_ratio: int, lanes: int) -> int:
    """down + per-lane latent matrices + up, with biases (`model.py:303-308`)."""
    fp = feature_dim // lte_ratio
    return feature_dim * fp + fp + lanes * fp * fp + fp * feature_dim + feature_dim


def dense_mixer_param_count(feature_dim: int) -> int:
    """The F x F linear the latent transform replaces (`model.py:311-313`)."""
    return feature_dim * feature_dim + feature_dim


def _mbrb_count(f: int, h: int, k: int) -> int:
    return 2 * f + k * (f * h + h) + h * f + f


def model_param_count(cfg: ModelConfig) -> int:
    """Closed-form total (`model.py:316-324`)."""
    f = cfg.feature_dim
    return (VOCAB * cfg.embed_dim + _mbrb_count(f, cfg.hidden_local, cfg.branches)
            + lte_param_count(f, cfg.lte_ratio, cfg.lanes)
            + _mbrb_count(f, cfg.hidden_global, cfg.branches) + f * VOCAB + VOCAB)


def model_param_count_dense_mixer(cfg: ModelConfig) -> int:
    """Total if the LTE were a dense mixer (`model.py:327-332`)."""
    f = cfg.feature_dim
    return (model_param_count(cfg) - lte_param_count(f, cfg.lte_ratio, cfg.lanes)
            + dense_mixer_param_count(f))


def param_layout(cfg: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    """(name, shape) in the reference's flat ``parameters()`` order."""
    f, fp, k = cfg.feature_dim, cfg.latent_dim, cfg.branches
    out: list[tuple[str, tuple[int, ...]]] = [("embedding", (VOCAB, cfg.embed_dim))]

    def mbrb(name: str, h: int) -> None:
        out.append((f"{name}.ln_gain", (1, f)))
        out.append((f"{name}.ln_bias", (1, f)))
        for i in range(k):
            out.append((f"{name}.branch{i}_w", (f, h)))
            out.append((f"{name}.branch{i}_b", (1, h)))
        out.append((f"{name}.out_w", (h, f)))
        out.append((f"{name}.out_b", (1, f)))

    mbrb("local", cfg.hidden_local)
    out += [("lte.down_w", (f, fp)), ("lte.down_b", (1, fp)),
            ("lte.lane_mats", (cfg.lanes, fp, fp)),
            ("lte.up_w", (fp, f)), ("lte.up_b", (1, f))]
    mbrb("global", cfg.hidden_global)
    out += [("head_w", (f, VOCAB)), ("head_b", (1, VOCAB))]
    return out


def param_offsets(cfg: ModelConfig) -> dict[str, tuple[int, tuple[int, ...]]]:
    """name -> (flat offset, shape) in the reference order."""
    res, off = {}, 0
    for name, shape in param_layout(cfg):
        size = 1
        for d in shape:
            size *= d
        res[name] = (off, shape)
        off += size
    return res
