"""Shared test helpers: configs from the reference suite, skip logic."""
import numpy as np
import pytest

from paper_2507_18969_b200.config import ModelConfig

# the reference test-suite's tiny pipeline config (test_pipeline.py:13-14)
TINY = ModelConfig(context_len=8, embed_dim=4, hidden_local=16, hidden_global=32,
                   lte_ratio=4, branches=2, lanes=8, seed=5)
# the reference test-suite's toy model config (test_model.py:15-16)
TOY = ModelConfig(context_len=4, embed_dim=4, hidden_local=8, hidden_global=8,
                  lte_ratio=2, branches=2, lanes=2, seed=7)
DESK = dict(context_len=16, embed_dim=8, hidden_local=256, hidden_global=512, lte_ratio=4,
            branches=2)
PAPER = dict(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lte_ratio=4,
             branches=2)
# BASELINE.json config 5 (scaled EDPC)
SCALED = dict(context_len=32, embed_dim=16, hidden_local=4096, hidden_global=8192, lte_ratio=4,
              branches=2)


def tiny_cfg(**kw):
    return TINY.with_overrides(**kw)


def softmax_rows(rng, n, scale=4.0):
    z = rng.normal(size=(n, 256)).astype(np.float32) * np.float32(scale)
    z = z - z.max(1, keepdims=True)
    e = np.exp(z)
    return (e / e.sum(1, keepdims=True)).astype(np.float32)
