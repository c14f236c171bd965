"""G-invariance of the sharded path on one B200: G contexts on the same GPU,
each owning 8/G lane groups and their segments, exchanging gradient partials
device-to-device every step, must produce exactly the single-GPU container
(`pipeline.py:117-118` bytes = f(data, cfg, S))."""
import numpy as np
import pytest

from paper_2507_18969_b200 import ModelConfig, compress, decompress, read_container, write_container
from paper_2507_18969_b200 import dist, synth
from helpers import PAPER, TINY

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,segments", [(2, 4), (4, 4), (8, 8)])
def test_sharded_tiny_is_bit_identical(world, segments):
    data = synth.text_like(6000, 3)
    ref = write_container(compress(data, TINY, segments))
    got = write_container(dist.compress_multi(data, TINY, segments, [0] * world))
    assert got == ref
    assert dist.decompress_multi(read_container(got), [0] * world) == data


@pytest.fixture(scope="module")
def paper1024():
    """Paper dims at 1024 lanes: the benchmark's numerics (tcgen05 GEMMs, fp16
    MBRB operands with 128-lane groups, fused LTE forward); single-GPU
    container as the reference bytes."""
    cfg = ModelConfig(**PAPER, lanes=1024)
    data = synth.text_like(1024 * 56, 5)
    c = compress(data, cfg, 16)
    assert c.header.numerics == 15, c.header.numerics
    return cfg, data, write_container(c)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_paper_dims_tcgen05_is_bit_identical(paper1024, world):
    """G contexts (the sharded optimizer, the fp16 weight-shadow pull, early
    side-stream Adam off) give exactly the single-GPU container."""
    cfg, data, ref = paper1024
    got = write_container(dist.compress_multi(data, cfg, 16, [0] * world))
    assert got == ref
    assert decompress(read_container(got), devices=[0] * world) == data


def test_lane_plan_rejects_straddling_geometry():
    with pytest.raises(ValueError):
        dist.lane_plan(TINY.with_overrides(lanes=12), 4, 2)   # 12 % 8
    with pytest.raises(ValueError):
        dist.lane_plan(TINY, 2, 4)                           # 4-lane segments over 2-lane shares
    with pytest.raises(ValueError):
        dist.lane_plan(TINY, 4, 3)                           # 3 does not divide 8


def _gpus():
    from paper_2507_18969_b200 import _lib
    return _lib.device_count()


@pytest.mark.skipif("_gpus() < 2")
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_ranks_match_single_gpu(paper1024, world):
    """One host thread per GPU, NCCL send/recv + all-gather captured in every
    rank's step graphs (dist._compress_nccl): the single-GPU container, bit
    for bit, and its decompression."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cfg, data, ref = paper1024
    assert dist._use_nccl(list(range(world)))
    stats = {}
    got = write_container(dist.compress_multi(data, cfg, 16, list(range(world)), stats=stats))
    assert stats["mode"] == "nccl"
    assert got == ref
    assert dist.decompress_multi(read_container(got), list(range(world))) == data
