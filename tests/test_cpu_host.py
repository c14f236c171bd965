"""CPU-side checks: host logic, formats, init, and the C-ABI library surface.

No GPU compute here (the driver runs these on a CPU-only box); compute
paths are exercised by the -m gpu tests.
"""
import ctypes
import os
import re
import struct
import zlib

import numpy as np
import pytest

from paper_2507_18969_b200 import _lib
from paper_2507_18969_b200.config import (ModelConfig, lte_param_count, model_param_count,
                                          param_layout, param_offsets)
from paper_2507_18969_b200.container import (BadMagicError, BadVersionError, ChecksumError,
                                             ContainerError, EdpcContainer, Header,
                                             InvalidHeaderError, TruncatedError, header_size,
                                             read_container, write_container)
from paper_2507_18969_b200.init import init_params_f64
from paper_2507_18969_b200.lanes import join_lanes, segment_spans, split_lanes, validate_geometry
from paper_2507_18969_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ config

def test_config_validation():
    toy = ModelConfig(context_len=4, embed_dim=4, hidden_local=8, hidden_global=8,
                      lte_ratio=2, branches=2, lanes=2, seed=7)
    for bad in (dict(lte_ratio=3), dict(branches=0), dict(lanes=0), dict(context_len=0),
                dict(hidden_local=0)):
        with pytest.raises(ValueError):
            toy.with_overrides(**bad).validate()


def test_param_counts_match_layout_and_closed_form():
    cfg = ModelConfig()
    total = sum(int(np.prod(s)) for _, s in param_layout(cfg))
    assert total == model_param_count(cfg) == 5_097_536  # test_model.py:270-289
    f = cfg.feature_dim
    assert lte_param_count(f, 4, 64) == f * 64 + 64 + 64 * 64 * 64 + 64 * f + f
    c2 = cfg.with_overrides(lanes=4096)
    assert model_param_count(c2) == 21_612_608


def test_param_offsets_are_contiguous():
    cfg = ModelConfig(context_len=8, embed_dim=4, hidden_local=16, hidden_global=32, lanes=8)
    offs = param_offsets(cfg)
    pos = 0
    for name, shape in param_layout(cfg):
        assert offs[name][0] == pos
        pos += int(np.prod(shape))


# ------------------------------------------------------------------- lanes

def test_split_join_property():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(0, 5000))
        lanes = int(rng.integers(1, 65))
        data = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        split, mat = split_lanes(data, lanes)
        assert mat.shape == (lanes, split.lane_len)
        assert join_lanes(split, mat) == data


def test_split_padding_and_spans():
    split, mat = split_lanes(bytes(range(10)), 4)
    assert split.lane_len == 3 and mat[3, 1] == 0 and mat[3, 2] == 0
    assert segment_spans(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        validate_geometry(ModelConfig(lanes=8), 3)
    with pytest.raises(ValueError):
        validate_geometry(ModelConfig(lanes=8), 0)


# -------------------------------------------------------------- container

def _container(S=3):
    cfg = ModelConfig(context_len=8, embed_dim=4, hidden_local=16, hidden_global=32, lanes=6)
    segs = [bytes([i]) * (i + 1) for i in range(S)]
    bits = [8 * (i + 1) - i for i in range(S)]
    return EdpcContainer(Header.from_config(cfg, 1234, bits), segs)


def test_container_roundtrip_and_sizes():
    c = _container()
    blob = write_container(c)
    assert len(blob) == header_size(3) + sum(len(s) for s in c.segments)
    back = read_container(blob)
    assert back.header == c.header and back.segments == c.segments
    assert write_container(back) == blob
    empty = EdpcContainer(Header.from_config(ModelConfig(), 0, []), [])
    assert len(write_container(empty)) == 89  # test_container.py:37-43


def test_container_rejects_corruption():
    blob = write_container(_container())
    hs = header_size(3)
    for pos in range(hs):  # every single-byte header corruption is detected
        bad = bytearray(blob)
        bad[pos] ^= 0x5A
        with pytest.raises(ContainerError):
            read_container(bytes(bad))
    with pytest.raises(BadMagicError):
        read_container(b"XXXX" + blob[4:])
    with pytest.raises(TruncatedError):
        read_container(blob[:3])
    for cut in range(5, len(blob)):
        with pytest.raises(ContainerError):
            read_container(blob[:cut])


def test_container_version_separates_numerics():
    blob = bytearray(write_container(_container()))
    assert blob[4] == 2
    # the encoder's numerics flags ride in the version byte's high nibble
    c = _container()
    c.header.numerics = 7
    b7 = write_container(c)
    assert b7[4] == 0x72 and read_container(b7).header.numerics == 7
    c.header.numerics = 16
    with pytest.raises(ContainerError):
        write_container(c)
    bad = bytearray(b7)
    bad[4] = 0x73  # bad low nibble
    with pytest.raises(ContainerError):
        read_container(bytes(bad))
    v1 = write_container(_container(), version=1)
    with pytest.raises(BadVersionError):
        read_container(v1)  # a reference (fp64) container is not GPU-decodable
    assert read_container(v1, version=1).header == _container().header


def test_container_random_blobs_rejected():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(0, 200))
        blob = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        if rng.random() < 0.5:
            blob = b"EDPC\x02" + blob
        with pytest.raises(ContainerError):
            read_container(blob)


def test_container_bounds_before_allocation():
    head = bytearray(b"EDPC\x02" + struct.pack("<QQ8I4d", 10, 0, 8, 4, 16, 32, 4, 2, 8,
                                                 (1 << 20) + 1, 1e-3, .9, .999, 1e-8))
    with pytest.raises(InvalidHeaderError):
        read_container(bytes(head))


# --------------------------------------------------------------------- init

def test_init_matches_reference_golden(golden):
    import json
    g = golden("model")
    i = 0
    while f"init_{i}" in g:
        cfg = ModelConfig(**json.loads(str(g[f"init_cfg_{i}"])))
        assert np.array_equal(init_params_f64(cfg), g[f"init_{i}"])
        i += 1


# ------------------------------------------------------------------- synth

def test_synth_is_seeded_and_textlike():
    a = synth.text_like(1 << 16, 3)
    assert a == synth.text_like(1 << 16, 3) and a != synth.text_like(1 << 16, 4)
    assert 3.8 < synth.order0_bpb(a) < 4.8
    m = synth.mixed(3 << 20, 0)
    assert len(m) == 3 << 20
    assert synth.order0_bpb(m[1 << 20: 2 << 20]) > 6.5  # image block


# ------------------------------------------------------------ C-ABI surface

def _header_functions():
    src = open(os.path.join(ROOT, "include", "edpc_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(edpc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2507_18969_b200 import build
    build.build()
    lib = _lib.load()
    declared = _header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.exported_symbols())
    assert lib.edpc_abi_version() == 1


def test_compute_without_gpu_fails_loudly():
    lib = _lib.load()
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.EdpcNativeError):
        _lib.require_device(0)
    p = np.full((1, 256), 1 / 256, dtype=np.float32)
    out = np.empty((1, 257), dtype=np.uint32)
    st = lib.edpc_quantize_rows(0, p.ctypes.data, 1, 0, out.ctypes.data)
    assert st == _lib.ERR_CUDA
    from paper_2507_18969_b200 import compress
    with pytest.raises(_lib.EdpcNativeError):
        compress(b"hello world" * 10, ModelConfig(context_len=4, embed_dim=2, hidden_local=8,
                                                   hidden_global=8, lanes=4), 2)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_18969_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def test_library_does_not_preload_a_conflicting_nccl():
    """torch must still import after the library is loaded (NCCL is dlopen'ed
    lazily, only for multi-GPU, so torch's bundled NCCL wins)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); from paper_2507_18969_b200 import _lib; "
            "_lib.load(); import torch; print('ok')" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_archive_format_roundtrip_and_corruption():
    """Chunked multi-container framing (archive.py): index round trip, every
    single-byte index corruption and every truncation detected."""
    from paper_2507_18969_b200.archive import (archive_header_size, read_archive,
                                               write_archive)
    blobs = [write_container(_container(S)) for S in (1, 2, 3)]
    arc = write_archive(1000, 2500, blobs)
    head, got = read_archive(arc)
    assert got == blobs and head.chunk_count == 3
    assert [head.chunk_span(k) for k in range(3)] == [(0, 1000), (1000, 2000), (2000, 2500)]
    hs = archive_header_size(3)
    for pos in range(hs):
        bad = bytearray(arc)
        bad[pos] ^= 0x5A
        with pytest.raises(ContainerError):
            read_archive(bytes(bad))
    for cut in range(0, len(arc)):
        with pytest.raises(ContainerError):
            read_archive(arc[:cut])
    with pytest.raises(ContainerError):
        read_archive(arc + b"x")
    with pytest.raises(ContainerError):
        write_archive(1000, 2500, blobs[:2])  # chunk count must match the length
    assert read_archive(write_archive(7, 0, []))[1] == []
