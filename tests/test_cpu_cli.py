"""CLI host-side contract on CPU (no GPU compute): the reference's exit codes
(`pkg/src/edpc/cli.py:3-4,24-28`, `:338-357`) for bad usage, invalid
configurations, corrupt containers and I/O failures, profile resolution, and
the metrics line.  Round trips through the CLI are in test_gpu_pipeline.py."""
import json
import os

import pytest

from paper_2507_18969_b200 import cli
from paper_2507_18969_b200.config import ModelConfig, model_param_count
from paper_2507_18969_b200.container import EdpcContainer, Header, write_container


def _args(argv):
    return cli.build_parser().parse_args(argv)


def test_profiles_and_overrides():
    cfg, seg = cli.resolve_config(_args(["compress", "-i", "a", "-o", "b"]))
    assert (cfg.lanes, seg, cfg.hidden_global, cfg.feature_dim) == (64, 32, 4096, 256)
    cfg, seg = cli.resolve_config(_args(["compress", "-i", "a", "-o", "b", "--profile", "desk",
                                         "--lanes", "4096", "--segments", "256", "--seed", "3"]))
    assert (cfg.lanes, seg, cfg.hidden_local, cfg.seed) == (4096, 256, 256, 3)


@pytest.mark.parametrize("argv", [
    ["compress", "-i", "x"],                                              # missing -o
    ["frobnicate"],                                                       # unknown command
    ["compress", "-i", "x", "-o", "y", "--lanes", "64", "--segments", "7"],  # S does not divide B
    ["compress", "-i", "x", "-o", "y", "--lte-ratio", "3"],                  # F' not integral
    ["compress", "-i", "x", "-o", "y", "--devices", "0,zero"],
    ["compress", "-i", "x", "-o", "y", "--devices", "1,1"],
])
def test_usage_errors_exit_64(argv, tmp_path):
    src = tmp_path / "x"
    src.write_bytes(b"abc")
    argv = [str(src) if a == "x" else str(tmp_path / "y") if a == "y" else a for a in argv]
    assert cli.main(argv) == cli.EXIT_USAGE


def test_corrupt_container_exit_3(tmp_path):
    cfg = ModelConfig(lanes=64)
    blob = bytearray(write_container(EdpcContainer(header=Header.from_config(cfg, 0, []),
                                                   segments=[])))
    blob[10] ^= 0xFF  # inside the CRC-covered header
    bad = tmp_path / "bad.edpc"
    bad.write_bytes(bytes(blob))
    assert cli.main(["decompress", "-i", str(bad), "-o", str(tmp_path / "out")]) == cli.EXIT_CORRUPT
    bad.write_bytes(b"EDPC")  # truncated
    assert cli.main(["verify", "-i", str(bad), "-c", str(bad)]) == cli.EXIT_CORRUPT


def test_missing_input_exit_2(tmp_path):
    assert cli.main(["decompress", "-i", str(tmp_path / "nope"), "-o", str(tmp_path / "o")]) == cli.EXIT_IO


def test_empty_container_decompresses_without_gpu(tmp_path):
    """n = 0: header-only container (89 bytes, S = 0, pipeline.py:123-128) ->
    b"" with no device work (pipeline.py:245-248)."""
    cfg = ModelConfig(lanes=64)
    blob = write_container(EdpcContainer(header=Header.from_config(cfg, 0, []), segments=[]))
    assert len(blob) == 89
    src, out = tmp_path / "e.edpc", tmp_path / "e.out"
    src.write_bytes(blob)
    assert cli.main(["decompress", "-i", str(src), "-o", str(out)]) == cli.EXIT_OK
    assert out.read_bytes() == b""


def test_metrics_line_and_order0():
    m = cli.Metrics(file="f", original_bytes=1000, compressed_bytes=400, ratio=2.5,
                    seconds={"wall": 2.0}, param_count=model_param_count(ModelConfig()),
                    mb_per_s=0.0005)
    d = json.loads(m.json_line())
    assert d["ratio"] == 2.5 and d["param_count"] == 5_097_536 and "mb_per_s" in d
    assert "1000 -> 400 bytes" in m.human()
    assert cli.order0_entropy_bits(b"") == 0.0
    assert abs(cli.order0_entropy_bits(bytes(range(256)) * 4) - 8.0) < 1e-12
    assert cli.order0_bound_ratio(b"aaaa") == float("inf")
    assert cli.first_divergence(b"abcd", b"abXd") == 2
    assert cli.first_divergence(b"abc", b"abcde") == 3
