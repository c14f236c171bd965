"""Multi-rank host logic on CPU (gloo, world size 2): id broadcast, lane plan,
container assembly order, and the G-invariance of the canonical reduction
(all-gather of lane-group partials + fixed tree == single-process tree)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_18969_b200 import dist as edist
from paper_2507_18969_b200.config import ModelConfig
from paper_2507_18969_b200.container import read_container, write_container


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tree(p):
    return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. rank 0's NCCL-style 128-byte id reaches every rank unchanged
        uid = bytes(range(128)) if rank == 0 else None
        got = edist.torch_broadcast_id(uid)
        # 2. lane plan: rank r owns groups [4r, 4r+4) of 8
        cfg = ModelConfig(context_len=4, embed_dim=4, hidden_local=8, hidden_global=8,
                          lte_ratio=2, lanes=64)
        plan = edist.lane_plan(cfg, 16, world)
        # 3. each rank's partials for its own groups, all-gathered, then the tree
        rng = np.random.default_rng(1234)
        full = rng.normal(size=(8, 1000)).astype(np.float32) * 1e3
        import torch
        mine = torch.from_numpy(full[4 * rank: 4 * rank + 4].copy())
        bufs = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(bufs, mine)
        gathered = torch.cat(bufs).numpy()
        q.put((rank, got == bytes(range(128)), plan, _tree(gathered).tobytes(),
               _tree(full).tobytes()))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_and_plan():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, id_ok, plan, tree_dist, tree_single in res:
        assert id_ok
        assert plan == [(0, 32), (32, 32)]
        assert tree_dist == tree_single  # bit-identical: G-invariant reduction


def test_assemble_orders_segments_by_rank():
    cfg = ModelConfig(context_len=4, embed_dim=4, hidden_local=8, hidden_global=8,
                      lte_ratio=2, lanes=8)
    c = edist.assemble(cfg, 100, [([9, 17], [b"\x01\x80", b"\x02\x03\x80"]),
                                  ([8, 1], [b"\x04", b"\x80"])])
    assert c.header.bit_lengths == [9, 17, 8, 1]
    assert read_container(write_container(c)).segments == [b"\x01\x80", b"\x02\x03\x80", b"\x04", b"\x80"]
