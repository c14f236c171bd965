"""Multi-rank host logic on CPU (gloo, world size 2): id broadcast, lane plan,
container assembly order, and the G-invariance of the sharded optimizer's
reduction (subtree sums, slice exchange, owner-side tree, all-gather ==
single-process 8-leaf tree, bit for bit)."""
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


def _sharded_step(rank, world, full):
    """The sharded optimizer's exchange exactly as the library runs it, over
    gloo: subtree sum of the rank's groups, slice r of every rank's subtree sum
    to rank r (send/recv), G-leaf tree on the owned slice, all-gather of the
    owned slices.  Returns the full reduced gradient on this rank."""
    import torch
    gc = 8 // world
    n = full.shape[1]
    sub = edist.tree_sum([full[g] for g in range(rank * gc, rank * gc + gc)])
    ranges = edist.shard_ranges(n, world)
    o, ln = ranges[rank]
    leaves = [None] * world
    leaves[rank] = torch.from_numpy(sub[o:o + ln].copy())
    reqs = []
    for j in range(world):
        if j == rank:
            continue
        jo, jl = ranges[j]
        reqs.append(dist.isend(torch.from_numpy(sub[jo:jo + jl].copy()), j))
        leaves[j] = torch.empty(ln, dtype=torch.float32)
        reqs.append(dist.irecv(leaves[j], j))
    for r in reqs:
        r.wait()
    mine = edist.tree_sum([x.numpy() for x in leaves])
    s = max(l for _, l in ranges)
    pad = torch.zeros(s, dtype=torch.float32)
    pad[:ln] = torch.from_numpy(mine)
    bufs = [torch.empty(s, dtype=torch.float32) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return np.concatenate([bufs[j].numpy()[:ranges[j][1]] for j in range(world)])


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
        # 3. the sharded optimizer's exchange == the single-context tree, bit
        #    for bit (n not a multiple of the 64-aligned slice: ragged last slice)
        rng = np.random.default_rng(1234)
        full = rng.normal(size=(8, 1000)).astype(np.float32) * 1e3
        sharded = _sharded_step(rank, world, full)
        q.put((rank, got == bytes(range(128)), plan, sharded.tobytes(), _tree(full).tobytes()))
    finally:
        dist.destroy_process_group()


def test_tree_sum_matches_canonical_order_and_subtrees():
    rng = np.random.default_rng(7)
    p = list(rng.normal(size=(8, 4096)).astype(np.float32) * 1e4)
    ref = _tree(p)
    assert edist.tree_sum(p).tobytes() == ref.tobytes()
    for world in (1, 2, 4, 8):
        gc = 8 // world
        subs = [edist.tree_sum(p[r * gc:(r + 1) * gc]) for r in range(world)]
        assert edist.tree_sum(subs).tobytes() == ref.tobytes()


@pytest.mark.parametrize("n,world", [(4835392, 8), (4835392, 2), (1000, 8), (100, 8), (5, 4)])
def test_shard_ranges_partition_the_parameters(n, world):
    r = edist.shard_ranges(n, world)
    assert len(r) == world
    pos = 0
    for o, ln in r:
        assert o == pos and ln >= 0
        pos += ln
    assert pos == n
    s = -(-(-(-n // world)) // 64) * 64
    assert all(o % 64 == 0 or ln == 0 for o, ln in r)
    assert world * s - n < 8 * 64  # fits the library's kShardPad padding


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
