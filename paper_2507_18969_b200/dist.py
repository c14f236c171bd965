"""Lane sharding of one container across GPUs.

Reference facts this follows: one model shared by all lanes and segments and
updated every step from the mean loss over all B lanes (`pipeline.py:136,196`,
`nn.py:206-209`, `model.py:265-281`); lanes are otherwise independent and
segments are contiguous lane ranges with their own coders (`pipeline.py:66-68`).

Partition: G ranks (G | 8, B % 8 == 0); rank r owns lanes [r*B/G, (r+1)*B/G)
= the 8/G consecutive lane groups of the canonical gradient reduction and the
segments inside them, their per-lane FDM state, coders and lane-matrix slice.
Sharded optimizer, per model step: each rank reduces its
groups' gradient partials to one subtree sum; the shared parameters are cut
into G slices (``shard_ranges``) and rank j's subtree sum of slice r goes to
rank r; rank r runs the top of the canonical tree over the G subtree sums and
Adam on its slice only; the updated weight slices are all-gathered.  (NCCL
send/recv + all-gather inside the library for one process per GPU;
stream-ordered peer copies for several contexts in one process.)  The tree is
the single-GPU one, so the trajectory -- and the container bytes -- do not
depend on G.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _lib
from .config import ModelConfig
from .container import EdpcContainer, Header
from .coder import CoderError
from .init import init_params_f32
from .lanes import lane_len_for, validate_geometry
from .model import DeviceContext

NUM_GROUPS = 8


def shard_ranges(n_shared: int, world: int) -> list[tuple[int, int]]:
    """[(offset, length)] of each rank's owned shared-parameter slice; mirrors
    ``shard_range`` in csrc/model.cu (64-aligned equal slices, last shorter)."""
    s = -(-n_shared // world)
    s = -(-s // 64) * 64
    out = []
    for r in range(world):
        o = min(n_shared, r * s)
        out.append((o, min(n_shared, (r + 1) * s) - o))
    return out


def tree_sum(parts):
    """Pairwise tree over 1/2/4/8 leaves, the order of ``tree_sum`` in
    csrc/kernels.cuh: 8 leaves -> ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7))."""
    if len(parts) == 1:
        return parts[0]
    h = len(parts) // 2
    return tree_sum(parts[:h]) + tree_sum(parts[h:])


def lane_plan(cfg: ModelConfig, segments: int, world: int) -> list[tuple[int, int]]:
    """[(lane_begin, lane_count)] per rank; raises ValueError if the geometry
    cannot be split on lane-group and segment boundaries."""
    validate_geometry(cfg, segments)
    B = cfg.lanes
    if world < 1 or NUM_GROUPS % world:
        raise ValueError(f"GPU count {world} must divide {NUM_GROUPS}")
    if world == 1:
        return [(0, B)]
    if B % NUM_GROUPS:
        raise ValueError(f"multi-GPU needs lanes ({B}) divisible by {NUM_GROUPS}")
    per = B // world
    spl = B // segments
    if per % spl:
        raise ValueError(f"segments of {spl} lanes straddle the {per}-lane GPU shares")
    return [(r * per, per) for r in range(world)]


def assemble(cfg: ModelConfig, n: int, shards: list[tuple[list[int], list[bytes]]],
             numerics: int = 0) -> EdpcContainer:
    """Container from per-rank (bit_lengths, payloads), rank order = segment order."""
    bits, pays = [], []
    for b, p in shards:
        bits += list(b)
        pays += list(p)
    return EdpcContainer(header=Header.from_config(cfg, n, bits, numerics), segments=pays)


def _split_payloads(bits, buf):
    out, pos = [], 0
    for b in bits:
        nb = (int(b) + 7) // 8
        out.append(bytes(buf[pos: pos + nb]))
        pos += nb
    return out


# ------------------------------------------------ single process, G contexts

class ShardSet:
    """G contexts (one per device in ``devices``; devices may repeat, e.g. to
    exercise the sharded path on one GPU) driven by one host thread."""

    def __init__(self, cfg: ModelConfig, segments: int, n: int, devices: list[int],
                 numerics: int | None = None):
        self.cfg = cfg
        self.plan = lane_plan(cfg, segments, len(devices))
        self.ctxs = []
        for d, (lb, lc) in zip(devices, self.plan):
            self.ctxs.append(DeviceContext(cfg, segments, n, d, lb, lc, numerics=numerics))
            numerics = self.ctxs[0].numerics_flags()  # every shard runs rank 0's numerics
        self.numerics = numerics
        params = init_params_f32(cfg)
        for c in self.ctxs:
            c.load_flat(params)
        self.lib = _lib.load()

    def close(self):
        for c in self.ctxs:
            c.close()

    def step(self, i: int, decompress: bool) -> None:
        lib = self.lib
        for c in self.ctxs:
            _lib.check(lib.edpc_step_phase(c.h, i, 0, int(decompress)))
        for dst in self.ctxs:
            for src in self.ctxs:
                if src is not dst:
                    _lib.check(lib.edpc_partials_pull(dst.h, src.h))
        for c in self.ctxs:
            _lib.check(lib.edpc_step_phase(c.h, i, 1, int(decompress)))
        for dst in self.ctxs:
            for src in self.ctxs:
                if src is not dst:
                    _lib.check(lib.edpc_weights_pull(dst.h, src.h))


# ------------------------------- one host thread per GPU, NCCL in the graphs

def nccl_available() -> bool:
    """True when the library can reach an NCCL (libnccl.so.2)."""
    buf = (ctypes.c_uint8 * 128)()
    return _lib.load().edpc_nccl_unique_id(buf, 128) == _lib.OK


def _use_nccl(devices: list[int]) -> bool:
    """Distinct GPUs (NCCL allows one rank per device) and an NCCL to load;
    contexts sharing a device (tests on one GPU) use stream-ordered peer
    copies (ShardSet) instead."""
    return len(set(devices)) == len(devices) and _lib.device_count() >= len(devices) and \
        nccl_available()


def _run_ranks(devices: list[int], fn) -> list:
    """fn(rank, device) on one host thread per device (each thread owns its
    context: the C ABI calls block only their own device's stream, and the
    NCCL collectives inside every rank's captured step graphs meet on the
    devices); exceptions are re-raised on the caller."""
    import threading
    out: list = [None] * len(devices)
    errs: list = []

    def run(r):
        try:
            out[r] = fn(r, devices[r])
        except BaseException as exc:
            errs.append(exc)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(len(devices))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


def _nccl_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _lib.check(_lib.load().edpc_nccl_unique_id(buf, 128))
    return bytes(buf)


def _join(ctx: DeviceContext, uid: bytes, world: int, rank: int) -> None:
    arr = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _lib.check(_lib.load().edpc_ctx_set_comm(ctx.h, arr, world, rank))


def _compress_nccl(data: bytes, cfg: ModelConfig, segments: int, devices: list[int],
                   chunk: int = 512) -> tuple[list, int]:
    """One context per GPU joined to an NCCL communicator; each rank's thread
    runs the same column blocks as the single-GPU pipeline (CUDA-graph model
    steps with the sharded optimizer's send/recv + all-gather captured inside)."""
    n = len(data)
    plan = lane_plan(cfg, segments, len(devices))
    uid = _nccl_id()
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    params = init_params_f32(cfg)
    spl = cfg.lanes // segments
    lib = _lib.load()

    def rank_fn(r, dev):
        lb, lc = plan[r]
        ctx = DeviceContext(cfg, segments, n, dev, lb, lc)
        try:
            ctx.load_flat(params)
            _join(ctx, uid, len(devices), r)
            L = ctx.lane_len
            for i0 in range(0, L, chunk):
                i1 = min(L, i0 + chunk)
                _lib.check(lib.edpc_set_input_columns(ctx.h, buf.ctypes.data, n, i0, i1))
                _lib.check(lib.edpc_compress_steps(ctx.h, i0, i1))
            bits = np.zeros(lc // spl, dtype=np.int64)
            tot = ctypes.c_int64()
            _lib.check(lib.edpc_compress_finish(ctx.h, bits.ctypes.data, ctypes.byref(tot)))
            pay = np.zeros(max(tot.value, 1), dtype=np.uint8)
            _lib.check(lib.edpc_get_payloads(ctx.h, pay.ctypes.data, pay.size))
            return bits.tolist(), _split_payloads(bits, pay), ctx.numerics_flags()
        finally:
            ctx.close()

    res = _run_ranks(devices, rank_fn)
    return [(b, p) for b, p, _ in res], res[0][2]


def _decompress_nccl(container: EdpcContainer, devices: list[int], chunk: int = 512) -> bytes:
    h = container.header
    cfg = h.model_config()
    n, segments = h.original_len, h.segment_count
    plan = lane_plan(cfg, segments, len(devices))
    uid = _nccl_id()
    params = init_params_f32(cfg)
    spl = cfg.lanes // segments
    lib = _lib.load()

    def rank_fn(r, dev):
        lb, lc = plan[r]
        ctx = DeviceContext(cfg, segments, n, dev, lb, lc, numerics=h.numerics)
        try:
            ctx.load_flat(params)
            _join(ctx, uid, len(devices), r)
            s0, s1 = lb // spl, (lb + lc) // spl
            pays = np.frombuffer(b"".join(container.segments[s0:s1]) or b"\0", dtype=np.uint8)
            bits = np.ascontiguousarray(h.bit_lengths[s0:s1], dtype=np.int64)
            _lib.check(lib.edpc_set_payloads(ctx.h, pays.ctypes.data, bits.ctypes.data))
            L = ctx.lane_len
            for i0 in range(0, L, chunk):
                _lib.check(lib.edpc_decompress_steps(ctx.h, i0, min(L, i0 + chunk)))
            out = np.empty(lc * L, dtype=np.uint8)
            st = lib.edpc_get_output(ctx.h, out.ctypes.data, out.size)
            if st == _lib.ERR_CODER:
                raise CoderError(lib.edpc_last_error().decode())
            _lib.check(st)
            return out
        finally:
            ctx.close()

    return np.concatenate(_run_ranks(devices, rank_fn))[:n].tobytes()


def compress_multi(data: bytes, cfg: ModelConfig, segments: int, devices: list[int], *,
                   stats: dict | None = None) -> EdpcContainer:
    t0 = time.perf_counter()
    n = len(data)
    if n == 0:
        return EdpcContainer(header=Header.from_config(cfg, 0, []), segments=[])
    for d in set(devices):
        _lib.require_device(d)
    lane_plan(cfg, segments, len(devices))  # geometry errors before any context
    if _use_nccl(list(devices)):
        shards, numerics = _compress_nccl(data, cfg, segments, list(devices))
        if stats is not None:
            stats.update(steps=max(0, lane_len_for(n, cfg.lanes) - cfg.context_len),
                         predict_s=0.0, train_s=0.0, encode_s=0.0, mode="nccl",
                         wall_s=time.perf_counter() - t0, peak_queue_depth=0,
                         devices=list(devices))
        return assemble(cfg, n, shards, numerics)
    ss = ShardSet(cfg, segments, n, list(devices))
    lib = ss.lib
    try:
        buf = np.frombuffer(bytes(data), dtype=np.uint8)
        T = cfg.context_len
        L = ss.ctxs[0].lane_len
        for c in ss.ctxs:
            _lib.check(lib.edpc_set_input(c.h, buf.ctypes.data, n, 0))
            _lib.check(lib.edpc_compress_steps(c.h, 0, min(T, L)))
        for i in range(T, L):
            ss.step(i, False)
            if (i + 1) % 256 == 0 or i + 1 == L:
                for c in ss.ctxs:
                    _lib.check(lib.edpc_encode_pending(c.h, i + 1))
        shards = []
        for c in ss.ctxs:
            sl = c.lane_count // (cfg.lanes // segments)
            bits = np.zeros(sl, dtype=np.int64)
            tot = ctypes.c_int64()
            _lib.check(lib.edpc_compress_finish(c.h, bits.ctypes.data, ctypes.byref(tot)))
            pay = np.zeros(max(tot.value, 1), dtype=np.uint8)
            _lib.check(lib.edpc_get_payloads(c.h, pay.ctypes.data, pay.size))
            shards.append((bits.tolist(), _split_payloads(bits, pay)))
        numerics = ss.numerics
    finally:
        ss.close()
    if stats is not None:
        stats.update(steps=max(0, L - T), predict_s=0.0, train_s=0.0, encode_s=0.0,
                     wall_s=time.perf_counter() - t0, peak_queue_depth=0, devices=list(devices))
    return assemble(cfg, n, shards, numerics)


def decompress_multi(container: EdpcContainer, devices: list[int], *,
                     stats: dict | None = None) -> bytes:
    t0 = time.perf_counter()
    h = container.header
    cfg = h.model_config()
    n = h.original_len
    segments = h.segment_count
    for d in set(devices):
        _lib.require_device(d)
    if _use_nccl(list(devices)):
        out = _decompress_nccl(container, list(devices))
        if stats is not None:
            stats.update(steps=max(0, lane_len_for(n, cfg.lanes) - cfg.context_len), mode="nccl",
                         wall_s=time.perf_counter() - t0, devices=list(devices))
        return out
    ss = ShardSet(cfg, segments, n, list(devices), numerics=h.numerics)
    lib = ss.lib
    try:
        spl = cfg.lanes // segments
        T = cfg.context_len
        L = ss.ctxs[0].lane_len
        for c, (lb, lc) in zip(ss.ctxs, ss.plan):
            s0, s1 = lb // spl, (lb + lc) // spl
            pays = b"".join(container.segments[s0:s1]) or b"\0"
            bits = np.ascontiguousarray(h.bit_lengths[s0:s1], dtype=np.int64)
            pb = np.frombuffer(pays, dtype=np.uint8)
            _lib.check(lib.edpc_set_payloads(c.h, pb.ctypes.data, bits.ctypes.data))
            _lib.check(lib.edpc_decompress_steps(c.h, 0, min(T, L)))
        for i in range(T, L):
            ss.step(i, True)
        parts = []
        for c in ss.ctxs:
            out = np.empty(c.lane_count * L, dtype=np.uint8)
            st = lib.edpc_get_output(c.h, out.ctypes.data, out.size)
            if st == _lib.ERR_CODER:
                raise CoderError(lib.edpc_last_error().decode())
            _lib.check(st)
            parts.append(out)
    finally:
        ss.close()
    if stats is not None:
        stats.update(steps=max(0, L - T), wall_s=time.perf_counter() - t0, devices=list(devices))
    return np.concatenate(parts)[:n].tobytes()


# ------------------------------------------- one process per GPU (torchrun)

def nccl_join(ctx: DeviceContext, rank: int, world: int, broadcast_id) -> None:
    """Joins ``ctx`` to an NCCL communicator; ``broadcast_id(bytes|None)``
    returns rank 0's 128-byte id on every rank (torch.distributed object
    broadcast under torchrun)."""
    lib = _lib.load()
    uid = None
    if rank == 0:
        buf = (ctypes.c_uint8 * 128)()
        _lib.check(lib.edpc_nccl_unique_id(buf, 128))
        uid = bytes(buf)
    uid = broadcast_id(uid)
    arr = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _lib.check(lib.edpc_ctx_set_comm(ctx.h, arr, world, rank))


def torch_broadcast_id(uid):
    import torch.distributed as dist
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def bench_multi(args, wl, clocks_cls=None, peaks=None, flops_per_lane=None) -> None:
    """bench.py at N GPUs under torchrun: the workload as defined (C3: fixed
    B, S and stream; per-GPU lanes B/G; identical container bytes at every G),
    the sharded optimizer's two NCCL exchanges per model step inside the
    captured step graph; the step time is the max over ranks of CUDA-event
    time."""
    import json

    import torch
    import torch.distributed as dist

    from . import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    # the workload as defined (C3: fixed B = 32768 lanes, S = 1024 segments,
    # 1 GiB): rank r runs lanes [r B/G, (r+1) B/G) -- per-GPU M = B/G -- and the
    # container bytes are the same at every G (strong scaling)
    cfg = ModelConfig(**wl["model"], lanes=wl["lanes"])
    S = wl["segments"]
    n = wl["nbytes"]
    plan = lane_plan(cfg, S, world)
    lb, lc = plan[rank]
    T = cfg.context_len
    chunk, K, W = args.chunk, args.steps, args.warmup
    L = lane_len_for(n, cfg.lanes)
    stream = np.frombuffer(synth.generate(wl["kind"], n, wl["seed"]), dtype=np.uint8)
    ctx = DeviceContext(cfg, S, n, local, lb, lc)
    ctx.load_flat(init_params_f32(cfg))
    numerics = ctx.numerics()
    _lib.check(lib.edpc_set_input(ctx.h, stream.ctypes.data, n, 0))  # this rank's lane slice
    nccl_join(ctx, rank, world, torch_broadcast_id)
    _lib.check(lib.edpc_compress_steps(ctx.h, 0, T))
    col = T
    for _ in range(W):
        _lib.check(lib.edpc_compress_steps(ctx.h, col, col + chunk))
        col += chunk
    _lib.check(lib.edpc_sync(ctx.h))
    dist.barrier()
    torch.cuda.synchronize()
    import contextlib
    sampler = clocks_cls(local) if (clocks_cls and rank == 0) else contextlib.nullcontext()
    with sampler as clk:
        _lib.check(lib.edpc_timer(ctx.h, 0, None))
        for k in range(K):
            _lib.check(lib.edpc_compress_steps(ctx.h, col, col + chunk))
            col += chunk
        _lib.check(lib.edpc_timer(ctx.h, 1, None))
        ms = ctypes.c_double()
        _lib.check(lib.edpc_timer(ctx.h, 2, ctypes.byref(ms)))
    clocks = getattr(clk, "result", None) if clk is not None else None
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([ms.value], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_bytes = cfg.lanes * chunk * K  # all ranks' lanes
    if rank == 0:
        dtype = ("fp16+tf32" if numerics["fp16_mbrb"] else "tf32") if numerics["tcgen05"] else "fp32"
        roof = None
        if peaks and flops_per_lane:
            # whole-step rate per GPU (this path has no per-kernel breakdown)
            fl = flops_per_lane(wl["model"]) * lc * chunk * K
            ach = fl / (ms_max / 1e3) / 1e12
            pk = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
            roof = dict(bound="tensor", kernel="whole model step per GPU (all kernels)",
                        achieved=ach, peak=pk, unit="TFLOP/s", frac=ach / pk, traffic=None)
        line = dict(metric="compress/decompress MB/s at 1/2/4/8 B200 + bits/byte vs CPU ref",
                    value=total_bytes / (ms_max / 1e3) / 1e6, unit="MB/s", n_gpus=world,
                    steps=K, warmup=W, ms_per_step=ms_max / K, higher_is_better=True,
                    scaling="strong", vs_baseline=None, numerics=numerics, clocks=clocks,
                    roofline=roof, cpu_baseline=None,
                    e2e=None, e2e_note="multi-GPU lines time the device-resident loop only",
                    dtype=dtype, data=f"synthetic {wl['kind']}-like (PCG64 seed {wl['seed']})",
                    config=dict(workload=f"{wl['desc']}; {world} GPUs: B={cfg.lanes}, S={S}, "
                                         f"{n >> 20} MiB, {lc} lanes per GPU (strong scaling)",
                                lanes=cfg.lanes, segments=S,
                                lanes_per_gpu=lc, columns_per_step=chunk,
                                exchange="sharded optimizer per model step, inside the step "
                                         "graph: NCCL send/recv of subtree-sum slices "
                                         "((G-1)/G x 19.3 MB out per GPU), G-leaf tree + Adam on "
                                         "the owned slice, NCCL all-gather of the updated fp32 "
                                         "weights + fp16 shadow"))
        print(json.dumps(line), flush=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
