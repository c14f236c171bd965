#!/usr/bin/env python
"""EDPC hot-path benchmark on B200 (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c4a|c4b|c3|c5] [--chunk COLS]

Workload (default ``c2``, BASELINE.json configs[1]): 64 MiB synthetic
text-like stream (PCG64 seed 0), the reference default model (t16 d_e16
h2048/4096 r4 k2), B=4096 lanes, S=256 segments.  A bench *step* is
``--chunk`` autoregressive lane columns (default 32) = B*chunk input bytes
of predict -> quantize -> encode -> backward -> Adam.

* ``value``     compress MB/s (10^6 input bytes / s), lane matrix resident in
                HBM, device-timed with CUDA events on the library's stream
                (the encoder stream is joined before the stop event).
* ``decompress_MBps``  the mirrored decode loop on the same columns (output
                verified bit-exact against the input).
* ``e2e``       the whole stream through the public API: ``compress(bytes)``
                + ``write_container`` (context setup, parameter upload,
                streaming H2D of the lane columns, graph-replayed steps, device
                payload assembly, payload D2H); ``full_stream_*`` adds the
                full ``decompress`` and its lossless check.
* ``bits_per_byte`` / ``ref_bits_per_byte``: the full C2-mini stream (4 MiB,
                same B/S/dims) compressed end to end by the public API vs the
                unmodified reference's run of the same stream
                (tests/golden/ref_ratio_c2mini_text_4m.json).
* ``roofline``  dominant kernel class (the per-step GEMMs): algorithmic
                FLOPs (6*(kF h_l + h_l F + 2F F' + kF h_g + h_g F
                + 256F) per lane-step) / CUDA-event time of those launches,
                against the FLOP-weighted peak of the numerics the context
                runs (kind::f16 MBRB GEMMs at the measured dense bf16/fp16
                rate, kind::tf32 LTE/head GEMMs at half of it); ``traffic`` is
                the GEMMs' DRAM bytes per model step from the committed ncu
                capture (profiles/r02_gemm_traffic.json).
* ``cpu_baseline`` the CPU oracle (numpy fp64 + C coder, restating the
                reference) step-sampled at the same B and dims on this host.

``--impl reference`` times that CPU implementation alone (rank 0) and prints
the same metric with "impl": "reference".
Working set per step (weights, Adam state, 4096 per-lane FDMs, activations)
is ~1 GB > 126 MB L2, so no explicit L2 flush is needed between steps.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER = dict(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lte_ratio=4,
             branches=2)
WORKLOADS = {
    "c2": dict(kind="text", nbytes=64 << 20, seed=0, lanes=4096, segments=256, model=PAPER,
               desc="C2: 64 MiB text-like stream, default EDPC (2-branch MBRB + LTE), B=4096, S=256"),
    "c4a": dict(kind="text", nbytes=64 << 20, seed=0, lanes=4096, segments=256,
                model=dict(PAPER, branches=1), desc="C4a: as C2 with single-branch MBRB"),
    "c4b": dict(kind="text", nbytes=64 << 20, seed=0, lanes=4096, segments=256,
                model=dict(PAPER, lte_ratio=1), desc="C4b: as C2 with full-width LTE (F'=F)"),
    "c3": dict(kind="mixed", nbytes=1 << 30, seed=0, lanes=32768, segments=1024, model=PAPER,
               desc="C3: 1 GiB mixed text/image stream, B=32768, S=1024 (lanes sharded over GPUs)"),
    "c5": dict(kind="mixed", nbytes=1 << 30, seed=0, lanes=32768, segments=1024,
               model=dict(PAPER, context_len=32, hidden_local=4096, hidden_global=8192),
               desc="C5: scaled EDPC (t=32, F=512, F'=128, h 4096/8192), 1 GiB mixed stream, "
                    "B=32768, S=1024, online adaptation (lanes sharded over GPUs)"),
}
METRIC = "compress/decompress MB/s at 1/2/4/8 B200 + bits/byte vs CPU ref"


_T0 = time.perf_counter()


def note(msg: str) -> None:
    """Progress on stderr (stdout carries only the JSON line)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def gemm_flops_per_lane(m) -> float:
    F = m["context_len"] * m["embed_dim"]
    Fp = F // m["lte_ratio"]
    k, hl, hg = m["branches"], m["hidden_local"], m["hidden_global"]
    return 6.0 * (k * F * hl + hl * F + 2 * F * Fp + k * F * hg + hg * F + 256 * F)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "25"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.p is None:
            return
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if sm:
            self.result = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                           "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------- CPU oracle

def cpu_sample(wl, min_seconds: float, max_steps: int, warm: int = 1, exact: bool = False,
               blas_threads: int | None = None):
    """Step-sampled CPU oracle at the workload's exact (B, dims).  BLAS runs on
    all host cores by default -- a non-default override: the reference pins
    OpenBLAS to one thread (`__init__.py:15-22`); blas_threads=1 restores that."""
    if blas_threads is not None:
        import threadpoolctl
        with threadpoolctl.threadpool_limits(blas_threads):
            return cpu_sample(wl, min_seconds, max_steps, warm, exact)
    from oracle import coder as oc
    from oracle.model import OracleModel
    from paper_2507_18969_b200.config import ModelConfig
    from paper_2507_18969_b200 import synth
    cfg = ModelConfig(**wl["model"], lanes=wl["lanes"])
    B, T, S = cfg.lanes, cfg.context_len, wl["segments"]
    nb = min(wl["nbytes"], B * (T + warm + max_steps + 1))
    data = synth.generate(wl["kind"], B * ((nb + B - 1) // B), wl["seed"])
    mat = np.frombuffer(data, np.uint8).reshape(B, -1)
    model = OracleModel(cfg)
    encs = [oc.ArithmeticEncoder() for _ in range(S)]
    spl = B // S

    def step(i):
        probs, cache = model.predict(mat[:, i - T: i])
        _, cums = oc.quantize_rows(probs)
        for s in range(S):
            encs[s].encode_rows(cums[s * spl:(s + 1) * spl], mat[s * spl:(s + 1) * spl, i])
        model.train_step(cache, mat[:, i])

    i = T
    for _ in range(warm):
        step(i)
        i += 1
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (n < 2 or exact or time.perf_counter() - t0 < min_seconds):
        step(i)
        i += 1
        n += 1
    dt = time.perf_counter() - t0
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        cores = max([d.get("num_threads", 1) for d in info] + [1])
    except Exception:
        cores = os.cpu_count() or 1
    return dict(value=B * n / dt / 1e6, unit="MB/s", cores=int(cores), kind="port",
                sample=f"{n} model steps x {B} lanes ({wl['desc']}), fp64 numpy/OpenBLAS + C coder,"
                       f" after {warm} warm-up step; {dt:.1f} s",
                seconds_per_step=dt / n, blas_threads=int(cores),
                blas_note="reference default" if cores == 1 else
                "non-default override: the reference pins BLAS to 1 thread (__init__.py:15-22)")


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B = wl["lanes"]
    # a bounded sample: up to --steps model steps, stopping after ~60 s
    r = cpu_sample(wl, min_seconds=60.0, max_steps=args.steps, warm=min(args.warmup, 1))
    r1 = cpu_sample(wl, min_seconds=0.0, max_steps=min(args.steps, 2), blas_threads=1)
    # treat each model step as one bench step (a bounded sample of the workload)
    line = dict(metric=METRIC, value=r["value"], unit="MB/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=r["seconds_per_step"] * 1e3,
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic", impl="reference",
                config=dict(workload=wl["desc"], lanes=B, segments=wl["segments"],
                            columns_per_step=1),
                cpu_baseline=dict(value=r["value"], unit="MB/s", cores=r["cores"], kind="port",
                                  sample=r["sample"], blas_note=r["blas_note"],
                                  one_thread=dict(value=r1["value"], cores=1, sample=r1["sample"],
                                                  blas_note=r1["blas_note"])),
                e2e=dict(value=r["value"], unit="MB/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- GPU arm

def run_ours(args, wl):
    from paper_2507_18969_b200 import _lib, synth
    from paper_2507_18969_b200.config import ModelConfig
    from paper_2507_18969_b200.init import init_params_f32
    from paper_2507_18969_b200.model import DeviceContext

    world = int(os.environ.get("WORLD_SIZE", "1"))
    # EDPC_BENCH_MULTI=1: the torchrun/NCCL path even at one rank (smoke test)
    if world > 1 or args.gpus > 1 or os.environ.get("EDPC_BENCH_MULTI") == "1":
        from paper_2507_18969_b200.dist import bench_multi
        return bench_multi(args, wl, clocks_cls=Clocks, peaks=peaks()[0],
                           flops_per_lane=gemm_flops_per_lane)
    lib = _lib.load()
    _lib.require_device(0)
    cfg = ModelConfig(**wl["model"], lanes=wl["lanes"])
    B, S, T = cfg.lanes, wl["segments"], cfg.context_len
    data = synth.generate(wl["kind"], wl["nbytes"], wl["seed"])
    n = len(data)
    buf = np.frombuffer(data, np.uint8)
    chunk, K, W = args.chunk, args.steps, args.warmup
    KP = max(2, min(K, 4))  # profiled bench steps (eager, per-kernel events)
    C = T + (W + K + KP) * chunk
    params = init_params_f32(cfg)

    def timed_loop(ctx, fn, nsteps, prof):
        """Device-timed loop on the library stream.  prof=False: CUDA graphs,
        no per-kernel events (the headline number); prof=True: eager launches
        with per-region CUDA events (breakdown, launch count, roofline)."""
        _lib.check(lib.edpc_prof(ctx.h, 1 if prof else 0))
        _lib.check(lib.edpc_timer(ctx.h, 0, None))
        for k in range(nsteps):
            fn(k)
        _lib.check(lib.edpc_timer(ctx.h, 1, None))
        ms = ctypes.c_double()
        _lib.check(lib.edpc_timer(ctx.h, 2, ctypes.byref(ms)))
        regions = {}
        for r, name in enumerate(_lib.REGIONS):
            t, c = ctypes.c_double(), ctypes.c_int64()
            _lib.check(lib.edpc_prof_read(ctx.h, r, ctypes.byref(t), ctypes.byref(c)))
            regions[name] = (t.value, c.value)
        t, c = ctypes.c_double(), ctypes.c_int64()
        _lib.check(lib.edpc_prof_read(ctx.h, -1, ctypes.byref(t), ctypes.byref(c)))
        _lib.check(lib.edpc_prof(ctx.h, 0))
        return ms.value, regions, c.value

    # ---- compress (device-resident input)
    note("compress loop")
    ctx = DeviceContext(cfg, S, n, 0)
    ctx.load_flat(params)
    numerics = ctx.numerics()
    _lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, n, 0))
    col = 0
    _lib.check(lib.edpc_compress_steps(ctx.h, 0, T))
    col = T
    for _ in range(W):
        _lib.check(lib.edpc_compress_steps(ctx.h, col, col + chunk))
        col += chunk
    _lib.check(lib.edpc_sync(ctx.h))
    start = col

    def comp_step(k):
        c0 = start + k * chunk
        _lib.check(lib.edpc_compress_steps(ctx.h, c0, c0 + chunk))

    with Clocks(0) as clk:
        c_ms, _, _ = timed_loop(ctx, comp_step, K, False)
    clocks = clk.result
    p_ms, c_regions, launches = timed_loop(ctx, lambda k: comp_step(K + k), KP, True)
    bits = np.zeros(S, dtype=np.int64)
    tot = ctypes.c_int64()
    _lib.check(lib.edpc_compress_finish(ctx.h, bits.ctypes.data, ctypes.byref(tot)))
    pay = np.zeros(max(tot.value, 1), dtype=np.uint8)
    _lib.check(lib.edpc_get_payloads(ctx.h, pay.ctypes.data, pay.size))
    ctx.close()
    region_bpb = 8.0 * tot.value / (B * C)

    # ---- decompress the same columns
    note("decompress loop")
    dctx = DeviceContext(cfg, S, n, 0)
    dctx.load_flat(params)
    _lib.check(lib.edpc_set_payloads(dctx.h, pay.ctypes.data, bits.ctypes.data))
    _lib.check(lib.edpc_decompress_steps(dctx.h, 0, start))
    _lib.check(lib.edpc_sync(dctx.h))

    def dec_step(k):
        c0 = start + k * chunk
        _lib.check(lib.edpc_decompress_steps(dctx.h, c0, c0 + chunk))

    d_ms, _, _ = timed_loop(dctx, dec_step, K, False)
    dp_ms, d_regions, d_launches = timed_loop(dctx, lambda k: dec_step(K + k), KP, True)
    got = np.empty((B, C), dtype=np.uint8)
    _lib.check(lib.edpc_get_columns(dctx.h, 0, C, got.ctypes.data))
    L = dctx.lane_len
    want = np.zeros(B * L, dtype=np.uint8)
    want[:n] = buf
    lossless = bool(np.array_equal(got, want.reshape(B, L)[:, :C]))
    dctx.close()

    # ---- e2e: the whole stream through the public API (host bytes in,
    note("full-stream e2e")
    # container bytes out): context setup, parameter upload, streaming column
    # H2D, graph-replayed model steps, device payload assembly + D2H, container
    # write; then the full decompress, checked lossless
    e2e, full = None, {}
    if not args.no_e2e:
        from paper_2507_18969_b200 import compress, decompress, read_container, write_container
        e_n = min(n, args.e2e_bytes) if args.e2e_bytes else n
        stream = bytes(data[:e_n])
        cstats: dict = {}
        t0 = time.perf_counter()
        blob = write_container(compress(stream, cfg, S, stats=cstats))
        ce_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        back = decompress(read_container(blob))
        de_s = time.perf_counter() - t0
        ok = back == stream
        e2e = dict(value=e_n / ce_s / 1e6, unit="MB/s", h2d_bytes_per_step=e_n,
                   d2h_bytes_per_step=len(blob), steps=1,
                   path="public compress(bytes) -> write_container of the whole "
                        f"{e_n >> 20} MiB stream (one step = the stream): context setup, "
                        "parameter upload, streaming column H2D, CUDA-graph model steps, "
                        "device-side payload assembly, one payload D2H, container write; "
                        "context buffers from the device memory pool the preceding bench "
                        "phases warmed (a long-lived process; the first call in a fresh "
                        "process adds ~1 s of CUDA/pool start-up)")
        full = dict(full_stream_bytes=e_n, full_stream_compress_MBps=e_n / ce_s / 1e6,
                    full_stream_decompress_MBps=e_n / de_s / 1e6, full_stream_lossless=ok,
                    full_stream_bits_per_byte=8.0 * len(blob) / e_n,
                    full_stream_compress_s=ce_s, full_stream_decompress_s=de_s,
                    full_stream_compress_breakdown_s={k: round(cstats[k], 4) for k in
                                                      ("setup_s", "device_loop_s", "encode_s",
                                                       "finish_s", "payload_d2h_s", "close_s")
                                                      if k in cstats})

    # ---- bits/byte vs the reference's own run of the C2-mini stream
    note("ratio")
    ratio = {}
    if not args.no_ratio and wl is WORKLOADS["c2"]:
        from paper_2507_18969_b200 import compress, write_container
        refp = os.path.join(ROOT, "tests", "golden", "ref_ratio_c2mini_text_4m.json")
        mini = synth.generate("text", 4 << 20, 0)
        t0 = time.perf_counter()
        blob = write_container(compress(mini, cfg, S))
        api_s = time.perf_counter() - t0
        ratio = dict(bits_per_byte=8.0 * len(blob) / len(mini), api_compress_s_4MiB=api_s)
        if os.path.exists(refp):
            ref = json.load(open(refp))
            ratio["ref_bits_per_byte"] = ref["bits_per_byte"]
            ratio["ratio_delta_vs_ref"] = (len(mini) / len(blob)) / ref["ratio"] - 1.0

    # ---- CPU baseline (bounded sample, rank 0, N=1)
    note("cpu baseline")
    cpu = None
    if not args.no_cpu:
        r = cpu_sample(wl, min_seconds=args.cpu_seconds, max_steps=20)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "blas_note")}
        r1 = cpu_sample(wl, min_seconds=0.0, max_steps=2, blas_threads=1)
        cpu["one_thread"] = {k: r1[k] for k in ("value", "cores", "sample", "blas_note")}

    pk, pk_src = peaks()
    tc, f16 = numerics["tcgen05"], numerics["fp16_mbrb"]
    fl_step = gemm_flops_per_lane(wl["model"]) * B  # per model step (lane column)
    steps_total = KP * chunk  # model steps in the profiled pass
    g_ms, g_n = c_regions["gemm"]
    achieved = fl_step * steps_total / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
    peak_16 = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))  # dense fp16 = bf16 rate
    # mixed peak: the MBRB GEMMs run kind::f16 (fp16 operands), the LTE / head
    # GEMMs kind::tf32 at half that rate -> t_min = sum_phase FLOP / peak
    fl_tf32 = gemm_flops_per_lane(dict(wl["model"], hidden_local=0, hidden_global=0)) * B
    if f16:
        peak_t = fl_step / ((fl_step - fl_tf32) / peak_16 + fl_tf32 / (peak_16 / 2))
        gemm_kind = "tcgen05 kind::f16 (MBRB branch/out-proj) + kind::tf32 (LTE, head)"
        dtype = "fp16+tf32"
    elif tc:
        peak_t, gemm_kind, dtype = peak_16 / 2, "tcgen05 kind::tf32", "tf32"
    else:
        peak_t, gemm_kind, dtype = peak_16 / 2, "SIMT fp32", "fp32"
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "r02_gemm_traffic.json")
    if not os.path.exists(tp):
        tp = os.path.join(ROOT, "profiles", "r01_gemm_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        traffic, traffic_src = tj["gemm_dram_bytes_per_step"], tj.get("source", tp)
    m = wl["model"]
    F = m["context_len"] * m["embed_dim"]
    Fp = F // m["lte_ratio"]
    fdm_bytes = B * Fp * Fp * 4 * 6.0
    kernels = {}
    for name, (t, c) in c_regions.items():
        kernels[name] = dict(ms_per_step=t / steps_total, launches_per_step=c / steps_total,
                             share=t / max(sum(v[0] for v in c_regions.values()), 1e-9))
    f_ms = c_regions["fdm_bwd_adam"][0]
    if f_ms > 0:
        gbs = fdm_bytes * steps_total / (f_ms / 1e3) / 1e9
        kernels["fdm_bwd_adam"].update(algorithmic_bytes=fdm_bytes, achieved_GBps=gbs,
                                       frac_hbm=gbs / pk["hbm_gbs"])
    line = dict(
        metric=METRIC, value=B * chunk * K / (c_ms / 1e3) / 1e6, unit="MB/s", n_gpus=1,
        steps=K, warmup=W, ms_per_step=c_ms / K, higher_is_better=True, scaling="weak",
        vs_baseline=None, dtype=dtype, data=f"synthetic {wl['kind']}-like (PCG64 seed {wl['seed']},"
                                              f" sha256 {synth.sha256(data)[:16]})",
        config=dict(workload=wl["desc"], lanes=B, segments=S, columns_per_step=chunk,
                    bytes_per_step=B * chunk, model=wl["model"],
                    l2="no flush: per-step working set ~1 GB > 126 MB L2"),
        decompress_MBps=B * chunk * K / (d_ms / 1e3) / 1e6, lossless_region=lossless,
        region_bits_per_byte=region_bpb, **ratio, **full,
        roofline=dict(bound="tensor",
                      kernel=f"per-step GEMMs ({gemm_kind})",
                      achieved=achieved,
                      peak=peak_t, unit="TFLOP/s", frac=achieved / peak_t, traffic=traffic,
                      peak_source=f"{pk_src} bf16 dense sustained ({peak_16} TFLOP/s) = fp16 rate;"
                                  f" tf32 at half; weighted by the FLOP mix",
                      traffic_unit="DRAM bytes per model step, all GEMM launches",
                      traffic_source=traffic_src, frac_vs_fp16_peak=achieved / peak_16,
                      flops_per_step=fl_step, gemm_ms_per_model_step=g_ms / steps_total),
        kernels=kernels, kernels_note=f"per-region CUDA events over {KP} extra eager bench steps "
                                      f"({steps_total} model steps); eager ms/step {p_ms / KP:.2f} vs "
                                      f"graph ms/step {c_ms / K:.2f}",
        decode_kernels={k: dict(ms_per_step=v[0] / steps_total) for k, v in d_regions.items() if v[0]},
        cpu_baseline=cpu, e2e=e2e, gpu_launches=int(launches * K // KP),
        clocks=clocks, numerics=numerics)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c2 on one GPU, c3 (the multi-GPU config) on N > 1")
    ap.add_argument("--chunk", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-bytes", type=int, default=None,
                    help="e2e / full-stream leg on this prefix of the stream (default: all)")
    ap.add_argument("--no-ratio", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if args.workload is None:
        multi = args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1
        args.workload = "c3" if multi else "c2"
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
