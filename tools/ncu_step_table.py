"""ncu per-kernel CSV -> markdown table (profiling helper, not collected).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none \
        -k regex:'^(?!k_boot)' --csv --log-file X.csv python tools/prof_step.py 4096 1
    python tools/ncu_step_table.py X.csv "title" profiles/rNN_gemm_traffic.json > profiles/rNN_step_kernels.md

Takes the LAST model step's launches (from the last k_embed_ln<1> on).
"""
import csv
import re
import sys
from collections import OrderedDict

M_T = "gpu__time_duration.sum"
M_R = "dram__bytes_read.sum"
M_W = "dram__bytes_write.sum"
M_TC = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
M_L2 = "lts__throughput.avg.pct_of_peak_sustained_elapsed"


def main(path, title):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    k = OrderedDict()
    for r in rd:
        key = int(r["ID"])
        e = k.setdefault(key, {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        v = r["Metric Value"].replace(",", "")
        unit = r["Metric Unit"]
        try:
            x = float(v)
        except ValueError:
            continue
        if r["Metric Name"] in (M_R, M_W):
            x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if r["Metric Name"] == M_T:
            x *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        e[r["Metric Name"]] = x
    ks = list(k.values())
    start = max(i for i, e in enumerate(ks) if e["name"].startswith("void k_embed_ln<1>"))
    ks = ks[start:]
    print(f"# {title}\n")
    print("| kernel | grid | us | DRAM read MB | DRAM write MB | tensor % | L2 % |")
    print("|---|---|---|---|---|---|---|")
    tot = gt = gb = 0.0
    for e in ks:
        name = re.sub(r"\(.*", "", e["name"]).replace("edpc::", "")
        name = re.sub(r"^void ", "", name)
        t = e.get(M_T, 0) / 1e3
        rb, wb = e.get(M_R, 0) / 1e6, e.get(M_W, 0) / 1e6
        if name.startswith("k_encode"):  # the coder's own stream, overlapped with the step
            print(f"| {name} (encoder stream, not in the total) | {e['grid']} | {t:.1f} | | | | |")
            continue
        tot += t
        if "k_tc_gemm" in name or "k_mbrb_" in name or "k_wgrad_" in name:
            gt += t
            gb += rb + wb
        print(f"| {name} | {e['grid']} | {t:.1f} | {rb:.1f} | {wb:.1f} | "
              f"{e.get(M_TC, 0):.1f} | {e.get(M_L2, 0):.1f} |")
    print(f"| **total** | | {tot:.1f} | | | | |")
    print(f"\ntcgen05 GEMM kernels (k_tc_gemm, fused k_mbrb_*, k_wgrad_*): {gt:.1f} us of {tot:.1f} us;"
          f" their DRAM traffic {gb:.1f} MB per step.")
    return dict(gemm_dram_bytes_per_step=gb * 1e6, gemm_us_per_step_serialized=gt,
                step_us_serialized=tot, source=path)


if __name__ == "__main__":
    import json
    r = main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "one model step")
    if len(sys.argv) > 3:  # also write the per-step GEMM traffic (bench.py roofline.traffic)
        with open(sys.argv[3], "w") as f:
            json.dump(r, f)
