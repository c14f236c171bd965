"""Runs the UNMODIFIED reference on a synthetic stream and records its ratio.

Dev-container only (needs /root/reference).  Output JSON goes to
tests/golden/ref_ratio_<name>.json and is the anchor for the 0.5% ratio
parity claim at that exact (data, B, S, dims).  Usage:

    PYTHONPATH=/root/reference/pkg/src:. python oracle/run_reference_ratio.py \
        NAME KIND NBYTES SEED LANES SEGMENTS [PROFILE] [--decompress]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2507_18969_b200 import synth  # noqa: E402  (data generator only)

import edpc  # noqa: E402
from edpc.container import write_container, read_container  # noqa: E402
from edpc.model import ModelConfig  # noqa: E402

PROFILES = {
    "paper": dict(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096,
                  lte_ratio=4, branches=2),
    "desk": dict(context_len=16, embed_dim=8, hidden_local=256, hidden_global=512,
                 lte_ratio=4, branches=2),
    # BASELINE configs 4a / 4b (bench.py --workload c4a / c4b)
    "paper_k1": dict(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096,
                     lte_ratio=4, branches=1),
    "paper_lte1": dict(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096,
                       lte_ratio=1, branches=2),
}


def main():
    name, kind, nbytes, seed, lanes, segs = sys.argv[1:7]
    profile = sys.argv[7] if len(sys.argv) > 7 and not sys.argv[7].startswith("--") else "paper"
    do_dec = "--decompress" in sys.argv
    data = synth.generate(kind, int(nbytes), int(seed))
    cfg = ModelConfig(**PROFILES[profile], lanes=int(lanes))
    stats = {}
    t0 = time.time()
    c = edpc.compress(data, cfg, int(segs), stats=stats)
    tc = time.time() - t0
    blob = write_container(c)
    rec = dict(name=name, kind=kind, nbytes=len(data), seed=int(seed), sha256=synth.sha256(data),
               profile=profile, lanes=int(lanes), segments=int(segs), container_bytes=len(blob),
               ratio=len(data) / len(blob), bits_per_byte=8 * len(blob) / len(data),
               bit_lengths=c.header.bit_lengths, compress_s=tc, stats=stats,
               nproc=os.cpu_count(), order0_bpb=synth.order0_bpb(data))
    if do_dec:
        t0 = time.time()
        out = edpc.decompress(read_container(blob))
        rec["decompress_s"] = time.time() - t0
        rec["roundtrip_ok"] = out == data
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "tests", "golden", f"ref_ratio_{name}.json")
    with open(out_path, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
