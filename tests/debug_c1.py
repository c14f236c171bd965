"""Debug helper (not collected): C1 ratio under the current env."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import ModelConfig, compress, write_container, synth
ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_ratio_c1_text_1m.json")))
data = synth.generate(ref["kind"], ref["nbytes"], ref["seed"])
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=ref["lanes"])
t = time.time()
blob = write_container(compress(data, cfg, ref["segments"]))
r = len(data) / len(blob)
print(os.environ.get("EDPC_TCGEN05", "1"), "ratio", r, "ref", ref["ratio"], "delta %.4f" % (r / ref["ratio"] - 1), "bytes", len(blob), ref["container_bytes"], "s", time.time() - t)
