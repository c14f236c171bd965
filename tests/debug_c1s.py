"""Debug helper (not collected): C1 ratio for each recorded reference seed."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import ModelConfig, compress, write_container, synth
for name in ("c1_text_1m", "c1_text_1m_s1", "c1_text_1m_s2"):
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"ref_ratio_{name}.json")))
    data = synth.generate(ref["kind"], ref["nbytes"], ref["seed"])
    assert synth.sha256(data) == ref["sha256"]
    cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=ref["lanes"])
    blob = write_container(compress(data, cfg, ref["segments"]))
    r = len(data) / len(blob)
    print(os.environ.get("EDPC_TCGEN05", "1"), name, "ratio %.5f ref %.5f delta %+.4f" % (r, ref["ratio"], r / ref["ratio"] - 1), flush=True)
