"""Context teardown cost across repeated public-API compress calls (debug helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import ModelConfig, compress, decompress, read_container, write_container, synth
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=4096)
data = synth.generate("text", mb << 20, 0)
for rep in range(3):
    st = {}
    t = time.time(); blob = write_container(compress(data, cfg, 256, stats=st))
    print("compress", rep, round(time.time() - t, 3), {k: round(v, 4) for k, v in st.items() if k.endswith("_s")}, flush=True)
    t = time.time(); out = decompress(read_container(blob)); print("decompress", rep, round(time.time() - t, 3), out == data, flush=True)
