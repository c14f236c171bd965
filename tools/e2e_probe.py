"""Public-API compress/decompress of a C2-shaped stream with progress prints (debug helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import ModelConfig, compress, decompress, read_container, write_container, synth
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=4096)
t = time.time(); data = synth.generate("text", mb << 20, 0); print("synth", time.time() - t, flush=True)
st = {}
t = time.time(); blob = write_container(compress(data, cfg, 256, stats=st)); print("compress", time.time() - t, st, flush=True)
t = time.time(); out = decompress(read_container(blob)); print("decompress", time.time() - t, out == data, flush=True)
