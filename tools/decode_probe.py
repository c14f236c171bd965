"""Chunk-by-chunk decompress of a C2-shaped stream with progress prints (debug helper)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import ModelConfig, compress, synth, _lib
from paper_2507_18969_b200.init import init_params_f32
from paper_2507_18969_b200.model import DeviceContext
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=4096)
data = synth.generate("text", mb << 20, 0)
t = time.time(); c = compress(data, cfg, 256); print("compress", time.time() - t, flush=True)
h = c.header
lib = _lib.load()
ctx = DeviceContext(cfg, 256, len(data), 0, numerics=h.numerics)
ctx.load_flat(init_params_f32(cfg))
pay = np.frombuffer(b"".join(c.segments), np.uint8)
bits = np.ascontiguousarray(h.bit_lengths, np.int64)
_lib.check(lib.edpc_set_payloads(ctx.h, pay.ctypes.data, bits.ctypes.data))
L = ctx.lane_len
t = time.time()
for i0 in range(0, L, 512):
    _lib.check(lib.edpc_decompress_steps(ctx.h, i0, min(L, i0 + 512)))
    _lib.check(lib.edpc_sync(ctx.h))
    print("chunk", i0, round(time.time() - t, 2), flush=True)
out = np.empty(len(data), np.uint8)
print("get_output", lib.edpc_get_output(ctx.h, out.ctypes.data, out.size), flush=True)
print("ok", out.tobytes() == data, flush=True)
