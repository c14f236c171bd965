"""Debug helper (not collected by pytest): a reduced bench-shaped compress."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib, synth
from paper_2507_18969_b200.config import ModelConfig
from paper_2507_18969_b200.init import init_params_f32
from paper_2507_18969_b200.model import DeviceContext
B, S, cols = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 4 * cols
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=B)
data = synth.text_like(B * L, 0)
lib = _lib.load()
ctx = DeviceContext(cfg, S, len(data), 0)
ctx.load_flat(init_params_f32(cfg))
buf = np.frombuffer(data, np.uint8)
_lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, len(data), 0))
_lib.check(lib.edpc_compress_steps(ctx.h, 0, cols))
_lib.check(lib.edpc_sync(ctx.h))
print("steps ok", flush=True)
bits = np.zeros(S, np.int64); tot = ctypes.c_int64()
_lib.check(lib.edpc_compress_finish(ctx.h, bits.ctypes.data, ctypes.byref(tot)))
print("finish ok", tot.value, bits[:4])
