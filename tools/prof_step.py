"""Profiling driver (not collected): C2-shaped context, a few model steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib, synth
from paper_2507_18969_b200.config import ModelConfig
from paper_2507_18969_b200.init import init_params_f32
from paper_2507_18969_b200.model import DeviceContext
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=B)
data = synth.text_like(B * 64, 0)
lib = _lib.load()
ctx = DeviceContext(cfg, B // 16, len(data), 0)
ctx.load_flat(init_params_f32(cfg))
buf = np.frombuffer(data, np.uint8)
_lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, len(data), 0))
_lib.check(lib.edpc_compress_steps(ctx.h, 0, 16 + steps))
_lib.check(lib.edpc_sync(ctx.h))
print("ok")
