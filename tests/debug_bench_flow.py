"""Debug helper (not collected): bench flow with checks between phases."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib, synth
from paper_2507_18969_b200.config import ModelConfig
from paper_2507_18969_b200.init import init_params_f32
from paper_2507_18969_b200.model import DeviceContext
B, S = 256, 16
use_prof = int(sys.argv[1]); use_timer = int(sys.argv[2])
cfg = ModelConfig(context_len=16, embed_dim=16, hidden_local=2048, hidden_global=4096, lanes=B)
data = synth.text_like(B * 200, 0)
lib = _lib.load()
p = init_params_f32(cfg)
ctx = DeviceContext(cfg, S, len(data), 0)
ctx.load_flat(p)
buf = np.frombuffer(data, np.uint8)
_lib.check(lib.edpc_set_input(ctx.h, buf.ctypes.data, len(data), 0))
if use_prof: _lib.check(lib.edpc_prof(ctx.h, 1))
if use_timer: _lib.check(lib.edpc_timer(ctx.h, 0, None))
_lib.check(lib.edpc_compress_steps(ctx.h, 0, 40))
if use_timer:
    _lib.check(lib.edpc_timer(ctx.h, 1, None)); ms = ctypes.c_double(); _lib.check(lib.edpc_timer(ctx.h, 2, ctypes.byref(ms))); print("ms", ms.value)
if use_prof: _lib.check(lib.edpc_prof(ctx.h, 0))
bits = np.zeros(S, np.int64); tot = ctypes.c_int64()
_lib.check(lib.edpc_compress_finish(ctx.h, bits.ctypes.data, ctypes.byref(tot)))
pay = np.zeros(tot.value, np.uint8)
_lib.check(lib.edpc_get_payloads(ctx.h, pay.ctypes.data, pay.size))
ctx.close()
print("closed", flush=True)
d = DeviceContext(cfg, S, len(data), 0)
_lib.check(lib.edpc_sync(d.h)); print("new ctx sync ok", flush=True)
d.load_flat(p)
_lib.check(lib.edpc_set_payloads(d.h, pay.ctypes.data, bits.ctypes.data))
_lib.check(lib.edpc_decompress_steps(d.h, 0, 40))
got = np.empty((B, 40), np.uint8); _lib.check(lib.edpc_get_columns(d.h, 0, 40, got.ctypes.data))
print("lossless", np.array_equal(got, np.frombuffer(data, np.uint8).reshape(B, -1)[:, :40]))
