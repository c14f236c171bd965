"""Finds the fp16 MN-major descriptor strides (not collected): tries LBO/SBO pairs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib
lib = _lib.load()
M, N, K = 128, 128, 128
rng = np.random.default_rng(0)
A = rng.normal(size=(M, K)).astype(np.float16)
B = rng.normal(size=(K, N)).astype(np.float16)
ref = A.astype(np.float64) @ B.astype(np.float64)
for a_mn, b_mn in [(0, 0), (1, 0), (0, 1), (1, 1)]:
    Ah = np.ascontiguousarray(A.T) if a_mn else A
    Bh = B if b_mn else np.ascontiguousarray(B.T)
    pairs = [(0, 0)] if not (a_mn or b_mn) else [(8192, 1024), (1024, 8192), (0, 1024), (8192, 0), (2048, 1024), (1024, 2048), (16, 1024), (4096, 1024)]
    for lbo, sbo in pairs:
        C = np.zeros((M, N), dtype=np.float32)
        st = lib.edpc_debug_gemm_h(M, N, K, a_mn, b_mn, Ah.ctypes.data, Bh.ctypes.data, C.ctypes.data, lbo, sbo)
        err = np.abs(C - ref).max() / np.abs(ref).max() if st == 0 else -1
        print(f"a_mn={a_mn} b_mn={b_mn} lbo={lbo} sbo={sbo}: status {st} err {err:.3g}", flush=True)
