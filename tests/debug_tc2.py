"""Debug helper (not collected)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib
lib = _lib.load()

def run(M, N, K, a_mn, b_mn, dist):
    rng = np.random.default_rng(M + N + K)
    if dist == "pos":
        A = rng.random((M, K)).astype(np.float32); B = rng.random((K, N)).astype(np.float32)
    else:
        A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(K, N)).astype(np.float32)
    Ah = np.ascontiguousarray(A.T) if a_mn else A
    Bh = B if b_mn else np.ascontiguousarray(B.T)
    C = np.full((M, N), -7, dtype=np.float32)
    st = lib.edpc_debug_gemm(M, N, K, a_mn, b_mn, Ah.ctypes.data, Bh.ctypes.data, C.ctypes.data, 0)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.abs(C - ref).max() / np.abs(ref).max()
    return st, err, C[0, :3], ref[0, :3]

for dist in ("normal", "pos", "normal"):
    for (M, N, K) in [(128, 64, 32), (128, 256, 64)]:
        for a_mn in (0, 1):
            for b_mn in (0, 1):
                st, err, c, r = run(M, N, K, a_mn, b_mn, dist)
                print(dist, M, N, K, a_mn, b_mn, "st", st, "err %.2e" % err, c, r, flush=True)
