"""Debug helper (not collected)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib
lib = _lib.load()
np.set_printoptions(precision=3, linewidth=160)
M, N, K = 128, 64, 32
rng = np.random.default_rng(1)
A = np.arange(M * K, dtype=np.float32).reshape(M, K) / 1000
B = rng.random((K, N)).astype(np.float32)
ref = A @ B
for a_mn, b_mn in ((1, 0), (0, 1)):
    Ah = np.ascontiguousarray(A.T) if a_mn else A
    Bh = B if b_mn else np.ascontiguousarray(B.T)
    for dbg in (2, 0, 3):
        C = np.full((M, N), -7, dtype=np.float32)
        st = lib.edpc_debug_gemm(M, N, K, a_mn, b_mn, Ah.ctypes.data, Bh.ctypes.data, C.ctypes.data, dbg)
        err = np.abs(C - ref).max() / np.abs(ref).max()
        print("a_mn", a_mn, "b_mn", b_mn, "dbg", dbg, "st", st, "err %.2e" % err)
        print(C[:2, :12]); print(C[40, :12])
print("ref", ref[:2, :6])
print("A^T rows", Ah[:2, :12] if True else None)
