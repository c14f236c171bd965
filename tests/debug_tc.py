"""Debug helper (not collected): probe the tcgen05 GEMM stages."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18969_b200 import _lib
lib = _lib.load()
M, N, K = 128, 64, 32
A = (np.arange(M * K, dtype=np.float32).reshape(M, K) % 97) / 97
B = (np.arange(K * N, dtype=np.float32).reshape(N, K) % 89) / 89   # [N][K]
np.set_printoptions(precision=3, linewidth=150)
for dbg in (1, 2, 0):
    C = np.full((M, N), -1, np.float32)
    st = lib.edpc_debug_gemm(M, N, K, 0, 0, A.ctypes.data, B.ctypes.data, C.ctypes.data, dbg)
    print("dbg", dbg, "status", st, lib.edpc_last_error())
    print(C[:3, :8]); print(C[64:66, :8])
ref = A @ B.T
print("ref", ref[:3, :8])
