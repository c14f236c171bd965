"""GEMM microbenchmark sweep (not collected)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import _lib
lib = _lib.load()
cases = [(4096, 4096, 256, 0, 0, 1), (4096, 4096, 256, 0, 1, 1), (4096, 4096, 1024, 0, 0, 1),
         (4096, 4096, 4096, 0, 0, 1), (16384, 4096, 256, 0, 0, 1), (4096, 256, 4096, 0, 0, 4)]
for M, N, K, am, bm, sp in cases:
    ms = ctypes.c_double()
    st = lib.edpc_bench_gemm(M, N, K, am, bm, sp, 20, ctypes.byref(ms))
    tf = 2.0 * M * N * K / (ms.value / 1e3) / 1e12
    print(f"BNmax={os.environ.get('EDPC_BN_MAX','256')} M={M:5d} N={N:5d} K={K:5d} a_mn={am} b_mn={bm} split={sp}: {ms.value*1e3:8.1f} us  {tf:7.1f} TF/s", flush=True)
