"""GEMM microbenchmark driver (not collected): bare tcgen05 kernel TF/s."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import _lib
lib = _lib.load()
cases = [(8192, 8192, 8192, 0, 0, 1), (8192, 8192, 8192, 0, 1, 1), (8192, 8192, 8192, 1, 1, 1),
         (4096, 4096, 256, 0, 1, 1), (4096, 4096, 256, 0, 0, 1), (4096, 256, 2048, 0, 1, 1),
         (4096, 256, 2048, 0, 1, 4), (4096, 256, 8192, 0, 0, 4), (256, 4096, 4096, 1, 1, 8),
         (4096, 256, 4096, 1, 1, 8)]
for M, N, K, am, bm, sp in cases:
    ms = ctypes.c_double()
    st = lib.edpc_bench_gemm(M, N, K, am, bm, sp, 20, ctypes.byref(ms))
    if st:
        print(M, N, K, am, bm, sp, "err", lib.edpc_last_error()); continue
    tf = 2.0 * M * N * K / (ms.value / 1e3) / 1e12
    print(f"M={M:5d} N={N:5d} K={K:5d} a_mn={am} b_mn={bm} split={sp}: {ms.value*1e3:8.1f} us  {tf:7.1f} TF/s")
