"""One GEMM microbenchmark case (not collected): M N K a_mn b_mn split iters."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18969_b200 import _lib
lib = _lib.load()
M, N, K, am, bm, sp, it = (int(x) for x in sys.argv[1:8])
ms = ctypes.c_double()
_lib.check(lib.edpc_bench_gemm(M, N, K, am, bm, sp, it, ctypes.byref(ms)))
print(f"M={M} N={N} K={K}: {ms.value*1e3:.1f} us  {2.0*M*N*K/(ms.value/1e3)/1e12:.1f} TF/s", flush=True)
