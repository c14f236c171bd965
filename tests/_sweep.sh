for am in 0 1; do for bm in 0 1; do timeout 100 python tests/bench_gemm1.py 256 4096 4096 $am $bm 8 30 | sed "s/^/a_mn=$am b_mn=$bm split8 /"; done; done
timeout 100 python tests/bench_gemm1.py 512 4096 4096 1 1 8 30 | sed "s/^/M512 mn split8 /"
timeout 100 python tests/bench_gemm1.py 256 4096 4096 1 1 4 30 | sed "s/^/mn split4 /"
