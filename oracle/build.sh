#!/usr/bin/env bash
# Builds the CPU oracle (test infrastructure; never linked by the product).
# No -ffast-math and no FMA contraction: float64 must round like the numba
# kernels of the reference.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$here/build"
gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -o "$here/build/libedpc_oracle.so" \
    "$here/edpc_oracle.c" -lm
