#!/usr/bin/env bash
# rebuild the C-ABI library (and fail loudly)
cd "$(dirname "$0")" && mkdir -p build && python -m paper_2507_18969_b200.build "$@" > build/last_build.log 2>&1 || { grep -iE "error|warning" build/last_build.log | head -20; tail -3 build/last_build.log; exit 1; }
ls -la paper_2507_18969_b200/_edpc_b200.so
