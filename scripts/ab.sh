#!/bin/bash
# A/B timing of library variants (run under gpurun): default lib vs each variants/libfdsdf_*.so named
# usage: bash scripts/ab.sh NAME...   (two interleaved rounds)
for r in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2511_08980_b200/variants/libfdsdf_$v.so"; fi
    FDSDF_LIB="$lib" timeout -s KILL 180 python bench.py --no-cpu-baseline --no-extras --no-e2e --no-c5 --no-eval-sweep --steps 20 > gpurun_out/ab_$v.log 2>&1
    echo "== $v (round $r)"; python scripts/show_bench.py gpurun_out/ab_$v.log || tail -3 gpurun_out/ab_$v.log
  done
done
