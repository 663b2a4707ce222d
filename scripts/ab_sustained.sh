#!/bin/bash
# A/B of library variants under the board's power limit (run under gpurun): the C2 step back to
# back for seconds (scripts/power_probe.py), default lib vs each variants/libfdsdf_NAME.so named
# usage: bash scripts/ab_sustained.sh NAME...   (two interleaved rounds)
for r in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2511_08980_b200/variants/libfdsdf_$v.so"; fi
    echo "== $v (round $r)"; FDSDF_LIB="$lib" timeout -s KILL 120 python scripts/power_probe.py 2 2>&1 | grep -v "^warm"
  done
done
