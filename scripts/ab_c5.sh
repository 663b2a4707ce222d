for r in 1 2; do
  for v in default poll; do
    if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2511_08980_b200/variants/libfdsdf_$v.so"; fi
    FDSDF_LIB="$lib" timeout -s KILL 300 python bench.py --config c5 --no-cpu-baseline --no-extras --no-e2e --no-c5 --no-eval-sweep --steps 40 > gpurun_out/abc5_$v.log 2>&1
    echo "== $v (round $r)"; python scripts/show_bench.py gpurun_out/abc5_$v.log || tail -3 gpurun_out/abc5_$v.log
    python - <<PY
import json
for l in open('gpurun_out/abc5_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('clocks', d.get('clocks'))
PY
  done
done
