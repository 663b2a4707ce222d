#!/bin/bash
# quick GPU check: the GPU test suite + a short bench (run under gpurun)
timeout -s KILL 300 python -m pytest tests -m gpu -q -x "$@" 2>&1 | tail -3
timeout -s KILL 180 python bench.py --no-cpu-baseline --no-extras --no-e2e --steps 10 > gpurun_out/b.log 2>&1
python scripts/show_bench.py gpurun_out/b.log || tail -5 gpurun_out/b.log
