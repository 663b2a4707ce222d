#!/bin/bash
# Round evidence (run under gpurun): the default bench line, the ncu launch list of a short
# bench run, and one `ncu --set full` capture of one step's kernels.  TAG names the outputs.
TAG=${1:-r02}
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python scripts/show_bench.py gpurun_out/bench_$TAG.log
QUICK="--no-extras --no-e2e --no-cpu-baseline --no-c5 --no-eval-sweep"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 $QUICK \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_tc|bwd_tc|wgrad_tc|finalize|pack_tc" --launch-skip 18 --launch-count 6 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 $QUICK \
  > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full capture rc=$?"
