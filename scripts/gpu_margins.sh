#!/bin/bash
# parity margins (loss / gradient / entry errors) of the step and the full-size C2 run
timeout -s KILL 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -s -k "c2_full or (step_parity and tensor)" 2>&1 | grep -E "lerr|c2 full|passed|failed" | cut -c1-260
