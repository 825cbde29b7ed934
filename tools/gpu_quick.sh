#!/bin/bash
# quick GPU iteration: GPU tests (optional), timeline, bench [+ ncu full of every kernel of one C5 step]
# usage: bash tools/gpu_quick.sh TAG [full=0|1] [tests=0|1]
tag=${1:-quick}; full=${2:-0}; tests=${3:-0}
out=gpurun_out/$tag; mkdir -p $out
if [ "$tests" = "1" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
fi
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
if [ "$full" = "1" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_ -c 16 -o $out/step_full \
     python tools/profile_driver.py c5 --mixes 4096 --reps 1 > $out/ncu_full.log 2>&1
fi
