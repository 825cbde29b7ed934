#!/bin/bash
# quick GPU iteration: GPU tests (optional), smoke, timeline, bench [+ ncu full of every kernel of one C5 step]
# usage: bash tools/gpu_quick.sh TAG [full=0|1] [tests=0|1]
tag=${1:-quick}; full=${2:-0}; tests=${3:-0}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
if [ "$tests" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --durations=25 -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
fi
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
if [ "$full" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttp --no-extra > $out/ncu_bench.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_ -c 16 -o $out/step_full \
     python tools/profile_driver.py c5 --mixes 4096 --reps 1 > $out/ncu_full.log 2>&1
fi
ls -la $out
