#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (N=1) + reference arm, launch lists and ncu --set full
# of every planner kernel of one bench-size C5 step.   usage: bash tools/gpu_check.sh TAG
tag=${1:-check}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttp > $out/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
   python tools/profile_driver.py c4 > $out/ncu_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_ -c 16 -o $out/step_full \
   python tools/profile_driver.py c5 --mixes 4096 --reps 1 > $out/ncu_full.log 2>&1
ls -la $out
