#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (N=1), launch list and one ncu --set full of pass 1.
# usage (from repo root, on the GPU box): bash tools/gpu_check.sh [tag]
tag=${1:-check}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttp > $out/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
   python tools/profile_driver.py c4 > $out/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -c 1 -o $out/pass1_full \
   python tools/profile_driver.py c5 --mixes 512 > $out/ncu_full.log 2>&1
ls -la $out
