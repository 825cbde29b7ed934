#!/bin/bash
# full round capture: GPU suite, smoke, bench (+ reference arm), launch lists, ncu --set full of one C5 step and
# of the C4 plan, timeline.   usage: bash tools/gpu_final.sh TAG
tag=${1:-final}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=20 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttp > $out/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
   python tools/profile_driver.py c4 > $out/ncu_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_ -c 20 -o $out/step_full \
   python tools/profile_driver.py c5 --mixes 4096 --reps 1 > $out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_levels|k_slice_f32|k_slice_exact" -c 3 -o $out/c4_full \
   python tools/profile_driver.py c4 --reps 1 > $out/ncu_c4full.log 2>&1
ls -la $out
