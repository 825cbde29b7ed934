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
# summaries on the box (the reports are too large to bring back whole): raw metrics of every kernel and
# per-line stall samples of the top kernels; only the pass-1 / K3 reports themselves travel back
ncu -i $out/step_full.ncu-rep --page raw --csv > $out/step_full_raw.csv 2>/dev/null
ncu -i $out/c4_full.ncu-rep --page raw --csv > $out/c4_full_raw.csv 2>/dev/null
for k in k_pass1_fast k_rowlb_fused k_pass2 k_prep_aux k_materialize; do
  python tools/ncu_lines.py $out/step_full.ncu-rep $k 40 > $out/lines_$k.txt 2>&1
done
for k in k_levels k_slice_f32 k_slice_exact; do python tools/ncu_lines.py $out/c4_full.ncu-rep $k 40 > $out/lines_c4_$k.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1_fast -c 1 -o $out/pass1_full \
   python tools/profile_driver.py c5 --mixes 4096 --reps 1 > $out/ncu_p1.log 2>&1
rm -f $out/step_full.ncu-rep $out/c4_full.ncu-rep
ls -la $out
