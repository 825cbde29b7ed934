#!/bin/bash
# round-2 iteration: new GPU tests, A/B of base vs current lib, K1 per-layer timing (K1_DEBUG variant),
# ncu --set full of the C4 plan (K1, K3) and of the exhaustive no-QoS C5 sweep.   usage: bash tools/gpu_r02b.sh TAG [k-expr]
tag=${1:-r02b}; K=${2:-"weight or c4 or c2 or random or worked or k1 or c3 or pruned or overflow or small_batch or planner"}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "$K" -p no:cacheprovider --durations=15 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for v in base ""; do
  lib=$PWD/paper_2506_12598_b200/libeclip${v:+_$v}.so
  ECLIP_LIB=$lib timeout 600 python tools/ab_kernels.py > $out/ab_${v:-new}.json 2> $out/ab_${v:-new}.err
done
ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_k1dbg.so timeout 300 python tools/profile_driver.py c4 --reps 3 > $out/k1dbg_c4.log 2>&1
ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_k1dbg.so timeout 300 python tools/profile_driver.py c3 --reps 3 > $out/k1dbg_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_levels|k_slice" -c 8 -o $out/c4_full \
   python tools/profile_driver.py c4 --reps 1 > $out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1_fast -c 1 -o $out/c5_exh_noqos \
   python tools/profile_driver.py c5 --mixes 512 --reps 1 --noqos --exhaustive > $out/ncu_exh.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
   python tools/profile_driver.py c4 > $out/ncu_c4l.log 2>&1
ls -la $out
