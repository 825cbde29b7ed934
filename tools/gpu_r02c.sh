#!/bin/bash
# full GPU suite + smoke, A/B (base vs current), K1 per-layer timing, bench.   usage: bash tools/gpu_r02c.sh TAG
tag=${1:-r02c}; K=${2:-}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 ${K:+-k "$K"} > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for v in ${VARIANTS:-base new}; do
  lib=$PWD/paper_2506_12598_b200/libeclip_$v.so; [ "$v" = new ] && lib=$PWD/paper_2506_12598_b200/libeclip.so
  ECLIP_LIB=$lib timeout 600 python tools/ab_kernels.py > $out/ab_$v.json 2> $out/ab_$v.err
done
ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_k1dbg.so timeout 300 python tools/profile_driver.py c4 --reps 2 > $out/k1dbg_c4.log 2>&1
ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_k1dbg.so timeout 300 python tools/profile_driver.py c3 --reps 2 > $out/k1dbg_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
   python tools/profile_driver.py c4 > $out/ncu_c4l.log 2>&1
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
ls -la $out
timeout 900 python bench.py --steps 10 --no-extra > $out/bench.json 2> $out/bench.err
