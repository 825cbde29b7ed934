#!/bin/bash
# exhaustive sweep check: parity tests of the exhaustive / pruned paths, A/B, ncu of the exhaustive no-QoS kernel
tag=${1:-r02h}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -k "pruned_equals or c5_small or many_workers or batch_paper or random_instances" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for v in base new; do
  lib=$PWD/paper_2506_12598_b200/libeclip_$v.so; [ "$v" = new ] && lib=$PWD/paper_2506_12598_b200/libeclip.so
  ECLIP_LIB=$lib timeout 600 python tools/ab_kernels.py > $out/ab_$v.json 2> $out/ab_$v.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1_fast -c 1 -o $out/c5_exh_noqos \
   python tools/profile_driver.py c5 --mixes 512 --reps 1 --noqos --exhaustive > $out/ncu_exh.log 2>&1
ls $out
