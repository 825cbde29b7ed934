#!/bin/bash
tag=${1:-c4ncu}; out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_levels|k_slice_f32|k_slice_exact" -c 3 -o $out/c4_full \
   python tools/profile_driver.py c4 --reps 1 > $out/ncu_c4.log 2>&1
ls $out
