#!/bin/bash
# memcheck on selected GPU tests, then the whole GPU suite.   usage: bash tools/gpu_memk.sh TAG "k-expr" ...
tag=${1:-memk}; shift
out=gpurun_out/$tag; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for t in "$@"; do
  n=$(echo $t | tr -c 'a-z0-9' '_')
  timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest -q -m gpu -p no:cacheprovider tests -k "$t" > $out/mc_$n.log 2>&1
  echo "rc=$?" >> $out/mc_$n.log
done
timeout 1500 python -m pytest tests -q -m gpu --durations=15 -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
