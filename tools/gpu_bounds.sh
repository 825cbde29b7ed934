#!/bin/bash
# the GPU suite and the bench workload against the bounds-checked test build (-DECLIP_BOUNDS: ECLIP_CHECK traps
# on an out-of-range index in the kernels; compute-sanitizer is not available on the pool)
#   usage: bash tools/gpu_bounds.sh TAG
tag=${1:-bounds}
out=gpurun_out/$tag; mkdir -p $out
export ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_bounds.so
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect "tests/test_gpu_parity.py::test_overflow_fallbacks_with_tiny_list_capacities" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
grep -c "ECLIP_CHECK failed" $out/*.log $out/*.err > $out/check_failures.txt 2>&1
ls $out
