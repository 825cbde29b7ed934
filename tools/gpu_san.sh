#!/bin/bash
# compute-sanitizer over the GPU suite: memcheck (all GPU tests), racecheck + synccheck (the planner's
# parity tests at small and bench sizes).   usage: bash tools/gpu_san.sh TAG
tag=${1:-san}
out=gpurun_out/$tag; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
K="random_instances_vs_oracle or c1_sweep or c2_all or edge or small_batch or pruned_equals_exhaustive_batch or overflow or sharded or many_workers or c4_full"
timeout 1800 $CS --tool memcheck --target-processes all --print-limit 200 --log-file $out/memcheck.log \
   python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/memcheck_pytest.log 2>&1; echo "rc=$?" >> $out/memcheck_pytest.log
timeout 1500 $CS --tool racecheck --racecheck-report analysis --target-processes all --print-limit 200 --log-file $out/racecheck.log \
   python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py -k "$K" > $out/racecheck_pytest.log 2>&1; echo "rc=$?" >> $out/racecheck_pytest.log
timeout 900 $CS --tool synccheck --target-processes all --print-limit 200 --log-file $out/synccheck.log \
   python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py -k "$K" > $out/synccheck_pytest.log 2>&1; echo "rc=$?" >> $out/synccheck_pytest.log
tail -3 $out/*.log
