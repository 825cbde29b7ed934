#!/bin/bash
# runtime experiment (f2): shared default stream (the paper's layout) and one full stream per worker
out=gpurun_out/${1:-rt}; mkdir -p $out
timeout 900 python tools/runtime_experiment.py --requests ${2:-150} --out $out/runtime_shared.json > $out/exp_shared.log 2>&1
timeout 900 python tools/runtime_experiment.py --requests ${2:-150} --own-default --out $out/runtime_own.json > $out/exp_own.log 2>&1
