#!/bin/bash
# the whole GPU suite, smoke, the bench (every timed step checked against the oracle's answers) and a timeline
#   usage: bash tools/gpu_full_iter.sh TAG
tag=${1:-fiter}
out=gpurun_out/$tag; mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > $out/bench.json 2> $out/bench.err
timeout 300 python tools/timeline.py --out $out/timeline.json > $out/timeline.txt 2>&1
ls $out
