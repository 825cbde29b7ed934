#!/bin/bash
# one GPU iteration: a parity subset of the GPU suite, the bench (every timed step checked against the
# oracle's answers), and timelines of the default library and of each libeclip_<name>.so variant given
#   usage: bash tools/gpu_iter.sh TAG [variant ...]
tag=${1:-iter}; shift
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "pruned or c5 or random_instances or batch or hetero or planner" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ttp --no-extra > $out/bench.json 2> $out/bench.err
bash tools/ab.sh $tag "$@" > $out/ab.txt 2>&1
ls $out
