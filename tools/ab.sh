#!/bin/bash
# A/B: timeline of the default library and of each variant given (libeclip_<name>.so)
out=gpurun_out/${1:-ab}; shift; mkdir -p $out
timeout 300 python tools/timeline.py --out $out/tl_default.json > $out/tl_default.txt 2>&1
for v in "$@"; do
  ECLIP_LIB=$PWD/paper_2506_12598_b200/libeclip_$v.so timeout 300 python tools/timeline.py --out $out/tl_$v.json > $out/tl_$v.txt 2>&1
done
for f in $out/tl_*.txt; do echo "== $f"; grep -A40 "step 2" $f | grep "pass1_fast\|rowlb\|pass2\|busy"; done
