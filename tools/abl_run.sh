#!/bin/bash
# swap in ablation builds of the library (tools/build_ablation.sh) for one timing
# run each (diagnostic only): tools/abl_run.sh <config> <variant>...
set -e
cfg=$1; shift
cp paper_2206_07244_b200/lib/libspgemm_b200.so /tmp/orig.so
for v in "$@"; do
  cp tools/abl_$v/libspgemm_b200.so paper_2206_07244_b200/lib/libspgemm_b200.so
  echo "== $v"; python tools/quick_timing.py $cfg | grep cfg
done
cp /tmp/orig.so paper_2206_07244_b200/lib/libspgemm_b200.so
echo "== base"; python tools/quick_timing.py $cfg | grep cfg
