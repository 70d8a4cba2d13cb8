#!/bin/bash
# swap in an ablation build of the library for one probe run (diagnostic only)
set -e
cp paper_2206_07244_b200/lib/libspgemm_b200.so /tmp/orig.so
for v in "$@"; do
  cp tools/abl_$v/libspgemm_b200.so paper_2206_07244_b200/lib/libspgemm_b200.so
  echo "== $v"; python tools/host_probe.py 2
done
cp /tmp/orig.so paper_2206_07244_b200/lib/libspgemm_b200.so
echo "== base"; python tools/host_probe.py 2
