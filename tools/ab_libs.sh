#!/bin/bash
# A/B several builds of libackpt.so on the fused d=8 launches at the C2 shape
# (same box, interleaved):  bash tools/ab_libs.sh reps A.so B.so ...
reps=$1; shift
cp paper_1806_01117_b200/libackpt.so /tmp/ackpt_orig.so
for rep in $(seq 1 $reps); do
  for lib in "$@"; do
    cp "$lib" paper_1806_01117_b200/libackpt.so
    echo -n "$lib "
    timeout 200 python tools/fused_times.py 2>/dev/null | tail -1
  done
done
cp /tmp/ackpt_orig.so paper_1806_01117_b200/libackpt.so
