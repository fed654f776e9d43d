#!/bin/bash
# A/B two builds of libackpt.so on the fused d=8 launches at the C2 shape
# (same box, interleaved):  bash tools/ab_fused.sh A.so B.so [reps]
cp paper_1806_01117_b200/libackpt.so /tmp/ackpt_orig.so
for rep in $(seq 1 ${3:-3}); do
  for lib in "$1" "$2"; do
    cp "$lib" paper_1806_01117_b200/libackpt.so
    echo -n "$lib "
    timeout 200 python tools/fused_times.py
  done
done
cp /tmp/ackpt_orig.so paper_1806_01117_b200/libackpt.so
