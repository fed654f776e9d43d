#!/bin/bash
# A/B two builds of libackpt.so on the CTA-per-sequence timings (same box):
#   bash tools/ab_sb.sh build/variants/A.so build/variants/B.so "d dtype batches..."
cp paper_1806_01117_b200/libackpt.so /tmp/ackpt_orig.so
for rep in 1 2; do
  for lib in "$1" "$2"; do
    cp "$lib" paper_1806_01117_b200/libackpt.so
    echo "== $lib"
    timeout 200 python tools/small_batch_times.py $3
  done
done
cp /tmp/ackpt_orig.so paper_1806_01117_b200/libackpt.so
