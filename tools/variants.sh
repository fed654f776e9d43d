#!/bin/bash
# A/B the d=8 fp32 step-kernel variants (chain timing at the C2 shape).
for v in ldg ldg3 tma tma128 tma_bwd2; do
  echo -n "$v "
  ACKPT_KERNEL_VARIANT=$v timeout 120 python tools/profile_kernels.py --steps 60 --fused 1
done
