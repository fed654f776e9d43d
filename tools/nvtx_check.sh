#!/bin/bash
# NVTX ranges (csrc/nvtx.h) seen by ncu: kernels inside the backward phase
# vs the forward sweep of tools/nvtx_probe.py (B200 box).
python tools/nvtx_probe.py || exit 1
for pat in "ackpt@pass/sweep/" "ackpt@pass/backward/"; do
  echo "== $pat"
  ncu --nvtx --nvtx-include "$pat" --metrics gpu__time_duration.sum --csv python tools/nvtx_probe.py 2>/dev/null \
    | python -c "import sys,csv,collections; r=[x for x in csv.reader(sys.stdin) if len(x)>5]; h=r[0]; i=h.index('Kernel Name'); c=collections.Counter(x[i].split('(')[0] for x in r[1:]); print(dict(c))"
done
