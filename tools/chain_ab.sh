#!/bin/bash
# Launch-chain check on a B200 box: the -m gpu suite with chaining on (the
# default), then the bench at C2 with ACKPT_TC_CHAIN=0 vs default, interleaved.
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/chain_tests.log
for rep in 1 2; do
  for m in 0 1; do
    ACKPT_TC_CHAIN=$m timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/chain_bench_${m}_${rep}.json 2>/dev/null
    echo "chain=$m rep=$rep $(python -c "import json,sys; d=json.loads(open('gpurun_out/chain_bench_${m}_${rep}.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'])")"
  done
done
