#!/bin/bash
# Launch chain on the d = 16 / 32 / 64 tensor-core kernels (B200 box):
# chain parity test, then tools/large_d_times.py with chaining off / forced
# (forced = what the executor does for back-to-back step launches), interleaved.
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q -p no:cacheprovider > gpurun_out/chain_test.log 2>&1
echo "chain test rc=$?"; tail -2 gpurun_out/chain_test.log
for rep in 1 2; do
  for m in 0 force; do
    echo "ACKPT_TC_CHAIN=$m rep=$rep"
    ACKPT_TC_CHAIN=$m timeout 300 python tools/large_d_times.py 16,32,64
  done
done > gpurun_out/chain_large_d.log 2>&1
cat gpurun_out/chain_large_d.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_long_chain.py tests/test_gpu_runtime.py -x -q -p no:cacheprovider > gpurun_out/chain_tests2.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/chain_tests2.log
