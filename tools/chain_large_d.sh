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
python - <<'PY'
import json
for l in open("gpurun_out/chain_large_d.log"):
    if l.startswith("ACKPT"): print(l.strip()); continue
    try: d = json.loads(l)
    except Exception: continue
    print(" d=%d fwd %.1f bwd %.1f adv %.1f tape %.1f rev %.1f" % (d["d"], d["fwd_us"], d["bwd_us"], d.get("adv_us", 0), d.get("tape_us", 0), d.get("rev_us", 0)))
PY
