"""Config-1 per-step passes (B=1 fp64, d=32, n=1000): wall vs GPU vs host-enqueue time, eager and CUDA-graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, tempfile
import paper_1806_01117_b200 as pkg, paper_1806_01117_b200.lstm as lstm
cell = lstm.random_cell(32, 1000, 0); ops = lstm.operator_pair(cell); s0 = lstm.random_state(32, 1)
for strat in (pkg.FullStorage(), pkg.Revolve(10)):
    for graph in (False, True):
        best=None
        for _ in range(5):
            _, st = pkg.execute(strat, ops, s0, graph=graph)
            if best is None or st.wall_seconds < best.wall_seconds: best = st
        print(type(strat).__name__, "graph" if graph else "eager", "wall %.2f ms gpu %.2f ms enqueue %.2f ms launches %d" % (best.wall_seconds*1e3, best.device["gpu_seconds"]*1e3, best.device["host_enqueue_seconds"]*1e3, best.device.get("kernel_launches", -1)))
