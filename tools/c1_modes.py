"""Config 1 (n=1000, d=32, s=10, B=1 fp64, file tier): wall ms of every strategy in per-step / fused x eager / CUDA-graph mode (min of 5)."""
import sys, os, json, tempfile
sys.path.insert(0, os.getcwd())
import paper_1806_01117_b200 as pkg, paper_1806_01117_b200.lstm as lstm
scratch = tempfile.mkdtemp()
out = {}
for name, strat in (("full", pkg.FullStorage()), ("revolve", pkg.Revolve(10)), ("multistage", pkg.Multistage(10))):
    r = {}
    for fuse in (False, True):
        for graph in (False, True):
            rep = lstm.bench(strat, n=1000, d=32, s=10, backend_config={"kind": "file", "dir": scratch}, runs=5, fuse=fuse, graph=graph)
            r[f"fuse={int(fuse)},graph={int(graph)}"] = round(rep.wall_seconds * 1e3, 3)
    out[name] = r
print(json.dumps(out))
