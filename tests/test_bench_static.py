"""CPU checks of bench.py: argument defaults and no undefined names in any
function (a NameError would only surface on the GPU box)."""

import ast
import builtins
import os

from conftest import ROOT


def _undefined_names(path):
    src = open(path).read()
    tree = ast.parse(src)
    top = {n.name for n in tree.body if isinstance(n, (ast.FunctionDef, ast.ClassDef))}
    top |= {t.id for n in tree.body if isinstance(n, ast.Assign) for t in n.targets if isinstance(t, ast.Name)}
    top |= {(a.asname or a.name).split(".")[0] for n in tree.body if isinstance(n, (ast.Import, ast.ImportFrom))
            for a in n.names}
    bad = []
    for fn in [n for n in tree.body if isinstance(n, ast.FunctionDef)]:
        known = set()
        for node in ast.walk(fn):
            if isinstance(node, ast.Name) and isinstance(node.ctx, (ast.Store, ast.Del)):
                known.add(node.id)
            elif isinstance(node, (ast.FunctionDef, ast.Lambda)):
                known.update(a.arg for a in node.args.args)
                if isinstance(node, ast.FunctionDef):
                    known.add(node.name)
            elif isinstance(node, (ast.Import, ast.ImportFrom)):
                known.update((a.asname or a.name).split(".")[0] for a in node.names)
            elif isinstance(node, ast.ExceptHandler) and node.name:
                known.add(node.name)
        for node in ast.walk(fn):
            if (isinstance(node, ast.Name) and isinstance(node.ctx, ast.Load) and node.id not in known
                    and node.id not in top and not hasattr(builtins, node.id)):
                bad.append((fn.name, node.id, node.lineno))
    return bad


def test_bench_has_no_undefined_names():
    assert _undefined_names(os.path.join(ROOT, "bench.py")) == []


def test_graft_entry_has_no_undefined_names():
    assert _undefined_names(os.path.join(ROOT, "__graft_entry__.py")) == []


def test_bench_defaults():
    import bench

    a = bench.parse_args([])
    assert (a.gpus, a.n, a.d, a.batch, a.memory_ratio) == (1, 10_000, 8, 1 << 20, 0.1)
    assert a.warmup >= 3 and a.fuse
    assert not bench.parse_args(["--per-step"]).fuse


def test_bench_config4_defaults():
    import bench

    a = bench.parse_args(["--config", "c4"])
    assert (a.batch, a.memory_ratio) == (1 << 24, 0.05)
    assert a.no_other_mode  # the per-step leg would need more pinned slots than the host holds
    cfg = bench.workload_config(a, int(a.memory_ratio * a.n) - 1)
    assert cfg["state_bytes_per_gpu"] == 1 << 30 and "config 4" in cfg["workload"]


def test_fused_pass_bytes_matches_the_launch_split():
    # sweep = one Advance launch (2S) per interval + a store (S
    # read from HBM, S over the link); backward = tape (L+1)S + reverse (L+2)S
    # per <= 64-step launch + a fetch (S) per interval.
    import bench

    class St:
        prefetches_issued = 3

    S, n = 1 << 20, 200
    b = bench.fused_pass_bytes(n, [0, 80, 160], S, True, St())
    launches = [64, 16, 64, 16, 40]  # intervals of 80, 80, 40 steps
    assert b["sweep_link"] == 3 * S and b["sweep_hbm"] == 3 * 2 * S + 3 * S
    assert b["backward_link"] == 3 * S
    assert b["backward_hbm"] == sum((c + 1) * S + (c + 2) * S for c in launches) + 3 * S
