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
