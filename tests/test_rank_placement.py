"""Host-side placement logic of a rank (CPU): the host-RAM budget that picks
the pinned tier or the three-stage cascade (C4 needs
ceil(n/I) x 1 GiB pinned per GPU, ~1 TiB per 8-GPU node), and NUMA binding
that degrades to a no-op without a GPU / NUMA topology."""

import paper_1806_01117_b200.distributed as D


class _FakePkg:
    class PinnedHostBackend:
        def __init__(self, slot_bytes):
            self.slot_bytes = slot_bytes

    class CascadeBackend:
        def __init__(self, directory, slot_bytes, dram_slots):
            self.directory, self.slot_bytes, self.dram_slots = directory, slot_bytes, dram_slots


GiB = 1 << 30


def test_budget_is_a_share_of_available_memory(monkeypatch):
    monkeypatch.setattr(D, "host_memory_available", lambda: 200 * GiB)
    assert D.pinned_key_budget(GiB, local_ranks=1) == 160  # 0.8 x 200 GiB
    assert D.pinned_key_budget(GiB, local_ranks=8) == 20
    assert D.pinned_key_budget(64 << 20, local_ranks=8) == 320


def test_c4_plan_spills_on_a_shared_node(monkeypatch, tmp_path):
    monkeypatch.setattr(D, "host_memory_available", lambda: 200 * GiB)
    # C4 per GPU: 1 GiB states, ~125 boundary keys (n = 10^4, I ~ 80)
    b1 = D.make_rank_backend(_FakePkg, GiB, 125, local_ranks=1)
    assert isinstance(b1, _FakePkg.PinnedHostBackend)
    b8 = D.make_rank_backend(_FakePkg, GiB, 125, local_ranks=8, spill_dir=str(tmp_path))
    assert isinstance(b8, _FakePkg.CascadeBackend)
    assert b8.dram_slots == 20 and b8.directory == str(tmp_path)


def test_meminfo_is_read():
    assert D.host_memory_available() > 0


def test_numa_binding_without_gpu_is_a_noop():
    out = D.bind_local_numa(0)
    assert out["cpus"] is None and out["numa_node"] is None
