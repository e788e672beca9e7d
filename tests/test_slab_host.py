"""z-slab decomposition host logic on CPU (gloo, world_size 2 and 4): geometry, halo exchange of the
vmult's K face planes, ghost-cell refresh of the smoother's extended slabs, all-reduced dots and the
coarse-level all-gather (paper_2407_09621_b200/slab.py)."""
import pytest

import paper_2407_09621_b200 as sf
from paper_2407_09621_b200 import slab

from slab_launch import run


def test_slab_levels_geometry():
    hier = sf.build_hierarchy(5, 1)
    for G in (1, 2, 4, 8):
        sls = [slab.slab_levels(hier, r, G) for r in range(G)]
        for lvl in sls[0]:
            n = hier.n_cells(lvl)
            assert sum(s[lvl].nz for s in sls) == n
            assert all(s[lvl].nz % 2 == 0 and s[lvl].nz >= 2 for s in sls)
            assert [s[lvl].z0 for s in sls] == [r * n // G for r in range(G)]
            assert sls[0][lvl].h_lo == 0 and sls[-1][lvl].h_hi == 0
            if G > 1:
                assert sls[0][lvl].h_hi == slab.GHOST_CELLS and sls[-1][lvl].h_lo == slab.GHOST_CELLS
        # distributable levels are a contiguous range ending at the finest level
        lv = sorted(sls[0])
        assert lv == list(range(lv[0], 6)) if lv else True
    # 8 ranks: level 4 (16 cells) is the lowest with 2-cell slabs
    assert min(slab.slab_levels(hier, 0, 8)) == 4
    assert min(slab.slab_levels(hier, 0, 1)) == 1


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_and_reductions_gloo(world):
    res = run(world, "--case", "host", "--degree", "1", "--level", "4", timeout=300)
    for r in res:
        assert r["ghost_cells_ok"], r
        assert r["face_planes_ok"], r
        assert r["gather_ok"], r
        assert r["dot_rel_err"] < 1e-14, r
        assert r["levels"] == res[0]["levels"]
