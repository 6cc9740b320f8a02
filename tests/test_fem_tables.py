"""Host tables of the device assembly (paper_2302_10917_b200/fem.py) against the
reference's fem_basis / assembly helpers (tests/golden/fem_tables.npz, made by
tests/golden/make_golden.py fem).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from paper_2302_10917_b200 import fem

CASES = ((1, 1), (2, 2), (3, 2), (2, 3), (1, 4), (2, 5))


@pytest.mark.parametrize("m,p", CASES)
def test_reference_element_tables_bit_exact(m, p):
    g = golden("fem_tables.npz")
    for deg in (2 * p + 1, 2 * p + 2):
        key = f"m{m}p{p}d{deg}"
        tab = fem.asm_tables(m, p, deg)
        assert np.array_equal(tab.qp, g[key + "_qp"])
        assert np.array_equal(tab.qw, g[key + "_qw"])
        assert np.array_equal(tab.val, g[key + "_val"])
        assert np.array_equal(tab.gref, g[key + "_grad"])
        assert np.array_equal(tab.href, g[key + "_hess"])
    tab = fem.asm_tables(m, p, 2 * p + 1)
    assert np.array_equal(tab.cell_map, g[f"m{m}p{p}_cell_map"])
    assert np.array_equal(tab.edge_nodes, g[f"m{m}p{p}_edge_nodes"])
    assert np.array_equal(tab.fs, g[f"m{m}p{p}_face_s"])  # incl. the m = 3 sliver segments
    assert np.array_equal(tab.fw[0, :tab.fs.size], g[f"m{m}p{p}_face_w"])
    assert np.array_equal(tab.th_fwd, g[f"m{m}p{p}_trace"])


@pytest.mark.parametrize("m,p", CASES)
def test_dirichlet_projection(m, p):
    g = golden("fem_tables.npz")
    fn = lambda x: np.cos(2.0 * x[:, 0]) + x[:, 1] ** 2  # noqa: E731
    gh = fem.dirichlet_projection(g[f"m{m}p{p}_dface_verts"], fn, p, m)
    ref = g[f"m{m}p{p}_ghat"]
    assert np.abs(gh - ref).max() <= 1e-13 * np.abs(ref).max()


def test_patch_dof_counts():
    for m in range(1, 5):
        for p in range(1, 6):
            assert fem.patch_dof_map(m, p)[4] == (m * p + 1) * (m * p + 2) // 2
