"""Host problem setup (paper_1808_01364_b200/grid.py) vs golden outputs of the reference grid.py."""
import numpy as np
import pytest

from paper_1808_01364_b200 import grid
from paper_1808_01364_b200.errors import ConfigurationError


def test_field_and_operator_golden(golden):
    for i in range(int(golden["grid_count"])):
        dim, n, m, seed, contrast, width, b = golden[f"grid_{i}_params"]
        spec = grid.GridSpec(int(dim), int(n), int(m))
        f = grid.generate_field(spec, int(seed), float(contrast), float(width))
        assert np.array_equal(f.values, golden[f"grid_{i}_field"])
        A = grid.assemble_operator(f, float(b))
        assert np.array_equal(A.csr.indptr, golden[f"grid_{i}_indptr"])
        assert np.array_equal(A.csr.indices, golden[f"grid_{i}_indices"])
        assert np.array_equal(A.csr.data, golden[f"grid_{i}_data"])


def test_gridspec_validation():
    for bad in [(4, 16, 4), (2, 16, 1), (2, 18, 4), (2, 24, 4), (2, 8, 8)]:
        with pytest.raises(ConfigurationError):
            grid.GridSpec(*bad)
    s = grid.GridSpec(3, 16, 4)
    assert s.levels == 2 and s.ndofs == 15 ** 3
    ids = np.arange(s.ndofs)
    assert np.array_equal(s.id_of(s.coords_of(ids)), ids)


def test_laplacian_stencil():
    spec = grid.GridSpec(2, 16, 4)
    f = grid.CoefficientField(spec, np.ones(spec.shape), 0, 1.0, 1.0)
    A = grid.assemble_operator(f).to_dense()
    i = spec.id_of([[5, 7]])[0]
    assert A[i, i] == 4.0 and sorted(A[i][A[i] != 0])[:4] == [-1.0] * 4
    spec3 = grid.GridSpec(3, 8, 4)
    A3 = grid.assemble_operator(grid.CoefficientField(spec3, np.ones(spec3.shape), 0, 1.0, 1.0)).to_dense()
    j = spec3.id_of([[3, 4, 5]])[0]
    assert A3[j, j] == 6.0 and np.count_nonzero(A3[j]) == 7
    assert np.array_equal(A, A.T)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_fields(name):
    cfg = grid.CONFIGS[name]
    small = {2: 32 if cfg.m == 8 else 64, 3: 16}[cfg.dim]
    spec, A, f = grid.baseline_problem(name, 0, small)
    assert f.values.shape == spec.shape and np.all(f.values > 0)
    if cfg.recipe.startswith("thresh"):
        assert set(np.unique(f.values)) <= {cfg_hi for cfg_hi in (1e3, 1e-3, 1e4, 1e-4)}
    assert abs(A.csr - A.csr.T).max() == 0.0
