"""Device-side level-0 planner (csrc/gpu_plan.cu) against the host planner
(csrc/planner.cpp, itself pinned to the reference's classify_active group order by
tests/test_capi.py): every level-0 plan array -- groups in classify order with ascending members
(hierarchy.py:124-145), block pattern with elimination fill, adjacency, pool offsets, cell lists,
Schur contribution lists in cell order, scaling blocks, skeleton neighbour / dependency lists and
wavefronts -- must be identical, at test sizes and at the full BASELINE sizes."""
import ctypes as C

import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_1808_01364_b200 import _lib  # noqa: E402
from paper_1808_01364_b200 import factorization as gfac  # noqa: E402
from paper_1808_01364_b200.grid import GridSpec, assemble_operator, baseline_problem, generate_field  # noqa: E402

CASES = [("2d-n32-m4", 2, 32, 4, None), ("3d-n16-m4", 3, 16, 4, None), ("c1", None, None, None, "c1"),
         ("c2", None, None, None, "c2"), ("c4", None, None, None, "c4"), ("c5", None, None, None, "c5")]


@pytest.mark.parametrize("name,dim,n,m,cfg", CASES, ids=[c[0] for c in CASES])
def test_device_plan_equals_host_plan(name, dim, n, m, cfg):
    if cfg:
        spec, A, _ = baseline_problem(cfg, 0, None)
    else:
        spec = GridSpec(dim, n, m)
        A = assemble_operator(generate_field(spec, 1))
    dm = gfac.device_matrix(A)
    buf = C.create_string_buffer(4096)
    bad = _lib.lib().phif_plan_check(dm.handle, spec.dim, spec.n, spec.m, buf, 4096)
    assert bad == 0, buf.value.decode()
