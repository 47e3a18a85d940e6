"""The edge-case sets of tests/edge_sets.py through the oracle alone: their expected outcomes
(closed form or listing-defect reading) and their grazing-band exclusion level, which the GPU
parity tests (test_gpu_edge.py) assert at 0."""
import numpy as np
import pytest

import oracle
from tests import edge_sets as es
from tests.parity import oracle_exclusions
from tests.test_oracle_closed_forms import finite_cylinder_hit
from workloads import gen


def _o(rays, ctrl, radii, depth):
    return oracle.intersect(rays, ctrl, radii, gen.make_pairs_1seg(rays.shape[0]), depth)


@pytest.mark.parametrize("depth", [0, 4, 16, 23])
def test_edge_sets_have_no_exclusions(depth):
    sets = [es.straight(a) for a in [(1, 0, 0), (0, 1, 0), (0, 0, 1)]]
    sets += [es.axial(), es.inside("A"), es.inside("C"), es.scaled("A"), es.scaled("C")]
    for rays, ctrl, radii in sets:
        o = _o(rays, ctrl, radii, depth)
        assert oracle_exclusions(o) == 0
    # perpendicular rays exactly ON a cap plane within the radius are in the band by
    # definition (the +eps run's cap moved out, the -eps run's in); nothing else is
    rays, ctrl, radii = es.perpendicular()
    o = _o(rays, ctrl, radii, depth)
    assert oracle_exclusions(o) == es.perpendicular_on_cap(rays).sum() == o["grazing"].sum() == 2


def test_perpendicular_and_axial_closed_form():
    for rays, ctrl, radii in (es.perpendicular(), es.axial()):
        A, B = ctrl[0, 0].astype(float), ctrl[0, 3].astype(float)
        for depth in (0, 9, 23):
            o = _o(rays, ctrl, radii, depth)
            on_cap = es.perpendicular_on_cap(rays)
            for i, ry in enumerate(rays.astype(np.float64)):
                if on_cap[i]:
                    continue  # in the band by definition (t depends on the cap's side)
                inside = abs(ry[1]) ** 2 + abs(ry[2]) ** 2 < 0.01 and 0 < ry[0] < 6
                e = None if inside else finite_cylinder_hit(ry[:3], ry[4:7], A, B, float(radii[0, 0]))
                if inside:
                    assert o["kind"][i] == oracle.KIND_INSIDE and o["t"][i] == 0
                elif e is None:
                    assert not o["hit"][i]
                else:
                    assert o["hit"][i] and abs(o["t"][i] - e[0]) <= 1e-12 * max(1, e[0])
                    assert o["kind"][i] == e[3]


def test_scaled_directions_follow_d_as_given():
    """Scaling d by s divides t by s and leaves u and n unchanged (t along d as given)."""
    rays, ctrl, radii = es.scaled("A")
    unit = rays.copy()
    unit[:, 4:7] /= np.linalg.norm(rays[:, 4:7].astype(np.float64), axis=1, keepdims=True)
    s = np.linalg.norm(rays[:, 4:7].astype(np.float64), axis=1)
    unit[:, 3] = np.inf
    a = _o(rays, ctrl, radii, 9)
    b = _o(unit, ctrl, radii, 9)
    m = a["hit"]
    assert m.sum() > 300
    assert np.all(b["hit"][m])
    assert np.allclose(a["t"][m] * s[m], b["t"][m], rtol=1e-6)
    assert np.allclose(a["u"][m], b["u"][m], atol=1e-6)
