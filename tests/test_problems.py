"""The seeded input generators: determinism, decomposition independence,
value ranges, and the structural properties the recipes promise."""
import numpy as np
import pytest

from problems import get_workload, slab_range, splitmix64, uniform
from problems.stencils import porous7, void_fraction


def _splitmix_python(x):
    """Independent pure-Python (arbitrary-precision int) splitmix64."""
    M = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_splitmix_matches_bigint_reference():
    xs = [0, 1, 2, 12345, (1 << 40) * 1000 + 77, (1 << 64) - 1]
    got = splitmix64(np.array(xs, dtype=np.uint64))
    assert [int(v) for v in got] == [_splitmix_python(x) for x in xs]


def test_uniform_range_and_moments():
    u = uniform(0, np.arange(1 << 20, dtype=np.uint64))
    assert u.min() >= -1.0 and u.max() < 1.0
    assert abs(u.mean()) < 5e-3 and abs(u.var() - 1 / 3) < 5e-3


@pytest.mark.parametrize("name", ["c2s", "c3s", "c4s"])
def test_slab_generation_is_decomposition_independent(name):
    prob = get_workload(name).problem()
    full_a = prob.bands(epoch=1)
    full_b = prob.rhs(2)
    for P in (2, 3, 4):
        for r in range(P):
            z0, z1 = slab_range(prob.nz, r, P)
            assert np.array_equal(prob.bands(z0, z1, epoch=1), full_a[:, z0:z1])
            assert np.array_equal(prob.rhs(2, z0, z1), full_b[z0:z1])


def test_channel_rhs_mean_free_and_pinned():
    prob = get_workload("c2s").problem()
    for t in (0, 3):
        b = prob.rhs(t).reshape(-1)
        assert b[0] == 0.0
        assert abs(b[1:].mean()) < 1e-15


def test_porous_void_fraction_near_quarter():
    prob = porous7(64, 6)
    assert abs(void_fraction(prob) - 0.25) < 0.03


def test_epoch_perturbation_relative_size():
    prob = get_workload("c4s").problem()
    a0, a1 = prob.bands(epoch=0), prob.bands(epoch=1)
    nz = a0 != 0
    rel = np.abs(a1[nz] / a0[nz] - 1)
    assert rel.max() <= 1e-3 and rel.max() > 5e-4
    assert np.array_equal(a0 == 0, a1 == 0)
