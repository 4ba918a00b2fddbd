"""y pencils: a 1 x py x pz process grid (ProcessGrid, config.hpp:33) with
y ghost rows in HBM, exchanged by pack / peer-copy / unpack kernels before
the z planes (fill_halos_periodic, field.cpp:9-48, distributed), on the
staged path.  Every decomposition must give the reference's state, series
and divergence event bit for bit."""
import numpy as np
import pytest

import pyoracle as po
from test_gpu_parity import CODES, assert_state, b200_solver, checker, same_bits

GRIDS = [(1, 2), (2, 2), (1, 3), (2, 4)]  # (pz, py)


@pytest.mark.gpu
@pytest.mark.parametrize("pz,py", GRIDS)
@pytest.mark.parametrize("preset", ["DP", "HPSP"])
def test_pencils_bitwise(b200, preset, pz, py):
    n, dt = 24, 0.002
    s = b200_solver(b200, n, preset, decomp=b200.Decomposition(pz=pz, py=py), path="staged")
    c = checker(n, preset=preset)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(dt, 3, 1))
    _, series, _, _ = c.advance(dt, 3, 1)
    assert not r.diverged
    assert_state(s, c, (0, 1, 2), f"{preset} pencils {pz}x{py}")
    got = np.array([[x.t, x.kinetic_energy, x.enstrophy] for x in r.series])
    assert same_bits(got, series[:, :3])
    # the reference Field carrier of Q, x/y/z halos included (field.hpp:45-51)
    if po.ref_available():
        for comp in range(5):
            assert same_bits(s.get_field_ext(0, comp), c.field_ext(0, comp))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["default", "storesome"])
def test_pencils_chunk_aligned_diagnostics(b200, strategy):
    """128^3 on 2 x 2 pencils: every pencil-plane holds whole 4096-point
    chunks, so the diagnostics gather chunk sums and reorder them into the
    global scan order -- still the reference's tree bit for bit."""
    n, dt = 128, 0.001
    s = b200_solver(b200, n, "SPDP", strategy=strategy, decomp=b200.Decomposition(pz=2, py=2), path="staged")
    c = checker(n, preset="SPDP", strategy=strategy)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(dt, 2, 1))
    _, series, _, _ = c.advance(dt, 2, 1)
    assert_state(s, c, (0, 1), f"SPDP {strategy} 128^3 pencils")
    got = np.array([[x.t, x.kinetic_energy, x.enstrophy] for x in r.series])
    assert same_bits(got, series[:, :3])


@pytest.mark.gpu
def test_pencils_divergence(b200):
    kw = dict(preset="DP", split="Divergence", viscous=False, mach=0.4)
    s = b200_solver(b200, 16, decomp=b200.Decomposition(pz=2, py=2), path="staged", **kw)
    c = checker(16, **kw)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(0.2, 400, 10))
    st, series, ev, it = c.advance(0.2, 400, 10)
    assert r.diverged and st == 2
    e = r.divergence
    assert [CODES[e.what], e.i, e.j, e.k, e.iteration, e.substep] == ev
    assert r.iterations_run == it


def test_pencil_config_errors(b200):
    with pytest.raises(b200.ConfigError):  # ny not divisible
        b200_solver(b200, 16, decomp=b200.Decomposition(pz=1, py=3))
    with pytest.raises(b200.ConfigError):  # pencils thinner than the halo
        b200_solver(b200, 16, decomp=b200.Decomposition(pz=1, py=8))
