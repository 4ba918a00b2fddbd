"""GPU parity: the B200 solver against the reference itself (oracle/_ref) and
the C restatement (oracle/), bit for bit.

Contract (parity build): Q, Qt and R are *bitwise*
equal to the reference after every substep, for every preset x emulation x
strategy; diagnostics agree bitwise on bitwise-equal states (same reduction
tree).  Checkers are run on the same seeded/deterministic inputs.
"""
import os

import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu

PRESETS = list(po.PRESETS)
EMUL = ["strict", "storeround"]
STRATS = ["default", "storesome"]


def checker(n, **kw):
    """The reference library when present, else the (reference-pinned) oracle."""
    if po.ref_available():
        return po.Reference(n, **kw)
    kw.pop("threads", None)
    return po.Oracle(n, **kw)


def b200_solver(m, n, preset="DP", emulation="strict", strategy="storesome", split="Blaisdell",
                mach=0.1, re=1600.0, pr=0.72, gamma=1.4, viscous=True, overrides=None,
                decomp=None, path=None):
    prec = m.resolve_preset(preset, emulation)
    if overrides:
        prec.custom_overrides = {k: po.KIND_NAMES[v] for k, v in overrides.items()}
    s = m.Solver(m.GridSpec(n), prec, strategy, m.FlowParams(mach, re, pr, gamma, viscous), split,
                 decomp)
    if path:
        s.set_path(path)
    return s


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


def assert_state(s, c, classes=(0, 1, 2), ctx=""):
    for cls in classes:
        for comp in range(5):
            g, r = s.get_field(cls, comp), c.field(cls, comp)
            if not same_bits(g, r):
                bad = np.argwhere(g.view(np.uint64) != r.view(np.uint64))
                k, j, i = bad[0]
                raise AssertionError(
                    f"{ctx} class {cls} comp {comp}: {len(bad)} mismatches, first (i,j,k)=({i},{j},{k})"
                    f" gpu={g[k, j, i]!r} ref={r[k, j, i]!r}")


def test_double_rounding_kat(b200):
    """Stores round once from binary64 (test_precision.cpp:141-146)."""
    s = b200_solver(b200, 8, "HP")
    x = 1.0 + 2.0**-11 + 2.0**-40
    s.set_field(0, 0, np.full((8, 8, 8), x))
    assert s.get_field(0, 0)[0, 0, 0] == 1.0 + 2.0**-10
    s.set_field(0, 0, np.full((8, 8, 8), 65520.0))
    assert np.isinf(s.get_field(0, 0)[0, 0, 0])
    s.set_field(0, 0, np.full((8, 8, 8), 2.0**-25))
    assert s.get_field(0, 0)[0, 0, 0] == 0.0


@pytest.mark.parametrize("preset", PRESETS)
def test_init_tgv(b200, preset):
    s = b200_solver(b200, 16, preset)
    s.init_tgv()
    c = checker(16, preset=preset)
    c.init()
    assert_state(s, c, (0, 1, 2), f"init {preset}")


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("emulation", EMUL)
@pytest.mark.parametrize("preset", PRESETS)
def test_substeps_bitwise(b200, preset, emulation, strategy):
    """evaluate -> rk_substep -> halo fill, 2 RK steps, every substep compared."""
    n, dt = 16, 0.002
    kw = dict(preset=preset, emulation=emulation, strategy=strategy)
    s = b200_solver(b200, n, **kw)
    c = checker(n, **kw)
    s.init_tgv()
    c.init()
    for it in range(2):
        for sub in range(3):
            assert s.evaluate() is None
            assert c.evaluate()[0] == 0
            assert_state(s, c, (2,), f"{kw} it{it} sub{sub} R")
            assert s.rk_substep(sub, dt) is None
            c.rk_substep(sub, dt)
            s.fill_state_halos()
            assert_state(s, c, (0, 1), f"{kw} it{it} sub{sub} Q/Qt")


@pytest.mark.parametrize("split", list(po.SPLITS))
@pytest.mark.parametrize("viscous", [True, False])
def test_splits(b200, split, viscous):
    kw = dict(preset="HPSP", split=split, viscous=viscous, mach=0.4)
    s = b200_solver(b200, 12, **kw)
    c = checker(12, **kw)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(0.004, 2, 0))
    st, _, _, _ = c.advance(0.004, 2, 0)
    assert not r.diverged and st == 0
    assert_state(s, c, (0, 1), f"split {split} visc {viscous}")


def test_overrides(b200):
    """wk-array name overrides (precision.cpp:46-56) are honoured."""
    ov = {"T": "B32", "dudx": "B32", "u": "B16"}
    for strategy in STRATS:
        kw = dict(preset="HPSP", strategy=strategy, overrides=ov)
        s = b200_solver(b200, 12, **kw)
        c = checker(12, **kw)
        s.init_tgv()
        c.init()
        s.advance(b200.StepConfig(0.003, 2, 0))
        c.advance(0.003, 2, 0)
        assert_state(s, c, (0, 1), f"overrides {strategy}")


@pytest.mark.parametrize("threads", [1, 8])
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_advance_series(b200, preset, threads):
    """advance with sampling: identical K / enstrophy series (same tree)."""
    n = 32
    s = b200_solver(b200, n, preset)
    c = checker(n, preset=preset, threads=threads) if po.ref_available() else checker(n, preset=preset)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(0.002, 6, 2), threads=threads)
    st, series, _, it = c.advance(0.002, 6, 2, threads=threads)
    assert not r.diverged and st == 0 and r.iterations_run == it == 6
    got = np.array([[x.t, x.kinetic_energy, x.enstrophy, x.eps_s] for x in r.series])
    assert got.shape[0] == series.shape[0]
    assert same_bits(got, series[:, :4])
    assert_state(s, c, (0, 1), f"advance {preset}")


def test_diagnostics_kat(b200):
    """K(0) = 0.125, eps_S(0) at Re=800."""
    s = b200_solver(b200, 64, "DP", mach=0.5, re=800.0)
    s.init_tgv()
    d = s.diagnostics(0, 0.0, 8)
    assert abs(d.kinetic_energy - 0.125) < 1e-12
    assert abs(d.eps_s - 9.375e-4) / 9.375e-4 < 1e-5


@pytest.mark.parametrize("preset", ["DP", "HPSP", "HP"])
def test_uniform_state_zero_residual(b200, preset):
    """Uniform quiescent state -> R == 0 exactly."""
    for strategy in STRATS:
        s = b200_solver(b200, 16, preset, strategy=strategy)
        s.init_uniform()
        assert s.evaluate() is None
        for comp in range(5):
            assert np.all(s.get_field(2, comp) == 0.0)


CODES = {"nonpositive or nonfinite density": 1, "nonfinite residual": 2, "nonfinite state": 3}


def _divergence_run(b200, preset, exact, pz=1, path=None, overlap=None):
    kw = dict(preset=preset, split="Divergence", viscous=False, mach=0.4)
    s = b200_solver(b200, 16, decomp=b200.Decomposition(pz=pz) if pz > 1 else None, path=path, **kw)
    if overlap is not None:
        s.set_overlap(overlap)
    if exact:
        s.set_exact_divergence(True)
    c = checker(16, **kw)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(0.2, 400, 10))
    st, series, ev, it = c.advance(0.2, 400, 10)
    assert r.diverged and st == 2
    e = r.divergence
    assert [CODES[e.what], e.i, e.j, e.k, e.iteration, e.substep] == ev
    assert r.iterations_run == it
    got = np.array([[x.t, x.kinetic_energy, x.enstrophy, x.eps_s, x.diverged] for x in r.series])
    np.testing.assert_array_equal(np.isnan(got), np.isnan(series))
    assert same_bits(np.nan_to_num(got), np.nan_to_num(series))
    return s, c, CODES[e.what]


@pytest.mark.parametrize("preset", ["DP", "HP"])
def test_divergence_event(b200, preset):
    """Inviscid Divergence split blows up: same event, iteration and series;
    in exact-divergence mode Q, Qt and R at the event are the reference's."""
    s, c, _ = _divergence_run(b200, preset, exact=True)
    assert_state(s, c, (0, 1, 2), "divergence (exact)")


@pytest.mark.parametrize("preset", ["DP", "HP"])
def test_divergence_event_lean(b200, preset):
    """Default (lean) layout -- Qt in place, R on demand: the event, the series
    and Q are the reference's; Qt for a nonfinite-state event and R for
    nonfinite-residual / nonfinite-state events too (mpfd_b200.h)."""
    s, c, code = _divergence_run(b200, preset, exact=False)
    assert_state(s, c, (0,), "divergence (lean) Q")
    if code == 3:
        assert_state(s, c, (1,), "divergence (lean) Qt")
    if code in (2, 3):
        assert_state(s, c, (2,), "divergence (lean) R")


@pytest.mark.parametrize("pz", [2, 4])
def test_divergence_event_slabs(b200, pz):
    """Several z-slabs (overlapped exchange): the records of every slab merge
    into the reference's first event; in exact mode the slabs run in
    lock-step per substep and the whole state at the event is the
    reference's."""
    s, c, _ = _divergence_run(b200, "DP", exact=True, pz=pz, overlap=True)
    assert_state(s, c, (0, 1, 2), f"divergence pz={pz} (exact)")
    _divergence_run(b200, "DP", exact=False, pz=pz, overlap=True)
    _divergence_run(b200, "DP", exact=False, pz=pz)  # default: exchange first on one device


def test_divergence_event_staged(b200):
    """The staged (one kernel per level) path stops at the same event."""
    s, c, _ = _divergence_run(b200, "DP", exact=False, path="staged")
    assert_state(s, c, (0, 1, 2), "divergence (staged)")


@pytest.mark.parametrize("pz", [2, 4])
def test_local_slabs_bitwise(b200, pz):
    """z-slab decomposition on one device: bitwise equal to one slab."""
    n = 32
    one = b200_solver(b200, n, "HPSP")
    many = b200_solver(b200, n, "HPSP", decomp=b200.Decomposition(pz=pz))
    one.init_tgv()
    many.init_tgv()
    r1 = one.advance(b200.StepConfig(0.002, 4, 2))
    r2 = many.advance(b200.StepConfig(0.002, 4, 2))
    for cls in (0, 1):
        for comp in range(5):
            assert same_bits(one.get_field(cls, comp), many.get_field(cls, comp))
    a = [(x.kinetic_energy, x.enstrophy) for x in r1.series]
    b = [(x.kinetic_energy, x.enstrophy) for x in r2.series]
    assert a == b


@pytest.mark.parametrize("pz", [2, 3, 4])
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_overlapped_exchange_bitwise(b200, preset, pz):
    """Interior launch overlapped with the ghost-plane exchange, boundary
    launches after it: bitwise equal to the exchange-first schedule and to
    one slab, state and diagnostics series."""
    n = 48
    one = b200_solver(b200, n, preset)
    ov = b200_solver(b200, n, preset, decomp=b200.Decomposition(pz=pz))
    ov.set_overlap(True)
    seq = b200_solver(b200, n, preset, decomp=b200.Decomposition(pz=pz))
    seq.set_overlap(False)
    runs = []
    for s in (one, ov, seq):
        s.init_tgv()
        runs.append(s.advance(b200.StepConfig(0.002, 5, 2)))
    for cls in (0, 1):
        for comp in range(5):
            a = one.get_field(cls, comp)
            assert same_bits(a, ov.get_field(cls, comp)), (cls, comp)
            assert same_bits(a, seq.get_field(cls, comp)), (cls, comp)
    ser = [[(x.kinetic_energy, x.enstrophy) for x in r.series] for r in runs]
    assert ser[0] == ser[1] == ser[2]


@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_weak_scaling_grid_replicates(b200, preset):
    """z_periods = P stacked TGV periods on P slabs (the weak-scaling
    configuration): every period is bitwise the single-cube run, and K is
    the cube's K (same mean over P exact copies, within 1 ulp-scale sums)."""
    n, P = 24, 3
    one = b200_solver(b200, n, preset)
    big = b200.Solver(b200.GridSpec(n, z_periods=P), b200.resolve_preset(preset), "storesome",
                      b200.FlowParams(0.1, 1600.0, 0.72, 1.4, True), "Blaisdell",
                      decomp=b200.Decomposition(pz=P))
    one.init_tgv()
    big.init_tgv()
    r1 = one.advance(b200.StepConfig(0.002, 3, 3))
    r2 = big.advance(b200.StepConfig(0.002, 3, 3))
    for cls in (0, 1):
        for comp in range(5):
            a = one.get_field(cls, comp)
            b = big.get_field(cls, comp)
            assert b.shape == (n * P, n, n)
            for k in range(P):
                assert same_bits(a, b[k * n:(k + 1) * n]), (cls, comp, k)
    for x, y in zip(r1.series, r2.series):
        assert abs(x.kinetic_energy - y.kinetic_energy) <= 1e-14 * abs(x.kinetic_energy)
        assert abs(x.enstrophy - y.enstrophy) <= 1e-13 * abs(x.enstrophy)
    e = big.get_field_ext(0, 0)
    assert e.shape == (n * P + 8, n + 8, n + 8)


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_64_cubed_step(b200, preset):
    """One full RK step at 64^3 (config C1 size) against the reference."""
    n = 64
    s = b200_solver(b200, n, preset)
    c = checker(n, preset=preset)
    s.init_tgv()
    c.init()
    s.advance(b200.StepConfig(0.002, 1, 0))
    c.advance(0.002, 1, 0)
    assert_state(s, c, (0, 1), f"64^3 {preset}")


@pytest.mark.parametrize("emulation", EMUL)
@pytest.mark.parametrize("preset", PRESETS)
def test_fused_64_every_plan(b200, preset, emulation):
    """Every precision plan on the kernels a 64-multiple grid selects (the
    TMA-staged warp-specialised fp16 kernel where Q is fp32, the cp.async
    one where Q is fp16, the fp32 and fp64 kernels): one RK step against the
    reference, Q and Qt bit for bit."""
    n, dt = 64, 0.002
    kw = dict(preset=preset, emulation=emulation)
    s = b200_solver(b200, n, path="fused", **kw)
    c = checker(n, **kw)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(dt, 1, 0))
    st, _, _, _ = c.advance(dt, 1, 0)
    assert not r.diverged and st == 0
    assert_state(s, c, (0, 1), f"fused 64^3 {kw}")


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("emulation", EMUL)
@pytest.mark.parametrize("preset", PRESETS)
def test_fused_path_bitwise(b200, preset, emulation, strategy):
    """The fused residual + RK kernel over 2 steps (6 substeps) on a grid
    that is not a multiple of the 32x8 tile, plus R of the last substep."""
    n, dt = 20, 0.002
    kw = dict(preset=preset, emulation=emulation, strategy=strategy)
    s = b200_solver(b200, n, path="fused", **kw)
    c = checker(n, **kw)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(dt, 2, 0))
    st, _, _, _ = c.advance(dt, 2, 0)
    assert not r.diverged and st == 0
    assert_state(s, c, (0, 1, 2), f"fused {kw}")


@pytest.mark.parametrize("pz", [1, 2])
@pytest.mark.parametrize("path", ["fused", "staged"])
def test_paths_agree_64(b200, path, pz):
    """Both paths, one and two slabs, 3 steps at 64^3 DP and HPSP."""
    for preset in ("DP", "HPSP"):
        s = b200_solver(b200, 64, preset, path=path, decomp=b200.Decomposition(pz=pz))
        c = checker(64, preset=preset)
        s.init_tgv()
        c.init()
        s.advance(b200.StepConfig(0.002, 3, 0))
        c.advance(0.002, 3, 0)
        assert_state(s, c, (0, 1), f"{path} pz{pz} {preset}")


def test_nccl_transport_single_rank(b200):
    """The NCCL code path (dlopen, ncclCommInitRank, grouped send/recv of the
    ghost planes, allgather of diagnostics partials, allreduce of the
    divergence record) with one rank exchanging with itself: bitwise equal
    to the LOCAL path."""
    n = 32
    ref = b200_solver(b200, n, "HPSP")
    nid = b200.Solver.nccl_unique_id()
    nc = b200_solver(b200, n, "HPSP", decomp=b200.Decomposition(pz=1, mode=1, rank=0, nccl_id=nid))
    ref.init_tgv()
    nc.init_tgv()
    r1 = ref.advance(b200.StepConfig(0.002, 4, 2))
    r2 = nc.advance(b200.StepConfig(0.002, 4, 2))
    for cls in (0, 1):
        for comp in range(5):
            assert same_bits(ref.get_field(cls, comp), nc.get_field(cls, comp))
    assert [(x.kinetic_energy, x.enstrophy) for x in r1.series] == \
           [(x.kinetic_energy, x.enstrophy) for x in r2.series]
    # measured halo volume (mpfd_b200_halo_bytes): every exchange is two
    # ncclSend messages of 4 ghost planes x 5 components in q storage (fp32
    # in HPSP); at least one exchange per substep (4 steps x 3 substeps)
    blk = 4 * 5 * n * n * 4
    sent = nc.halo_bytes()
    assert sent % (2 * blk) == 0 and sent >= 2 * blk * 4 * 3
    assert ref.halo_bytes() == 0
    # divergence through the NCCL reduction of the event record
    kw = dict(preset="DP", split="Divergence", viscous=False, mach=0.4)
    a = b200_solver(b200, 16, **kw)
    b = b200_solver(b200, 16, decomp=b200.Decomposition(pz=1, mode=1, rank=0,
                                                        nccl_id=b200.Solver.nccl_unique_id()), **kw)
    a.init_tgv()
    b.init_tgv()
    ra = a.advance(b200.StepConfig(0.2, 400, 10))
    rb = b.advance(b200.StepConfig(0.2, 400, 10))
    assert ra.diverged and rb.diverged and ra.divergence == rb.divergence
    assert ra.iterations_run == rb.iterations_run


def _vs_reference(b200, n, preset, dt, steps, threads=None):
    """advance `steps` RK steps on the fused path the bench times and on the
    unmodified reference (oracle/_ref, all host threads); Q and Qt bit for bit."""
    threads = threads or os.cpu_count() or 8
    s = b200_solver(b200, n, preset)
    s.init_tgv()
    r = s.advance(b200.StepConfig(dt, steps, 0))
    assert not r.diverged
    c = checker(n, preset=preset, threads=threads)
    c.init()
    st, _, _, _ = c.advance(dt, steps, 0, threads=threads)
    assert st == 0
    for cls in (0, 1):
        for comp in range(5):
            g = s.get_field(cls, comp)
            ref = c.field(cls, comp)
            if not same_bits(g, ref):
                bad = np.argwhere(g.view(np.uint64) != ref.view(np.uint64))
                raise AssertionError(f"{n}^3 {preset} class {cls} comp {comp}: {len(bad)} mismatches")
            del g, ref
    s.close()


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_256_cubed_step_vs_reference(b200, preset):
    """BASELINE configs 2/3 (256^3 DP, SPDP; HPSP too): one RK step, bitwise
    against the reference at the size the bench's per-precision lines run at
    half scale (one step at 256^3)."""
    _vs_reference(b200, 256, preset, 5e-4, 1)


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_128_cubed_10_steps_vs_reference(b200, preset):
    """128^3, 10 RK steps, bitwise against the reference."""
    _vs_reference(b200, 128, preset, 1e-3, 10)


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_512_cubed_step_vs_reference(b200, preset):
    """The bench's workloads (TGV 512^3, BASELINE.json metric, every precision
    mode it reports): one RK step on the kernels the bench times, bitwise
    against the reference (22.5 GB of binary64 host carriers; the HPSP
    reference step emulates binary16 on the CPU, ~2 min on 16 threads)."""
    _vs_reference(b200, 512, preset, 2.5e-4, 1)


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_1024_cubed_fits_and_steps(b200, preset):
    """BASELINE configs[4] size on ONE B200: Q (double-buffered) + Qt in HBM
    (DP 129.9 GB), R and the diagnostics integrand never allocated; one RK
    step; size-independent checks -- the state stays finite, K stays the
    TGV's 1/8 to the decay of one step, and the solver holds exactly the
    lean footprint."""
    n = 1024
    s = b200_solver(b200, n, preset)
    bq, bt = {"DP": (8, 8), "SPDP": (8, 8), "HPSP": (4, 4)}[preset]
    q_bytes = (n + 8) * 5 * n * n * bq
    qt_bytes = 5 * n ** 3 * bt
    dev = s.memory()[0]
    assert 2 * q_bytes + qt_bytes <= dev <= 2 * q_bytes + qt_bytes + (1 << 30)
    s.init_tgv()
    d0 = s.diagnostics(0, 0.0, 8)
    r = s.advance(b200.StepConfig(1.25e-4, 1, 1))
    assert not r.diverged
    k0, k1 = r.series[0].kinetic_energy, r.series[-1].kinetic_energy
    assert k0 == d0.kinetic_energy and abs(k0 - 0.125) < 1e-6
    assert 0 < k0 - k1 < 1e-6 and np.isfinite(r.series[-1].enstrophy)
    assert s.memory()[0] == dev  # nothing allocated on the way
    s.close()


def test_lean_footprint_and_lazy_r(b200):
    """The fused path holds Q twice and Qt once; R appears only when read,
    bitwise the residual of the last substep's input; exact mode adds the
    Qt and R double buffers and returns them when switched off."""
    n = 32
    s = b200_solver(b200, n, "DP")
    c = checker(n, preset="DP")
    q_bytes, qt_bytes = (n + 8) * 5 * n * n * 8, 5 * n ** 3 * 8
    base = s.memory()[0]
    assert 2 * q_bytes + qt_bytes <= base <= 2 * q_bytes + qt_bytes + (8 << 20)
    s.init_tgv()
    c.init()
    assert np.all(s.get_field(2, 0) == 0.0) and s.memory()[0] == base
    s.advance(b200.StepConfig(0.002, 2, 0))
    c.advance(0.002, 2, 0)
    assert_state(s, c, (0, 1, 2), "lazy R")
    assert s.memory()[0] == base + qt_bytes  # R, allocated on the read
    s.set_exact_divergence(True)
    assert s.memory()[0] == base + 3 * qt_bytes
    s.advance(b200.StepConfig(0.002, 1, 0))
    c.advance(0.002, 1, 0)
    assert_state(s, c, (0, 1, 2), "exact mode")
    s.set_exact_divergence(False)
    assert s.memory()[0] == base + qt_bytes
    assert_state(s, c, (0, 1, 2), "exact mode off")
    s.advance(b200.StepConfig(0.002, 1, 0))
    c.advance(0.002, 1, 0)
    assert_state(s, c, (0, 1, 2), "lean again")


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_full_size_paths_agree(b200, preset):
    """BASELINE.json's 512^3 workload, one RK step: the fused kernel the bench
    times (warp-specialised for HPSP and SPDP, scalar fp64 for DP) and the staged one-kernel-per-level path -- two independent
    kernel implementations, each pinned bit for bit to the reference at small
    sizes -- leave bitwise identical Q and Qt at full size; the state stays
    finite and the density positive (a size-independent property check)."""
    n, dt = 512, 2.5e-4
    out = {}
    for path in ("fused", "staged"):
        s = b200_solver(b200, n, preset, path=path)
        s.init_tgv()
        r = s.advance(b200.StepConfig(dt, 1, 0))
        assert not r.diverged
        out[path] = [s.get_field(cls, comp) for cls in (0, 1) for comp in range(5)]
        s.close()
        del s
    for i, (a, b) in enumerate(zip(out["fused"], out["staged"])):
        assert same_bits(a, b), f"{preset} 512^3 class {i // 5} comp {i % 5}"
    rho = out["fused"][0]
    assert np.isfinite(rho).all() and (rho > 0).all()


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["DP", "SPDP", "HPSP"])
def test_history_64(b200, preset):
    """KE / enstrophy history contract: TGV 64^3,
    M=0.1, Re=1600, dt=0.002, t in [0, 0.5] sampled every 25 steps, against
    the reference -- bit for bit (the states are bitwise equal and the
    reduction tree is the reference's), far inside the stated tolerance
    (max rel dK, d enstrophy <= 1e-12); the fused kernels the bench times."""
    n, dt, steps, every = 64, 0.002, 250, 25
    s = b200_solver(b200, n, preset)
    c = checker(n, preset=preset, threads=8) if po.ref_available() else checker(n, preset=preset)
    s.init_tgv()
    c.init()
    r = s.advance(b200.StepConfig(dt, steps, every), threads=8)
    st, series, _, it = c.advance(dt, steps, every, threads=8)
    assert not r.diverged and st == 0 and r.iterations_run == it == steps
    got = np.array([[x.t, x.kinetic_energy, x.enstrophy, x.eps_s] for x in r.series])
    assert got.shape == (steps // every + 1, 4)
    assert same_bits(got, series[:, :4])
    rel = np.abs(got[:, 1:3] - series[:, 1:3]) / np.abs(series[:, 1:3])
    assert rel.max() <= 1e-12


@pytest.mark.parametrize("emulation", EMUL)
@pytest.mark.parametrize("preset", ["DP", "SPDP-wk", "SPDP-res", "HPSP", "HPSP-res", "HP"])
def test_materialised_default_gradients(b200, preset, emulation):
    """The reference's Default dataflow: the 12 ddx1-staged gradients
    (stencil.cpp:11-28 via physics.cpp:503-517) written to HBM at their wk
    storage, then read back by the level-2 kernel -- every substep's R, Q and
    Qt bit for bit the reference's, and the 12 arrays show up in the measured
    device bytes (the paper's memory table)."""
    n, dt = 16, 0.002
    kw = dict(preset=preset, emulation=emulation, strategy="default")
    s = b200_solver(b200, n, path="materialised", **kw)
    c = checker(n, **kw)
    s.init_tgv()
    c.init()
    before = s.memory()[0]
    for it in range(2):
        for sub in range(3):
            assert s.evaluate() is None
            assert c.evaluate()[0] == 0
            assert_state(s, c, (2,), f"{kw} it{it} sub{sub} R")
            assert s.rk_substep(sub, dt) is None
            c.rk_substep(sub, dt)
            s.fill_state_halos()
            assert_state(s, c, (0, 1), f"{kw} it{it} sub{sub} Q/Qt")
    planes, plane = n + 8, n * n
    # (res, wk) storage bytes; every staged gradient is exact at its wk storage
    res, wk = {"DP": (8, 8), "SPDP-wk": (8, 4), "SPDP-res": (4, 8), "HPSP": (2, 2), "HPSP-res": (2, 4),
               "HP": (2, 2)}[preset]
    lev2 = res if emulation == "strict" else 8  # level-2 fields at the residual compute type
    grown = s.memory()[0] - before
    # the 12 gradient arrays, primitives (5) and level-2 fields (7) with
    # ghost planes, and R (interior)
    assert grown == (12 * wk + 5 * wk + 7 * lev2) * planes * plane + 5 * n * plane * res


def test_materialised_rejects_wide_gradient_override(b200):
    prec = b200.resolve_preset("HPSP")
    prec.custom_overrides = {"dTdz": b200.B64}
    s = b200.Solver(b200.GridSpec(16), prec, "default", b200.FlowParams(0.1, 1600.0, 0.72, 1.4, True))
    with pytest.raises(b200.ConfigError):
        s.set_path("materialised")
