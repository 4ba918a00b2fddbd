"""CPU: the C-ABI library builds for sm_100a, loads, exports every symbol the
header declares, and rejects bad configurations before touching a device."""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpfd_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpfd_b200_\w+)\s*\(", txt)))


def test_exports_every_header_symbol(b200):
    L = b200.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="no cuobjdump")
def test_fatbin_is_sm100a(b200):
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", b200.library_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_presets_match_reference_table(b200):
    for name, (q, rk, res, wk) in po.PRESETS.items():
        p = b200.resolve_preset(name)
        assert (p.q_vector, p.rk_arrays, p.residuals, p.wk_arrays) == (q, rk, res, wk)
    for bad in ("QP", "spdp", ""):
        with pytest.raises(b200.ConfigError):
            b200.resolve_preset(bad)


def test_split_presets(b200):
    for name, w in po.SPLITS.items():
        s = b200.split_preset(name)
        assert (s.alpha, s.beta_rho, s.beta_u, s.beta_phi, s.gamma_rho, s.gamma_u,
                s.gamma_phi) == tuple(float(x) for x in w)
    with pytest.raises(b200.ConfigError):
        b200.split_preset("Upwind")


def _solver(b200, n=16, prec=None, split="Blaisdell", flow=None, decomp=None, strategy="storesome"):
    return b200.Solver(b200.GridSpec(n) if isinstance(n, int) else n,
                       prec or b200.resolve_preset("DP"), strategy,
                       flow or b200.FlowParams(), split, decomp)


def test_config_errors_before_device(b200):
    with pytest.raises(b200.ConfigError):
        b200.GridSpec(4)
    with pytest.raises(b200.ConfigError):  # inconsistent split (physics.cpp:479-480)
        _solver(b200, split=b200.SplitCoefficients(0.5, 0, 0, 0, 0, 0, 0))
    with pytest.raises(b200.ConfigError):  # FlowParams::validate
        _solver(b200, flow=b200.FlowParams(mach=-1.0))
    with pytest.raises(b200.ConfigError):  # class combination outside the presets
        _solver(b200, prec=b200.PrecisionConfig(0, 2, 1, 0))
    p = b200.resolve_preset("HPSP")
    p.custom_overrides = {"rho": po.B64}
    with pytest.raises(b200.ConfigError):  # per-component Q override
        _solver(b200, prec=p)
    with pytest.raises(b200.ConfigError):  # n not divisible by pz
        _solver(b200, n=18, decomp=b200.Decomposition(pz=4))
    with pytest.raises(b200.ConfigError):  # slab thinner than the halo
        _solver(b200, n=16, decomp=b200.Decomposition(pz=8))
    with pytest.raises(b200.ConfigError):
        _solver(b200, strategy="fast")


def test_halo_plan_arithmetic(b200):
    L = b200.lib()
    out = (C.c_longlong * 9)()
    assert L.mpfd_b200_halo_plan(64, 4, 1, 4, out) == 0
    send_up, recv_lo, send_dn, recv_hi, blk, up, dn, z0, nzl = list(out)
    plane5 = 5 * 64 * 64 * 4
    assert (nzl, z0, up, dn) == (16, 16, 2, 0)
    assert blk == 4 * plane5
    assert send_up == 16 * plane5 and recv_lo == 0
    assert send_dn == 4 * plane5 and recv_hi == 20 * plane5
    assert L.mpfd_b200_halo_plan(64, 3, 0, 4, out) == 1  # not divisible


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    """The product path fails loudly without its extension."""
    import paper_2505_20911_b200.solver as sv

    monkeypatch.setattr(sv, "library_path", str(tmp_path / "missing.so"))
    monkeypatch.setattr(sv, "_lib", None)
    with pytest.raises(ImportError):
        sv.lib()
    # monkeypatch restores the loaded library afterwards (no module reload:
    # that would leave the ctypes argtypes on classes the callers no longer use)
