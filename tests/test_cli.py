"""CLI level: `mpfd run <cfg>` (reference, oracle/_ref/mpfd) and the B200
drop-in `tools/mpfd_b200_run run <cfg>` write byte-identical diagnostics
CSVs (io.cpp:19-36) and the same exit codes (tools/mpfd.cpp:4-5)."""
import os
import subprocess

import pytest

import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "mpfd_b200_run")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "mpfd")


def build_tool(b200):
    src = os.path.join(ROOT, "tools", "mpfd_b200_run.cpp")
    if not os.path.exists(TOOL) or os.path.getmtime(TOOL) < max(
            os.path.getmtime(src), os.path.getmtime(b200.library_path)):
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-I" + os.path.join(ROOT, "include"), src,
                        "-L" + os.path.dirname(b200.library_path), "-lmpfd_b200",
                        "-Wl,-rpath," + os.path.dirname(b200.library_path), "-o", TOOL], check=True)
    return TOOL


def test_tool_builds_and_rejects_bad_config(b200, tmp_path):
    tool = build_tool(b200)
    bad = tmp_path / "bad.cfg"
    bad.write_text("nonsense_key = 42\n")  # tests/data/bad.cfg of the reference
    r = subprocess.run([tool, "run", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown key" in r.stderr


@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
def test_reference_cli_exit_codes(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("nonsense_key = 42\n")
    assert subprocess.run([REF_CLI, "run", str(bad)], capture_output=True).returncode == 1


CFGS = {
    "smoke_uniform": "case = uniform\nn = 8\ndt = 0.01\nn_iterations = 3\ndiagnostics_interval = 1\n",
    "tgv_dp": "n = 32\nM = 0.1\nRe = 1600\ndt = 0.002\nn_iterations = 40\ndiagnostics_interval = 10\n"
              "strategy = storesome\n",
    "tgv_hpsp_default": "n = 32\nprecision = HPSP\ndt = 0.002\nn_iterations = 30\n"
                        "diagnostics_interval = 10\nthreads = 4\n",
    "tgv_spdp_storeround": "n = 24\nprecision = SPDP\nemulation = storeround\ndt = 0.003\n"
                           "n_iterations = 20\ndiagnostics_interval = 5\nsplit = KGP\n",
    "diverge": "n = 16\nM = 0.4\nviscous = false\nsplit = Divergence\ndt = 0.2\nn_iterations = 400\n"
               "diagnostics_interval = 10\nstrategy = storesome\n",
}


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
@pytest.mark.parametrize("name", list(CFGS))
def test_csv_byte_identical(b200, tmp_path, name):
    tool = build_tool(b200)
    outs = {}
    codes = {}
    for who, exe in (("ref", REF_CLI), ("b200", tool)):
        cfg = tmp_path / f"{who}.cfg"
        out = tmp_path / f"{who}.csv"
        cfg.write_text(CFGS[name] + f"output = {out}\n")
        r = subprocess.run([exe, "run", str(cfg)], capture_output=True, text=True, cwd=tmp_path)
        codes[who] = r.returncode
        outs[who] = out.read_bytes()
    assert codes["ref"] == codes["b200"]
    assert outs["ref"] == outs["b200"]


def _csv(rows):
    s = "t,kinetic_energy,enstrophy,solenoidal_dissipation,ke_normalized,diverged\n"
    for r in rows:
        s += ",".join("%.17g" % x for x in r) + ",0\n"
    return s


@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
def test_compare_matches_reference_cli(b200, tmp_path):
    """`compare a.csv b.csv` (tools/mpfd.cpp:28-38, compare_series tgv.cpp:177-197):
    same per-sample |delta eps_S|, pairwise mean and max, same text; sample-grid
    mismatches are errors (exit 1) in both."""
    tool = build_tool(b200)
    import numpy as np
    rng = np.random.default_rng(3)
    t = np.arange(70) * 0.5
    a = np.c_[t, rng.random((70, 4))]
    b = np.c_[t, rng.random((70, 4))]
    (tmp_path / "a.csv").write_text(_csv(a))
    (tmp_path / "b.csv").write_text(_csv(b))
    (tmp_path / "c.csv").write_text(_csv(b[:-1]))
    (tmp_path / "d.csv").write_text(_csv(np.c_[t + 0.25, b[:, 1:]]))
    args = [str(tmp_path / "a.csv"), str(tmp_path / "b.csv")]
    r1 = subprocess.run([REF_CLI, "compare", *args], capture_output=True, text=True)
    r2 = subprocess.run([tool, "compare", *args], capture_output=True, text=True)
    assert r1.returncode == r2.returncode == 0
    assert r1.stdout == r2.stdout
    for bad in ("c.csv", "d.csv"):
        args = [str(tmp_path / "a.csv"), str(tmp_path / bad)]
        assert subprocess.run([REF_CLI, "compare", *args], capture_output=True).returncode == 1
        assert subprocess.run([tool, "compare", *args], capture_output=True).returncode == 1


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
def test_sweep_matrix_identical(b200, tmp_path):
    """`sweep <spec>` (run_sweep, runner.cpp:108-173): DP reference plus each
    preset over dt x M; the mean |delta eps_S| matrix (the paper's accuracy
    heat-map methodology) and the log are the reference CLI's, byte for byte."""
    tool = build_tool(b200)
    spec = ("n = 16\nRe = 1600\nt_end = 1.0\nstrategy = storesome\nthreads = 4\n"
            "sweep.dt = 0.01, 0.02\nsweep.M = 0.1, 0.3\nsweep.presets = SPDP, HPSP, SP\n")
    outs = {}
    for who, exe in (("ref", REF_CLI), ("b200", tool)):
        f = tmp_path / f"{who}.spec"
        f.write_text(spec + f"sweep.output = {tmp_path / (who + '.csv')}\n")
        r = subprocess.run([exe, "sweep", str(f)], capture_output=True, text=True, cwd=tmp_path)
        assert r.returncode == 0, r.stderr
        outs[who] = (r.stdout.replace(who + ".csv", "X.csv"), (tmp_path / f"{who}.csv").read_bytes())
    assert outs["ref"] == outs["b200"]
    assert outs["ref"][1].count(b"\n") == 5


REPORTS = {
    "dp_default": "n = 64\n",
    "hpsp_default_pencils": "n = 64\nprecision = HPSP\nprocs = 1,2,4\n",
    "spdp_storesome_slabs": "n = 128\nprecision = SPDP\nstrategy = storesome\nprocs = 1,1,8\n",
    "spdp_res_override": "n = 32\nprecision = SPDP-res\nprecision.custom.u = B16\nprecision.custom.dTdz = B32\n"
                         "procs = 2,2,2\ncomm.rk_arrays = 1\ncomm.wk_arrays = 2\n",
    "hp_pencils": "n = 96\nprecision = HP\nprocs = 2,2,2\n",
    "bad_procs": "n = 30\nprocs = 1,1,4\n",
}


@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
@pytest.mark.parametrize("name", list(REPORTS))
def test_report_identical(b200, tmp_path, name):
    """`report <config>` (print_report, runner.cpp:90-106): the analytic memory
    census of the field set and the modelled halo volume per process, byte for
    byte the reference CLI's (and the same exit code on a bad process grid)."""
    tool = build_tool(b200)
    cfg = tmp_path / "r.cfg"
    cfg.write_text(REPORTS[name])
    r1 = subprocess.run([REF_CLI, "report", str(cfg)], capture_output=True, text=True)
    r2 = subprocess.run([tool, "report", str(cfg)], capture_output=True, text=True)
    assert r1.returncode == r2.returncode
    assert r1.stdout == r2.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="reference CLI not built")
def test_snapshots_identical(b200, tmp_path):
    """snapshot_times / snapshot_path (advance integrate.cpp:154-158, runner.cpp:
    34-41, write_snapshot io.cpp:69-85): the same files, byte for byte."""
    tool = build_tool(b200)
    base = ("n = 24\nprecision = HPSP\nM = 0.1\nRe = 1600\ndt = 0.002\nn_iterations = 30\n"
            "diagnostics_interval = 10\nstrategy = storesome\nsnapshot_times = 0.01, 0.035, 0.06\n")
    files = {}
    for who, exe in (("ref", REF_CLI), ("b200", tool)):
        d = tmp_path / who
        d.mkdir()
        (d / "c.cfg").write_text(base + f"snapshot_path = {d / 'snap.bin'}\noutput = {d / 'o.csv'}\n")
        r = subprocess.run([exe, "run", str(d / "c.cfg")], capture_output=True, text=True, cwd=d)
        assert r.returncode == 0, r.stderr
        files[who] = {p.name: p.read_bytes() for p in d.iterdir() if p.name.startswith("snap")}
    assert sorted(files["ref"]) == sorted(files["b200"]) and len(files["ref"]) == 3
    for k in files["ref"]:
        assert files["ref"][k] == files["b200"][k], k
