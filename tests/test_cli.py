"""The drop-in boundary, compiled: the reference's OWN CLI (proj/tools/mpfd.cpp)
and runner (proj/src/runner.cpp) built with integration/runner_b200.patch,
so run_simulation (runner.cpp:11-48) drives the B200 path through
include/mpfd_b200.hpp.  `mpfd run / sweep` of the patched CLI and of the stock
CLI (oracle/_ref/mpfd) write byte-identical CSVs, snapshots, sweep matrices
and run summaries (wall time aside), with the same exit codes
(tools/mpfd.cpp:4-5).  Built by integration/Makefile (build()); the GPU box
runs the prebuilt binary."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATCHED = os.path.join(ROOT, "integration", "_build", "mpfd_b200cli")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "mpfd")

needs_clis = pytest.mark.skipif(not (os.path.exists(REF_CLI) and os.path.exists(PATCHED)),
                                reason="reference CLI / patched CLI not built (integration/Makefile)")


@needs_clis
def test_patched_cli_links_the_b200_library():
    """The patched CLI resolves run_simulation's hot path to libmpfd_b200.so."""
    out = subprocess.run(["ldd", PATCHED], capture_output=True, text=True).stdout
    lib = [l for l in out.splitlines() if "libmpfd_b200.so" in l]
    assert lib and "not found" not in lib[0], out
    assert os.path.realpath(lib[0].split("=>")[1].split("(")[0].strip()) == os.path.realpath(
        os.path.join(ROOT, "paper_2505_20911_b200", "libmpfd_b200.so"))


@needs_clis
def test_bad_config_exit_codes(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("nonsense_key = 42\n")  # tests/data/bad.cfg of the reference
    for exe in (REF_CLI, PATCHED):
        r = subprocess.run([exe, "run", str(bad)], capture_output=True, text=True)
        assert r.returncode == 1 and "unknown key" in r.stderr


CFGS = {
    "smoke_uniform": "case = uniform\nn = 8\ndt = 0.01\nn_iterations = 3\ndiagnostics_interval = 1\n",
    "tgv_dp": "n = 32\nM = 0.1\nRe = 1600\ndt = 0.002\nn_iterations = 40\ndiagnostics_interval = 10\n"
              "strategy = storesome\n",
    "tgv_hpsp_default": "n = 32\nprecision = HPSP\ndt = 0.002\nn_iterations = 30\n"
                        "diagnostics_interval = 10\nthreads = 4\n",
    "tgv_spdp_storeround": "n = 24\nprecision = SPDP\nemulation = storeround\ndt = 0.003\n"
                           "n_iterations = 20\ndiagnostics_interval = 5\nsplit = KGP\n",
    "tgv_override": "n = 16\nprecision = SPDP-res\nprecision.custom.u = B16\ndt = 0.003\n"
                    "n_iterations = 10\ndiagnostics_interval = 5\n",
    "diverge": "n = 16\nM = 0.4\nviscous = false\nsplit = Divergence\ndt = 0.2\nn_iterations = 400\n"
               "diagnostics_interval = 10\nstrategy = storesome\n",
}

WALL = re.compile(r"^iterations: (\d+), wall time (\S+) s \((\S+) s/iteration\)$")


def _summary(stdout, who):
    """run_to_files' log (runner.cpp:69-88) with the wall-time figures split off."""
    lines, wall = [], None
    for line in stdout.replace(who + ".csv", "X.csv").splitlines():
        m = WALL.match(line)
        if m:
            wall = (int(m.group(1)), float(m.group(2)), float(m.group(3)))
            line = f"iterations: {m.group(1)}, wall time W"
        lines.append(line)
    return lines, wall


@pytest.mark.gpu
@needs_clis
@pytest.mark.parametrize("name", list(CFGS))
def test_run_byte_identical(b200, tmp_path, name):
    """`mpfd run <cfg>`: same CSV bytes (io.cpp:19-36), same exit code, same
    summary -- sample count, iterations, the memory census (memory_report,
    registry.cpp:24-39, which the patched runner takes from
    mpfd_b200_memory_census) and the divergence line; the wall time is the
    B200 path's own and positive."""
    outs, codes, logs = {}, {}, {}
    for who, exe in (("ref", REF_CLI), ("b200", PATCHED)):
        cfg = tmp_path / f"{who}.cfg"
        out = tmp_path / f"{who}.csv"
        cfg.write_text(CFGS[name] + f"output = {out}\n")
        r = subprocess.run([exe, "run", str(cfg)], capture_output=True, text=True, cwd=tmp_path)
        codes[who] = r.returncode
        outs[who] = out.read_bytes()
        logs[who] = _summary(r.stdout, who)
    assert codes["ref"] == codes["b200"]
    assert outs["ref"] == outs["b200"]
    assert logs["ref"][0] == logs["b200"][0]
    it, wall, spi = logs["b200"][1]
    assert wall > 0.0 and (it == 0 or spi > 0.0)
    assert any("memory census" in l for l in logs["b200"][0])


@pytest.mark.gpu
@needs_clis
def test_sweep_matrix_identical(b200, tmp_path):
    """`sweep <spec>` (run_sweep, runner.cpp:108-173) calls the patched
    run_simulation for the DP reference and each preset over dt x M; the mean
    |delta eps_S| matrix (the paper's accuracy heat-map methodology) and the
    log are the stock CLI's, byte for byte."""
    spec = ("n = 16\nRe = 1600\nt_end = 1.0\nstrategy = storesome\nthreads = 4\n"
            "sweep.dt = 0.01, 0.02\nsweep.M = 0.1, 0.3\nsweep.presets = SPDP, HPSP, SP\n")
    outs = {}
    for who, exe in (("ref", REF_CLI), ("b200", PATCHED)):
        f = tmp_path / f"{who}.spec"
        f.write_text(spec + f"sweep.output = {tmp_path / (who + '.csv')}\n")
        r = subprocess.run([exe, "sweep", str(f)], capture_output=True, text=True, cwd=tmp_path)
        assert r.returncode == 0, r.stderr
        outs[who] = (r.stdout.replace(who + ".csv", "X.csv"), (tmp_path / f"{who}.csv").read_bytes())
    assert outs["ref"] == outs["b200"]
    assert outs["ref"][1].count(b"\n") == 5


@pytest.mark.gpu
@needs_clis
def test_snapshots_identical(b200, tmp_path):
    """snapshot_times / snapshot_path (advance integrate.cpp:154-158, runner.cpp:
    34-41, write_snapshot io.cpp:69-85): the same files, byte for byte."""
    base = ("n = 24\nprecision = HPSP\nM = 0.1\nRe = 1600\ndt = 0.002\nn_iterations = 30\n"
            "diagnostics_interval = 10\nstrategy = storesome\nsnapshot_times = 0.01, 0.035, 0.06\n")
    files = {}
    for who, exe in (("ref", REF_CLI), ("b200", PATCHED)):
        d = tmp_path / who
        d.mkdir()
        (d / "c.cfg").write_text(base + f"snapshot_path = {d / 'snap.bin'}\noutput = {d / 'o.csv'}\n")
        r = subprocess.run([exe, "run", str(d / "c.cfg")], capture_output=True, text=True, cwd=d)
        assert r.returncode == 0, r.stderr
        files[who] = {p.name: p.read_bytes() for p in d.iterdir() if p.name.startswith("snap")}
    assert sorted(files["ref"]) == sorted(files["b200"]) and len(files["ref"]) == 3
    for k in files["ref"]:
        assert files["ref"][k] == files["b200"][k], k
