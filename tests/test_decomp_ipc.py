"""GPU, two or three processes on one B200: the solver's own multi-rank code path.

Each process creates a Solver with one z-slab of a pz = 2 decomposition in
MPFD_DECOMP_IPC mode: the neighbours' Q buffers are mapped with CUDA IPC,
ghost planes are pulled by copy-engine transfers ordered by epoch flags in
device memory (cuStreamWaitValue32 / cuStreamWriteValue32), and the host
collective behind the divergence keys, the divergence records and the
diagnostics partials is torch.distributed on gloo (Decomposition.allgather).
Everything the solver does in that mode runs here for real -- plan, pulls,
overlap of the exchange with the interior planes, divergence reduction,
diagnostics gather and merge -- with the NCCL calls swapped for the
copy-engine transport (NCCL refuses two ranks on one device).

Checks, against the unmodified reference (oracle/_ref) on the whole domain:
Q and Qt of every slab bit for bit, the KE/enstrophy series bit for bit, and
the divergence event (what, where, when).
"""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    # name: (n, preset, path, overlap, steps, diag interval, dt, flow kw[, ranks])
    "hpsp_fused_overlap": (32, "HPSP", "fused", True, 6, 3, 0.002, {}),
    # three ranks: distinct lower and upper neighbours (two ranks share one)
    "spdp_three_ranks": (48, "SPDP", "fused", True, 3, 3, 0.002, {"ranks": 3}),
    # y pencils (staged path): a 2 x 2 grid of ranks, and 3 pencils in y
    "dp_pencils_2x2": (32, "DP", "staged", False, 3, 3, 0.002, {"ranks": 4, "py": 2}),
    "hpsp_pencils_1x3": (24, "HPSP", "staged", False, 3, 3, 0.002, {"ranks": 3, "py": 3}),
    "dp_fused_no_overlap": (32, "DP", "fused", False, 4, 2, 0.002, {}),
    "spdp_staged": (24, "SPDP", "staged", True, 3, 3, 0.002, {}),
    "diverge": (16, "DP", "fused", True, 400, 10, 0.2, dict(split="Divergence", viscous=False, mach=0.4)),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_20911_b200 as m

    n, preset, path, overlap, steps, di, dt, kw = CASES[name]
    py = kw.get("py", 1)
    kw = {k: v for k, v in kw.items() if k not in ("ranks", "py")}
    flow = m.FlowParams(kw.get("mach", 0.1), 1600.0, 0.72, 1.4, kw.get("viscous", True))
    dec = m.Decomposition(pz=world // py, py=py, mode=m.IPC, rank=rank, device=0,
                          allgather=m.gloo_allgather())
    s = m.Solver(m.GridSpec(n), m.resolve_preset(preset), "storesome", flow, kw.get("split", "Blaisdell"), dec)
    s.set_path(path)
    s.set_overlap(overlap)
    s.init_tgv()
    r = s.advance(m.StepConfig(dt, steps, di))
    pz = world // py
    nzl, nyl = n // pz, n // py
    z0, y0 = (rank // py) * nzl, (rank % py) * nyl
    res = {
        "z0": z0, "y0": y0,
        "q": np.stack([s.get_field(0, c)[z0:z0 + nzl, y0:y0 + nyl] for c in range(5)]),
        "qt": np.stack([s.get_field(1, c)[z0:z0 + nzl, y0:y0 + nyl] for c in range(5)]),
        "series": [(x.t, x.kinetic_energy, x.enstrophy, x.diverged) for x in r.series],
        "diverged": r.diverged,
        "event": None if r.divergence is None else tuple(vars(r.divergence).values()),
        "iters": r.iterations_run,
        "halo": s.halo_bytes(),
    }
    s.close()
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_ipc_ranks_vs_reference(b200, tmp_path, name):
    import pyoracle as po

    world = CASES[name][7].get("ranks", 2)
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    parts = [pickle.load(open(tmp_path / f"r{r}.pkl", "rb")) for r in range(world)]
    n, preset, path, overlap, steps, di, dt, kw = CASES[name]
    py = kw.get("py", 1)
    kw = {k: v for k, v in kw.items() if k not in ("ranks", "py")}
    ckw = dict(preset=preset, split=kw.get("split", "Blaisdell"), viscous=kw.get("viscous", True),
               mach=kw.get("mach", 0.1))
    c = po.Reference(n, **ckw) if po.ref_available() else po.Oracle(n, **ckw)
    c.init()
    st, series, ev, iters = c.advance(dt, steps, di, threads=8)
    # every rank holds the same collective results
    for p in parts[1:]:
        assert parts[0]["series"] == p["series"]
        assert parts[0]["event"] == p["event"] and parts[0]["iters"] == p["iters"]
    assert parts[0]["iters"] == iters
    got = np.array([[t, k, e, d] for t, k, e, d in parts[0]["series"]], dtype=np.float64)
    want = series[:, [0, 1, 2, 4]]
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.nan_to_num(got).view(np.uint64), np.nan_to_num(want).view(np.uint64))
    if kw:
        codes = {"nonpositive or nonfinite density": 1, "nonfinite residual": 2, "nonfinite state": 3}
        assert parts[0]["diverged"] and st == 2
        what, i, j, k, _time, it, sub = parts[0]["event"]
        assert [codes[what], i, j, k, it, sub] == ev
        return
    assert not parts[0]["diverged"] and st == 0
    pz = world // py
    nzl, nyl = n // pz, n // py
    for p in parts:
        z0, y0 = p["z0"], p["y0"]
        for cls, key in ((0, "q"), (1, "qt")):
            ref = np.stack([c.field(cls, comp)[z0:z0 + nzl, y0:y0 + nyl] for comp in range(5)])
            assert np.array_equal(p[key].view(np.uint64), ref.view(np.uint64)), (name, key, z0, y0)
        # every state: two pulls of 4 planes x 5 components in q storage (the
        # planes carry the 4 y ghost rows per side with pencils), plus two
        # packed y faces of 4 rows
        bq = 4 if preset == "HPSP" else 8  # q storage
        rows = nyl + (8 if py > 1 else 0)
        per_state = 2 * 4 * 5 * rows * n * bq + (2 * nzl * 5 * 4 * n * bq if py > 1 else 0)
        assert p["halo"] % per_state == 0 and p["halo"] >= per_state * steps * 3
