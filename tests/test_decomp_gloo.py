"""CPU, world_size 2 (gloo): the host-side logic of the multi-rank path,
driven through the library's own C-ABI host functions -- the ones the solver
runs around its collectives -- with torch.distributed (gloo) as the
transport:

  * mpfd_b200_halo_plan: the byte offsets the NCCL and IPC transports use.
    Each rank lays its slab out exactly like the device Q buffer
    ([nzl+8 planes][5][n][n]) and moves the planned blocks; the ghosts must
    equal the periodic wrap of the global field (fill_halos_periodic's z
    pass, field.cpp:29-36).
  * the IPC transport's host collective (Decomposition.allgather =
    gloo_allgather, called through the same ctypes callback the solver
    receives) gathers each rank's 4096-chunk diagnostics partials;
    mpfd_b200_merge_diagnostics must then equal the reference's
    deterministic_sum over the whole field for both tree shapes
    (reduce.cpp:14-36), i.e. diagnostics are decomposition independent.
  * per-rank divergence record tables, gathered the same way, merged by
    mpfd_b200_merge_divergence, give the single-domain event: earliest
    substep, the reference's check order, the first point in scan order
    (physics.cpp:573-584, integrate.cpp:135-147, reduce.cpp:57-81) -- also
    when the other rank ran ahead and recorded a later substep.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIFT = 39  # kDivKeyShift: (key << 39) | global index


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _first_in_scan(mask_slab, z0, n):
    idx = np.flatnonzero(mask_slab.reshape(-1))
    return None if idx.size == 0 else int(idx[0]) + z0 * n * n


def _table(bad, key_of_code, z0, nzl, n):
    """Record table of one slab: bad[code][comp] is the global boolean mask."""
    t = np.full(15, np.iinfo(np.uint64).max, dtype=np.uint64)
    for code in range(3):
        for comp in range(5):
            gi = _first_in_scan(bad[code][comp][z0:z0 + nzl], z0, n)
            if gi is not None:
                t[code * 5 + comp] = np.uint64((key_of_code[code] << SHIFT) | gi)
    return t


def _worker(rank, world, port, n, result_dir):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_20911_b200 as m
    import pyoracle as po

    # ---- halo plan ---------------------------------------------------------
    bq = 8
    p = m.halo_plan(n, world, rank, bq)
    send_up, recv_lo, send_dn, recv_hi, blk = (p[k] for k in ("send_up", "recv_lo", "send_dn", "recv_hi", "block"))
    up, dn, z0, nzl = p["up"], p["dn"], p["z0"], p["nzl"]
    rng = np.random.default_rng(7)
    glob = rng.standard_normal((n, 5, n, n))  # [z][comp][y][x]
    q = np.zeros((nzl + 8, 5, n, n))
    q[4:4 + nzl] = glob[z0:z0 + nzl]
    buf = torch.from_numpy(q.reshape(-1).view(np.uint8))
    reqs = [dist.isend(buf[send_up:send_up + blk].clone(), up), dist.isend(buf[send_dn:send_dn + blk].clone(), dn)]
    lo = torch.empty(blk, dtype=torch.uint8)
    hi = torch.empty(blk, dtype=torch.uint8)
    dist.recv(lo, dn)
    dist.recv(hi, up)
    for r in reqs:
        r.wait()
    buf[recv_lo:recv_lo + blk] = lo
    buf[recv_hi:recv_hi + blk] = hi
    q = buf.numpy().view(np.float64).reshape(nzl + 8, 5, n, n)
    for g in range(4):
        assert np.array_equal(q[g], glob[(z0 - 4 + g) % n])
        assert np.array_equal(q[nzl + 4 + g], glob[(z0 + nzl + g) % n])

    ag = m.gloo_allgather()  # the IPC transport's host collective

    # ---- diagnostics partials -> merge -------------------------------------
    Lo = po.oracle_lib()
    for comp in (0, 3):
        integ = np.ascontiguousarray(glob[z0:z0 + nzl, comp]).reshape(-1)
        nch = integ.size // 4096
        parts = np.array([Lo.orc_pairwise_sum(integ[i * 4096:].ctypes.data_as(C.POINTER(C.c_double)), 4096)
                          for i in range(nch)])
        allp = np.frombuffer(ag(parts.tobytes()), dtype=np.float64)
        full = np.ascontiguousarray(glob[:, comp]).reshape(-1)
        for threads in (1, 8):
            got = m.merge_diagnostics(allp, full.size, threads, chunked=True)
            want = Lo.orc_deterministic_sum(full.ctypes.data_as(C.POINTER(C.c_double)), full.size, threads)
            assert got == want, (comp, threads)
        # unaligned / raw-integrand path: every rank's points, concatenated
        raw = np.frombuffer(ag(integ.tobytes()), dtype=np.float64)
        assert m.merge_diagnostics(raw, full.size, 8, chunked=False) == \
            Lo.orc_deterministic_sum(full.ctypes.data_as(C.POINTER(C.c_double)), full.size, 8)

    # ---- divergence records -> merge ---------------------------------------
    dt = 0.002
    it = 17
    bad = [[np.zeros((n, n, n), bool) for _ in range(5)] for _ in range(3)]
    # substep 1 of iteration 17: a nonfinite residual on both slabs (rank 1's
    # earlier in scan order is not what counts: rank 0's slab comes first),
    # and a density event on the upper slab only
    bad[1][2][n // 2 + 3, 5, 9] = True
    bad[1][2][n // 2 - 2, 7, 1] = True
    bad[1][4][1, 0, 0] = True
    bad[0][0][n - 1, 3, 3] = True
    key = 3 * it + 1
    # rank 1 also ran ahead one substep and saw a nonfinite state there
    keys = {0: [key, key, key], 1: [key, key, key + 1]}
    bad_state = [np.zeros((n, n, n), bool) for _ in range(5)]
    bad_state[0][n - 2, 0, 0] = True
    tabs = _table(bad, keys[rank], z0, nzl, n)
    if rank == 1:
        t2 = _table([bad[0], bad[1], bad_state], keys[1], z0, nzl, n)
        tabs = np.minimum(tabs, t2)
    allt = np.frombuffer(ag(tabs.tobytes()), dtype=np.uint64).reshape(world, 15)
    ev = m.merge_divergence(allt, n, dt)
    # single domain: density is checked first (primitives), at the earliest key
    assert ev is not None and ev.iteration == it and ev.substep == 1
    assert ev.what.startswith("nonpositive") and (ev.i, ev.j, ev.k) == (3, 3, n - 1)
    assert abs(ev.time - it * dt) == 0.0
    # without the density event: the residual check, component 2, slab 0 first
    bad[0][0][:] = False
    tabs = _table(bad, keys[rank], z0, nzl, n)
    allt = np.frombuffer(ag(tabs.tobytes()), dtype=np.uint64).reshape(world, 15)
    ev = m.merge_divergence(allt, n, dt)
    assert ev.what == "nonfinite residual" and (ev.i, ev.j, ev.k) == (1, 7, n // 2 - 2)
    assert ev.time == it * dt
    assert m.merge_divergence(np.full((world, 15), np.iinfo(np.uint64).max, np.uint64), n, dt) is None

    with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_plan_gather_and_merges(tmp_path, world):
    import paper_2505_20911_b200 as m

    m.lib()  # fail here, not in the workers, if the library is missing
    mp.spawn(_worker, args=(world, _free_port(), 64, str(tmp_path)), nprocs=world, join=True)
    assert all(os.path.exists(tmp_path / f"ok{r}") for r in range(world))
