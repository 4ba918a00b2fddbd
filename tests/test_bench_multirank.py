"""bench.py's multi-rank path end to end on one GPU: two torchrun ranks
pinned to cuda:0 (MPFD_BENCH_DEVICE) on the IPC transport -- the barrier,
the max-over-ranks timing, the per-rank e2e through the C-ABI and the
measured halo bytes.  Ranks sharing one GPU give no scaling number; this
checks that the path the driver's N-GPU runs take works."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_bench_two_ranks_ipc(b200):
    n = 64
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--grid", str(n), "--precision", "HPSP", "--transport", "ipc",
           "--modes", "", "--no-cpu-baseline", "--no-memory-table", "--no-issue-ceiling", "--slab-sweep", ""]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "MPFD_BENCH_DEVICE": "0"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 prints one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert "IPC" in d["config"]["decomposition"]
    # weak scaling: n^3 per rank, two TGV periods stacked in z
    assert abs(d["value"] * d["ms_per_step"] * 1e-3 - 2 * n ** 3) < 1e-6 * 2 * n ** 3
    # every state: two pulls of 4 planes x 5 components in fp32 (HPSP q storage)
    per_state = 2 * 4 * 5 * n * n * 4
    assert d["halo"]["measured_bytes_per_step"] >= 3 * per_state
    assert d["e2e"]["value"] > 0 and not d["e2e"]["diverged"]
