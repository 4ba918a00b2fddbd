#!/usr/bin/env python3
"""bench.py -- TGV explicit-FD RK time step on B200 (one JSON line on rank 0).

Metric (BASELINE.json): grid-point updates per second per RK step, TGV,
per precision mode; one step = one full low-storage RK3 step (3 substeps of
residual + stage update + halo refresh).  Inputs are the deterministic TGV
initial condition (synthetic, no RNG); the state (>= 5.4 GB at 512^3 DP) is
far larger than the 126 MB L2, so no explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 512] [--precision DP]
  python bench.py --impl reference ...     # the reference CPU implementation

Multi-GPU: launched by torch.distributed.run, one rank per GPU; z-slab
decomposition with NCCL halo exchange overlapped with the interior planes.
Default --scaling weak: every rank owns one n^3 period (the grid stacks N
TGV periods along z, GridSpec.z_periods = N), so per-GPU work is fixed;
--scaling strong splits one n^3 cube over the N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# keep stdout to the one JSON line: NCCL prints its version banner at
# NCCL_DEBUG >= VERSION (WARN included), so the level stays unset (errors only)
if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "WARN"):
    del os.environ["NCCL_DEBUG"]

METRIC = ("grid-pt updates/s per RK step (TGV 512^3, per precision mode) at 1/2/4/8 B200; "
          "% HBM roofline")
UNIT = "grid-pt updates/s"
BYTES = {"B16": 2, "B32": 4, "B64": 8}
PRESET_KINDS = {  # (q, rk, res, wk) byte widths, precision.cpp:58-88
    "DP": (8, 8, 8, 8), "SP": (4, 4, 4, 4), "HP": (2, 2, 2, 2), "SPDP": (8, 8, 4, 4),
    "SPDP-wk": (8, 8, 8, 4), "SPDP-res": (8, 8, 4, 8), "HPSP": (4, 4, 2, 2),
    "HPSP-wk": (4, 4, 4, 2), "HPSP-res": (4, 4, 2, 4),
}
DT = {64: 0.002, 128: 0.001, 256: 5e-4, 512: 2.5e-4, 1024: 1.25e-4}


def b_alg(preset: str) -> int:
    """B_alg = 45 bq + 30 br + 25 bt bytes / point / RK step."""
    bq, bt, br, _ = PRESET_KINDS[preset]
    return 45 * bq + 30 * br + 25 * bt


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def cpu_reference_run(preset, strategy, emulation, n, steps, warmup, threads=None):
    """Time the reference CPU implementation (oracle/_ref: the unmodified
    reference sources, else the C port) through its advance() on this host's
    cores, on the n^3 TGV grid itself; returns (pt/s, cores, kind, sample)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    threads = threads or os.cpu_count() or 1
    kind = "reference" if po.ref_available() else "port"
    kw = dict(preset=preset, strategy=strategy, emulation=emulation)
    if kind == "reference":
        c = po.Reference(n, threads=threads, **kw)
    else:
        po.oracle_lib().orc_set_threads(threads)
        c = po.Oracle(n, **kw)
    c.init()
    dt = DT.get(n, 0.002)
    if warmup:
        c.advance(dt, warmup, 0, threads=threads)
    t0 = time.perf_counter()
    c.advance(dt, steps, 0, threads=threads)
    el = time.perf_counter() - t0
    del c
    rate = n ** 3 * steps / el
    sample = (f"TGV {n}^3 {preset} {strategy} {emulation}, {steps} timed RK step(s) after {warmup} "
              f"warm-up, {'reference advance() (oracle/_ref)' if kind == 'reference' else 'C port (oracle/)'}, "
              f"threads={threads}, {el / steps:.2f} s/step")
    return rate, threads, kind, sample


# CPU steps are ~1e4x slower than the GPU's: the reference runs the bench's
# own grid for a bounded number of steps (1 warm-up + 2 timed)
CPU_STEPS, CPU_WARMUP = 2, 1
# per-precision CPU lines run at 256^3, one timed step (HPSP Strict emulates
# binary16 in software: ~8x a DP step on the CPU)
CPU_PP_GRID = 256


def cpu_per_precision(modes, args):
    out = {}
    for p in modes:
        try:
            rate, cores, kind, sample = cpu_reference_run(p, args.strategy, args.emulation,
                                                          min(args.grid, CPU_PP_GRID), 1, 0)
            out[p] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        except Exception as e:  # report, never hide
            out[p] = {"value": None, "error": str(e)}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps, warmup = min(args.steps, CPU_STEPS), min(args.warmup, CPU_WARMUP)
    rate, cores, kind, sample = cpu_reference_run(args.precision, args.strategy, args.emulation,
                                                  args.grid, steps, warmup)
    bound = (f"{steps} timed + {warmup} warm-up step(s) of the {args.grid}^3 grid instead of "
             f"{args.steps} + {args.warmup}: a CPU step of this grid takes tens of seconds")
    modes = [x for x in args.modes.split(",") if x and x != args.precision]
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_ms(rate, args.grid), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": dtype_of(args.precision), "data": "synthetic",
        "config": {"workload": f"TGV {args.grid}^3 {args.precision} (M=0.1, Re=1600, {args.split}, "
                               f"{args.strategy}, {args.emulation})",
                   "n": args.grid, "precision": args.precision, "sample": sample, "bounded": bound},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_precision": cpu_per_precision(modes, args),
    }
    print(json.dumps(line), flush=True)
    return 0


def n_ms(rate, n):
    return n ** 3 / rate * 1e3 if rate else None


def dtype_of(preset):
    q, t, r, w = PRESET_KINDS[preset]
    names = {8: "f64", 4: "f32", 2: "f16"}
    return names[r] if q == r else f"{names[q]}/{names[r]}"


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--grid", type=int, default=512, help="n of the n^3 TGV grid")
    ap.add_argument("--precision", default="DP")
    ap.add_argument("--strategy", default="storesome")
    ap.add_argument("--emulation", default="strict")
    ap.add_argument("--split", default="Blaisdell")
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "staged"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--modes", default="SPDP,HPSP",
                    help="extra precision modes measured after the headline (per_precision)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl", action="store_true",
                    help="use the NCCL transport even on one rank (self-exchange)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="halo transport between ranks: ncclSend/Recv, or copy-engine pulls from "
                         "CUDA-IPC-mapped neighbour buffers (host collectives over gloo)")
    ap.add_argument("--slab-sweep", default="2,4,8",
                    help="LOCAL z-slab counts timed on one GPU (decomposition overhead); '' to skip")
    ap.add_argument("--slab-preset", default="HPSP")
    ap.add_argument("--no-issue-ceiling", action="store_true",
                    help="skip the issue-ceiling microbenchmark (compute roofline denominators)")
    ap.add_argument("--no-memory-table", action="store_true",
                    help="skip the measured per-preset memory table (Default strategy, materialised)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-overlap", action="store_true",
                    help="exchange ghost planes before the substep instead of overlapping")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2505_20911_b200 as m

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # MPFD_BENCH_DEVICE pins every rank to one device: a functional check of
    # the multi-rank path on a one-GPU box (IPC transport only; the timing of
    # ranks sharing a GPU is not a scaling number)
    local = int(os.environ.get("MPFD_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    use_nccl = world > 1 or args.nccl  # multi-rank (the transport is args.transport)
    ipc = use_nccl and args.transport == "ipc"
    if use_nccl:
        if "RANK" not in os.environ:  # --nccl without a launcher: a 1-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        if ipc:  # host collectives only: the halo moves by copy engines
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gloo = None  # the IPC transport's host all-gather runs on the default (gloo) group
    red_dev = "cpu" if ipc else "cuda"
    hbm, peak_src = peaks()
    try:
        ceil = {"skipped": True} if args.no_issue_ceiling else m.issue_ceiling(local)
    except Exception as e:  # report, never hide
        ceil = {"error": str(e)}

    def measure(preset, with_extras, local_pz=1, overlap=None, zper_override=None):
        n = args.grid
        dt = DT.get(n, 2.5e-4)
        prec = m.resolve_preset(preset, args.emulation)
        decomp = None
        if local_pz > 1:  # LOCAL z-slabs on this device (the decomposition's own cost)
            decomp = m.Decomposition(pz=local_pz, device=local)
        elif use_nccl and args.transport == "ipc":
            decomp = m.Decomposition(pz=world, mode=m.IPC, rank=rank, device=local,
                                     allgather=m.gloo_allgather(gloo))
        elif use_nccl:
            obj = [m.Solver.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            decomp = m.Decomposition(pz=world, mode=1, rank=rank, device=local, nccl_id=obj[0])
        else:
            decomp = m.Decomposition(device=local)
        zper = world if args.scaling == "weak" else 1
        if zper_override:
            zper = zper_override
        s = m.Solver(m.GridSpec(n, z_periods=zper), prec, args.strategy,
                     m.FlowParams(0.1, 1600.0, 0.72, 1.4, True), args.split, decomp)
        if args.path != "auto":
            s.set_path(args.path)
        if args.no_overlap or overlap is False:
            s.set_overlap(False)
        elif overlap is True:
            s.set_overlap(True)
        s.init_tgv()
        s.run_steps(args.warmup, dt)
        s.synchronize()
        stream = torch.cuda.ExternalStream(s.stream)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.profile(True)
        if use_nccl:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            ev0.record(stream)
            s.run_steps(args.steps, dt)
            ev1.record(stream)
            s.synchronize()
            torch.cuda.synchronize()
        ms_total = ev0.elapsed_time(ev1)
        if use_nccl:
            t = torch.tensor([ms_total], device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_total = float(t.item())
        kms, klaunch = s.profile_read()
        halo_sent = s.halo_bytes()
        s.profile(False)
        ms_step = ms_total / args.steps
        npts = n ** 3 * zper  # whole job
        rate = npts / (ms_step * 1e-3)
        # roofline of the dominant kernel (class 0: residual / fused step)
        bq, bt, br, bw = PRESET_KINDS[preset]
        nloc = npts // world
        fused = klaunch[1] == 0
        if fused:
            # the kernel's own compulsory bytes per substep: read Q, write Q;
            # Qt read (substeps 1,2) + write
            comp_pt = (10 * bq + 5 * bt) / 3 + 2 * (10 * bq + 10 * bt) / 3
            kname = "fused residual + RK stage update"
        else:
            comp_pt = 5 * bq + 5 * br
            kname = "staged residual (k_resid)"
        # dominant-kernel time per substep (an overlapped substep is one
        # interior + two boundary launches covering the slab once)
        avg_ms = kms[0] / (3 * args.steps) if fused else kms[0] / max(1, klaunch[0])
        # achieved = SURVEY 8(d)'s algorithmic bytes (B_alg per point per RK
        # step / 3 per substep launch) x the points one launch updates / the
        # CUDA-event launch time
        alg_pt = b_alg(preset) / 3
        achieved = alg_pt * nloc / (avg_ms * 1e-3) / 1e9
        res = {
            "preset": preset, "value": rate, "ms_per_step": ms_step,
            "b_alg_bytes_per_pt": b_alg(preset),
            "b_alg_frac": rate * b_alg(preset) / 1e9 / hbm,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic_lookup(preset, nloc, fused),
                         "kernel": kname, "avg_ms_per_substep": avg_ms,
                         "basis": "B_alg/3 bytes per point per launch (SURVEY.md 8(d)); traffic = "
                                  "ncu dram bytes of the same launch (profiles/ncu_traffic.json)",
                         "bytes_per_pt_per_launch": alg_pt,
                         "compulsory_bytes_per_pt_per_launch": comp_pt,
                         "compulsory_frac": comp_pt * nloc / (avg_ms * 1e-3) / 1e9 / hbm,
                         "compute": compute_roofline(preset, nloc, avg_ms, ceil),
                         "peak_source": peak_src},
            "kernel_ms": {"dominant": kms[0], "rk": kms[1], "halo": kms[2], "other": kms[3]},
            "gpu_launches": int(klaunch[0] + klaunch[1] + klaunch[3]),
            "clocks": clk.summary(),
            "path": "fused" if fused else "staged",
        }
        if with_extras and not args.no_e2e:
            res["e2e"] = (e2e_run_slab(m, s, n, dt, args.steps, world, rank, zper, red_dev) if use_nccl
                          else e2e_run(m, s, n, dt, args.steps, world, rank))
        mc = s.memory_census()
        bq_ = PRESET_KINDS[preset][0]
        res["memory"] = {
            "device_bytes": mc["device_bytes"], "census_bytes": mc["total_bytes"],
            "census_b64_bytes": mc["baseline_b64_bytes"], "census_gain": mc["gain"],
            "device_gain_vs_census_b64": mc["baseline_b64_bytes"] / mc["device_bytes"],
            "census_per_class": mc["per_class"],
            "note": "device_bytes: HBM this solver holds (Q double-buffered, Qt in place, R never "
                    "allocated on the fused path); census: the reference's analytic memory_report "
                    "of its field set (registry.cpp:24-39)"}
        if use_nccl:
            # measured ncclSend bytes per RK step vs comm_volume_report's model
            # (registry.cpp:41-66; depth 2, q exchanged 3x per iteration)
            steps_run = args.warmup + args.steps
            res["halo"] = {"measured_bytes_per_step": halo_sent / steps_run,
                           "model_bytes_per_step": (2 * 2 * n * n * bq_ * 3 * 5 if world > 1 else 0),
                           "note": "we exchange Q only, 4 ghost planes deep (primitives and "
                                   "gradients are rebuilt from ghost Q), in q storage precision"}
        s.close()
        del s
        torch.cuda.synchronize()
        return res

    head = measure(args.precision, True)
    extra = {}
    for p in [x for x in args.modes.split(",") if x and x != args.precision]:
        try:
            r = measure(p, False)
            extra[p] = {k: r[k] for k in ("value", "ms_per_step", "b_alg_frac", "path", "memory")}
            extra[p]["roofline_frac"] = r["roofline"]["frac"]
            extra[p]["compute"] = r["roofline"]["compute"]
        except Exception as e:  # report, never hide
            extra[p] = {"error": str(e)}
    # the decomposition's own cost on one GPU: the same grid cut into P
    # LOCAL z-slabs (ghost-plane recompute, the interior / boundary launch
    # split, the overlapped exchange by device copies) -- the per-GPU part of
    # weak-scaling efficiency, everything but the link
    sweep = {}
    if world == 1 and args.slab_sweep:
        base = None
        for P in [1] + [int(x) for x in args.slab_sweep.split(",") if x]:
            for ov in ((True,) if P == 1 else (True, False)):
                key = str(P) if P == 1 else f"{P}/{'overlap' if ov else 'exchange_first'}"
                try:
                    r = measure(args.slab_preset, False, local_pz=P, overlap=ov)
                    base = base or r["ms_per_step"]
                    sweep[key] = {"ms_per_step": r["ms_per_step"], "value": r["value"],
                                  "efficiency_vs_1_slab": base / r["ms_per_step"]}
                except Exception as e:  # report, never hide
                    sweep[key] = {"error": str(e)}
        # weak scaling's slab: a whole n^3 period per slab (z_periods = P)
        P = max([int(x) for x in args.slab_sweep.split(",") if x] or [1])
        try:
            r = measure(args.slab_preset, False, local_pz=P, zper_override=P)
            sweep[f"{P}/weak"] = {"ms_per_step": r["ms_per_step"], "value": r["value"],
                                  "efficiency_vs_1_slab": r["value"] / (args.grid ** 3 * 1e3 / base)}
        except Exception as e:
            sweep[f"{P}/weak"] = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": dtype_of(args.precision), "data": "synthetic",
            "config": {"workload": (f"TGV {args.grid}^3 {args.precision} (M=0.1, Re=1600, "
                                    f"{args.split}, {args.strategy}, {args.emulation})"
                                    + (f", {args.grid}^3 per GPU ({args.grid}x{args.grid}x"
                                       f"{args.grid * world} stacked periods)"
                                       if args.scaling == "weak" and world > 1 else "")),
                       "n": args.grid, "precision": args.precision, "path": head["path"],
                       "decomposition": f"z-slabs x{world}" + ((" (IPC copy engines)" if args.transport == "ipc"
                                                                  else " (NCCL)") if use_nccl else ""),
                       "halo_exchange": ("overlapped with interior planes (2 streams)"
                                         if use_nccl and not args.no_overlap
                                         and args.grid * (world if args.scaling == "weak" else 1) // world >= 128
                                         else "before each substep (slabs < 128 planes)" if use_nccl
                                         and not args.no_overlap else
                                         "before each substep" if use_nccl else
                                         "periodic self-copy (1 slab)"),
                       "l2": "state >> 126 MB L2 (no flush needed)"},
            "roofline": head["roofline"],
            "b_alg": {"bytes_per_pt_per_step": head["b_alg_bytes_per_pt"],
                      "frac_of_hbm": head["b_alg_frac"]},
            "gpu_launches": head["gpu_launches"],
            "memory": head.get("memory"),
            "clocks": head["clocks"],
            "kernel_ms": head["kernel_ms"],
            "per_precision": {args.precision: {"value": head["value"],
                                               "ms_per_step": head["ms_per_step"],
                                               "b_alg_frac": head["b_alg_frac"],
                                               "memory": head.get("memory")}, **extra},
            "issue_ceiling_lane_ops_per_s": ceil,
        }
        if "e2e" in head:
            line["e2e"] = head["e2e"]
        if sweep:
            sweep["note"] = (f"{args.slab_preset}: the {args.grid}^3 grid cut into P LOCAL z-slabs on one GPU "
                             "(P/overlap: interior launch overlapped with the exchange, then the boundary "
                             "planes; P/exchange_first: exchange, then one launch), and P slabs of one "
                             f"{args.grid}^3 period each (P/weak, z_periods = P): the decomposition's own cost at "
                             "P GPUs' slab thickness, without the link")
            line["slab_sweep"] = sweep
        if not args.no_memory_table and world == 1:
            line["memory_table"] = memory_table(m, args, local)
        if "halo" in head:
            line["halo"] = head["halo"]
        if not args.no_cpu_baseline and world == 1:
            try:
                rate, cores, kind, sample = cpu_reference_run(args.precision, args.strategy,
                                                              args.emulation, args.grid,
                                                              CPU_STEPS, CPU_WARMUP)
                line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores,
                                        "kind": kind, "sample": sample}
            except Exception as e:
                line["cpu_baseline"] = {"value": None, "error": str(e)}
            for p, v in cpu_per_precision([p for p in extra if "error" not in extra[p]], args).items():
                extra[p]["cpu_baseline"] = v
        print(json.dumps(line), flush=True)
    if use_nccl:
        dist.destroy_process_group()
    return 0


def memory_table(m, args, device):
    """The paper's memory table measured: per preset, the
    HBM the solver holds against the reference's analytic census of the same
    field set (memory_report, registry.cpp:24-39), for the Default strategy
    on the materialised path (the reference's dataflow: the 12 ddx1-staged
    gradients held at wk storage, plus primitives and level-2 fields) and
    for Storesome on the fused path the bench times (primitives, gradients
    and level-2 fields never reach HBM).  Allocation only: one residual
    evaluation on a uniform state allocates the staged arrays."""
    out = {}
    for preset in ("DP", "SPDP", "HPSP"):
        row = {}
        for strategy, path in (("default", "materialised"), ("storesome", "fused")):
            try:
                s = m.Solver(m.GridSpec(args.grid), m.resolve_preset(preset, args.emulation), strategy,
                             m.FlowParams(0.1, 1600.0, 0.72, 1.4, True), args.split, m.Decomposition(device=device))
                s.set_path(path)
                s.init_uniform()
                if path == "materialised":
                    s.evaluate()
                mc = s.memory_census()
                row[f"{strategy}/{path}"] = {"device_bytes": mc["device_bytes"], "census_bytes": mc["total_bytes"],
                                             "census_b64_bytes": mc["baseline_b64_bytes"],
                                             "census_gain": mc["gain"],
                                             "device_over_census": mc["device_bytes"] / mc["total_bytes"]}
                s.close()
            except Exception as e:  # report, never hide
                row[f"{strategy}/{path}"] = {"error": str(e)}
        out[preset] = row
    out["note"] = (f"{args.grid}^3; device_bytes = HBM held (Q double-buffered on the fused path, "
                   "staged arrays with ghost planes on the materialised path); census = the "
                   "reference's memory_report for the same field set, halos included")
    return out


PIPE = {8: "fp64 (DADD/DMUL)", 4: "fp32 pairs (FADD2/FFMA2)", 2: "fp16 pairs (HADD2/HMUL2)"}
CEIL_KEY = {8: "fp64", 4: "fp32", 2: "fp16"}


def compute_roofline(preset, npts, avg_ms, ceil):
    """Secondary (compute) roofline of the fused kernel: its floating-point
    lane operations per point per launch, counted by ncu on the committed
    capture (profiles/ncu_ops.json: smsp__sass_thread_inst_executed_op_*
    summed over the residual compute type's add/mul/fma, packed
    instructions counted per lane), at the CUDA-event launch time, against
    the measured issue ceiling of that arithmetic (mpfd_b200_issue_ceiling)."""
    rb = PRESET_KINDS[preset][2]
    out = {"pipe": PIPE[rb], "ceiling_gops": None, "ops_per_pt_per_launch": None,
           "achieved_gops": None, "frac": None}
    if isinstance(ceil, dict) and CEIL_KEY[rb] in ceil:
        out["ceiling_gops"] = ceil[CEIL_KEY[rb]] / 1e9
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_ops.json")) as f:
            d = json.load(f)
    except Exception:
        d = {}
    ops = d.get(f"{preset}/fused/ops_per_pt")
    pct = d.get(f"{preset}/fused/pipe_active_pct")
    if ops:
        out["ops_per_pt_per_launch"] = ops
        out["achieved_gops"] = ops * npts / (avg_ms * 1e-3) / 1e9
        if out["ceiling_gops"]:
            out["frac"] = out["achieved_gops"] / out["ceiling_gops"]
    out["ncu_pipe_active_pct"] = pct
    issue = d.get(f"{preset}/fused/issue_active_pct")
    stalls = d.get(f"{preset}/fused/top_stalls")
    if issue is not None:
        # what bounds the kernel, from the committed capture: the HBM
        # fraction above is far from 1, so it is the instruction stream
        out["limiter"] = (f"issue/latency: issue {issue}% of peak, {PIPE[rb].split()[0]} pipe {pct}% active, "
                          f"warps {d.get(f'{preset}/fused/warps_active_pct')}% of max; top stalls "
                          + ", ".join(f"{a} {b}" for a, b in (stalls or [])[:3]))
    return out


def traffic_lookup(preset, npts, fused):
    """DRAM bytes per launch of the dominant kernel: the per-point
    dram__bytes_read.sum + dram__bytes_write.sum of the committed ncu --set
    full capture (profiles/ncu_traffic.json, 256^3) times this launch's
    points; None when no capture exists for this preset and path."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(f"{preset}/{'fused' if fused else 'staged'}/bytes_per_pt")
        return None if v is None else v * npts
    except Exception:
        return None


def e2e_run_slab(m, s, n, dt, steps, world, rank, zper, red_dev="cuda"):
    """e2e under the NCCL decomposition: every rank uploads its own z-slab of
    Q from pinned interior binary64 host carriers (the C-ABI's global-index
    set/get with the carrier pointer offset to the slab), advances `steps`
    RK steps with a diagnostics sample at the end (NCCL-reduced), reads its
    slab back; the time is the max over ranks of the wall clock around all
    of it.  Bytes are whole-job per step."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    nz_glob = n * zper
    nzl = nz_glob // world
    z0 = rank * nzl
    host = [torch.empty((nzl, n, n), dtype=torch.float64, pin_memory=True) for _ in range(5)]
    s.init_tgv()
    plane = n * n * 8
    ptrs = [C.c_void_p(h.data_ptr() - z0 * plane) for h in host]  # global-index view of the slab
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_get_state_interior(s.h, 0, c, C.cast(ptrs[c], C.POINTER(C.c_double))))
    s.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_set_state_interior(s.h, 0, c, C.cast(ptrs[c], C.POINTER(C.c_double))))
    r = s.advance(m.StepConfig(dt, steps, steps))
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_get_state_interior(s.h, 0, c, C.cast(ptrs[c], C.POINTER(C.c_double))))
    el = time.perf_counter() - t0
    t = torch.tensor([el], device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t.item())
    pts = n * n * nz_glob
    return {"value": pts * steps / el, "unit": UNIT, "h2d_bytes_per_step": 5 * pts * 8 / steps,
            "d2h_bytes_per_step": (5 * pts * 8 + 2 * 2 * (pts // 4096) * 8) / steps,
            "note": "advance() through the C-ABI on every rank: its Q slab uploaded from pinned "
                    "interior binary64 host carriers, diagnostics sampled at t=0 and t_end (gathered), "
                    "the slab read back; max over ranks; bytes whole-job, amortised over the steps",
            "diverged": r.diverged}


def e2e_run(m, s_unused, n, dt, steps, world, rank):
    """Same metric through the reference-facing C-ABI with HOST buffers:
    pinned ext^3 binary64 carriers (the reference Field layout) uploaded,
    `steps` RK steps advanced with a diagnostics sample (D2H) at the end,
    the state read back; all inside the timed region."""
    import ctypes as C

    import numpy as np
    import torch

    if world > 1:
        return None
    e = n + 8
    # pinned host carriers for the 5 components of Q
    host = [torch.empty((e, e, e), dtype=torch.float64, pin_memory=True) for _ in range(5)]
    s = s_unused
    s.init_tgv()
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_get_state(
            s.h, 0, c, C.cast(host[c].data_ptr(), C.POINTER(C.c_double))))
    s.synchronize()
    t0 = time.perf_counter()
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_set_state(
            s.h, 0, c, C.cast(host[c].data_ptr(), C.POINTER(C.c_double))))
    r = s.advance(m.StepConfig(dt, steps, steps))
    for c in range(5):
        m.solver._check(s.L.mpfd_b200_get_state(
            s.h, 0, c, C.cast(host[c].data_ptr(), C.POINTER(C.c_double))))
    el = time.perf_counter() - t0
    h2d = 5 * n ** 3 * 8 / steps
    d2h = (5 * n ** 3 * 8 + 2 * 2 * (n ** 3 // 4096) * 8) / steps
    return {"value": n ** 3 * steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "note": "advance() through the C-ABI: Q uploaded from pinned ext^3 binary64 host "
                    "carriers, diagnostics sampled at t=0 and t_end, Q read back; bytes "
                    "amortised over the steps", "diverged": r.diverged}


if __name__ == "__main__":
    sys.exit(main())
