"""Python mirror of the reference solver API over the B200 C-ABI.

Reference names kept (file:line in /root/reference/proj):
  PrecisionConfig / resolve_preset     precision.hpp:181-199, precision.cpp:58-88
  GridSpec                             field.hpp:20-56
  FlowParams                           physics.hpp:26-34
  SplitCoefficients / split_preset     physics.hpp:40-63, physics.cpp:19-43
  RKScheme / StepConfig                integrate.hpp:18-28
  DivergenceEvent                      physics.hpp:85-91
  DiagnosticsRecord                    tgv.hpp:13-20
  AdvanceResult                        integrate.hpp:35-43
  Solver = make_solver_fields + ResidualEvaluator + rk_substep + advance +
           DiagnosticsComputer         physics.cpp:441-587, integrate.cpp:47-167,
                                       tgv.cpp:29-175
Errors mirror the reference: ConfigError for configuration problems,
divergence reported as a value (DivergenceEvent), DeviceError for CUDA/NCCL.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MPFD_B200_LIB selects an alternative in-tree build (developer A/B runs)
library_path = os.environ.get("MPFD_B200_LIB") or os.path.join(HERE, "libmpfd_b200.so")

B16, B32, B64 = 0, 1, 2
STRICT, STOREROUND = 0, 1
DEFAULT, STORESOME = 0, 1
_KIND = {"B16": B16, "B32": B32, "B64": B64}


class ConfigError(ValueError):
    """ConfigError / RegistryError (precision.hpp:23-28)."""


class DeviceError(RuntimeError):
    """CUDA or NCCL failure inside the B200 library."""


# ---------------------------------------------------------------------------
# C structs (include/mpfd_b200.h)
class _Grid(C.Structure):
    _fields_ = [("n", C.c_int), ("domain_length", C.c_double), ("z_periods", C.c_int)]


class _Prec(C.Structure):
    _fields_ = [("q_vector", C.c_int), ("rk_arrays", C.c_int), ("residuals", C.c_int),
                ("wk_arrays", C.c_int), ("emulation", C.c_int), ("n_overrides", C.c_int),
                ("override_names", C.POINTER(C.c_char_p)), ("override_kinds", C.POINTER(C.c_int))]


class _Flow(C.Structure):
    _fields_ = [("mach", C.c_double), ("reynolds", C.c_double), ("prandtl", C.c_double),
                ("gamma", C.c_double), ("viscous", C.c_int)]


class _Split(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("alpha", "beta_rho", "beta_u", "beta_phi", "gamma_rho", "gamma_u", "gamma_phi")]


# int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes)
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class _HostComm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", _ALLGATHER)]


class _Decomp(C.Structure):
    _fields_ = [("pz", C.c_int), ("mode", C.c_int), ("rank", C.c_int), ("device", C.c_int),
                ("devices", C.POINTER(C.c_int)), ("nccl_id", C.c_void_p),
                ("hostcomm", C.POINTER(_HostComm)), ("py", C.c_int)]


class _Div(C.Structure):
    _fields_ = [("code", C.c_int), ("i", C.c_int), ("j", C.c_int), ("k", C.c_int),
                ("time", C.c_double), ("iteration", C.c_long), ("substep", C.c_int)]


class _Diag(C.Structure):
    _fields_ = [("t", C.c_double), ("kinetic_energy", C.c_double), ("enstrophy", C.c_double),
                ("eps_s", C.c_double), ("ke_normalized", C.c_double), ("diverged", C.c_int)]


class _Step(C.Structure):
    _fields_ = [("a", C.c_double * 3), ("b", C.c_double * 3), ("dt", C.c_double),
                ("n_iterations", C.c_long), ("diagnostics_interval", C.c_int),
                ("ke_weighting", C.c_int), ("threads", C.c_int)]


class _AdvInfo(C.Structure):
    _fields_ = [("iterations_run", C.c_long), ("wall_seconds", C.c_double),
                ("seconds_per_iteration", C.c_double)]


class _Census(C.Structure):
    _fields_ = [("count", C.c_long * 5), ("bytes", C.c_size_t * 5), ("total_bytes", C.c_size_t),
                ("baseline_b64_bytes", C.c_size_t), ("gain", C.c_double), ("device_bytes", C.c_size_t)]


_lib = None


def lib():
    """The loaded C-ABI library.  Raises if the sm_100a extension is missing:
    the product path has no CPU fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(
                f"{library_path} is missing: build it with `python -m "
                "paper_2505_20911_b200.build` (nvcc, sm_100a)")
        L = C.CDLL(library_path)
        P = C.c_void_p
        I = C.c_int
        D = C.c_double
        L.mpfd_b200_last_error.restype = C.c_char_p
        L.mpfd_b200_version.restype = C.c_char_p
        L.mpfd_b200_resolve_preset.argtypes = [C.c_char_p, C.POINTER(_Prec)]
        L.mpfd_b200_split_preset.argtypes = [C.c_char_p, C.POINTER(_Split)]
        L.mpfd_b200_nccl_unique_id.argtypes = [P]
        L.mpfd_b200_create.argtypes = [C.POINTER(_Grid), C.POINTER(_Prec), I, C.POINTER(_Flow),
                                       C.POINTER(_Split), C.POINTER(_Decomp), C.POINTER(P)]
        L.mpfd_b200_destroy.argtypes = [P]
        L.mpfd_b200_init_tgv.argtypes = [P]
        L.mpfd_b200_init_uniform.argtypes = [P]
        DP = C.POINTER(D)
        for fn in ("set_state", "get_state", "set_state_interior", "get_state_interior"):
            getattr(L, "mpfd_b200_" + fn).argtypes = [P, I, I, DP]
        L.mpfd_b200_residual.argtypes = [P, C.POINTER(_Div)]
        L.mpfd_b200_rk_substep.argtypes = [P, I, DP, DP, D, C.POINTER(_Div)]
        L.mpfd_b200_halo_refresh.argtypes = [P]
        L.mpfd_b200_diagnostics.argtypes = [P, I, D, I, C.POINTER(_Diag)]
        L.mpfd_b200_advance.argtypes = [P, C.POINTER(_Step), C.POINTER(_Diag), C.c_long,
                                        C.POINTER(C.c_long), C.POINTER(_Div), C.POINTER(C.c_long)]
        L.mpfd_b200_stream.restype = P
        L.mpfd_b200_stream.argtypes = [P]
        L.mpfd_b200_synchronize.argtypes = [P]
        L.mpfd_b200_run_steps.argtypes = [P, C.POINTER(_Step), C.c_long]
        L.mpfd_b200_profile.argtypes = [P, I]
        L.mpfd_b200_profile_read.argtypes = [P, DP, C.POINTER(C.c_long)]
        L.mpfd_b200_halo_bytes.argtypes = [P, C.POINTER(C.c_ulonglong)]
        L.mpfd_b200_field_kind.argtypes = [P, I, C.c_char_p, C.POINTER(I)]
        L.mpfd_b200_memory.argtypes = [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                       C.POINTER(C.c_size_t)]
        L.mpfd_b200_set_path.argtypes = [P, I]
        L.mpfd_b200_set_overlap.argtypes = [P, I]
        L.mpfd_b200_set_exact_divergence.argtypes = [P, I]
        L.mpfd_b200_advance_info.argtypes = [P, C.POINTER(_AdvInfo)]
        L.mpfd_b200_memory_census.argtypes = [P, C.POINTER(_Census)]
        L.mpfd_b200_issue_ceiling.argtypes = [I, C.POINTER(D)]
        L.mpfd_b200_halo_plan.argtypes = [I, I, I, I, C.POINTER(C.c_longlong)]
        L.mpfd_b200_merge_divergence.argtypes = [C.POINTER(C.c_ulonglong), I, I, D, C.POINTER(_Div)]
        L.mpfd_b200_merge_diagnostics.argtypes = [DP, C.c_size_t, C.c_size_t, I, I, DP]
        _lib = L
    return _lib


def issue_ceiling(device: int = 0) -> dict:
    """Measured lane-op/s of unfused add/mul on `device`: fp64 (DADD/DMUL),
    fp32 pairs (FADD2/FFMA2), fp16 pairs (HADD2/HMUL2)."""
    out = (C.c_double * 3)()
    _check(lib().mpfd_b200_issue_ceiling(device, out))
    return {"fp64": out[0], "fp32": out[1], "fp16": out[2]}


def _check(rc: int):
    if rc == 0 or rc == 2:
        return rc
    msg = lib().mpfd_b200_last_error().decode()
    if rc == 1:
        raise ConfigError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------------------
@dataclass
class PrecisionConfig:
    q_vector: int = B64
    rk_arrays: int = B64
    residuals: int = B64
    wk_arrays: int = B64
    custom_overrides: Dict[str, int] = field(default_factory=dict)
    emulation: int = STRICT

    def resolve(self, cls: int, name: str) -> int:
        if name in self.custom_overrides:
            return self.custom_overrides[name]
        if cls == 4:
            return B64
        return (self.q_vector, self.rk_arrays, self.residuals, self.wk_arrays)[cls]


def resolve_preset(name: str, emulation: str | int = STRICT) -> PrecisionConfig:
    p = _Prec()
    _check(lib().mpfd_b200_resolve_preset(name.encode(), C.byref(p)))
    emu = emulation if isinstance(emulation, int) else (
        STRICT if emulation == "strict" else STOREROUND)
    return PrecisionConfig(p.q_vector, p.rk_arrays, p.residuals, p.wk_arrays, {}, emu)


@dataclass
class GridSpec:
    """GridSpec (field.hpp:20-56).  z_periods > 1 is a B200 extension for weak
    scaling: n x n x (z_periods*n) points, the 2 pi-periodic TGV repeated
    exactly along z (include/mpfd_b200.h)."""
    n: int = 32
    domain_length: float = 2.0 * math.pi
    z_periods: int = 1

    halo_depth = 4

    def __post_init__(self):
        if self.n < 5:
            raise ConfigError("GridSpec: n must be >= 5")
        if self.z_periods < 1:
            raise ConfigError("GridSpec: z_periods must be >= 1")

    @property
    def nz(self) -> int:
        return self.n * self.z_periods

    def spacing(self) -> float:
        return self.domain_length / self.n

    def ext(self) -> int:
        return self.n + 2 * self.halo_depth


@dataclass
class FlowParams:
    mach: float = 0.5
    reynolds: float = 800.0
    prandtl: float = 0.72
    gamma: float = 1.4
    viscous: bool = True


@dataclass
class SplitCoefficients:
    alpha: float = 1.0
    beta_rho: float = 0.0
    beta_u: float = 0.0
    beta_phi: float = 0.0
    gamma_rho: float = 0.0
    gamma_u: float = 0.0
    gamma_phi: float = 0.0


def split_preset(name: str) -> SplitCoefficients:
    s = _Split()
    _check(lib().mpfd_b200_split_preset(name.encode(), C.byref(s)))
    return SplitCoefficients(*(getattr(s, k) for k, _ in _Split._fields_))


@dataclass
class RKScheme:
    a: Tuple[float, float, float] = (0.0, -5.0 / 9.0, -153.0 / 128.0)
    b: Tuple[float, float, float] = (1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0)


@dataclass
class StepConfig:
    dt: float = 0.005
    n_iterations: int = 4000
    diagnostics_interval: int = 100


@dataclass
class DivergenceEvent:
    what: str
    i: int
    j: int
    k: int
    time: float = -1.0
    iteration: int = -1
    substep: int = -1


_WHAT = {1: "nonpositive or nonfinite density", 2: "nonfinite residual", 3: "nonfinite state"}


@dataclass
class DiagnosticsRecord:
    t: float = 0.0
    kinetic_energy: float = 0.0
    enstrophy: float = 0.0
    eps_s: float = 0.0
    ke_normalized: float = 0.0
    diverged: bool = False


@dataclass
class AdvanceResult:
    diverged: bool
    divergence: Optional[DivergenceEvent]
    iterations_run: int
    series: List[DiagnosticsRecord]
    wall_seconds: float = 0.0            # integrate.hpp:41-42
    seconds_per_iteration: float = 0.0


LOCAL, NCCL, IPC = 0, 1, 2  # decomposition transports (mpfd_b200.h)


@dataclass
class Decomposition:
    """z-slab decomposition: pz slabs, LOCAL (all slabs in this process),
    NCCL (one slab per rank, `nccl_id` from Solver.nccl_unique_id()) or IPC
    (one slab per rank, ghost planes pulled by copy engines from the
    neighbours' CUDA-IPC-mapped buffers; `allgather(bytes) -> bytes` is the
    host collective, every rank's contribution concatenated in rank order)."""
    pz: int = 1
    mode: int = LOCAL
    rank: int = 0
    device: int = 0
    devices: Optional[List[int]] = None
    nccl_id: Optional[bytes] = None
    allgather: Optional[object] = None
    py: int = 1  # y pencils (LOCAL, staged path): a 1 x py x pz process grid


def gloo_allgather(group=None):
    """A Decomposition.allgather over torch.distributed (CPU tensors, e.g. the
    gloo backend)."""
    import torch
    import torch.distributed as dist

    def ag(data: bytes) -> bytes:
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, t, group=group)
        return b"".join(o.numpy().tobytes() for o in out)
    return ag


def halo_plan(n: int, pz: int, rank: int, bytes_q: int) -> dict:
    """The z-slab halo plan the solver uses (mpfd_b200_halo_plan)."""
    out = (C.c_longlong * 9)()
    _check(lib().mpfd_b200_halo_plan(n, pz, rank, bytes_q, out))
    keys = ("send_up", "recv_lo", "send_dn", "recv_hi", "block", "up", "dn", "z0", "nzl")
    return dict(zip(keys, list(out)))


def merge_divergence(tables: np.ndarray, n: int, dt: float) -> Optional["DivergenceEvent"]:
    """The solver's merge of per-slab / per-rank divergence records
    (mpfd_b200_merge_divergence): tables of shape (count, 15) uint64."""
    t = np.ascontiguousarray(tables, dtype=np.uint64).reshape(-1, 15)
    ev = _Div()
    rc = _check(lib().mpfd_b200_merge_divergence(t.ctypes.data_as(C.POINTER(C.c_ulonglong)), t.shape[0], n,
                                                  dt, C.byref(ev)))
    return _div(ev) if rc == 2 else None


def merge_diagnostics(parts: np.ndarray, npoints: int, threads: int, chunked: bool) -> float:
    """The solver's host reduction of gathered diagnostics partials
    (mpfd_b200_merge_diagnostics)."""
    p = np.ascontiguousarray(parts, dtype=np.float64)
    out = C.c_double()
    _check(lib().mpfd_b200_merge_diagnostics(_dp(p), p.size, npoints, threads, 1 if chunked else 0,
                                             C.byref(out)))
    return out.value


def _div(d: _Div) -> DivergenceEvent:
    return DivergenceEvent(_WHAT.get(d.code, "?"), d.i, d.j, d.k, d.time, d.iteration, d.substep)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Solver:
    """make_solver_fields + ResidualEvaluator + the RK driver on B200."""

    def __init__(self, grid: GridSpec, precision: PrecisionConfig, strategy: int | str,
                 flow: FlowParams, split: SplitCoefficients | str = "Blaisdell",
                 decomp: Optional[Decomposition] = None):
        L = lib()
        if isinstance(strategy, str):
            if strategy not in ("default", "storesome"):
                raise ConfigError(f"unknown strategy '{strategy}' (expected default or storesome)")
            strategy = DEFAULT if strategy == "default" else STORESOME
        if isinstance(split, str):
            split = split_preset(split)
        self.grid, self.precision, self.flow, self.split = grid, precision, flow, split
        self.n = grid.n
        self.nz = grid.nz
        names = list(precision.custom_overrides)
        self._keep = [n.encode() for n in names]
        p = _Prec(precision.q_vector, precision.rk_arrays, precision.residuals,
                  precision.wk_arrays, precision.emulation, len(names),
                  (C.c_char_p * max(1, len(names)))(*self._keep),
                  (C.c_int * max(1, len(names)))(*[precision.custom_overrides[k] for k in names]))
        g = _Grid(grid.n, grid.domain_length, grid.z_periods)
        f = _Flow(flow.mach, flow.reynolds, flow.prandtl, flow.gamma, 1 if flow.viscous else 0)
        s = _Split(*(getattr(split, k) for k, _ in _Split._fields_))
        d = decomp or Decomposition()
        self._devs = (C.c_int * max(1, len(d.devices or [])))(*(d.devices or [0]))
        self._nid = C.create_string_buffer(d.nccl_id, 128) if d.nccl_id else None
        self._hc = None
        if d.allgather is not None:
            fn = d.allgather

            def _ag(ctx, send, recv, nbytes):
                try:
                    out = fn(C.string_at(send, nbytes))
                    C.memmove(recv, out, len(out))
                    return 0
                except Exception:  # reported to the solver as a failed collective
                    return 1
            self._agf = _ALLGATHER(_ag)  # kept alive with the solver
            self._hc = _HostComm(None, self._agf)
        dd = _Decomp(d.pz, d.mode, d.rank, d.device,
                     self._devs if d.devices else None,
                     C.cast(self._nid, C.c_void_p) if self._nid else None,
                     C.pointer(self._hc) if self._hc is not None else None, d.py)
        self.h = C.c_void_p()
        _check(L.mpfd_b200_create(C.byref(g), C.byref(p), strategy, C.byref(f), C.byref(s),
                                  C.byref(dd), C.byref(self.h)))
        self.L = L

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.L.mpfd_b200_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().mpfd_b200_nccl_unique_id(buf))
        return buf.raw

    # --- setup ------------------------------------------------------------
    def init_tgv(self):
        _check(self.L.mpfd_b200_init_tgv(self.h))

    def init_uniform(self):
        _check(self.L.mpfd_b200_init_uniform(self.h))

    # --- carriers ----------------------------------------------------------
    def get_field(self, cls: int, comp: int) -> np.ndarray:
        """Interior n^3 binary64 carrier, indexed [k, j, i]."""
        out = np.empty((self.nz, self.n, self.n))
        _check(self.L.mpfd_b200_get_state_interior(self.h, cls, comp, _dp(out)))
        return out

    def set_field(self, cls: int, comp: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        if a.shape != (self.nz, self.n, self.n):
            raise ConfigError(f"carrier shape {a.shape} != {(self.nz, self.n, self.n)}")
        _check(self.L.mpfd_b200_set_state_interior(self.h, cls, comp, _dp(a)))

    def get_state(self, cls: int) -> np.ndarray:
        return np.stack([self.get_field(cls, c) for c in range(5)])

    def set_state(self, cls: int, arr: np.ndarray):
        for c in range(5):
            self.set_field(cls, c, arr[c])

    def get_field_ext(self, cls: int, comp: int) -> np.ndarray:
        e = self.n + 8
        out = np.zeros((self.nz + 8, e, e))
        _check(self.L.mpfd_b200_get_state(self.h, cls, comp, _dp(out)))
        return out

    def set_field_ext(self, cls: int, comp: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        e = self.n + 8
        if a.shape != (self.nz + 8, e, e):
            raise ConfigError(f"carrier shape {a.shape} != {(self.nz + 8, e, e)}")
        _check(self.L.mpfd_b200_set_state(self.h, cls, comp, _dp(a)))

    # --- hot path ----------------------------------------------------------
    def evaluate(self) -> Optional[DivergenceEvent]:
        """ResidualEvaluator::evaluate (physics.cpp:485-587)."""
        d = _Div()
        rc = _check(self.L.mpfd_b200_residual(self.h, C.byref(d)))
        return _div(d) if rc == 2 else None

    def rk_substep(self, substep: int, dt: float, scheme: RKScheme = RKScheme()
                   ) -> Optional[DivergenceEvent]:
        """rk_substep (integrate.cpp:47-91) + advance's finite guard."""
        a = np.array(scheme.a, dtype=np.float64)
        b = np.array(scheme.b, dtype=np.float64)
        d = _Div()
        rc = _check(self.L.mpfd_b200_rk_substep(self.h, substep, _dp(a), _dp(b), dt, C.byref(d)))
        return _div(d) if rc == 2 else None

    def fill_state_halos(self):
        _check(self.L.mpfd_b200_halo_refresh(self.h))

    def diagnostics(self, weighting: int = 0, t: float = 0.0, threads: int = 8
                    ) -> DiagnosticsRecord:
        d = _Diag()
        _check(self.L.mpfd_b200_diagnostics(self.h, weighting, t, threads, C.byref(d)))
        return DiagnosticsRecord(d.t, d.kinetic_energy, d.enstrophy, d.eps_s, d.ke_normalized,
                                 bool(d.diverged))

    def _step(self, step: StepConfig, scheme: RKScheme, weighting: int, threads: int) -> _Step:
        return _Step((C.c_double * 3)(*scheme.a), (C.c_double * 3)(*scheme.b), step.dt,
                     step.n_iterations, step.diagnostics_interval, weighting, threads)

    def advance(self, step: StepConfig, scheme: RKScheme = RKScheme(), weighting: int = 0,
                threads: int = 8, cap: int = 100000) -> AdvanceResult:
        """advance (integrate.cpp:97-167) with diagnostics sampling."""
        st = self._step(step, scheme, weighting, threads)
        cap = min(cap, 2 + (step.n_iterations // max(1, step.diagnostics_interval)
                            if step.diagnostics_interval > 0 else 0) + 2)
        series = (_Diag * cap)()
        ln, it = C.c_long(0), C.c_long(0)
        d = _Div()
        rc = _check(self.L.mpfd_b200_advance(self.h, C.byref(st), series, cap, C.byref(ln),
                                             C.byref(d), C.byref(it)))
        recs = [DiagnosticsRecord(x.t, x.kinetic_energy, x.enstrophy, x.eps_s, x.ke_normalized,
                                  bool(x.diverged)) for x in series[: ln.value]]
        info = _AdvInfo()
        _check(self.L.mpfd_b200_advance_info(self.h, C.byref(info)))
        return AdvanceResult(rc == 2, _div(d) if rc == 2 else None, it.value, recs,
                             info.wall_seconds, info.seconds_per_iteration)

    # --- measurement hooks --------------------------------------------------
    def run_steps(self, iters: int, dt: float, scheme: RKScheme = RKScheme()):
        st = self._step(StepConfig(dt, iters, 0), scheme, 0, 8)
        _check(self.L.mpfd_b200_run_steps(self.h, C.byref(st), iters))

    def synchronize(self):
        _check(self.L.mpfd_b200_synchronize(self.h))

    @property
    def stream(self) -> int:
        return self.L.mpfd_b200_stream(self.h) or 0

    def profile(self, enable: bool):
        _check(self.L.mpfd_b200_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        ms = np.zeros(4)
        ln = (C.c_long * 4)()
        _check(self.L.mpfd_b200_profile_read(self.h, _dp(ms), ln))
        return ms, list(ln)

    def memory(self):
        a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(self.L.mpfd_b200_memory(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def memory_census(self) -> dict:
        """memory_report (registry.cpp:24-39) of the reference's field set for
        this config, plus the HBM this solver holds (device_bytes)."""
        m = _Census()
        _check(self.L.mpfd_b200_memory_census(self.h, C.byref(m)))
        names = ("q_vector", "rk_arrays", "residuals", "wk_arrays", "diagnostics")
        return {"per_class": {nm: {"count": m.count[i], "bytes": m.bytes[i]} for i, nm in enumerate(names)},
                "total_bytes": m.total_bytes, "baseline_b64_bytes": m.baseline_b64_bytes,
                "gain": m.gain, "device_bytes": m.device_bytes}

    def set_exact_divergence(self, enable: bool):
        """Exact divergence state: Qt and R double-buffered, slabs/ranks in
        lock-step per substep (see mpfd_b200.h).  Default off."""
        _check(self.L.mpfd_b200_set_exact_divergence(self.h, 1 if enable else 0))

    def halo_bytes(self) -> int:
        """Bytes of ghost planes this rank moved so far (ncclSend or IPC pulls)."""
        v = C.c_ulonglong()
        _check(self.L.mpfd_b200_halo_bytes(self.h, C.byref(v)))
        return v.value

    def set_path(self, path: str):
        """"fused" (default), "staged" (one kernel per level) or "materialised"
        (staged, with the Default strategy's 12 gradients stored in HBM at wk
        storage -- the reference's dataflow and memory footprint)."""
        codes = {"staged": 0, "fused": 1, "materialised": 2}
        if path not in codes:
            raise ConfigError(f"unknown path '{path}' (expected one of {sorted(codes)})")
        _check(self.L.mpfd_b200_set_path(self.h, codes[path]))

    def set_overlap(self, enable: Optional[bool]):
        """Overlap the z-halo exchange with the interior planes: True, False,
        or None for the default policy (overlap where the exchange crosses a
        link and slabs are >= 128 planes thick).  Bitwise identical results
        either way."""
        _check(self.L.mpfd_b200_set_overlap(self.h, -1 if enable is None else (1 if enable else 0)))
