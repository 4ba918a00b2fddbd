"""pyoracle -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers of the B200 product:

* ``Oracle``: the C restatement in ``oracle/mpfd_oracle.c`` (always buildable
  with gcc; built into ``oracle/build/``).
* ``Reference``: the unmodified reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libmpfd_ref.so`` (present in
  this container and shipped prebuilt to the GPU box; absent otherwise).

Both expose the same methods so a test can run either side by side with the
B200 solver.  Only tests/, __graft_entry__.smoke() and bench.py's CPU leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libmpfd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpfd_ref.so")

B16, B32, B64 = 0, 1, 2

# PrecisionConfig presets (precision.cpp:58-88): (q, rk, res, wk)
PRESETS = {
    "DP": (B64, B64, B64, B64),
    "SP": (B32, B32, B32, B32),
    "HP": (B16, B16, B16, B16),
    "SPDP": (B64, B64, B32, B32),
    "SPDP-wk": (B64, B64, B64, B32),
    "SPDP-res": (B64, B64, B32, B64),
    "HPSP": (B32, B32, B16, B16),
    "HPSP-wk": (B32, B32, B32, B16),
    "HPSP-res": (B32, B32, B16, B32),
}

# SplitCoefficients presets (physics.cpp:19-43):
# alpha, beta_rho, beta_u, beta_phi, gamma_rho, gamma_u, gamma_phi
SPLITS = {
    "Divergence": (1.0, 0, 0, 0, 0, 0, 0),
    "Feiereisen": (0.5, 0, 0, 0.5, 0, 0, 0.5),
    "Blaisdell": (0.5, 0, 0.5, 0, 0, 0.5, 0),
    "Kok": (0.5, 0.5, 0, 0, 0.5, 0, 0),
    "KGP": (0.25,) * 7,
}

# field names per slot (make_solver_fields physics.cpp:441-475) and class
FIELD_NAMES = (
    ["rho", "rhou", "rhov", "rhow", "rhoE"]
    + ["rk_rho", "rk_rhou", "rk_rhov", "rk_rhow", "rk_rhoE"]
    + ["res_rho", "res_rhou", "res_rhov", "res_rhow", "res_rhoE"]
    + ["u", "v", "w", "p", "T"]
    + ["dudx", "dudy", "dudz", "dvdx", "dvdy", "dvdz", "dwdx", "dwdy", "dwdz"]
    + ["dTdx", "dTdy", "dTdz"]
)
FIELD_CLASS = [0] * 5 + [1] * 5 + [2] * 5 + [3] * 17
KIND_NAMES = {"B16": B16, "B32": B32, "B64": B64}


def resolve_kinds(preset: str, overrides: dict | None = None):
    """PrecisionConfig::resolve for every solver field (precision.cpp:46-56)."""
    cls = PRESETS[preset]
    ov = {k: (KIND_NAMES[v] if isinstance(v, str) else int(v)) for k, v in (overrides or {}).items()}
    kinds = [ov.get(name, cls[c]) for name, c in zip(FIELD_NAMES, FIELD_CLASS)]
    return list(cls), kinds


def ensure_built():
    if not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "mpfd_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


_orc = None
_ref = None


def oracle_lib():
    global _orc
    if _orc is None:
        ensure_built()
        L = C.CDLL(ORACLE_SO)
        P = C.c_void_p
        D = C.c_double
        L.orc_create.restype = P
        L.orc_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.c_int,
                                 C.POINTER(D), D, D, D, D, C.c_int]
        L.orc_destroy.argtypes = [P]
        L.orc_init.argtypes = [P, C.c_int]
        L.orc_evaluate.argtypes = [P, C.POINTER(C.c_longlong)]
        L.orc_rk_substep.argtypes = [P, C.c_int, D]
        L.orc_advance.argtypes = [P, D, C.c_long, C.c_int, C.c_int, C.c_int, C.POINTER(D), C.c_long,
                                  C.POINTER(C.c_long), C.POINTER(C.c_longlong), C.POINTER(C.c_long)]
        L.orc_diagnostics.argtypes = [P, C.c_int, D, C.c_int, C.POINTER(D)]
        L.orc_get_field.argtypes = [P, C.c_int, C.c_int, C.POINTER(D)]
        L.orc_set_field.argtypes = [P, C.c_int, C.c_int, C.POINTER(D)]
        L.orc_encode_b16.restype = C.c_uint16
        L.orc_encode_b16.argtypes = [D]
        L.orc_decode_b16.restype = D
        L.orc_decode_b16.argtypes = [C.c_uint16]
        L.orc_round_to.restype = D
        L.orc_round_to.argtypes = [C.c_int, D]
        L.orc_emulated_op.restype = D
        L.orc_emulated_op.argtypes = [C.c_int, C.c_int, C.c_char, D, D]
        L.orc_pairwise_sum.restype = D
        L.orc_pairwise_sum.argtypes = [C.POINTER(D), C.c_long]
        L.orc_deterministic_sum.restype = D
        L.orc_deterministic_sum.argtypes = [C.POINTER(D), C.c_long, C.c_int]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_set_threads(os.cpu_count() or 1)
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        P = C.c_void_p
        D = C.c_double
        L.ref_create.restype = P
        L.ref_create.argtypes = [C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_char_p, D, D, D, D,
                                 C.c_int, C.c_char_p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_destroy.argtypes = [P]
        L.ref_init.argtypes = [P, C.c_int]
        L.ref_fill_halos.argtypes = [P]
        L.ref_evaluate.argtypes = [P, C.c_int, C.POINTER(C.c_longlong)]
        L.ref_rk_substep.argtypes = [P, C.c_int, D, C.c_int]
        L.ref_advance.argtypes = [P, D, C.c_long, C.c_int, C.c_int, C.c_int, C.POINTER(D), C.c_long,
                                  C.POINTER(C.c_long), C.POINTER(C.c_longlong), C.POINTER(C.c_long),
                                  C.POINTER(D)]
        L.ref_diagnostics.argtypes = [P, C.c_int, D, C.c_int, C.POINTER(D)]
        L.ref_get_field.argtypes = [P, C.c_int, C.c_int, C.POINTER(D)]
        L.ref_set_field.argtypes = [P, C.c_int, C.c_int, C.POINTER(D)]
        L.ref_get_field_ext.argtypes = [P, C.c_int, C.c_int, C.POINTER(D)]
        L.ref_storage_kind.argtypes = [P, C.c_int, C.c_int]
        L.ref_encode_b16.restype = C.c_uint16
        L.ref_encode_b16.argtypes = [D]
        L.ref_decode_b16.restype = D
        L.ref_decode_b16.argtypes = [C.c_uint16]
        L.ref_round_to.restype = D
        L.ref_round_to.argtypes = [C.c_int, D]
        L.ref_emulated_op.restype = D
        L.ref_emulated_op.argtypes = [C.c_int, C.c_int, C.c_char, D, D]
        L.ref_deterministic_sum.restype = D
        L.ref_deterministic_sum.argtypes = [C.POINTER(D), C.c_long, C.c_int]
        _ref = L
    return _ref


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class _Base:
    """Shared driver surface: fields are (n, n, n) arrays indexed [k, j, i]."""

    n: int

    def field(self, cls: int, comp: int) -> np.ndarray:
        out = np.empty((self.n, self.n, self.n), dtype=np.float64)
        self._get(cls, comp, out)
        return out

    def state(self, cls: int) -> np.ndarray:
        return np.stack([self.field(cls, c) for c in range(5)])

    def set_state(self, cls: int, arr: np.ndarray):
        for c in range(5):
            a = np.ascontiguousarray(arr[c], dtype=np.float64)
            self._set(cls, c, a)


class Oracle(_Base):
    """The C restatement (oracle/mpfd_oracle.c)."""

    def __init__(self, n, preset="DP", emulation="strict", strategy="storesome",
                 split="Blaisdell", mach=0.1, re=1600.0, pr=0.72, gamma=1.4, viscous=True,
                 overrides=None):
        L = oracle_lib()
        self.L, self.n = L, n
        cls, kinds = resolve_kinds(preset, overrides)
        w = (C.c_double * 7)(*SPLITS[split])
        self.h = L.orc_create(n, (C.c_int * 4)(*cls), (C.c_int * 32)(*kinds),
                              0 if emulation == "strict" else 1,
                              0 if strategy == "default" else 1, w, mach, re, pr, gamma,
                              1 if viscous else 0)
        if not self.h:
            raise ValueError("orc_create failed")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_destroy(self.h)
            self.h = None

    def init(self, case="tgv"):
        self.L.orc_init(self.h, 0 if case == "tgv" else 1)

    def evaluate(self):
        ev = (C.c_longlong * 6)()
        st = self.L.orc_evaluate(self.h, ev)
        return st, list(ev)

    def rk_substep(self, sub, dt):
        self.L.orc_rk_substep(self.h, sub, dt)

    def step(self, dt):
        for s in range(3):
            st, ev = self.evaluate()
            if st:
                return st, ev
            self.rk_substep(s, dt)
        return 0, None

    def advance(self, dt, n_iter, diag_interval=0, weighting=0, threads=8, cap=4096):
        series = np.zeros((cap, 5))
        ln, it = C.c_long(0), C.c_long(0)
        ev = (C.c_longlong * 6)()
        st = self.L.orc_advance(self.h, dt, n_iter, diag_interval, weighting, threads,
                                _dp(series), cap, C.byref(ln), ev, C.byref(it))
        return st, series[: ln.value].copy(), list(ev), it.value

    def diagnostics(self, weighting=0, t=0.0, threads=8):
        out = np.zeros(4)
        self.L.orc_diagnostics(self.h, weighting, t, threads, _dp(out))
        return out

    def _get(self, cls, comp, out):
        self.L.orc_get_field(self.h, cls, comp, _dp(out))

    def _set(self, cls, comp, a):
        self.L.orc_set_field(self.h, cls, comp, _dp(a))


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libmpfd_ref.so)."""

    def __init__(self, n, preset="DP", emulation="strict", strategy="storesome",
                 split="Blaisdell", mach=0.1, re=1600.0, pr=0.72, gamma=1.4, viscous=True,
                 overrides=None, threads=8):
        L = ref_lib()
        self.L, self.n, self.threads = L, n, threads
        ov = ";".join(f"{k}={v if isinstance(v, str) else ['B16', 'B32', 'B64'][v]}"
                      for k, v in (overrides or {}).items())
        self.h = L.ref_create(n, preset.encode(), 0 if emulation == "strict" else 1,
                              0 if strategy == "default" else 1, split.encode(), mach, re, pr,
                              gamma, 1 if viscous else 0, ov.encode())
        if not self.h:
            raise ValueError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def init(self, case="tgv"):
        if self.L.ref_init(self.h, 0 if case == "tgv" else 1):
            raise ValueError(self.L.ref_last_error().decode())

    def fill_halos(self):
        self.L.ref_fill_halos(self.h)

    def evaluate(self):
        ev = (C.c_longlong * 6)()
        st = self.L.ref_evaluate(self.h, self.threads, ev)
        return st, list(ev)

    def rk_substep(self, sub, dt):
        self.L.ref_rk_substep(self.h, sub, dt, self.threads)
        self.L.ref_fill_halos(self.h)

    def step(self, dt):
        for s in range(3):
            st, ev = self.evaluate()
            if st:
                return st, ev
            self.rk_substep(s, dt)
        return 0, None

    def advance(self, dt, n_iter, diag_interval=0, weighting=0, threads=None, cap=4096):
        series = np.zeros((cap, 5))
        ln, it = C.c_long(0), C.c_long(0)
        secs = C.c_double(0)
        ev = (C.c_longlong * 6)()
        st = self.L.ref_advance(self.h, dt, n_iter, diag_interval, weighting,
                                threads or self.threads, _dp(series), cap, C.byref(ln), ev,
                                C.byref(it), C.byref(secs))
        self.wall_seconds = secs.value
        return st, series[: ln.value].copy(), list(ev), it.value

    def diagnostics(self, weighting=0, t=0.0, threads=None):
        out = np.zeros(4)
        self.L.ref_diagnostics(self.h, weighting, t, threads or self.threads, _dp(out))
        return out

    def field_ext(self, cls, comp):
        e = self.n + 8
        out = np.empty((e, e, e))
        self.L.ref_get_field_ext(self.h, cls, comp, _dp(out))
        return out

    def storage_kind(self, cls, comp):
        return self.L.ref_storage_kind(self.h, cls, comp)

    def _get(self, cls, comp, out):
        self.L.ref_get_field(self.h, cls, comp, _dp(out))

    def _set(self, cls, comp, a):
        self.L.ref_set_field(self.h, cls, comp, _dp(a))
