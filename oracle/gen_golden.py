"""gen_golden.py -- TEST INFRASTRUCTURE ONLY.

Generates tests/golden/ from the unmodified reference library
(oracle/_ref/libmpfd_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  The fixtures pin the C restatement (tests/test_oracle.py)
and the B200 path (tests/test_gpu_parity.py) on machines where the reference
sources are absent (the GPU box).

  python oracle/gen_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import pyoracle as po  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

N_STEP = 8          # grid for the per-config step digests
DT = 0.002


def digest(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    if not po.ref_available():
        sys.exit("oracle/_ref missing: run `make -C oracle ref` with /root/reference present")
    os.makedirs(OUT, exist_ok=True)
    gold = {"source": "oracle/_ref (reference sources, unmodified)", "n": N_STEP, "dt": DT,
            "steps": {}, "series": {}, "divergence": {}, "codec": {}}
    arrays = {}
    # 1. one RK step (3 substeps) per preset x emulation x strategy; digests of
    #    Q, Qt, R after the step and R after the first evaluate
    for preset in po.PRESETS:
        for emu in ("strict", "storeround"):
            for strat in ("default", "storesome"):
                key = f"{preset}/{emu}/{strat}"
                r = po.Reference(N_STEP, preset=preset, emulation=emu, strategy=strat, threads=1)
                r.init()
                r.evaluate()
                r0 = r.state(2)
                for s in range(3):
                    if s:
                        r.evaluate()
                    r.rk_substep(s, DT)
                q, qt, rr = r.state(0), r.state(1), r.state(2)
                gold["steps"][key] = {"R0": digest(r0), "Q": digest(q), "Qt": digest(qt),
                                      "R": digest(rr)}
                if strat == "storesome" and emu == "strict" and preset in ("DP", "SPDP", "HPSP"):
                    arrays[f"{preset}_Q"] = q
                    arrays[f"{preset}_Qt"] = qt
                    arrays[f"{preset}_R"] = rr
    # 2. diagnostics series (advance with sampling), both reduction trees
    for preset in ("DP", "HPSP"):
        for threads in (1, 8):
            r = po.Reference(16, preset=preset, threads=threads)
            r.init()
            st, series, _, it = r.advance(DT, 8, 2, threads=threads)
            gold["series"][f"{preset}/t{threads}"] = series.tolist()
    # 3. a divergence event (inviscid Divergence split)
    for preset in ("DP", "HP"):
        r = po.Reference(16, preset=preset, split="Divergence", viscous=False, mach=0.4)
        r.init()
        st, series, ev, it = r.advance(0.2, 400, 10)
        gold["divergence"][preset] = {"status": st, "event": ev, "iterations": it,
                                      "series": np.nan_to_num(series, nan=-1.0).tolist()}
    # 4. codec table on a fixed sample (precision.hpp:78-140)
    L = po.ref_lib()
    rng = np.random.default_rng(0x5EED)
    xs = np.ldexp(rng.uniform(-2, 2, 4000), rng.integers(-26, 17, 4000)).tolist()
    xs += [1.0, 65520.0, -65520.0, 65519.999, 0.1, 0.0, 2.0**-25, 2.0**-25 * 1.0000001,
           1.0 + 2.0**-11 + 2.0**-40]
    gold["codec"] = {"x": xs, "h": [int(L.ref_encode_b16(x)) for x in xs]}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(gold, f)
    np.savez_compressed(os.path.join(OUT, "golden_n8.npz"), **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
