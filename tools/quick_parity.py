"""Developer check: fused / staged paths vs the reference on a few presets."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import paper_2505_20911_b200 as m
import pyoracle as po
from test_gpu_parity import b200_solver, checker, assert_state

presets = sys.argv[1].split(",") if len(sys.argv) > 1 else ["DP", "SPDP", "HPSP"]
for preset in presets:
    for strategy in ("storesome", "default"):
        for n, steps in ((20, 2), (64, 2)):
            s = b200_solver(m, n, preset, strategy=strategy, path="fused")
            c = checker(n, preset=preset, strategy=strategy)
            s.init_tgv(); c.init()
            s.advance(m.StepConfig(0.002, steps, 0)); c.advance(0.002, steps, 0)
            assert_state(s, c, (0, 1, 2), f"{preset} {strategy} n{n}")
            print("ok", preset, strategy, n, flush=True)
