import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import paper_2505_20911_b200 as m
from test_gpu_parity import b200_solver, checker
for preset in ["HPSP", "SPDP"]:
    for n in (64, 20):
        for visc in (True, False):
            s = b200_solver(m, n, preset, path="fused", viscous=visc)
            c = checker(n, preset=preset, viscous=visc)
            s.init_tgv(); c.init()
            s.advance(m.StepConfig(0.002, 1, 0)); c.advance(0.002, 1, 0)
            for cls in (2, 1, 0):
                for comp in range(5):
                    g, r = s.get_field(cls, comp), c.field(cls, comp)
                    bad = np.argwhere(g.view(np.uint64) != r.view(np.uint64))
                    if len(bad):
                        odd = np.mean(bad[:, 2] % 2)
                        k, j, i = bad[0]
                        print(f"{preset} n{n} visc{visc} cls{cls} comp{comp}: {len(bad)} bad, frac odd-i {odd:.2f}, first ({i},{j},{k}) rel {abs(g[k,j,i]-r[k,j,i])/abs(r[k,j,i]):.2e}")
            print("done", preset, n, visc, flush=True)
