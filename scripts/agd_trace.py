"""Print an AGD trace on BASELINE configs[1] (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.matching import CONFIGS, generate
from paper_2603_04621_b200 import MatchingProblem
inst = generate(CONFIGS["1M_x_10k"], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
for cfg in (dict(gamma0=0.16, gamma_min=0.01), dict(gamma0=0.01)):
    gp.agd_init(halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5, history_cap=6000, **cfg)
    gp.solve(6000); gp.sync()
    h = gp.history()
    print(cfg)
    for t in (0, 50, 100, 200, 500, 800, 1000, 1200, 1400, 1600, 2000, 2500, 3000, 4000, 5000, 5999):
        print(f"  t={t:5d} g={h['g'][t]:.8e} eta={h['eta'][t]:.2e} gnorm={h['gnorm'][t]:.3e} infeas={h['infeas'][t]:.3e} nnzx={h['nnz_x'][t]:.0f}")
    best = np.maximum.accumulate(h["g"])
    print("  best", best[-1], "argmax", int(np.argmax(h["g"])))
