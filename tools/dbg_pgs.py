import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests")); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
import paper_2306_06946_b200 as cn
from test_gpu_pgs_pipe import _problem
for (G, mu) in [(140, 0.0), (140, 0.4), (300, 0.0), (104, 0.0), (130, 0.0)]:
    W, d = _problem(G, G)
    for sw in [1, 2, 3]:
        os.environ["CNB_PGS_GRID"] = "1"
        r1 = cn.pgs(W, d, 0.01, cn.PgsConfig(sw, 1e-300, mu)); l1 = r1.lam.cpu().numpy()
        os.environ["CNB_PGS_GRID"] = "0"
        r0 = cn.pgs(W, d, 0.01, cn.PgsConfig(sw, 1e-300, mu)); l0 = r0.lam.cpu().numpy()
        bad = np.nonzero(np.abs(l1 - l0) > 1e-9 * np.abs(l0).max())[0]
        print(G, mu, sw, "maxrel", float(np.abs(l1 - l0).max() / np.abs(l0).max()), "first bad group", (bad[0] // 3) if len(bad) else None, flush=True)
