"""Step-by-step comparison of a one-brick group with the single-domain engine."""
import sys

import numpy as np

sys.path[:0] = [".", "tests"]
import dpdsys as _sys  # noqa: E402
import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200 import domain as D  # noqa: E402

box, obox, st = _sys.fluid((10, 10, 10), 3.0, seed=5)
run = dpd.RunConfig(rebuild_every=int(sys.argv[4]) if len(sys.argv) > 4 else 4)
dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1, 1, 1)
e = _sys.engine(box, st, run=run)
e.setup()
g = D.BrickGroup(box, dpd.PairParams(), run, dims, capacity=len(st[0]))
g.upload(dpd.ParticleStore.from_arrays(*st))
g.setup()
for s in range(8):
    a, b = e.download(), g.download()
    oa = np.argsort(a.tag)
    dx = max(np.abs(a.coord[k][oa] - b.coord[k]).max() for k in range(3))
    dv = max(np.abs(a.veloc[k][oa] - b.veloc[k]).max() for k in range(3))
    df = max(np.abs(a.force[k][oa] - b.force[k]).max() for k in range(3))
    nf = np.abs(a.force[0]).max()
    xb = b.coord[0]
    interior = (np.abs(xb - 5.0) > 2.0) & (np.minimum(xb, 10 - xb) > 2.0)
    dfi = max(np.abs(a.force[k][oa] - b.force[k])[interior].max() for k in range(3))
    print(f"   interior df {dfi:.3e} ({interior.sum()} particles)")
    print(f"step {s}: n {len(a.tag)} {len(b.tag)} dx {dx:.3e} dv {dv:.3e} df {df:.3e} |f| {nf:.3e}"
          f" ghosts {g.ghost_counts()}", flush=True)
    # ghosts must be exact (shifted) copies of their owners
    idx = {int(t): i for i, t in enumerate(b.tag)}
    for q, br in enumerate(g.bricks):
        gx, gv, gt = br.ghosts()
        at = np.array([idx[int(t)] for t in gt], np.int64)
        bad = 0
        for k in range(3):
            d = gx[k] - b.coord[k][at]
            d = d - np.round(d / 10.0) * 10.0
            bad = max(bad, np.abs(d).max(initial=0))
        dvg = max(np.abs(gv[k] - b.veloc[k][at]).max(initial=0) for k in range(3))
        print(f"   brick {q}: ghosts {len(gt)} pos err {bad:.3e} vel err {dvg:.3e}", flush=True)
    e.step(1)
    g.step(1)
