"""Step-1 forces of single/group engines with and without a rebuild (kbT = 0)."""
import sys

import numpy as np

sys.path[:0] = [".", "tests"]
import dpdsys as _sys  # noqa: E402
import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200 import domain as D  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (2, 1, 1)
box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=11)
p = dpd.PairParams.make(1, 25.0, 4.5, 0.0, 1.0, 1.0, 0.01)
res = {}
for R in (1, 3):
    run = dpd.RunConfig(rebuild_every=R)
    e = _sys.engine(box, st, params=p, run=run)
    e.setup()
    e.step(1)
    a = e.download()
    o = np.argsort(a.tag)
    res[f"single R{R}"] = (np.stack([f[o] for f in a.force], 1), np.stack([x[o] for x in a.coord], 1))
    g = D.BrickGroup(box, p, run, dims, capacity=len(st[0]))
    g.upload(dpd.ParticleStore.from_arrays(*st))
    g.setup()
    g.step(1)
    b = g.download()
    res[f"group R{R}"] = (np.stack(b.force, 1), np.stack(b.coord, 1))
keys = list(res)
for i in range(len(keys)):
    for j in range(i + 1, len(keys)):
        Fa, Xa = res[keys[i]]
        Fb, Xb = res[keys[j]]
        rel = np.linalg.norm(Fa - Fb) / np.linalg.norm(Fa)
        nbad = int((np.abs(Fa - Fb).max(1) > 1e-3).sum())
        print(f"{keys[i]:>10} vs {keys[j]:>10}: F rel {rel:.3e} bad {nbad} dx {np.abs(Xa - Xb).max():.3e}")
# where are the bad particles of group R3 vs single R3
Fa, Xa = res["single R3"]
Fb, Xb = res["group R3"]
bad = np.abs(Fa - Fb).max(1) > 1e-3
print("bad x-coords:", np.round(np.sort(Xa[bad, 0]), 2)[:60])
