"""C4 vesicle chemistry at scale on one GPU (BASELINE.json configs[3]:
amphiphilic BBBAABBB chains, 10% of the particles, in solvent at rho = 5;
P:362-374; the harmonic bonds K = 80, r0 = 0.38 and the repulsion matrix of
configs/self_assembly.cfg).  Every `every` steps: the largest B-bead cluster
(union-find at r_c) and its shape (observables.aggregate_shape:
vesicle / micelle / bilayer / irregular), kT, throughput.

  python scripts/vesicle_run.py N STEPS EVERY OUT
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200.observables import aggregate_shape  # noqa: E402
from paper_1311_0402_b200.scenario import cluster_members  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2**24
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", "vesicle_run.txt")
S, A, B = 0, 1, 2
rho = 5.0
L = (n / rho) ** (1.0 / 3.0)
box = dpd.SimBox((0.0, 0.0, 0.0), (L, L, L))
a = np.full((3, 3), 15.0)
a[A, B] = a[B, A] = a[B, S] = a[S, B] = 120.0
p = dpd.PairParams.make(3, a.ravel(), 4.5, 1.0, 1.0, 1.0, 0.01)
nch = int(0.1 * n) // 8
e = dpd.Engine(box, p, dpd.RunConfig(), capacity=n)
e.init_random(n, 1.0, 5, nch, [B, B, B, A, A, B, B, B], S, 0.38, 80.0)
e.setup()
nb = nch * 8
log = open(out, "w")


def report(step, wall):
    st = e.download()
    mol = np.where(st.tag <= nb, (st.tag - 1) // 8 + 1, 0)
    beads, chains, idx = cluster_members(st.coord, st.species, mol, box, [B], 1.0)
    X = np.stack([st.coord[k][idx] for k in range(3)], 1)
    shp = aggregate_shape(X, box)
    line = (f"step {step}: largest B cluster {chains} of {nch} chains ({beads} beads), shape {shp.kind} "
            f"(Rg {shp.radius_of_gyration:.2f}, asphericity {shp.asphericity:.3f}, hollowness "
            f"{shp.hollowness:.2f}, closure {shp.closure:.2f}), kT {e.thermo()['kbt']:.4f}, "
            f"{wall:.1f} s")
    print(line, flush=True)
    log.write(line + "\n")
    log.flush()


t0 = time.time()
report(0, 0.0)
done = 0
while done < steps:
    k = min(every, steps - done)
    ms, _, _ = e.step_timed(k)
    done += k
    rate = n * k / (ms * 1e-3) / 1e6
    log.write(f"  steps {done - k + 1}-{done}: {ms / k:.3f} ms/step, {rate:.1f} M particle-steps/s\n")
    report(done, time.time() - t0)
log.close()
