import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1311_0402_b200.scenario import parse_config, largest_cluster
s = parse_config(os.path.join(ROOT, "configs", "self_assembly.cfg"))
e = s.engine()
e.setup()
nb = s.n_chains * 8
t0 = time.time()
done = 0
for target in (10000, 25000, 50000, 100000, 150000, 200000):
    e.step(target - done)
    done = target
    st = e.download()
    mol = np.where(st.tag <= nb, (st.tag - 1) // 8 + 1, 0)
    beads, chains = largest_cluster(st.coord, st.species, mol, s.box, [2])
    print(f"step {target}: {time.time() - t0:.1f}s largest B cluster {beads} beads, {chains} chains of {s.n_chains}; kbt {e.thermo()['kbt']:.3f}", flush=True)
