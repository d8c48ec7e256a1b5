"""Long statistical acceptance runs behind the SPEC invariants:
10-replica steady double-Poiseuille viscosity (paper 2.089 +- 0.009; SPEC
2.089 +- 0.03 over 10 replicas), quiescent thermostat over 1e5 steps (kT within
2%), self-assembly over the SPEC's 2e5 steps (largest hydrophobic cluster).
Usage: python scripts/validation_long.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1311_0402_b200 as dpd  # noqa: E402
import test_gpu_observables as T  # noqa: E402
from paper_1311_0402_b200.observables import estimate_viscosity, velocity_profile  # noqa: E402
from paper_1311_0402_b200.scenario import largest_cluster, parse_config  # noqa: E402

t0 = time.time()
mus = []
for seed in range(11, 21):
    e = T.poiseuille_engine((12.0, 32.0, 8.0), 6.0, 0.0, 4.5, 0.5, 0.001, 0.055, seed)
    e.step(60000)
    e.profile_reset(32, 2, 0)
    for _ in range(600):
        e.step(100)
        e.profile_sample()
    p = velocity_profile(*e.profile(), 0.0, 8.0, fold=True)
    mus.append(estimate_viscosity(p.centers - 4.0, -p.mean_v, 0.055, 6.0, 4.0)[0])
    e.close()
mus = np.array(mus)
print(f"viscosity, 10 replicas (12x32x8, paper 4.2 parameters): mean {mus.mean():.4f} +- "
      f"{mus.std(ddof=1) / np.sqrt(len(mus)):.4f} (sd {mus.std(ddof=1):.4f}); "
      f"values {np.round(mus, 3).tolist()}  [{time.time() - t0:.0f}s]", flush=True)

# quiescent thermostat: kT = 1, 1e5 steps, C1 parameters on a 16^3 box
box = dpd.SimBox((0.0, 0.0, 0.0), (16.0, 16.0, 16.0))
e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=12288)
e.init_random(12288, 1.0, 3)
e.setup()
kts = []
for _ in range(100):
    rec = e.step_thermo(1000)
    kts.append(rec["kbt"].mean())
kts = np.array(kts)
print(f"thermostat, 1e5 steps at kT = 1 (12,288 particles): mean kT {kts[10:].mean():.4f}, "
      f"block means in [{kts[10:].min():.4f}, {kts[10:].max():.4f}] (SPEC: within 2%)  "
      f"[{time.time() - t0:.0f}s]", flush=True)
e.close()

s = parse_config(os.path.join(ROOT, "configs", "self_assembly.cfg"))
e = s.engine()
e.setup()
nb = s.n_chains * 8
done = 0
for target in (0, 20000, 50000, 100000, 200000):
    e.step(target - done)
    done = target
    st = e.download()
    mol = np.where(st.tag <= nb, (st.tag - 1) // 8 + 1, 0)
    beads, chains = largest_cluster(st.coord, st.species, mol, s.box, [s.species.index("B")])
    print(f"self-assembly step {target}: largest B cluster {chains} of {s.n_chains} chains "
          f"({beads} beads), kT {e.thermo()['kbt']:.3f}  [{time.time() - t0:.0f}s]", flush=True)
