"""Print the statistical-acceptance numbers behind tests/test_gpu_observables.py
(steady double-Poiseuille viscosity, transient deviation from Eq. 9, ideal-gas
g(r)) for profiles/.  Usage: python scripts/validate_observables.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import test_gpu_observables as T  # noqa: E402
from paper_1311_0402_b200.observables import (analytic_transient_profile, estimate_viscosity,  # noqa: E402
                                              velocity_profile)

g = 0.055
for seed in (7, 8, 9, 10):
    e = T.poiseuille_engine((12.0, 32.0, 8.0), 6.0, 0.0, 4.5, 0.5, 0.001, g, seed)
    e.step(60000)
    e.profile_reset(32, 2, 0)
    for _ in range(600):
        e.step(100)
        e.profile_sample()
    p = velocity_profile(*e.profile(), 0.0, 8.0, fold=True)
    mu, se, rel = estimate_viscosity(p.centers - 4.0, -p.mean_v, g, 6.0, 4.0)
    print(f"steady double Poiseuille (paper 4.2: 2.089 +- 0.009), seed {seed}: mu = {mu:.4f} +- {se:.4f}, "
          f"fit residual {rel:.3f}")
s = T.poiseuille_engine((12.0, 8.0, 8.0), 5.0, 15.0, 3.0, 1.0, 0.01, g, 21)
s.step(20000)
s.profile_reset(32, 2, 0)
for _ in range(400):
    s.step(50)
    s.profile_sample()
p = velocity_profile(*s.profile(), 0.0, 8.0, fold=True)
mu, se, rel = estimate_viscosity(p.centers - 4.0, -p.mean_v, g, 5.0, 4.0)
print(f"transient parameter set (rho 5, a 15, sigma 3): steady mu = {mu:.4f} +- {se:.4f}")
e = T.poiseuille_engine((20.0, 8.0, 40.0), 5.0, 15.0, 3.0, 1.0, 0.01, g, 22)
t_now = 0
for Tt in (100, 200, 500):
    e.step(int(round((Tt - 0.5) / 0.01)) - t_now)
    e.profile_reset(40, 2, 0)
    for _ in range(100):
        e.step(1)
        e.profile_sample()
    t_now = int(round((Tt + 0.5) / 0.01))
    q = velocity_profile(*e.profile(), 0.0, 40.0, fold=True)
    ref = analytic_transient_profile(q.centers - 30.0, float(Tt), g, 20.0, mu / 5.0)
    dev = np.linalg.norm(-q.mean_v - ref) / np.linalg.norm(ref)
    print(f"transient t = {Tt}: L2 deviation from Eq. 9 = {100 * dev:.2f}% (bar 7%), centre u = "
          f"{-q.mean_v[9]:.4f} vs {ref[9]:.4f}")
