"""BASELINE config C2 on one B200: reverse (double) Poiseuille flow of
1,048,576 particles in the paper's transient box with y x 4 (59.4123 x 29.7062
x 118.825, rho 5, a 15, sigma 3, kT 1, dt 0.01, g 0.055; drive x, profile z),
started from rest; folded profiles vs Eq. 9 with nu from a steady fit of the
same parameters on a 12 x 8 x 8 box.  Prints the deviations and the device
throughput of the run.  Usage: python scripts/validate_c2.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200.observables import (analytic_transient_profile, estimate_viscosity,  # noqa: E402
                                              velocity_profile)

g, rho, kbt, dt = 0.055, 5.0, 1.0, 0.01
p = dpd.PairParams.make(1, 15.0, 4.5, kbt, 1.0, 1.0, dt)
run = dpd.RunConfig(body_force=g, drive_axis=0, partition_axis=2)


def engine(L, seed):
    box = dpd.SimBox((0.0, 0.0, 0.0), L)
    n = int(round(rho * L[0] * L[1] * L[2]))
    e = dpd.Engine(box, p, run, capacity=n)
    e.init_random(n, kbt, seed)
    e.setup()
    return e, n


s, _ = engine((12.0, 8.0, 8.0), 21)
s.step(20000)
s.profile_reset(32, 2, 0)
for _ in range(400):
    s.step(50)
    s.profile_sample()
prof = velocity_profile(*s.profile(), 0.0, 8.0, fold=True)
mu, se, rel = estimate_viscosity(prof.centers - 4.0, -prof.mean_v, g, rho, 4.0)
nu = mu / rho
print(f"steady fit (12x8x8): mu = {mu:.4f} +- {se:.4f}, nu = {nu:.4f}")

L = (59.4123, 29.7062, 118.825)
e, n = engine(L, 22)
print(f"C2: {n} particles")
d = L[2] / 2
t_now, dev_t, steps = 0, 0.0, 0
for T in (100, 200, 500):
    k = int(round((T - 0.5) / dt)) - t_now
    ms = e.step_timed(k)[0]
    dev_t += ms
    steps += k
    e.profile_reset(60, 2, 0)
    for _ in range(100):
        e.step(1)
        e.profile_sample()
    t_now = int(round((T + 0.5) / dt))
    q = velocity_profile(*e.profile(), 0.0, L[2], fold=True)
    ref = analytic_transient_profile(q.centers - 3 * d / 2, float(T), g, d, nu)
    dev = np.linalg.norm(-q.mean_v - ref) / np.linalg.norm(ref)
    mid = len(ref) // 2
    print(f"t = {T}: L2 deviation from Eq. 9 = {100 * dev:.2f}%, centre u = {-q.mean_v[mid]:.4f} "
          f"(Eq. 9 {ref[mid]:.4f})")
print(f"device time {dev_t:.1f} ms for {steps} steps: {n * steps / dev_t / 1e3:.1f} M particle-steps/s")
