"""Device throughput of every BASELINE config that fits one B200 (the bench
line is C3; this is the supporting table for profiles/):
  C1  32^3 fluid, 98,304 particles (the CPU reference's own case)
  C2  reverse Poiseuille, 1,048,576 particles, body force (rho 5, a 15)
  C3  4,194,304 particle fluid, rho 3 (the roofline config)
  C4  vesicle chemistry per GPU: 2,097,152 particles (16M / 8 GPUs), rho 5, 10% BBBAABBB
      chains with harmonic bonds, 3 species, paper repulsion matrix
  C5  weak-scaling brick size: 16,777,216 particles, rho 3
Usage: python scripts/bench_configs.py [steps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1311_0402_b200 as dpd  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100


ONLY = os.environ.get("CONFIGS")  # e.g. CONFIGS=C3,C4


def run(name, L, n, params, run_cfg, chains=None):
    if ONLY and name not in ONLY.split(","):
        return
    box = dpd.SimBox((0.0, 0.0, 0.0), L)
    e = dpd.Engine(box, params, run_cfg, capacity=n)
    if chains:
        e.init_random(n, params.kbt, 5, *chains)
    else:
        e.init_random(n, params.kbt, 5)
    e.setup()
    e.step(20)
    ms, st, ln = e.step_timed(steps, stages=True)
    rate = n * steps / (ms * 1e-3) / 1e6
    out = dict(config=name, particles=n, steps=steps, ms_per_step=round(ms / steps, 5),
               m_particle_steps_per_s=round(rate, 1),
               stage_ms_per_step={k: round(st[i] / steps, 5) for i, k in
                                  enumerate(["integrate", "sort_permute", "build", "force", "other"])})
    print(json.dumps(out), flush=True)
    e.close()


flu = dpd.PairParams()
run("C1", (32.0, 32.0, 32.0), 98304, flu, dpd.RunConfig())
p2 = dpd.PairParams.make(1, 15.0, 4.5, 1.0, 1.0, 1.0, 0.01)
run("C2", (59.4123, 29.7062, 118.825), 1048576, p2,
    dpd.RunConfig(body_force=0.055, drive_axis=0, partition_axis=2))
L3 = (4194304 / 3.0) ** (1 / 3)
run("C3", (L3, L3, L3), 4194304, flu, dpd.RunConfig())
L4 = (2097152 / 5.0) ** (1 / 3)
S, A, B = 0, 1, 2
a = [[15, 15, 120], [15, 15, 120], [120, 120, 15]]  # rows S, A, B: a(A,B) = a(B,S) = 120
p4 = dpd.PairParams.make(3, [a[i][j] for i in range(3) for j in range(3)], 4.5, 1.0, 1.0, 1.0, 0.01)
nch = int(0.1 * 2097152) // 8
run("C4", (L4, L4, L4), 2097152, p4, dpd.RunConfig(), chains=(nch, [B, B, B, A, A, B, B, B], S, 0.38, 80.0))
L5 = (16777216 / 3.0) ** (1 / 3)
run("C5", (L5, L5, L5), 16777216, flu, dpd.RunConfig())
