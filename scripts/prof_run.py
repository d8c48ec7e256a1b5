"""Short C3 run for ncu captures: setup + N steps (one rebuild per 10)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1311_0402_b200 as dpd  # noqa: E402

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
L = bench.c3_box()
state = bench.synth_state(bench.N_C3, L)
e = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), (L, L, L)), dpd.PairParams(), dpd.RunConfig(),
               capacity=bench.N_C3)
e.upload(dpd.ParticleStore.from_arrays(*state))
e.setup()
e.step(nsteps)
print("done", e.thermo())
