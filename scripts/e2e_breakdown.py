"""Wall-clock breakdown of bench.py's e2e leg (C3, pinned host buffers):
upload / setup / step_thermo(K) / download, three repetitions.

    python scripts/e2e_breakdown.py [K]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1311_0402_b200 as dpd  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L = bench.c3_box()
state = bench.synth_state(bench.N_C3, L, seed=2024)
box = dpd.SimBox((0.0, 0.0, 0.0), (L, L, L))
e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=bench.N_C3)
pinned = [torch.from_numpy(a).pin_memory().numpy() for a in state]
out = [torch.empty(bench.N_C3, dtype=torch.float64).pin_memory().numpy() for _ in range(6)]
e.upload(dpd.ParticleStore.from_arrays(*pinned))
e.setup()
e.step_thermo(20)
for rep in range(int(os.environ.get("REPS", "3"))):
    t = [time.perf_counter()]
    e.upload(dpd.ParticleStore.from_arrays(*pinned))
    t.append(time.perf_counter())
    e.setup()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    rec = e.step_thermo(K)
    t.append(time.perf_counter())
    e.download_state(out[0:3], out[3:6])
    t.append(time.perf_counter())
    ms = np.diff(t) * 1e3
    tot = (t[-1] - t[0])
    print(f"rep {rep}: upload {ms[0]:.2f} ms, setup {ms[1]:.2f}, step_thermo({K}) {ms[2]:.2f} "
          f"({ms[2] / K:.4f}/step), download {ms[3]:.2f}; e2e {bench.N_C3 * K / tot / 1e6:.1f} M/s")
    ms_dev, _, _ = e.step_timed(K)
    w0 = time.perf_counter()
    e.step(K)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    print(f"   device-timed step {ms_dev / K:.4f} ms; dpdb_step({K}) wall {(w1 - w0) * 1e3:.2f} ms")
