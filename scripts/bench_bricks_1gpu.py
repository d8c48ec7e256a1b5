"""Cost of the brick decomposition on ONE B200 (the multi-GPU path without the
NVLink hops): the C3 system (4,194,304 particles) as 1 domain vs 2x1x1, 2x2x1
and 2x2x2 bricks of the in-process group transport (every brick on GPU 0,
own stream each; ghost update overlapped with interior forces).  Wall clock
around K group steps with a device sync (supporting measurement, not a bench
line).  Usage: python scripts/bench_bricks_1gpu.py [steps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200 import domain as D  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
L = bench.c3_box()
state = bench.synth_state(bench.N_C3, L)
box = dpd.SimBox((0.0, 0.0, 0.0), (L, L, L))
for dims in [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]:
    nb = dims[0] * dims[1] * dims[2]
    if nb == 1:
        e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=bench.N_C3)
    else:
        e = D.BrickGroup(box, dpd.PairParams(), dpd.RunConfig(), dims,
                         capacity=int(bench.N_C3 / nb * 1.3))
    e.upload(dpd.ParticleStore.from_arrays(*state))
    e.setup()
    e.step(20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.step(K)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    extra = {}
    if nb > 1:
        gh = sum(e.ghost_counts())
        split = [b.block_split() for b in e.bricks]
        extra = dict(ghosts=gh, ghost_frac=round(gh / bench.N_C3, 4),
                     interior_blocks=round(sum(i for _, i in split) / sum(n for n, _ in split), 3))
    print(json.dumps(dict(dims=dims, bricks=nb, steps=K, ms_per_step=round(1e3 * dt / K, 4),
                          m_particle_steps_per_s=round(bench.N_C3 * K / dt / 1e6, 1), **extra)),
          flush=True)
    e.close()

# weak-scaling proxy: nb bricks of 4,194,304 particles each (the bench's
# per-GPU size), all on this one GPU -> nb * t(1 brick) / t(nb bricks) is the
# per-brick work efficiency of the decomposition (ghost pairs, halo kernels,
# rebuild exchange), everything but the NVLink transfer time
t1 = None
for dims in [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]:
    nb = dims[0] * dims[1] * dims[2]
    bigbox = dpd.SimBox((0.0, 0.0, 0.0), tuple(L * d for d in dims))

    import numpy as np
    parts = []
    for q in range(nb):
        c = D.coords_of(q, dims)
        s_ = bench.synth_state(bench.N_C3, L, seed=2024 + q)
        for k in range(3):
            s_[k] = s_[k] + c[k] * L
        s_[6] = s_[6] + np.uint32(q * bench.N_C3)
        parts.append(s_)
    allst = [np.concatenate([p[k] for p in parts]) for k in range(7)]
    if nb == 1:
        e = dpd.Engine(bigbox, dpd.PairParams(), dpd.RunConfig(), capacity=bench.N_C3)
    else:
        e = D.BrickGroup(bigbox, dpd.PairParams(), dpd.RunConfig(), dims, capacity=int(bench.N_C3 * 1.2))
    e.upload(dpd.ParticleStore.from_arrays(*allst))
    e.setup()
    e.step(20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.step(K)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    t1 = dt if nb == 1 else t1
    print(json.dumps(dict(weak=True, dims=dims, bricks=nb, particles=bench.N_C3 * nb,
                          ms_per_step=round(1e3 * dt, 4),
                          per_brick_efficiency=round(nb * t1 / dt, 3))), flush=True)
    e.close()
