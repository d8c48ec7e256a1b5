"""Command line of the engine: run / bench / verify / ulp-sweep.

    python -m paper_1311_0402_b200 run configs/poiseuille_steady.cfg --out out/
    python -m paper_1311_0402_b200 bench configs/c3_fluid.cfg --steps 200
    python -m paper_1311_0402_b200 verify
    python -m paper_1311_0402_b200 ulp-sweep gaussian32

Exit code 0 on success, the reference's error category (inc/error.hpp:8-13;
5 = device) on failure.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import time

import numpy as np

from . import DPDError
from . import io as dio
from .domain import BrickGroup
from .engine import ParticleStore
from .observables import velocity_profile
from .scenario import Scenario, parse_config


def _engine(sc: Scenario, domains, device):
    """Single domain, or a brick group (bricks spread over the visible GPUs)."""
    if domains is None or domains == (1, 1, 1):
        return sc.engine(device), False
    import torch
    init = sc.engine(device)  # init_random on the device, then split into bricks
    st = init.download()
    init.close()
    nb = domains[0] * domains[1] * domains[2]
    ng = max(torch.cuda.device_count(), 1)
    g = BrickGroup(sc.box, sc.params, sc.run, domains, capacity=int(sc.n / nb * 2) + 4096,
                   devices=[(device + q) % ng for q in range(nb)])
    mol = None
    if sc.chains:
        mol = np.where(st.tag <= sc.n_chains * len(sc.chains["sequence"]),
                       (st.tag - 1) // len(sc.chains["sequence"]) + 1, 0).astype(np.uint32)
    g.upload(ParticleStore(st.coord, st.veloc, st.tag, st.species, mol))
    return g, True


def cmd_run(a) -> int:
    sc = parse_config(a.config)
    if a.seed is not None:
        sc.seed = sc.run.seed = a.seed
    os.makedirs(a.out, exist_ok=True)
    e, bricks = _engine(sc, a.domains, a.device)
    e.setup()
    thermo = {"step": [], "kbt": [], "momentum": []}
    th0 = e.thermo()
    thermo["step"].append(0)
    thermo["kbt"].append(th0["kbt"])
    thermo["momentum"].append(th0["momentum"])
    prof = sc.profile
    if prof and not bricks:
        e.profile_reset(prof["bins"], prof["axis"], sc.run.drive_axis)
    chunk = prof["every"] if prof else 1000
    done = 0
    t0 = time.perf_counter()
    while done < sc.steps:
        k = min(chunk, sc.steps - done)
        rec = e.step_thermo(k)
        done += k
        for key in thermo:
            thermo[key].extend(list(rec[key]))
        if prof and not bricks and done >= prof["start"]:
            e.profile_sample()
    wall = time.perf_counter() - t0
    rec = {k: np.asarray(v) for k, v in thermo.items()}
    dio.write_thermo_csv(os.path.join(a.out, "thermo.csv"), rec, sc.params.dt, sc.n)
    st = e.download()
    dio.write_xyz(os.path.join(a.out, "final.xyz"), st, names=list(sc.species) + ["X"] * 4,
                  comment=f"step {done}")
    if prof and not bricks:
        ax = prof["axis"]
        p = velocity_profile(*e.profile(), sc.box.lo[ax], sc.box.hi[ax])
        dio.write_profile_csv(os.path.join(a.out, "profile.csv"), p)
    if not bricks:
        dio.save_restart(os.path.join(a.out, "restart.bin"), e)
    print(f"run {a.config}: {sc.n} particles, {done} steps in {wall:.2f} s "
          f"({sc.n * done / max(wall, 1e-9) / 1e6:.1f} M particle-steps/s wall), final kT "
          f"{rec['kbt'][-1]:.4f}; outputs in {a.out}")
    e.close()
    return 0


def cmd_bench(a) -> int:
    sc = parse_config(a.config)
    e = sc.engine(a.device)
    e.setup()
    e.step(min(20, a.steps))
    ms, _, _ = e.step_timed(a.steps)
    print(f"bench {a.config}: {sc.n} particles, {a.steps} steps, {ms / a.steps:.4f} ms/step, "
          f"{sc.n * a.steps / (ms * 1e-3) / 1e6:.1f} M particle-steps/s (device time)")
    e.close()
    return 0


def cmd_verify(a) -> int:
    """The acceptance scenarios as the GPU test suites that
    assert them: thermostat, viscosity, transient Eq. 9, g(r), self-assembly."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = [os.path.join(root, "tests", t) for t in
             ("test_gpu_observables.py", "test_gpu_init.py", "test_gpu_run.py")]
    return subprocess.call([sys.executable, "-m", "pytest", "-q", "-m", "gpu"] + tests, cwd=root)


def cmd_ulp_sweep(a) -> int:
    """CSV (input, output, reference, ulp_error) of a device kernel
    against the bit-exact fp64 path of the same function."""
    from .engine import fastlog, gaussian
    rng = np.random.default_rng(a.seed or 1)
    n = a.samples
    u = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    if a.kernel in ("gaussian32", "gaussian_hot"):
        ref = gaussian(u, v)
        out = gaussian(u, v, fp32=a.kernel == "gaussian32", hot=a.kernel == "gaussian_hot").astype(np.float64)
        inp = [f"{x} {y}" for x, y in zip(u, v)]
    elif a.kernel == "fastlog32":
        u = np.maximum(u, 1)
        ref = fastlog(u)
        out = fastlog(u, fp32=True).astype(np.float64)
        inp = [str(x) for x in u]
    else:
        raise DPDError(1, f"ulp-sweep: unknown kernel {a.kernel} (gaussian32, gaussian_hot, fastlog32)")
    ulp = np.abs(out - ref) / np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    w = sys.stdout
    w.write("input,output,reference,ulp_error\n")
    for i in range(n):
        w.write(f"{inp[i]},{out[i]!r},{ref[i]!r},{ulp[i]:.3f}\n")
    h = np.histogram(ulp, bins=[0, 0.5, 1, 2, 4, 8, 16, np.inf])[0]
    sys.stderr.write(f"ulp histogram [0,.5,1,2,4,8,16,inf): {h.tolist()}, max {ulp.max():.2f}\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1311_0402_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("config")
    r.add_argument("--domains", type=lambda s: tuple(int(x) for x in s.lower().split("x")), default=None)
    r.add_argument("--seed", type=int, default=None)
    r.add_argument("--out", default="out")
    r.add_argument("--device", type=int, default=0)
    b = sub.add_parser("bench")
    b.add_argument("config")
    b.add_argument("--steps", type=int, default=100)
    b.add_argument("--device", type=int, default=0)
    sub.add_parser("verify")
    u = sub.add_parser("ulp-sweep")
    u.add_argument("kernel")
    u.add_argument("--samples", type=int, default=10000)
    u.add_argument("--seed", type=int, default=None)
    a = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "bench": cmd_bench, "verify": cmd_verify, "ulp-sweep": cmd_ulp_sweep}[a.cmd](a)
    except DPDError as ex:
        sys.stderr.write(f"error [{ex.code}]: {ex}\n")
        return ex.code


if __name__ == "__main__":
    sys.exit(main())
