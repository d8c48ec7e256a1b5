import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_1311_0402_b200 as dpd

L = (8.0, 8.0, 8.0)
obox = O.make_box((0, 0, 0), L)
n = 1536
st = O.init_fluid(obox, n, 1.0, 7)
box = dpd.SimBox((0.0, 0.0, 0.0), L)
def mk():
    e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=n)
    e.upload(dpd.ParticleStore.from_arrays(*st))
    return e
a = mk(); a.setup()
b = mk(); b.reorder_particles(); b.build_neighbor_table(); b.compute_forces(0)
sim = O.Sim(obox, O.make_params(), st, nthreads=4)
for step in range(1, 13):
    a.step(1)
    b.verlet_phase1()
    if step % 10 == 0:
        b.reorder_particles(); b.build_neighbor_table()
    b.compute_forces(step)
    b.verlet_phase2()
    sim.run(1)
    sa, sb = a.download(), b.download()
    r = sim.state()
    oa, ob, orr = np.argsort(sa.tag), np.argsort(sb.tag), np.argsort(r["tag"])
    dxa = np.abs(sa.coord[0][oa] - r["x"][orr]).max()
    dxb = np.abs(sb.coord[0][ob] - r["x"][orr]).max()
    dva = np.abs(sa.veloc[0][oa] - r["vx"][orr]).max()
    dvb = np.abs(sb.veloc[0][ob] - r["vx"][orr]).max()
    dfa = np.abs(sa.force[0][oa] - r["fx"][orr]).max()
    dfb = np.abs(sb.force[0][ob] - r["fx"][orr]).max()
    print(step, "T", round(a.thermo()["kbt"], 4), round(b.thermo()["kbt"], 4), round(sim.temperature(), 4),
          "dx %.2e %.2e dv %.2e %.2e df %.2e %.2e" % (dxa, dxb, dva, dvb, dfa, dfb))
