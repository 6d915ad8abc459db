import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1703_00185_b200 as tl
vs = tl.build_velocity_set("D2Q37")
for arith in ("exact", "fast"):
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9*vs.cs2, Twall_bot=1.1*vs.cs2, arith=arith)
    for L in [(256,128),(512,256)]:
        cfg = tl.SimConfig(Lx=L[0], Ly=L[1], steps=2048, params=p, init="rayleigh-taylor", output="device")
        tl.run(tl.SimConfig(Lx=L[0], Ly=L[1], steps=64, params=p, init="rayleigh-taylor", output="device"))
        r = tl.run(cfg)
        tb = np.array([m["t_bulk"] for m in r.metrics])
        print(arith, L, "wall us/step", round(r.wall_seconds/2048*1e6,2), "device us/step (graph avg)", round(np.nanmedian(tb)*1e6,2))
