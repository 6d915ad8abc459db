"""Minimal launch sequence for an ncu capture of the NVLink peer-store step
kernel (k_peer_step): ONE process drives two 1920x2048 tiles on GPUs 0 and
1 (configs[2] at N=2, exchange="p2p", linked in-process with
tlb_peer_create_local), a few steps in lock step.  Under ncu's serialised
kernel replay this cannot deadlock: a border block of step s waits only for
the neighbour's step s-1, launched before it.

    ncu --replay-mode application --metrics gpu__time_duration.sum,nvltx__bytes.sum,... \
        -k regex:"k_peer_step|k_tb2" -c 8 -o X python tools/peer_ncu.py fast on
(kernel replay of one rank's launch while the other GPU's waits on it
hangs; application replay re-runs the deterministic program per pass)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
    temporal = sys.argv[2] if len(sys.argv) > 2 else "off"    # "on": tlb_peer_step2
    # "0": both ranks on GPU 0 (kernel replay works: a rank's launch waits
    # only on the other rank's previous launch, already done when serialised)
    devices = tuple(int(d) for d in (sys.argv[3] if len(sys.argv) > 3 else "0,1").split(","))
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith=arith)
    res = tl.run(tl.SimConfig(Lx=3840, Ly=2048, Np=2, steps=4, params=p,
                              init="rayleigh-taylor", devices=devices, exchange="p2p",
                              output="device", recv_timeout=60.0, temporal=temporal))
    print("peer_ncu done", res.mlups, flush=True)


if __name__ == "__main__":
    main()
