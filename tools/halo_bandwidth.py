"""NVLink halo-exchange bandwidth vs message size on B200 (paper Fig. 11 /
reference bench.bench_halo_exchange analog), feeding the planner.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/halo_bandwidth.py [--out profiles/r01_halo_bw.csv]

For tile heights Ly the X-face message is 26 x (Ly+6) doubles per direction.
Measured per size (CUDA events, 50 reps, max over ranks):
  x_face_ring : tlb_ring_exchange = pack both faces + grouped NCCL
                send/recv with both ring neighbours + unpack (what a step does)
  nccl_p2p    : raw torch.distributed batched send/recv of the same bytes
Bandwidth = 2 faces x message bytes / time (the planner's B, for two faces
sent per step).  Rank 0 writes the table and the planner's 1-D predictions
for the C2-per-GPU weak-scaling workload at Np = 1, 2, 4, 8.
"""
import argparse
import csv
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib, planner  # noqa: E402
from paper_1703_00185_b200.kernels import field_desc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "halo_bw.csv"))
    ap.add_argument("--beta", type=float, default=None,
                    help="s per site update (default: measured N=1 fast step here)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    vs = tl.build_velocity_set("D2Q37")
    fab = tl.DistFabric()
    lib = _lib.load()
    s = torch.cuda.Stream(dev)
    rows = []
    for Ly in (64, 256, 1024, 2048, 4096, 8192, 16384):
        tiles = tl.decompose(8 * world, Ly, world, "1d")
        w = tl.RankWorker(tiles[rank], vs, tl.PhysicsParams(tau=0.8), fab,
                          schedule="overlapped", device=dev)
        msg = 26 * (Ly + 6) * 8
        fd = field_desc(w.prv)

        def ring():
            _lib.check(lib.tlb_ring_exchange(w._ring, fd, 1, w.sbuf2.data_ptr(),
                                             w.rbuf2.data_ptr(), s.cuda_stream), "exchange")

        sb = torch.ones(2 * msg // 8, dtype=torch.float64, device=dev)
        rb = torch.empty_like(sb)
        left, right = (rank - 1) % world, (rank + 1) % world

        def p2p():
            n = msg // 8
            ops = [dist.P2POp(dist.isend, sb[:n], right), dist.P2POp(dist.irecv, rb[:n], left),
                   dist.P2POp(dist.isend, sb[n:], left), dist.P2POp(dist.irecv, rb[n:], right)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()

        for kind, fn in (("x_face_ring", ring), ("nccl_p2p", p2p)):
            with torch.cuda.stream(s):
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                reps = 50
                for _ in range(reps):
                    fn()
                e1.record(s)
                torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item()) * 1e-3
            rows.append((kind, msg, 2 * msg / sec, sec))
        del w
    if rank == 0:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w", newline="") as fh:
            cw = csv.writer(fh)
            cw.writerow(["kind", "message_bytes", "bandwidth [bytes/s]", "seconds"])
            for r in rows:
                cw.writerow([r[0], r[1], repr(r[2]), repr(r[3])])
        ring_rows = [r for r in rows if r[0] == "x_face_ring"]
        table = planner.BandwidthTable([r[1] for r in ring_rows], [r[2] for r in ring_rows])
        beta = a.beta or 0.3917e-3 / (1920 * 2048)   # r01 N=1 fast step (bench.py)
        preds = {}
        for Np in (1, 2, 4, 8):
            inp = planner.CostModelInput(1920 * Np, 2048, Np, table, table, beta)
            p1, po = planner.predict_1d(inp), planner.predict_1d_overlap(inp)
            preds[Np] = {"1d_ms": p1.T_total * 1e3, "1d_overlap_ms": po.T_total * 1e3,
                         "1d_eff": 1 / p1.scale_violation, "1d_overlap_eff": 1 / po.scale_violation}
        print(json.dumps({"table": rows, "beta_s_per_site": beta, "predictions": preds}))
    dist.barrier()
    fab.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
