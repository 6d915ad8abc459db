"""Per-step launch-gap probe on the N=1 C2 step: back-to-back fused steps
(a) bare, (b) with the RankWorker's 4 timing events per step, (c) captured
in a CUDA graph.  Prints ms/step for each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.kernels import field_desc  # noqa: E402


def main(n=100, arith="fast"):
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith=arith)
    g = tl.LatticeGeometry(1920, 2048, 3, 3, 37)
    A, B = tl.allocate_field(g, vs)
    macro = tl.init.rayleigh_taylor_macro(1920, 2048, vs)
    A.pops[:, g.phys_x, g.phys_y] = tl.equilibrium(*[torch.as_tensor(m).cuda() for m in macro], vs)
    lib = _lib.load()
    st = _lib.Status(A.device)
    tp = _lib.params(p)
    fa, fb = field_desc(A), field_desc(B)
    s = torch.cuda.Stream()

    def step(i, sp):
        src, dst = (fa, fb) if i % 2 == 0 else (fb, fa)
        _lib.check(lib.tlb_step_self(src, dst, tp, 1, 0, 1, st.ptr, sp), "step")

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    with torch.cuda.stream(s):
        for i in range(6):
            step(i, s.cuda_stream)
    bare = timed(lambda: [step(i, s.cuda_stream) for i in range(n)])

    def with_events():
        for i in range(n):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(s)
            ev[1].record(s)
            step(i, s.cuda_stream)
            ev[2].record(s)
            ev[3].record(s)
    evs = timed(with_events)

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for i in range(n):
            step(i, s.cuda_stream)
    with torch.cuda.stream(s):
        graph.replay()
    torch.cuda.synchronize()

    def replay():
        with torch.cuda.stream(s):
            graph.replay()
    gr = timed(replay)
    print(f"{arith}: bare {bare:.5f} ms/step, with 4 events {evs:.5f}, cuda graph {gr:.5f}",
          flush=True)


if __name__ == "__main__":
    main(arith="fast")
    main(arith="exact")
