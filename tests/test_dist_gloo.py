"""Multi-process X-face exchange (DistFabric) on CPU with the gloo backend.

The N>1 path exchanges the face-plan payloads of runtime.py:199-224 between
one process per GPU with torch.distributed point-to-point.  Here the same
DistFabric code runs with world_size 2 and 3 over gloo on CPU tensors: every
rank packs its edge columns (numpy restatement of pack_x), exchanges, unpacks
into its halo, and the halo must equal the periodic wrap of the global
lattice -- the ring protocol of runtime.py:269-284, including Np=2 where left
and right are the same peer.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

Q, H = 37, 3


def _c():
    from paper_1703_00185_b200.velocity_set import d2q37_vectors
    return d2q37_vectors()


def plan(c, sign):
    return [np.nonzero(sign * c[:, 0] >= d)[0] for d in range(1, H + 1)]


def pack_x(pops, c, sign, Lx):
    out = []
    for d, ls in enumerate(plan(c, sign), start=1):
        col = H + Lx - d if sign == 1 else H + d - 1
        out.append(pops[ls, col, :].reshape(-1))
    return np.concatenate(out)


def unpack_x(pops, c, sign, payload, Lx):
    off = 0
    NY = pops.shape[2]
    for d, ls in enumerate(plan(c, sign), start=1):
        col = H - d if sign == 1 else H + Lx - 1 + d
        n = len(ls) * NY
        pops[ls, col, :] = payload[off:off + n].reshape(len(ls), NY)
        off += n


class _W:
    """The slice of RankWorker that DistFabric touches."""

    def __init__(self, tile, n):
        self.tile = tile
        self.rbuf_plus = torch.zeros(n, dtype=torch.float64)
        self.rbuf_minus = torch.zeros(n, dtype=torch.float64)


def _worker(rank, world, port, Lx_tile, Ly, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1703_00185_b200.runtime import DistFabric, decompose
        c = _c()
        Lx = Lx_tile * world
        NY = Ly + 2 * H
        rng = np.random.default_rng(0)
        glob = rng.random((Q, Lx, NY))          # same global lattice on every rank
        tiles = decompose(Lx, Ly, world, "1d")
        t = tiles[rank]
        pops = np.zeros((Q, Lx_tile + 2 * H, NY))
        pops[:, H:H + Lx_tile, :] = glob[:, t.x0:t.x0 + Lx_tile, :]
        out_p = torch.from_numpy(pack_x(pops, c, 1, Lx_tile))
        out_m = torch.from_numpy(pack_x(pops, c, -1, Lx_tile))
        w = _W(t, out_p.numel())
        fab = DistFabric()
        assert not fab.native and fab.rank == rank and fab.Np == world
        for step in range(3):                   # repeated steps reuse the buffers
            h = fab.start_x(w, step, out_p, out_m)
            fab.finish_x(w, h, w.rbuf_plus, w.rbuf_minus)
        unpack_x(pops, c, 1, w.rbuf_plus.numpy(), Lx_tile)
        unpack_x(pops, c, -1, w.rbuf_minus.numpy(), Lx_tile)
        ok = True
        for sign in (1, -1):
            for d, ls in enumerate(plan(c, sign), start=1):
                col = H - d if sign == 1 else H + Lx_tile - 1 + d
                gx = (t.x0 + col - H) % Lx
                ok &= np.array_equal(pops[ls, col, :], glob[ls, gx, :])
        q.put((rank, bool(ok), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # report to the parent
        q.put((rank, False, repr(exc)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_distfabric_ring_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 8, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in results:
        assert ok, (rank, err)
