"""bench.py's N > 1 exchange (the data-parallel layer step): the packed
lower-triangle factor all-reduce and the digit-form inverse broadcasts, run
for real over gloo at world size 2 on CPU tensors."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2211_14133_b200.engine import _tril_index
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(rank)
        dims = (8, 24, 16)
        factors = [torch.randn((d, d), generator=g) for d in dims]
        upper_before = [torch.triu(f, 1).clone() for f in factors]
        tril = [_tril_index(d, "cpu") for d in dims]
        bench.sync_factors(torch, dist, factors, tril)
        digits = [torch.full((5 + i,), float(10 * rank + i)).to(torch.uint8) for i in range(len(dims))]
        bench.share_inverses(dist, digits, world)
        # numpy copies travel by value: tensors would go through shared-memory
        # fds that vanish if this process exits before the parent unpickles
        # them (an intermittent ConnectionResetError)
        q.put((rank, [f.numpy().copy() for f in factors], [u.numpy().copy() for u in upper_before],
               [d.numpy().copy() for d in digits]))
    finally:
        dist.destroy_process_group()


def test_packed_factor_allreduce_and_digit_broadcast():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, f, up, dg = q.get(timeout=120)
        res[r] = tuple([torch.from_numpy(a) for a in lst] for lst in (f, up, dg))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dims = (8, 24, 16)
    for k, d in enumerate(dims):
        # lower triangle = replica average, identical on both ranks; upper untouched
        lows = [torch.tril(res[r][0][k]) for r in range(world)]
        assert torch.equal(lows[0], lows[1])
        for r in range(world):
            assert torch.equal(torch.triu(res[r][0][k], 1), res[r][1][k])
        orig = []
        for r in range(world):
            g = torch.Generator().manual_seed(r)
            fs = [torch.randn((dd, dd), generator=g) for dd in dims]
            orig.append(torch.tril(fs[k]))
        assert torch.allclose(lows[0], (orig[0] + orig[1]) / 2)
    # digit forms: factor i from rank i % world on every rank
    for r in range(world):
        for i, dg in enumerate(res[r][2]):
            assert torch.all(dg == (10 * (i % world) + i))
