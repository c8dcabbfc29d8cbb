"""Virtual devices: a D x W pipeline on ONE GPU, for running the multi-device
programs of runtime.py with the product backend (engine.CudaBackend) where a
single B200 is all there is.

Each virtual rank is a host thread with its own CUDA streams (torch's
current stream is per thread) running the unchanged PipeFisherTrainer /
Executor / CudaBackend code.  ``VirtualDist`` stands in for the subset of
torch.distributed they use, in process and on the device:

* P2P (isend / irecv): a FIFO per (src, dst, group) channel carrying
  (tensor, event recorded on the sender's stream); the receiver's stream
  waits on the event and copies -- the stream-ordered semantics of an NCCL
  send/recv pair.
* Collectives (all_reduce AVG / SUM / MAX, broadcast): members rendezvous on
  (group, call index) -- every member issues a group's collectives in one
  order (runtime.check_collective_order) -- and the last one to arrive
  enqueues the reduction on its stream after every member's event, in rank
  order (deterministic), writes the result into every member's tensor and
  hands back an event the others' streams wait on.

Timing between virtual devices is not a multi-GPU measurement (they share
one GPU's SMs); what this checks is that the multi-device programs --
stage-to-stage P2P, SyncCurvature, inverse broadcast, SyncGrad, K-FAC items
in the bubbles -- execute with the real kernels and produce the right
numbers (tests/test_vdev_gpu.py).
"""
from __future__ import annotations

import collections
import threading
from typing import Dict, List, Optional, Sequence, Tuple

import torch


class _ReduceOp:
    SUM, AVG, MAX = "sum", "avg", "max"


class _Work:
    def __init__(self, fn=None):
        self._fn = fn

    def wait(self):
        if self._fn is not None:
            fn, self._fn = self._fn, None
            fn()
        return True


class _Group:
    def __init__(self, ranks: Tuple[int, ...]):
        self.ranks = ranks


class VirtualWorld:
    """Shared state of one virtual cluster of `size` ranks on `device`."""

    def __init__(self, size: int, device=None, timeout: float = 600.0):
        self.size = size
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.timeout = timeout
        self._lock = threading.Condition()
        self._chan: Dict[Tuple, collections.deque] = collections.defaultdict(collections.deque)
        self._rdv: Dict[Tuple, dict] = {}
        self._groups: Dict[Tuple[int, ...], _Group] = {}
        self.world_group = self.group_of(tuple(range(size)))
        self.collectives: List[dict] = []  # log: (kind, group, members' inputs/outputs) when `log` is set
        self.log = False
        self.failed: Optional[BaseException] = None
        # torch's CPU generator is process-global: ranks building their (seeded)
        # stages must take turns, or the seeds of different threads interleave
        self.init_lock = threading.Lock()

    def group_of(self, ranks: Tuple[int, ...]) -> _Group:
        with self._lock:
            if ranks not in self._groups:
                self._groups[ranks] = _Group(ranks)
            return self._groups[ranks]

    def dist(self, rank: int) -> "VirtualDist":
        return VirtualDist(self, rank)

    def _wait(self, pred):
        # called with the lock held
        if not self._lock.wait_for(lambda: pred() or self.failed is not None, timeout=self.timeout):
            raise TimeoutError("virtual world: a rank never arrived (deadlocked program?)")
        if self.failed is not None:
            raise RuntimeError("virtual world: another rank failed") from self.failed

    def fail(self, e: BaseException):
        with self._lock:
            self.failed = e
            self._lock.notify_all()


class VirtualDist:
    """The torch.distributed calls of runtime.Comm and engine.CudaBackend, for
    one virtual rank."""

    ReduceOp = _ReduceOp

    def __init__(self, world: VirtualWorld, rank: int):
        self.w, self.rank = world, rank
        self._calls: Dict[Tuple[int, ...], int] = collections.defaultdict(int)

    @property
    def init_lock(self):
        """Hold while constructing seeded modules (PipeFisherTrainer)."""
        return self.w.init_lock

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.w.size

    def new_group(self, ranks: Sequence[int]):
        return self.w.group_of(tuple(sorted(ranks)))

    # ---------------------------------------------------------------- P2P
    def isend(self, tensor: torch.Tensor, dst: int, group=None):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        key = (self.rank, dst, (group or self.w.world_group).ranks)
        with self.w._lock:
            self.w._chan[key].append((tensor, ev))
            self.w._lock.notify_all()
        return _Work()

    def irecv(self, buf: torch.Tensor, src: int, group=None):
        key = (src, self.rank, (group or self.w.world_group).ranks)

        def done():
            with self.w._lock:
                self.w._wait(lambda: len(self.w._chan[key]) > 0)
                t, ev = self.w._chan[key].popleft()
            s = torch.cuda.current_stream()
            s.wait_event(ev)
            buf.copy_(t)
            t.record_stream(s)

        return _Work(done)

    # ---------------------------------------------------------------- collectives
    def _collective(self, kind: str, tensor: torch.Tensor, group, op=None, src=None):
        g = group or self.w.world_group
        if self.rank not in g.ranks:
            raise ValueError("rank not in group")
        n = self._calls[g.ranks]
        self._calls[g.ranks] += 1
        key = (g.ranks, n)
        ev_in = torch.cuda.Event()
        ev_in.record(torch.cuda.current_stream())
        with self.w._lock:
            r = self.w._rdv.setdefault(key, {"in": {}, "done": None, "left": len(g.ranks)})
            r["in"][self.rank] = (tensor, ev_in, kind, op, src)
            if len(r["in"]) == len(g.ranks):
                r["done"] = self._reduce(g.ranks, r["in"])
                self.w._lock.notify_all()
            else:
                self.w._wait(lambda: r["done"] is not None)
            ev_out = r["done"]
            r["left"] -= 1
            if r["left"] == 0:
                del self.w._rdv[key]
        torch.cuda.current_stream().wait_event(ev_out)
        return _Work()

    def _reduce(self, ranks, inputs) -> torch.cuda.Event:
        kinds = {v[2] for v in inputs.values()}
        if len(kinds) != 1:
            raise RuntimeError(f"collective mismatch in group {ranks}: {kinds}")
        kind = kinds.pop()
        s = torch.cuda.current_stream()
        for t, ev, *_ in inputs.values():
            s.wait_event(ev)
        ts = [inputs[r][0] for r in ranks]
        before = [t.clone() for t in ts] if self.w.log else None
        if kind == "all_reduce":
            op = inputs[ranks[0]][3]
            acc = ts[0].clone()
            for t in ts[1:]:  # rank order: deterministic
                if op == _ReduceOp.MAX:
                    torch.maximum(acc, t, out=acc)
                else:
                    acc.add_(t)
            if op == _ReduceOp.AVG:
                acc.div_(len(ts))
            for t in ts:
                t.copy_(acc)
        elif kind == "broadcast":
            src = inputs[ranks[0]][4]
            for r, t in zip(ranks, ts):
                if r != src:
                    t.copy_(inputs[src][0])
        else:  # pragma: no cover
            raise ValueError(kind)
        if self.w.log:
            self.w.collectives.append({"kind": kind, "ranks": ranks, "before": before,
                                       "after": [t.clone() for t in ts]})
        ev = torch.cuda.Event()
        ev.record(s)
        return ev

    def all_reduce(self, tensor, op=_ReduceOp.SUM, group=None, async_op=False):
        return self._collective("all_reduce", tensor, group, op=op)

    def broadcast(self, tensor, src, group=None, async_op=False):
        return self._collective("broadcast", tensor, group, src=src)

    def barrier(self, group=None):
        t = torch.zeros(1, device=self.w.device)
        return self._collective("all_reduce", t, group, op=_ReduceOp.SUM)


def run_virtual(size: int, body, device=None, timeout: float = 600.0, log: bool = False):
    """Run body(rank, dist) on `size` threads, one virtual rank each; returns
    the per-rank results (re-raises the first failure)."""
    world = VirtualWorld(size, device, timeout)
    world.log = log
    out: List = [None] * size
    errs: List[Optional[BaseException]] = [None] * size

    def worker(rank):
        try:
            torch.cuda.set_device(world.device)
            out[rank] = body(rank, world.dist(rank))
        except BaseException as e:  # noqa: BLE001
            errs[rank] = e
            world.fail(e)

    threads = [threading.Thread(target=worker, args=(r,), name=f"vdev{r}") for r in range(size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = next((e for e in errs if e is not None and not isinstance(e, RuntimeError)), None) or \
        next((e for e in errs if e is not None), None)
    if first is not None:
        raise first
    return out, world
