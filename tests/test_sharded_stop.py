"""The time-budget stop of a row-sharded run is one collective decision
(factorize._ShardedDeviceLoop.stop_vote): with per-rank clocks that disagree,
every rank still leaves the outer loop after the same iteration, so the
all-reduced objective of every emit has all its partners (world size 2, gloo,
CPU).  The loop under test is the product's _run_outer; only the device
arithmetic is replaced by a stub."""
import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Stream:
    def synchronize(self):
        pass


class _TorchShim:
    class cuda:  # noqa: N801
        @staticmethod
        def current_stream():
            return _Stream()


class _SkewedClock:
    """Rank 0's clock runs out after 3 ticks, rank 1's never does."""

    def __init__(self, rank):
        self.rank, self.ticks = rank, 0

    def pause(self):
        pass

    def resume(self):
        pass

    def tick(self):
        self.ticks += 1

    def elapsed(self):
        return 100.0 if (self.rank == 0 and self.ticks >= 3) else 0.001 * self.ticks

    def wall_elapsed(self):
        return self.elapsed()


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(REPO))
    import torch
    import torch.distributed as dist

    from paper_1812_04315_b200 import factorize, sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = sharded.Comm()

    class StubRun(factorize._ShardedDeviceLoop):
        def __init__(self):
            self.comm, self.torch = comm, _TorchShim
            self.n, self.m, self.p = 6, 5, 2
            self.steps = 0

        def norm_x(self):
            t = torch.tensor([1.0])
            self.comm.all_reduce(t)
            return float(t[0])

        def prepare(self, init):
            pass

        def half_steps(self, t, icfg):
            self.steps += 1

        def drain(self):
            pass

        def objective(self):
            t = torch.tensor([0.5 / (1 + self.steps)])
            self.comm.all_reduce(t)
            return float(t[0])

        def host_factors(self):
            return np.ones((6, 2)), np.ones((2, 5))

    run = StubRun()
    init = factorize.FactorPair(G=np.ones((6, 2)), F=np.ones((2, 5)), p=2)
    cfg = factorize.OuterConfig(time_budget_seconds=5.0, max_outer_iterations=10, trace_every=1)
    recs = []
    factorize._run_outer(None, init, cfg, lambda r, G, F: recs.append(r.outer_iter), _SkewedClock(rank), None,
                         "fp64", run=run)
    np.save(Path(out_dir) / f"r{rank}.npy", np.array([run.steps] + recs))
    dist.barrier()
    dist.destroy_process_group()


def test_time_budget_stop_is_collective():
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r0, r1 = np.load(Path(d) / "r0.npy"), np.load(Path(d) / "r1.npy")
    assert list(r0) == list(r1)
    assert r0[0] == 3  # rank 0's budget ran out after 3 iterations; rank 1 stopped with it
