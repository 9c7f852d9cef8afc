"""Multi-GPU work division on CPU: partition logic, the row-strip halo split
checked against the oracle (bit-exact counts, flows equal to the unsplit
slice), and a world_size-2 gloo run of the distributed assembly."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import veckm_oracle as vo
from paper_2504_19417_b200 import sharding


def test_slice_range_covers_exactly_once():
    for n in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in sharding.slice_range(n, r, world)]
            assert got == list(range(n))
            sizes = [len(sharding.slice_range(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_row_strips_balance_and_halo():
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 100, size=720)
    for world in (1, 2, 4, 8):
        strips = sharding.row_strips(counts, world, 10)
        assert strips[0].lo == 0 and strips[-1].hi == 720
        for a, b in zip(strips[:-1], strips[1:]):
            assert a.hi == b.lo
        for s in strips:
            assert s.in_lo == max(0, s.lo - 10) and s.in_hi == min(720, s.hi + 10)
        owned = np.array([counts[s.lo:s.hi].sum() for s in strips])
        assert owned.max() - owned.min() <= 2 * counts.max() + 1


class _OracleEngine:
    """Stands in for FlowEngine: the oracle on a strip geometry (test only)."""

    def __init__(self, width, height, dx, dy, fr, w):
        self.args = (width, height, dx, dy, fr, w)

    def predict_host(self, events, t_start, return_counts=False):
        W, H, dx, dy, fr, w = self.args
        t = events[:, 0] - t_start
        x = events[:, 1].astype(np.int64)
        y = events[:, 2].astype(np.int64)
        g = vo.accumulate(t, x, y, W, H, dx, dy, fr, 0.016)
        emb, cnt = vo.pool(g, vo.spatial_table(fr, dx, dy), t, x, y, fr, 0.016)
        flows = vo.mlp(w[0], w[1], w[2], w[3], vo.to_features(emb)).astype(np.float32)
        return (flows, cnt.astype(np.int32)) if return_counts else flows


def _setup(n=6000, W=40, H=48, seed=3):
    X = vo.synth_uniform_noise(n, W, H, seed=seed)
    fr = vo.make_freqs(16)
    g = np.random.default_rng(1)
    w = (g.normal(0, 0.25, (8, 32)).astype(np.float32), np.zeros(8, np.float32),
         g.normal(0, 0.5, (2, 8)).astype(np.float32), np.zeros(2, np.float32))
    return X, fr, w


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_spatial_split_equals_unsplit_oracle(world):
    X, fr, w = _setup()
    W, H, d = 40, 48, 4
    full = _OracleEngine(W, H, d, d, fr, w).predict_host(X, float(X[0, 0]), return_counts=True)
    parts_flows = []
    for rank in range(world):
        out = sharding.predict_spatial(lambda h: _OracleEngine(W, h, d, d, fr, w), X, float(X[0, 0]), W, H, d,
                                       world=1, rank=0, return_counts=True) if world == 1 else None
        parts_flows.append(out)
    if world == 1:
        flows, counts = parts_flows[0]
    else:
        rows = np.bincount(X[:, 2].astype(np.int64), minlength=H)
        strips = sharding.row_strips(rows, world, d)
        ses = [sharding.strip_events(X, s) for s in strips]
        res = [_OracleEngine(W, s.height, d, d, fr, w).predict_host(se.events, float(X[0, 0]), True)
               for s, se in zip(strips, ses)]
        flows, counts = sharding.assemble(len(X), ses, [r[0] for r in res], [r[1] for r in res])
    np.testing.assert_array_equal(counts, full[1])
    np.testing.assert_array_equal(flows, full[0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, fr, w = _setup()
        W, H, d = 40, 48, 4
        out = sharding.predict_spatial(lambda h: _OracleEngine(W, h, d, d, fr, w), X, float(X[0, 0]), W, H, d,
                                       world=world, rank=rank, return_counts=True)
        if rank == 0:
            q.put(out)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_spatial_split():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    flows, counts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    X, fr, w = _setup()
    full = _OracleEngine(40, 48, 4, 4, fr, w).predict_host(X, float(X[0, 0]), return_counts=True)
    np.testing.assert_array_equal(counts, full[1])
    np.testing.assert_array_equal(flows, full[0])
