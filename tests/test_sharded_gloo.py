"""World-size-2 gloo test of the row-sharded ingest protocol (CPU).

Each rank drives an oracle-backed stand-in engine (test double with the C-ABI engine's
sharded interface) over its row slab through paper_2405_16076_b200.sharded.ShardedIngest; the
all-reduced runs must reproduce the unsharded oracle: same selected columns J, coefficients P
and error estimate.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleParams, OracleOID
from oracle.oid import sketch, column_norms2
from synth import c1_matrix


class OracleShardEngine:
    """Test double: the engine's sharded interface on the CPU oracle, for rows [rb, re)."""

    def __init__(self, params):
        self.p = params
        self.o = OracleOID(params)
        self.ell = params.ell
        self._part0 = None
        self._part1 = None
        self._nc = 0

    def ingest_sketch(self, X):
        X = np.asarray(X, dtype=np.float64)
        Y = sketch(self.p, X, self.o._Q)
        n = column_norms2(X)
        self._nc = X.shape[1]
        self._part0 = torch.from_numpy(np.concatenate([Y.T.ravel(), n]))   # [Y col-major; n] as in oid.h

    def partials(self, which):
        return self._part0 if which == 0 else self._part1

    def ingest_commit(self, X):
        v = self._part0.numpy()
        nc, ell = self._nc, self.ell
        Y = v[:ell * nc].reshape(nc, ell).T
        self.o.ingest_block(np.asarray(X, dtype=np.float64), partial_sketch=Y, partial_norms=v[ell * nc:])

    def estimate_begin(self):
        C = self.o.C                                  # this rank's rows of the basis
        self._part1 = torch.from_numpy(np.ascontiguousarray(C.T @ C).ravel())

    def estimate_end(self, out=None):
        t = self.p.t
        G = self._part1.numpy().reshape(t, t)
        return self.o.error_estimate(G=G)


M, N, B, K, ELL = 1500, 64, 16, 8, 24
SPLIT = (4, 8, 12)


def _params(rb=0, re=-1):
    return OracleParams(m=M, k=K, ell=ELL, ell1=SPLIT[0], ell2=SPLIT[1], ell3=SPLIT[2], lam=-1.0, seed=11,
                        row_begin=rb, row_end=re)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_16076_b200.sharded import ShardedIngest, row_slab
        A = c1_matrix(seed=5, m=M, n=N, rank=6, noise=1e-5)
        rb, re = row_slab(M, rank, world)
        drv = ShardedIngest(OracleShardEngine(_params(rb, re)))
        for j in range(0, N, B):
            drv.ingest(A[rb:re, j:j + B])
        est = drv.estimate()
        o = drv.engine.o
        q.put((rank, o.J.copy(), o.P.copy(), est["est_rel"], (rb, re)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_row_slab_partition():
    from paper_2405_16076_b200.sharded import row_slab
    for m in (1000, 14266368, 12345):
        for world in (1, 2, 4, 8):
            cuts = [row_slab(m, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == m
            assert all(cuts[r][1] == cuts[r + 1][0] for r in range(world - 1))
            assert all(c[0] % 32 == 0 for c in cuts)


def test_two_rank_gloo_matches_single():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = c1_matrix(seed=5, m=M, n=N, rank=6, noise=1e-5)
    ref = OracleOID(_params())
    for j in range(0, N, B):
        ref.ingest_block(A[:, j:j + B])
    ref_est = ref.error_estimate()
    assert res[0][4][1] == res[1][4][0]                     # slabs tile the rows
    for rank, J, P, est_rel, _ in res:
        assert np.array_equal(J, ref.J), (rank, J, ref.J)
        assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) < 1e-10
        assert abs(est_rel - ref_est["est_rel"]) < 1e-10
