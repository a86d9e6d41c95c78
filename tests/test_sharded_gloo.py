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


# ---------------------------------------------------------------- gradient variant across slabs
# SURVEY 8(e) route (ii): each block's stencil halos come from the neighbouring ranks, so the
# shards' parts Omega[:, slab] (G^p X)[slab] of the gradient sketches sum to Omega G^p X.
GNF, GNX, GNY, GNC = 2, 10, 12, 5


class HaloShardEngine:
    """Test double of the engine's sharded gradient interface: (G^p X)[slab] from the halo-extended
    slab with the oracle's stencil matrices, sketched by a test-local dense Omega on global rows."""

    def __init__(self, rb, re, m, Om):
        from oracle.gradient import grid_gradient_operators
        self.rb, self.re, self.m, self.Om = rb, re, m, Om
        self.G = grid_gradient_operators(GNF, GNX, GNY)
        self.reach = GNY                         # one axis-0 neighbour = ny rows (2-D grid)
        self.halos = None
        self._p0 = self._p2 = None

    def grad_halo(self):
        return min(self.rb, self.reach), min(self.m - self.re, self.reach)

    def ingest_sketch(self, X, lo=None, hi=None):
        hlo, hhi = self.grad_halo()
        assert (0 if lo is None else lo.shape[0]) == hlo and (0 if hi is None else hi.shape[0]) == hhi
        parts = [t.numpy() for t in (lo, X, hi) if t is not None]
        ext = np.vstack(parts)
        self.halos = (None if lo is None else lo.numpy().copy(), None if hi is None else hi.numpy().copy())
        Om = self.Om[:, self.rb:self.re]
        self._p0 = torch.from_numpy(np.ascontiguousarray(Om @ X.numpy()).ravel())
        gx = [Gp[self.rb:self.re, self.rb - hlo:self.re + hhi] @ ext for Gp in self.G]
        self._p2 = torch.from_numpy(np.concatenate([(Om @ g).ravel() for g in gx]))

    def partials(self, which):
        return {0: self._p0, 2: self._p2}[which]

    def ingest_commit(self, X):
        self.committed = (self._p0.numpy().copy(), self._p2.numpy().copy())


def _halo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_16076_b200.sharded import ShardedIngest
        m = GNF * GNX * GNY
        rng = np.random.default_rng(3)
        A = rng.standard_normal((m, GNC))
        Om = rng.standard_normal((7, m))
        cuts = [0, 64, 160, m][: world + 1] if world == 3 else [0, 128, m]
        rb, re = cuts[rank], cuts[rank + 1]
        eng = HaloShardEngine(rb, re, m, Om)
        drv = ShardedIngest(eng)
        drv.ingest(torch.from_numpy(np.asfortranarray(A[rb:re])))
        q.put((rank, (rb, re), eng.halos, eng.committed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gradient_halo_exchange_gloo(world):
    from oracle.gradient import grid_gradient_operators
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = GNF * GNX * GNY
    rng = np.random.default_rng(3)
    A = rng.standard_normal((m, GNC))
    Om = rng.standard_normal((7, m))
    G = grid_gradient_operators(GNF, GNX, GNY)
    for rank, (rb, re), (lo, hi), (p0, p2) in res:
        # halos are exactly the neighbouring global rows (clipped at the ends of the row range)
        if rb == 0:
            assert lo is None
        else:
            assert np.array_equal(lo, A[rb - min(rb, GNY):rb])
        if re == m:
            assert hi is None
        else:
            assert np.array_equal(hi, A[re:re + min(m - re, GNY)])
        # the reduced partials equal the unsharded sketches [Omega X] and [Omega G^p X]
        assert np.allclose(p0, (Om @ A).ravel(), rtol=0, atol=1e-12)
        ref2 = np.concatenate([(Om @ (Gp @ A)).ravel() for Gp in G])
        assert np.allclose(p2, ref2, rtol=0, atol=1e-10)
