"""Full-size parity (BASELINE config 2, C3: m = 14,266,368 fp64, b = 32, k = 200, l = 512) in the
launch configuration bench.py times (tensor-core K1, all SMs), on outputs the oracle can compute
one by one and on properties that hold at any size.  Run with -m gpu on a B200.

* sampled sketch rows: y_r = sum_i Omega(r, i) x_i over all 14.3M rows, recomputed by the oracle
  row by row (oracle.gauss16 + fp64 dot products), against the GPU partial buffer;
* column norms ||x_j||^2 (exact fp64 sums);
* after the commit: the basis slab holds the admitted columns bit-exactly, the Gram is
  Y Y^T (trace = sum of the sketch energy), ||A_obs||^2 equals the norms, J is valid.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.gauss16 import omega_rows, gauss16_scale          # noqa: E402
from synth import ChannelFlow, C3                               # noqa: E402


@pytest.fixture(scope="module")
def oid():
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid
    assert torch.cuda.is_available()
    return oid


def _oracle_row(seed, r, X, chunk=1 << 22):
    """y_r = s sum_i L(n(r, i)) x_i in fp64, in row chunks (oracle Philox + Gauss-16)."""
    acc = np.zeros(X.shape[1])
    for i0 in range(0, X.shape[0], chunk):
        i1 = min(X.shape[0], i0 + chunk)
        L = omega_rows(seed, [r], i0, i1)[0]
        acc += L @ X[i0:i1]
    return gauss16_scale() * acc


def test_c3_fullsize_sampled_parity(oid):
    gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
    m, b, ell, k = gen.m, C3.b, C3.ell, C3.k
    dev = torch.device("cuda", 0)
    X = gen.block_torch(0, b, dev).T                       # (m, b) column-major, as bench.py
    p = oid.make_params(m=m, k=k, ell=ell, b_max=b, n_cap=64, lam=-1.0, seed=0)
    eng = oid.Engine(p)
    eng.ingest_sketch(X)
    part = eng.partials(0).cpu().numpy()
    assert eng.stats()["k1_mode_used"] == oid.K1_TC_INT8
    Yg = part[:ell * b].reshape(b, ell).T
    ng = part[ell * b:ell * b + b]
    Xh = X.cpu().numpy()                                    # host copy of the same bytes
    nref = np.einsum("ij,ij->j", Xh, Xh)
    assert np.max(np.abs(ng - nref) / nref) < 1e-12
    for r in (0, 1, 127, 128, 255, 256, 300, 511):        # both M tiles, both halves, Hutch++ blocks
        yr = _oracle_row(0, r, Xh)
        rel = np.max(np.abs(Yg[r] - yr)) / np.max(np.abs(yr))
        assert rel < 1e-12, (r, rel)
    # commit: Gram, energy, selection, exact basis copy
    eng.ingest_commit(X)
    G = eng.get(3)
    assert np.allclose(G, Yg @ Yg.T, rtol=1e-12, atol=1e-12 * np.max(np.abs(G)))
    sc = eng.scalars()
    assert abs(sc["frob2"] - nref.sum()) <= 1e-12 * nref.sum()
    J = eng.J()
    occ = J[J >= 0]
    assert len(occ) > 0 and len(set(occ.tolist())) == len(occ) and occ.max() < b
    basis = eng.finalize(basis=True)["basis"]
    rows = torch.randint(0, m, (4096,), generator=torch.Generator().manual_seed(1)).to(dev)
    for slot, col in enumerate(J):
        if col >= 0:
            assert torch.equal(basis[rows, slot], X[rows, col]), slot
    eng.close()


def test_c3_fullsize_basis_gram(oid):
    """A9 at full size in the bench launch configuration: after each estimate, sampled entries
    of G = A_J^T A_J equal fp64 dot products of the basis columns (computed on the host from the
    finalized basis), across several blocks so the incremental (dirty-slot) update is covered."""
    gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
    m, b = gen.m, C3.b
    dev = torch.device("cuda", 0)
    p = oid.make_params(m=m, k=C3.k, ell=C3.ell, b_max=b, n_cap=128, lam=-1.0, seed=0)
    eng = oid.Engine(p)
    rng = np.random.default_rng(3)
    for blk in range(3):
        X = gen.block_torch(blk * b, (blk + 1) * b, dev).T
        eng.ingest_block(X)
        est = eng.error_estimate()
        assert np.isfinite(est["est_rel"])
        del X
        G = eng.get(11)
        J = eng.J()
        occ = np.flatnonzero(J >= 0)
        basis = eng.finalize(basis=True)["basis"]
        pick = rng.choice(occ, size=min(6, len(occ)), replace=False)
        cols = {int(i): basis[:, int(i)].cpu().numpy() for i in pick}
        for i in pick:
            for j in pick:
                ref = float(np.dot(cols[int(i)], cols[int(j)]))
                scale = np.sqrt(np.dot(cols[int(i)], cols[int(i)]) * np.dot(cols[int(j)], cols[int(j)]))
                assert abs(G[i, j] - ref) <= 1e-13 * scale, (blk, i, j, G[i, j], ref)
        vac = np.flatnonzero(J < 0)
        assert np.all(G[vac, :] == 0) and np.all(G[:, vac] == 0)
        del basis
    eng.close()
