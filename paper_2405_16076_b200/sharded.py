"""Row-sharded ingest over torch.distributed.

The spatial dimension m is split into contiguous row slabs, one per rank, as a
domain-decomposed solver holds its snapshots.  Omega is keyed on GLOBAL rows (reading R1),
so every rank sketches its own slab and the ell x b partial sketches (plus the column norms)
sum to the unsharded sketch: the only data-path exchange of a block is one all-reduce of
(ell + 1) * b fp64 values between ``oid_ingest_sketch`` and ``oid_ingest_commit``.
Everything after it (Gram, spectrum, scores, selection, Alg 4) is replicated on identical
inputs.  An error estimate adds one all-reduce of the t x t basis-Gram partials
(``oid_estimate_begin`` -> reduce -> ``oid_estimate_end``).

Gradient variant (A11) across slabs: the stencils G^p X of a slab's edge
rows need the neighbouring slabs' rows, so each block first exchanges stencil halos with the two
neighbouring ranks (route (ii): ``exchange_halos``, point-to-point, grad_ny * grad_nz rows each
way), and the d gradient sketches are all-reduced beside [Y; n] (``oid_partials(2)``).
Omega G^p Omega^T needs no exchange (route (i): Omega is generated at any global row) and is
reduced once (``oid_gradient_ogo`` -> ``oid_partials(3)``) before the first GCV.

This module is host-side plumbing only: it calls the engine's C-ABI entry points and
``torch.distributed.all_reduce`` (NCCL on B200, gloo in the CPU tests); it does no arithmetic
of the method.
"""

import contextlib

import torch
import torch.distributed as dist


def _null():
    return contextlib.nullcontext()

ROW_ALIGN = 32   # Philox row-group size of the sketch entries (reading R2): slab starts stay aligned


def row_slab(m, rank, world, align=ROW_ALIGN):
    """[begin, end) of rank's contiguous row slab; interior boundaries rounded to `align` rows."""
    if world <= 1:
        return 0, m
    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return m
        c = (m * r) // world
        return min(m, (c // align) * align)
    return cut(rank), cut(rank + 1)


class ShardedIngest:
    """Drives one engine (this rank's slab) through the sharded ingest / estimate protocol.

    engine: anything with ingest_sketch(X), partials(which) -> tensor (in-place reducible),
    ingest_commit(X), estimate_begin(), estimate_end(out), i.e. paper_2405_16076_b200.Engine.
    group: torch.distributed process group (None = default); world size 1 skips the reductions.
    """

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1

    def _reduce(self, t):
        if self.world <= 1:
            return
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            # gloo (CPU tests, single-GPU runs) reduces host copies; staged on the current stream
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _halo_rows(self):
        f = getattr(self.engine, "grad_halo", None)
        return f() if f is not None else (0, 0)

    def exchange_halos(self, X, rows_lo, rows_hi):
        """Stencil halos of this rank's block X (m_loc x ncols, column-major): returns (lo, hi),
        the rows_lo rows just below the slab (from rank - 1) and the rows_hi rows just above it
        (from rank + 1), each a column-major (rows, ncols) tensor, or None when 0 rows.  A rank
        sends its first rows to rank - 1 and its last rows to rank + 1; the widths a neighbour
        needs are its own rows_hi / rows_lo, exchanged first (so ranks whose halos are clipped
        at the ends of the row range still pair up).  Needs every slab >= its neighbours' halo."""
        if self.world <= 1:
            return None, None
        rank = dist.get_rank(self.group)
        nc = X.shape[1]
        stage = X.is_cuda and dist.get_backend(self.group) == "gloo"
        dev = torch.device("cpu") if stage else X.device
        # widths the neighbours need from this rank: (rank - 1)'s rows_hi, (rank + 1)'s rows_lo
        mine = torch.tensor([rows_lo, rows_hi], dtype=torch.int64, device=dev)
        allw = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allw, mine, group=self.group)
        need_prev = int(allw[rank - 1][1]) if rank > 0 else 0
        need_next = int(allw[rank + 1][0]) if rank + 1 < self.world else 0
        if need_prev > X.shape[0] or need_next > X.shape[0]:
            raise ValueError("a slab is thinner than its neighbour's stencil halo (grad_ny * grad_nz rows)")
        gr = lambda r: dist.get_global_rank(self.group, r) if self.group is not None else r
        ops, bufs = [], {}
        # buffers are (ncols, rows) row-major = (rows, ncols) column-major after .T
        if need_prev:
            ops.append(dist.P2POp(dist.isend, X[:need_prev].T.contiguous().to(dev), gr(rank - 1), self.group))
        if need_next:
            ops.append(dist.P2POp(dist.isend, X[X.shape[0] - need_next:].T.contiguous().to(dev), gr(rank + 1),
                                  self.group))
        if rows_lo:
            bufs["lo"] = torch.empty((nc, rows_lo), dtype=X.dtype, device=dev)
            ops.append(dist.P2POp(dist.irecv, bufs["lo"], gr(rank - 1), self.group))
        if rows_hi:
            bufs["hi"] = torch.empty((nc, rows_hi), dtype=X.dtype, device=dev)
            ops.append(dist.P2POp(dist.irecv, bufs["hi"], gr(rank + 1), self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        out = []
        for key in ("lo", "hi"):
            b = bufs.get(key)
            out.append(None if b is None else b.to(X.device).T)
        return tuple(out)

    def ingest(self, X):
        """One block (this rank's rows, column-major m_loc x ncols).  The all-reduce runs on the
        engine's ingest stream (torch.distributed enqueues on the current stream), between the
        sketch that writes the partials and the commit that reads them.  Gradient variant: the
        stencil halos are exchanged first and the gradient sketches reduced beside [Y; n]."""
        st = getattr(self.engine, "stream", None)
        ctx = torch.cuda.stream(st) if st is not None and self.world > 1 else _null()
        with ctx:
            rows_lo, rows_hi = self._halo_rows()
            if rows_lo or rows_hi:
                lo, hi = self.exchange_halos(X, rows_lo, rows_hi)
                self.engine.ingest_sketch(X, lo, hi)
                self._reduce(self.engine.partials(0))
                self._reduce(self.engine.partials(2))
            else:
                self.engine.ingest_sketch(X)
                self._reduce(self.engine.partials(0))
            self.engine.ingest_commit(X)

    def gradient_ogo(self):
        """Omega G^p Omega^T of the gradient variant, once, before the first GCV: each rank forms
        its rows' part (no exchange) and the parts are summed (oid_partials(3))."""
        st = getattr(self.engine, "stream", None)
        ctx = torch.cuda.stream(st) if st is not None and self.world > 1 else _null()
        with ctx:
            self.engine.gradient_ogo()
            self._reduce(self.engine.partials(3))

    def estimate(self, out=None):
        """NA-Hutch++ estimate (Alg 8); out: 8 fp64 values (see include/oid.h).  The reduction runs
        on the engine's estimate stream when it has one (torch.distributed uses the current stream)."""
        est = getattr(self.engine, "estimate_stream", None)
        ctx = torch.cuda.stream(est) if est is not None and self.world > 1 else _null()
        with ctx:
            self.engine.estimate_begin()
            self._reduce(self.engine.partials(1))
            return self.engine.estimate_end(out)
