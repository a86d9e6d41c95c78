"""Row-sharded ingest over torch.distributed.

The spatial dimension m is split into contiguous row slabs, one per rank, as a
domain-decomposed solver holds its snapshots.  Omega is keyed on GLOBAL rows (reading R1),
so every rank sketches its own slab and the ell x b partial sketches (plus the column norms)
sum to the unsharded sketch: the only data-path exchange of a block is one all-reduce of
(ell + 1) * b fp64 values between ``oid_ingest_sketch`` and ``oid_ingest_commit``.
Everything after it (Gram, spectrum, scores, selection, Alg 4) is replicated on identical
inputs.  An error estimate adds one all-reduce of the t x t basis-Gram partials
(``oid_estimate_begin`` -> reduce -> ``oid_estimate_end``).

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

    def ingest(self, X):
        """One block (this rank's rows, column-major m_loc x ncols).  The all-reduce runs on the
        engine's ingest stream (torch.distributed enqueues on the current stream), between the
        sketch that writes the partials and the commit that reads them."""
        st = getattr(self.engine, "stream", None)
        ctx = torch.cuda.stream(st) if st is not None and self.world > 1 else _null()
        with ctx:
            self.engine.ingest_sketch(X)
            self._reduce(self.engine.partials(0))
            self.engine.ingest_commit(X)

    def estimate(self, out=None):
        """NA-Hutch++ estimate (Alg 8); out: 8 fp64 values (see include/oid.h).  The reduction runs
        on the engine's estimate stream when it has one (torch.distributed uses the current stream)."""
        est = getattr(self.engine, "estimate_stream", None)
        ctx = torch.cuda.stream(est) if est is not None and self.world > 1 else _null()
        with ctx:
            self.engine.estimate_begin()
            self._reduce(self.engine.partials(1))
            return self.engine.estimate_end(out)
