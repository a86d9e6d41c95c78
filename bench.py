"""Snapshot-ingest benchmark of the B200 single-pass randomized ID path (BASELINE.json metric:
"snapshot ingest GB/s (sketch+CSS+Hutch++) at 1/2/4/8 B200; % of roofline").

One step = one block of b snapshots through the whole hot path:
oid_ingest_block (fused sketch incl. the NA-Hutch++ row blocks + norms, [all-reduce], Gram,
ridge regulariser, ridge scores, selection, basis copy, Alg 4) followed by the Alg 8 error
estimate (basis Gram + NA-Hutch++), i.e. Alg 3 steps 9-32 with Alg 4 only.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl reference]

N > 1 is launched by torchrun: rows are sharded (strong scaling, fixed m), one NCCL
all-reduce of the (l+1) x b partial sketch per block and one of the t x t basis-Gram
partials per estimate.  Prints ONE JSON line on rank 0.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (generator spec, b, k, ell, dtype, description)
    "C3": (("channel", (192, 129, 192)), 32, 200, 512, "f64",
           "C3 channel-flow stand-in: 3 components on 192x129x192 (m=14,266,368) fp64, b=32, k=200, l=512"),
    "C3r": (("channel", (48, 33, 48)), 32, 200, 512, "f64", "C3r: C3 on a 48x33x48 grid (m=228,096)"),
    "C5": (("lowrank", 1 << 27), 64, 400, 1024, "f32",
           "C5 scaling sweep: m=2^27 fp32 rows split over the GPUs, rank-500 (sigma_i=i^-1.5) + 1e-5 noise, "
           "n=4096, b=64, k=400, l=1024"),
    "C5r": (("lowrank", 1 << 18), 64, 400, 1024, "f32", "C5r: C5 with m=2^18 rows"),
    # latency-bound configs: K1 reads 0.5 / 1.3 MB per block, the replicated
    # post-pass dominates
    "C1": (("c1", None), 16, 20, 48, "f64",
           "C1: m=4096 fp64, rank-10 (sigma_i=10^(-i/3)) + 1e-6 noise, n=512, b=16, k=20, l=48, "
           "lambda=||A-A_k||^2/k by the harness (P:203)"),
    "C2": (("image", None), 64, 100, 256, "f32",
           "C2: NSTX GPI stand-in, 64x80 frames (m=5120) fp32, n=20000, b=64, k=100, l=256"),
}


class _HostStream:
    """A host-generated stream (C1 matrix / C2 frames) exposed like the device generators:
    .m, block_torch (device upload, outside any timed region), block (host)."""

    def __init__(self, kind):
        from synth import c1_matrix, ImageStream, C1
        self.kind = kind
        if kind == "c1":
            self.A = c1_matrix(seed=C1.data_seed)
            self.m = self.A.shape[0]
            s = np.linalg.svd(self.A, compute_uv=False)
            self.lam = float(np.sum(s[C1.k:] ** 2) / C1.k)          # P:203, computed by the harness
            self.split = C1.split
        else:
            self.img = ImageStream(seed=1002)
            self.m = ImageStream.H * ImageStream.W
            self.lam, self.split = -1.0, None

    def block(self, t0, t1, row_begin=0, row_end=None):
        row_end = self.m if row_end is None else row_end
        # C1 has n = 512 snapshots: longer runs cycle through it (stated in config.blocks)
        X = self.A[:, np.arange(t0, t1) % self.A.shape[1]] if self.kind == "c1" else self.img.block(t0, t1)
        return X[row_begin:row_end]

    def block_torch(self, t0, t1, device, row_begin=0, row_end=None):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.block(t0, t1, row_begin, row_end).T)).to(device)


def make_gen(workload):
    from synth import ChannelFlow, LowRankStream
    (kind, arg) = WORKLOADS[workload][0]
    if kind in ("c1", "image"):
        return _HostStream(kind)
    return ChannelFlow(*arg, seed=1003) if kind == "channel" else LowRankStream(m=arg, seed=1005)


def gen_lam_split(gen, ell):
    """lambda mode and NA-Hutch++ split of a workload (C1: the harness lambda and 16/16/16, R11)."""
    lam = getattr(gen, "lam", -1.0)
    split = getattr(gen, "split", None) or (ell // 6, ell // 3, ell - ell // 6 - ell // 3)
    return lam, split


def host_rows(workload, gen, t0, t1, rows):
    """Rows [0, rows) of a block on the host (numpy, the generator's host formula)."""
    if WORKLOADS[workload][0][0] == "channel":
        return _host_rows(gen, t0, t1, rows)
    return np.asarray(gen.block(t0, t1, 0, rows), dtype=np.float64)


METRIC = "snapshot ingest GB/s (sketch+CSS+Hutch++) at 1/2/4/8 B200; % of roofline"
FP64_NOMINAL_TF, BF16_NOMINAL_TF = 40.0, 2250.0    # B200 datasheet ratio used to derive the fp64 peak


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=28)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--workload", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--k1-mode", type=int, default=4,
                    help="oid_k1_mode: 4 = K1F (31-bit fixed point, parity-tested at full C3 size in "
                         "tests/test_gpu_k1fast.py; the default), 2 = exact int8 digit planes, 0 = auto (exact)")
    ap.add_argument("--a9", default="q", choices=["q", "fp64"],
                    help="basis Gram: q = A9Q (int8 tensor cores on the 31-bit quantised basis copy, a9_mode = 1; "
                         "with --k1-mode 4, the default) or fp64 (exact DMMA Gram)")
    ap.add_argument("--no-estimate", action="store_true", help="ingest only (estimate not in the step)")
    ap.add_argument("--no-pipeline", dest="pipeline", action="store_false",
                    help="single shard: end each estimate before the next block's ingest is issued (the default "
                         "ends it after, so the library runs the estimate's basis Gram beside the next block's "
                         "post-pass: C3 609 vs 587 GB/s with A9Q in at most 6 clusters)")
    ap.add_argument("--one-stream", action="store_true", help="estimates on the ingest stream (no overlap)")
    ap.add_argument("--cpu-sample-rows", type=int, default=1 << 18)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp["hbm_gbs"], mp["bf16_tflops"], mp.get("bf16_tflops_sustained", mp["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.idx = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "-i", str(self.idx),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU oracle legs
def oracle_sample(workload, rows, steps=1, warmup=0):
    """Time the CPU oracle (as it stands) on row-sampled blocks of the workload.

    Each step = OracleOID.ingest_block + error_estimate on rows [0, rows) of one fresh block.
    Returns (GB/s over the timed steps, seconds per step, BLAS threads, sample description).
    """
    from oracle import OracleParams, OracleOID
    _, b, k, ell, dt, _ = WORKLOADS[workload]
    gen = make_gen(workload)
    m = gen.m
    rows = min(rows, m)
    lam, sp = gen_lam_split(gen, ell)
    o = OracleOID(OracleParams(m=m, k=k, ell=ell, ell1=sp[0], ell2=sp[1], ell3=sp[2], lam=lam, seed=0,
                               row_begin=0, row_end=rows), cache_omega=False)
    blocks = [host_rows(workload, gen, s * b, (s + 1) * b, rows) for s in range(warmup + steps)]
    for X in blocks[:warmup]:
        o.ingest_block(X)
        o.error_estimate()
    t0 = time.perf_counter()
    for X in blocks[warmup:]:
        o.ingest_block(X)
        o.error_estimate()
    dt_s = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        thr = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        thr = 1
    gbs = steps * rows * b * 8 / dt_s / 1e9
    sample = (f"{workload} rows [0,{rows}) of {m} x {b} snapshots per block, all {ell} sketch rows, "
              f"{steps} timed block(s) after {warmup} warm-up: oracle ingest_block + error_estimate")
    return gbs, dt_s / steps, thr, sample


def _host_rows(gen, t0, t1, rows):
    """Rows [0, rows) of a ChannelFlow block on the host (numpy), same formula as synth.ChannelFlow.block."""
    import numpy as np
    plane = gen.ny * gen.nx
    nz_needed = (rows + plane - 1) // plane
    a = gen._coeff(t0, t1)
    ex = np.exp(1j * gen.alpha[None, :] * gen.x[:, None] / 4)
    ez = np.exp(1j * 2 * gen.beta[None, :] * gen.z[:, None] / 3)
    out = np.empty((nz_needed * plane, t1 - t0))
    for zi in range(nz_needed):
        F = (ez[zi][None, None, :] * gen.g[:, None, :] * ex[None, :, :]).reshape(-1, gen.NMODE)
        out[zi * plane:(zi + 1) * plane] = (F @ a[0]).real + (1 - gen.y ** 2).repeat(gen.nx)[:, None]
    out = out[:rows]
    for j, t in enumerate(range(t0, t1)):
        out[:, j] += gen.noise * np.random.default_rng([gen.seed, t]).standard_normal(rows)
    return out


def run_reference(args, rank, world):
    """Reference arm = the CPU oracle (no runnable reference implementation exists)."""
    if rank != 0:
        return
    steps = max(1, args.steps)
    rows = min(args.cpu_sample_rows, 1 << 16)
    gbs, secs, thr, sample = oracle_sample(args.workload, rows, steps=steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload][5], "sample_rows": rows},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": thr, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ B200 arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _, b, k, ell, dt, desc = WORKLOADS[args.workload]
    gen = make_gen(args.workload)
    m = gen.m
    from paper_2405_16076_b200.sharded import ShardedIngest, row_slab
    rb, re = row_slab(m, rank, world)
    m_loc = re - rb
    W, K, E = args.warmup, args.steps, args.e2e_steps
    nblk = W + K + E
    n_cap = max(1000, (nblk + 8) * b)   # + the ingest-only blocks
    # distinct device-resident blocks: the whole stream when it fits (C3: 31 blocks of 3.65 GB),
    # else a ring cycled in order (stated in config.blocks)
    dsz = 8 if dt == "f64" else 4
    free = torch.cuda.mem_get_info(dev)[0]
    blk_bytes_loc = (re - rb) * b * dsz
    lam, split = gen_lam_split(gen, ell)
    ws_bytes = oid.workspace_bytes(oid.make_params(m=m, k=k, ell=ell, b_max=b, n_cap=n_cap, lam=lam, split=split,
                                                   seed=0, dtype=dt, row_begin=rb, row_end=re))
    if ws_bytes + 2 * blk_bytes_loc + (4 << 30) > free:
        # e.g. C5 at N = 1: the 400-column basis alone is 215 GB; E(P) is taken from P = 2
        if rank == 0:
            print(json.dumps({"metric": METRIC, "n_gpus": world, "config": {"workload": desc},
                              "unavailable": f"workspace {ws_bytes / 1e9:.1f} GB + two blocks of "
                                             f"{blk_bytes_loc / 1e9:.1f} GB exceed the {free / 1e9:.0f} GB free "
                                             f"on this GPU at {world} GPU(s)"}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    ring = max(2, min(W + K, int((free - ws_bytes - (8 << 30)) // blk_bytes_loc)))
    p = oid.make_params(m=m, k=k, ell=ell, b_max=b, n_cap=n_cap, lam=lam, split=split, seed=0, dtype=dt,
                        row_begin=rb, row_end=re, k1_mode=args.k1_mode, profile=True, device=local,
                        a9q=(args.a9 == "q" and args.k1_mode == 4))
    # ingest on a high-priority stream, estimates on a second stream: the basis Gram of block k
    # (HBM/DMMA-bound) overlaps the latency-bound post-pass of block k+1
    stream = torch.cuda.Stream(dev, priority=-1)
    est_stream = torch.cuda.Stream(dev, priority=0) if not args.one_stream else stream
    eng = oid.Engine(p, stream=stream, estimate_stream=est_stream)

    # synthetic blocks, generated on the device outside any timed region (inputs >> L2)
    blocks = []
    for s in range(ring):
        blocks.append(gen.block_torch(s * b, (s + 1) * b, dev, row_begin=rb, row_end=re).T)   # (m_loc, b) col-major
    torch.cuda.synchronize()
    est_out = torch.empty(8, dtype=torch.float64, device=dev)
    sharded = world > 1

    drv = ShardedIngest(eng)

    # inputs smaller than L2 (C1, C2): flush L2 before every step by writing 256 MB on the ingest
    # stream, inside the timed region (the reported step time is an upper bound)
    small = ring * blk_bytes_loc < (256 << 20)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None

    # --pipeline (single shard): the estimate of block e ends after block e+1's ingest has been issued
    # (the begin/end split of the ABI; the library then launches the basis Gram beside e+1's
    # post-pass).  Every timed step still issues one ingest and one complete estimate; the last
    # estimate ends inside the timed region.
    pipelined = not sharded and not args.no_estimate and not args.one_stream and args.pipeline
    pending = [False]

    def step(X):
        if flush is not None:
            flush.fill_(1)
        if sharded:
            drv.ingest(X)                 # sketch -> all-reduce of the (l+1) x b partials -> commit
        else:
            eng.ingest_block(X)
        if not args.no_estimate:
            if pipelined:
                if pending[0]:
                    eng.estimate_end(est_out)     # the previous block's estimate
                eng.estimate_begin()
                pending[0] = True
            else:
                drv.estimate(est_out)     # basis-Gram partials all-reduced when sharded

    def finish():
        if pending[0]:
            eng.estimate_end(est_out)
            pending[0] = False

    for s in range(W):
        with torch.cuda.stream(stream):
            step(blocks[s % ring])
    with torch.cuda.stream(stream):
        finish()
    torch.cuda.synchronize()
    eng.stats_reset()
    st0 = eng.stats()                    # device counters (admissions, dirty slots) before the timed region
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for s in range(W, W + K):
            step(blocks[s % ring])
        finish()
    stream.wait_stream(est_stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    st = eng.stats()
    if sharded:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    dsz = 8 if dt == "f64" else 4
    block_bytes = m * b * dsz                       # all ranks together
    value = K * block_bytes / (ms * 1e-3) / 1e9
    est_val = est_out.cpu().tolist()

    # ingest GB/s alone (K1 -> AR1 -> K2-K7, no estimate), on the next blocks of
    # the stream after the timed region (reported beside the step metric, not instead of it)
    ingest_only = None
    KI = min(8, K)
    if not args.no_estimate and KI > 0:
        # the next KI snapshots blocks of the stream, generated into ring slots the timed region is
        # done with (cycling back to block 0 would feed the engine columns it has already seen)
        for s in range(W + K, W + K + KI):
            blocks[s % ring] = None
            blocks[s % ring] = gen.block_torch(s * b, (s + 1) * b, dev, row_begin=rb, row_end=re).T
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for s in range(W + K, W + K + KI):
                X = blocks[s % ring]
                if flush is not None:
                    flush.fill_(1)
                if sharded:
                    drv.ingest(X)
                else:
                    eng.ingest_block(X)
        e1.record(stream)
        torch.cuda.synchronize()
        ims = e0.elapsed_time(e1)
        if sharded:
            t = torch.tensor([ims], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ims = t.item()
        ingest_only = {"ms_per_block": ims / KI, "value": KI * block_bytes / (ims * 1e-3) / 1e9, "unit": "GB/s",
                       "blocks": KI, "definition": "SURVEY 8(d) D(1): ingest_block only (no estimate), the "
                                                   f"{KI} blocks after the timed region"}

    # roofline of the dominant kernel (K1, fused ingest) on this rank, as SURVEY.md section 8(d)
    # defines it: t_roof = max(HBM read of the block, 2 l m b sketch flops at the chosen pipe's peak),
    # frac = t_roof / t_K1 (DESIGN.md section 7 lists the per-unit figures)
    hbm, bf16, bf16_sus, src = peaks()
    int8_tops = 2.0 * bf16_sus                      # B200 dense int8 = 2 x bf16 (nominal 4.5 / 2.25 PFLOP/s);
                                                    # sustained: K1 is timed inside the long step
    k1_avg_ms = st["k1_ms"] / max(1, st["k1_launches"])
    k1_bytes = m_loc * b * dsz
    k1_flops = 2.0 * ell * m_loc * b
    mode = st["k1_mode_used"]
    t_hbm = k1_bytes / (hbm * 1e9) * 1e3
    tc_modes = (oid.K1_TC_INT8, oid.K1_TC_PAIR, oid.K1_TC_FAST)
    t_flop = k1_flops / (int8_tops * 1e12) * 1e3 if mode in tc_modes else \
        k1_flops / (bf16_sus * FP64_NOMINAL_TF / BF16_NOMINAL_TF * 1e12) * 1e3
    t_roof = max(t_hbm, t_flop)
    traffic, traffic_src = _traffic_from_profiles(args.workload, mode)
    roof = {"bound": "hbm" if t_hbm >= t_flop else "tensor",
            "achieved": k1_bytes / (k1_avg_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": t_roof / k1_avg_ms, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": {oid.K1_TC_INT8: "k1_tc_kernel", oid.K1_TC_PAIR: "k1p::k1_tc_kernel",
                       oid.K1_TC_FAST: "k1f_kernel"}.get(mode, "k1_simt_kernel"),
            "k1_ms": k1_avg_ms, "hbm_roof_ms": t_hbm, "flop_roof_ms": t_flop, "peak_source": src,
            "definition": "frac = max(block bytes / HBM peak, 2 l m b / int8 peak) / t_K1 (SURVEY 8(d)); "
                          "t_K1 = CUDA events on the ingest stream inside the timed region"}
    planes = {oid.K1_TC_INT8: 7 if dt == "f64" else 6, oid.K1_TC_PAIR: 6, oid.K1_TC_FAST: 4}.get(mode, 0)
    emul = None
    if mode in tc_modes:
        ops = planes * k1_flops
        emul = {"planes": planes, "int8_ops_per_launch": ops, "achieved_tops": ops / (k1_avg_ms * 1e-3) / 1e12,
                "peak_tops": int8_tops, "frac": ops / (k1_avg_ms * 1e-3) / 1e12 / int8_tops,
                "note": ("fixed-point emulation: one int8 MAC per digit plane per sketch multiply-add; " +
                         ("31-bit fixed point (K1F), |x - x_q| <= 2^-27 max|x_j|" if mode == oid.K1_TC_FAST
                          else "exact (56-bit / 48-bit fixed point)"))}
    # sketch-entry (RNG) roof: l m_loc Gauss-16 entries per launch; ALU-pipe bound at 1.5 ALU ops per
    # entry (Philox4x32-10: 20 LOP3 per 32 entries; Gauss-16 decode: 7 ALU ops per 8 entries, sm_100a
    # SASS) on 148 SMs x 64 ALU lanes per clock
    clk = clocks.get("sm_mhz") or 1965.0
    entries = float(ell) * m_loc
    rng_peak = 148 * 64 * clk * 1e6 / 1.5
    rng = {"entries_per_launch": entries, "entries_per_s": entries / (k1_avg_ms * 1e-3),
           "alu_ops_per_entry": 1.5, "peak_entries_per_s": rng_peak, "rng_roof_ms": entries / rng_peak * 1e3,
           "frac": entries / rng_peak * 1e3 / k1_avg_ms, "sm_mhz": clk}
    # A9 (exact basis Gram, one read of the basis slab per estimate) and the whole step
    a9 = None
    if st.get("a9_launches", 0):
        a9_ms = st["a9_ms"] / st["a9_launches"]
        basis_bytes = m_loc * k * dsz
        nd = (st["dirty_slots"] - st0["dirty_slots"]) / max(1, st["estimates"] - st0["estimates"])
        fp64_tf = bf16_sus * FP64_NOMINAL_TF / BF16_NOMINAL_TF
        t_a9_hbm = basis_bytes / (hbm * 1e9) * 1e3
        t_a9_flop = 2.0 * nd * k * m_loc / (fp64_tf * 1e12) * 1e3
        a9 = {"kernel": "basis_gram_tc_kernel", "ms_per_launch": a9_ms, "bytes_per_launch": basis_bytes,
              "achieved_gbs": basis_bytes / (a9_ms * 1e-3) / 1e9, "dirty_slots_per_estimate": nd,
              "hbm_roof_ms": t_a9_hbm, "dmma_roof_ms": t_a9_flop, "fp64_tensor_peak_tflops": fp64_tf,
              "frac": max(t_a9_hbm, t_a9_flop) / a9_ms}
        if args.a9 == "q" and mode == oid.K1_TC_FAST:
            # A9Q: 4 bytes per basis element (quantised copy), 16 int8 plane pairs per fp64 MAC
            qbytes = m_loc * k * 4
            t_q_hbm = qbytes / (hbm * 1e9) * 1e3
            t_q_mma = 16 * 2.0 * nd * k * m_loc / (int8_tops * 1e12) * 1e3
            a9 = {"kernel": "a9q::gram_q_kernel (a9_mode = 1)", "ms_per_launch": a9_ms, "bytes_per_launch": qbytes,
                  "achieved_gbs": qbytes / (a9_ms * 1e-3) / 1e9, "dirty_slots_per_estimate": nd,
                  "hbm_roof_ms": t_q_hbm, "int8_roof_ms": t_q_mma, "frac": max(t_q_hbm, t_q_mma) / a9_ms}
    adm = (st["admissions"] - st0["admissions"]) / K
    step_bytes = block_bytes + (0 if args.no_estimate else m * k * dsz) + 2.0 * m * dsz * adm
    step_roof = {"algorithmic_bytes_per_step": step_bytes, "admissions_per_step": adm,
                 "hbm_floor_ms": step_bytes / (hbm * 1e9) * 1e3, "ms_per_step": ms / K,
                 "frac": step_bytes / (hbm * 1e9) * 1e3 / (ms / K),
                 "terms": "block read + basis read by the estimate (A9) + 2 column bytes per admission (A7)"}
    latency = {"min_ms": st["lat_min_ms"], "median_ms": st["lat_med_ms"], "max_ms": st["lat_max_ms"],
               "span": "start of the block's K1 to the end of its commit (ingest stream)"}

    # e2e through the public API with HOST buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if E > 0:
        host = []
        for s in range(E):
            t0_ = (W + K + (KI if ingest_only is not None else 0) + s) * b
            hb = torch.empty((b, m_loc), dtype=blocks[0].dtype, pin_memory=True)
            hb.copy_(gen.block_torch(t0_, t0_ + b, dev, row_begin=rb, row_end=re).cpu())
            host.append(hb)
        # double-buffered device blocks: the H2D copy of block k+1 (copy stream) overlaps the
        # ingest + estimate of block k; every step still copies its whole block in and its
        # estimate out inside the timed region
        dbufs = [torch.empty((b, m_loc), dtype=blocks[0].dtype, device=dev) for _ in range(2)]
        est_host = torch.empty(8, dtype=torch.float64, pin_memory=True)
        cstream = torch.cuda.Stream(dev)
        ev_copied = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]
        del blocks
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cstream.wait_event(e0)
        for i, hb in enumerate(host):
            bsel = i % 2
            with torch.cuda.stream(cstream):
                if i >= 2:
                    cstream.wait_event(ev_used[bsel])
                dbufs[bsel].copy_(hb, non_blocking=True)
                ev_copied[bsel].record(cstream)
            stream.wait_event(ev_copied[bsel])
            with torch.cuda.stream(stream):
                step(dbufs[bsel].T)
                ev_used[bsel].record(stream)
            with torch.cuda.stream(est_stream):
                est_host.copy_(est_out, non_blocking=True)
        with torch.cuda.stream(stream):
            finish()                      # the last block's estimate (pipelined mode)
        with torch.cuda.stream(est_stream):
            est_host.copy_(est_out, non_blocking=True)
        stream.wait_stream(est_stream)
        stream.wait_stream(cstream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if sharded:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": E * block_bytes / (ems * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": block_bytes, "d2h_bytes_per_step": 8 * 8, "steps": E}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu_baseline:
        gbs, secs, thr, sample = oracle_sample(args.workload, args.cpu_sample_rows)
        cpu = {"value": gbs, "unit": "GB/s", "cores": thr, "kind": "oracle", "sample": sample, "seconds": secs}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if world > 1 else "strong",
            "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": {"workload": desc, "m": m, "b": b, "k": k, "ell": ell,
                       "lambda": "paper surrogate (-1)" if lam == -1.0 else f"fixed {lam:.6g} (harness, P:203)",
                       "step": ("ingest_block + error_estimate" + (" (estimate of block e ended after the ingest of "
                                                                    "e+1 is issued; the last one inside the timed region)"
                                                                    if pipelined else "")) if not args.no_estimate else "ingest_block",
                       "l2": ("inputs larger than L2 (each block %.2f GB, fresh block per step)" % (block_bytes / 1e9))
                             if flush is None else "inputs smaller than L2: 256 MB L2 flush on the ingest stream before "
                                                   "every step, inside the timed region",
                       "blocks": f"stream snapshots [0, {(W + K) * b}) in blocks of {b}, {ring} distinct device-resident blocks"
                                 + ("" if ring >= W + K else " (cycled)"),
                       "parallelism": f"rows sharded over {world} GPU(s)"},
            "roofline": roof,
            "emulation_pipe": emul,
            "rng": rng,
            "a9": a9,
            "step_roofline": step_roof,
            "block_latency": latency,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": st["launches"],
            "breakdown_ms_per_step": {"k1": st["k1_ms"] / K, "post": st["post_ms"] / K, "estimate": st["est_ms"] / K},
            "ingest_only": ingest_only,
            "last_estimate": {"est_rel": est_val[5], "e2": est_val[0], "flags": int(est_val[6])},
            "k1_mode": {oid.K1_TC_INT8: "tc_int8 (exact)", oid.K1_TC_PAIR: "tc_pair (exact)",
                        oid.K1_TC_FAST: "tc_fast (K1F: 31-bit fixed point, int8 digit planes, int32 accumulate, "
                                        "fp64 assembly)"}.get(mode, "simt_f64"),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if sharded:
        dist.destroy_process_group()


def _traffic_from_profiles(workload, mode):
    """dram bytes per K1 launch (read + write) copied from a committed ncu --set full capture of the
    same kernel on the same workload (profiles/k1_traffic.json names the capture), or None."""
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        key = f"{workload}:{ {2: 'tc', 3: 'pair', 4: 'fast'}.get(mode, 'simt') }"
        ent = d.get(key)
        if isinstance(ent, dict):
            return ent.get("bytes"), "copied from " + ent.get("capture", "profiles/k1_traffic.json")
        return ent, "copied from profiles/k1_traffic.json"
    except Exception:
        return None, None


if __name__ == "__main__":
    main()
