/*
 * oid.h — C ABI of liboid.so, the B200 (sm_100a) hot path of the single-pass online
 * randomized interpolative decomposition with NA-Hutch++ error estimation
 * (Li, Becker, Doostan, arxiv 2405.16076).  Citations: P:n = line n of the paper's LaTeX
 * source; readings R1..R14 are in DESIGN.md section 3.
 *
 * Problem: A = [a_1 .. a_n] (m x n) arrives column by column; the library keeps a
 * sketch S = Omega A_obs, a basis of t = k selected columns A_J and coefficients P with
 * A_obs ~ A_J P (eqn:id), following Algorithm 3 with Algorithm 4
 * coefficients and Algorithm 8 error estimates.
 *
 * Conventions for every entry point
 *   - All matrices are column-major.  Device pointers are CUDA global memory on the context's
 *     device; "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every call returns an oid_status.  Parameters are validated before any data is touched
 *     (OID_EINVAL / OID_ESHAPE); call order is checked (OID_ESTATE).  CUDA launch failures
 *     return OID_ECUDA.  oid_last_error(ctx) returns a message for the last failure.
 *   - Numerical degradation that is not an error (non-finite input, rank-deficient S_J,
 *     negative estimated ||E||^2) is reported in flag bits (OID_FLAG_*), never silently.
 *   - Ingest calls are asynchronous: nothing is copied to the host and the host never waits.
 *   - Determinism: identical parameters and data give bitwise-identical J, P and estimates.
 *   - The context is single-threaded.  With several row shards, all ranks make the same calls
 *     in the same order (collective semantics) and reduce the exposed partial buffers between
 *     the *_sketch/_begin and *_commit/_end halves (sum, fp64), e.g. with an NCCL all-reduce.
 */
#ifndef OID_H_
#define OID_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oid_ctx_s* oid_ctx;

typedef enum {
  OID_OK = 0,
  OID_EINVAL = -1,   /* bad parameter values                                               */
  OID_ESHAPE = -2,   /* ncols > b_max, ld < m_loc, capacity n_cap exceeded, small workspace */
  OID_ENOMEM = -3,   /* host allocation failed                                              */
  OID_ECUDA = -4,    /* CUDA error (launch, copy, no device / unsupported arch)             */
  OID_ENCCL = -5,    /* reserved: collective failure reported by the caller's reducer       */
  OID_ENUMERIC = -6, /* reserved                                                            */
  OID_ESTATE = -7    /* call out of order (e.g. commit without sketch)                      */
} oid_status;

typedef enum { OID_F32 = 0, OID_F64 = 1 } oid_dtype;

/* K1 (fused ingest) implementation.  Modes 0-3 are exact to fp64 rounding. */
typedef enum {
  OID_K1_AUTO = 0,      /* tensor-core path when available for the shape, else SIMT       */
  OID_K1_SIMT_F64 = 1,  /* CUDA-core DFMA, Omega generated in registers                    */
  OID_K1_TC_INT8 = 2,   /* tcgen05 kind::i8, Omega generated into TMEM (A operand), data
                           split into exact int8 digit planes in shared memory (sm_100a);
                           needs row_begin % 32 == 0, 16-byte aligned X and ld            */
  OID_K1_TC_PAIR = 3,   /* experimental: 2-CTA (cta_group::2) variant of OID_K1_TC_INT8 with
                           48-bit digit planes converted by integer arithmetic            */
  OID_K1_TC_FAST = 4    /* K1F: tcgen05 kind::i8 with the data quantised to a 31-bit per-column
                           fixed point (4 signed digit planes stacked in M, Omega^T generated
                           into shared memory as the B operand, each X element converted once
                           for ell <= 512).  Not exact: |x - x_q| <= 2^-26 max_i |x_ij| per
                           element, within north_star's 1e-5 tolerance.
                           Used for the snapshot blocks; the gradient passes stay exact.  Same
                           alignment needs as OID_K1_TC_INT8, else the exact kernels run.  */
} oid_k1_mode;

/* flag bits (oid_stats.flags, estimate out[6]) */
#define OID_FLAG_NONFINITE_INPUT 1u   /* a block contained NaN/Inf (column norm not finite)   */
#define OID_FLAG_SJ_RANK_DEFICIENT 2u /* S_J had singular values below the 1e-12 cutoff (R9)   */
#define OID_FLAG_E2_NEGATIVE 4u       /* NA-Hutch++ ||E||^2 estimate < 0, clamped (R13 / S:434) */
#define OID_FLAG_K1_RECOMPUTED 8u     /* tensor-core K1 re-ran a slab with exact exponents     */

typedef struct {
  int64_t m;          /* global rows (spatial points of one snapshot)              */
  int64_t row_begin;  /* this shard's global rows [row_begin, row_end); Omega is keyed   */
  int64_t row_end;    /*   on GLOBAL rows so the sketch is independent of the sharding   */
  int64_t n_cap;      /* max columns ever ingested (sizes S: ell x n_cap, P: k x n_cap)  */
  int32_t k;          /* target rank = basis size t (k = t); 1 <= k <= min(ell, 416) */
  int32_t ell;        /* sketch rows l = k + p; 1 <= ell <= 1024                  */
  int32_t b_max;      /* max columns per ingest call, 1..64                              */
  int32_t ell1, ell2, ell3; /* NA-Hutch++ contiguous row split, sum = ell (R11)    */
  double lambda;      /* >= 0 fixed ridge; -1 streaming surrogate;
                         -2 sketch-tail surrogate (R8)                                   */
  double eps, delta;  /* accuracy / failure probability of the admission rate    */
  double c;           /* admission constant (R5: 1)                                      */
  uint64_t seed;      /* Philox key (R1): tag 0 sketch entries, tag 1 selection draws    */
  int32_t dtype;      /* oid_dtype of the snapshot data and of the stored basis          */
  int32_t k1_mode;    /* oid_k1_mode                                                     */
  int32_t profile;    /* 1: time K1 and the other kernel groups with CUDA events          */
  int32_t device;     /* CUDA device ordinal the workspace lives on                      */
  /* Gradient-enhanced variant (reading Q17).  grad_nfields > 0 enables
     it: a snapshot stacks grad_nfields fields on a grad_nx x grad_ny grid (field f at rows
     [f nx ny, (f+1) nx ny), node (i, j) at f nx ny + i ny + j); simplex gradients over the axis
     neighbours with spacings grad_hx, grad_hy (0: 1/(N-1)).  The ridge scores then use the
     augmented sketch [Omega a; Omega G^1 a; Omega G^2 a] and the augmented energy; the
     estimate keeps Alg 4's P; oid_gradient_* give P(mu) and the sketched GCV.  Requires
     grad_nfields grad_nx grad_ny (grad_nz) = m and (d + 1) ell <= 2048.  Row-sharded contexts
     (route (ii) for G^p X): each block comes with its stencil halos
     (oid_ingest_sketch_halo, widths from oid_grad_halo), the gradient sketches are summed with
     oid_partials(2) beside oid_partials(0), and Omega G^p Omega^T (route (i): Omega generated at
     the neighbouring global rows, no exchange) with oid_gradient_ogo + oid_partials(3).  */
  int32_t grad_nfields, grad_nx, grad_ny;
  int32_t omega_cache; /* NEXT-3 ablation: 1 = store the sketch entries (their Philox words,
                          ell * m_loc / 2 bytes of workspace, filled at oid_init) and stream them
                          into the tensor-core K1 instead of generating them; 0 = generate in
                          registers (the default).  Same entries, bitwise-identical results.   */
  double grad_hx, grad_hy;
  /* Coefficients (NEXT-1, Alg 3 steps 28-32).  0: Alg 4 every epoch, P kept implicit
     (the hot path).  1: every epoch also Algs 5-7 (readings R15-R17 of DESIGN.md) and
     the NA-Hutch++ estimate of each of the four candidates (A9 every epoch); P = the candidate
     with the smallest unclamped estimate (lowest algorithm number on ties), kept explicit
     (t x n_cap) as the next epoch's P_prev.  oid_finalize then returns that P and
     oid_error_estimate the chosen candidate's estimate; oid_get field 14 logs the choices.
     Requires a single shard (row_begin = 0, row_end = m) and ell1, ell2 > 0.                  */
  int32_t coeff_mode;
  /* Epochs (NEXT-2).  0: one ingest block = one epoch (reading R4, the hot path).  1: the paper's
     buffer: every column is sketched, counted and copied into a device buffer
     D (m_loc x k in the data dtype, part of the workspace); an epoch over D's k columns runs
     whenever k are buffered, across block boundaries.  Not combined with coeff_mode = 1 or the
     gradient variant.  oid_error_estimate is available once the first epoch has run.           */
  int32_t epoch_mode;
  /* NEXT-4: a 3-D grid for the gradient variant.  grad_nz > 1: the fields live on grad_nx x
     grad_ny x grad_nz nodes (node (i, j, l) of field f at row f nx ny nz + (i ny + j) nz + l),
     three gradient components with spacings grad_hx, grad_hy, grad_hz (0: 1/(N-1)), augmented
     sketch of 4 ell rows ((d + 1) ell <= 2048).  0 or 1: the 2-D grid above.                    */
  int32_t grad_nz;
  /* Basis Gram (A9).  0: exact fp64 (DMMA) from the stored basis (the default).  1: A9Q - int8
     tensor cores from a second copy of the basis quantised by A7 to a 31-bit per-column fixed
     point (4 bytes per element, half the read, no DMMA bound; |dG_ij| <= 2^-27 (M_j ||a_i||_1 +
     M_i ||a_j||_1) + m 2^-54 M_i M_j; measured 2e-10 relative on C1 and
     C3).  Needs k1_mode = OID_K1_TC_FAST (the per-column exponents come from K1F), epoch_mode = 0
     and no gradient variant; otherwise the exact A9 runs.  The fast mode of bench.py.           */
  int32_t a9_mode;
  double grad_hz;
} oid_params;

typedef struct {
  int64_t n_obs;          /* columns ingested so far                                    */
  int64_t epochs;         /* non-empty ingest calls                                     */
  int64_t launches;       /* kernels launched by this context                          */
  int64_t k1_launches;    /* launches of the fused ingest kernel                        */
  double k1_ms;           /* summed CUDA-event time of K1 (profile = 1), launch stream   */
  double post_ms;         /* summed CUDA-event time of the post-pass (commit)           */
  double est_ms;          /* summed CUDA-event time of error estimates                  */
  uint32_t flags;         /* OR of OID_FLAG_* seen so far (read at this call; syncs)     */
  int32_t k1_mode_used;   /* oid_k1_mode actually used by the last ingest               */
  double a9_ms;           /* summed CUDA-event time of the basis-Gram kernel (A9, profile) */
  int64_t a9_launches;    /* timed basis-Gram launches                                   */
  int64_t admissions;     /* basis admissions so far (A6; each costs one A7 column copy)  */
  int64_t dirty_slots;    /* slots whose Gram rows estimates recomputed (A9), summed      */
  int64_t estimates;      /* estimates begun                                             */
  double lat_min_ms, lat_med_ms, lat_max_ms;  /* per-block ingest latency, K1 start to the
                             end of the commit (profile = 1; 0 when not measured)        */
} oid_stats_t;

/* Size in bytes of the device workspace oid_init needs for these parameters.
   Errors: OID_EINVAL on invalid parameters. */
oid_status oid_workspace_query(const oid_params* p, size_t* bytes);

/* Create a context.  workspace: caller-owned device buffer of >= oid_workspace_query bytes
   (256-byte aligned), kept alive and untouched until oid_destroy.  stream: used for the
   initial clears.  Errors: OID_EINVAL, OID_ESHAPE (workspace too small), OID_ECUDA. */
oid_status oid_init(const oid_params* p, void* workspace, size_t bytes, void* stream, oid_ctx* out);

/* Single-shard ingest of one block = one epoch (R4): Alg 3 steps 9-27 for ncols columns,
   then Alg 4.  X: device, m_loc x ncols, leading dimension ld >= m_loc, dtype p->dtype,
   read by kernels enqueued on `stream`; X must stay valid until those kernels complete
   (the caller may record an event after this call).  Global column indices continue from
   the previous call (0-based).  ncols == 0 is a no-op.
   Errors: OID_ESHAPE (ncols > b_max, ld < m_loc, n_obs + ncols > n_cap), OID_ECUDA. */
oid_status oid_ingest_block(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream);

/* Multi-shard ingest, first half: K1 on this shard's rows.  Afterwards the partial buffer
   (oid_partials, which = 0) holds [Y (ell x ncols, col-major); n (ncols)] for this shard's rows;
   the caller sums it over shards in place before oid_ingest_commit. */
oid_status oid_ingest_sketch(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream);

/* Multi-shard ingest, second half: Gram, ridge scores, selection, basis copy of this shard's
   rows of the admitted columns (reads X again, admitted columns only), Alg 4.
   Same X, ld, ncols as the preceding oid_ingest_sketch.  Errors: OID_ESTATE if no sketch. */
oid_status oid_ingest_commit(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream);

/* Device pointer and element count (fp64) of a partial buffer to be summed over shards:
   which = 0: ingest partials ((ell + 1) * ncols of the last sketch);
   which = 1: basis-Gram partials (k * k) of the last oid_estimate_begin;
   which = 2: gradient variant, the gradient sketches of the last sketch: d buffers
              [Y_p (ell x ncols); n_p (ncols)], buffer p - 1 at offset (p - 1)(ell + 1) b_max
              (count = d (ell + 1) b_max: summing the whole range is allowed, entries past
              (ell + 1) ncols of a buffer are never read);
   which = 3: gradient variant, Omega G^p Omega^T (d ell x ell, p = 1..d) after oid_gradient_ogo.
   Errors: OID_EINVAL (unknown which, or 2/3 without the gradient variant). */
oid_status oid_partials(oid_ctx ctx, int32_t which, double** dev_ptr, int64_t* count);

/* Sharded gradient variant (P:684 stencils G^p X across row slabs, SURVEY 8(e) route (ii)):
   oid_ingest_sketch with the block's stencil halos.  X_lo: device, rows_lo x ncols (ld_lo >=
   rows_lo), the global rows [row_begin - rows_lo, row_begin) of the same block; X_hi: rows_hi x
   ncols (ld_hi >= rows_hi), the rows [row_end, row_end + rows_hi); dtype p->dtype; both read by
   kernels on `stream` and borrowed like X.  rows_lo / rows_hi = oid_grad_halo (grad_ny grad_nz
   rows, clipped at 0 and m; 0 without the gradient variant, when the pointers may be NULL).
   oid_ingest_sketch = this call with NULL halos.  Errors: those of oid_ingest_sketch, and
   OID_EINVAL when a needed halo is NULL or its ld too small. */
oid_status oid_ingest_sketch_halo(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, const void* X_lo,
                                  int64_t ld_lo, const void* X_hi, int64_t ld_hi, void* stream);
oid_status oid_grad_halo(oid_ctx ctx, int64_t* rows_lo, int64_t* rows_hi);

/* NA-Hutch++ estimate of ||A_obs - A_J P||_F for the current J and P (Alg 8).
   _begin computes this shard's part of G = A_J^T A_J; after the caller's reduction
   _end evaluates eq:NAhutchPP_2nd_term and eq:NAhutchPP_expansion.
   out_dev: device array of 8 doubles receiving
     [0] ||E||^2 estimate (unclamped), [1] T = estimate of tr(A (A_J P)^T), [2] tr(G P P^T),
     [3] ||A_obs||_F^2, [4] ||E||_F estimate (clamped at 0), [5] relative estimate,
     [6] flags (as double), [7] kappa(S_J).  Errors: OID_ESTATE before the first block.
   Ordering: the estimate reads the state of the last committed ingest (whatever stream it ran
   on); its internal work runs on library streams ordered by events after that commit, and
   `stream` (which may differ from the ingest stream and overlap the next ingest) waits for the
   partials at the end of _begin and for the whole estimate at the end of _end, so out_dev is
   written in `stream` order.  The partials (oid_partials 1) alternate between two buffers by
   estimate parity: reduce them between _begin and _end of the same estimate. */
oid_status oid_estimate_begin(oid_ctx ctx, void* stream);
oid_status oid_estimate_end(oid_ctx ctx, double* out_dev, void* stream);

/* Single-shard convenience: begin + end, then copies the 8 values to host memory out_host
   (synchronizes `stream`). */
oid_status oid_error_estimate(oid_ctx ctx, double* out_host, void* stream);

/* Final outputs: J (k int64 to host memory, slot order, -1 = vacant) and
   P (k x n_obs, column-major, ld = k) to device memory (P_on_device = 1) or host memory
   (0); basis_dev (may be NULL): device m_loc x k buffer (ld = m_loc, dtype) receiving the
   basis slab A_J (vacant columns zero).  Synchronizes `stream`.  The context stays usable. */
oid_status oid_finalize(oid_ctx ctx, int64_t* J_host, double* P, int32_t P_on_device,
                        void* basis_dev, void* stream);

/* Gradient variant (grad_nfields > 0), after an ingest and with no sketch pending:
   oid_gradient_gcv       sketched GCV(mu) of eq:GCV_COmega for the current basis,
                          computed on the device (Omega G^p Omega^T is regenerated once per
                          context); synchronizes `stream`.
   oid_gradient_coefficients  P(mu) = argmin ||Omega(A_J X - A)||^2 + mu sum_p ||Omega G^p (A_J X - A)||^2
                          (eq:opt_grad_fullsketch), k x n_obs column-major (ld k) into
                          device memory P_dev (vacant-slot rows zero); asynchronous.
   oid_gradient_finalize  mu* by golden-section search of GCV over log10(mu) in [lo, hi] to
                          tolerance tol (the paper: [-3, 3]); P(mu*) into P_dev when not
                          NULL; synchronizes.
   oid_gradient_ogo       this shard's part of Omega G^p Omega^T, into oid_partials(3);
                          sharded contexts call it once and sum the partials over the shards
                          before the first GCV (single shard: optional, done on first use).
   Errors: OID_ESTATE (variant off, nothing ingested, sketch pending; sharded GCV before
   oid_gradient_ogo), OID_EINVAL (mu < 0, lo >= hi, tol <= 0). */
oid_status oid_gradient_ogo(oid_ctx ctx, void* stream);
oid_status oid_gradient_gcv(oid_ctx ctx, double mu, double* gcv, void* stream);
oid_status oid_gradient_coefficients(oid_ctx ctx, double mu, double* P_dev, void* stream);
oid_status oid_gradient_finalize(oid_ctx ctx, double lo, double hi, double tol, double* mu_star, double* P_dev,
                                 void* stream);

/* Copy internal state to host memory (synchronizes `stream`), for tests and diagnostics.
   field: 0 J (k int64), 1 tau_old (k), 2 S (ell x n_obs), 3 Gram (ell x ell; 3 ell x 3 ell with
          the gradient variant),
          4 scalars [frob2, lambda_eff, E_k, shift, trace, dmax, min_margin, kappa],
          5 last scores (k + ncols: basis slots then candidates), 6 eigenvalues of Gram (ell; on the
          tridiagonal fast path only the k largest, entries 0..k-1, are computed - the rest are
          stale),
          7 last ingest partials ((ell+1) * ncols), 8 S_J^+ (k x ell),
          9 Jacobi rotation counts per sweep (3 x 48 int32: Gram, S_J, NA-Hutch++ core),
          10 K1 role timestamps of CTA 0 (10 x 4096 int64 clock64; recorded when the environment
             variable OID_K1_DEBUG=1 was set at oid_init),
          11 basis Gram G = A_J^T A_J of the last estimate (k x k; rows/columns of vacant
             slots zero),
          12 tridiagonalisation phase timestamps of the last ingest (4 x 1024 int64 clock64 of
             cluster CTA 0; recorded with OID_K1_DEBUG=1),
          14 coefficient choices (coeff_mode = 1): per epoch [epoch, q*, e2 of Algs 4, 5, 6, 7]
             (epochs x 6 doubles),
          15 K1F exponent state (OID_K1_TC_FAST): 256 units x 32 columns of observed maximum
             biased exponents (INT_MIN before the first block), then 8 int32 counters summed over
             launches: [first-tile raises, mid-stream raises (accumulator drains), reruns of a
             unit after a precision loss, int32-overflow epochs, 0, 0, 0, 0]. */
oid_status oid_get(oid_ctx ctx, int32_t field, void* host_dst, size_t bytes, void* stream);

/* Counters and CUDA-event timings (synchronizes the context's recorded events).
   oid_stats_reset clears the launch counters and the recorded timings. */
oid_status oid_stats(oid_ctx ctx, oid_stats_t* out);

/* Run report (A12; the outputs of P:357 and the error metrics of P:729) as one JSON
   object written to host memory buf (cap bytes, NUL-terminated): totals (n_obs, epochs,
   estimates, OR of the OID_FLAG_* bits, admissions, dirty slots), "epoch_log" (per epoch: epoch,
   n_obs, admissions, evictions, lambda_eff, E_k, the minimum decision margin of reading R14,
   kappa(S_J) of Alg 4) and "estimate_log" (per estimate: the epoch it follows, the unclamped
   ||E||^2 estimate e2, T, tr(G P P^T), ||A_obs||^2, the relative estimate, flags, kappa(S_J)).
   At most n_cap rows each.  *needed (may be NULL) receives the size including the NUL.
   Synchronizes `stream` and the library's streams.  Errors: OID_ESHAPE if cap is too small. */
oid_status oid_report(oid_ctx ctx, char* buf, size_t cap, size_t* needed, void* stream);
oid_status oid_stats_reset(oid_ctx ctx);

/* Host-only: the Gauss-16 sketch-entry table (reading R2): for a 4-bit Philox draw n,
   Omega = s * (q[n] + 1/2), q[n] integer in [-111, 110]; needs no GPU.
   Errors: OID_EINVAL on NULL pointers. */
oid_status oid_sketch_table(int32_t q[16], double* scale);

/* Diagnostics and tuning knobs (environment variables read at oid_init; none changes a result:
   every one only moves work between streams / SMs or records timings, and the tests compare
   the affected paths bitwise or against the oracle):
     OID_K1_DEBUG=1     record K1 role timestamps (oid_get field 10) and the tridiagonalisation
                        phase timestamps (field 12)
     OID_K1_EXP=bits    K1 ablations for timing only (1: no Philox, 2: no digit conversion; the
                        pair kernel: 4 no TMEM store, 32 no fence, 64 no dp4a, 128 no conversion,
                        256 no MMA, 512 no TMA) - results are WRONG with any bit set
     OID_K1_FREE=n      SMs the persistent K1 grid leaves free (default 2: the estimate's single-SM
                        core SVD and side kernels hold no K1 CTA back)
     OID_A9Q_SERIAL=1   K1 waits for the previous A9Q instead of sharing the SMs with it
     OID_A9Q_CL=n       A9Q launched as at most n 16-CTA clusters (default 6, two GPCs stay free
                        for the A4 and A8 tridiagonalisation clusters)
     OID_A9_DEFER=0     single-shard contexts launch an estimate's basis Gram in oid_estimate_begin
                        (default: after the next block's K1, or when anything needs it)
     OID_TIMELINE=1     per-stream timeline marks (oid_get field 13)
     OID_NO_SIDE=1      run every kernel on the caller's stream (race check of the event graph)
     OID_JACOBI_COLD=1  A4/A5 always by cold-started Jacobi (reference path for tests)
     OID_SIDE_PRIO, OID_SIDE2_PRIO, OID_GS_PRIO   stream priorities of the side / A9 streams
     OID_BG_FREE, OID_BG_WAVES, OID_BG_CLUSTER, OID_BG_SMEM, OID_GS_GATE   A9 launch shape
                        (SMs left free, waves per SM, cluster size, ring KB, gate behind A8) */
void oid_destroy(oid_ctx ctx);
const char* oid_last_error(oid_ctx ctx);   /* ctx == NULL: last oid_init failure (this thread) */
const char* oid_version(void);

#ifdef __cplusplus
}
#endif
#endif /* OID_H_ */
