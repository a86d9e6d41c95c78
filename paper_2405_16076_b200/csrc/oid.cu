// liboid: host engine and C ABI (include/oid.h) of the B200 ingest hot path of the
// single-pass randomized ID (arxiv 2405.16076, Alg 3 / Alg 4 / Alg 8).
//
// The caller owns all device memory (one workspace buffer, sized by oid_workspace_query);
// every step runs in the kernels below on the caller's stream; the host never waits during
// ingest.  See DESIGN.md sections 1 and 6 for the kernel list and the data layout.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: named ranges per API call for nsys / ncu --nvtx

#include "../../include/oid.h"
#include "common.cuh"
#include "dense.cuh"
#include "k1_simt.cuh"
#include "k1_tc.cuh"
#include "k1_pair.cuh"
#include "k1_fast.cuh"
#include "gram_q.cuh"
#include "coeff.cuh"
#include "gram_tc.cuh"
#include "grad.cuh"
#include "path.cuh"
#include "tri.cuh"

using namespace oid;

namespace {
// one NVTX range per public call (the step structure in a profiler timeline)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

constexpr int kK1MaxCtas = 1024;
thread_local char g_init_err[512] = "no error";
constexpr int kGramChunks = 296;            // cp.async fallback kernel
constexpr size_t kGramPartBudget = size_t(1536) << 20;  // per-chunk A9 partials (TMA kernel)
inline int gram_tc_chunks(int t) {           // short CTAs (several waves) so higher-priority work interleaves
  const size_t per = static_cast<size_t>(t) * t * sizeof(double);
  return static_cast<int>(std::max<size_t>(kGramChunks, std::min<size_t>(148 * 32, kGramPartBudget / per)));
}
constexpr int kMaxSweeps = 48;
constexpr int kNumJacobiUses = 3;
constexpr int kSymMaxPairs = 65;   // ceil(2048 / 16) / 2 + 1
constexpr size_t kSmallSvdSmem = 200 * 1024;
constexpr int kCrossChunks = 64;    // row chunks of the NEXT-1 cross dots (fixed-order sum)

// ------------------------------------------------------------------ Gauss-16 table (reading R2)
// Inverse normal CDF (for the bin centroids of the 16-level law): Acklam's rational approximation refined by one Halley step on erfc.
double inv_norm_cdf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  double x;
  if (p < 0.02425) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - 0.02425) {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = std::sqrt(-2.0 * std::log(1.0 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  for (int it = 0; it < 2; ++it) {
    const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    const double u = e * std::sqrt(2.0 * M_PI) * std::exp(0.5 * x * x);
    x = x - u / (1.0 + 0.5 * x * u);
  }
  return x;
}

// Gauss-16 (reading R2): magnitudes m_k = round(56 c_k - 1/2) of the centroids c_k of the 8
// positive equiprobable N(0,1) bins; nibble n -> L(n) = (m_{n&7} + 1/2)(1 - 2(n >> 3)),
// q(n) = L(n) - 1/2 (int8), entry = s L(n), s = 1/sqrt(mean L^2).
void gauss16(int32_t m[8], int32_t q[16], double* scale) {
  const double inv_sqrt_2pi = 0.3989422804014327;
  auto phi = [&](double x) { return std::isfinite(x) ? inv_sqrt_2pi * std::exp(-0.5 * x * x) : 0.0; };
  for (int k = 0; k < 8; ++k) {
    const double a = k == 0 ? 0.0 : inv_norm_cdf((k + 8) / 16.0);
    const double b = k == 7 ? INFINITY : inv_norm_cdf((k + 9) / 16.0);
    m[k] = static_cast<int32_t>(std::lround(56.0 * 16.0 * (phi(a) - phi(b)) - 0.5));
  }
  double sum2 = 0.0;
  for (int n = 0; n < 16; ++n) {
    const double L = (m[n & 7] + 0.5) * (n >> 3 ? -1.0 : 1.0);
    q[n] = (n >> 3) ? -m[n & 7] - 1 : m[n & 7];
    sum2 += L * L;
  }
  *scale = 1.0 / std::sqrt(sum2 / 16.0);
}

// ------------------------------------------------------------------ workspace layout
struct Bump {
  size_t off = 0;
  size_t take(size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) & ~static_cast<size_t>(255);
    return o;
  }
};

struct Layout {
  size_t S, gram, Ypart, k1part, k1npart, gB, gV, mu, mu_sorted, Yc, Tsc, tau, scal, J, tau_old, admit, counts,
      flags, counters, C, SJ, sjB, sjV, sjsig, sjw, sjZ, Sjpinv, Pexp, AJP, G, Gsum, Gpart, cB, cV, csig, cw, cZ, M,
      X1, X2, Q1, Q2, R1, R2t, R3, PPt, est, tc, k1g, Cq, Fq, qadm, Gfull, dirty, dlist, jfro2, symU, symF, symTol, gT, td, te, Vh, tauv, gv, gp, gate, ldl, wyT, sjG, cG, cBt, cZ2, dbg, Jsnap, Dsnap, gcnt, Sg, YpG, GX, OGO, gH, gHV, gHs, gHw, gHZ, gHp, gR, gCm, gE, gLst, gLV, gLs, gLw, gLZ, gLp, gRhs, gscal, td2, te2, Vh2, tauv2, wyT2, ldl2, mu2, cum, elog, eslog, omega, trA, trW, Pcand, Pchosen, Pext, Rres, Gprev, gpH, gpV, gpMu, gpW, Gpinv, Xc, Dx, Dxp, Tm, cest, est_ch, est4, qlog, Jprev, olds, nold, qsel, Dpool, Dnorm, total;
};

int64_t m_local(const oid_params& p) { return p.row_end - p.row_begin; }
constexpr int kElogCols = 8;   // report row: epoch log [epoch, n_obs, admissions, evictions, lambda, E_k,
                               // min margin, kappa(S_J)]; estimate log [epoch, e2, T, gpp, frob2, est_rel,
                               // flags, kappa]
size_t dsize(const oid_params& p) { return p.dtype == OID_F64 ? 8 : 4; }

// A9Q (the basis Gram on int8 tensor cores from a quantised basis copy) needs K1F's per-column
// exponents of the block the admitted columns come from: the snapshot-block path only (not the
// t-column buffer, not the gradient variant); opt-in (a9_mode = 1, oid.h)
inline bool a9q_wanted(const oid_params& p) {
  return p.a9_mode == 1 && p.k1_mode == OID_K1_TC_FAST && p.epoch_mode == 0 && p.grad_nfields == 0;
}

Layout make_layout(const oid_params& p) {
  Layout L{};
  Bump b;
  const size_t d = sizeof(double);
  const size_t ell = p.ell, t = p.k, n = p.n_cap;
  // candidates per epoch: the block (b_max) or, with paper-literal epochs, the t buffered columns
  const size_t bm = p.epoch_mode == 1 ? std::max<size_t>(p.b_max, p.k) : p.b_max;
  const size_t ncb = 64;
  // augmented sketch [Y; Y_1; ..; Y_d] (A11): d = 2 gradient components on a 2-D grid, 3 in 3-D
  const size_t ga = p.grad_nfields > 0 ? (p.grad_nz > 1 ? 4 : 3) : 1;
  const size_t gd = ga - 1;
  const size_t ellg = ga * ell;                     // order of the Gram whose spectrum A4/A5 use
  L.S = b.take(ell * n * d);
  L.gram = b.take(ellg * ellg * d);
  L.Ypart = b.take((ell + 1) * p.b_max * d);
  L.k1part = b.take(static_cast<size_t>(kK1MaxCtas) * ell * ncb * d);
  L.k1npart = b.take(static_cast<size_t>(kK1MaxCtas) * ncb * d);
  L.gB = b.take(ellg * ellg * d);
  L.gV = b.take(ellg * ellg * d);
  L.mu = b.take(ellg * d);
  L.mu_sorted = b.take(ellg * d);
  L.Yc = b.take(ellg * (t + bm) * d);
  L.Tsc = b.take(ellg * (t + bm) * d);
  L.tau = b.take((t + bm) * d);
  L.scal = b.take(SC_COUNT * d);
  L.J = b.take(t * sizeof(int64_t));
  L.tau_old = b.take(t * d);
  L.admit = b.take(2 * (t + bm) * sizeof(int));
  L.counts = b.take(4 * sizeof(int));
  L.cum = b.take(4 * sizeof(unsigned long long));   // [admissions, dirty slots at estimates, estimates]
  L.elog = b.take(n * kElogCols * d);                 // per-epoch report rows (A12)
  L.eslog = b.take(n * kElogCols * d);                // per-estimate report rows (A12)
  L.flags = b.take(4 * sizeof(unsigned));
  L.counters = b.take(kNumJacobiUses * kMaxSweeps * sizeof(int));
  {
    // row-tiled basis C_blk[tile][slot][RL] (RL = 128 bytes of rows), padded to whole tiles
    const int64_t RL = 128 / static_cast<int64_t>(dsize(p));
    L.C = b.take(static_cast<size_t>((m_local(p) + RL - 1) / RL * RL) * t * dsize(p));
  }
  L.SJ = b.take(2 * ell * t * d);          // per epoch parity (the next A8 overlaps this estimate)
  L.sjB = b.take(ell * t * d);
  L.sjV = b.take(t * t * d);
  L.sjsig = b.take(t * d);
  L.sjw = b.take(t * d);
  L.sjZ = b.take(t * ell * d);
  L.Sjpinv = b.take(2 * t * ell * d);
  L.Pexp = b.take(t * n * d);
  L.AJP = b.take(ell * n * d);
  L.G = b.take(t * t * d);
  L.Gsum = b.take(2 * t * t * d);           // by estimate parity (A9 stream vs estimate tail)
  L.Gpart = b.take(static_cast<size_t>(gram_tc_chunks(static_cast<int>(t)) + 64) * t * t * d);   // + 64 segment sums
  const size_t l1 = p.ell1, l2 = p.ell2, l3 = p.ell3;
  L.cB = b.take(std::max<size_t>(1, l1 * l2) * d);
  L.cV = b.take(std::max<size_t>(1, l2 * l2) * d);
  L.csig = b.take(std::max<size_t>(1, l2) * d);
  L.cw = b.take(std::max<size_t>(1, l2) * d);
  L.cZ = b.take(std::max<size_t>(1, l2 * l1) * d);
  L.M = b.take(std::max<size_t>(1, l2 * l1) * d);
  L.X1 = b.take(std::max<size_t>(1, l1 * t) * d);
  L.X2 = b.take(std::max<size_t>(1, l2 * t) * d);
  L.Q1 = b.take(std::max<size_t>(1, l2 * t) * d);
  L.Q2 = b.take(std::max<size_t>(1, l2 * t) * d);
  L.R1 = b.take(std::max<size_t>(1, l3 * l2) * d);
  L.R2t = b.take(std::max<size_t>(1, l3 * l1) * d);
  L.R3 = b.take(std::max<size_t>(1, l3 * l1) * d);
  L.PPt = b.take(t * t * d);
  L.est = b.take(8 * d);
  L.Gfull = b.take(t * t * d);
  L.dirty = b.take(t * sizeof(int));
  L.dlist = b.take(2 * t * sizeof(int));
  L.gcnt = b.take(8 * sizeof(int));          // [4 par + 2] = dirty count of estimate parity par
  L.jfro2 = b.take(kNumJacobiUses * d);
  L.symU = b.take(static_cast<size_t>(kSymMaxPairs) * kSymB * kSymB * d);
  L.symF = b.take(kSymMaxPairs * sizeof(int));
  L.symTol = b.take(kNumJacobiUses * d);
  L.gT = b.take(ellg * ellg * d);
  L.td = b.take(ellg * d);
  L.te = b.take(ellg * d);
  L.Vh = b.take(ellg * (ellg + 1) * d);   // leading dimension tri_ldv(n) <= n + 1
  L.tauv = b.take(ellg * d);
  L.gv = b.take((ellg + 1) * d);
  L.gp = b.take((ellg + 16) * d);
  L.gate = b.take(8 * sizeof(int));
  L.sjG = b.take(t * t * d);
  L.dbg = b.take((k1p::kDbgRows + 1) * k1tc::kDbgTiles * sizeof(long long));
  L.cBt = b.take(std::max<size_t>(1, l1 * l2) * d);
  L.cZ2 = b.take(std::max<size_t>(1, l1 * l2) * d);
  L.cG = b.take(std::max<size_t>(1, std::min(l1, l2) * std::min(l1, l2)) * d);
  L.ldl = b.take(2 * ellg * d);
  L.wyT = b.take(static_cast<size_t>(kMaxRefChunksG) * kRefChunk * kRefChunk * d);
  if (ellg > kTriMaxN && ellg <= kTriMaxG) {
    // panel reduction of Gram orders 512 < n <= 1024: working copy of the Gram and the panel's W
    L.trA = b.take(ellg * ellg * d);
    L.trW = b.take(ellg * kPanNb * d);
  }
  // second tridiagonal workspace: the Alg 4 SPD solve (side stream) runs beside A4 of the next block
  L.td2 = b.take(ell * d);
  L.te2 = b.take(ell * d);
  L.Vh2 = b.take(ell * (ell + 1) * d);
  L.tauv2 = b.take(ell * d);
  L.wyT2 = b.take(static_cast<size_t>(kMaxRefChunks) * kRefChunk * kRefChunk * d);
  L.ldl2 = b.take(2 * ell * d);
  L.mu2 = b.take(ell * d);
  L.Jsnap = b.take(2 * t * sizeof(int64_t));
  L.Dsnap = b.take(2 * t * sizeof(int));
  if (ga > 1) {
    // gradient variant (A11): S^p, their K1 outputs, G^p X, Omega G^p Omega^T, GCV / P(mu) scratch
    const size_t ml = static_cast<size_t>(m_local(p));
    L.Sg = b.take(gd * ell * n * d);   // S^p = Omega G^p A_obs, p = 1..d
    L.YpG = b.take(std::max<size_t>(2, gd) * (ell + 1) * bm * d);
    L.GX = b.take(std::max<size_t>(2, gd) * ml * bm * d);
    L.OGO = b.take(gd * ell * ell * d);
    L.gH = b.take(t * t * d);
    L.gHV = b.take(t * t * d);
    L.gHs = b.take(t * d);
    L.gHw = b.take(t * d);
    L.gHZ = b.take(t * t * d);
    L.gHp = b.take(t * t * d);
    L.gR = b.take(ell * t * d);
    L.gCm = b.take(ell * ell * d);
    L.gE = b.take(ell * n * d);
    L.gLst = b.take(ga * ell * t * d);
    L.gLV = b.take(t * t * d);
    L.gLs = b.take(t * d);
    L.gLw = b.take(t * d);
    L.gLZ = b.take(ga * ell * t * d);
    L.gLp = b.take(t * ga * ell * d);
    L.gRhs = b.take(ga * ell * n * d);
    L.gscal = b.take(8 * d);
  }
  if (p.epoch_mode == 1) {   // NEXT-2: the buffer D (m_loc x t, data dtype) and its squared norms
    L.Dpool = b.take(static_cast<size_t>(m_local(p)) * t * dsize(p));
    L.Dnorm = b.take(t * d);
  }
  if (p.coeff_mode == 1) {
    // NEXT-1: candidates of Algs 5-7, the chosen P (= next P_prev), P_prev extended, a residual,
    // G_prev, G^+ and its eigen-decomposition, the cross Gram, cross dots and their chunk partials
    L.Pcand = b.take(3 * t * n * d);
    L.Pchosen = b.take(t * n * d);
    L.Pext = b.take(t * n * d);
    L.Rres = b.take(ell * n * d);
    L.Gprev = b.take(t * t * d);
    L.gpH = b.take(t * t * d);
    L.gpV = b.take(t * t * d);
    L.gpMu = b.take(t * d);
    L.gpW = b.take(t * d);
    L.Gpinv = b.take(t * t * d);
    L.Xc = b.take(t * t * d);
    L.Dx = b.take(t * t * d);
    L.Dxp = b.take(static_cast<size_t>(kCrossChunks) * t * t * d);
    L.Tm = b.take(t * t * d);
    L.cest = b.take(3 * 8 * d);
    L.est_ch = b.take(8 * d);
    L.est4 = b.take(8 * d);
    L.qlog = b.take(n * 6 * d);
    L.Jprev = b.take(t * sizeof(int64_t));
    L.olds = b.take(t * sizeof(int));
    L.nold = b.take(4 * sizeof(int));
    L.qsel = b.take(4 * sizeof(int));
  }
  if (a9q_wanted(p)) {   // A9Q: the quantised basis (4 digit planes per element) and its exponents
    L.Cq = b.take(a9q::qbasis_bytes(m_local(p), static_cast<int>(t)));
    L.Fq = b.take(t * sizeof(int));
    L.qadm = b.take((static_cast<size_t>(p.b_max) + t) * 4 * sizeof(int));   // (slot, column, C, -) per admission
  }
  if (p.omega_cache == 1) {   // omega_cache (NEXT-3): Philox words of ell x m_loc sketch entries
    // + 1 group: the last 64-row K1 tile may run one 32-row group past the shard (zero rows of X)
    const int64_t ng = (p.row_end + 31) / 32 - p.row_begin / 32 + 1;
    L.omega = b.take(static_cast<size_t>(ng) * ell * 16);
  }
  L.tc = b.take(std::max(std::max(k1tc_workspace_bytes(p.ell, p.b_max, m_local(p), p.dtype == OID_F64),
                                  k1p_workspace_bytes(p.ell, p.b_max, m_local(p), p.dtype == OID_F64)),
                         k1f_workspace_bytes()));
  L.k1g = b.take(static_cast<size_t>(k1f::kMaxUnits * 32 + 8) * sizeof(int));   // K1F exponent guesses + counters
  L.total = b.off;
  return L;
}

const char* validate(const oid_params* p) {
  if (!p) return "null params";
  if (p->m <= 0) return "m must be > 0";
  if (p->row_begin < 0 || p->row_end > p->m || p->row_begin >= p->row_end) return "need 0 <= row_begin < row_end <= m";
  if (p->k < 1) return "k must be >= 1";
  if (p->ell < 1 || p->ell > 1024) return "ell must be in [1, 1024]";
  if (p->k > p->ell) return "k must be <= ell";
  if (p->k > 416) return "k must be <= 416";
  if (p->b_max < 1 || p->b_max > 64) return "b_max must be in [1, 64]";
  if (p->n_cap < 1) return "n_cap must be >= 1";
  if (p->ell1 < 0 || p->ell2 < 0 || p->ell3 < 0 || p->ell1 + p->ell2 + p->ell3 != p->ell)
    return "ell1 + ell2 + ell3 must equal ell (all >= 0)";
  if (!(p->lambda >= 0.0 || p->lambda == -1.0 || p->lambda == -2.0)) return "lambda must be >= 0, -1 or -2";
  if (!(p->eps > 0.0) || !(p->delta > 0.0 && p->delta < 1.0) || !(p->c > 0.0)) return "need eps > 0, 0 < delta < 1, c > 0";
  if (p->dtype != OID_F32 && p->dtype != OID_F64) return "dtype must be OID_F32 or OID_F64";
  if (p->k1_mode < 0 || p->k1_mode > 4) return "bad k1_mode";
  if (p->m / 32 >= (int64_t(1) << 32)) return "m too large for the 32-bit Philox row counter";
  if (p->grad_nfields < 0) return "grad_nfields must be >= 0";
  if (p->omega_cache != 0 && p->omega_cache != 1) return "omega_cache must be 0 or 1";
  if (p->coeff_mode != 0 && p->coeff_mode != 1) return "coeff_mode must be 0 or 1";
  if (p->coeff_mode == 1 && (p->row_begin != 0 || p->row_end != p->m))
    return "coeff_mode = 1 needs a single shard (row_begin = 0, row_end = m)";
  if (p->coeff_mode == 1 && (p->ell1 <= 0 || p->ell2 <= 0)) return "coeff_mode = 1 needs ell1, ell2 > 0";
  if (p->coeff_mode == 1 && p->grad_nfields > 0) return "coeff_mode = 1 is not combined with the gradient variant";
  if (p->epoch_mode != 0 && p->epoch_mode != 1) return "epoch_mode must be 0 or 1";
  if (p->epoch_mode == 1 && (p->coeff_mode != 0 || p->grad_nfields > 0))
    return "epoch_mode = 1 (t-column epochs) is not combined with coeff_mode = 1 or the gradient variant";
  if (p->grad_nfields > 0) {
    const int64_t nz = p->grad_nz > 1 ? p->grad_nz : 1;
    if (p->grad_nz < 0) return "gradient variant: grad_nz must be >= 0 (0 or 1: a 2-D grid)";
    if (p->grad_nx < 1 || p->grad_ny < 1 || int64_t(p->grad_nfields) * p->grad_nx * p->grad_ny * nz != p->m)
      return "gradient variant: grad_nfields * grad_nx * grad_ny (* grad_nz) must equal m";
    if (!(p->grad_hz >= 0.0)) return "gradient variant: grad_hz must be >= 0";
    if ((p->grad_nz > 1 ? 4 : 3) * p->ell > 2048) return "gradient variant: (d + 1) ell must be <= 2048";
    if (!(p->grad_hx >= 0.0) || !(p->grad_hy >= 0.0)) return "gradient variant: spacings must be >= 0 (0 = 1/(N-1))";
  }
  return nullptr;
}

}  // namespace

// ------------------------------------------------------------------ context
struct oid_ctx_s {
  oid_params p{};
  Layout L{};
  char* ws = nullptr;
  int64_t m_loc = 0;
  int t = 0;
  int num_sms = 0;
  int coop_max = 0;   // max co-resident CTAs of the Jacobi kernel
  int sym_coop_max = 0;
  int k1_ctas_per_sm = 1;
  double qscale = 0.0;
  int32_t qmag[8] = {0};
  double factor = 0.0;
  uint32_t key0 = 0, key1 = 0;
  int64_t n_obs = 0, epoch = 0;
  int pending_nc = -1;        // ncols of a sketch awaiting commit
  bool estimate_ready = false;
  int64_t launches = 0, k1_launches = 0;
  int k1_mode_used = 0;
  bool tc_ok = false;
  CUtensorMap bg_map{};       // basis slab C as a 2-D tensor {m_loc rows, t columns}
  bool cold_jacobi = false;   // diagnostics: OID_JACOBI_COLD=1 disables the warm starts
  bool k1_debug = false;      // diagnostics: OID_K1_DEBUG=1 records K1 role timestamps (oid_get 10)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_k1, ev_post, ev_est, ev_a9;
  // Side stream (highest priority) for the latency-bound chains that do not depend on the
  // HBM-bound kernels of the caller's stream: the Alg 4 factorisation (A8) runs beside the basis
  // copy (A7) and the basis-Gram-independent part of Alg 8 (A10) beside the basis Gram (A9).
  cudaStream_t side = nullptr;    // Alg 4 chains (A8)
  cudaStream_t side2 = nullptr;   // estimate factors and tail (A10)
  cudaStream_t side3 = nullptr;   // A4 spectrum -> lambda chain beside the Q^T application of A5
  cudaStream_t gs = nullptr;      // A9 basis Gram (and its dirty list / sums), lowest priority
  cudaEvent_t ev_gs_done = nullptr;                  // the last estimate's A9 partial sums are ready
  cudaEvent_t ev_gsum_free[2] = {nullptr, nullptr};  // the estimate tail scattered that parity's sums
  int n_est = 0, est_par = 0;  // estimates begun; parity of the current one
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_sj_done[2] = {nullptr, nullptr};   // A8 of an epoch parity finished (S_J, S_J^+ ready)
  cudaEvent_t ev_sj_free[2] = {nullptr, nullptr};   // the estimate finished reading that parity's S_J, S_J^+
  cudaEvent_t ev_snap_free[2] = {nullptr, nullptr}; // the estimate finished reading that parity's snapshot
  int last_est_tag = 0;       // admission tag of the last estimated epoch (dirty = newer tags)
  int ga = 1;                 // 3 with the gradient variant (augmented sketch), else 1
  GradGrid grid{};
  bool ogo_ready = false;     // Omega G^p Omega^T formed (gradient variant; sharded: this shard's
                              // partial until the caller's reduction of oid_partials(3))
  // stencil halos of the pending sketch (sharded gradient variant, oid_ingest_sketch_halo)
  const void* halo_lo = nullptr;
  const void* halo_hi = nullptr;
  int64_t halo_ld_lo = 0, halo_ld_hi = 0;
  // cross-stream hazards when estimates run on another stream than the ingests:
  // committed = end of a commit (its snapshot taken); gram_done = estimate's basis reads
  // finished; sj_j = Alg 4 chain finished reading J; est_done = end of an estimate.
  cudaEvent_t ev_committed = nullptr, ev_gram_done = nullptr, ev_sj_j = nullptr, ev_est_done = nullptr;
  int bg_free_sms = 0;        // SMs the A9 kernel leaves free (diagnostics: OID_BG_FREE)
  int bg_waves = 32;          // A9 CTAs per SM (short CTAs; diagnostics: OID_BG_WAVES)
  int bg_smem_kb = 200;       // A9 ring budget (diagnostics: OID_BG_SMEM)
  int bg_cluster = 1;         // A9 CTAs per cluster: whole groups of SMs retire together (OID_BG_CLUSTER)
  int gs_gate = 0;            // A9 also waits for the epoch's A8 chain (diagnostics: OID_GS_GATE)
  bool use_side = true;       // diagnostics: OID_NO_SIDE=1 runs everything on the caller's stream
  int k1_free_sms = 2;        // SMs the persistent K1 grid leaves to concurrent streams (OID_K1_FREE):
                              // the estimate's single-SM core SVD and side-stream kernels then hold no
                              // K1 CTA back (C3 pipelined: 623 vs 605 GB/s with 0)
  bool a9q = false;           // A9 on the quantised basis (K1F mode; off for good once a block skips K1F)
  bool a9q_serial = false;    // K1 waits for the last A9Q (diagnostics: OID_A9Q_SERIAL=1)
  int a9q_cl = 6;             // A9Q 16-CTA clusters at most (OID_A9Q_CL): two GPCs stay free for the
                              // A4 and A8 tridiagonalisation clusters (C3: 587 vs 547 GB/s with 7)
  bool a9_defer = false;      // single shard: A9 launched after the next block's K1 (OID_A9_DEFER=0: at once)
  bool a9_pending = false;    // an estimate's A9 queued but not launched
  int a9_gp = 0;
  cudaStream_t a9_gs = nullptr;
  cudaEvent_t ev_k1_end = nullptr;
  int last_nc = 0;            // columns of the last committed epoch (NEXT-1's P_prev extension)
  int dcount = 0;             // NEXT-2: columns buffered in D since the last epoch
  int64_t dbase = 0;          //         global index of D's first column
  bool timeline = false;      // diagnostics: OID_TIMELINE=1 records tagged events (oid_get 13)
  std::vector<std::pair<int, cudaEvent_t>> tl;
  char err[512] = {0};

  template <typename T> T* ptr(size_t off) const { return reinterpret_cast<T*>(ws + off); }
  double* d(size_t off) const { return ptr<double>(off); }

  oid_status fail(oid_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, sizeof(err), fmt, ap);
    va_end(ap);
    return s;
  }
};

#define CK(expr)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return ctx->fail(OID_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CKL()                                                                                      \
  do {                                                                                             \
    ++ctx->launches;                                                                               \
    cudaError_t e_ = cudaGetLastError();                                                           \
    if (e_ != cudaSuccess) return ctx->fail(OID_ECUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

namespace {

unsigned blocks_for(int64_t n, int threads = 256) { return static_cast<unsigned>((n + threads - 1) / threads); }

// C = alpha op(A) op(B) + beta C (column-major); skipped on the device when *gate == 0
oid_status gemm(oid_ctx ctx, cudaStream_t st, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                const int* gate = nullptr) {
  if (M <= 0 || N <= 0) return OID_OK;
  dim3 grid((M + 31) / 32, (N + 31) / 32);
  if (!ta && !tb) dgemm_kernel<false, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, gate);
  else if (!ta && tb) dgemm_kernel<false, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, gate);
  else if (ta && !tb) dgemm_kernel<true, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, gate);
  else dgemm_kernel<true, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, gate);
  CKL();
  return OID_OK;
}

// Block one-sided Jacobi SVD of B (L x n) in place.  warm = false: V <- I first (B = A);
// warm = true: V holds an orthogonal start and the caller has set B = A V.  sig = column norms.
oid_status jacobi(oid_ctx ctx, cudaStream_t st, double* B, int L, int n, double* V, double* sig, int use,
                  bool warm = false, const int* gate = nullptr) {
  if (n <= 0) return OID_OK;
  if (!warm) {
    set_identity_kernel<<<blocks_for(int64_t(n) * n), 256, 0, st>>>(V, n, gate);
    CKL();
  }
  int* counters = ctx->ptr<int>(ctx->L.counters) + use * kMaxSweeps;
  CK(cudaMemsetAsync(counters, 0, kMaxSweeps * sizeof(int), st));
  if (n > 1) {
    const bool w8 = (L + n) <= 1600;
    const int Wd = w8 ? 8 : 4;
    const size_t smem = sizeof(double) * 2 * Wd * (L + n);
    const void* fn = w8 ? reinterpret_cast<const void*>(bjacobi_kernel<8>) : reinterpret_cast<const void*>(bjacobi_kernel<4>);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * Wd, smem));
    const int nb = (n + Wd - 1) / Wd;
    const int npairs = (nb + (nb & 1)) / 2;
    const int grid = std::max(1, std::min(npairs, std::max(1, per_sm) * ctx->num_sms));
    double* fro2 = ctx->d(ctx->L.jfro2) + use;
    fro2_kernel<<<1, 256, 0, st>>>(B, int64_t(L) * n, fro2, gate);
    CKL();
    int Li = L, ni = n, ms = kMaxSweeps;
    // relative orthogonality target: well above the dot-product rounding level (~L eps)
    double tol = 4e-14 * std::max(1.0, std::sqrt(static_cast<double>(L) / 16.0));
    void* args[] = {&B, &Li, &ni, &V, &counters, &ms, &tol, &fro2, &gate};
    CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(32 * Wd), args, smem, st));
    CKL();
  }
  col_norms_kernel<<<n, 256, 0, st>>>(B, L, n, sig, gate);
  CKL();
  return OID_OK;
}

// pinv(A) for A = B_orig (L x n) given the Jacobi result (B, V, sig): out (n x L) = V diag(w) B^T
oid_status pinv_assemble(oid_ctx ctx, cudaStream_t st, const double* B, int L, int n, const double* V,
                         const double* sig, double* w, double* Z, double* out, double* kappa, unsigned flagbit,
                         const int* gate = nullptr) {
  if (n <= 0 || L <= 0) return OID_OK;
  pinv_weights_kernel<<<1, 256, 0, st>>>(sig, n, 1e-12, w, kappa, flagbit ? ctx->ptr<unsigned>(ctx->L.flags) : nullptr,
                                         flagbit, gate);
  CKL();
  scale_transpose_kernel<<<blocks_for(int64_t(L) * n), 256, 0, st>>>(B, L, n, w, Z, gate);
  CKL();
  return gemm(ctx, st, false, false, n, L, n, 1.0, V, n, Z, n, 0.0, out, n, gate);
}

// X = A^-1 R for a symmetric positive definite n x n A (overwritten) by the cluster
// tridiagonalisation when kappa(A) <= kmax2 (gate[0] set on the device); otherwise gate[1] is set
// and nothing is written (the caller's pseudo-inverse fallback runs).  n <= kTriMaxN.
oid_status spd_solve(oid_ctx ctx, cudaStream_t st, const double* A, int n, const double* R, int64_t ldr, bool in_t,
                     int nrhs, double* X, int64_t ldx, bool out_t, double kmax2, int* gate, double* kappa_out) {
  const Layout& L = ctx->L;   // second tridiagonal workspace (td2 ...)
  const size_t smem = sizeof(double) * static_cast<size_t>(n) * tri_rows(n);
  tridiag_cluster_kernel<<<kTriCtas, 256, smem, st>>>(A, n, n, ctx->d(L.td2), ctx->d(L.te2), ctx->d(L.Vh2), tri_ldv(n), ctx->d(L.tauv2),
                                                      nullptr, ctx->d(L.wyT2));
  CKL();
  // the SPD gate needs only the extreme eigenvalues
  multisect_kernel<<<1, 64, sizeof(double) * multisect_smem_doubles(n), st>>>(ctx->d(L.td2), ctx->d(L.te2), n,
                                                                            ctx->d(L.mu2), 1, 1);
  CKL();
  spd_gate_kernel<<<1, 32, 0, st>>>(ctx->d(L.mu2), n, kmax2, ctx->d(L.td2), ctx->d(L.te2), ctx->d(L.ldl2), gate,
                                    kappa_out);
  CKL();
  tri_solve_kernel<<<nrhs, 256, sizeof(double) * kQStages * kRefChunk * tri_ldv(n), st>>>(R, ldr, in_t ? 1 : 0, n, nrhs, ctx->d(L.Vh2), ctx->d(L.wyT2), ctx->d(L.ldl2), gate, X, ldx,
                                         out_t ? 1 : 0);
  CKL();
  return OID_OK;
}

// Householder tridiagonalisation of the Gram (order 512 < n <= kTriMaxG) into (td, te, Vh, tauv,
// wyT): panels of kPanNb columns (tridiag_panel_kernel + the two-GEMM trailing update) down to
// the last 512 columns, which the register-resident cluster kernel finishes (tri.cuh).
oid_status tridiag_big(oid_ctx ctx, cudaStream_t st, int n, long long* dbg) {
  const Layout& L = ctx->L;
  const int ldv = tri_ldv(n);
  double* A = ctx->d(L.trA);
  double* Vh = ctx->d(L.Vh);
  double* Wp = ctx->d(L.trW);
  CK(cudaMemcpyAsync(A, ctx->d(L.gram), sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(Vh, 0, sizeof(double) * static_cast<size_t>(ldv) * n, st));   // rows no reflector writes
  const int n0 = n - kTriMaxN;
  for (int k0 = 0; k0 < n0; k0 += kPanNb) {
    const int nb = std::min(kPanNb, n0 - k0);
    tridiag_panel_kernel<<<kTriCtas, 256, kPanSmem, st>>>(A, n, k0, nb, ctx->d(L.td), ctx->d(L.te), Vh, ldv,
                                                          ctx->d(L.tauv), Wp);
    CKL();
    // A(k1:, k1:) -= V W^T + W V^T over the panel's reflectors (k1 = k0 + nb)
    const int k1 = k0 + nb, m = n - k1;
    double* C = A + k1 + static_cast<int64_t>(k1) * n;
    const double* V = Vh + k1 + static_cast<int64_t>(k0) * ldv;
    oid_status s = gemm(ctx, st, false, true, m, m, nb, -1.0, V, ldv, Wp + k1, n, 1.0, C, n);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, false, true, m, m, nb, -1.0, Wp + k1, n, V, ldv, 1.0, C, n);
    if (s != OID_OK) return s;
  }
  const size_t smem = sizeof(double) * static_cast<size_t>(kTriMaxN) * tri_rows(kTriMaxN);
  tridiag_cluster_kernel<<<kTriCtas, 256, smem, st>>>(A + n0 + static_cast<int64_t>(n0) * n, n, kTriMaxN, ctx->d(L.td) + n0,
                                                      ctx->d(L.te) + n0, Vh + n0 + static_cast<int64_t>(n0) * ldv, ldv,
                                                      ctx->d(L.tauv) + n0, dbg, nullptr);
  CKL();
  wy_t_kernel<<<(n - 2 + kRefChunk - 1) / kRefChunk, 256, 0, st>>>(Vh, ctx->d(L.tauv), n, ctx->d(L.wyT));
  CKL();
  return OID_OK;
}

// Symmetric eigen-decomposition by two-sided block Jacobi (sym_bjacobi_kernel): H (n x n) is
// overwritten by (numerically) diag(mu); V holds the eigenvectors.  warm = true: the caller set
// H = V0^T A V0 and V = V0.  mu receives diag(H).
oid_status sym_eig(oid_ctx ctx, cudaStream_t st, double* H, int n, double* V, double* mu, int use, bool warm,
                   const int* gate = nullptr) {
  if (n <= 0) return OID_OK;
  if (!warm) {
    set_identity_kernel<<<blocks_for(int64_t(n) * n), 256, 0, st>>>(V, n);
    CKL();
  }
  int* counters = ctx->ptr<int>(ctx->L.counters) + use * kMaxSweeps;
  CK(cudaMemsetAsync(counters, 0, kMaxSweeps * sizeof(int), st));
  double* tolp = ctx->d(ctx->L.symTol) + use;
  frob_scale_kernel<<<1, 256, 0, st>>>(H, int64_t(n) * n, 1e-15, tolp, gate);
  CKL();
  if (n > 1) {
    const int nb = (n + kSymW - 1) / kSymW, nbb = nb + (nb & 1), npairs = nbb / 2;
    const int work = npairs * (npairs + 1) / 2 + npairs * ((n + kSymB - 1) / kSymB);
    const int grid = std::max(1, std::min(work, ctx->sym_coop_max));
    double* Ub = ctx->d(ctx->L.symU);
    int* fl = ctx->ptr<int>(ctx->L.symF);
    int ni = n, ms = kMaxSweeps;
    double tol = 1e-14;
    void* args[] = {&H, &V, &ni, &Ub, &fl, &counters, &ms, &tol, &tolp, &gate};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(sym_bjacobi_kernel), dim3(grid), dim3(256), args, 0, st));
    CKL();
  }
  diag_kernel<<<blocks_for(n), 256, 0, st>>>(H, n, mu, gate);
  CKL();
  return OID_OK;
}


struct EvScope {
  oid_ctx ctx;
  cudaStream_t st;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* v;
  cudaEvent_t b = nullptr, e = nullptr;
  EvScope(oid_ctx c, cudaStream_t s, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* vec) : ctx(c), st(s), v(vec) {
    if (!ctx->p.profile) return;
    cudaEventCreate(&b);
    cudaEventCreate(&e);
    cudaEventRecord(b, st);
  }
  ~EvScope() {
    if (!ctx->p.profile) return;
    cudaEventRecord(e, st);
    v->emplace_back(b, e);
  }
};

// diagnostics timeline: tagged event on st (OID_TIMELINE=1)
void tl_mark(oid_ctx ctx, cudaStream_t st, int tag) {
  if (!ctx->timeline || ctx->tl.size() >= 4096) return;
  cudaEvent_t ev;
  if (cudaEventCreate(&ev) != cudaSuccess) return;
  cudaEventRecord(ev, st);
  ctx->tl.emplace_back(tag, ev);
}

// side stream waits for all work enqueued on st so far
oid_status fork_to(oid_ctx ctx, cudaStream_t st, cudaStream_t to) {
  if (!ctx->use_side) return OID_OK;
  CK(cudaEventRecord(ctx->ev_fork, st));
  CK(cudaStreamWaitEvent(to, ctx->ev_fork, 0));
  return OID_OK;
}
oid_status fork_side(oid_ctx ctx, cudaStream_t st) { return fork_to(ctx, st, ctx->side); }
// st waits for all work enqueued on the side stream so far
oid_status join_from(oid_ctx ctx, cudaStream_t st, cudaStream_t from) {
  if (!ctx->use_side) return OID_OK;
  CK(cudaEventRecord(ctx->ev_join, from));
  CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
  return OID_OK;
}
// st waits for all work enqueued on both side streams so far
oid_status join_side(oid_ctx ctx, cudaStream_t st) {
  oid_status s = join_from(ctx, st, ctx->side);
  return s != OID_OK ? s : join_from(ctx, st, ctx->side2);
}

template <typename T>
oid_status launch_k1_simt(oid_ctx ctx, cudaStream_t st, const T* X, int64_t ld, int nc, double* out) {
  const oid_params& p = ctx->p;
  const int ncb = nc <= 16 ? 16 : (nc <= 32 ? 32 : 64);
  const int rpt = ncb <= 32 ? 2 : 1;
  const int ysplit = (p.ell + 256 * rpt - 1) / (256 * rpt);
  const int64_t g_begin = p.row_begin / kGrp, g_end = (p.row_end + kGrp - 1) / kGrp;
  const int64_t ngroups = g_end - g_begin;
  int64_t want = std::max<int64_t>(1, (int64_t(ctx->num_sms) * ctx->k1_ctas_per_sm) / ysplit);
  want = std::min<int64_t>(want, std::min<int64_t>(ngroups, kK1MaxCtas));
  const int64_t per = (ngroups + want - 1) / want;
  const int gx = static_cast<int>((ngroups + per - 1) / per);
  dim3 grid(gx, ysplit);
  double* part = ctx->d(ctx->L.k1part);
  double* npart = ctx->d(ctx->L.k1npart);
  {
    EvScope ev(ctx, st, &ctx->ev_k1);
#define K1_LAUNCH(NCB, RPT)                                                                              \
  k1_simt_kernel<T, NCB, RPT><<<grid, kThreads, 0, st>>>(X, ld, nc, p.row_begin, p.row_end, g_begin, g_end, per, \
                                                         p.ell, ctx->key0, ctx->key1, part, npart)
    if (ncb == 16) K1_LAUNCH(16, 2);
    else if (ncb == 32) K1_LAUNCH(32, 2);
    else K1_LAUNCH(64, 1);
#undef K1_LAUNCH
    CKL();
    ++ctx->k1_launches;
  }
  const int64_t nout = int64_t(p.ell) * nc + nc;
  k1_reduce_kernel<<<blocks_for(nout), 256, 0, st>>>(part, npart, gx, ncb, p.ell, nc, ctx->qscale, out,
                                                    ctx->ptr<unsigned>(ctx->L.flags));
  CKL();
  ctx->k1_mode_used = OID_K1_SIMT_F64;
  return OID_OK;
}

// K1 on one block (X of dtype f64 / f32) into out = [Y (ell x nc); n (nc)]
oid_status sketch_one(oid_ctx ctx, const void* X, int64_t ld, int nc, cudaStream_t st, double* out, bool f64,
                      bool strict_mode, bool main_x = false) {
  const oid_params& p = ctx->p;
  const bool want_pair = p.k1_mode == OID_K1_TC_PAIR;
  const bool want_tc = (p.k1_mode == OID_K1_TC_INT8) || want_pair || p.k1_mode == OID_K1_TC_FAST ||
                       (p.k1_mode == OID_K1_AUTO && ctx->tc_ok);
  K1TcArgs a{};
  a.X = X; a.ld = ld; a.ncols = nc; a.row_begin = p.row_begin; a.row_end = p.row_end; a.ell = p.ell;
  a.key0 = ctx->key0; a.key1 = ctx->key1; a.scale = ctx->qscale; a.f64 = f64;
  a.ws = ctx->ws + ctx->L.tc; a.out = out; a.flags = ctx->ptr<unsigned>(ctx->L.flags);
  a.t0 = static_cast<uint32_t>(ctx->qmag[0]) | (static_cast<uint32_t>(ctx->qmag[1]) << 8) |
         (static_cast<uint32_t>(ctx->qmag[2]) << 16) | (static_cast<uint32_t>(ctx->qmag[3]) << 24);
  a.t1 = static_cast<uint32_t>(ctx->qmag[4]) | (static_cast<uint32_t>(ctx->qmag[5]) << 8) |
         (static_cast<uint32_t>(ctx->qmag[6]) << 16) | (static_cast<uint32_t>(ctx->qmag[7]) << 24);
  a.num_sms = std::max(2, ctx->num_sms - ctx->k1_free_sms);
  a.dbg = ctx->k1_debug ? ctx->ptr<long long>(ctx->L.dbg) : nullptr;
  a.omega = (p.omega_cache == 1 && strict_mode) ? reinterpret_cast<const uint4*>(ctx->ws + ctx->L.omega) : nullptr;
  // K1F (OID_K1_TC_FAST): the snapshot blocks themselves (its exponent guesses follow one data
  // stream); the gradient / Omega G Omega^T passes keep the exact kernel
  if (p.k1_mode == OID_K1_TC_FAST && main_x && ctx->tc_ok && k1f_call_ok(a)) {
    int nl = 0;
    cudaError_t e;
    {
      EvScope ev(ctx, st, &ctx->ev_k1);
      tl_mark(ctx, st, 1);
      e = k1f_launch(a, ctx->ptr<int>(ctx->L.k1g), st, &nl);
      tl_mark(ctx, st, 2);
    }
    ctx->launches += nl;
    ctx->k1_launches += 1;
    if (e != cudaSuccess) return ctx->fail(OID_ECUDA, "k1 fast: %s", cudaGetErrorString(e));
    ctx->k1_mode_used = OID_K1_TC_FAST;
    return OID_OK;
  }
  const bool tc_call = want_tc && ctx->tc_ok && (want_pair ? k1p_call_ok(a) : k1tc_call_ok(a));
  if (strict_mode && (p.k1_mode == OID_K1_TC_INT8 || want_pair) && !tc_call)
    return ctx->fail(OID_EINVAL, "tensor-core K1 unavailable for this device/shape/alignment");
  if (tc_call) {
    int nl = 0;
    cudaError_t e;
    {
      EvScope ev(ctx, st, &ctx->ev_k1);
      tl_mark(ctx, st, 1);
      e = want_pair ? k1p_launch(a, st, &nl) : k1tc_launch(a, st, &nl);
      tl_mark(ctx, st, 2);
    }
    ctx->launches += nl;
    ctx->k1_launches += 1;
    if (e != cudaSuccess) return ctx->fail(OID_ECUDA, "k1 tc: %s", cudaGetErrorString(e));
    ctx->k1_mode_used = want_pair ? OID_K1_TC_PAIR : OID_K1_TC_INT8;
    return OID_OK;
  }
  if (f64) return launch_k1_simt<double>(ctx, st, static_cast<const double*>(X), ld, nc, out);
  return launch_k1_simt<float>(ctx, st, static_cast<const float*>(X), ld, nc, out);
}

// A9 of the pending estimate: exact basis Gram (or A9Q) of parity ctx->a9_gp on the A9 stream, then
// the fixed-order sums; records ev_gram_done (the next basis copy waits for it) and ev_gs_done.
static oid_status launch_a9(oid_ctx ctx) {
  if (!ctx->a9_pending) return OID_OK;
  ctx->a9_pending = false;
  const Layout& L = ctx->L;
  const int t = ctx->t;
  const int gp = ctx->a9_gp;
  cudaStream_t gs = ctx->a9_gs;
  int* dl = ctx->ptr<int>(L.dlist) + static_cast<size_t>(gp) * t;
  int* gc = ctx->ptr<int>(L.gcnt) + 4 * gp;
  double* Gs = ctx->d(L.Gsum) + static_cast<size_t>(gp) * t * t;
  tl_mark(ctx, gs, 8);
  // A9: exact basis Gram G = A_J^T A_J, incremental: only the rows/columns of
  // slots admitted since the last estimate are recomputed, over this shard's rows.
  {
    const bool f64 = ctx->p.dtype == OID_F64;
    const int64_t RL = f64 ? 16 : 32;
    const int64_t ntiles = (ctx->m_loc + RL - 1) / RL;
    // many short CTAs (waves of num_sms - bg_free_sms): kernels of higher-priority streams (the next
    // block's K1 and post-pass, the side stream) are scheduled as they retire
    const int sms = std::max(1, ctx->num_sms - ctx->bg_free_sms);
    const int cl = ctx->bg_cluster;   // CTAs per cluster (1: plain launch)
    int want = std::min(gram_tc_chunks(t), sms * ctx->bg_waves);
    want = std::max(cl, want / cl * cl);
    int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, (ntiles + 7) / 8)));
    const int64_t per = (ntiles + grid - 1) / grid;
    grid = static_cast<int>((ntiles + per - 1) / per);
    grid = (grid + cl - 1) / cl * cl;   // CTAs past the last tile contribute zero partials
    const int nbox = (t + 255) / 256;
    const int stage_bytes = (nbox * std::min(t, 256) * 128 + 1023) / 1024 * 1024;
    const int nstage = std::max(2, std::min(bgtc::kMaxStages, (ctx->bg_smem_kb * 1024) / stage_bytes));
    const size_t smem = static_cast<size_t>(nstage) * stage_bytes + 1024;
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute la[1];
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(32 * (bgtc::kCW + 1));
    lc.dynamicSmemBytes = smem;
    lc.stream = gs;
    if (cl > 1) {
      la[0].id = cudaLaunchAttributeClusterDimension;
      la[0].val.clusterDim.x = cl;
      la[0].val.clusterDim.y = 1;
      la[0].val.clusterDim.z = 1;
      lc.attrs = la;
      lc.numAttrs = 1;
    }
    if (ctx->a9q) {
      // A9Q: (row-tile set, slot chunk) CTAs, one per SM, launched as 16-CTA clusters (at most 7,
      // so each occupies one GPC and at least one GPC stays free: the A4 tridiagonalisation's
      // 16-CTA cluster, which runs concurrently, can always be placed)
      const int nch = a9q::nchunks(t);
      const int64_t nt128 = (ctx->m_loc + a9q::kTR - 1) / a9q::kTR;
      int ncl = std::min(ctx->a9q_cl, (sms - 20) / 16);
      while (ncl > 0 && (16 * ncl) % nch != 0) --ncl;
      const bool clustered = ncl > 0 && (16 * ncl) / nch <= nt128;
      const int nr = clustered ? (16 * ncl) / nch
                               : static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((sms - 20) / nch, nt128)));
      grid = nr * nch;
      EvScope eva9(ctx, gs, &ctx->ev_a9);
      cudaLaunchConfig_t qc = {};
      cudaLaunchAttribute qa[1];
      qc.gridDim = dim3(grid);
      qc.blockDim = dim3(a9q::kThreads);
      qc.dynamicSmemBytes = a9q::smem_bytes();
      qc.stream = gs;
      if (clustered) {
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = 16;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
      }
      CK(cudaLaunchKernelEx(&qc, a9q::gram_q_kernel, static_cast<const uint8_t*>(ctx->ptr<uint8_t>(L.Cq)),
                            static_cast<const int*>(ctx->ptr<int>(L.Fq)), nt128, t, nr, static_cast<const int*>(dl),
                            static_cast<const int*>(gc), ctx->d(L.Gpart)));
      CKL();
    } else {
      EvScope eva9(ctx, gs, &ctx->ev_a9);
      if (f64)
        CK(cudaLaunchKernelEx(&lc, bgtc::basis_gram_tc_kernel<double>, ctx->bg_map, ntiles, t, per, nstage, stage_bytes,
                              nbox, static_cast<const int*>(dl), static_cast<const int*>(gc), ctx->d(L.Gpart)));
      else
        CK(cudaLaunchKernelEx(&lc, bgtc::basis_gram_tc_kernel<float>, ctx->bg_map, ntiles, t, per, nstage, stage_bytes,
                              nbox, static_cast<const int*>(dl), static_cast<const int*>(gc), ctx->d(L.Gpart)));
      CKL();
    }
    CK(cudaEventRecord(ctx->ev_gram_done, gs));
    tl_mark(ctx, gs, 9);
    // two-level fixed-order sum: up to 64 segment sums into the tail of Gpart, then one
    const int nseg = std::min(64, std::max(1, grid / 16));
    double* seg = ctx->d(L.Gpart) + static_cast<size_t>(grid) * t * t;
    sum_dirty_chunks_kernel<<<dim3(blocks_for(int64_t(t) * t), nseg), 256, 0, gs>>>(ctx->d(L.Gpart), grid, t, gc, seg);
    CKL();
    sum_dirty_chunks_kernel<<<dim3(blocks_for(int64_t(t) * t), 1), 256, 0, gs>>>(seg, nseg, t, gc, Gs);
    CKL();
  }

  CK(cudaEventRecord(ctx->ev_gs_done, gs));
  return OID_OK;
}

// rows of the stencil halo below (lo) / above this shard: an axis-0 neighbour is ny nz rows
// away and no stencil reaches further (grad.cuh); 0 at the ends of the row range
int64_t grad_halo_rows(oid_ctx ctx, bool lo) {
  if (ctx->ga == 1) return 0;
  const int64_t reach = static_cast<int64_t>(ctx->grid.ny) * ctx->grid.nz;
  return lo ? std::min<int64_t>(ctx->p.row_begin, reach) : std::min<int64_t>(ctx->p.m - ctx->p.row_end, reach);
}

oid_status do_sketch(oid_ctx ctx, const void* X, int64_t ld, int nc, cudaStream_t st) {
  const oid_params& p = ctx->p;
  const Layout& L = ctx->L;
  // diagnostics (OID_A9Q_SERIAL=1): K1 waits for the last A9Q instead of sharing the SMs with it
  // (measured: 482 vs 513 GB/s on C3, the overlap wins although each kernel stretches)
  if (ctx->a9q && ctx->a9q_serial && ctx->use_side) CK(cudaStreamWaitEvent(st, ctx->ev_gram_done, 0));
  oid_status s = sketch_one(ctx, X, ld, nc, st, ctx->d(L.Ypart), p.dtype == OID_F64, true, true);

  if (s != OID_OK || ctx->ga == 1) return s;
  // gradient variant (A11): G^p X by the axis-neighbour stencils, then K1 on each
  // (same Omega, so the three sketches stack into [Omega a; Omega G^1 a; Omega G^2 a])
  const int64_t m = ctx->m_loc;
  double* GX = ctx->d(L.GX);
  const int64_t gstride = m * p.b_max;
  const unsigned gb = static_cast<unsigned>(std::min<int64_t>(blocks_for(m * nc), 8 * ctx->num_sms));
  const int64_t hlo = grad_halo_rows(ctx, true);
  if (p.dtype == OID_F64)
    grad_stencil_kernel<double><<<gb, 256, 0, st>>>(static_cast<const double*>(X), ld, m, nc, ctx->grid, GX, gstride,
                                                    p.row_begin, static_cast<const double*>(ctx->halo_lo), ctx->halo_ld_lo,
                                                    hlo, static_cast<const double*>(ctx->halo_hi), ctx->halo_ld_hi);
  else
    grad_stencil_kernel<float><<<gb, 256, 0, st>>>(static_cast<const float*>(X), ld, m, nc, ctx->grid, GX, gstride,
                                                   p.row_begin, static_cast<const float*>(ctx->halo_lo), ctx->halo_ld_lo,
                                                   hlo, static_cast<const float*>(ctx->halo_hi), ctx->halo_ld_hi);
  CKL();
  for (int q = 0; q < ctx->ga - 1; ++q) {
    s = sketch_one(ctx, GX + q * gstride, m, nc, st, ctx->d(L.YpG) + static_cast<size_t>(q) * (p.ell + 1) * p.b_max, true,
                   false);
    if (s != OID_OK) return s;
  }
  return OID_OK;
}

oid_status coeff_argmin(oid_ctx ctx, cudaStream_t st);   // NEXT-1, after the extern "C" block

// One epoch of Alg 3 (steps 15-27 + Alg 4) over nc candidate columns X (ld), whose
// sketches are Ycand (ell x nc, ld ell), squared norms nrm and global indices base, base + 1, ...
// do_a3: the block mode, where the candidates are the block itself and A3 (S, Gram, ||A_obs||^2)
// runs here first; the t-column mode runs A3 per column segment itself (commit_tcols).
oid_status post_epoch(oid_ctx ctx, const void* X, int64_t ld, int nc, cudaStream_t st, const double* Ycand,
                      const double* nrm, int64_t base, bool do_a3) {
  const oid_params& p = ctx->p;
  const Layout& L = ctx->L;
  const int ell = p.ell, t = ctx->t;
  double* Yp = ctx->d(L.Ypart);
  double* scal = ctx->d(L.scal);
  EvScope ev(ctx, st, &ctx->ev_post);
  tl_mark(ctx, st, 3);
  oid_status s = OID_OK;
  const int ns = t + nc;
  const int ng = ctx->ga * ell;              // order of the (augmented) Gram
  const int frob_idx = ctx->ga > 1 ? SC_FROB2_AUG : SC_FROB2;
  if (ctx->ga == 1) {
    // A3: S <- [S, Y], SS^T += YY^T, ||A_obs||^2 += sum n_j
    if (do_a3) {
      gram_update_kernel<<<blocks_for(int64_t(ell) * ell), 256, 0, st>>>(Yp, Yp + static_cast<int64_t>(ell) * nc, ell, nc,
                                                                        ctx->d(L.gram), ctx->d(L.S), ctx->n_obs, scal);
      CKL();
    }
    // A4: spectrum of the Gram and lambda; A5: ridge scores
    gather_scored_kernel<<<blocks_for(int64_t(ell) * ns), 256, 0, st>>>(ctx->d(L.S), ctx->ptr<int64_t>(L.J), t, Ycand, nc,
                                                                        ell, ctx->d(L.Yc));
    CKL();
  } else {
    // A11: augmented sketch [Y; Y_1; ..; Y_d], its ((d+1) ell)^2 Gram and energy
    const int64_t ystride = static_cast<int64_t>(ell + 1) * p.b_max, sstride = static_cast<int64_t>(ell) * p.n_cap;
    gram_update_aug_kernel<<<blocks_for(int64_t(ng) * ng), 256, 0, st>>>(Yp, ctx->d(L.YpG), ystride, ctx->ga, ell, nc,
                                                                         ctx->d(L.gram), ctx->d(L.S), ctx->d(L.Sg), sstride,
                                                                         ctx->n_obs, scal);
    CKL();
    gather_scored_aug_kernel<<<blocks_for(int64_t(ng) * ns), 256, 0, st>>>(ctx->d(L.S), ctx->d(L.Sg), sstride,
                                                                           ctx->ptr<int64_t>(L.J), t, Yp, ctx->d(L.YpG),
                                                                           ystride, ctx->ga, nc, ell, ctx->d(L.Yc));
    CKL();
  }
  int* gate = ctx->ptr<int>(L.gate);
  // the deferred A9 of the last estimate (estimate_begin) starts once the work before this point is
  // done, i.e. after this block's K1: queued behind the tridiagonalisation below on the block
  // scheduler (the cluster kernel on the higher-priority stream is placed first and keeps its 16
  // SMs; the Gram then takes the rest), so the Gram overlaps the latency-bound A4-A6 chain
  auto launch_deferred_a9 = [&]() -> oid_status {
    if (!(ctx->a9_pending && ctx->use_side)) return OID_OK;
    CK(cudaEventRecord(ctx->ev_k1_end, st));
    CK(cudaStreamWaitEvent(ctx->a9_gs, ctx->ev_k1_end, 0));
    return launch_a9(ctx);
  };
  if (ng <= kTriMaxG && !ctx->cold_jacobi) {
    // tridiagonal fast path (tri.cuh); the eigenvector path below runs only when gate[1] is set
    long long* tdbg = ctx->k1_debug ? ctx->ptr<long long>(L.dbg) + k1p::kDbgRows * k1tc::kDbgTiles : nullptr;
    if (ng <= kTriMaxN) {
      const size_t smem = sizeof(double) * static_cast<size_t>(ng) * tri_rows(ng);
      // (event before the cluster launch: the Gram becomes ready together with the cluster kernel)
      s = launch_deferred_a9();
      if (s != OID_OK) return s;
      tridiag_cluster_kernel<<<kTriCtas, 256, smem, st>>>(ctx->d(L.gram), ng, ng, ctx->d(L.td), ctx->d(L.te), ctx->d(L.Vh),
                                                          tri_ldv(ng), ctx->d(L.tauv), tdbg,
                                                          ctx->d(L.wyT));   // the compact-WY T factors too
      CKL();
    } else {
      s = tridiag_big(ctx, st, ng, tdbg);
      if (s != OID_OK) return s;
    }
    tl_mark(ctx, st, 15);
    // the spectrum -> lambda -> LDL^T chain on side stream 3, beside z = Q^T y for all scored columns
    cudaStream_t s3 = ctx->use_side ? ctx->side3 : st;
    s = fork_to(ctx, st, s3);
    if (s != OID_OK) return s;
    // lambda needs E_k (the k largest) and mu_0 only
    const int nev = std::min(p.k, ng);
    multisect_kernel<<<(nev * 32 + 255) / 256, 256, sizeof(double) * multisect_smem_doubles(ng), s3>>>(
        ctx->d(L.td), ctx->d(L.te), ng, ctx->d(L.mu), nev, 0);
    CKL();
    lambda_sorted_kernel<<<1, 256, sizeof(double) * 3 * ng, s3>>>(ctx->d(L.mu), ng, p.k, ctx->d(L.gram), p.lambda, ell,
                                                                  scal, gate, ctx->d(L.td), ctx->d(L.te), ctx->d(L.ldl), 1,
                                                                  frob_idx);
    CKL();
    {
      const unsigned qg = (ns + kQV - 1) / kQV;
      const size_t ring = sizeof(double) * kRefChunk * tri_ldv(ng);   // one stage
      if (ng <= 512)
        tri_scores_multi_kernel<2, 256, kQStages><<<qg, 256, kQStages * ring, st>>>(
            ctx->d(L.Yc), ng, ns, ctx->d(L.Vh), ctx->d(L.wyT), ctx->d(L.ldl), gate, ctx->d(L.tau), ctx->d(L.Tsc));
      else if (ng <= 1024)
        tri_scores_multi_kernel<4, 256, kQStages><<<qg, 256, kQStages * ring, st>>>(
            ctx->d(L.Yc), ng, ns, ctx->d(L.Vh), ctx->d(L.wyT), ctx->d(L.ldl), gate, ctx->d(L.tau), ctx->d(L.Tsc));
      else   // n <= 2048: 512 threads, one ring stage (a stage is 128 KB)
        tri_scores_multi_kernel<4, 512, 1><<<qg, 512, ring, st>>>(
            ctx->d(L.Yc), ng, ns, ctx->d(L.Vh), ctx->d(L.wyT), ctx->d(L.ldl), gate, ctx->d(L.tau), ctx->d(L.Tsc));
      CKL();
    }
    s = join_from(ctx, st, s3);
    if (s != OID_OK) return s;
    tri_scores_chain_kernel<<<(ns + kQV - 1) / kQV, 128, sizeof(double) * (kQV + 2) * ng, st>>>(
        ctx->d(L.Tsc), ng, ns, ctx->d(L.ldl), gate, ctx->d(L.tau));
    CKL();
    tl_mark(ctx, st, 16);
    const int* g1 = gate + 1;
    s = gemm(ctx, st, false, false, ng, ng, ng, 1.0, ctx->d(L.gram), ng, ctx->d(L.gV), ng, 0.0, ctx->d(L.gT), ng, g1);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, true, false, ng, ng, ng, 1.0, ctx->d(L.gV), ng, ctx->d(L.gT), ng, 0.0, ctx->d(L.gB), ng, g1);
    if (s != OID_OK) return s;
    s = sym_eig(ctx, st, ctx->d(L.gB), ng, ctx->d(L.gV), ctx->d(L.mu), 0, true, g1);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, true, false, ng, ns, ng, 1.0, ctx->d(L.gV), ng, ctx->d(L.Yc), ng, 0.0, ctx->d(L.Tsc), ng, g1);
    if (s != OID_OK) return s;
    scores_kernel<<<ns, 256, 0, st>>>(ctx->d(L.Tsc), ctx->d(L.mu), ng, ns, scal, ctx->d(L.tau), g1);
    CKL();
  } else {
    // eigenvector path only: warm-started two-sided block Jacobi (gV starts as the identity)
    s = gemm(ctx, st, false, false, ng, ng, ng, 1.0, ctx->d(L.gram), ng, ctx->d(L.gV), ng, 0.0, ctx->d(L.gT), ng);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, true, false, ng, ng, ng, 1.0, ctx->d(L.gV), ng, ctx->d(L.gT), ng, 0.0, ctx->d(L.gB), ng);
    if (s != OID_OK) return s;
    s = sym_eig(ctx, st, ctx->d(L.gB), ng, ctx->d(L.gV), ctx->d(L.mu), 0, true);
    if (s != OID_OK) return s;
    lambda_kernel<<<1, 256, 0, st>>>(ctx->d(L.mu), ng, p.k, ctx->d(L.gram), p.lambda, ell, scal, ctx->d(L.mu_sorted),
                                     frob_idx);
    CKL();
    s = gemm(ctx, st, true, false, ng, ns, ng, 1.0, ctx->d(L.gV), ng, ctx->d(L.Yc), ng, 0.0, ctx->d(L.Tsc), ng);
    if (s != OID_OK) return s;
    scores_kernel<<<ns, 256, 0, st>>>(ctx->d(L.Tsc), ctx->d(L.mu), ng, ns, scal, ctx->d(L.tau), nullptr);
    CKL();
  }
  // A6: selection / replacement; the previous block's Alg 4 chain reads J first
  tl_mark(ctx, st, 4);
  if (p.coeff_mode == 1)   // NEXT-1: J_prev of Algs 6 and 7
    CK(cudaMemcpyAsync(ctx->ws + L.Jprev, ctx->ws + L.J, sizeof(int64_t) * t, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamWaitEvent(st, ctx->ev_sj_j, 0));
  select_kernel<<<1, 256, 0, st>>>(ctx->ptr<int64_t>(L.J), ctx->d(L.tau_old), ctx->d(L.tau), nrm, t, nc,
                                  ctx->factor, static_cast<uint32_t>(ctx->epoch), base, ctx->key0, ctx->key1,
                                  ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), scal, ctx->ptr<int>(L.dirty),
                                  static_cast<int>(ctx->epoch + 1), ctx->ptr<unsigned long long>(L.cum),
                                  ctx->d(L.elog) + static_cast<size_t>(ctx->epoch) * kElogCols);
  CKL();
  // A8 runs on the side stream, beside the basis copy
  s = fork_side(ctx, st);
  if (s != OID_OK) return s;
  // A7: basis copy of this shard's rows, after the last estimate's basis reads
  CK(cudaStreamWaitEvent(st, ctx->ev_gram_done, 0));
  if (p.coeff_mode == 1) {
    // NEXT-1: <x_r, c_old_i> for the admitted columns and the columns about to be replaced or
    // vacated, before the copy overwrites them (Alg 7's A_J^T A_Jprev)
    changed_slots_kernel<<<1, 32, 0, st>>>(ctx->ptr<int64_t>(L.J), ctx->ptr<int64_t>(L.Jprev), t, ctx->ptr<int>(L.olds),
                                           ctx->ptr<int>(L.nold));
    CKL();
    const int64_t per = (ctx->m_loc + kCrossChunks - 1) / kCrossChunks;
    const dim3 grid(static_cast<unsigned>((nc * t + 7) / 8 < 64 ? (nc * t + 7) / 8 : 64), kCrossChunks);
    if (p.dtype == OID_F64)
      cross_dots_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(X), ld, ctx->ptr<double>(L.C), ctx->m_loc, t,
                                                      ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), ctx->ptr<int>(L.olds),
                                                      ctx->ptr<int>(L.nold), per, ctx->d(L.Dxp));
    else
      cross_dots_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(X), ld, ctx->ptr<float>(L.C), ctx->m_loc, t,
                                                     ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), ctx->ptr<int>(L.olds),
                                                     ctx->ptr<int>(L.nold), per, ctx->d(L.Dxp));
    CKL();
    cross_dots_sum_kernel<<<blocks_for(int64_t(t) * t), 256, 0, st>>>(ctx->d(L.Dxp), kCrossChunks, t, ctx->d(L.Dx));
    CKL();
  }
  tl_mark(ctx, st, 5);
  {
    dim3 grid(std::max(1u, std::min(blocks_for(ctx->m_loc), static_cast<unsigned>(8 * ctx->num_sms))));
    if (ctx->a9q && ctx->k1_mode_used != OID_K1_TC_FAST) ctx->a9q = false;   // no exponents for this block
    if (!ctx->a9q) {
      if (p.dtype == OID_F64)
        basis_copy_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(X), ld, ctx->ptr<double>(L.C), ctx->m_loc,
                                                        ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), nc, t);
      else
        basis_copy_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(X), ld, ctx->ptr<float>(L.C), ctx->m_loc,
                                                       ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), nc, t);
      CKL();
    } else {
      // A7 + the quantised copy in one pass over the admitted columns: per-admission exponents
      // (one warp each, blocks past the device-side count exit at once), then a GPU-filling
      // grid-stride pass over (admission, 512-row) items
      const k1f::Geom kg = k1f::make_geom(p.ell, nc, ctx->m_loc, p.dtype == OID_F64, std::max(2, ctx->num_sms - ctx->k1_free_sms));
      a9q::quant_adm_kernel<<<static_cast<unsigned>((nc + t + 7) / 8), 256, 0, st>>>(
          ctx->ptr<int>(L.admit), ctx->ptr<int>(L.counts), nc, t, ctx->ptr<int>(L.k1g), kg.nunits(), kg.nsg,
          p.dtype == OID_F64 ? 1021 : 125, ctx->ptr<int>(L.Fq), reinterpret_cast<int4*>(ctx->ptr<int>(L.qadm)));
      CKL();
      if (static_cast<int64_t>(nc + t) * ((ctx->m_loc + 511) / 512) >= (int64_t(1) << 31))
        return ctx->fail(OID_ESHAPE, "quantised copy: %lld rows per shard too many", (long long)ctx->m_loc);
      grid = dim3(static_cast<unsigned>(3 * ctx->num_sms));
      if (p.dtype == OID_F64)
        a9q::basis_quant_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(X), ld, ctx->ptr<uint8_t>(L.Cq),
                                                             ctx->m_loc, t, ctx->ptr<int>(L.counts),
                                                             reinterpret_cast<const int4*>(ctx->ptr<int>(L.qadm)),
                                                             ctx->ptr<double>(L.C));
      else
        a9q::basis_quant_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(X), ld, ctx->ptr<uint8_t>(L.Cq),
                                                            ctx->m_loc, t, ctx->ptr<int>(L.counts),
                                                            reinterpret_cast<const int4*>(ctx->ptr<int>(L.qadm)),
                                                            ctx->ptr<float>(L.C));
      CKL();
    }
  }
  tl_mark(ctx, st, 6);
  if (do_a3) ctx->n_obs += nc;
  ctx->last_nc = nc;
  cudaStream_t cs = ctx->use_side ? ctx->side : st;
  const int par = static_cast<int>(ctx->epoch & 1);
  double* SJp = ctx->d(L.SJ) + static_cast<size_t>(par) * ell * t;
  double* Sjpinvp = ctx->d(L.Sjpinv) + static_cast<size_t>(par) * ell * t;
  // the estimate of epoch - 2 (same parity) must have finished reading S_J, S_J^+
  CK(cudaStreamWaitEvent(cs, ctx->ev_sj_free[par], 0));
  tl_mark(ctx, cs, 11);
  // A8: Alg 4 kept implicit: S_J^+ per epoch.  Fast path: S_J^+ = (S_J^T S_J)^-1 S_J^T
  // by the cluster tridiagonalisation when kappa(S_J) <= 1e5 (no R9 cutoff can act); else the
  // one-sided Jacobi SVD pseudo-inverse (gated on the device).
  gather_sj_kernel<<<blocks_for(int64_t(ell) * t), 256, 0, cs>>>(ctx->d(L.S), ctx->ptr<int64_t>(L.J), t, ell, SJp);
  CKL();
  int* sjgate = ctx->ptr<int>(L.gate) + 2;
  if (t <= kTriMaxN) {
    s = gemm(ctx, cs, true, false, t, t, ell, 1.0, SJp, ell, SJp, ell, 0.0, ctx->d(L.sjG), t);
    if (s != OID_OK) return s;
    fill_vacant_diag_kernel<<<1, 256, 0, cs>>>(ctx->d(L.sjG), t, ctx->ptr<int64_t>(L.J));
    CKL();
    CK(cudaEventRecord(ctx->ev_sj_j, cs));   // last read of J in this chain
    s = spd_solve(ctx, cs, ctx->d(L.sjG), t, SJp, ell, true, ell, Sjpinvp, t, false, 1e10, sjgate,
                  scal + SC_KAPPA_SNAP + par);
    if (s != OID_OK) return s;
  } else {
    CK(cudaEventRecord(ctx->ev_sj_j, cs));
    set_flag_kernel<<<1, 1, 0, cs>>>(sjgate, 0, 1);
    CKL();
  }
  const int* fb = sjgate + 1;
  s = gemm(ctx, cs, false, false, ell, t, t, 1.0, SJp, ell, ctx->d(L.sjV), t, 0.0, ctx->d(L.sjB), ell, fb);
  if (s != OID_OK) return s;
  s = jacobi(ctx, cs, ctx->d(L.sjB), ell, t, ctx->d(L.sjV), ctx->d(L.sjsig), 1, true, fb);
  if (s != OID_OK) return s;
  s = pinv_assemble(ctx, cs, ctx->d(L.sjB), ell, t, ctx->d(L.sjV), ctx->d(L.sjsig), ctx->d(L.sjw), ctx->d(L.sjZ),
                    Sjpinvp, scal + SC_KAPPA_SNAP + par, OID_FLAG_SJ_RANK_DEFICIENT, fb);
  if (s != OID_OK) return s;
  CK(cudaMemcpyAsync(scal + SC_KAPPA, scal + SC_KAPPA_SNAP + par, sizeof(double), cudaMemcpyDeviceToDevice, cs));
  log_scalar_kernel<<<1, 32, 0, cs>>>(scal + SC_KAPPA_SNAP + par, ctx->d(L.elog) + static_cast<size_t>(ctx->epoch) * kElogCols + 7);
  CKL();
  CK(cudaEventRecord(ctx->ev_sj_done[par], cs));
  tl_mark(ctx, cs, 12);
  // snapshot of this epoch for an estimate that may overlap the next commit (after the
  // estimate of epoch - 2 has released this parity's snapshot)
  CK(cudaStreamWaitEvent(st, ctx->ev_snap_free[par], 0));
  commit_snapshot_kernel<<<1, 256, 0, st>>>(ctx->ptr<int64_t>(L.J), ctx->ptr<int>(L.dirty), t,
                                            ctx->ptr<int64_t>(L.Jsnap) + static_cast<size_t>(par) * t,
                                            ctx->ptr<int>(L.Dsnap) + static_cast<size_t>(par) * t, scal, par);
  CKL();
  CK(cudaEventRecord(ctx->ev_committed, st));
  ctx->epoch += 1;
  ctx->estimate_ready = true;
  if (p.coeff_mode == 1) return coeff_argmin(ctx, st);
  return OID_OK;
}

// NEXT-2, paper-literal epochs: every column is sketched and counted and goes
// into the buffer D (a device copy: the caller's block is gone by the time D fills); an epoch runs
// over D's t columns whenever t are buffered, at the exact column where that happens.  A commit
// that completes no epoch only moves the estimate's snapshot on (||A_obs||^2; J, S_J^+ unchanged).
oid_status commit_tcols(oid_ctx ctx, const void* X, int64_t ld, int nc, cudaStream_t st) {
  const oid_params& p = ctx->p;
  const Layout& L = ctx->L;
  const int ell = p.ell, t = ctx->t;
  const int64_t m = ctx->m_loc;
  double* Yp = ctx->d(L.Ypart);
  const double* nrm_blk = Yp + static_cast<int64_t>(ell) * nc;
  const size_t es = p.dtype == OID_F64 ? 8 : 4;
  bool epoch_done = false;
  for (int c0 = 0; c0 < nc;) {
    const int q = std::min(nc - c0, t - ctx->dcount);
    gram_update_kernel<<<blocks_for(int64_t(ell) * ell), 256, 0, st>>>(Yp + static_cast<int64_t>(ell) * c0, nrm_blk + c0, ell,
                                                                      q, ctx->d(L.gram), ctx->d(L.S), ctx->n_obs,
                                                                      ctx->d(L.scal));
    CKL();
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(m * q), 8 * ctx->num_sms));
    const uint8_t* src = static_cast<const uint8_t*>(X) + static_cast<size_t>(c0) * ld * es;
    uint8_t* dst = reinterpret_cast<uint8_t*>(ctx->ws + L.Dpool) + static_cast<size_t>(ctx->dcount) * m * es;
    if (p.dtype == OID_F64)
      copy_cols_kernel<double><<<g, 256, 0, st>>>(reinterpret_cast<const double*>(src), ld, reinterpret_cast<double*>(dst), m, m, q);
    else
      copy_cols_kernel<float><<<g, 256, 0, st>>>(reinterpret_cast<const float*>(src), ld, reinterpret_cast<float*>(dst), m, m, q);
    CKL();
    CK(cudaMemcpyAsync(ctx->d(L.Dnorm) + ctx->dcount, nrm_blk + c0, sizeof(double) * q, cudaMemcpyDeviceToDevice, st));
    ctx->n_obs += q;
    ctx->dcount += q;
    c0 += q;
    if (ctx->dcount == t) {
      oid_status s = post_epoch(ctx, ctx->ws + L.Dpool, m, t, st, ctx->d(L.S) + static_cast<int64_t>(ell) * ctx->dbase,
                                ctx->d(L.Dnorm), ctx->dbase, false);
      if (s != OID_OK) return s;
      ctx->dbase += t;
      ctx->dcount = 0;
      epoch_done = true;
    }
  }
  if (!epoch_done && ctx->epoch > 0) {
    const int par = static_cast<int>((ctx->epoch + 1) & 1);   // the last epoch's parity
    CK(cudaStreamWaitEvent(st, ctx->ev_snap_free[par], 0));
    commit_snapshot_kernel<<<1, 256, 0, st>>>(ctx->ptr<int64_t>(L.J), ctx->ptr<int>(L.dirty), t,
                                              ctx->ptr<int64_t>(L.Jsnap) + static_cast<size_t>(par) * t,
                                              ctx->ptr<int>(L.Dsnap) + static_cast<size_t>(par) * t, ctx->d(L.scal), par);
    CKL();
    CK(cudaEventRecord(ctx->ev_committed, st));
  }
  return OID_OK;
}

oid_status do_commit(oid_ctx ctx, const void* X, int64_t ld, int nc, cudaStream_t st) {
  if (ctx->p.epoch_mode == 1) return commit_tcols(ctx, X, ld, nc, st);
  double* Yp = ctx->d(ctx->L.Ypart);
  return post_epoch(ctx, X, ld, nc, st, Yp, Yp + static_cast<int64_t>(ctx->p.ell) * nc, ctx->n_obs, true);
}

oid_status check_block(oid_ctx ctx, const void* X, int64_t ld, int32_t nc) {
  if (nc < 0 || nc > ctx->p.b_max) return ctx->fail(OID_ESHAPE, "ncols=%d outside [0, b_max=%d]", nc, ctx->p.b_max);
  if (nc > 0 && X == nullptr) return ctx->fail(OID_EINVAL, "X is NULL");
  if (nc > 0 && ld < ctx->m_loc) return ctx->fail(OID_ESHAPE, "ld=%lld < m_loc=%lld", (long long)ld, (long long)ctx->m_loc);
  if (ctx->n_obs + nc > ctx->p.n_cap)
    return ctx->fail(OID_ESHAPE, "n_obs + ncols = %lld exceeds n_cap = %lld", (long long)(ctx->n_obs + nc),
                     (long long)ctx->p.n_cap);
  if (ctx->n_obs + nc >= (int64_t(1) << 31)) return ctx->fail(OID_ESHAPE, "too many columns");
  return OID_OK;
}

oid_status explicit_P(oid_ctx ctx, cudaStream_t st) {
  const Layout& L = ctx->L;
  const int par = static_cast<int>((ctx->epoch + 1) & 1);   // parity of the last committed epoch (epoch - 1)
  return gemm(ctx, st, false, false, ctx->t, static_cast<int>(ctx->n_obs), ctx->p.ell, 1.0,
              ctx->d(L.Sjpinv) + static_cast<size_t>(par) * ctx->t * ctx->p.ell, ctx->t,
              ctx->d(L.S), ctx->p.ell, 0.0, ctx->d(L.Pexp), ctx->t);
}

// Alg 8 factors that do not involve the basis Gram G (A10): P = S_J^+ S, Omega A_J P, the core
// pseudo-inverse M, Omega_k A P^T, the third-block trace terms and P P^T; enqueued on stream cs.
// The G-independent factors of Alg 8 for an explicit t x n_obs coefficient matrix P (ld t) and the
// sketched basis SJ (l x t): Omega A_J P, the core pseudo-inverse M, Omega_k A P^T, the third-block
// traces and P P^T; sc[0..3] = [T1 (set later with G), t3a, t3b, tr(G P P^T) (later)].
oid_status hutch_pre(oid_ctx ctx, cudaStream_t st, const double* P, const double* SJ, double* sc);

oid_status estimate_pre(oid_ctx ctx, cudaStream_t st, int par) {
  oid_status s = explicit_P(ctx, st);                                                 // P = S_J^+ S
  if (s != OID_OK) return s;
  return hutch_pre(ctx, st, ctx->d(ctx->L.Pexp), ctx->d(ctx->L.SJ) + static_cast<size_t>(par) * ctx->p.ell * ctx->t,
                   ctx->d(ctx->L.scal) + SC_T1);
}

oid_status hutch_pre(oid_ctx ctx, cudaStream_t st, const double* P, const double* SJ, double* sc) {
  const Layout& L = ctx->L;
  const oid_params& p = ctx->p;
  const int t = ctx->t, ell = p.ell, l1 = p.ell1, l2 = p.ell2, l3 = p.ell3;
  const int n = static_cast<int>(ctx->n_obs);
  double* S = ctx->d(L.S);
  double* AJP = ctx->d(L.AJP);
  oid_status s = gemm(ctx, st, false, false, ell, n, t, 1.0, SJ, ell, P, t, 0.0, AJP, ell);   // Omega A_J P
  if (s != OID_OK) return s;
  CK(cudaMemsetAsync(sc, 0, 4 * sizeof(double), st));
  if (l1 > 0 && l2 > 0) {
    // M = (Omega1 A (Omega2 A_J P)^T)^+   
    s = gemm(ctx, st, false, true, l1, l2, n, 1.0, S, ell, AJP + l1, ell, 0.0, ctx->d(L.cB), l1);
    if (s != OID_OK) return s;
    // M = B^+ (l2 x l1) by the one-sided Jacobi SVD pseudo-inverse with the R9 cutoff: the core
    // is routinely ill-conditioned (kappa 1e5-1e17 on C3), so no normal-equation fast path
    const int* cgate = nullptr;
    const int lo = std::min(l1, l2), hi = std::max(l1, l2);
    if (static_cast<size_t>(hi + lo) * lo * sizeof(double) <= kSmallSvdSmem) {
      // small pseudo-inverse in one CTA: SVD of the tall orientation (hi x lo)
      double* Bt = ctx->d(L.cBt);
      if (l1 < l2) {
        transpose_kernel<<<blocks_for(int64_t(l1) * l2), 256, 0, st>>>(ctx->d(L.cB), l1, l2, Bt, cgate);
        CKL();
      } else {
        CK(cudaMemcpyAsync(Bt, ctx->d(L.cB), sizeof(double) * l1 * l2, cudaMemcpyDeviceToDevice, st));
      }
      int* counters = ctx->ptr<int>(L.counters) + 2 * kMaxSweeps;
      small_svd_kernel<<<1, 1024, static_cast<size_t>(hi + lo) * lo * sizeof(double), st>>>(
          Bt, hi, lo, ctx->d(L.cV), ctx->d(L.csig), counters, kMaxSweeps, 4e-14 * std::max(1.0, std::sqrt(hi / 16.0)),
          cgate);
      CKL();
      if (l1 < l2) {
        // pinv(B^T) (l1 x l2) = V diag(w) Bt^T; M = pinv(B) = pinv(B^T)^T (l2 x l1)
        s = pinv_assemble(ctx, st, Bt, hi, lo, ctx->d(L.cV), ctx->d(L.csig), ctx->d(L.cw), ctx->d(L.cZ), ctx->d(L.cZ2),
                          nullptr, 0, cgate);
        if (s != OID_OK) return s;
        transpose_kernel<<<blocks_for(int64_t(l1) * l2), 256, 0, st>>>(ctx->d(L.cZ2), l1, l2, ctx->d(L.M), cgate);
        CKL();
      } else {
        s = pinv_assemble(ctx, st, Bt, hi, lo, ctx->d(L.cV), ctx->d(L.csig), ctx->d(L.cw), ctx->d(L.cZ), ctx->d(L.M),
                          nullptr, 0, cgate);
        if (s != OID_OK) return s;
      }
    } else {
      s = jacobi(ctx, st, ctx->d(L.cB), l1, l2, ctx->d(L.cV), ctx->d(L.csig), 2, false, cgate);
      if (s != OID_OK) return s;
      s = pinv_assemble(ctx, st, ctx->d(L.cB), l1, l2, ctx->d(L.cV), ctx->d(L.csig), ctx->d(L.cw), ctx->d(L.cZ), ctx->d(L.M),
                        nullptr, 0, cgate);
      if (s != OID_OK) return s;
    }
    // term1 = tr(M (Omega1 A P^T) G (Omega2 A P^T)^T)
    s = gemm(ctx, st, false, true, l1, t, n, 1.0, S, ell, P, t, 0.0, ctx->d(L.X1), l1);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, false, true, l2, t, n, 1.0, S + l1, ell, P, t, 0.0, ctx->d(L.X2), l2);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, false, false, l2, t, l1, 1.0, ctx->d(L.M), l2, ctx->d(L.X1), l1, 0.0, ctx->d(L.Q1), l2);
    if (s != OID_OK) return s;
  }
  if (l3 > 0) {
    // t3a = tr((Omega3 A)(Omega3 A_J P)^T)
    frob_dot_kernel<<<1, 256, 0, st>>>(S + l1 + l2, ell, AJP + l1 + l2, ell, l3, n, sc + 1);
    CKL();
    if (l1 > 0 && l2 > 0) {
      // t3b = tr((Omega3 A_J P)(Omega2 A)^T M (Omega1 A)(Omega3 A_J P)^T)
      s = gemm(ctx, st, false, true, l3, l2, n, 1.0, AJP + l1 + l2, ell, S + l1, ell, 0.0, ctx->d(L.R1), l3);
      if (s != OID_OK) return s;
      s = gemm(ctx, st, false, true, l3, l1, n, 1.0, AJP + l1 + l2, ell, S, ell, 0.0, ctx->d(L.R2t), l3);
      if (s != OID_OK) return s;
      s = gemm(ctx, st, false, false, l3, l1, l2, 1.0, ctx->d(L.R1), l3, ctx->d(L.M), l2, 0.0, ctx->d(L.R3), l3);
      if (s != OID_OK) return s;
      frob_dot_kernel<<<1, 256, 0, st>>>(ctx->d(L.R3), l3, ctx->d(L.R2t), l3, l3, l1, sc + 2);
      CKL();
    }
  }
  // tr(G P P^T) = ||A_J P||_F^2
  s = gemm(ctx, st, false, true, t, t, n, 1.0, P, t, P, t, 0.0, ctx->d(L.PPt), t);
  if (s != OID_OK) return s;
  return OID_OK;
}

// ---------------------------------------------------------------- gradient variant (A11)
// Omega G^p Omega^T (l x l, p = 0, 1), regenerated once per context (finalize-time only)
// Omega G^p Omega^T (l x l, p = 0, 1), once per context: for chunks of sketch rows s, W = G^p
// Omega(s, :)^T (the stencil applied to the generated rows, m x chunk), then Omega W through the
// tensor-core K1 like any block (O(l m) generation + l/chunk K1 passes instead of O(l^2 m) Philox)
oid_status grad_ogo(oid_ctx ctx, cudaStream_t st, bool explicit_call = false) {
  if (ctx->ogo_ready) return OID_OK;
  if (!explicit_call && (ctx->p.row_begin != 0 || ctx->p.row_end != ctx->p.m))
    return ctx->fail(OID_ESTATE, "sharded gradient variant: call oid_gradient_ogo and sum oid_partials(3) over the "
                     "shards before the GCV");
  const Layout& L = ctx->L;
  const int ell = ctx->p.ell;
  const int64_t m = ctx->m_loc;
  const int chunk = std::min(64, 2 * ctx->p.b_max);   // W lives in L.GX (2 m b_max doubles)
  double* W = ctx->d(L.GX);
  double* Y = ctx->d(L.YpG);                             // (l + 1) x chunk K1 output
  for (int p = 0; p < ctx->ga - 1; ++p)
    for (int s0 = 0; s0 < ell; s0 += chunk) {
      const int ns = std::min(chunk, ell - s0);
      const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(m * ns), 8 * ctx->num_sms));
      omega_g_cols_kernel<<<g, 256, 0, st>>>(s0, ns, m, ctx->grid, p, ctx->key0, ctx->key1, ctx->qscale, W,
                                             ctx->p.row_begin);
      CKL();
      oid_status s = sketch_one(ctx, W, m, ns, st, Y, true, false);
      if (s != OID_OK) return s;
      CK(cudaMemcpyAsync(ctx->d(L.OGO) + static_cast<size_t>(p) * ell * ell + static_cast<size_t>(s0) * ell, Y,
                         sizeof(double) * ell * ns, cudaMemcpyDeviceToDevice, st));
    }
  ctx->ogo_ready = true;
  return OID_OK;
}

// [S_J; c S^1_J; ..; c S^d_J] ((d+1) l x t) into L.gLst
oid_status grad_stack_j(oid_ctx ctx, cudaStream_t st, double c) {
  const Layout& L = ctx->L;
  const int ell = ctx->p.ell, t = ctx->t;
  stack_aug_kernel<<<blocks_for(int64_t(ctx->ga) * ell * t), 256, 0, st>>>(
      ctx->d(L.S), ctx->d(L.Sg), static_cast<int64_t>(ell) * ctx->p.n_cap, ctx->ga, ell, t, ctx->ptr<int64_t>(L.J), c,
      ctx->d(L.gLst));
  CKL();
  return OID_OK;
}

// sketched GCV(mu) of eq:GCV_COmega -> L.gscal[0]
oid_status grad_gcv(oid_ctx ctx, cudaStream_t st, double mu) {
  const Layout& L = ctx->L;
  const int ell = ctx->p.ell, t = ctx->t, n = static_cast<int>(ctx->n_obs), l3 = ctx->ga * ell, gd = ctx->ga - 1;
  oid_status s = grad_ogo(ctx, st);
  if (s != OID_OK) return s;
  s = grad_stack_j(ctx, st, 1.0);
  if (s != OID_OK) return s;
  const double* SJ = ctx->d(L.gLst);              // rows 0..l-1 of the stack (ld (d+1) l); S^p_J at SJ + p l
  // H = S_J^T S_J + mu sum_p S^p_J^T S^p_J      (t x t)
  s = gemm(ctx, st, true, false, t, t, ell, 1.0, SJ, l3, SJ, l3, 0.0, ctx->d(L.gH), t);
  if (s != OID_OK) return s;
  for (int q = 1; q <= gd; ++q) {
    s = gemm(ctx, st, true, false, t, t, ell, mu, SJ + q * ell, l3, SJ + q * ell, l3, 1.0, ctx->d(L.gH), t);
    if (s != OID_OK) return s;
  }
  // R = S_J + mu sum_p (Omega G^p Omega^T)^T S^p_J   (l x t)
  for (int q = 1; q <= gd; ++q) {
    s = gemm(ctx, st, true, false, ell, t, ell, mu, ctx->d(L.OGO) + static_cast<size_t>(q - 1) * ell * ell, ell,
             SJ + q * ell, l3, q == 1 ? 0.0 : 1.0, ctx->d(L.gR), ell);
    if (s != OID_OK) return s;
  }
  add_strided_kernel<<<blocks_for(int64_t(ell) * t), 256, 0, st>>>(SJ, l3, ell, t, ctx->d(L.gR), ell);
  CKL();
  // H^+ by the one-sided Jacobi SVD (R9 cutoff)
  CK(cudaMemcpyAsync(ctx->d(L.gHp), ctx->d(L.gH), sizeof(double) * t * t, cudaMemcpyDeviceToDevice, st));
  s = jacobi(ctx, st, ctx->d(L.gHp), t, t, ctx->d(L.gHV), ctx->d(L.gHs), 2, false);
  if (s != OID_OK) return s;
  s = pinv_assemble(ctx, st, ctx->d(L.gHp), t, t, ctx->d(L.gHV), ctx->d(L.gHs), ctx->d(L.gHw), ctx->d(L.gHZ),
                    ctx->d(L.gH), nullptr, 0);
  if (s != OID_OK) return s;
  // C = S_J H^+ R^T (l x l); E = S - C S; GCV = ||E||^2 / tr(I - C)^2
  s = gemm(ctx, st, false, false, ell, t, t, 1.0, SJ, l3, ctx->d(L.gH), t, 0.0, ctx->d(L.gLZ), ell);
  if (s != OID_OK) return s;
  s = gemm(ctx, st, false, true, ell, ell, t, 1.0, ctx->d(L.gLZ), ell, ctx->d(L.gR), ell, 0.0, ctx->d(L.gCm), ell);
  if (s != OID_OK) return s;
  CK(cudaMemcpyAsync(ctx->d(L.gE), ctx->d(L.S), sizeof(double) * ell * n, cudaMemcpyDeviceToDevice, st));
  s = gemm(ctx, st, false, false, ell, n, ell, -1.0, ctx->d(L.gCm), ell, ctx->d(L.S), ell, 1.0, ctx->d(L.gE), ell);
  if (s != OID_OK) return s;
  gcv_final_kernel<<<1, 256, 0, st>>>(ctx->d(L.gE), int64_t(ell) * n, ctx->d(L.gCm), ell, ctx->d(L.gscal));
  CKL();
  return OID_OK;
}

// P(mu) of eq:opt_grad_fullsketch: [S_J; sqrt(mu) S^p_J]^+ [S; sqrt(mu) S^p]  (t x n, ld t)
oid_status grad_coefficients(oid_ctx ctx, cudaStream_t st, double mu, double* P) {
  const Layout& L = ctx->L;
  const int ell = ctx->p.ell, t = ctx->t, n = static_cast<int>(ctx->n_obs), l3 = ctx->ga * ell;
  const double c = std::sqrt(mu);
  oid_status s = grad_stack_j(ctx, st, c);
  if (s != OID_OK) return s;
  s = jacobi(ctx, st, ctx->d(L.gLst), l3, t, ctx->d(L.gLV), ctx->d(L.gLs), 2, false);
  if (s != OID_OK) return s;
  s = pinv_assemble(ctx, st, ctx->d(L.gLst), l3, t, ctx->d(L.gLV), ctx->d(L.gLs), ctx->d(L.gLw), ctx->d(L.gLZ),
                    ctx->d(L.gLp), nullptr, 0);
  if (s != OID_OK) return s;
  stack_aug_kernel<<<blocks_for(int64_t(l3) * n), 256, 0, st>>>(ctx->d(L.S), ctx->d(L.Sg),
                                                                 static_cast<int64_t>(ell) * ctx->p.n_cap, ctx->ga, ell, n,
                                                                 nullptr, c, ctx->d(L.gRhs));
  CKL();
  return gemm(ctx, st, false, false, t, n, l3, 1.0, ctx->d(L.gLp), t, ctx->d(L.gRhs), l3, 0.0, P, t);
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* oid_version(void) { return "liboid 0.1 (sm_100a)"; }

const char* oid_last_error(oid_ctx ctx) { return ctx ? ctx->err : g_init_err; }

oid_status oid_workspace_query(const oid_params* p, size_t* bytes) {
  if (!bytes || validate(p)) return OID_EINVAL;
  *bytes = make_layout(*p).total;
  return OID_OK;
}

oid_status oid_sketch_table(int32_t q[16], double* scale) {
  if (!q || !scale) return OID_EINVAL;
  int32_t m[8];
  gauss16(m, q, scale);
  return OID_OK;
}

oid_status oid_init(const oid_params* p, void* workspace, size_t bytes, void* stream, oid_ctx* out) {
  if (!out) return OID_EINVAL;
  *out = nullptr;
  if (validate(p)) return OID_EINVAL;
  oid_ctx ctx = new (std::nothrow) oid_ctx_s();
  if (!ctx) return OID_ENOMEM;
  ctx->p = *p;
  ctx->L = make_layout(*p);
  if (!workspace || bytes < ctx->L.total || (reinterpret_cast<uintptr_t>(workspace) & 255)) {
    oid_destroy(ctx);   // releases the streams / events created so far
    return OID_ESHAPE;
  }
  ctx->ws = static_cast<char*>(workspace);
  ctx->m_loc = m_local(*p);
  ctx->t = p->k;
  if (p->grad_nfields > 0) {
    const bool d3 = p->grad_nz > 1;   // NEXT-4: three gradient components on a 3-D grid
    ctx->ga = d3 ? 4 : 3;
    ctx->grid.nf = p->grad_nfields;
    ctx->grid.nx = p->grad_nx;
    ctx->grid.ny = p->grad_ny;
    ctx->grid.nz = d3 ? p->grad_nz : 1;
    ctx->grid.d = d3 ? 3 : 2;
    ctx->grid.hx = p->grad_hx > 0.0 ? p->grad_hx : (p->grad_nx > 1 ? 1.0 / (p->grad_nx - 1) : 1.0);
    ctx->grid.hy = p->grad_hy > 0.0 ? p->grad_hy : (p->grad_ny > 1 ? 1.0 / (p->grad_ny - 1) : 1.0);
    ctx->grid.hz = p->grad_hz > 0.0 ? p->grad_hz : (p->grad_nz > 1 ? 1.0 / (p->grad_nz - 1) : 1.0);
  }
  const int ng = ctx->ga * p->ell;
  ctx->key0 = static_cast<uint32_t>(p->seed & 0xffffffffu);
  ctx->key1 = static_cast<uint32_t>(p->seed >> 32);
  const double k = p->k;
  ctx->factor = p->c * (k * std::log(k) + k * std::log(1.0 / p->delta) / p->eps) / ctx->t;
  int32_t q[16];
  gauss16(ctx->qmag, q, &ctx->qscale);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto bad = [&](cudaError_t e) {
    snprintf(g_init_err, sizeof(g_init_err), "init: %s", cudaGetErrorString(e));
    oid_destroy(ctx);   // releases the streams / events created so far
    return OID_ECUDA;
  };
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return bad(e);
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, p->device)) != cudaSuccess) return bad(e);
  ctx->num_sms = prop.multiProcessorCount;
  int per_sm = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_svd_kernel, 256, 0)) != cudaSuccess) return bad(e);
  ctx->coop_max = std::max(1, per_sm * ctx->num_sms);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sym_bjacobi_kernel, 256, 0)) != cudaSuccess) return bad(e);
  ctx->sym_coop_max = std::max(1, std::min(per_sm, 2) * ctx->num_sms);
  {
    const int big = static_cast<int>(prop.sharedMemPerBlockOptin) - 2048;
    if ((e = cudaFuncSetAttribute(bjacobi_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)) != cudaSuccess) return bad(e);
    if ((e = cudaFuncSetAttribute(bjacobi_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)) != cudaSuccess) return bad(e);
  }
  if (std::min(ng, p->k) <= kTriMaxG) {
    // the cluster tridiagonalisation serves A4 (order ell, or 3 ell with gradients: alone up to
    // 512, as the last 512 columns up to 1024) and the A8 SPD solve (order k, when k <= 512)
    const int ntri = std::min(std::max(ng, p->k), kTriMaxN);
    if ((e = cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(double) * ntri * tri_rows(ntri)))) !=
        cudaSuccess)
      return bad(e);
    const int ref_smem = static_cast<int>(sizeof(double) * kQStages * kRefChunk * tri_ldv(kTriMaxN));
    const int ref_smem_1k = static_cast<int>(sizeof(double) * kQStages * kRefChunk * tri_ldv(1024));
    const int ref_smem_2k = static_cast<int>(sizeof(double) * kRefChunk * tri_ldv(kTriMaxG));
    if ((e = cudaFuncSetAttribute(tri_scores_multi_kernel<2, 256, kQStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ref_smem)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tri_scores_multi_kernel<4, 256, kQStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ref_smem_1k)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tri_scores_multi_kernel<4, 512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ref_smem_2k)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tri_scores_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(double) * (kQV + 2) * kTriMaxG))) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(lambda_sorted_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(double) * 3 * kTriMaxG))) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tridiag_panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tridiag_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanSmem)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(tri_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ref_smem)) != cudaSuccess)
      return bad(e);
  }
  if ((e = cudaFuncSetAttribute(small_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmallSvdSmem))) != cudaSuccess)
    return bad(e);
  {
    int lo = 0, hi = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return bad(e);
    // Both side streams at the priority of the ingest stream given at init (measured best on C3
    // among above / equal / below, profiles/r01_summary.md): above it they starve the next block's
    // persistent K1 of SMs, below it (with a low-priority estimate stream) the estimate chain lags.
    int p_ing = 0;
    if (cudaStreamGetPriority(st, &p_ing) != cudaSuccess) p_ing = lo;
    (void)hi;
    const int p_side = getenv("OID_SIDE_PRIO") ? atoi(getenv("OID_SIDE_PRIO")) : p_ing;
    const int p_side2 = getenv("OID_SIDE2_PRIO") ? atoi(getenv("OID_SIDE2_PRIO")) : p_ing;
    if ((e = cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, p_side)) != cudaSuccess) return bad(e);
    if ((e = cudaStreamCreateWithPriority(&ctx->side2, cudaStreamNonBlocking, p_side2)) != cudaSuccess) return bad(e);
    if ((e = cudaStreamCreateWithPriority(&ctx->side3, cudaStreamNonBlocking, p_ing)) != cudaSuccess) return bad(e);
    // A9 at the lowest priority: throughput work that fills whatever the latency-bound chains leave
    const int p_gs = getenv("OID_GS_PRIO") ? atoi(getenv("OID_GS_PRIO")) : lo;
    if ((e = cudaStreamCreateWithPriority(&ctx->gs, cudaStreamNonBlocking, p_gs)) != cudaSuccess) return bad(e);
    if ((e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming)) != cudaSuccess) return bad(e);
    if ((e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming)) != cudaSuccess) return bad(e);
    for (cudaEvent_t* ev : {&ctx->ev_committed, &ctx->ev_gram_done, &ctx->ev_sj_j, &ctx->ev_est_done, &ctx->ev_sj_done[0],
                            &ctx->ev_sj_done[1], &ctx->ev_sj_free[0], &ctx->ev_sj_free[1], &ctx->ev_snap_free[0],
                            &ctx->ev_snap_free[1], &ctx->ev_gs_done, &ctx->ev_gsum_free[0], &ctx->ev_gsum_free[1]})
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return bad(e);
    if (getenv("OID_BG_FREE")) ctx->bg_free_sms = std::max(0, atoi(getenv("OID_BG_FREE")));
    if (getenv("OID_BG_WAVES")) ctx->bg_waves = std::max(1, atoi(getenv("OID_BG_WAVES")));
    if (getenv("OID_GS_GATE")) ctx->gs_gate = atoi(getenv("OID_GS_GATE"));
    if (getenv("OID_BG_CLUSTER")) {
      const int v = atoi(getenv("OID_BG_CLUSTER"));
      ctx->bg_cluster = (v == 2 || v == 4 || v == 8 || v == 16) ? v : 1;
    }
    if (getenv("OID_BG_SMEM")) ctx->bg_smem_kb = std::min(200, std::max(8, atoi(getenv("OID_BG_SMEM"))));
    ctx->use_side = !(getenv("OID_NO_SIDE") && atoi(getenv("OID_NO_SIDE")) != 0);
    if (getenv("OID_K1_FREE")) ctx->k1_free_sms = std::max(0, atoi(getenv("OID_K1_FREE")));
    ctx->timeline = getenv("OID_TIMELINE") && atoi(getenv("OID_TIMELINE")) != 0;
  }
  ctx->k1_ctas_per_sm = 1;
  ctx->cold_jacobi = getenv("OID_JACOBI_COLD") && atoi(getenv("OID_JACOBI_COLD")) != 0;
  ctx->k1_debug = getenv("OID_K1_DEBUG") && atoi(getenv("OID_K1_DEBUG")) != 0;
  ctx->tc_ok = (prop.major == 10 && prop.minor == 0) && k1tc_supported(p->ell, p->b_max, p->dtype == OID_F64);
  {
    // A9 tensor-map of the basis slab (fixed for the life of the context)
    const bool f64 = p->dtype == OID_F64;
    const int es = f64 ? 8 : 4;
    const Layout& Lb = ctx->L;
    // {RL rows, t slots, tiles} over the row-tiled basis: one box = one tile of all slots,
    // t x 128 contiguous bytes (two boxes of <= 256 slots when t > 256)
    const int64_t RL = 128 / es;
    const int64_t ntiles = (ctx->m_loc + RL - 1) / RL;
    if (k1tc_encoder() == nullptr) {
      snprintf(g_init_err, sizeof(g_init_err), "init: cuTensorMapEncodeTiled unavailable");
      oid_destroy(ctx);   // releases the streams / events created so far
      return OID_ECUDA;
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(RL), static_cast<cuuint64_t>(ctx->t), static_cast<cuuint64_t>(ntiles)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(RL * es), static_cast<cuuint64_t>(RL * es * ctx->t)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(RL), static_cast<cuuint32_t>(std::min(ctx->t, 256)), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = k1tc_encoder()(&ctx->bg_map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                 ctx->ws + Lb.C, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      snprintf(g_init_err, sizeof(g_init_err), "init: basis tensor map encoding failed (%d)", static_cast<int>(cr));
      oid_destroy(ctx);   // releases the streams / events created so far
      return OID_ECUDA;
    }
    const int bgmax = 200 * 1024 + 1024;
    if ((e = cudaFuncSetAttribute(a9q::gram_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(a9q::smem_bytes()))) != cudaSuccess) return bad(e);
    if ((e = cudaFuncSetAttribute(a9q::gram_q_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return bad(e);
    if ((e = cudaFuncSetAttribute(bgtc::basis_gram_tc_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bgmax)) != cudaSuccess) return bad(e);
    if ((e = cudaFuncSetAttribute(bgtc::basis_gram_tc_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bgmax)) != cudaSuccess) return bad(e);
    if ((e = cudaFuncSetAttribute(bgtc::basis_gram_tc_kernel<double>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return bad(e);
    if ((e = cudaFuncSetAttribute(bgtc::basis_gram_tc_kernel<float>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return bad(e);
  }
  double qd[16];
  for (int i = 0; i < 16; ++i) qd[i] = q[i] + 0.5;
  if ((e = cudaMemcpyToSymbolAsync(c_qtab_f64, qd, sizeof(qd), 0, cudaMemcpyHostToDevice, st)) != cudaSuccess) return bad(e);
  // state: J = -1, tau_old = 1, Gram = 0, S = 0, scalars, flags
  const Layout& L = ctx->L;
  if ((e = cudaMemsetAsync(ctx->ws + L.J, 0xff, sizeof(int64_t) * ctx->t, st)) != cudaSuccess) return bad(e);
  std::vector<double> ones(ctx->t, 1.0);
  if ((e = cudaMemcpyAsync(ctx->ws + L.tau_old, ones.data(), sizeof(double) * ctx->t, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.gram, 0, sizeof(double) * ng * ng, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.Vh, 0, sizeof(double) * ng * (ng + 1), st)) != cudaSuccess) return bad(e);
  set_identity_kernel<<<static_cast<unsigned>((int64_t(ng) * ng + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<double*>(ctx->ws + L.gV), ng);
  set_identity_kernel<<<static_cast<unsigned>((int64_t(p->k) * p->k + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<double*>(ctx->ws + L.sjV), p->k);
  if ((e = cudaGetLastError()) != cudaSuccess) return bad(e);
  double sc[SC_COUNT] = {0};
  sc[SC_MINMARGIN] = INFINITY;
  sc[SC_KAPPA] = 1.0;
  if ((e = cudaMemcpyAsync(ctx->ws + L.scal, sc, sizeof(sc), cudaMemcpyHostToDevice, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.flags, 0, 4 * sizeof(unsigned), st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.Gfull, 0, sizeof(double) * ctx->t * ctx->t, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.dirty, 0, sizeof(int) * ctx->t, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.counts, 0, 4 * sizeof(int), st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.cum, 0, 4 * sizeof(unsigned long long), st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.elog, 0, sizeof(double) * kElogCols * p->n_cap, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.eslog, 0, sizeof(double) * kElogCols * p->n_cap, st)) != cudaSuccess) return bad(e);
  if ((e = cudaMemsetAsync(ctx->ws + L.gcnt, 0, 8 * sizeof(int), st)) != cudaSuccess) return bad(e);
  k1f::fill_int_kernel<<<(k1f::kMaxUnits * 32 + 255) / 256, 256, 0, st>>>(ctx->ptr<int>(L.k1g), k1f::kMaxUnits * 32,
                                                                        k1f::kNoGuess);
  if ((e = cudaMemsetAsync(ctx->ws + L.k1g + k1f::kMaxUnits * 32 * sizeof(int), 0, 8 * sizeof(int), st)) != cudaSuccess)
    return bad(e);
  if ((e = cudaGetLastError()) != cudaSuccess) return bad(e);
  {
    const int64_t RL = 128 / static_cast<int64_t>(dsize(*p));
    const size_t cb = static_cast<size_t>((ctx->m_loc + RL - 1) / RL * RL) * ctx->t * dsize(*p);
    if ((e = cudaMemsetAsync(ctx->ws + L.C, 0, cb, st)) != cudaSuccess) return bad(e);
  }
  ctx->a9q = a9q_wanted(*p) && ctx->tc_ok;
  ctx->a9q_serial = getenv("OID_A9Q_SERIAL") && atoi(getenv("OID_A9Q_SERIAL")) != 0;
  if (getenv("OID_A9Q_CL")) ctx->a9q_cl = std::max(1, std::min(7, atoi(getenv("OID_A9Q_CL"))));
  ctx->a9_defer = p->row_begin == 0 && p->row_end == p->m && !(getenv("OID_A9_DEFER") && atoi(getenv("OID_A9_DEFER")) == 0);
  if ((e = cudaEventCreateWithFlags(&ctx->ev_k1_end, cudaEventDisableTiming)) != cudaSuccess) return bad(e);
  if (a9q_wanted(*p)) {
    if ((e = cudaMemsetAsync(ctx->ws + L.Cq, 0, a9q::qbasis_bytes(ctx->m_loc, ctx->t), st)) != cudaSuccess) return bad(e);
    if ((e = cudaMemsetAsync(ctx->ws + L.Fq, 0, sizeof(int) * ctx->t, st)) != cudaSuccess) return bad(e);
  }
  if (p->omega_cache == 1) {
    const int64_t g0 = p->row_begin / 32, ng = (p->row_end + 31) / 32 - g0 + 1;
    k1tc::omega_fill_kernel<<<static_cast<unsigned>(ctx->num_sms * 8), 256, 0, st>>>(
        reinterpret_cast<uint4*>(ctx->ws + L.omega), ng, g0, p->ell, ctx->key0, ctx->key1);
    if ((e = cudaGetLastError()) != cudaSuccess) return bad(e);
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return bad(e);   // host arrays above go out of scope
  *out = ctx;
  return OID_OK;
}

oid_status oid_ingest_sketch(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream) {
  return oid_ingest_sketch_halo(ctx, X, ld, ncols, nullptr, 0, nullptr, 0, stream);
}

oid_status oid_ingest_sketch_halo(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, const void* X_lo,
                                  int64_t ld_lo, const void* X_hi, int64_t ld_hi, void* stream) {
  NvtxRange nvtx_range("oid_ingest_sketch");
  if (!ctx) return OID_EINVAL;
  oid_status s = check_block(ctx, X, ld, ncols);
  if (s != OID_OK) return s;
  const int64_t hlo = grad_halo_rows(ctx, true), hhi = grad_halo_rows(ctx, false);
  if (ncols > 0 && ((hlo > 0 && (!X_lo || ld_lo < hlo)) || (hhi > 0 && (!X_hi || ld_hi < hhi))))
    return ctx->fail(OID_EINVAL, "sharded gradient variant: the block needs stencil halos of %lld rows below and %lld "
                     "above (oid_grad_halo; got %p ld %lld, %p ld %lld)", static_cast<long long>(hlo),
                     static_cast<long long>(hhi), X_lo, static_cast<long long>(ld_lo), X_hi,
                     static_cast<long long>(ld_hi));
  ctx->halo_lo = X_lo;
  ctx->halo_hi = X_hi;
  ctx->halo_ld_lo = ld_lo;
  ctx->halo_ld_hi = ld_hi;
  ctx->pending_nc = ncols;
  if (ncols == 0) return OID_OK;
  return do_sketch(ctx, X, ld, ncols, static_cast<cudaStream_t>(stream));
}

oid_status oid_grad_halo(oid_ctx ctx, int64_t* rows_lo, int64_t* rows_hi) {
  if (!ctx || !rows_lo || !rows_hi) return OID_EINVAL;
  *rows_lo = grad_halo_rows(ctx, true);
  *rows_hi = grad_halo_rows(ctx, false);
  return OID_OK;
}

oid_status oid_ingest_commit(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream) {
  NvtxRange nvtx_range("oid_ingest_commit");
  if (!ctx) return OID_EINVAL;
  if (ctx->pending_nc < 0 || ctx->pending_nc != ncols)
    return ctx->fail(OID_ESTATE, "commit without a matching sketch (pending ncols %d, got %d)", ctx->pending_nc, ncols);
  oid_status s = check_block(ctx, X, ld, ncols);
  if (s != OID_OK) return s;
  ctx->pending_nc = -1;
  if (ncols == 0) return OID_OK;
  return do_commit(ctx, X, ld, ncols, static_cast<cudaStream_t>(stream));
}

oid_status oid_ingest_block(oid_ctx ctx, const void* X, int64_t ld, int32_t ncols, void* stream) {
  if (!ctx) return OID_EINVAL;
  if (ctx->p.row_begin != 0 || ctx->p.row_end != ctx->p.m)
    return ctx->fail(OID_ESTATE, "sharded context: use oid_ingest_sketch / reduce / oid_ingest_commit");
  oid_status s = oid_ingest_sketch(ctx, X, ld, ncols, stream);
  if (s != OID_OK) return s;
  return oid_ingest_commit(ctx, X, ld, ncols, stream);
}

oid_status oid_partials(oid_ctx ctx, int32_t which, double** dev_ptr, int64_t* count) {
  if (ctx && ctx->a9_pending) {   // a deferred A9 (estimate_begin) is launched before anything reads state
    oid_status sp = launch_a9(ctx);
    if (sp != OID_OK) return sp;
  }
  if (!ctx || !dev_ptr || !count) return OID_EINVAL;
  if (which == 0) {
    *dev_ptr = ctx->d(ctx->L.Ypart);
    *count = int64_t(ctx->p.ell + 1) * std::max(0, ctx->pending_nc);
  } else if (which == 1) {
    *dev_ptr = ctx->d(ctx->L.Gsum) + static_cast<size_t>(ctx->est_par) * ctx->t * ctx->t;
    *count = int64_t(ctx->t) * ctx->t;
  } else if (which == 2 && ctx->ga > 1) {   // [Y_p; n_p], p = 1..d, each (ell + 1) b_max apart
    *dev_ptr = ctx->d(ctx->L.YpG);
    *count = int64_t(ctx->ga - 1) * (ctx->p.ell + 1) * ctx->p.b_max;
  } else if (which == 3 && ctx->ga > 1) {   // Omega G^p Omega^T, p = 1..d (ell x ell each)
    *dev_ptr = ctx->d(ctx->L.OGO);
    *count = int64_t(ctx->ga - 1) * ctx->p.ell * ctx->p.ell;
  } else {
    return OID_EINVAL;
  }
  return OID_OK;
}

static oid_status estimate_begin_impl(oid_ctx ctx, void* stream) {
  if (!ctx) return OID_EINVAL;
  if (!ctx->estimate_ready) return ctx->fail(OID_ESTATE, "no block ingested yet");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  oid_status sp = launch_a9(ctx);   // an estimate begun but never ended
  if (sp != OID_OK) return sp;
  const Layout& L = ctx->L;
  const int t = ctx->t;
  EvScope ev(ctx, st, &ctx->ev_est);
  // this estimate may run on another stream than the ingests: it reads the snapshot (J,
  // admission tags, ||A_obs||^2) and the S_J, S_J^+ buffers of the last committed epoch's parity
  const int par = static_cast<int>((ctx->epoch + 1) & 1);
  CK(cudaStreamWaitEvent(st, ctx->ev_committed, 0));
  tl_mark(ctx, st, 7);
  // A9 on its own stream, ordered after the commit it reads (and after the tail of the estimate
  // two back, which read this parity's sums) but not behind the previous estimate's tail on `st`:
  // the Gram of estimate e+1 must not wait for the A10 factors of estimate e.
  const int gp = ctx->n_est & 1;
  ctx->est_par = gp;
  ctx->n_est += 1;
  cudaStream_t gs = ctx->use_side ? ctx->gs : st;
  if (ctx->use_side) {
    CK(cudaStreamWaitEvent(gs, ctx->ev_committed, 0));
    CK(cudaStreamWaitEvent(gs, ctx->ev_gsum_free[gp], 0));
    if (ctx->gs_gate) CK(cudaStreamWaitEvent(gs, ctx->ev_sj_done[par], 0));
  }
  int* dl = ctx->ptr<int>(L.dlist) + static_cast<size_t>(gp) * t;
  int* gc = ctx->ptr<int>(L.gcnt) + 4 * gp;
  double* Gs = ctx->d(L.Gsum) + static_cast<size_t>(gp) * t * t;
  dirty_compact_kernel<<<1, 32, 0, gs>>>(ctx->ptr<int>(L.Dsnap) + static_cast<size_t>(par) * t, t, ctx->last_est_tag, dl, gc,
                                         ctx->ptr<unsigned long long>(L.cum));
  CKL();
  ctx->last_est_tag = static_cast<int>(ctx->epoch);   // newest admission tag of this state
  // A10 factors that do not need G: on the second side stream, concurrently with A9 below
  cudaStream_t cs2 = ctx->use_side ? ctx->side2 : st;
  oid_status s0 = fork_to(ctx, st, cs2);
  if (s0 != OID_OK) return s0;
  CK(cudaStreamWaitEvent(cs2, ctx->ev_sj_done[par], 0));
  tl_mark(ctx, cs2, 13);
  s0 = estimate_pre(ctx, cs2, par);
  if (s0 != OID_OK) return s0;
  est_kappa_kernel<<<1, 1, 0, cs2>>>(ctx->d(L.scal), par);
  CKL();
  CK(cudaEventRecord(ctx->ev_sj_free[par], cs2));   // S_J, S_J^+ (and kappa) of this parity are free again
  tl_mark(ctx, cs2, 14);
  // A9 (below, launch_a9) reads what this call has queued on gs; single-shard contexts defer its
  // launch until the next ingest has launched its K1 (or until anything needs the Gram): the two
  // full-GPU kernels then run back to back and A9 overlaps the latency-bound post-pass instead
  ctx->a9_gs = gs;
  ctx->a9_gp = gp;
  ctx->a9_pending = true;
  if (ctx->a9_defer && ctx->use_side) return OID_OK;
  oid_status sa = launch_a9(ctx);
  if (sa != OID_OK) return sa;
  // the caller's stream sees the partial sums (the sharded path reduces them on it)
  if (ctx->use_side) CK(cudaStreamWaitEvent(st, ctx->ev_gs_done, 0));
  return OID_OK;
}

static oid_status estimate_end_impl(oid_ctx ctx, double* out_dev, void* stream) {
  if (!ctx) return OID_EINVAL;
  if (!ctx->estimate_ready) return ctx->fail(OID_ESTATE, "no block ingested yet");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  {
    oid_status sp = launch_a9(ctx);   // deferred and not yet launched by an ingest
    if (sp != OID_OK) return sp;
    if (ctx->use_side) CK(cudaStreamWaitEvent(st, ctx->ev_gs_done, 0));
  }
  const Layout& L = ctx->L;
  const oid_params& p = ctx->p;
  const int t = ctx->t, l1 = p.ell1, l2 = p.ell2;
  double* scal = ctx->d(L.scal);
  EvScope ev(ctx, st, &ctx->ev_est);
  // The G-dependent tail runs on the (highest-priority) second side stream, after the
  // G-independent factors already queued there (estimate_pre): it is short and must not wait
  // behind the next block's K1 on a lower-priority estimate stream.  `st` joins it at the end.
  const int par = static_cast<int>((ctx->epoch + 1) & 1);
  cudaStream_t cs = ctx->use_side ? ctx->side2 : st;
  oid_status s = fork_to(ctx, st, cs);
  if (s != OID_OK) return s;
  est_scalars_kernel<<<1, 1, 0, cs>>>(scal, par);
  CKL();
  const int gp = ctx->est_par;
  gram_scatter_kernel<<<blocks_for(int64_t(t) * t), 256, 0, cs>>>(ctx->d(L.Gsum) + static_cast<size_t>(gp) * t * t,
                                                                  ctx->ptr<int>(L.dlist) + static_cast<size_t>(gp) * t,
                                                                  ctx->ptr<int>(L.gcnt) + 4 * gp, t, ctx->d(L.Gfull));
  CKL();
  CK(cudaEventRecord(ctx->ev_gsum_free[gp], cs));   // the A9 stream may reuse this parity
  CK(cudaMemcpyAsync(ctx->d(L.G), ctx->d(L.Gfull), sizeof(double) * t * t, cudaMemcpyDeviceToDevice, cs));
  mask_gram_kernel<<<blocks_for(int64_t(t) * t), 256, 0, cs>>>(ctx->d(L.G), ctx->ptr<int64_t>(L.Jsnap) + static_cast<size_t>(par) * t, t);
  CKL();
  if (l1 > 0 && l2 > 0) {
    // term1 = tr(M (Omega1 A P^T) G (Omega2 A P^T)^T) = <Q1 G, X2>
    s = gemm(ctx, cs, false, false, l2, t, t, 1.0, ctx->d(L.Q1), l2, ctx->d(L.G), t, 0.0, ctx->d(L.Q2), l2);
    if (s != OID_OK) return s;
    frob_dot_kernel<<<1, 256, 0, cs>>>(ctx->d(L.Q2), l2, ctx->d(L.X2), l2, l2, t, scal + SC_T1);
    CKL();
  }
  // tr(G P P^T) = ||A_J P||_F^2
  frob_dot_kernel<<<1, 256, 0, cs>>>(ctx->d(L.G), t, ctx->d(L.PPt), t, t, t, scal + SC_GPP);
  CKL();
  hutch_final_kernel<<<1, 32, 0, cs>>>(scal, p.ell3, ctx->ptr<unsigned>(L.flags), ctx->d(L.est));
  CKL();
  if (out_dev) CK(cudaMemcpyAsync(out_dev, ctx->d(L.est), 8 * sizeof(double), cudaMemcpyDeviceToDevice, cs));
  if (ctx->n_est <= p.n_cap) {
    est_log_kernel<<<1, 32, 0, cs>>>(ctx->d(L.est), static_cast<double>(ctx->epoch - 1),
                                     ctx->d(L.eslog) + static_cast<size_t>(ctx->n_est - 1) * kElogCols);
    CKL();
  }
  CK(cudaEventRecord(ctx->ev_snap_free[par], cs));   // this parity's snapshot may be rewritten
  s = join_from(ctx, st, cs);
  if (s != OID_OK) return s;
  CK(cudaEventRecord(ctx->ev_est_done, st));
  tl_mark(ctx, st, 10);
  return OID_OK;
}

// With coeff_mode = 1 every commit already ran the estimate of all four candidates (coeff_argmin):
// these return the chosen candidate's estimate, ordered after that work.
oid_status oid_estimate_begin(oid_ctx ctx, void* stream) {
  NvtxRange nvtx_range("oid_estimate_begin");
  if (!ctx) return OID_EINVAL;
  if (ctx->p.coeff_mode != 1) return estimate_begin_impl(ctx, stream);
  if (!ctx->estimate_ready) return ctx->fail(OID_ESTATE, "no block ingested yet");
  CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->ev_est_done, 0));
  return OID_OK;
}

oid_status oid_estimate_end(oid_ctx ctx, double* out_dev, void* stream) {
  NvtxRange nvtx_range("oid_estimate_end");
  if (!ctx) return OID_EINVAL;
  if (ctx->p.coeff_mode != 1) return estimate_end_impl(ctx, out_dev, stream);
  if (!ctx->estimate_ready) return ctx->fail(OID_ESTATE, "no block ingested yet");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  CK(cudaMemcpyAsync(ctx->d(ctx->L.est), ctx->d(ctx->L.est_ch), 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (out_dev) CK(cudaMemcpyAsync(out_dev, ctx->d(ctx->L.est_ch), 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return OID_OK;
}

oid_status oid_error_estimate(oid_ctx ctx, double* out_host, void* stream) {
  if (!ctx || !out_host) return OID_EINVAL;
  oid_status s = oid_estimate_begin(ctx, stream);
  if (s != OID_OK) return s;
  s = oid_estimate_end(ctx, nullptr, stream);
  if (s != OID_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaMemcpyAsync(out_host, ctx->d(ctx->L.est), 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OID_OK;
}

oid_status oid_gradient_ogo(oid_ctx ctx, void* stream) {
  if (!ctx) return OID_EINVAL;
  if (ctx->ga == 1) return ctx->fail(OID_ESTATE, "gradient variant not enabled (grad_nfields = 0)");
  if (ctx->ogo_ready) return OID_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  oid_status s = join_side(ctx, st);
  if (s != OID_OK) return s;
  return grad_ogo(ctx, st, true);
}

oid_status oid_gradient_gcv(oid_ctx ctx, double mu, double* gcv_out, void* stream) {
  if (!ctx || !gcv_out) return OID_EINVAL;
  if (ctx->ga == 1) return ctx->fail(OID_ESTATE, "gradient variant not enabled (grad_nfields = 0)");
  if (!(mu >= 0.0)) return ctx->fail(OID_EINVAL, "mu must be >= 0");
  if (ctx->pending_nc >= 0) return ctx->fail(OID_ESTATE, "a sketch is pending commit");
  if (ctx->n_obs == 0) return ctx->fail(OID_ESTATE, "no block ingested yet");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  oid_status s = join_side(ctx, st);
  if (s != OID_OK) return s;
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  s = grad_gcv(ctx, st, mu);
  if (s != OID_OK) return s;
  CK(cudaMemcpyAsync(gcv_out, ctx->d(ctx->L.gscal), sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OID_OK;
}

oid_status oid_gradient_coefficients(oid_ctx ctx, double mu, double* P_dev, void* stream) {
  if (!ctx || !P_dev) return OID_EINVAL;
  if (ctx->ga == 1) return ctx->fail(OID_ESTATE, "gradient variant not enabled (grad_nfields = 0)");
  if (!(mu >= 0.0)) return ctx->fail(OID_EINVAL, "mu must be >= 0");
  if (ctx->pending_nc >= 0) return ctx->fail(OID_ESTATE, "a sketch is pending commit");
  if (ctx->n_obs == 0) return ctx->fail(OID_ESTATE, "no block ingested yet");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  oid_status s = join_side(ctx, st);
  if (s != OID_OK) return s;
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  return grad_coefficients(ctx, st, mu, P_dev);
}

oid_status oid_gradient_finalize(oid_ctx ctx, double lo, double hi, double tol, double* mu_star, double* P_dev,
                                 void* stream) {
  if (!ctx || !mu_star) return OID_EINVAL;
  if (!(hi > lo) || !(tol > 0.0)) return ctx->fail(OID_EINVAL, "need lo < hi and tol > 0");
  // golden-section search on log10(mu); each probe is one device GCV evaluation
  const double invphi = (std::sqrt(5.0) - 1.0) / 2.0;
  double a = lo, b = hi;
  double c = b - invphi * (b - a), d = a + invphi * (b - a);
  double fc, fd;
  oid_status s = oid_gradient_gcv(ctx, std::pow(10.0, c), &fc, stream);
  if (s != OID_OK) return s;
  s = oid_gradient_gcv(ctx, std::pow(10.0, d), &fd, stream);
  if (s != OID_OK) return s;
  while (b - a > tol) {
    if (fc < fd) {
      b = d; d = c; fd = fc;
      c = b - invphi * (b - a);
      s = oid_gradient_gcv(ctx, std::pow(10.0, c), &fc, stream);
    } else {
      a = c; c = d; fc = fd;
      d = a + invphi * (b - a);
      s = oid_gradient_gcv(ctx, std::pow(10.0, d), &fd, stream);
    }
    if (s != OID_OK) return s;
  }
  *mu_star = std::pow(10.0, 0.5 * (a + b));
  if (P_dev) {
    s = oid_gradient_coefficients(ctx, *mu_star, P_dev, stream);
    if (s != OID_OK) return s;
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  }
  return OID_OK;
}

oid_status oid_finalize(oid_ctx ctx, int64_t* J_host, double* P, int32_t P_on_device, void* basis_dev, void* stream) {
  if (ctx && ctx->a9_pending) {   // a deferred A9 (estimate_begin) is launched before anything reads state
    oid_status sp = launch_a9(ctx);
    if (sp != OID_OK) return sp;
  }
  NvtxRange nvtx_range("oid_finalize");
  if (!ctx) return OID_EINVAL;
  if (ctx->pending_nc >= 0) return ctx->fail(OID_ESTATE, "a sketch is pending commit");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout& L = ctx->L;
  const int t = ctx->t;
  oid_status sj = join_side(ctx, st);
  if (sj != OID_OK) return sj;
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  if (ctx->n_obs > 0 && P) {
    if (ctx->p.coeff_mode == 1) {   // NEXT-1: the chosen candidate of the last epoch
      CK(cudaMemcpyAsync(P, ctx->d(L.Pchosen), sizeof(double) * t * ctx->n_obs,
                         P_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    } else {
      oid_status s = explicit_P(ctx, st);
      if (s != OID_OK) return s;
      CK(cudaMemcpyAsync(P, ctx->d(L.Pexp), sizeof(double) * t * ctx->n_obs,
                         P_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    }
  }
  if (J_host) CK(cudaMemcpyAsync(J_host, ctx->ws + L.J, sizeof(int64_t) * t, cudaMemcpyDeviceToHost, st));
  if (basis_dev)
  {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(ctx->m_loc * t), 8 * ctx->num_sms));
    if (ctx->p.dtype == OID_F64)
      basis_untile_kernel<double><<<g, 256, 0, st>>>(ctx->ptr<double>(L.C), ctx->m_loc, t, static_cast<double*>(basis_dev));
    else
      basis_untile_kernel<float><<<g, 256, 0, st>>>(ctx->ptr<float>(L.C), ctx->m_loc, t, static_cast<float*>(basis_dev));
    CKL();
  }
  CK(cudaStreamSynchronize(st));
  return OID_OK;
}

oid_status oid_get(oid_ctx ctx, int32_t field, void* host_dst, size_t bytes, void* stream) {
  if (ctx && ctx->a9_pending) {   // a deferred A9 (estimate_begin) is launched before anything reads state
    oid_status sp = launch_a9(ctx);
    if (sp != OID_OK) return sp;
  }
  if (!ctx || !host_dst) return OID_EINVAL;
  const Layout& L = ctx->L;
  const oid_params& p = ctx->p;
  size_t off = 0, need = 0;
  switch (field) {
    case 0: off = L.J; need = sizeof(int64_t) * ctx->t; break;
    case 1: off = L.tau_old; need = sizeof(double) * ctx->t; break;
    case 2: off = L.S; need = sizeof(double) * p.ell * ctx->n_obs; break;
    case 3: off = L.gram; need = sizeof(double) * ctx->ga * p.ell * ctx->ga * p.ell; break;
    case 4: off = L.scal; need = sizeof(double) * 8; break;
    case 5: off = L.tau; need = sizeof(double) * (ctx->t + p.b_max); break;
    case 6: off = L.mu; need = sizeof(double) * ctx->ga * p.ell; break;
    case 7: off = L.Ypart; need = sizeof(double) * (p.ell + 1) * p.b_max; break;
    case 8: off = L.Sjpinv + static_cast<size_t>((ctx->epoch + 1) & 1) * ctx->t * p.ell * sizeof(double);
            need = sizeof(double) * ctx->t * p.ell; break;
    case 9: off = L.counters; need = sizeof(int) * kNumJacobiUses * kMaxSweeps; break;
    case 10: off = L.dbg; need = k1p::kDbgRows * k1tc::kDbgTiles * sizeof(long long); break;
    case 11: off = L.G; need = sizeof(double) * ctx->t * ctx->t; break;
    case 12: off = L.dbg + k1p::kDbgRows * k1tc::kDbgTiles * sizeof(long long); need = k1tc::kDbgTiles * sizeof(long long); break;
    case 15: off = L.k1g; need = sizeof(int) * (k1f::kMaxUnits * 32 + 8); break;
    case 14:
      if (p.coeff_mode != 1) return ctx->fail(OID_ESTATE, "field 14 needs coeff_mode = 1");
      off = L.qlog; need = sizeof(double) * 6 * ctx->epoch; break;
    case 13: {   // timeline: up to 4096 (tag, ms since the first mark) pairs, then cleared
      if (bytes < 2 * 4096 * sizeof(double)) return ctx->fail(OID_ESHAPE, "field 13 needs %zu bytes", 2 * 4096 * sizeof(double));
      CK(cudaDeviceSynchronize());
      double* o = static_cast<double*>(host_dst);
      for (size_t i = 0; i < 4096; ++i) { o[2 * i] = -1.0; o[2 * i + 1] = 0.0; }
      for (size_t i = 0; i < ctx->tl.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->tl[0].second, ctx->tl[i].second);
        o[2 * i] = ctx->tl[i].first;
        o[2 * i + 1] = ms;
      }
      for (auto& pr : ctx->tl) cudaEventDestroy(pr.second);
      ctx->tl.clear();
      return OID_OK;
    }
    default: return ctx->fail(OID_EINVAL, "unknown field %d", field);
  }
  if (bytes < need) return ctx->fail(OID_ESHAPE, "field %d needs %zu bytes", field, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  oid_status sj = join_side(ctx, st);
  if (sj != OID_OK) return sj;
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  if (need) CK(cudaMemcpyAsync(host_dst, ctx->ws + off, need, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OID_OK;
}

oid_status oid_stats(oid_ctx ctx, oid_stats_t* out) {
  if (ctx && ctx->a9_pending) {   // a deferred A9 (estimate_begin) is launched before anything reads state
    oid_status sp = launch_a9(ctx);
    if (sp != OID_OK) return sp;
  }
  if (!ctx || !out) return OID_EINVAL;
  std::memset(out, 0, sizeof(*out));
  out->n_obs = ctx->n_obs;
  out->epochs = ctx->epoch;
  out->launches = ctx->launches;
  out->k1_launches = ctx->k1_launches;
  out->k1_mode_used = ctx->k1_mode_used;
  auto sum = [&](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v, double* dst) -> cudaError_t {
    double s = 0.0;
    for (auto& pr : v) {
      cudaError_t e = cudaEventSynchronize(pr.second);
      if (e != cudaSuccess) return e;
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, pr.first, pr.second);
      if (e != cudaSuccess) return e;
      s += ms;
    }
    *dst = s;
    return cudaSuccess;
  };
  CK(sum(ctx->ev_k1, &out->k1_ms));
  CK(sum(ctx->ev_post, &out->post_ms));
  CK(sum(ctx->ev_est, &out->est_ms));
  CK(sum(ctx->ev_a9, &out->a9_ms));
  out->a9_launches = static_cast<int64_t>(ctx->ev_a9.size());
  // per-block ingest latency: start of the block's K1 to the end of its commit (one K1 per block
  // on the plain path; the gradient variant runs three)
  {
    const size_t nb = ctx->ev_post.size();
    const size_t per = nb ? ctx->ev_k1.size() / nb : 0;
    std::vector<double> lat;
    if (per >= 1 && ctx->ev_k1.size() == per * nb) {
      for (size_t i = 0; i < nb; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev_k1[i * per].first, ctx->ev_post[i].second));
        lat.push_back(ms);
      }
    }
    if (!lat.empty()) {
      std::sort(lat.begin(), lat.end());
      out->lat_min_ms = lat.front();
      out->lat_med_ms = lat[lat.size() / 2];
      out->lat_max_ms = lat.back();
    }
  }
  unsigned f = 0;
  CK(cudaStreamSynchronize(ctx->side));
  CK(cudaStreamSynchronize(ctx->side2));
  CK(cudaEventSynchronize(ctx->ev_est_done));
  CK(cudaStreamSynchronize(ctx->side3));
  CK(cudaStreamSynchronize(ctx->gs));
  CK(cudaEventSynchronize(ctx->ev_committed));
  CK(cudaMemcpy(&f, ctx->ws + ctx->L.flags, sizeof(unsigned), cudaMemcpyDeviceToHost));
  out->flags = f;
  unsigned long long cum[4] = {0, 0, 0, 0};
  CK(cudaMemcpy(cum, ctx->ws + ctx->L.cum, sizeof(cum), cudaMemcpyDeviceToHost));
  out->admissions = static_cast<int64_t>(cum[0]);
  out->dirty_slots = static_cast<int64_t>(cum[1]);
  out->estimates = static_cast<int64_t>(cum[2]);
  return OID_OK;
}

oid_status oid_report(oid_ctx ctx, char* buf, size_t cap, size_t* needed, void* stream) {
  if (ctx && ctx->a9_pending) {   // a deferred A9 (estimate_begin) is launched before anything reads state
    oid_status sp = launch_a9(ctx);
    if (sp != OID_OK) return sp;
  }
  if (!ctx) return OID_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaStreamSynchronize(st));
  for (cudaStream_t sp : {ctx->side, ctx->side2, ctx->side3, ctx->gs})
    if (sp) CK(cudaStreamSynchronize(sp));
  CK(cudaEventSynchronize(ctx->ev_est_done));
  const int64_t ne = std::min<int64_t>(ctx->epoch, ctx->p.n_cap);
  const int64_t nest = std::min<int64_t>(ctx->n_est, ctx->p.n_cap);
  std::vector<double> el(static_cast<size_t>(std::max<int64_t>(1, ne)) * kElogCols),
      es(static_cast<size_t>(std::max<int64_t>(1, nest)) * kElogCols);
  if (ne) CK(cudaMemcpy(el.data(), ctx->ws + ctx->L.elog, sizeof(double) * kElogCols * ne, cudaMemcpyDeviceToHost));
  if (nest) CK(cudaMemcpy(es.data(), ctx->ws + ctx->L.eslog, sizeof(double) * kElogCols * nest, cudaMemcpyDeviceToHost));
  std::vector<double> ql;
  if (ctx->p.coeff_mode == 1 && ne) {
    ql.resize(static_cast<size_t>(ne) * 6);
    CK(cudaMemcpy(ql.data(), ctx->ws + ctx->L.qlog, sizeof(double) * 6 * ne, cudaMemcpyDeviceToHost));
  }
  unsigned f = 0;
  CK(cudaMemcpy(&f, ctx->ws + ctx->L.flags, sizeof(unsigned), cudaMemcpyDeviceToHost));
  unsigned long long cum[4] = {0, 0, 0, 0};
  CK(cudaMemcpy(cum, ctx->ws + ctx->L.cum, sizeof(cum), cudaMemcpyDeviceToHost));
  std::string j;
  char tmp[512];
  auto num = [&](double v) {
    if (std::isfinite(v)) snprintf(tmp, sizeof(tmp), "%.17g", v);
    else snprintf(tmp, sizeof(tmp), "%s", std::isnan(v) ? "\"nan\"" : (v > 0 ? "\"inf\"" : "\"-inf\""));
    return std::string(tmp);
  };
  snprintf(tmp, sizeof(tmp),
           "{\"n_obs\": %lld, \"epochs\": %lld, \"estimates\": %lld, \"flags\": %u, \"admissions\": %llu, "
           "\"dirty_slots_at_estimates\": %llu, \"k\": %d, \"ell\": %d, \"lambda_mode\": ",
           static_cast<long long>(ctx->n_obs), static_cast<long long>(ctx->epoch), static_cast<long long>(ctx->n_est), f,
           cum[0], cum[1], ctx->p.k, ctx->p.ell);
  j += tmp;
  j += num(ctx->p.lambda);
  j += ", \"epoch_log\": [";
  for (int64_t e = 0; e < ne; ++e) {
    const double* r = el.data() + e * kElogCols;
    j += e ? ", " : "";
    j += "{\"epoch\": " + num(r[0]) + ", \"n_obs\": " + num(r[1]) + ", \"admissions\": " + num(r[2]) +
         ", \"evictions\": " + num(r[3]) + ", \"lambda_eff\": " + num(r[4]) + ", \"E_k\": " + num(r[5]) +
         ", \"min_margin\": " + num(r[6]) + ", \"kappa_SJ\": " + num(r[7]);
    if (!ql.empty()) {   // NEXT-1: the chosen algorithm and the four candidates' estimates
      const double* q = ql.data() + e * 6;
      j += ", \"coeff_alg\": " + num(q[1]) + ", \"e2_alg4_7\": [" + num(q[2]) + ", " + num(q[3]) + ", " + num(q[4]) +
           ", " + num(q[5]) + "]";
    }
    j += "}";
  }
  j += "], \"estimate_log\": [";
  for (int64_t q = 0; q < nest; ++q) {
    const double* r = es.data() + q * kElogCols;
    j += q ? ", " : "";
    j += "{\"after_epoch\": " + num(r[0]) + ", \"e2\": " + num(r[1]) + ", \"T\": " + num(r[2]) +
         ", \"gpp\": " + num(r[3]) + ", \"frob2\": " + num(r[4]) + ", \"est_rel\": " + num(r[5]) +
         ", \"flags\": " + num(r[6]) + ", \"kappa_SJ\": " + num(r[7]) + "}";
  }
  j += "]}";
  if (needed) *needed = j.size() + 1;
  if (!buf || cap < j.size() + 1) return ctx->fail(OID_ESHAPE, "report needs %zu bytes (cap %zu)", j.size() + 1, cap);
  std::memcpy(buf, j.c_str(), j.size() + 1);
  return OID_OK;
}

oid_status oid_stats_reset(oid_ctx ctx) {
  if (!ctx) return OID_EINVAL;
  for (auto* v : {&ctx->ev_k1, &ctx->ev_post, &ctx->ev_est, &ctx->ev_a9}) {
    for (auto& pr : *v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    v->clear();
  }
  ctx->launches = 0;
  ctx->k1_launches = 0;
  return OID_OK;
}

void oid_destroy(oid_ctx ctx) {
  if (!ctx) return;
  for (cudaStream_t* sp : {&ctx->side, &ctx->side2, &ctx->side3, &ctx->gs})
    if (*sp) {
      cudaStreamSynchronize(*sp);
      cudaStreamDestroy(*sp);
    }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_k1_end) cudaEventDestroy(ctx->ev_k1_end);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  for (cudaEvent_t ev : {ctx->ev_committed, ctx->ev_gram_done, ctx->ev_sj_j, ctx->ev_est_done, ctx->ev_sj_done[0],
                         ctx->ev_sj_done[1], ctx->ev_sj_free[0], ctx->ev_sj_free[1], ctx->ev_snap_free[0], ctx->ev_snap_free[1],
                         ctx->ev_gs_done, ctx->ev_gsum_free[0], ctx->ev_gsum_free[1]})
    if (ev) cudaEventDestroy(ev);
  oid_stats_reset(ctx);
  delete ctx;
}

}  // extern "C"

namespace {
// NEXT-1 (Alg 3 steps 28-32) at the end of a commit: the Alg 4 candidate and its
// estimate through the standard A9/A10 machinery (so G is the exact basis Gram of this epoch),
// then Algs 5-7 (readings R15-R17) by GEMMs on the stream, their estimates, the device-side argmin
// and P <- P_{q*} (kept explicit as the next epoch's P_prev).
oid_status coeff_argmin(oid_ctx ctx, cudaStream_t st) {
  const Layout& L = ctx->L;
  const oid_params& p = ctx->p;
  const int t = ctx->t, ell = p.ell, l1 = p.ell1, l2 = p.ell2;
  const int nn = static_cast<int>(ctx->n_obs);
  const int nc = ctx->last_nc, nprev = nn - nc;
  oid_status s = estimate_begin_impl(ctx, st);
  if (s != OID_OK) return s;
  s = estimate_end_impl(ctx, ctx->d(L.est4), st);
  if (s != OID_OK) return s;
  CK(cudaStreamWaitEvent(st, ctx->ev_est_done, 0));
  const int par = static_cast<int>((ctx->epoch + 1) & 1);   // parity of the epoch just committed
  const double* S = ctx->d(L.S);
  const double* SJ = ctx->d(L.SJ) + static_cast<size_t>(par) * ell * t;
  const double* Z = ctx->d(L.Sjpinv) + static_cast<size_t>(par) * ell * t;
  const double* Zprev = ctx->d(L.Sjpinv) + static_cast<size_t>(par ^ 1) * ell * t;
  const double* G = ctx->d(L.G);
  const int64_t* J = ctx->ptr<int64_t>(L.J);
  const int64_t* Jp = ctx->ptr<int64_t>(L.Jprev);
  const size_t cs = static_cast<size_t>(t) * p.n_cap;
  double* P5 = ctx->d(L.Pcand);
  double* P6 = P5 + cs;
  double* P7 = P6 + cs;
  double* Gp = ctx->d(L.Gpinv);
  double* Pext = ctx->d(L.Pext);
  double* Rres = ctx->d(L.Rres);
  // G^+ (P:468's G^-1, reading R9 on G's eigenvalues; vacant slots are zero rows / columns of G)
  CK(cudaMemcpyAsync(ctx->d(L.gpH), G, sizeof(double) * t * t, cudaMemcpyDeviceToDevice, st));
  s = sym_eig(ctx, st, ctx->d(L.gpH), t, ctx->d(L.gpV), ctx->d(L.gpMu), 0, false);
  if (s != OID_OK) return s;
  psd_pinv_weights_kernel<<<1, 256, 0, st>>>(ctx->d(L.gpMu), t, ctx->d(L.gpW));
  CKL();
  scale_cols_kernel<<<blocks_for(int64_t(t) * t), 256, 0, st>>>(ctx->d(L.gpV), t, ctx->d(L.gpW), ctx->d(L.Tm));
  CKL();
  s = gemm(ctx, st, false, true, t, t, t, 1.0, ctx->d(L.Tm), t, ctx->d(L.gpV), t, 0.0, Gp, t);
  if (s != OID_OK) return s;
  // Alg 5: P5 = G^+ (S_J^T S) / l (reading R16: the 1/l of the JL-scaled Omega)
  s = gemm(ctx, st, true, false, t, nn, ell, 1.0, SJ, ell, S, ell, 0.0, Rres, t);
  if (s != OID_OK) return s;
  s = gemm(ctx, st, false, false, t, nn, t, 1.0 / ell, Gp, t, Rres, t, 0.0, P5, t);
  if (s != OID_OK) return s;
  // P_prev extended to this epoch's block (reading R15): (Omega A_Jprev)^+ Omega A_new
  if (nprev > 0) CK(cudaMemcpyAsync(Pext, ctx->d(L.Pchosen), sizeof(double) * t * nprev, cudaMemcpyDeviceToDevice, st));
  if (ctx->epoch == 1) {
    CK(cudaMemsetAsync(Pext + static_cast<size_t>(t) * nprev, 0, sizeof(double) * t * nc, st));
  } else {
    s = gemm(ctx, st, false, false, t, nc, ell, 1.0, Zprev, t, S + static_cast<size_t>(ell) * nprev, ell, 0.0,
             Pext + static_cast<size_t>(t) * nprev, t);
    if (s != OID_OK) return s;
  }
  // Alg 6 (the box's full Omega A_J, reading R17): P6 = Pz + S_J^+ (S - S_J Pz)
  CK(cudaMemcpyAsync(P6, Pext, sizeof(double) * t * nn, cudaMemcpyDeviceToDevice, st));
  zero_changed_rows_kernel<<<blocks_for(int64_t(t) * nn), 256, 0, st>>>(P6, t, nn, J, Jp);
  CKL();
  CK(cudaMemcpyAsync(Rres, S, sizeof(double) * ell * nn, cudaMemcpyDeviceToDevice, st));
  s = gemm(ctx, st, false, false, ell, nn, t, -1.0, SJ, ell, P6, t, 1.0, Rres, ell);
  if (s != OID_OK) return s;
  s = gemm(ctx, st, false, false, t, nn, ell, 1.0, Z, t, Rres, ell, 1.0, P6, t);
  if (s != OID_OK) return s;
  // Alg 7: T = A_J^+ A_Jprev = G^+ (A_J^T A_Jprev) (the QR transform R^+ Q^T written
  // with the exact Gram), P7 = T P_prev
  cross_gram_kernel<<<blocks_for(int64_t(t) * t), 256, 0, st>>>(G, ctx->d(L.Gprev), ctx->d(L.Dx), J, Jp, t, ctx->d(L.Xc));
  CKL();
  s = gemm(ctx, st, false, false, t, t, t, 1.0, Gp, t, ctx->d(L.Xc), t, 0.0, ctx->d(L.Tm), t);
  if (s != OID_OK) return s;
  s = gemm(ctx, st, false, false, t, nn, t, 1.0, ctx->d(L.Tm), t, Pext, t, 0.0, P7, t);
  if (s != OID_OK) return s;
  // NA-Hutch++ of each candidate (Alg 8 with the exact G of this epoch)
  double* cest = ctx->d(L.cest);
  for (int q = 0; q < 3; ++q) {
    double* sc = cest + 8 * q;
    s = hutch_pre(ctx, st, P5 + static_cast<size_t>(q) * cs, SJ, sc);
    if (s != OID_OK) return s;
    s = gemm(ctx, st, false, false, l2, t, t, 1.0, ctx->d(L.Q1), l2, G, t, 0.0, ctx->d(L.Q2), l2);
    if (s != OID_OK) return s;
    frob_dot_kernel<<<1, 256, 0, st>>>(ctx->d(L.Q2), l2, ctx->d(L.X2), l2, l2, t, sc);
    CKL();
    frob_dot_kernel<<<1, 256, 0, st>>>(G, t, ctx->d(L.PPt), t, t, t, sc + 3);
    CKL();
    cand_e2_kernel<<<1, 32, 0, st>>>(sc, p.ell3, ctx->d(L.scal) + SC_FROB2_EST);
    CKL();
  }
  (void)l1;
  // argmin over the unclamped estimates (first minimum), P <- P_{q*}
  argmin_pick_kernel<<<1, 32, 0, st>>>(ctx->d(L.est4), cest + 4, 8, static_cast<double>(ctx->epoch - 1),
                                       ctx->d(L.qlog) + static_cast<size_t>(ctx->epoch - 1) * 6, ctx->ptr<int>(L.qsel));
  CKL();
  copy_chosen_kernel<<<std::max(1u, std::min(blocks_for(int64_t(t) * nn), 1024u)), 256, 0, st>>>(
      ctx->d(L.Pexp), P5, static_cast<int64_t>(cs), ctx->ptr<int>(L.qsel), static_cast<int64_t>(t) * nn, ctx->d(L.Pchosen));
  CKL();
  chosen_estimate_kernel<<<1, 32, 0, st>>>(ctx->d(L.est4), cest, 8, ctx->ptr<int>(L.qsel), p.ell3,
                                           ctx->d(L.scal) + SC_FROB2_EST, ctx->d(L.est_ch));
  CKL();
  CK(cudaMemcpyAsync(ctx->d(L.Gprev), G, sizeof(double) * t * t, cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(ctx->ev_est_done, st));
  return OID_OK;
}
}  // namespace
