// Fast path of A4/A5 (ridge regulariser and ridge scores) for
// ell <= kTriMaxN: the sketch Gram G = S S^T is reduced to tridiagonal form T = Q^T G Q by
// Householder reflections on one 16-CTA thread-block cluster (G held in the cluster's shared
// memory, 32 rows per CTA); the eigenvalues of T (= of G) come from Sturm-count multisection,
// which gives E_k and lambda; when the ridge shift s = ell*lambda keeps every eigenvalue of
// G + sI above the pseudo-inverse cutoff (s >= 1e-8 (mu_max + s), reading R9 then drops no
// term), the scores are tau(y) = (Q^T y)^T (T + sI)^-1 (Q^T y), one LDL^T solve of a
// tridiagonal.  Otherwise the eigenvector (Jacobi) path runs instead, gated on the device.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "path.cuh"

namespace oid {
namespace cg2 = cooperative_groups;

constexpr int kTriCtas = 16;
constexpr int kTriMaxN = 512;
constexpr int kTriRows = kTriMaxN / kTriCtas;   // 32 rows per CTA at the maximum size

// Householder tridiagonalisation of the symmetric n x n matrix A (col-major), n <= 512.
// Outputs: d (n), e (n-1) of T; reflectors H_k = I - tau_k v_k v_k^T, k = 0..n-3, with v_k
// stored in Vh(:, k) (rows k+1..n-1; zero elsewhere) and tau_k in tauv[k].
// gv (n + 1), gp (n + kTriCtas): global broadcast buffers.  Launch: 16 CTAs in one cluster.
__global__ void __cluster_dims__(kTriCtas, 1, 1) __launch_bounds__(256)
tridiag_cluster_kernel(const double* __restrict__ A, int n, double* __restrict__ d, double* __restrict__ e,
                       double* __restrict__ Vh, double* __restrict__ tauv, double* __restrict__ gv,
                       double* __restrict__ gp) {
  cg2::cluster_group cluster = cg2::this_cluster();
  extern __shared__ double tri_smem[];
  const int c = static_cast<int>(cluster.block_rank());
  const int R = (n + kTriCtas - 1) / kTriCtas;
  const int r0 = c * R, r1 = min(n, r0 + R);
  double* Al = tri_smem;                 // [R][n] rows r0..r1-1 (row-major)
  double* vv = Al + R * n;               // [n]
  double* pw = vv + n;                   // [n]  p, then w
  __shared__ double red[8];
  __shared__ double sc[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < (r1 - r0) * n; idx += 256) {
    const int i = idx / n, j = idx - i * n;
    Al[i * n + j] = A[j + static_cast<int64_t>(r0 + i) * n];     // row r0+i = column r0+i (symmetric)
  }
  __syncthreads();
  cluster.sync();
  for (int k = 0; k < n - 2; ++k) {
    const int owner = k / R;
    const int len = n - k - 1;
    if (c == owner) {
      // Householder vector of row k (columns k+1..n-1): v = x - alpha e1, tau = 2 / v^T v
      const double* x = Al + (k - r0) * n + (k + 1);
      double ss = 0.0;
      for (int j = tid; j < len; j += 256) ss = fma(x[j], x[j], ss);
      ss = block_sum<256>(ss, red);
      const double x0 = x[0];
      double alpha = 0.0, tau = 0.0, v0 = 0.0;
      const double tail = ss - x0 * x0;
      if (tail > 0.0) {
        alpha = -copysign(sqrt(ss), x0);
        v0 = x0 - alpha;
        tau = 2.0 / (tail + v0 * v0);
      } else {
        alpha = x0;    // already tridiagonal in this column: H_k = I
      }
      for (int j = tid; j < len; j += 256) {
        const double vj = (j == 0) ? v0 : x[j];
        const double out = tau != 0.0 ? vj : 0.0;
        gv[k + 1 + j] = out;
        Vh[(k + 1 + j) + static_cast<int64_t>(k) * n] = out;
      }
      if (tid == 0) {
        gv[0] = tau;
        tauv[k] = tau;
        d[k] = Al[(k - r0) * n + k];
        e[k] = alpha;
      }
    }
    cluster.sync();
    const double tau = __ldcg(gv);
    for (int j = k + 1 + tid; j < n; j += 256) vv[j] = __ldcg(gv + j);
    __syncthreads();
    // p = tau A v on my rows i > k; K partial = v^T p
    const int i0 = max(r0, k + 1);
    double kp = 0.0;
    if (tau != 0.0) {
      for (int i = i0 + warp; i < r1; i += 8) {
        const double* row = Al + (i - r0) * n;
        double s = 0.0;
        for (int j = k + 1 + lane; j < n; j += 32) s = fma(row[j], vv[j], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          const double pi = tau * s;
          gp[i] = pi;
          pw[i] = pi;
        }
      }
    }
    __syncthreads();
    if (tau != 0.0 && tid == 0) {
      for (int i = i0; i < r1; ++i) kp = fma(vv[i], pw[i], kp);   // fixed order
      gp[n + c] = kp;
    }
    cluster.sync();
    if (tau != 0.0) {
      if (tid == 0) {
        double K = 0.0;
        for (int q = 0; q < kTriCtas; ++q) K += __ldcg(gp + n + q);
        sc[0] = 0.5 * tau * K;
      }
      for (int j = k + 1 + tid; j < n; j += 256) pw[j] = __ldcg(gp + j);
      __syncthreads();
      const double h = sc[0];
      for (int j = k + 1 + tid; j < n; j += 256) pw[j] = pw[j] - h * vv[j];   // w = p - (tau K / 2) v
      __syncthreads();
      // A <- A - v w^T - w v^T on my rows i > k, columns j > k
      for (int i = i0; i < r1; ++i) {
        double* row = Al + (i - r0) * n;
        const double vi = vv[i], wi = pw[i];
        for (int j = k + 1 + tid; j < n; j += 256) row[j] = row[j] - vi * pw[j] - wi * vv[j];
      }
    }
    __syncthreads();
  }
  // trailing 2 x 2 block
  if (n >= 2) {
    const int a = n - 2, b = n - 1;
    if (tid == 0 && a >= r0 && a < r1) { d[a] = Al[(a - r0) * n + a]; e[a] = Al[(a - r0) * n + b]; }
    if (tid == 0 && b >= r0 && b < r1) d[b] = Al[(b - r0) * n + b];
  } else if (n == 1 && c == 0 && tid == 0) {
    d[0] = Al[0];
  }
  cluster.sync();
}

// Eigenvalues of the symmetric tridiagonal (d, e) in descending order, mu[i] = (i+1)-th
// largest, by Sturm-count multisection: one warp per eigenvalue, 32 shifts per iteration.
__device__ __forceinline__ int sturm_count_gt(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                              double x, double pivmin) {
  // number of eigenvalues < x (negative pivots of LDL^T of T - x I)
  int neg = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  neg += q < 0.0;
  for (int j = 1; j < n; ++j) {
    q = d[j] - x - e2[j - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    neg += q < 0.0;
  }
  return n - neg;   // eigenvalues >= x
}

__global__ void __launch_bounds__(256) multisect_kernel(const double* __restrict__ d, const double* __restrict__ e, int n,
                                                        double* __restrict__ mu) {
  extern __shared__ double ms_smem[];
  double* ds = ms_smem;
  double* e2 = ms_smem + n;
  __shared__ double bnd[3];
  const int tid = threadIdx.x;
  for (int j = tid; j < n; j += blockDim.x) {
    ds[j] = d[j];
    if (j < n - 1) e2[j] = e[j] * e[j];
  }
  __syncthreads();
  if (tid == 0) {
    double lo = INFINITY, hi = -INFINITY, tmax = 0.0, emax2 = 0.0;
    for (int j = 0; j < n; ++j) {
      const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + (j < n - 1 ? fabs(e[j]) : 0.0);
      lo = fmin(lo, d[j] - r);
      hi = fmax(hi, d[j] + r);
      tmax = fmax(tmax, fabs(d[j]) + r);
      if (j < n - 1) emax2 = fmax(emax2, e[j] * e[j]);
    }
    const double eps = 2.220446049250313e-16;
    const double pad = 2.0 * eps * tmax + 1e-300;
    bnd[0] = lo - pad;
    bnd[1] = hi + pad;
    bnd[2] = 2.2250738585072014e-308 * fmax(1.0, emax2);   // LAPACK pivmin
  }
  __syncthreads();
  const double pivmin = bnd[2];
  const int warp = (blockIdx.x * blockDim.x + tid) >> 5, lane = tid & 31;
  if (warp >= n) return;
  const int i = warp;                     // target: (i+1)-th largest
  double lo = bnd[0], hi = bnd[1];
  const double eps = 2.220446049250313e-16;
  for (int it = 0; it < 40; ++it) {
    if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + pivmin) break;
    const double x = lo + (hi - lo) * static_cast<double>(lane + 1) / 33.0;
    const int gt = sturm_count_gt(ds, e2, n, x, pivmin);   // #eigenvalues >= x
    // new lo: largest x with gt >= i+1; new hi: smallest x with gt <= i
    const unsigned okm = __ballot_sync(0xffffffffu, gt >= i + 1);
    const int last_ok = okm ? 31 - __clz(okm) : -1;          // lanes with larger x have smaller counts
    const double nlo = last_ok >= 0 ? lo + (hi - lo) * static_cast<double>(last_ok + 1) / 33.0 : lo;
    const double nhi = last_ok < 31 ? lo + (hi - lo) * static_cast<double>(last_ok + 2) / 33.0 : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) mu[i] = 0.5 * (lo + hi);
}

// lambda (reading R8) from the descending eigenvalues mu; ridge shift s = ell lambda (R3);
// gate[0] = 1 when the tridiagonal score path is exact (s >= 1e-8 (mu_0 + s), n <= 512),
// gate[1] = 1 - gate[0] (eigenvector path).  With gate[0], also the LDL^T of T + sI:
// ldl[0..n) = 1/D_j, ldl[n..2n-1) = L_j.
__global__ void lambda_sorted_kernel(const double* __restrict__ mu, int n, int k, const double* __restrict__ gram,
                                     double lam_param, int ell, double* __restrict__ scal, int* __restrict__ gate,
                                     const double* __restrict__ d, const double* __restrict__ e,
                                     double* __restrict__ ldl, int tri_ok) {
  __shared__ double red[8];
  double tr = 0.0;
  for (int i = threadIdx.x; i < ell; i += blockDim.x) tr += gram[static_cast<int64_t>(i) * ell + i];
  tr = block_sum<256>(tr, red);
  if (threadIdx.x != 0) return;
  double Ek = 0.0;
  for (int i = 0; i < k && i < n; ++i) Ek += mu[i];
  const double frob2 = scal[SC_FROB2];
  double lam;
  if (lam_param >= 0.0) lam = lam_param;
  else if (lam_param == -1.0) lam = fmax(0.0, (frob2 - Ek / ell) / k);
  else lam = fmax(0.0, (tr - Ek) / (static_cast<double>(ell) * k));
  const double shift = ell * lam;
  const double dmax = (n > 0 ? mu[0] : 0.0) + shift;
  scal[SC_LAM] = lam;
  scal[SC_EK] = Ek;
  scal[SC_SHIFT] = shift;
  scal[SC_TRACE] = tr;
  scal[SC_DMAX] = dmax;
  const int fast = tri_ok && shift > 0.0 && shift >= 1e-8 * dmax;
  gate[0] = fast;
  gate[1] = !fast;
  if (fast) {
    double Dj = d[0] + shift;
    ldl[0] = 1.0 / Dj;
    for (int j = 1; j < n; ++j) {
      const double Lj = e[j - 1] / Dj;
      ldl[n + j - 1] = Lj;
      Dj = d[j] + shift - Lj * e[j - 1];
      ldl[j] = 1.0 / Dj;
    }
  }
}

// tau(y) = z^T (T + sI)^-1 z, z = Q^T y = H_{n-3} ... H_0 y; y = column j of Yc (ell x ncol).
// One CTA per column.  Runs when gate[0] != 0.
__global__ void __launch_bounds__(256) tri_scores_kernel(const double* __restrict__ Yc, int n, int ncol,
                                                         const double* __restrict__ Vh, const double* __restrict__ tauv,
                                                         const double* __restrict__ ldl, const int* __restrict__ gate,
                                                         double* __restrict__ tau_out) {
  if (gate[0] == 0) return;
  __shared__ double z[kTriMaxN];
  __shared__ double red[8];
  const int j = blockIdx.x, tid = threadIdx.x;
  if (j >= ncol) return;
  for (int i = tid; i < n; i += 256) z[i] = Yc[static_cast<int64_t>(j) * n + i];
  __syncthreads();
  for (int k = 0; k < n - 2; ++k) {
    const double tk = tauv[k];
    if (tk == 0.0) continue;                      // uniform across the CTA
    const double* v = Vh + static_cast<int64_t>(k) * n;
    double s = 0.0;
    for (int i = k + 1 + tid; i < n; i += 256) s = fma(v[i], z[i], s);
    s = block_sum<256>(s, red);
    const double f = tk * s;
    for (int i = k + 1 + tid; i < n; i += 256) z[i] = fma(-f, v[i], z[i]);
    __syncthreads();
  }
  if (tid == 0) {
    double y = z[0];
    double acc = y * y * ldl[0];
    for (int i = 1; i < n; ++i) {
      y = z[i] - ldl[n + i - 1] * y;
      acc = fma(y * y, ldl[i], acc);
    }
    tau_out[j] = acc;
  }
}

// SPD solve gate for A = Q T Q^T (tridiagonalised): mu = eigenvalues (descending).  gate[0] = 1
// when mu_min > 0 and mu_max <= kmax2 mu_min (no pseudo-inverse cutoff can act, reading R9, and
// the normal-equation error kmax2 eps stays far below the 1e-5 parity bar); then ldl holds the
// LDL^T of T (1/D_j, L_j) and *kappa_out = sqrt(mu_max / mu_min).  gate[1] = !gate[0].
__global__ void spd_gate_kernel(const double* __restrict__ mu, int n, double kmax2, const double* __restrict__ d,
                                const double* __restrict__ e, double* __restrict__ ldl, int* __restrict__ gate,
                                double* __restrict__ kappa_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double mx = n > 0 ? mu[0] : 0.0, mn = n > 0 ? mu[n - 1] : 0.0;
  const int ok = n > 0 && mn > 0.0 && mx <= kmax2 * mn;
  gate[0] = ok;
  gate[1] = !ok;
  if (!ok) return;
  if (kappa_out) *kappa_out = sqrt(mx / mn);
  double Dj = d[0];
  ldl[0] = 1.0 / Dj;
  for (int j = 1; j < n; ++j) {
    const double Lj = e[j - 1] / Dj;
    ldl[n + j - 1] = Lj;
    Dj = d[j] - Lj * e[j - 1];
    ldl[j] = 1.0 / Dj;
  }
}

// X(:, c) = A^-1 R(:, c) with A = Q T Q^T: z = Q^T r, solve T u = z (LDL^T), x = Q u.
// One CTA per right-hand side; runs when gate[0] != 0.  in_transposed: R(i, c) = R[c + i ldr];
// out_transposed: write X^T (nrhs x n).
__global__ void __launch_bounds__(256) tri_solve_kernel(const double* __restrict__ R, int64_t ldr, int in_transposed,
                                                        int n, int nrhs,
                                                        const double* __restrict__ Vh, const double* __restrict__ tauv,
                                                        const double* __restrict__ ldl, const int* __restrict__ gate,
                                                        double* __restrict__ X, int64_t ldx, int out_transposed) {
  if (gate[0] == 0) return;
  __shared__ double z[kTriMaxN];
  __shared__ double red[8];
  const int c = blockIdx.x, tid = threadIdx.x;
  if (c >= nrhs) return;
  for (int i = tid; i < n; i += 256)
    z[i] = in_transposed ? R[c + static_cast<int64_t>(i) * ldr] : R[static_cast<int64_t>(c) * ldr + i];
  __syncthreads();
  for (int k = 0; k < n - 2; ++k) {                 // z = H_{n-3} ... H_0 r
    const double tk = tauv[k];
    if (tk == 0.0) continue;
    const double* v = Vh + static_cast<int64_t>(k) * n;
    double s = 0.0;
    for (int i = k + 1 + tid; i < n; i += 256) s = fma(v[i], z[i], s);
    s = block_sum<256>(s, red);
    for (int i = k + 1 + tid; i < n; i += 256) z[i] = fma(-tk * s, v[i], z[i]);
    __syncthreads();
  }
  if (tid == 0) {                                   // T u = z by LDL^T
    for (int i = 1; i < n; ++i) z[i] -= ldl[n + i - 1] * z[i - 1];
    for (int i = 0; i < n; ++i) z[i] *= ldl[i];
    for (int i = n - 2; i >= 0; --i) z[i] -= ldl[n + i] * z[i + 1];
  }
  __syncthreads();
  for (int k = n - 3; k >= 0; --k) {               // x = H_0 ... H_{n-3} u
    const double tk = tauv[k];
    if (tk == 0.0) continue;
    const double* v = Vh + static_cast<int64_t>(k) * n;
    double s = 0.0;
    for (int i = k + 1 + tid; i < n; i += 256) s = fma(v[i], z[i], s);
    s = block_sum<256>(s, red);
    for (int i = k + 1 + tid; i < n; i += 256) z[i] = fma(-tk * s, v[i], z[i]);
    __syncthreads();
  }
  for (int i = tid; i < n; i += 256) {
    if (out_transposed) X[static_cast<int64_t>(i) * ldx + c] = z[i];
    else X[static_cast<int64_t>(c) * ldx + i] = z[i];
  }
}

// A(i, i) = cval for zero rows/columns of a Gram (vacant basis slots, reading R10) where cval =
// max diagonal, so the inverse leaves their coefficient rows zero and the spectrum bounds of the
// occupied block are unchanged.
__global__ void fill_vacant_diag_kernel(double* __restrict__ A, int n, const int64_t* __restrict__ J) {
  __shared__ double mx;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, A[i + static_cast<int64_t>(i) * n]);
    mx = m > 0.0 ? m : 1.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (J[i] < 0) A[i + static_cast<int64_t>(i) * n] = mx;
}

}  // namespace oid
