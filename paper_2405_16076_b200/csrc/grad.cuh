// Gradient-enhanced variant (paper P:625-719, reading Q17): simplex-gradient
// stencils on a 2-D grid per field, the augmented sketch [Omega a; Omega G^1 a; Omega G^2 a]
// and its Gram, and the pieces of the sketched GCV (eq:GCV_COmega).
//
// Grid layout (Q17): a snapshot stacks nf fields, field f at rows [f nx ny, (f+1) nx ny),
// node (i, j) at f nx ny + i ny + j.  For axis p with step h_p, the least-squares gradient over
// the axis neighbours (eq:gradient_estimation_mat) decouples per axis: with both neighbours it
// is the central difference (x_+ - x_-) / (2 h), with one neighbour the one-sided difference,
// with none zero -- (x_+' - x_-') / (n_p h) where x_+' = x_+ if present else x_q (same for -).
#pragma once
#include <cstdint>
#include "common.cuh"
#include "path.cuh"

namespace oid {

struct GradGrid {
  int nf, nx, ny;
  double hx, hy;
};

// stencil coefficient form of one axis at node (i, j): returns the neighbour offsets (rows) and
// 1 / (n_p h_p) (0 when the axis has no neighbour)
__device__ __forceinline__ void grad_axis(const GradGrid& g, int i, int j, int p, int64_t& op, int64_t& om, double& w) {
  if (p == 0) {
    const bool hp = i + 1 < g.nx, hm = i > 0;
    op = hp ? g.ny : 0;
    om = hm ? -g.ny : 0;
    const int n = int(hp) + int(hm);
    w = n ? 1.0 / (n * g.hx) : 0.0;
  } else {
    const bool hp = j + 1 < g.ny, hm = j > 0;
    op = hp ? 1 : 0;
    om = hm ? -1 : 0;
    const int n = int(hp) + int(hm);
    w = n ? 1.0 / (n * g.hy) : 0.0;
  }
}

// GX[p] (m x nc, ld m, fp64) = G^p X for p = 0, 1 (the block's rows are the whole grid: single shard)
template <typename T>
__global__ void grad_stencil_kernel(const T* __restrict__ X, int64_t ld, int64_t m, int nc, GradGrid g,
                                    double* __restrict__ GX0, double* __restrict__ GX1) {
  const int64_t total = m * nc;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e / m);
    const int64_t q = e - static_cast<int64_t>(c) * m;
    const int64_t local = q % (static_cast<int64_t>(g.nx) * g.ny);
    const int i = static_cast<int>(local / g.ny), j = static_cast<int>(local % g.ny);
    const T* col = X + static_cast<int64_t>(c) * ld;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      int64_t op, om;
      double w;
      grad_axis(g, i, j, p, op, om, w);
      const double v = (static_cast<double>(col[q + op]) - static_cast<double>(col[q + om])) * w;
      (p == 0 ? GX0 : GX1)[e] = v;
    }
  }
}

// A3 of the augmented sketch: Yh = [Y0; Y1; Y2] (3 ell x nc, each Yp col-major ell x nc followed
// by its nc norms); gram (3 ell)^2 += Yh Yh^T; S, S1, S2 <- append; scal[FROB2] += sum n0,
// scal[FROB2_AUG] += sum (n0 + n1 + n2)
__global__ void gram_update_aug_kernel(const double* __restrict__ Y0, const double* __restrict__ Y1,
                                       const double* __restrict__ Y2, int ell, int nc, double* __restrict__ gram,
                                       double* __restrict__ S, double* __restrict__ S1, double* __restrict__ S2,
                                       int64_t n0, double* __restrict__ scal) {
  const int ng = 3 * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(ng) * ng;
  auto yh = [&](int r, int j) -> double {
    const double* Y = r < ell ? Y0 : (r < 2 * ell ? Y1 : Y2);
    return Y[(r % ell) + static_cast<int64_t>(j) * ell];
  };
  if (idx < nn) {
    const int r = static_cast<int>(idx % ng), c = static_cast<int>(idx / ng);
    double s = gram[idx];
    for (int j = 0; j < nc; ++j) s = fma(yh(r, j), yh(c, j), s);
    gram[idx] = s;
  }
  const int64_t ny = static_cast<int64_t>(ell) * nc;
  if (idx < ny) {
    S[n0 * ell + idx] = Y0[idx];
    S1[n0 * ell + idx] = Y1[idx];
    S2[n0 * ell + idx] = Y2[idx];
  }
  if (idx == 0) {
    double f = scal[SC_FROB2], fa = scal[SC_FROB2_AUG];
    for (int j = 0; j < nc; ++j) {
      f += Y0[ny + j];
      fa += Y0[ny + j] + Y1[ny + j] + Y2[ny + j];
    }
    scal[SC_FROB2] = f;
    scal[SC_FROB2_AUG] = fa;
  }
}

// Yc (3 ell x (t + nc)): augmented sketches of the basis slots (zero for vacant) then candidates
__global__ void gather_scored_aug_kernel(const double* __restrict__ S, const double* __restrict__ S1,
                                         const double* __restrict__ S2, const int64_t* __restrict__ J, int t,
                                         const double* __restrict__ Y0, const double* __restrict__ Y1,
                                         const double* __restrict__ Y2, int nc, int ell, double* __restrict__ Yc) {
  const int ng = 3 * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(ng) * (t + nc);
  if (idx >= total) return;
  const int col = static_cast<int>(idx / ng), r = static_cast<int>(idx % ng);
  const int part = r / ell, rr = r % ell;
  double v = 0.0;
  if (col < t) {
    const int64_t j = J[col];
    const double* Sp = part == 0 ? S : (part == 1 ? S1 : S2);
    if (j >= 0) v = Sp[j * ell + rr];
  } else {
    const double* Yp = part == 0 ? Y0 : (part == 1 ? Y1 : Y2);
    v = Yp[static_cast<int64_t>(col - t) * ell + rr];
  }
  Yc[idx] = v;
}

// unit-variance Omega(r, i) (readings R1, R2): Philox block (i >> 5, r), nibble i & 31
__device__ __forceinline__ double omega_entry(int r, int64_t i, uint32_t key0, uint32_t key1, const double* qd,
                                              double scale) {
  const U4 w = philox4x32_10(static_cast<uint32_t>(i >> 5), static_cast<uint32_t>(r), 0u, 0u, key0, key1);
  const uint32_t words[4] = {w.x, w.y, w.z, w.w};
  const int rr = static_cast<int>(i & 31);
  return scale * qd[(words[rr >> 3] >> (4 * (rr & 7))) & 15u];
}

// OGO_p(r, s) = (Omega G^p Omega^T)(r, s) = sum_q Omega(r, q) (G^p row q) . Omega(s, :)^T, for
// p = blockIdx.z; one thread per (r, s), Omega regenerated (finalize-only; cost ell^2 m Philox)
__global__ void omega_g_omega_kernel(int ell, int64_t m, GradGrid g, uint32_t key0, uint32_t key1, double scale,
                                     double* __restrict__ OGO) {
  __shared__ double qd[16];
  if (threadIdx.x < 16) qd[threadIdx.x] = c_qtab_f64[threadIdx.x];
  __syncthreads();
  const int p = blockIdx.z;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(ell) * ell) return;
  const int r = static_cast<int>(idx % ell), s = static_cast<int>(idx / ell);
  double acc = 0.0;
  for (int64_t q = 0; q < m; ++q) {
    const int64_t local = q % (static_cast<int64_t>(g.nx) * g.ny);
    const int i = static_cast<int>(local / g.ny), j = static_cast<int>(local % g.ny);
    int64_t op, om;
    double w;
    grad_axis(g, i, j, p, op, om, w);
    if (w == 0.0) continue;
    const double gq = (omega_entry(s, q + op, key0, key1, qd, scale) - omega_entry(s, q + om, key0, key1, qd, scale)) * w;
    acc = fma(omega_entry(r, q, key0, key1, qd, scale), gq, acc);
  }
  OGO[static_cast<int64_t>(p) * ell * ell + idx] = acc;
}

// W(:, j) = G^p omega_{s0 + j} (m x ns, ld m): the stencil applied to sketch row s0 + j, so that
// Omega W = (Omega G^p Omega^T)(:, s0 .. s0 + ns) comes out of the tensor-core K1 (grad_ogo)
__global__ void omega_g_cols_kernel(int s0, int ns, int64_t m, GradGrid g, int p, uint32_t key0, uint32_t key1,
                                    double scale, double* __restrict__ W) {
  __shared__ double qd[16];
  if (threadIdx.x < 16) qd[threadIdx.x] = c_qtab_f64[threadIdx.x];
  __syncthreads();
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < m * ns;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx / m);
    const int64_t q = idx - static_cast<int64_t>(j) * m;
    const int64_t local = q % (static_cast<int64_t>(g.nx) * g.ny);
    const int i = static_cast<int>(local / g.ny), jj = static_cast<int>(local % g.ny);
    int64_t op, om;
    double w;
    grad_axis(g, i, jj, p, op, om, w);
    W[idx] = (w == 0.0) ? 0.0
                        : (omega_entry(s0 + j, q + op, key0, key1, qd, scale) -
                           omega_entry(s0 + j, q + om, key0, key1, qd, scale)) * w;
  }
}

// out (rows x ncol) = [A0; c A1; c A2] stacked by rows (each A_p rows_p = ell x ncol, ld ell);
// with J != nullptr, column j of A_p is A_p(:, J[j]) (zero for vacant slots)
__global__ void stack3_kernel(const double* __restrict__ A0, const double* __restrict__ A1, const double* __restrict__ A2,
                              int ell, int ncol, const int64_t* __restrict__ J, double c, double* __restrict__ out) {
  const int ng = 3 * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(ng) * ncol) return;
  const int col = static_cast<int>(idx / ng), r = static_cast<int>(idx % ng);
  const int part = r / ell, rr = r % ell;
  int64_t src = col;
  if (J) src = J[col];
  double v = 0.0;
  if (src >= 0) {
    const double* A = part == 0 ? A0 : (part == 1 ? A1 : A2);
    v = (part == 0 ? 1.0 : c) * A[src * ell + rr];
  }
  out[idx] = v;
}

// C (rows x cols, ld ldc) += A (ld lda)
__global__ void add_strided_kernel(const double* __restrict__ A, int64_t lda, int rows, int cols, double* __restrict__ C,
                                   int64_t ldc) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * cols) return;
  const int r = static_cast<int>(idx % rows), c = static_cast<int>(idx / rows);
  C[r + c * ldc] += A[r + c * lda];
}

// C = A + mu B (elementwise, n entries)
__global__ void axpby_kernel(const double* __restrict__ A, const double* __restrict__ B, double mu, int64_t n,
                             double* __restrict__ C) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < n) C[idx] = fma(mu, B[idx], A[idx]);
}

// out[0] = ||E||_F^2 / (ell - tr C)^2 with E = S - C S (ell x n, C ell x ell): GCV
__global__ void gcv_final_kernel(const double* __restrict__ E, int64_t nE, const double* __restrict__ C, int ell,
                                 double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nE; i += blockDim.x) s = fma(E[i], E[i], s);
  s = block_sum<256>(s, red);
  double tr = 0.0;
  for (int i = threadIdx.x; i < ell; i += blockDim.x) tr += C[static_cast<int64_t>(i) * ell + i];
  tr = block_sum<256>(tr, red);
  if (threadIdx.x == 0) {
    const double d = static_cast<double>(ell) - tr;
    out[0] = s / (d * d);
  }
}

}  // namespace oid
