// Gradient-enhanced variant (paper P:625-719, reading Q17): simplex-gradient
// stencils on a 2-D or 3-D grid per field (d = 2 or 3 gradient components; d = 3 is NEXT-4, the
// channel-flow analogue of P:862-908), the augmented sketch [Omega a; Omega G^1 a; ...;
// Omega G^d a] and its Gram, and the pieces of the sketched GCV (eq:GCV_COmega).
//
// Grid layout (Q17): a snapshot stacks nf fields, field f at rows [f nx ny nz, (f+1) nx ny nz),
// node (i, j, l) at f nx ny nz + (i ny + j) nz + l (2-D: nz = 1).  For axis p with step h_p, the
// least-squares gradient over the axis neighbours (eq:gradient_estimation_mat) decouples per
// axis: with both neighbours it is the central difference (x_+ - x_-) / (2 h), with one
// neighbour the one-sided difference, with none zero -- (x_+' - x_-') / (n_p h) where x_+' = x_+
// if present else x_q (same for -).
#pragma once
#include <cstdint>
#include "common.cuh"
#include "path.cuh"

namespace oid {

struct GradGrid {
  int nf, nx, ny, nz, d;   // d = 2 (nz = 1) or 3
  double hx, hy, hz;
};

// node (i, j, l) of local row q
__device__ __forceinline__ void grad_node(const GradGrid& g, int64_t q, int& i, int& j, int& l) {
  const int64_t local = q % (static_cast<int64_t>(g.nx) * g.ny * g.nz);
  const int64_t ij = local / g.nz;
  l = static_cast<int>(local - ij * g.nz);
  i = static_cast<int>(ij / g.ny);
  j = static_cast<int>(ij - static_cast<int64_t>(i) * g.ny);
}

// stencil coefficient form of axis p at node (i, j, l): the neighbour offsets (rows) and
// 1 / (n_p h_p) (0 when the axis has no neighbour)
__device__ __forceinline__ void grad_axis(const GradGrid& g, int i, int j, int l, int p, int64_t& op, int64_t& om,
                                          double& w) {
  const int idx = p == 0 ? i : (p == 1 ? j : l);
  const int len = p == 0 ? g.nx : (p == 1 ? g.ny : g.nz);
  const int64_t stride = p == 0 ? static_cast<int64_t>(g.ny) * g.nz : (p == 1 ? g.nz : 1);
  const double h = p == 0 ? g.hx : (p == 1 ? g.hy : g.hz);
  const bool hp = idx + 1 < len, hm = idx > 0;
  op = hp ? stride : 0;
  om = hm ? -stride : 0;
  const int n = int(hp) + int(hm);
  w = n ? 1.0 / (n * h) : 0.0;
}

// GX + p gstride (m x nc, ld m, fp64) = G^p X for p < d on this shard's rows: local row q is
// global row row0 + q (its grid node); a neighbour outside [0, m) is read from the halos (SURVEY
// 8(e) route (ii)): Xlo holds the hlo global rows [row0 - hlo, row0) (ld ldlo), Xhi the hhi rows
// [row0 + m, row0 + m + hhi) (ld ldhi).  Single shard: row0 = 0, no halo is ever read.
template <typename T>
__global__ void grad_stencil_kernel(const T* __restrict__ X, int64_t ld, int64_t m, int nc, GradGrid g,
                                    double* __restrict__ GX, int64_t gstride, int64_t row0,
                                    const T* __restrict__ Xlo, int64_t ldlo, int64_t hlo,
                                    const T* __restrict__ Xhi, int64_t ldhi) {
  const int64_t total = m * nc;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e / m);
    const int64_t q = e - static_cast<int64_t>(c) * m;
    int i, j, l;
    grad_node(g, row0 + q, i, j, l);
    const T* col = X + static_cast<int64_t>(c) * ld;
    auto at = [&](int64_t r) -> double {   // local row r (possibly in a halo)
      if (r < 0) return static_cast<double>(Xlo[static_cast<int64_t>(c) * ldlo + (hlo + r)]);
      if (r >= m) return static_cast<double>(Xhi[static_cast<int64_t>(c) * ldhi + (r - m)]);
      return static_cast<double>(col[r]);
    };
    for (int p = 0; p < g.d; ++p) {
      int64_t op, om;
      double w;
      grad_axis(g, i, j, l, p, op, om, w);
      GX[p * gstride + e] = (at(q + op) - at(q + om)) * w;
    }
  }
}

// A3 of the augmented sketch: Yh = [Y_0; ...; Y_d] ((d+1) ell x nc; Y_0 = Y0, Y_p = Yg +
// (p-1) ystride, each col-major ell x nc followed by its nc norms); gram ((d+1) ell)^2 += Yh Yh^T;
// S_0 = S, S_p = Sg + (p-1) sstride <- append; scal[FROB2] += sum n_0, scal[FROB2_AUG] += sum_p n_p
__global__ void gram_update_aug_kernel(const double* __restrict__ Y0, const double* __restrict__ Yg, int64_t ystride,
                                       int na, int ell, int nc, double* __restrict__ gram, double* __restrict__ S,
                                       double* __restrict__ Sg, int64_t sstride, int64_t n0, double* __restrict__ scal) {
  const int ng = na * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(ng) * ng;
  auto blk = [&](int part) -> const double* { return part == 0 ? Y0 : Yg + (part - 1) * ystride; };
  auto yh = [&](int r, int j) -> double { return blk(r / ell)[(r % ell) + static_cast<int64_t>(j) * ell]; };
  if (idx < nn) {
    const int r = static_cast<int>(idx % ng), c = static_cast<int>(idx / ng);
    double s = gram[idx];
    for (int j = 0; j < nc; ++j) s = fma(yh(r, j), yh(c, j), s);
    gram[idx] = s;
  }
  const int64_t ny = static_cast<int64_t>(ell) * nc;
  if (idx < ny) {
    S[n0 * ell + idx] = Y0[idx];
    for (int part = 1; part < na; ++part) Sg[(part - 1) * sstride + n0 * ell + idx] = blk(part)[idx];
  }
  if (idx == 0) {
    double f = scal[SC_FROB2], fa = scal[SC_FROB2_AUG];
    for (int j = 0; j < nc; ++j) {
      f += Y0[ny + j];
      for (int part = 0; part < na; ++part) fa += blk(part)[ny + j];
    }
    scal[SC_FROB2] = f;
    scal[SC_FROB2_AUG] = fa;
  }
}

// Yc ((d+1) ell x (t + nc)): augmented sketches of the basis slots (zero for vacant) then candidates
__global__ void gather_scored_aug_kernel(const double* __restrict__ S, const double* __restrict__ Sg, int64_t sstride,
                                         const int64_t* __restrict__ J, int t, const double* __restrict__ Y0,
                                         const double* __restrict__ Yg, int64_t ystride, int na, int nc, int ell,
                                         double* __restrict__ Yc) {
  const int ng = na * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(ng) * (t + nc);
  if (idx >= total) return;
  const int col = static_cast<int>(idx / ng), r = static_cast<int>(idx % ng);
  const int part = r / ell, rr = r % ell;
  double v = 0.0;
  if (col < t) {
    const int64_t j = J[col];
    const double* Sp = part == 0 ? S : Sg + (part - 1) * sstride;
    if (j >= 0) v = Sp[j * ell + rr];
  } else {
    const double* Yp = part == 0 ? Y0 : Yg + (part - 1) * ystride;
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

// W(:, j) = G^p omega_{s0 + j} (m x ns, ld m, this shard's rows row0 ..): the stencil applied to
// sketch row s0 + j (neighbours of a slab-edge row are generated, not exchanged), so that
// Omega W = (Omega G^p Omega^T)(:, s0 .. s0 + ns) comes out of the tensor-core K1 (grad_ogo)
__global__ void omega_g_cols_kernel(int s0, int ns, int64_t m, GradGrid g, int p, uint32_t key0, uint32_t key1,
                                    double scale, double* __restrict__ W, int64_t row0) {
  __shared__ double qd[16];
  if (threadIdx.x < 16) qd[threadIdx.x] = c_qtab_f64[threadIdx.x];
  __syncthreads();
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < m * ns;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx / m);
    const int64_t q = row0 + (idx - static_cast<int64_t>(j) * m);   // global row: Omega is keyed on it (8(e)
    int i, jj, l;                                                     // route (i), no halo needed)
    grad_node(g, q, i, jj, l);
    int64_t op, om;
    double w;
    grad_axis(g, i, jj, l, p, op, om, w);
    W[idx] = (w == 0.0) ? 0.0
                        : (omega_entry(s0 + j, q + op, key0, key1, qd, scale) -
                           omega_entry(s0 + j, q + om, key0, key1, qd, scale)) * w;
  }
}

// out ((d+1) ell x ncol) = [A0; c A_1; ...; c A_d] stacked by rows (A_p = Ag + (p-1) astride,
// each ell x ncol, ld ell); with J != nullptr, column j of A_p is A_p(:, J[j]) (zero for vacant slots)
__global__ void stack_aug_kernel(const double* __restrict__ A0, const double* __restrict__ Ag, int64_t astride, int na,
                                 int ell, int ncol, const int64_t* __restrict__ J, double c, double* __restrict__ out) {
  const int ng = na * ell;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(ng) * ncol) return;
  const int col = static_cast<int>(idx / ng), r = static_cast<int>(idx % ng);
  const int part = r / ell, rr = r % ell;
  int64_t src = col;
  if (J) src = J[col];
  double v = 0.0;
  if (src >= 0) {
    const double* A = part == 0 ? A0 : Ag + (part - 1) * astride;
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
