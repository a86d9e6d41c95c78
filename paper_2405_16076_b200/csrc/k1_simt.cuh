// K1, CUDA-core variant: Y_part = Z(:, slab) * X_blk and n_j = sum_i x_ij^2 in one read of X
// (Alg 3 steps 10 and 13).  Z entries are generated in registers from Philox
// (reading R1) through the Gauss-16 levels (reading R2); products and sums in fp64 (DFMA).
#pragma once
#include "common.cuh"

namespace oid {

__constant__ double c_qtab_f64[16];    // L(n) = q(n) + 1/2 as exact doubles (set at init)

constexpr int kGrp = 32;               // data rows per Philox block (8 nibbles x 4 words)

// One CTA owns a contiguous range of global 32-row groups and 256*RPT sketch rows
// (blockIdx.y selects the sketch-row slice).  Rows outside [row_begin, row_end) read as 0.
template <typename T, int NCB, int RPT>
__global__ void __launch_bounds__(kThreads, 1)
k1_simt_kernel(const T* __restrict__ X, int64_t ld, int ncols, int64_t row_begin, int64_t row_end,
               int64_t grp_begin, int64_t grp_end, int64_t grp_per_cta, int ell, uint32_t key0, uint32_t key1,
               double* __restrict__ part, double* __restrict__ npart) {
  __shared__ double xs[2][kGrp][NCB];
  __shared__ double qd[16];
  const int tid = threadIdx.x;
  if (tid < 16) qd[tid] = c_qtab_f64[tid];

  const int64_t g0 = grp_begin + static_cast<int64_t>(blockIdx.x) * grp_per_cta;
  const int64_t g1 = min(grp_end, g0 + grp_per_cta);
  const int rbase = blockIdx.y * (kThreads * RPT);

  double acc[RPT][NCB];
#pragma unroll
  for (int k = 0; k < RPT; ++k)
#pragma unroll
    for (int j = 0; j < NCB; ++j) acc[k][j] = 0.0;
  double nrm = 0.0;

  constexpr int kLoads = (kGrp * NCB + kThreads - 1) / kThreads;
  double pre[kLoads];
  auto fetch = [&](int64_t gq) {
#pragma unroll
    for (int it = 0; it < kLoads; ++it) {
      const int e = tid + it * kThreads;
      const int rr = e & (kGrp - 1), j = e / kGrp;
      const int64_t g = gq * kGrp + rr;
      double v = 0.0;
      if (j < ncols && g >= row_begin && g < row_end) v = static_cast<double>(X[(g - row_begin) + j * ld]);
      pre[it] = v;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int it = 0; it < kLoads; ++it) {
      const int e = tid + it * kThreads;
      if (e < kGrp * NCB) xs[buf][e & (kGrp - 1)][e / kGrp] = pre[it];
    }
  };

  if (g0 < g1) { fetch(g0); }
  int buf = 0;
  for (int64_t gq = g0; gq < g1; ++gq) {
    stash(buf);
    __syncthreads();
    if (gq + 1 < g1) fetch(gq + 1);
    if (blockIdx.y == 0 && tid < NCB) {
#pragma unroll
      for (int rr = 0; rr < kGrp; ++rr) { const double v = xs[buf][rr][tid]; nrm = fma(v, v, nrm); }
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = rbase + k * kThreads + tid;
      if (r < ell) {
        const U4 w = philox4x32_10(static_cast<uint32_t>(gq), static_cast<uint32_t>(r), 0u, 0u, key0, key1);
        const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int rr = 0; rr < kGrp; ++rr) {
          const double q = qd[(words[rr >> 3] >> (4 * (rr & 7))) & 15u];
#pragma unroll
          for (int j = 0; j < NCB; j += 2) {
            const double2 xv = *reinterpret_cast<const double2*>(&xs[buf][rr][j]);
            acc[k][j] = fma(q, xv.x, acc[k][j]);
            acc[k][j + 1] = fma(q, xv.y, acc[k][j + 1]);
          }
        }
      }
    }
    buf ^= 1;
  }
  // partials: part[cta][j][r]  (cta = blockIdx.x), npart[cta][j]
  const int64_t cta = blockIdx.x;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = rbase + k * kThreads + tid;
    if (r < ell) {
#pragma unroll
      for (int j = 0; j < NCB; ++j)
        if (j < ncols) part[(cta * NCB + j) * ell + r] = acc[k][j];
    }
  }
  if (blockIdx.y == 0 && tid < NCB && tid < ncols) npart[cta * NCB + tid] = nrm;
}

// Fixed-order reduction over CTAs: out = [s * sum part (ell x ncols); sum npart (ncols)].
__global__ void k1_reduce_kernel(const double* __restrict__ part, const double* __restrict__ npart, int nctas,
                                 int ncb, int ell, int ncols, double scale, double* __restrict__ out,
                                 unsigned* __restrict__ flags) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ny = static_cast<int64_t>(ell) * ncols;
  if (idx < ny) {
    const int j = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
    double s = 0.0;
    for (int c = 0; c < nctas; ++c) s += part[(static_cast<int64_t>(c) * ncb + j) * ell + r];
    out[idx] = scale * s;
  } else if (idx < ny + ncols) {
    const int j = static_cast<int>(idx - ny);
    double s = 0.0;
    for (int c = 0; c < nctas; ++c) s += npart[static_cast<int64_t>(c) * ncb + j];
    out[idx] = s;
    if (!isfinite(s)) atomicOr(flags, 1u);
  }
}

}  // namespace oid
