// NEXT-1: Algs 5-7 beside Alg 4 and the per-epoch NA-Hutch++ argmin (Alg 3 steps 28-32,
// P:390-396), enabled by oid_params.coeff_mode = 1.  The candidates are formed with
// small GEMMs in oid.cu; the kernels here are the pieces that are not GEMMs:
//   * cross_dots_kernel: <x_r, c_old_i> for every column x_r admitted this epoch and every basis
//     column c_old_i replaced or vacated this epoch, over this shard's rows, BEFORE the basis copy
//     (A7) overwrites the old columns - Alg 7's A_J^T A_Jprev needs them;
//   * cross_gram_kernel: X = A_J^T A_Jprev from the current exact Gram G, the previous one and the
//     cross dots (unchanged slots keep their Gram entries);
//   * psd_pinv_weights_kernel: 1/mu above the R9 cutoff for G^+ (P:468's G^-1);
//   * zero_changed_rows_kernel: eq:coeff_update_residual_zeroout;
//   * argmin_pick_kernel / copy_chosen_kernel: q* = first minimum of the unclamped estimates
//     (lowest algorithm number on ties) and P <- P_{q*}, decided on the device.
#pragma once
#include "common.cuh"

namespace oid {

// partial dots over a row chunk: part[chunk](j_a, i_e) = sum_rows X(:, r_a) C_old(:, i_e), with
// the admitted pairs (slot, r) in admit[0 .. 2 na) and the changed old slots in olds[0 .. ne)
template <typename T>
__global__ void __launch_bounds__(256) cross_dots_kernel(const T* __restrict__ X, int64_t ld, const T* __restrict__ Cb,
                                                         int64_t m_loc, int t, const int* __restrict__ admit,
                                                         const int* __restrict__ counts, const int* __restrict__ olds,
                                                         const int* __restrict__ ne_p, int64_t rows_per_chunk,
                                                         double* __restrict__ part) {
  constexpr int RL = 128 / sizeof(T);
  const int na = counts[0], ne = *ne_p;
  const int npair = na * ne;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = min(m_loc, r0 + rows_per_chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pr = blockIdx.x * 8 + warp; pr < npair; pr += gridDim.x * 8) {
    const int a = pr / ne, e = pr - a * ne;
    const int r = admit[2 * a + 1], slot = olds[e];
    const T* x = X + static_cast<int64_t>(r) * ld;
    double acc = 0.0;
    for (int64_t i = r0 + lane; i < r1; i += 32)
      acc = fma(static_cast<double>(x[i]), static_cast<double>(Cb[((i / RL) * t + slot) * RL + (i % RL)]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    // column-major (new slot j, old slot i): j + i t
    if (lane == 0) part[(static_cast<int64_t>(blockIdx.y) * t + slot) * t + admit[2 * a]] = acc;
  }
}

// Dx(j, i) = sum over chunks (fixed order) of part[chunk][j][i]
__global__ void cross_dots_sum_kernel(const double* __restrict__ part, int nchunk, int t, double* __restrict__ Dx) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * t) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += part[static_cast<int64_t>(c) * t * t + idx];
  Dx[idx] = s;
}

// Changed old slots of this epoch (J_prev[i] >= 0, J[i] != J_prev[i]) in slot order; *ne = count.
__global__ void changed_slots_kernel(const int64_t* __restrict__ J, const int64_t* __restrict__ Jprev, int t,
                                     int* __restrict__ olds, int* __restrict__ ne) {
  if (threadIdx.x != 0) return;
  int c = 0;
  for (int i = 0; i < t; ++i)
    if (Jprev[i] >= 0 && J[i] != Jprev[i]) olds[c++] = i;
  *ne = c;
}

// X = A_J^T A_Jprev (t x t, column i = previous slot i): 0 for a vacant previous slot; the current
// Gram column for an unchanged slot; for a changed old column c_old_i, row j = <c_j, c_old_i>:
// 0 if slot j is vacant now, Gprev(j, i) if slot j is unchanged, Dx(j, i) if j was filled this epoch.
__global__ void cross_gram_kernel(const double* __restrict__ G, const double* __restrict__ Gprev,
                                  const double* __restrict__ Dx, const int64_t* __restrict__ J,
                                  const int64_t* __restrict__ Jprev, int t, double* __restrict__ X) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * t) return;
  const int j = idx % t, i = idx / t;
  double v = 0.0;
  if (Jprev[i] >= 0 && J[j] >= 0) {
    if (J[i] == Jprev[i]) v = G[idx];
    else if (J[j] == Jprev[j]) v = Gprev[idx];
    else v = Dx[idx];
  }
  X[idx] = v;
}

// w_i = 1/mu_i for mu_i > 1e-12 max(mu) (reading R9), else 0
__global__ void psd_pinv_weights_kernel(const double* __restrict__ mu, int n, double* __restrict__ w) {
  __shared__ double mx;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, mu[i]);
    mx = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = (mx > 0.0 && mu[i] > 1e-12 * mx) ? 1.0 / mu[i] : 0.0;
}

// P(i, :) = 0 for slots whose basis column changed this epoch (J[i] != J_prev[i])
__global__ void zero_changed_rows_kernel(double* __restrict__ P, int t, int64_t n, const int64_t* __restrict__ J,
                                         const int64_t* __restrict__ Jprev) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= t * n) return;
  const int i = static_cast<int>(idx % t);
  if (J[i] != Jprev[i]) P[idx] = 0.0;
}

// e2[q] (q = 0..3 for Algs 4..7) -> q* (first minimum), logged with the four estimates:
// log row = [epoch, 4 + q*, e2_4, e2_5, e2_6, e2_7]; qsel[0] = q*
__global__ void argmin_pick_kernel(const double* __restrict__ e4, const double* __restrict__ cest, int cstride,
                                   double epoch, double* __restrict__ logrow, int* __restrict__ qsel) {
  if (threadIdx.x != 0) return;
  double e[4] = {e4[0], cest[0], cest[cstride], cest[2 * cstride]};
  int q = 0;
  for (int k = 1; k < 4; ++k)
    if (e[k] < e[q]) q = k;
  qsel[0] = q;
  if (logrow) {
    logrow[0] = epoch;
    logrow[1] = 4.0 + q;
    for (int k = 0; k < 4; ++k) logrow[2 + k] = e[k];
  }
}

// dst <- the chosen candidate (t x n, ld t): src0 = Alg 4's P, src1 + (q-1) t n_cap = Algs 5-7
__global__ void copy_chosen_kernel(const double* __restrict__ src0, const double* __restrict__ src1, int64_t cand_stride,
                                   const int* __restrict__ qsel, int64_t count, double* __restrict__ dst) {
  const int q = qsel[0];
  const double* src = q == 0 ? src0 : src1 + static_cast<int64_t>(q - 1) * cand_stride;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// out(:, j) = V(:, j) w_j (n x n)
__global__ void scale_cols_kernel(const double* __restrict__ V, int n, const double* __restrict__ w,
                                  double* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n * n) out[idx] = V[idx] * w[idx / n];
}

// e2 of one candidate from its scalar slots [T1, T3A, T3B, GPP] and ||A_obs||^2
__global__ void cand_e2_kernel(double* __restrict__ cs, int ell3, const double* __restrict__ frob2) {
  if (threadIdx.x != 0) return;
  const double T = ell3 > 0 ? cs[0] + (cs[1] - cs[2]) / ell3 : cs[0];
  cs[4] = *frob2 - 2.0 * T + cs[3];
}

// out[8] of the chosen candidate, in the layout of hutch_final_kernel's output
__global__ void chosen_estimate_kernel(const double* __restrict__ est4, const double* __restrict__ cest, int cstride,
                                       const int* __restrict__ qsel, int ell3, const double* __restrict__ frob2,
                                       double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  const int q = qsel[0];
  for (int k = 0; k < 8; ++k) out[k] = est4[k];
  if (q == 0) return;
  const double* cs = cest + (q - 1) * cstride;
  const double T = ell3 > 0 ? cs[0] + (cs[1] - cs[2]) / ell3 : cs[0];
  const double e2 = cs[4], f2 = *frob2;
  const double est = sqrt(fmax(e2, 0.0));
  unsigned f = static_cast<unsigned>(est4[6]) & ~4u;
  if (e2 < 0.0) f |= 4u;
  out[0] = e2; out[1] = T; out[2] = cs[3]; out[3] = f2; out[4] = est;
  out[5] = f2 > 0.0 ? est / sqrt(f2) : 0.0;
  out[6] = static_cast<double>(f);
}

}  // namespace oid
