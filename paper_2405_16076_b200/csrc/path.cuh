// Post-pass kernels specific to Algorithm 3: ridge regulariser, ridge scores, selection,
// basis copy, S_J gather, NA-Hutch++ final combination.
#pragma once
#include "common.cuh"

namespace oid {

// scalars layout (device double array)
enum Scal : int {
  SC_FROB2 = 0, SC_LAM = 1, SC_EK = 2, SC_SHIFT = 3, SC_TRACE = 4, SC_DMAX = 5, SC_MINMARGIN = 6, SC_KAPPA = 7,
  SC_T1 = 8, SC_T3A = 9, SC_T3B = 10, SC_GPP = 11, SC_COUNT = 16
};

// Ridge regulariser (reading R8): eigenvalues mu of the unscaled Gram, E_k = sum of the k
// largest (descending order), lambda per mode, shift = ell * lambda (reading R3),
// dmax = max(mu) + shift.  One CTA (n <= 1024): rank sort, then sequential sums.
__global__ void lambda_kernel(const double* __restrict__ mu, int n, int k, const double* __restrict__ gram,
                              double lam_param, int ell, double* __restrict__ scal, double* __restrict__ sorted) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = mu[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double u = mu[j];
      rank += (u > v) || (u == v && j < i);
    }
    sorted[rank] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double Ek = 0.0;
    for (int i = 0; i < k && i < n; ++i) Ek += sorted[i];
    double tr = 0.0;
    for (int i = 0; i < ell; ++i) tr += gram[static_cast<int64_t>(i) * ell + i];
    const double frob2 = scal[SC_FROB2];
    double lam;
    if (lam_param >= 0.0) lam = lam_param;
    else if (lam_param == -1.0) lam = fmax(0.0, (frob2 - Ek / ell) / k);
    else lam = fmax(0.0, (tr - Ek) / (static_cast<double>(ell) * k));
    const double shift = ell * lam;
    scal[SC_LAM] = lam;
    scal[SC_EK] = Ek;
    scal[SC_SHIFT] = shift;
    scal[SC_TRACE] = tr;
    scal[SC_DMAX] = (n > 0 ? sorted[0] : 0.0) + shift;
  }
}

// Yc = [S(:, J_i) for slots (zero if vacant) | Y_block]  (ell x (t + nc))
__global__ void gather_scored_kernel(const double* __restrict__ S, const int64_t* __restrict__ J, int t,
                                     const double* __restrict__ Yp, int nc, int ell, double* __restrict__ Yc) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(ell) * (t + nc);
  if (idx >= total) return;
  const int col = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
  double v = 0.0;
  if (col < t) {
    const int64_t j = J[col];
    if (j >= 0) v = S[j * ell + r];
  } else {
    v = Yp[static_cast<int64_t>(col - t) * ell + r];
  }
  Yc[idx] = v;
}

// tau_j = sum_{i: mu_i + shift > 1e-12 dmax} T(i, j)^2 / (mu_i + shift), T = W^T Yc
// (eq:sketch_ridge_leverage_score; readings R3, R9).  One CTA per column.
__global__ void scores_kernel(const double* __restrict__ T, const double* __restrict__ mu, int ell, int ncol,
                              const double* __restrict__ scal, double* __restrict__ tau, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[8];
  const int j = blockIdx.x;
  if (j >= ncol) return;
  const double shift = scal[SC_SHIFT], dmax = scal[SC_DMAX];
  double s = 0.0;
  if (dmax > 0.0) {
    for (int i = threadIdx.x; i < ell; i += blockDim.x) {
      const double d = mu[i] + shift;
      if (d > 1e-12 * dmax) { const double x = T[static_cast<int64_t>(j) * ell + i]; s += x * x / d; }
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) tau[j] = s;
}

// Alg 3 steps 15-27, readings R4-R7, R14.  Single thread (sequential by nature:
// slot i+1 sees the candidates consumed by slot i).
// tau: [t slot scores | nc candidate scores]; nrm: candidate norms (zero columns skipped).
// Outputs: admit list (slot, r) pairs, count; zero list (slots vacated, not refilled).
__global__ void select_kernel(int64_t* __restrict__ J, double* __restrict__ tau_old, const double* __restrict__ tau,
                              const double* __restrict__ nrm, int t, int nc, double factor, uint32_t epoch,
                              int64_t base, uint32_t key0, uint32_t key1, int* __restrict__ admit,
                              int* __restrict__ counts, double* __restrict__ scal, int* __restrict__ dirty) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned consumed[2] = {0u, 0u};   // nc <= 64
  int na = 0, nz = 0;
  double minm = scal[SC_MINMARGIN];
  for (int i = 0; i < t; ++i) {
    bool occupied = J[i] >= 0;
    bool evicted = false;
    if (occupied) {
      const double told = tau_old[i];
      const double ti = fmin(told, tau[i]);
      const double rho = told > 0.0 ? ti / told : 1.0;
      const double pev = 1.0 - rho;
      const double u = select_uniform(epoch, static_cast<uint32_t>(i), 0xFFFFFFFFu, key0, key1);
      minm = fmin(minm, fabs(u - pev) / fmax(rho, 0x1p-24));
      if (u < pev) { J[i] = -1; tau_old[i] = 1.0; occupied = false; evicted = true; }
      else tau_old[i] = ti;
    }
    if (!occupied) {
      bool filled = false;
      for (int r = 0; r < nc; ++r) {
        if ((consumed[r >> 5] >> (r & 31)) & 1u) continue;
        if (nrm[r] == 0.0) continue;
        const double praw = tau[t + r] * factor;
        const double p = fmin(1.0, praw);
        const double u = select_uniform(epoch, static_cast<uint32_t>(i), static_cast<uint32_t>(r), key0, key1);
        minm = fmin(minm, fabs(u - praw) / fmax(praw, 0x1p-24));
        if (u < p) {
          J[i] = base + r;
          tau_old[i] = tau[t + r];
          consumed[r >> 5] |= 1u << (r & 31);
          admit[2 * na] = i;
          admit[2 * na + 1] = r;
          dirty[i] = 1;
          ++na;
          filled = true;
          break;
        }
      }
      if (evicted && !filled) { admit[2 * (nc + t) - 2 - 2 * nz] = i; ++nz; }
    }
  }
  counts[0] = na;
  counts[1] = nz;
  scal[SC_MINMARGIN] = minm;
}

// C(:, slot) <- X(:, r) for admissions, C(:, slot) <- 0 for vacated slots.
template <typename T>
__global__ void basis_copy_kernel(const T* __restrict__ X, int64_t ld, T* __restrict__ C, int64_t m_loc,
                                  const int* __restrict__ admit, const int* __restrict__ counts, int nc, int t) {
  const int a = blockIdx.y;
  const int na = counts[0], nz = counts[1];
  int slot, r = -1;
  if (a < na) { slot = admit[2 * a]; r = admit[2 * a + 1]; }
  else if (a - na < nz) { slot = admit[2 * (nc + t) - 2 - 2 * (a - na)]; }
  else return;
  T* dst = C + static_cast<int64_t>(slot) * m_loc;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (r >= 0) {
    const T* src = X + static_cast<int64_t>(r) * ld;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m_loc; i += stride) dst[i] = src[i];
  } else {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m_loc; i += stride) dst[i] = T(0);
  }
}

// S_J = S(:, J) with zero columns for vacant slots (ell x t)
__global__ void gather_sj_kernel(const double* __restrict__ S, const int64_t* __restrict__ J, int t, int ell,
                                 double* __restrict__ SJ) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(ell) * t) return;
  const int col = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
  const int64_t j = J[col];
  SJ[idx] = j >= 0 ? S[j * ell + r] : 0.0;
}

// G(i, j) masked to occupied slots: G <- G .* [J_i >= 0][J_j >= 0]
__global__ void mask_gram_kernel(double* __restrict__ G, const int64_t* __restrict__ J, int t) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * t) return;
  const int i = idx % t, j = idx / t;
  if (J[i] < 0 || J[j] < 0) G[idx] = 0.0;
}

// Final combination of Alg 8: T = term1 + (t3a - t3b)/ell3;
// e2 = frob2 - 2T + tr(G P P^T).  out[8] as documented in oid.h.
__global__ void hutch_final_kernel(const double* __restrict__ scal, int ell3, const unsigned* __restrict__ flags,
                                   double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  const double term1 = scal[SC_T1];
  const double T = ell3 > 0 ? term1 + (scal[SC_T3A] - scal[SC_T3B]) / ell3 : term1;
  const double gpp = scal[SC_GPP];
  const double frob2 = scal[SC_FROB2];
  const double e2 = frob2 - 2.0 * T + gpp;
  unsigned f = *flags;
  if (e2 < 0.0) f |= 4u;
  const double est = sqrt(fmax(e2, 0.0));
  out[0] = e2; out[1] = T; out[2] = gpp; out[3] = frob2; out[4] = est;
  out[5] = frob2 > 0.0 ? est / sqrt(frob2) : 0.0;
  out[6] = static_cast<double>(f);
  out[7] = scal[SC_KAPPA];
}

// Slots admitted since the last estimate (dirty flags set by select_kernel), compacted in
// slot order; flags cleared.  counts[2] = number of dirty slots.
__global__ void dirty_compact_kernel(int* __restrict__ dirty, int t, int* __restrict__ list, int* __restrict__ counts) {
  if (threadIdx.x != 0) return;
  int c = 0;
  for (int i = 0; i < t; ++i)
    if (dirty[i]) { list[c++] = i; dirty[i] = 0; }
  counts[2] = c;
}

// Incremental exact basis Gram (A9): Dpart[chunk](q, j) = sum_{rows in chunk} C(r, d_q) C(r, j)
// for the dirty slots d_q.  Each CTA streams its row chunk of the basis once per
// group of 32 dirty slots, 32 rows at a time through a 2-stage cp.async ring (column-major tile,
// pitch BG_PITCH elements: conflict-free column-strided reads).  Thread (tq, tj) = (tid % 8,
// tid / 8) owns the 4 x JB register tile q = tq + 8a, j = tj + 32b (fp64 FMA, fixed order).
constexpr int kBgRows = 32;
template <typename T> struct BgPitch { static constexpr int v = sizeof(T) == 8 ? 34 : 36; };

template <typename T>
__host__ __device__ constexpr size_t bg_stage_elems(int t) { return static_cast<size_t>(t) * BgPitch<T>::v; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// fp64 tensor-core MMA (DMMA): D (8x8) += A (8x4, row) * B (4x8, col).  Fragments: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], c = C[lane/4][2 (lane%4) + {0, 1}].
__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Warp w owns the output columns j in [32 (w + 8 i), +32) for i < JBW (t <= 256 JBW); the 32 dirty
// slots q of the group are the M dimension (4 m8 blocks), the basis rows the K dimension.
template <typename T, int JBW>
__global__ void __launch_bounds__(256) basis_gram_dirty_kernel(const T* __restrict__ C, int64_t m_loc, int t,
                                                               int64_t rows_per_chunk, int nstage,
                                                               const int* __restrict__ list,
                                                               const int* __restrict__ counts,
                                                               double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char bg_smem[];
  constexpr int P = BgPitch<T>::v;
  constexpr int EPC = 16 / sizeof(T);                  // elements per 16-byte copy
  T* tiles = reinterpret_cast<T*>(bg_smem);            // [nstage][t][P]
  __shared__ double dt[kBgRows][33];                   // dirty columns of the current tile
  __shared__ int dl[32];
  const int nd = counts[2];
  if (nd == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g4 = lane >> 2, i4 = lane & 3;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_chunk;
  const int64_t r1 = min(m_loc, r0 + rows_per_chunk);
  const int ntile = static_cast<int>((r1 - r0 + kBgRows - 1) / kBgRows);
  const size_t stage = bg_stage_elems<T>(t);
  const bool vec = ((m_loc * sizeof(T)) % 16 == 0) && (r0 % EPC == 0);
  double* out = part + static_cast<int64_t>(blockIdx.x) * t * t;

  auto load = [&](int it, int buf) {
    T* dst = tiles + buf * stage;
    const int64_t rb = r0 + static_cast<int64_t>(it) * kBgRows;
    constexpr int CH = kBgRows / EPC;                  // 16-byte chunks per column
    for (int e = tid; e < t * CH; e += 256) {
      const int col = e / CH, c = e - col * CH;
      const int64_t r = rb + c * EPC;
      T* d = dst + col * P + c * EPC;
      const T* src = C + static_cast<int64_t>(col) * m_loc + r;
      if (vec && r + EPC <= r1) {
        cp_async16(d, src);
      } else {
#pragma unroll
        for (int k = 0; k < EPC; ++k) d[k] = (r + k < r1) ? src[k] : T(0);
      }
    }
  };

  for (int q0 = 0; q0 < nd; q0 += 32) {
    if (tid < 32) dl[tid] = (q0 + tid < nd) ? list[q0 + tid] : -1;
    double acc[JBW][4][4][2];
#pragma unroll
    for (int b = 0; b < JBW; ++b)
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
#pragma unroll
        for (int n = 0; n < 4; ++n) { acc[b][mm][n][0] = 0.0; acc[b][mm][n][1] = 0.0; }
    __syncthreads();
    load(0, 0);
    cp_async_commit();
    for (int it = 0; it < ntile; ++it) {
      const int buf = nstage == 2 ? (it & 1) : 0;
      if (nstage == 2 && it + 1 < ntile) load(it + 1, buf ^ 1);
      cp_async_commit();
      if (nstage == 2) cp_async_wait<1>(); else cp_async_wait<0>();
      __syncthreads();
      const T* tile = tiles + buf * stage;
      for (int e = tid; e < 32 * kBgRows; e += 256) {        // gather the dirty columns
        const int q = e >> 5, rr = e & 31;
        const int d = dl[q];
        dt[rr][q] = d >= 0 ? static_cast<double>(tile[d * P + rr]) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int ks = 0; ks < kBgRows; ks += 4) {
        double a[4];
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) a[mm] = dt[ks + i4][8 * mm + g4];
#pragma unroll
        for (int b = 0; b < JBW; ++b) {
          const int jb = 32 * (warp + 8 * b);
          if (jb >= t) continue;                             // warp-uniform
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const int j = jb + 8 * n + g4;
            const double bv = j < t ? static_cast<double>(tile[j * P + ks + i4]) : 0.0;
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) dmma_m8n8k4(acc[b][mm][n], a[mm], bv);
          }
        }
      }
      __syncthreads();
      if (nstage == 1 && it + 1 < ntile) load(it + 1, 0);
    }
#pragma unroll
    for (int b = 0; b < JBW; ++b) {
      const int jb = 32 * (warp + 8 * b);
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const int q = 8 * mm + g4;
        if (q0 + q >= nd) continue;
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = jb + 8 * n + 2 * i4 + h;
            if (j < t) out[(q0 + q) + static_cast<int64_t>(j) * t] = acc[b][mm][n][h];
          }
      }
    }
  }
}

// G(d_q, j) = G(j, d_q) = D(q, j) for the dirty slots (after the cross-shard reduction).
__global__ void gram_scatter_kernel(const double* __restrict__ D, const int* __restrict__ list,
                                    const int* __restrict__ counts, int t, double* __restrict__ G) {
  const int nd = counts[2];
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(nd) * t) return;
  const int q = static_cast<int>(idx % nd), j = static_cast<int>(idx / nd);
  const int d = list[q];
  const double v = D[q + static_cast<int64_t>(j) * t];
  G[d + static_cast<int64_t>(j) * t] = v;
  G[j + static_cast<int64_t>(d) * t] = v;
}

__global__ void sum_chunks_kernel(const double* __restrict__ part, int nchunks, int64_t n, double* __restrict__ out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[static_cast<int64_t>(c) * n + idx];
  out[idx] = s;
}

// gate[0] = a, gate[1] = b
__global__ void set_flag_kernel(int* __restrict__ gate, int a, int b) {
  gate[0] = a;
  gate[1] = b;
}

}  // namespace oid
