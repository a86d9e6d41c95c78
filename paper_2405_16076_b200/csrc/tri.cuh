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
constexpr int kTriMaxG = 2048;   // largest Gram order on the tridiagonal A4/A5 path (panels + cluster)
constexpr int kTriRows = kTriMaxN / kTriCtas;   // 32 rows per CTA at the maximum size

// Householder tridiagonalisation of the symmetric n x n matrix A (col-major), n <= 512.
// Outputs: d (n), e (n-1) of T; reflectors H_k = I - tau_k v_k v_k^T, k = 0..n-3, with v_k
// stored in Vh(:, k) (rows k+1..n-1; zero elsewhere) and tau_k in tauv[k].
// Launch: 16 CTAs in one cluster.  CTA c owns rows [c R, c R + R) (R = tri_rows(n) <= 32, even);
// warp w of the CTA owns 4 of them and lane l the columns l + 32 q (q < 16), held in REGISTERS
// (64 doubles per thread), so the matrix-vector product and the rank-2 update never touch
// shared memory.
// Step k: every CTA pushes its slice of column k (= row k by symmetry) and its partial ||x||^2
// into every CTA's shared memory with st.async (distributed shared memory), which completes
// bytes on the receiver's mbarrier; each CTA waits on its own mbarrier only (no cluster-wide
// barrier), forms the reflector redundantly, computes p = tau A v on its rows and pushes its p
// slice and partial v^T p the same way; then it applies A <- A - v w^T - w v^T,
// w = p - (tau v^T p / 2) v.  Buffers and mbarriers alternate between even and odd steps: a
// CTA can only send step k+2's data after every CTA has sent its step-k+1 p, i.e. after every
// receiver has finished step k, so a buffer is never overwritten while it is read.
constexpr int kTriRW = 4;     // rows per warp
constexpr int kTriCL = 16;    // column registers per lane

__host__ __device__ constexpr int tri_rows(int n) { return 2 * ((n + 2 * kTriCtas - 1) / (2 * kTriCtas)); }
// leading dimension of the reflector matrix Vh (even, so every column start is 16-byte aligned)
__host__ __device__ constexpr int tri_ldv(int n) { return (n + 1) & ~1; }

// 1/x for normal x: hardware approximation refined by two Newton steps (about 1 ulp); keeps the
// divide off the sequential LDL^T pivot chains
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double q = fma(-x, r, 1.0);
  r = fma(r, q, r);
  q = fma(-x, r, 1.0);
  return fma(r, q, r);
}

// column block q of all kTriRW rows, q warp-uniform: one indexed branch instead of a select chain
__device__ __forceinline__ void tri_pick_rows(const double (&a)[kTriRW][kTriCL], int q, double (&x)[kTriRW]) {
  switch (q) {
#define TRI_CASE(Q) \
  case Q: { _Pragma("unroll") for (int r = 0; r < kTriRW; ++r) x[r] = a[r][Q]; } break;
    TRI_CASE(0) TRI_CASE(1) TRI_CASE(2) TRI_CASE(3) TRI_CASE(4) TRI_CASE(5) TRI_CASE(6) TRI_CASE(7)
    TRI_CASE(8) TRI_CASE(9) TRI_CASE(10) TRI_CASE(11) TRI_CASE(12) TRI_CASE(13) TRI_CASE(14)
    default: { _Pragma("unroll") for (int r = 0; r < kTriRW; ++r) x[r] = a[r][15]; } break;
#undef TRI_CASE
  }
}
__device__ __forceinline__ double tri_pick(const double (&a)[kTriCL], int q) {
  double x = 0.0;
#pragma unroll
  for (int c = 0; c < kTriCL; ++c) x = (c == q) ? a[c] : x;
  return x;
}

__device__ __forceinline__ uint32_t tri_saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t tri_mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void tri_st_async2(uint32_t raddr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr), "d"(x),
               "d"(y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void tri_st_async1(uint32_t raddr, double x, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(x), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void tri_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tri_saddr(bar)), "r"(count));
}
__device__ __forceinline__ void tri_mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tri_saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tri_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TRI_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TRI_WAIT_%=;\n\t}" ::"r"(tri_saddr(bar)),
      "r"(parity)
      : "memory");
}

// Compact-WY form of the reflectors in chunks of kRefChunk: for chunk b (k = 8b .. 8b+7, k < n-2)
// H_{8b} H_{8b+1} ... H_{8b+7} = I - V_b T_b V_b^T with T_b upper triangular (LAPACK larft,
// forward columnwise: T(i,i) = tau_i, T(0:i, i) = -tau_i T(0:i, 0:i) V(:, 0:i)^T v_i).  One CTA per
// chunk; T_b row-major in wyT[64 b ..].  Reflectors with tau = 0 give zero rows/columns.
constexpr int kRefChunk = 8;
constexpr int kMaxRefChunks = (kTriMaxN + kRefChunk - 1) / kRefChunk;
constexpr int kMaxRefChunksG = (kTriMaxG + kRefChunk - 1) / kRefChunk;
constexpr int kQStages = 3;
// T factor of reflector chunk b (256 threads; G: 8 x 8 shared scratch); tau from tau_src.
__device__ __forceinline__ void wy_t_chunk(int b, const double* __restrict__ Vh, const double* tau_src, int n,
                                           double* __restrict__ wyT, double (*G)[kRefChunk]) {
  const int k0 = b * kRefChunk, nk = n - 2, ldv = tri_ldv(n);
  const int nr = min(kRefChunk, nk - k0);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // V^T V, pairs r < c (28), one warp per pair, fixed-order shuffle reduction
  for (int pr = w; pr < kRefChunk * (kRefChunk - 1) / 2; pr += 8) {
    int r = 0, rem = pr;
    while (rem >= kRefChunk - 1 - r) { rem -= kRefChunk - 1 - r; ++r; }
    const int c = r + 1 + rem;
    double acc = 0.0;
    if (c < nr) {
      const double* vr = Vh + static_cast<int64_t>(k0 + r) * ldv;
      const double* vc = Vh + static_cast<int64_t>(k0 + c) * ldv;
      for (int i = k0 + 1 + lane; i < n; i += 32) acc = fma(__ldcg(vr + i), __ldcg(vc + i), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) G[r][c] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double T[kRefChunk][kRefChunk];
#pragma unroll
    for (int r = 0; r < kRefChunk; ++r)
#pragma unroll
      for (int c = 0; c < kRefChunk; ++c) T[r][c] = 0.0;
#pragma unroll
    for (int c = 0; c < kRefChunk; ++c) {
      if (c < nr) {
        const double tc = tau_src[k0 + c];
        T[c][c] = tc;
#pragma unroll
        for (int r = 0; r < c; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int q = r; q < c; ++q) acc = fma(T[r][q], G[q][c], acc);
          T[r][c] = -tc * acc;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kRefChunk; ++r)
#pragma unroll
      for (int c = 0; c < kRefChunk; ++c) wyT[b * kRefChunk * kRefChunk + r * kRefChunk + c] = T[r][c];
  }
  __syncthreads();   // G reused by the next chunk
}

__global__ void __cluster_dims__(kTriCtas, 1, 1) __launch_bounds__(256, 1)
tridiag_cluster_kernel(const double* __restrict__ A, int lda, int n, double* __restrict__ d, double* __restrict__ e,
                       double* __restrict__ Vh, int ldv_out, double* __restrict__ tauv, long long* __restrict__ dbg,
                       double* __restrict__ wyT) {
  cg2::cluster_group cluster = cg2::this_cluster();
  const int c = static_cast<int>(cluster.block_rank());
  const int R = tri_rows(n);
  const int r0 = c * R, r1 = min(n, r0 + R);
  __shared__ __align__(16) double xb[2][kTriCtas * kTriRows];   // column k, all CTAs' slices
  __shared__ __align__(16) double pb[2][kTriCtas * kTriRows];   // p, all CTAs' slices
  __shared__ __align__(16) double locx[kTriRows], locp[kTriRows];
  __shared__ double ssb[2][kTriCtas];
  __shared__ double kb[2][kTriCtas];
  __shared__ double wred[8];
  __shared__ __align__(8) uint64_t barx[2], barp[2];
  __shared__ double tau_s[kTriMaxN], d_s[kTriMaxN], e_s[kTriMaxN];
  extern __shared__ double vh_s[];       // [n][R]: this CTA's rows of every reflector (dynamic)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t phase_bytes = static_cast<uint32_t>(kTriCtas) * (R + 1) * 8u;
  if (tid == 0) {
    tri_mbar_init(&barx[0], 1); tri_mbar_init(&barx[1], 1);
    tri_mbar_init(&barp[0], 1); tri_mbar_init(&barp[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double a[kTriRW][kTriCL];
  int gi[kTriRW];
#pragma unroll
  for (int r = 0; r < kTriRW; ++r) {
    const int i = r0 + warp * kTriRW + r;
    gi[r] = (warp * kTriRW + r < R && i < r1) ? i : -1;
#pragma unroll
    for (int q = 0; q < kTriCL; ++q) {
      const int j = lane + 32 * q;
      a[r][q] = (gi[r] >= 0 && j < n) ? A[j + static_cast<int64_t>(gi[r]) * lda] : 0.0;   // row i = column i
    }
  }
  // sender roles: thread -> (target CTA, pair of rows)
  const int hp = R >> 1;                          // v2 stores per slice
  const int tq = hp > 0 ? tid / hp : 0, tu = hp > 0 ? tid - tq * hp : 0;
  const bool sender = hp > 0 && tq < kTriCtas;
  // entries past the senders' slices (rows >= kTriCtas R) are never pushed: keep them zero, so the
  // unmasked products below see v_j = p_j = 0 there
  for (int i = kTriCtas * R + tid; i < kTriCtas * kTriRows; i += blockDim.x) {
    xb[0][i] = 0.0; xb[1][i] = 0.0; pb[0][i] = 0.0; pb[1][i] = 0.0;
  }
  cluster.sync();                                 // mbarrier inits visible cluster-wide
  const bool rec = dbg != nullptr && c == 0 && tid == 0;   // diagnostics: phase timestamps of CTA 0
  for (int k = 0; k < n - 2; ++k) {
    const int buf = k & 1;
    const uint32_t par = (k >> 1) & 1;
    double* xk = xb[buf];
    const int qk = k >> 5, lk = k & 31;
    if (rec && k < 1024) dbg[4 * k] = clock64();
    if (tid == 0) { tri_mbar_expect(&barx[buf], phase_bytes); tri_mbar_expect(&barp[buf], phase_bytes); }
    // phase 1: x_i = A(i, k) for my rows i > k -> every CTA, with the partial sum of squares
    double ssw = 0.0;
    double colk[kTriRW];
    tri_pick_rows(a, qk, colk);
#pragma unroll
    for (int r = 0; r < kTriRW; ++r) {
      const double xi = __shfl_sync(0xffffffffu, colk[r], lk);
      if (gi[r] > k) { ssw = fma(xi, xi, ssw); if (lane == 0) locx[gi[r] - r0] = xi; }
      else if (lane == 0 && warp * kTriRW + r < R) locx[warp * kTriRW + r] = 0.0;
      if (gi[r] == k && lane == 0) d_s[k] = xi;   // the diagonal entry A(k, k)
    }
    if (lane == 0) wred[warp] = ssw;
    __syncthreads();
    if (sender) {
      const uint32_t la = tri_saddr(&xk[r0 + 2 * tu]);
      tri_st_async2(tri_mapa(la, tq), locx[2 * tu], locx[2 * tu + 1], tri_mapa(tri_saddr(&barx[buf]), tq));
    }
    if (tid < kTriCtas) {
      double ss = 0.0;
      for (int w = 0; w < 8; ++w) ss += wred[w];
      tri_st_async1(tri_mapa(tri_saddr(&ssb[buf][c]), tid), ss, tri_mapa(tri_saddr(&barx[buf]), tid));
    }
    if (rec && k < 1024) dbg[4 * k + 1] = clock64();
    tri_mbar_wait(&barx[buf], par);
    if (rec && k < 1024) dbg[4 * k + 2] = clock64();
    // phase 2: reflector (redundant in every CTA)
    double ss = 0.0;
    for (int q = 0; q < kTriCtas; ++q) ss += ssb[buf][q];
    const double x0 = xk[k + 1];
    const double tail = ss - x0 * x0;
    double alpha, tau = 0.0, v0 = 0.0;
    if (tail > 0.0) {
      alpha = -copysign(sqrt(ss), x0);
      v0 = x0 - alpha;
      tau = 2.0 * rcp_nr(tail + v0 * v0);
    } else {
      alpha = x0;
    }
    if (tid == 0) { tau_s[k] = tau; e_s[k] = alpha; }
    // v_i for my rows; p_i = tau sum_j A_ij v_j
    double vi[kTriRW], pi[kTriRW];
#pragma unroll
    for (int r = 0; r < kTriRW; ++r) {
      vi[r] = (gi[r] > k) ? (gi[r] == k + 1 ? v0 : xk[gi[r]]) : 0.0;
      pi[r] = 0.0;
    }
    // The received slices are zero at rows <= k and past n (the senders zero them), so
    // v_j = x_j except v_{k+1} = v0, and w_j = p_j - h v_j needs no masks either: the stale
    // entries of A in finished rows / columns only ever meet zeros.
    if (tau != 0.0) {
      double p2[kTriRW];   // second accumulator per row (odd column blocks): half the FMA chain
#pragma unroll
      for (int r = 0; r < kTriRW; ++r) p2[r] = 0.0;
#pragma unroll
      for (int q = 0; q < kTriCL; ++q) {
        const int j = lane + 32 * q;
        const double vj = j == k + 1 ? v0 : xk[j];
#pragma unroll
        for (int r = 0; r < kTriRW; ++r) {
          if (q & 1) p2[r] = fma(a[r][q], vj, p2[r]);
          else pi[r] = fma(a[r][q], vj, pi[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < kTriRW; ++r) pi[r] += p2[r];
    }
    // warp sums of the 4 rows by a butterfly reduce-scatter (row 2 b4 + b3 ends in the lanes with
    // lane bits b4, b3), then broadcast: 10 shuffles instead of 20
    static_assert(kTriRW == 4, "butterfly below is written for 4 rows per warp");
    {
      const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
      const double s0 = h16 ? pi[0] : pi[2], s1 = h16 ? pi[1] : pi[3];
      const double k0 = h16 ? pi[2] : pi[0], k1 = h16 ? pi[3] : pi[1];
      const double q0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
      const double q1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
      double t = (h8 ? q1 : q0) + __shfl_xor_sync(0xffffffffu, h8 ? q0 : q1, 8);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
#pragma unroll
      for (int r = 0; r < kTriRW; ++r) pi[r] = __shfl_sync(0xffffffffu, t, (r >> 1) * 16 + (r & 1) * 8);
    }
    double kw = 0.0;
#pragma unroll
    for (int r = 0; r < kTriRW; ++r) {
      pi[r] *= tau;
      if (gi[r] > k) kw = fma(vi[r], pi[r], kw);
      if (lane == 0 && warp * kTriRW + r < R) {
        locp[warp * kTriRW + r] = gi[r] > k ? pi[r] : 0.0;
        if (gi[r] >= 0) vh_s[k * R + (gi[r] - r0)] = (gi[r] > k && tau != 0.0) ? vi[r] : 0.0;
      }
    }
    if (lane == 0) wred[warp] = kw;
    __syncthreads();
    if (sender) {
      const uint32_t la = tri_saddr(&pb[buf][r0 + 2 * tu]);
      tri_st_async2(tri_mapa(la, tq), locp[2 * tu], locp[2 * tu + 1], tri_mapa(tri_saddr(&barp[buf]), tq));
    }
    if (tid < kTriCtas) {
      double kp = 0.0;
      for (int w = 0; w < 8; ++w) kp += wred[w];
      tri_st_async1(tri_mapa(tri_saddr(&kb[buf][c]), tid), kp, tri_mapa(tri_saddr(&barp[buf]), tid));
    }
    tri_mbar_wait(&barp[buf], par);
    if (rec && k < 1024) dbg[4 * k + 3] = clock64();
    // phase 3: w = p - (tau K / 2) v; A <- A - v w^T - w v^T (zeros outside i, j > k)
    if (tau != 0.0) {
      double K = 0.0;
      for (int q = 0; q < kTriCtas; ++q) K += kb[buf][q];
      const double h = 0.5 * tau * K;
      const double* pk = pb[buf];
      double wi[kTriRW];
#pragma unroll
      for (int r = 0; r < kTriRW; ++r) wi[r] = (gi[r] > k) ? pi[r] - h * vi[r] : 0.0;
#pragma unroll
      for (int q = 0; q < kTriCL; ++q) {
        const int j = lane + 32 * q;
        const double vj = j == k + 1 ? v0 : xk[j];
        const double wj = pk[j] - h * vj;
#pragma unroll
        for (int r = 0; r < kTriRW; ++r) a[r][q] = a[r][q] - vi[r] * wj - wi[r] * vj;
      }
    }
  }
  // trailing 2 x 2 block
#pragma unroll
  for (int r = 0; r < kTriRW; ++r) {
    if (n >= 2 && gi[r] == n - 2) {
      const double dd = __shfl_sync(0xffffffffu, tri_pick(a[r], (n - 2) >> 5), (n - 2) & 31);
      const double ee = __shfl_sync(0xffffffffu, tri_pick(a[r], (n - 1) >> 5), (n - 1) & 31);
      if (lane == 0) { d_s[n - 2] = dd; e_s[n - 2] = ee; }
    }
    if (gi[r] == n - 1) {
      const double dd = __shfl_sync(0xffffffffu, tri_pick(a[r], (n - 1) >> 5), (n - 1) & 31);
      if (lane == 0) d_s[n - 1] = dd;
    }
  }
  __syncthreads();
  // bulk writes: reflector rows of this CTA (Vh(i, k) for i in [r0, r1), k < n - 2; leading
  // dimension tri_ldv(n), the pad row of odd n written as zero by the last CTA), tau/d/e
  // (ldv_out > tri_ldv(n): the trailing block of a larger reduction, whose Vh the caller zeroed)
  const int ldv = ldv_out;
  for (int idx = tid; idx < (r1 - r0) * (n - 2); idx += 256) {
    const int k = idx / (r1 - r0), il = idx - k * (r1 - r0);
    Vh[(r0 + il) + static_cast<int64_t>(k) * ldv] = vh_s[k * R + il];
  }
  if (ldv == tri_ldv(n) && ldv > n && r0 <= n - 1 && n - 1 < r0 + R)
    for (int k = tid; k < n - 2; k += 256) Vh[n + static_cast<int64_t>(k) * ldv] = 0.0;
  for (int k = tid; k < n; k += 256) {
    if (c == 0 && k < n - 2) tauv[k] = tau_s[k];
    if (k >= r0 && k < r1) { d[k] = d_s[k]; if (k < n - 1) e[k] = e_s[k]; }
  }
  cluster.sync();   // also: every CTA's Vh rows are visible to the whole cluster (global memory)
  // compact-WY T factors of the reflector chunks, chunk b on CTA b mod 16 (wy_t_kernel fused)
  if (wyT != nullptr && n > 2) {
    __shared__ double G[kRefChunk][kRefChunk];
    const int nch = (n - 2 + kRefChunk - 1) / kRefChunk;
    for (int b = c; b < nch; b += kTriCtas) wy_t_chunk(b, Vh, tau_s, n, wyT, G);
  }
}


// ---------------------------------------------------------------------------------------------
// Gram orders 512 < n <= kTriMaxG (l = 1024 on C5): the first n - 512 columns are reduced in
// panels of kPanNb by tridiag_panel_kernel, the LAPACK sytrd/latrd blocking restated for one
// 16-CTA cluster: within a panel the trailing matrix is not touched; column k and the product
// p = tau A v are corrected for the panel's earlier reflectors through their (v, w) pairs,
//   A_cur = A - V W^T - W V^T,
// and after the panel two GEMMs apply A <- A - V W^T - W V^T to the trailing block.  The
// remaining 512 x 512 block goes to tridiag_cluster_kernel.  The reflectors are those of the
// unblocked reduction (same H_k = I - tau_k v_k v_k^T, same d, e), only summed in another order.
// A lives in global memory (L2-resident: 8 MB at n = 1024); CTA c owns rows [c R, c R + R).
// Per column, three distributed-shared-memory exchanges (st.async onto the receivers'
// mbarriers, buffers alternating by step parity as in the cluster kernel):
//   A: the corrected column k below the diagonal (= x, slices of every CTA) and its partial norms
//   B: partial V^T v, W^T v over each CTA's rows
//   C: partial v^T p, and from the owner of row k + 1 that row of V and W (and p_{k+1}), which
//      the next column's correction needs.
constexpr int kPanNb = 32;
constexpr int kPanMaxR = kTriMaxG / kTriCtas;   // 128
__host__ __device__ constexpr int pan_rows(int n) { return 2 * ((n + 2 * kTriCtas - 1) / (2 * kTriCtas)); }
// dynamic shared memory: V, W rows of this CTA (2 kPanMaxR (kPanNb + 1)) + the column buffers
// xb[2][kTriCtas kPanMaxR]
constexpr int kPanSmem = (2 * kPanMaxR * (kPanNb + 1) + 2 * kTriCtas * kPanMaxR) * static_cast<int>(sizeof(double));

__global__ void __cluster_dims__(kTriCtas, 1, 1) __launch_bounds__(256, 1)
tridiag_panel_kernel(const double* __restrict__ A, int n, int k0, int nb, double* __restrict__ d,
                     double* __restrict__ e, double* __restrict__ Vh, int ldv, double* __restrict__ tauv,
                     double* __restrict__ W) {
  cg2::cluster_group cluster = cg2::this_cluster();
  const int c = static_cast<int>(cluster.block_rank());
  const int R = pan_rows(n);
  const int r0 = c * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // V, W rows of this CTA and the two column buffers (dynamic, kPanSmem bytes)
  extern __shared__ __align__(16) double pan_smem[];
  double (*Vs)[kPanNb + 1] = reinterpret_cast<double (*)[kPanNb + 1]>(pan_smem);
  double (*Ws)[kPanNb + 1] = reinterpret_cast<double (*)[kPanNb + 1]>(pan_smem + kPanMaxR * (kPanNb + 1));
  double (*xb)[kTriCtas * kPanMaxR] =
      reinterpret_cast<double (*)[kTriCtas * kPanMaxR]>(pan_smem + 2 * kPanMaxR * (kPanNb + 1));
  __shared__ double ssb[2][kTriCtas];
  __shared__ double vtb[2][kTriCtas][2 * kPanNb];
  __shared__ double kb[2][kTriCtas];
  __shared__ double rowb[2][1 + 2 * kPanNb];
  __shared__ double rowV[kPanNb], rowW[kPanNb];
  __shared__ __align__(16) double locx[kPanMaxR];
  __shared__ double locs[kPanMaxR], locp[kPanMaxR];
  __shared__ double vtot[2 * kPanNb];
  __shared__ double wred[8];
  __shared__ double tau_s[kPanNb], e_s[kPanNb];
  __shared__ __align__(8) uint64_t barA[2], barB[2], barC[2];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) { tri_mbar_init(&barA[b], 1); tri_mbar_init(&barB[b], 1); tri_mbar_init(&barC[b], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kTriCtas * kPanMaxR; i += blockDim.x) { xb[0][i] = 0.0; xb[1][i] = 0.0; }
  cluster.sync();
  const uint32_t bytesA = static_cast<uint32_t>(kTriCtas) * (R + 1) * 8u;
  const uint32_t bytesB = static_cast<uint32_t>(kTriCtas) * 2 * kPanNb * 8u;
  const uint32_t bytesC = static_cast<uint32_t>(kTriCtas) * 8u + (1 + 2 * kPanNb) * 8u;
  const int hp = R >> 1;                          // v2 stores per slice
  for (int j = 0; j < nb; ++j) {
    const int k = k0 + j;
    const int buf = j & 1;
    const uint32_t par = (j >> 1) & 1;
    if (tid == 0) {
      tri_mbar_expect(&barA[buf], bytesA);
      tri_mbar_expect(&barB[buf], bytesB);
      tri_mbar_expect(&barC[buf], bytesC);
    }
    // ---- phase A: column k of A_cur on my rows (x_i for i > k, d_k on its owner)
    double ssw = 0.0;
    if (tid < R) {
      const int i = r0 + tid;
      double a = 0.0;
      if (i < n && i >= k) {
        a = A[i + static_cast<int64_t>(k) * n];
        for (int q = 0; q < j; ++q) a -= Vs[tid][q] * rowW[q] + Ws[tid][q] * rowV[q];
      }
      if (i == k) d[k] = a;
      const double xi = (i < n && i > k) ? a : 0.0;
      locx[tid] = xi;
      ssw = xi * xi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssw += __shfl_xor_sync(0xffffffffu, ssw, o);
    if (lane == 0) wred[warp] = ssw;
    __syncthreads();
    for (int idx = tid; idx < kTriCtas * hp; idx += blockDim.x) {
      const int tq = idx / hp, tu = idx - tq * hp;   // (target CTA, pair of rows)
      const uint32_t la = tri_saddr(&xb[buf][r0 + 2 * tu]);
      tri_st_async2(tri_mapa(la, tq), locx[2 * tu], locx[2 * tu + 1], tri_mapa(tri_saddr(&barA[buf]), tq));
    }
    if (tid < kTriCtas) {
      double ss = 0.0;
      for (int w = 0; w < 8; ++w) ss += wred[w];
      tri_st_async1(tri_mapa(tri_saddr(&ssb[buf][c]), tid), ss, tri_mapa(tri_saddr(&barA[buf]), tid));
    }
    tri_mbar_wait(&barA[buf], par);
    // ---- reflector (redundant in every CTA), as in the unblocked reduction
    double ss = 0.0;
    for (int q = 0; q < kTriCtas; ++q) ss += ssb[buf][q];
    const double* xk = xb[buf];
    const double x0 = xk[k + 1];
    const double tail = ss - x0 * x0;
    double alpha, tau = 0.0, v0 = 0.0;
    if (tail > 0.0) {
      alpha = -copysign(sqrt(ss), x0);
      v0 = x0 - alpha;
      tau = 2.0 * rcp_nr(tail + v0 * v0);
    } else {
      alpha = x0;
    }
    if (tid == 0) { tau_s[j] = tau; e_s[j] = alpha; }
    // ---- phase B: s = A v on my rows (column i of the symmetric A = row i), V^T v, W^T v partials
    // warp w: rows w, w + 8, ... of this CTA (8 at R = 64), lanes over the columns j' > k
    {
      constexpr int RW = kPanMaxR / 8;
      double acc[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) acc[r] = 0.0;
      if (tau != 0.0) {
        for (int jj = k + 1 + lane; jj < n; jj += 32) {
          const double vj = jj == k + 1 ? v0 : xk[jj];
#pragma unroll
          for (int r = 0; r < RW; ++r) {
            const int il = warp + 8 * r, i = r0 + il;
            if (il < R && i < n && i > k) acc[r] = fma(__ldcg(A + jj + static_cast<int64_t>(i) * n), vj, acc[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        double t = acc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0 && warp + 8 * r < R) locs[warp + 8 * r] = t;
      }
    }
    if (tid < 2 * kPanNb) {
      const int q = tid & (kPanNb - 1);
      const bool isw = tid >= kPanNb;
      double t = 0.0;
      if (q < j && tau != 0.0)
        for (int il = 0; il < R; ++il) {
          const int i = r0 + il;
          if (i > k && i < n) {
            const double vi = i == k + 1 ? v0 : xk[i];
            t = fma(isw ? Ws[il][q] : Vs[il][q], vi, t);
          }
        }
      vtot[tid] = t;   // staging of this CTA's partials
    }
    __syncthreads();
    for (int idx = tid; idx < kTriCtas * 2 * kPanNb; idx += blockDim.x) {
      const int dst = idx / (2 * kPanNb), q = idx - dst * (2 * kPanNb);
      tri_st_async1(tri_mapa(tri_saddr(&vtb[buf][c][q]), dst), vtot[q], tri_mapa(tri_saddr(&barB[buf]), dst));
    }
    tri_mbar_wait(&barB[buf], par);
    __syncthreads();   // vtot (staging) is rewritten below
    if (tid < 2 * kPanNb) {
      double t = 0.0;
      for (int q = 0; q < kTriCtas; ++q) t += vtb[buf][q][tid];
      vtot[tid] = t;    // [0, nb): V^T v, [nb, 2 nb): W^T v
    }
    __syncthreads();
    // ---- phase C: p = tau (A v - V (W^T v) - W (V^T v)) on my rows; K = v^T p
    double kw = 0.0;
    if (tid < R) {
      const int i = r0 + tid;
      double p = 0.0, vi = 0.0;
      if (i < n && i > k && tau != 0.0) {
        p = locs[tid];
        for (int q = 0; q < j; ++q) p -= Vs[tid][q] * vtot[kPanNb + q] + Ws[tid][q] * vtot[q];
        p *= tau;
        vi = i == k + 1 ? v0 : xk[i];
      }
      locp[tid] = p;
      kw = vi * p;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kw += __shfl_xor_sync(0xffffffffu, kw, o);
    if (lane == 0) wred[warp] = kw;
    __syncthreads();
    if (tid < kTriCtas) {
      double kp = 0.0;
      for (int w = 0; w < 8; ++w) kp += wred[w];
      tri_st_async1(tri_mapa(tri_saddr(&kb[buf][c]), tid), kp, tri_mapa(tri_saddr(&barC[buf]), tid));
    }
    // the owner of row k + 1 (k + 1 < n: panels stop 512 columns before the end): p_{k+1} and
    // that row of V, W (columns < j) for every CTA
    const int own = (k + 1) / R;
    if (c == own) {
      const int il = k + 1 - r0;
      for (int idx = tid; idx < kTriCtas * (1 + 2 * kPanNb); idx += blockDim.x) {
        const int dst = idx / (1 + 2 * kPanNb), q = idx - dst * (1 + 2 * kPanNb);
        double val;
        if (q == 0) val = locp[il];
        else if (q <= kPanNb) val = (q - 1 < j) ? Vs[il][q - 1] : 0.0;
        else val = (q - 1 - kPanNb < j) ? Ws[il][q - 1 - kPanNb] : 0.0;
        tri_st_async1(tri_mapa(tri_saddr(&rowb[buf][q]), dst), val, tri_mapa(tri_saddr(&barC[buf]), dst));
      }
    }
    tri_mbar_wait(&barC[buf], par);
    double K = 0.0;
    for (int q = 0; q < kTriCtas; ++q) K += kb[buf][q];
    const double h = 0.5 * tau * K;
    if (tid < R) {
      const int i = r0 + tid;
      const bool act = i < n && i > k && tau != 0.0;
      const double vi = act ? (i == k + 1 ? v0 : xk[i]) : 0.0;
      Vs[tid][j] = vi;
      Ws[tid][j] = act ? locp[tid] - h * vi : 0.0;
    }
    if (tid < kPanNb) {
      // row k + 1 of V and W for the next column's correction
      const int q = tid;
      if (q < j) { rowV[q] = rowb[buf][1 + q]; rowW[q] = rowb[buf][1 + kPanNb + q]; }
      else if (q == j) { rowV[q] = tau != 0.0 ? v0 : 0.0; rowW[q] = tau != 0.0 ? rowb[buf][0] - h * v0 : 0.0; }
    }
    __syncthreads();
  }
  // panel outputs: reflector columns (all rows of this CTA), W rows, tau / e
  for (int idx = tid; idx < R * nb; idx += blockDim.x) {
    const int q = idx / R, il = idx - q * R, i = r0 + il;
    if (i < n) {
      Vh[i + static_cast<int64_t>(k0 + q) * ldv] = Vs[il][q];
      W[i + static_cast<int64_t>(q) * n] = Ws[il][q];
    }
  }
  if (c == 0)
    for (int q = tid; q < nb; q += blockDim.x) { tauv[k0 + q] = tau_s[q]; e[k0 + q] = e_s[q]; }
  cluster.sync();
}

// Number of eigenvalues >= x of the symmetric tridiagonal (d, e2 = e^2): n minus the number of
// sign changes of the Sturm sequence p_{-1} = 1, p_j = (d_j - x) p_{j-1} - e_{j-1}^2 p_{j-2}
// (e2[0] = 0; no divisions; a zero p_j takes the sign opposite to p_{j-1}).  The caller scales
// (d, e2, x) by (s, s^2, s) with s an exact power of two so that |d|, |x| <= 2 and e2 <= 1:
// every p_j scales by s^(j+1) exactly, so the count is unchanged, and |p_j| grows by at most 2^3
// per step, which lets the power-of-two renormalisation run once per 8 steps.  d and e2 are
// padded to a multiple of 8 with (d = 4, e2 = 0): d - x > 0 there, no sign change.
constexpr int kSturmUnroll = 8;
__device__ __forceinline__ int sturm_count_gt(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                              double x) {
  int neg = 0;
  double pm = 0.0, pc = 1.0;
  const int npad = (n + kSturmUnroll - 1) & ~(kSturmUnroll - 1);
  for (int j0 = 0; j0 < npad; j0 += kSturmUnroll) {
    double dv[kSturmUnroll], ev[kSturmUnroll];
#pragma unroll
    for (int u = 0; u < kSturmUnroll; u += 2) {
      const double2 a = *reinterpret_cast<const double2*>(d + j0 + u);
      const double2 b = *reinterpret_cast<const double2*>(e2 + j0 + u);
      dv[u] = a.x; dv[u + 1] = a.y; ev[u] = b.x; ev[u + 1] = b.y;
    }
#pragma unroll
    for (int u = 0; u < kSturmUnroll; ++u) {
      double pn = fma(dv[u] - x, pc, -ev[u] * pm);
      if (pn == 0.0) pn = (pc < 0.0) ? 0x1p-1000 : -0x1p-1000;
      neg += (pn < 0.0) != (pc < 0.0);
      pm = pc;
      pc = pn;
    }
    const double a = fabs(pc);
    if (a > 0x1p+400 || a < 0x1p-400) {
      const double sc = ldexp(1.0, -ilogb(pc));
      pc *= sc;
      pm *= sc;
    }
  }
  return n - neg;
}

// smem doubles multisect_kernel needs for order n
__host__ __device__ constexpr int multisect_smem_doubles(int n) { return 2 * ((n + kSturmUnroll - 1) & ~(kSturmUnroll - 1)); }

// Eigenvalues mu[i] (descending) for i < nev, plus mu[n-1] when `smallest` (one warp each).
__global__ void __launch_bounds__(256) multisect_kernel(const double* __restrict__ d, const double* __restrict__ e, int n,
                                                        double* __restrict__ mu, int nev, int smallest) {
  extern __shared__ double ms_smem[];
  const int npad = (n + kSturmUnroll - 1) & ~(kSturmUnroll - 1);
  double* ds = ms_smem;
  double* e2 = ms_smem + npad;
  __shared__ double bnd[4];
  const int tid = threadIdx.x;
  if (tid == 0) {
    double lo = INFINITY, hi = -INFINITY, tmax = 0.0;
    for (int j = 0; j < n; ++j) {
      const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + (j < n - 1 ? fabs(e[j]) : 0.0);
      lo = fmin(lo, d[j] - r);
      hi = fmax(hi, d[j] + r);
      tmax = fmax(tmax, fabs(d[j]) + r);
    }
    const double eps = 2.220446049250313e-16;
    const double pad = 2.0 * eps * tmax + 1e-300;
    bnd[0] = lo - pad;
    bnd[1] = hi + pad;
    bnd[2] = tmax > 0.0 ? ldexp(1.0, -ilogb(tmax) - 1) : 1.0;   // s: s tmax in [0.5, 1)
    bnd[3] = 4.0 * eps * tmax;                                    // absolute accuracy of a Sturm count
  }
  __syncthreads();
  const double sc = bnd[2];
  for (int j = tid; j < npad; j += blockDim.x) {
    // |d_j| + |e_j| <= tmax, so s |d_j| < 1, s^2 e_j^2 < 1; |s x| < 2 for x in [lo, hi]
    ds[j] = j < n ? sc * d[j] : 4.0;
    const double ev = (j > 0 && j < n) ? sc * e[j - 1] : 0.0;
    e2[j] = ev * ev;
  }
  __syncthreads();
  const int warp = (blockIdx.x * blockDim.x + tid) >> 5, lane = tid & 31;
  if (warp >= nev + smallest) return;
  const int i = warp < nev ? warp : n - 1;   // target: (i+1)-th largest
  double lo = bnd[0], hi = bnd[1];
  const double eps = 2.220446049250313e-16;
  for (int it = 0; it < 40; ++it) {
    if (hi - lo <= fmax(2.0 * eps * fmax(fabs(lo), fabs(hi)), bnd[3]) + 1e-300) break;
    const double x = lo + (hi - lo) * static_cast<double>(lane + 1) / 33.0;
    const int gt = sturm_count_gt(ds, e2, n, sc * x);   // #eigenvalues >= x
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
                                     double* __restrict__ ldl, int tri_ok, int frob_idx) {
  __shared__ double red[8];
  extern __shared__ double ls_smem[];   // mus, ds, es: 3 n doubles (the serial loops read shared memory)
  double* mus = ls_smem;
  double* ds = ls_smem + n;
  double* es = ls_smem + 2 * n;
  double tr = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    tr += gram[static_cast<int64_t>(i) * n + i];   // Gram order n
    mus[i] = mu[i];
    ds[i] = d[i];
    if (i < n - 1) es[i] = e[i];
  }
  tr = block_sum<256>(tr, red);   // (synchronises the block)
  if (threadIdx.x != 0) return;
  d = ds;
  e = es;
  double Ek = 0.0;
  for (int i = 0; i < k && i < n; ++i) Ek += mus[i];
  const double frob2 = scal[frob_idx];
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
    // D_j >= shift > 0 (T + sI is positive definite); one reciprocal per pivot on the sequential
    // chain, from the hardware approximation refined by two Newton steps (about 1 ulp)
    const auto rcp = rcp_nr;
    double Dj = d[0] + shift;
    double rj = rcp(Dj);
    ldl[0] = rj;
    for (int j = 1; j < n; ++j) {
      const double ej = e[j - 1];
      const double Lj = ej * rj;
      ldl[n + j - 1] = Lj;
      Dj = fma(-Lj, ej, d[j] + shift);
      rj = rcp(Dj);
      ldl[j] = rj;
    }
  }
}

__global__ void __launch_bounds__(256) wy_t_kernel(const double* __restrict__ Vh, const double* __restrict__ tauv, int n,
                                                   double* __restrict__ wyT) {
  __shared__ double G[kRefChunk][kRefChunk];
  wy_t_chunk(blockIdx.x, Vh, tauv, n, wyT, G);
}

// Shared-memory state of cta_apply_q (one vector per CTA): kQStages ring of reflector chunks
// (V rows [k0_even, ldv) of 8 reflectors + their T) filled by cp.async.bulk on mbarriers.
struct QSmem {
  double* v;          // [kQStages][kRefChunk][ldv] (dynamic)
  double* t;          // [kQStages][64]
  uint64_t* full;     // [kQStages]
  double (*red)[8][kRefChunk];   // [2][warps][8]
};

__device__ __forceinline__ void q_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tri_saddr(dst)),
               "l"(src), "r"(bytes), "r"(tri_saddr(bar))
               : "memory");
}

// z <- Q^T z (forward: H_{n-3} ... H_0 z) or Q z (backward: H_0 ... H_{n-3} z) for ONE vector held in
// registers (thread tid owns rows tid and tid + 256), one compact-WY chunk at a time:
// w = V^T z (per-thread partial products, fixed-order warp and cross-warp sums), u = T^T w
// (forward) or T w (backward), z -= V u.  `uses` counts the ring's fills across calls (parity).
__device__ __forceinline__ void cta_apply_q(double (&z)[2], int n, const double* __restrict__ Vh,
                                            const double* __restrict__ wyT, bool forward, QSmem& sm, int& uses) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = n - 2, ldv = tri_ldv(n);
  if (nk <= 0) return;
  const int nch = (nk + kRefChunk - 1) / kRefChunk;
  auto chunk_of = [&](int it) { return forward ? it : nch - 1 - it; };
  auto issue = [&](int it) {        // thread 0 only
    const int b = chunk_of(it), k0 = b * kRefChunk, k0e = k0 & ~1;
    const int nr = min(kRefChunk, nk - k0);
    const int st = (uses + it) % kQStages;
    const uint32_t row_bytes = static_cast<uint32_t>(ldv - k0e) * 8u;
    tri_mbar_expect(&sm.full[st], static_cast<uint32_t>(nr) * row_bytes + 64u * 8u);
    q_bulk(sm.t + st * 64, wyT + b * 64, 64u * 8u, &sm.full[st]);
    for (int r = 0; r < nr; ++r)
      q_bulk(sm.v + (static_cast<size_t>(st) * kRefChunk + r) * ldv + k0e, Vh + static_cast<int64_t>(k0 + r) * ldv + k0e,
             row_bytes, &sm.full[st]);
  };
  if (tid == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }
  for (int it = 0; it < nch; ++it) {
    const int b = chunk_of(it), k0 = b * kRefChunk;
    const int nr = min(kRefChunk, nk - k0);
    const int g = uses + it, st = g % kQStages;
    tri_mbar_wait(&sm.full[st], (g / kQStages) & 1);
    const double* vb = sm.v + static_cast<size_t>(st) * kRefChunk * ldv;
    double v[kRefChunk][2], pr[kRefChunk];
#pragma unroll
    for (int r = 0; r < kRefChunk; ++r) {
      pr[r] = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int i = tid + 256 * s;
        v[r][s] = (r < nr && i > k0 && i < n) ? vb[r * ldv + i] : 0.0;   // rows <= k0 are zero in V
        pr[r] = fma(v[r][s], z[s], pr[r]);
      }
    }
    // warp sums by a butterfly reduce-scatter: value r ends in lanes 4 r .. 4 r + 3 (9 shuffles
    // instead of 40)
    static_assert(kRefChunk == 8, "butterfly below is written for 8 values");
#pragma unroll
    for (int half = 4; half > 0; half >>= 1) {
      const bool hi = (lane & (4 * half)) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const double send = hi ? pr[i] : pr[i + half];
        const double keep = hi ? pr[i + half] : pr[i];
        pr[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4 * half);
      }
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) pr[0] += __shfl_xor_sync(0xffffffffu, pr[0], o);
    double (*red)[kRefChunk] = sm.red[it & 1];
    if ((lane & 3) == 0) red[warp][lane >> 2] = pr[0];
    double T[kRefChunk * kRefChunk];
#pragma unroll
    for (int q = 0; q < kRefChunk * kRefChunk; ++q) T[q] = sm.t[st * 64 + q];
    __syncthreads();                      // V_it in registers, red complete; stage (it-1) % 3 free
    if (tid == 0 && it + 2 < nch) issue(it + 2);
    double w[kRefChunk];
#pragma unroll
    for (int r = 0; r < kRefChunk; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += red[q][r];
      w[r] = acc;
    }
    double u[kRefChunk];
#pragma unroll
    for (int c = 0; c < kRefChunk; ++c) {
      double acc = 0.0;
      if (forward) {
#pragma unroll
        for (int r = 0; r <= c; ++r) acc = fma(T[r * kRefChunk + c], w[r], acc);    // (T^T w)_c
      } else {
#pragma unroll
        for (int q = c; q < kRefChunk; ++q) acc = fma(T[c * kRefChunk + q], w[q], acc);   // (T w)_c
      }
      u[c] = acc;
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      double zi = z[s];
#pragma unroll
      for (int r = 0; r < kRefChunk; ++r) zi = fma(-v[r][s], u[r], zi);
      z[s] = zi;
    }
  }
  uses += nch;
  __syncthreads();                        // red / ring reuse by a following call
}

// z_v <- Q^T z_v for kQV vectors at once (the reflector chunks are read once per CTA for all of
// them).  Per chunk: the 8 kQV partial dot products of each thread are reduced over the warp by a
// butterfly reduce-scatter (lane l ends with value l: 31 shuffles instead of 5 per value), over
// the warps through shared memory; warp 0 forms u = T^T w (one (vector, column) per lane) and
// every thread applies z -= V u.
constexpr int kQV = 4;   // vectors per CTA (kQV * kRefChunk == 32: one reduced value per lane)
static_assert(kQV * kRefChunk == 32, "one reduced value per lane");
// NS entries per thread, NT threads (n <= NT NS), QST ring stages (chunks 0 .. QST-1 issued up
// front; chunk it + QST into stage it % QST once chunk it is fully consumed)
template <int NS, int NT, int QST>
__device__ __forceinline__ void cta_apply_qt_multi(double (&z)[kQV][NS], int n, const double* __restrict__ Vh,
                                                   const double* __restrict__ wyT, double* vring, double* tring,
                                                   uint64_t* full, double (*redm)[NT / 32][32], double* us) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = n - 2, ldv = tri_ldv(n);
  if (nk <= 0) return;
  const int nch = (nk + kRefChunk - 1) / kRefChunk;
  auto issue = [&](int b) {        // thread 0 only
    const int k0 = b * kRefChunk, k0e = k0 & ~1;
    const int nr = min(kRefChunk, nk - k0);
    const int st = b % QST;
    const uint32_t row_bytes = static_cast<uint32_t>(ldv - k0e) * 8u;
    tri_mbar_expect(&full[st], static_cast<uint32_t>(nr) * row_bytes + 64u * 8u);
    q_bulk(tring + st * 64, wyT + b * 64, 64u * 8u, &full[st]);
    for (int r = 0; r < nr; ++r)
      q_bulk(vring + (static_cast<size_t>(st) * kRefChunk + r) * ldv + k0e, Vh + static_cast<int64_t>(k0 + r) * ldv + k0e,
             row_bytes, &full[st]);
  };
  if (tid == 0)
    for (int b = 0; b < QST && b < nch; ++b) issue(b);
  for (int it = 0; it < nch; ++it) {
    const int k0 = it * kRefChunk;
    const int nr = min(kRefChunk, nk - k0);
    const int st = it % QST;
    tri_mbar_wait(&full[st], (it / QST) & 1);
    const double* vb = vring + static_cast<size_t>(st) * kRefChunk * ldv;
    double v[kRefChunk][NS];
#pragma unroll
    for (int r = 0; r < kRefChunk; ++r)
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int i = tid + NT * s;
        v[r][s] = (r < nr && i > k0 && i < n) ? vb[r * ldv + i] : 0.0;   // rows <= k0 are zero in V
      }
    double val[32];
#pragma unroll
    for (int q = 0; q < kQV; ++q)
#pragma unroll
      for (int r = 0; r < kRefChunk; ++r) {
        double acc = v[r][0] * z[q][0];
#pragma unroll
        for (int s = 1; s < NS; ++s) acc = fma(v[r][s], z[q][s], acc);
        val[q * kRefChunk + r] = acc;
      }
#pragma unroll
    for (int half = 16; half > 0; half >>= 1) {
      const bool hi = (lane & half) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const double send = hi ? val[i] : val[i + half];
        const double keep = hi ? val[i + half] : val[i];
        val[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
      }
    }
    redm[it & 1][warp][lane] = val[0];   // warp sum of value `lane` = (vector lane / 8, row lane % 8)
    __syncthreads();                     // V_it in registers, redm complete
    if (warp == 0) {
      double w = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) w += redm[it & 1][q][lane];
      const int c = lane & (kRefChunk - 1), base = lane & ~(kRefChunk - 1);
      const double* T = tring + st * 64;
      double u = 0.0;
#pragma unroll
      for (int r = 0; r < kRefChunk; ++r) {
        const double wr = __shfl_sync(0xffffffffu, w, base + r);
        if (r <= c) u = fma(T[r * kRefChunk + c], wr, u);   // (T^T w)_c
      }
      us[(it & 1) * 32 + lane] = u;
    }
    __syncthreads();                     // stage st (V and T) fully consumed
    if (tid == 0 && it + QST < nch) issue(it + QST);
#pragma unroll
    for (int q = 0; q < kQV; ++q)
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        double zi = z[q][s];
#pragma unroll
        for (int r = 0; r < kRefChunk; ++r) zi = fma(-v[r][s], us[(it & 1) * 32 + q * kRefChunk + r], zi);
        z[q][s] = zi;
      }
  }
  __syncthreads();
}

// A5 fast path: tau(y) = z^T (T + sI)^-1 z with z = Q^T y = H_{n-3} ... H_0 y, y = column j of Yc
// (ell x ncol), for kQV columns per CTA; the LDL^T chains run on kQV threads.  Runs when gate[0] != 0.
template <int NS, int NT, int QST>
__global__ void __launch_bounds__(NT) tri_scores_multi_kernel(const double* __restrict__ Yc, int n, int ncol,
                                                               const double* __restrict__ Vh, const double* __restrict__ wyT,
                                                               const double* __restrict__ ldl, const int* __restrict__ gate,
                                                               double* __restrict__ tau_out, double* __restrict__ zout) {
  // zout != nullptr: only z = Q^T y (n x ncol into zout), before the gate and the LDL^T factors
  // exist (tri_scores_chain_kernel finishes); otherwise the whole score
  if (zout == nullptr && gate[0] == 0) return;
  extern __shared__ __align__(16) double ref_smem[];
  __shared__ __align__(16) double tsm[QST * 64];
  __shared__ __align__(8) uint64_t full[QST];
  __shared__ double redm[2][NT / 32][32];
  __shared__ double us[64];
  const int tid = threadIdx.x, j0 = blockIdx.x * kQV;
  if (tid == 0) {
    for (int q = 0; q < QST; ++q) tri_mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double z[kQV][NS];
#pragma unroll
  for (int q = 0; q < kQV; ++q)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int i = tid + NT * s;
      z[q][s] = (i < n && j0 + q < ncol) ? Yc[static_cast<int64_t>(j0 + q) * n + i] : 0.0;
    }
  __syncthreads();
  cta_apply_qt_multi<NS, NT, QST>(z, n, Vh, wyT, ref_smem, tsm, full, redm, us);
  if (zout != nullptr) {
#pragma unroll
    for (int q = 0; q < kQV; ++q)
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int i = tid + NT * s;
        if (i < n && j0 + q < ncol) zout[static_cast<int64_t>(j0 + q) * n + i] = z[q][s];
      }
    return;
  }
  // the reflector ring is free again (cta_apply_qt_multi ends with a barrier): z and the LDL^T
  // factors go to the start of the dynamic shared memory (kQV n + 2 n doubles <= the ring)
  double* zs = ref_smem;
  double* ls = ref_smem + kQV * n;
#pragma unroll
  for (int q = 0; q < kQV; ++q)
#pragma unroll
    for (int s = 0; s < NS; ++s) if (tid + NT * s < n) zs[q * n + tid + NT * s] = z[q][s];
  for (int i = tid; i < 2 * n - 1; i += blockDim.x) ls[i] = ldl[i];
  __syncthreads();
  if (tid < kQV && j0 + tid < ncol) {
    const double* zq = zs + tid * n;
    double y = zq[0];
    double acc = y * y * ls[0];
    for (int i = 1; i < n; ++i) {
      y = zq[i] - ls[n + i - 1] * y;
      acc = fma(y * y, ls[i], acc);
    }
    tau_out[j0 + tid] = acc;
  }
}

// tau_j = z_j^T (T + sI)^-1 z_j from z = Q^T y (tri_scores_multi_kernel with zout): kQV columns
// per CTA, the serial LDL^T chains on kQV threads; runs when gate[0] != 0.
__global__ void __launch_bounds__(128) tri_scores_chain_kernel(const double* __restrict__ Z, int n, int ncol,
                                                               const double* __restrict__ ldl, const int* __restrict__ gate,
                                                               double* __restrict__ tau_out) {
  if (gate[0] == 0) return;
  extern __shared__ double chain_smem[];   // zs[kQV][n], ls[2 n]: (kQV + 2) n doubles
  double* zs = chain_smem;
  double* ls = chain_smem + kQV * n;
  const int tid = threadIdx.x, j0 = blockIdx.x * kQV;
  for (int e = tid; e < kQV * n; e += blockDim.x) {
    const int q = e / n, i = e - q * n;
    zs[q * n + i] = j0 + q < ncol ? Z[static_cast<int64_t>(j0 + q) * n + i] : 0.0;
  }
  for (int i = tid; i < 2 * n - 1; i += blockDim.x) ls[i] = ldl[i];
  __syncthreads();
  if (tid < kQV && j0 + tid < ncol) {
    const double* zq = zs + tid * n;
    double y = zq[0];
    double acc = y * y * ls[0];
    for (int i = 1; i < n; ++i) {
      y = zq[i] - ls[n + i - 1] * y;
      acc = fma(y * y, ls[i], acc);
    }
    tau_out[j0 + tid] = acc;
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
  double rj = rcp_nr(Dj);   // D_j > 0: A is positive definite here
  ldl[0] = rj;
  for (int j = 1; j < n; ++j) {
    const double ej = e[j - 1];
    const double Lj = ej * rj;
    ldl[n + j - 1] = Lj;
    Dj = fma(-Lj, ej, d[j]);
    rj = rcp_nr(Dj);
    ldl[j] = rj;
  }
}

// X(:, c) = A^-1 R(:, c) with A = Q T Q^T: z = Q^T r, solve T u = z (LDL^T), x = Q u.
// One right-hand side per CTA; runs when gate[0] != 0.  in_transposed: R(i, c) = R[c + i ldr];
// out_transposed: write X^T (nrhs x n).  Dynamic smem: kQStages kRefChunk tri_ldv(n) doubles.
__global__ void __launch_bounds__(256) tri_solve_kernel(const double* __restrict__ R, int64_t ldr, int in_transposed,
                                                        int n, int nrhs, const double* __restrict__ Vh,
                                                        const double* __restrict__ wyT, const double* __restrict__ ldl,
                                                        const int* __restrict__ gate, double* __restrict__ X,
                                                        int64_t ldx, int out_transposed) {
  if (gate[0] == 0) return;
  extern __shared__ __align__(16) double ref_smem[];
  __shared__ __align__(16) double tsm[kQStages * 64];
  __shared__ __align__(8) uint64_t full[kQStages];
  __shared__ double red[2][8][kRefChunk];
  __shared__ double zs[kTriMaxN];
  __shared__ double ls[2 * kTriMaxN];   // LDL^T factors (1/D, L)
  const int tid = threadIdx.x, c = blockIdx.x;
  if (tid == 0) {
    for (int q = 0; q < kQStages; ++q) tri_mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double z[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = tid + 256 * s;
    z[s] = i < n ? (in_transposed ? R[c + static_cast<int64_t>(i) * ldr] : R[static_cast<int64_t>(c) * ldr + i]) : 0.0;
  }
  __syncthreads();
  QSmem sm{ref_smem, tsm, full, red};
  int uses = 0;
  cta_apply_q(z, n, Vh, wyT, true, sm, uses);                                // z = Q^T r
#pragma unroll
  for (int s = 0; s < 2; ++s) if (tid + 256 * s < n) zs[tid + 256 * s] = z[s];
  __syncthreads();
  for (int i = tid; i < 2 * n - 1; i += blockDim.x) ls[i] = ldl[i];   // the chains below read shared memory
  __syncthreads();
  if (tid == 0) {                                                            // T u = z by LDL^T
    double y = zs[0];
    for (int i = 1; i < n; ++i) { y = zs[i] - ls[n + i - 1] * y; zs[i] = y; }
    for (int i = 0; i < n; ++i) zs[i] *= ls[i];
    y = zs[n - 1];
    for (int i = n - 2; i >= 0; --i) { y = zs[i] - ls[n + i] * y; zs[i] = y; }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) z[s] = tid + 256 * s < n ? zs[tid + 256 * s] : 0.0;
  cta_apply_q(z, n, Vh, wyT, false, sm, uses);                               // x = Q u
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = tid + 256 * s;
    if (i < n) {
      if (out_transposed) X[static_cast<int64_t>(i) * ldx + c] = z[s];
      else X[static_cast<int64_t>(c) * ldx + i] = z[s];
    }
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
