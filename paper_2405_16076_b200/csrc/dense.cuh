// Small dense fp64 kernels of the post-pass (Gram, GEMM, one-sided Jacobi SVD / eigen,
// traces).  All reductions run in a fixed order, so results are bitwise reproducible.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace oid {
namespace cg = cooperative_groups;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// out = ||A||_F^2 over len doubles (one CTA, fixed order)
__global__ void fro2_kernel(const double* __restrict__ A, int64_t len, double* __restrict__ out,
                            const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s = fma(A[i], A[i], s);
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = s;
}

// C (M x N, ldc) = alpha * op(A) * op(B) + beta * C, column-major, op = transpose if T*.
// 32x32 output tile per CTA, 256 threads x 4 outputs, K staged in 16-wide smem panels.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) dgemm_kernel(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                    int64_t lda, const double* __restrict__ B, int64_t ldb, double beta,
                                                    double* __restrict__ C, int64_t ldc, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double As[16][33];
  __shared__ double Bs[16][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 0..7
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 32; e += 256) {
      const int kk = e >> 5, ii = e & 31;
      const int i = i0 + ii, k = k0 + kk;
      double a = 0.0;
      if (i < M && k < K) a = TA ? A[k + static_cast<int64_t>(i) * lda] : A[i + static_cast<int64_t>(k) * lda];
      As[kk][ii] = a;
      const int j = j0 + ii;
      double b = 0.0;
      if (j < N && k < K) b = TB ? B[j + static_cast<int64_t>(k) * ldb] : B[k + static_cast<int64_t>(j) * ldb];
      Bs[kk][ii] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const double a = As[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(a, Bs[kk][ty + 8 * q], acc[q]);
    }
    __syncthreads();
  }
  const int i = i0 + tx;
  if (i < M) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + ty + 8 * q;
      if (j < N) {
        double* c = C + i + static_cast<int64_t>(j) * ldc;
        *c = (beta == 0.0) ? alpha * acc[q] : fma(beta, *c, alpha * acc[q]);
      }
    }
  }
}

// Gram += Y Y^T (ell x ell), S(:, n0:n0+nc) = Y, frob2 += sum n_j  (Alg 3 steps 10-13).
// Y: ell x nc sketches (ld ell), nrm: their nc squared column norms
__global__ void gram_update_kernel(const double* __restrict__ Yp, const double* __restrict__ nrm, int ell, int nc,
                                   double* __restrict__ gram, double* __restrict__ S, int64_t n0,
                                   double* __restrict__ scal) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(ell) * ell;
  if (idx < nn) {
    const int r = static_cast<int>(idx % ell), c = static_cast<int>(idx / ell);
    double s = gram[idx];
    for (int j = 0; j < nc; ++j) s = fma(Yp[r + static_cast<int64_t>(j) * ell], Yp[c + static_cast<int64_t>(j) * ell], s);
    gram[idx] = s;
  }
  const int64_t ny = static_cast<int64_t>(ell) * nc;
  if (idx < ny) S[n0 * ell + idx] = Yp[idx];
  if (idx == 0) {
    double f = scal[0];
    for (int j = 0; j < nc; ++j) f += nrm[j];
    scal[0] = f;
  }
}

// dst(:, j) = src(:, j), j < ncols, rows < m (column-major, leading dimensions lds / ldd)
template <typename T>
__global__ void copy_cols_kernel(const T* __restrict__ src, int64_t lds, T* __restrict__ dst, int64_t ldd, int64_t m,
                                 int ncols) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m * ncols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i / m, r = i - j * m;
    dst[j * ldd + r] = src[j * lds + r];
  }
}

// One-sided (Hestenes) Jacobi: orthogonalise the n columns of B (L x n) by plane rotations
// accumulated in V (n x n, initialised by the caller).  Round-robin pair ordering, one
// pair per CTA per round, one grid-wide barrier per round.  Sweeps stop when a sweep
// applies no rotation (|b_p.b_q| <= tol sqrt(|b_p|^2 |b_q|^2)).  Cooperative launch.
__global__ void __launch_bounds__(256) jacobi_svd_kernel(double* __restrict__ B, int L, int n, double* __restrict__ V,
                                                         int* __restrict__ counters, int max_sweeps, double tol) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[3][8];
  const int nn = n + (n & 1);
  const int npairs = nn / 2;
  const int m1 = nn - 1;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int k = 0; k < m1; ++k) {
      for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
        int a, b;
        if (pi == 0) { a = m1; b = k; } else { a = (k + pi) % m1; b = (k - pi + m1) % m1; }
        const int p = min(a, b), q = max(a, b);
        if (q >= n) continue;
        double* bp = B + static_cast<int64_t>(p) * L;
        double* bq = B + static_cast<int64_t>(q) * L;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
          const double x = bp[i], y = bq[i];
          al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) { red[0][w] = al; red[1][w] = be; red[2][w] = ga; }
        __syncthreads();
        al = 0.0; be = 0.0; ga = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { al += red[0][i]; be += red[1][i]; ga += red[2][i]; }
        __syncthreads();
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          double t;
          if (fabs(zeta) > 1e150) t = 0.5 / zeta;
          else t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = 1.0 / sqrt(fma(t, t, 1.0)), s = c * t;
          for (int i = threadIdx.x; i < L; i += blockDim.x) {
            const double x = bp[i], y = bq[i];
            bp[i] = c * x - s * y;
            bq[i] = s * x + c * y;
          }
          double* vp = V + static_cast<int64_t>(p) * n;
          double* vq = V + static_cast<int64_t>(q) * n;
          for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
          if (threadIdx.x == 0) atomicAdd(&counters[sweep], 1);
        }
      }
      grid.sync();
    }
    const int rotated = atomicAdd(&counters[sweep], 0);
    if (rotated == 0) break;
  }
}

// Block one-sided Jacobi: the n columns of B (L x n) are cut into blocks of W columns; each
// outer round pairs blocks round-robin and one CTA (W warps) orthogonalises the 2W columns of
// its block pair with one inner cyclic sweep held in shared memory (B and V columns staged),
// one warp per column pair, warp-shuffle dot products.  One grid-wide barrier per outer round;
// outer sweeps stop when a sweep applies no rotation.  V (n x n) must hold the initial
// orthogonal matrix (identity or a warm start) and B = A V on entry.  Cooperative launch,
// dynamic smem = 2W (L + n) doubles.
template <int W>
__global__ void __launch_bounds__(32 * W) bjacobi_kernel(double* __restrict__ B, int L, int n, double* __restrict__ V,
                                                         int* __restrict__ counters, int max_sweeps, double tol,
                                                         const double* __restrict__ fro2, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* Bs = sm;                       // [2W][L]
  double* Vs = sm + 2 * W * L;           // [2W][n]
  __shared__ int gcol[2 * W];
  __shared__ int nrot;
  const int nb = (n + W - 1) / W;
  const int nbb = nb + (nb & 1);
  const int npairs = nbb / 2;
  const int m1 = nbb - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double floor2 = 1e-28 * (*fro2);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int k = 0; k < max(m1, 1); ++k) {
      for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
        int a, b;
        if (pi == 0) { a = m1; b = k; } else { a = (k + pi) % m1; b = (k - pi + m1) % m1; }
        if (m1 == 0) { a = 0; b = 1; }
        const int P = min(a, b), Q = max(a, b);
        if (P >= nb) continue;
        if (threadIdx.x < 2 * W) {
          const int c = threadIdx.x;
          const int blk = c < W ? P : Q;
          const int g = blk * W + (c % W);
          gcol[c] = (blk < nb && g < n) ? g : -1;
        }
        if (threadIdx.x == 0) nrot = 0;
        __syncthreads();
        // stage the 2W columns of B and V with asynchronous 8-byte copies (all in flight at once)
        for (int e = threadIdx.x; e < 2 * W * L; e += blockDim.x) {
          const int c = e / L, i = e - c * L;
          const int g = gcol[c];
          if (g >= 0) cp_async8(Bs + e, B + static_cast<int64_t>(g) * L + i);
        }
        for (int e = threadIdx.x; e < 2 * W * n; e += blockDim.x) {
          const int c = e / n, i = e - c * n;
          const int g = gcol[c];
          if (g >= 0) cp_async8(Vs + e, V + static_cast<int64_t>(g) * n + i);
        }
        cp_async_wait_all();
        __syncthreads();
        const int m2 = 2 * W - 1;
        for (int r = 0; r < m2; ++r) {
          int p, q;
          if (warp == 0) { p = m2; q = r; } else { p = (r + warp) % m2; q = (r - warp + m2) % m2; }
          if (p > q) { const int tmp = p; p = q; q = tmp; }
          if (gcol[p] >= 0 && gcol[q] >= 0) {
            double* bp = Bs + p * L;
            double* bq = Bs + q * L;
            double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll 4
            for (int i = lane; i < L; i += 32) {
              const double x = bp[i], y = bq[i];
              al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              al += __shfl_xor_sync(0xffffffffu, al, o);
              be += __shfl_xor_sync(0xffffffffu, be, o);
              ga += __shfl_xor_sync(0xffffffffu, ga, o);
            }
            // columns at the rounding-noise level of B (||b||^2 <= (1e-14 ||B||_F)^2) are not rotated:
            // they carry no information and would never satisfy the relative test.
            if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be) && fmin(al, be) > floor2) {
              const double zeta = (be - al) / (2.0 * ga);
              double t;
              if (fabs(zeta) > 1e150) t = 0.5 / zeta;
              else t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              const double cs = 1.0 / sqrt(fma(t, t, 1.0)), sn = cs * t;
#pragma unroll 4
              for (int i = lane; i < L; i += 32) {
                const double x = bp[i], y = bq[i];
                bp[i] = cs * x - sn * y;
                bq[i] = sn * x + cs * y;
              }
              double* vp = Vs + p * n;
              double* vq = Vs + q * n;
#pragma unroll 4
              for (int i = lane; i < n; i += 32) {
                const double x = vp[i], y = vq[i];
                vp[i] = cs * x - sn * y;
                vq[i] = sn * x + cs * y;
              }
              if (lane == 0) atomicAdd(&nrot, 1);
            }
          }
          __syncthreads();
        }
        for (int c = 0; c < 2 * W; ++c) {
          const int g = gcol[c];
          if (g < 0) continue;
          for (int i = threadIdx.x; i < L; i += blockDim.x) B[static_cast<int64_t>(g) * L + i] = Bs[c * L + i];
          for (int i = threadIdx.x; i < n; i += blockDim.x) V[static_cast<int64_t>(g) * n + i] = Vs[c * n + i];
        }
        if (threadIdx.x == 0 && nrot) atomicAdd(&counters[sweep], nrot);
        __syncthreads();
      }
      grid.sync();
    }
    const int rotated = atomicAdd(&counters[sweep], 0);
    if (rotated == 0) break;
  }
}

// Two-sided block Jacobi eigen-solver for a symmetric n x n matrix H (col-major, ld n):
// on exit H is (numerically) diagonal and V <- V U holds the accumulated rotations, so with
// H = V0^T A V0 on entry (warm start: V0 = previous eigenvectors), A = V diag(H) V^T.
// Indices are cut into blocks of W; each outer round pairs blocks round-robin.  Phase A: one
// CTA per block pair runs one cyclic sweep of scalar rotations on the 2W x 2W diagonal
// block in shared memory (parallel ordering, W rotations per step) and publishes its
// accumulated 2W x 2W rotation U_p.  Phase B: every CTA applies H[I,K] <- U_I^T H[I,K] U_K
// to 2W x 2W tiles (pairs I <= K, mirrored) and V[:, I] <- V[:, I] U_I.  Two grid barriers
// per round; sweeps stop when a sweep applies no rotation.  A rotation of (p, q) is applied
// when |h_pq| > max(tol sqrt(|h_pp h_qq|), abs_tol).  Cooperative launch.
constexpr int kSymW = 16;
constexpr int kSymB = 2 * kSymW;     // 32
constexpr int kSymP = kSymB + 1;     // smem pitch

__device__ __forceinline__ void sym_pair(int k, int pi, int m1, int& P, int& Q) {
  int a, b;
  if (pi == 0) { a = m1; b = k; } else { a = (k + pi) % m1; b = (k - pi + m1) % m1; }
  if (m1 == 0) { a = 0; b = 1; }
  P = min(a, b); Q = max(a, b);
}
__device__ __forceinline__ int sym_idx(int P, int Q, int i) { return i < kSymW ? P * kSymW + i : Q * kSymW + (i - kSymW); }

__global__ void __launch_bounds__(256) sym_bjacobi_kernel(double* __restrict__ H, double* __restrict__ V, int n,
                                                          double* __restrict__ Ubuf, int* __restrict__ flags,
                                                          int* __restrict__ counters, int max_sweeps, double tol,
                                                          const double* __restrict__ abs_tol_p,
                                                          const int* __restrict__ gate) {
  if (gate && *gate == 0) return;   // uniform over the grid: no grid.sync reached
  cg::grid_group grid = cg::this_grid();
  const double abs_tol = *abs_tol_p;
  __shared__ double S[kSymB][kSymP];
  __shared__ double U[kSymB][kSymP];
  __shared__ double T[kSymB][kSymP];
  __shared__ double rot[kSymW][2];
  __shared__ int rp[kSymW][2];
  __shared__ int nrot;
  const int tid = threadIdx.x;
  const int nb = (n + kSymW - 1) / kSymW;
  const int nbb = nb + (nb & 1);
  const int npairs = nbb / 2;
  const int m1 = nbb - 1;
  const int rounds = max(m1, 1);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int k = 0; k < rounds; ++k) {
      // ---------------- phase A: one inner cyclic sweep per block pair
      for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
        int P, Q;
        sym_pair(k, pi, m1, P, Q);
        for (int e = tid; e < kSymB * kSymB; e += 256) {
          const int i = e % kSymB, j = e / kSymB;
          const int gi = sym_idx(P, Q, i), gj = sym_idx(P, Q, j);
          S[i][j] = (gi < n && gj < n) ? H[gi + static_cast<int64_t>(gj) * n] : 0.0;
          U[i][j] = (i == j) ? 1.0 : 0.0;
        }
        if (tid == 0) nrot = 0;
        __syncthreads();
        for (int step = 0; step < kSymB - 1; ++step) {
          if (tid < kSymW) {
            int p, q;
            if (tid == 0) { p = kSymB - 1; q = step; }
            else { p = (step + tid) % (kSymB - 1); q = (step - tid + kSymB - 1) % (kSymB - 1); }
            if (p > q) { const int x = p; p = q; q = x; }
            const double app = S[p][p], aqq = S[q][q], apq = S[p][q];
            double cs = 1.0, sn = 0.0;
            if (apq != 0.0 && fabs(apq) > fmax(tol * sqrt(fabs(app * aqq)), abs_tol)) {
              const double zeta = (aqq - app) / (2.0 * apq);
              double t;
              if (fabs(zeta) > 1e150) t = 0.5 / zeta;
              else t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              cs = 1.0 / sqrt(fma(t, t, 1.0));
              sn = cs * t;
              atomicAdd(&nrot, 1);
            }
            rot[tid][0] = cs; rot[tid][1] = sn; rp[tid][0] = p; rp[tid][1] = q;
          }
          __syncthreads();
          for (int e = tid; e < kSymW * kSymB; e += 256) {      // rows: S <- J^T S
            const int r = e / kSymB, j = e % kSymB;
            const double cs = rot[r][0], sn = rot[r][1];
            if (sn == 0.0) continue;
            const int p = rp[r][0], q = rp[r][1];
            const double x = S[p][j], y = S[q][j];
            S[p][j] = cs * x - sn * y;
            S[q][j] = sn * x + cs * y;
          }
          __syncthreads();
          for (int e = tid; e < kSymW * kSymB; e += 256) {      // columns: S <- S J, U <- U J
            const int r = e / kSymB, i = e % kSymB;
            const double cs = rot[r][0], sn = rot[r][1];
            if (sn == 0.0) continue;
            const int p = rp[r][0], q = rp[r][1];
            const double x = S[i][p], y = S[i][q];
            S[i][p] = cs * x - sn * y;
            S[i][q] = sn * x + cs * y;
            const double u = U[i][p], v = U[i][q];
            U[i][p] = cs * u - sn * v;
            U[i][q] = sn * u + cs * v;
          }
          __syncthreads();
        }
        double* Ug = Ubuf + static_cast<int64_t>(pi) * kSymB * kSymB;
        for (int e = tid; e < kSymB * kSymB; e += 256) Ug[e] = U[e % kSymB][e / kSymB];
        if (tid == 0) {
          flags[pi] = nrot > 0;
          if (nrot) atomicAdd(&counters[sweep], nrot);
        }
        __syncthreads();
      }
      grid.sync();
      // ---------------- phase B: apply the rotations to H tiles and V column blocks
      const int ntri = npairs * (npairs + 1) / 2;
      const int nvt = npairs * ((n + kSymB - 1) / kSymB);
      for (int w = blockIdx.x; w < ntri + nvt; w += gridDim.x) {
        if (w < ntri) {
          int I = 0, rem = w;
          while (rem >= npairs - I) { rem -= npairs - I; ++I; }
          const int K = I + rem;
          const bool fi = flags[I] != 0, fk = flags[K] != 0;
          if (!fi && !fk) continue;
          int PI, QI, PK, QK;
          sym_pair(k, I, m1, PI, QI);
          sym_pair(k, K, m1, PK, QK);
          const double* UI = Ubuf + static_cast<int64_t>(I) * kSymB * kSymB;
          const double* UK = Ubuf + static_cast<int64_t>(K) * kSymB * kSymB;
          for (int e = tid; e < kSymB * kSymB; e += 256) {
            const int i = e % kSymB, j = e / kSymB;
            const int gi = sym_idx(PI, QI, i), gj = sym_idx(PK, QK, j);
            T[i][j] = (gi < n && gj < n) ? H[gi + static_cast<int64_t>(gj) * n] : 0.0;
            S[i][j] = UI[e];           // S = U_I (i, j) col-major source
            U[i][j] = UK[e];
          }
          __syncthreads();
          // R = T U_K  (kept in registers: each thread 4 entries)
          double r4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int e = tid + 256 * c;
            const int i = e % kSymB, j = e / kSymB;
            double acc = 0.0;
#pragma unroll 8
            for (int l = 0; l < kSymB; ++l) acc = fma(T[i][l], U[l][j], acc);
            r4[c] = acc;
          }
          __syncthreads();
#pragma unroll
          for (int c = 0; c < 4; ++c) { const int e = tid + 256 * c; T[e % kSymB][e / kSymB] = r4[c]; }
          __syncthreads();
          // out = U_I^T R
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int e = tid + 256 * c;
            const int i = e % kSymB, j = e / kSymB;
            double acc = 0.0;
#pragma unroll 8
            for (int l = 0; l < kSymB; ++l) acc = fma(S[l][i], T[l][j], acc);
            const int gi = sym_idx(PI, QI, i), gj = sym_idx(PK, QK, j);
            if (gi < n && gj < n) {
              H[gi + static_cast<int64_t>(gj) * n] = acc;
              if (I != K) H[gj + static_cast<int64_t>(gi) * n] = acc;
            }
          }
          __syncthreads();
        } else {
          const int v = w - ntri;
          const int I = v % npairs, rc = v / npairs;
          if (!flags[I]) continue;
          int PI, QI;
          sym_pair(k, I, m1, PI, QI);
          const double* UI = Ubuf + static_cast<int64_t>(I) * kSymB * kSymB;
          const int r0 = rc * kSymB;
          for (int e = tid; e < kSymB * kSymB; e += 256) {
            const int i = e % kSymB, j = e / kSymB;
            const int gj = sym_idx(PI, QI, j);
            T[i][j] = (r0 + i < n && gj < n) ? V[(r0 + i) + static_cast<int64_t>(gj) * n] : 0.0;
            U[i][j] = UI[e];
          }
          __syncthreads();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int e = tid + 256 * c;
            const int i = e % kSymB, j = e / kSymB;
            double acc = 0.0;
#pragma unroll 8
            for (int l = 0; l < kSymB; ++l) acc = fma(T[i][l], U[l][j], acc);
            const int gj = sym_idx(PI, QI, j);
            if (r0 + i < n && gj < n) V[(r0 + i) + static_cast<int64_t>(gj) * n] = acc;
          }
          __syncthreads();
        }
      }
      grid.sync();
    }
    const int rotated = atomicAdd(&counters[sweep], 0);
    if (rotated == 0) break;
  }
}

// d[i] = H(i, i)
__global__ void diag_kernel(const double* __restrict__ H, int n, double* __restrict__ d, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = H[i + static_cast<int64_t>(i) * n];
}

// abs_tol = c * ||A||_F (fixed order, one CTA)
__global__ void frob_scale_kernel(const double* __restrict__ A, int64_t len, double c, double* __restrict__ out,
                                  const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s = fma(A[i], A[i], s);
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = c * sqrt(s);
}

// One-sided (Hestenes) Jacobi SVD of a small L x n matrix B (col-major) in ONE CTA with B and V
// resident in shared memory (no grid barriers): round-robin parallel ordering, kSvdG lanes per
// column pair (two pairs per warp, so every pair of a round runs at once), shuffle dot
// products, the same rotation rule and stopping test as bjacobi_kernel.
// On exit B <- B V (orthogonal columns), V (n x n), sig = column norms.  Dynamic smem: (L + n) n.
constexpr int kSvdG = 16;
__global__ void __launch_bounds__(1024) small_svd_kernel(double* __restrict__ Bg, int L, int n, double* __restrict__ Vg,
                                                        double* __restrict__ sig, int* __restrict__ counters,
                                                        int max_sweeps, double tol, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double ss_smem[];
  double* B = ss_smem;            // [n][L]
  double* V = ss_smem + static_cast<int64_t>(L) * n;   // [n][n]
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int sub = lane / kSvdG, gl = lane % kSvdG;
  constexpr int ppw = 32 / kSvdG;
  double f2 = 0.0;
  for (int e = tid; e < L * n; e += blockDim.x) { const double x = Bg[e]; B[e] = x; f2 = fma(x, x, f2); }
  for (int e = tid; e < n * n; e += blockDim.x) V[e] = (e % n == e / n) ? 1.0 : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, o);
  if (lane == 0) red[warp] = f2;
  __syncthreads();
  double fro2 = 0.0;
  for (int w = 0; w < nw; ++w) fro2 += red[w];
  const double floor2 = 1e-28 * fro2;
  const double tol2 = tol * tol;
  const int nn = n + (n & 1), np = nn / 2, m1 = nn - 1;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int k = 0; k < max(m1, 1); ++k) {
      for (int base = warp * ppw; base < np; base += nw * ppw) {    // warp-uniform
        const int pi = base + sub;
        int a, b;
        if (m1 == 0) { a = 0; b = 1; }
        else if (pi == 0) { a = m1; b = k; }
        else {
          a = k + pi; if (a >= m1) a -= m1;
          b = k - pi; if (b < 0) b += m1;
        }
        const int p = min(a, b), q = max(a, b);
        const bool act = pi < np && q < n;
        double* bp = B + static_cast<int64_t>(p) * L;
        double* bq = B + static_cast<int64_t>(q) * L;
        double al = 0.0, be = 0.0, ga = 0.0;
        if (act) {
          for (int i = gl; i < L; i += kSvdG) {
            const double x = bp[i], y = bq[i];
            al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
          }
        }
#pragma unroll
        for (int o = kSvdG / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (act && ga != 0.0 && ga * ga > tol2 * (al * be) && fmin(al, be) > floor2) {
          // rotation parameters from the reciprocal square root (rsqrt + Newton), one division
          const double zeta = (be - al) / (2.0 * ga);
          double t;
          if (fabs(zeta) > 1e150) t = 0.5 / zeta;
          else {
            const double z2 = fma(zeta, zeta, 1.0);
            double r = rsqrt(z2);
            r = r * fma(-0.5 * z2, r * r, 1.5);
            t = copysign(1.0, zeta) / fma(z2, r, fabs(zeta));        // 1 / (|zeta| + sqrt(1 + zeta^2))
          }
          const double u = fma(t, t, 1.0);
          double cs = rsqrt(u);
          cs = cs * fma(-0.5 * u, cs * cs, 1.5);
          const double sn = cs * t;
          for (int i = gl; i < L; i += kSvdG) {
            const double x = bp[i], y = bq[i];
            bp[i] = cs * x - sn * y;
            bq[i] = sn * x + cs * y;
          }
          double* vp = V + static_cast<int64_t>(p) * n;
          double* vq = V + static_cast<int64_t>(q) * n;
          for (int i = gl; i < n; i += kSvdG) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    const int any = __syncthreads_or(rotated);
    if (tid == 0) counters[sweep] = any;
    if (!any) break;
  }
  for (int e = tid; e < L * n; e += blockDim.x) Bg[e] = B[e];
  for (int e = tid; e < n * n; e += blockDim.x) Vg[e] = V[e];
  for (int c = warp; c < n; c += nw) {
    double s2 = 0.0;
    for (int i = lane; i < L; i += 32) { const double x = B[static_cast<int64_t>(c) * L + i]; s2 = fma(x, x, s2); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) sig[c] = sqrt(s2);
  }
}

// out (n x m) = A^T for A (m x n), both col-major
__global__ void transpose_kernel(const double* __restrict__ A, int m, int n, double* __restrict__ out,
                                 const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(m) * n) return;
  const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
  out[j + static_cast<int64_t>(i) * n] = A[idx];
}

// col_norm[i] = ||B(:, i)||_2 (fixed order), one CTA per column.
__global__ void col_norms_kernel(const double* __restrict__ B, int L, int n, double* __restrict__ out,
                                 const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[8];
  const int i = blockIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = threadIdx.x; r < L; r += blockDim.x) { const double v = B[static_cast<int64_t>(i) * L + r]; s = fma(v, v, s); }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[i] = sqrt(s);
}

__global__ void set_identity_kernel(double* __restrict__ V, int n, const int* __restrict__ gate = nullptr) {
  if (gate && *gate == 0) return;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < static_cast<int64_t>(n) * n) V[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
}

// Z(i, r) = w_i * B(r, i) with w_i = 1/sigma_i^2 if sigma_i > rcond * max sigma else 0
// (pseudo-inverse assembly pinv = V Z, reading R9).  Z is n x L.  One CTA.
__global__ void pinv_weights_kernel(const double* __restrict__ sig, int n, double rcond, double* __restrict__ w,
                                    double* __restrict__ kappa_out, unsigned* __restrict__ flags, unsigned flagbit,
                                    const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[8];
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, sig[i]);
  mx = block_max<256>(mx, red);
  double mn = INFINITY;
  int cut = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double s = sig[i];
    const bool keep = mx > 0.0 && s > rcond * mx;
    w[i] = keep ? 1.0 / (s * s) : 0.0;
    if (keep) mn = fmin(mn, s); else if (s > 0.0) cut = 1;
  }
  mn = -block_max<256>(-mn, red);
  const double anycut = block_max<256>(static_cast<double>(cut), red);
  if (threadIdx.x == 0) {
    if (kappa_out) *kappa_out = (mx > 0.0) ? mx / mn : 1.0;
    if (flags && anycut > 0.0) atomicOr(flags, flagbit);
  }
}

__global__ void scale_transpose_kernel(const double* __restrict__ B, int L, int n, const double* __restrict__ w,
                                       double* __restrict__ Z, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(L) * n) return;
  const int i = static_cast<int>(idx % n), r = static_cast<int>(idx / n);   // Z(i, r), ld = n
  Z[idx] = w[i] * B[static_cast<int64_t>(i) * L + r];
}

// sum_{i < rows, j < cols} A(i, j) * B(i, j)  (fixed order), written to *out (one CTA).
__global__ void frob_dot_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                                int rows, int64_t cols, double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  const int64_t total = static_cast<int64_t>(rows) * cols;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t j = e / rows;
    const int i = static_cast<int>(e % rows);
    s = fma(A[i + j * lda], B[i + j * ldb], s);
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace oid
