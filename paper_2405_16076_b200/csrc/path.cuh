// Post-pass kernels specific to Algorithm 3: ridge regulariser, ridge scores, selection,
// basis copy, S_J gather, NA-Hutch++ final combination.
#pragma once
#include "common.cuh"

namespace oid {

// scalars layout (device double array)
enum Scal : int {
  SC_FROB2 = 0, SC_LAM = 1, SC_EK = 2, SC_SHIFT = 3, SC_TRACE = 4, SC_DMAX = 5, SC_MINMARGIN = 6, SC_KAPPA = 7,
  SC_T1 = 8, SC_T3A = 9, SC_T3B = 10, SC_GPP = 11, SC_FROB2_EST = 12, SC_KAPPA_EST = 13,
  SC_FROB2_SNAP = 16,   // + epoch parity: ||A_obs||^2 snapshot taken at the end of a commit
  SC_KAPPA_SNAP = 18,   // + epoch parity: kappa(S_J) of that epoch's Alg 4 chain
  SC_FROB2_AUG = 20,    // gradient variant: ||A_obs||^2 + sum_p ||G^p A_obs||^2 (A11(2))
  SC_GCV = 21,          // gradient variant: last sketched GCV value
  SC_COUNT = 24
};

// Ridge regulariser (reading R8): eigenvalues mu of the unscaled Gram, E_k = sum of the k
// largest (descending order), lambda per mode, shift = ell * lambda (reading R3),
// dmax = max(mu) + shift.  One CTA (n <= 1024): rank sort, then sequential sums.
__global__ void lambda_kernel(const double* __restrict__ mu, int n, int k, const double* __restrict__ gram,
                              double lam_param, int ell, double* __restrict__ scal, double* __restrict__ sorted,
                              int frob_idx) {
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
    for (int i = 0; i < n; ++i) tr += gram[static_cast<int64_t>(i) * n + i];   // Gram order n (3 ell with gradients)
    const double frob2 = scal[frob_idx];
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

constexpr int kSelMaxT = 416;   // validated maximum of k
constexpr int kSelH = 14;       // candidate chunks of 32 per selection (448 >= max(b_max, k))

// Alg 3 steps 15-27, readings R4-R7, R14.  The t evictions are independent (one
// thread per slot); the vacant slots are then filled in slot order (sequential by nature: slot
// i+1 sees the candidates consumed by slot i), each by one warp testing its candidates at once
// (the first success in candidate order is the sequential scan's admission).
// tau: [t slot scores | nc candidate scores]; nrm: candidate norms (zero columns skipped).
// Outputs: admit list (slot, r) pairs, count; zero list (slots vacated, not refilled).
__global__ void __launch_bounds__(256) select_kernel(int64_t* __restrict__ J, double* __restrict__ tau_old,
                                                      const double* __restrict__ tau, const double* __restrict__ nrm, int t,
                                                      int nc, double factor, uint32_t epoch, int64_t base, uint32_t key0,
                                                      uint32_t key1, int* __restrict__ admit, int* __restrict__ counts,
                                                      double* __restrict__ scal, int* __restrict__ dirty, int dtag,
                                                      unsigned long long* __restrict__ cum, double* __restrict__ elog) {
  // The decisions are sequential only through the candidates consumed by earlier slots: the
  // eviction of slot i depends on slot i alone (steps 16-19), so
  //   (1) the evictions are decided in parallel, one thread per slot;
  //   (2) one warp walks the vacant slots in order; for each, the lanes draw and test the
  //       candidates r = lane, lane + 32 at once and the first success in index order is the
  //       admission (the same as the sequential scan: candidates before it fail, later draws
  //       are never looked at).
  // The R14 margin is the min over exactly the draws the sequential scan evaluates.  Small
  // footprint (256 threads, no dynamic shared memory) so the kernel fits beside the Gram CTAs.
  __shared__ unsigned char s_vac[kSelMaxT], s_ev[kSelMaxT];
  __shared__ double s_red[32];
  double mm = INFINITY;
  for (int i = threadIdx.x; i < t; i += blockDim.x) {
    bool vac = J[i] < 0, ev = false;
    if (!vac) {
      const double told = tau_old[i];
      const double ti = fmin(told, tau[i]);
      const double rho = told > 0.0 ? ti / told : 1.0;
      const double pev = 1.0 - rho;
      const double u = select_uniform(epoch, static_cast<uint32_t>(i), 0xFFFFFFFFu, key0, key1);
      mm = fmin(mm, fabs(u - pev) / fmax(rho, 0x1p-24));
      if (u < pev) { J[i] = -1; tau_old[i] = 1.0; vac = ev = true; }
      else tau_old[i] = ti;
    }
    s_vac[i] = vac;
    s_ev[i] = ev;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    // candidate r = lane + 32 h (h < kSelH: up to 448 candidates - a block of b_max <= 64, or
    // the t buffered columns of a paper-literal epoch); fp64 probabilities
    double praw[kSelH], pr[kSelH];
    bool ok[kSelH];
#pragma unroll
    for (int h = 0; h < kSelH; ++h) {
      const int r = lane + 32 * h;
      ok[h] = r < nc && nrm[r] != 0.0;
      praw[h] = r < nc ? tau[t + r] * factor : 0.0;
      pr[h] = fmin(1.0, praw[h]);
    }
    const int nh = (nc + 31) >> 5;
    int na = 0, nz = 0;
    for (int i0 = 0; i0 < t; i0 += 32) {
      uint32_t vm = __ballot_sync(0xffffffffu, i0 + lane < t && s_vac[i0 + lane]);
      while (vm) {
        const int i = i0 + __ffs(vm) - 1;
        vm &= vm - 1;
        // first success in candidate order: chunks of 32 in order, the lowest hit of the first
        // chunk that has one (the sequential scan's admission); draws past it are not evaluated
        int rs = kSelH * 32;   // no admission
#pragma unroll
        for (int h = 0; h < kSelH; ++h) {
          if (h >= nh) break;
          const double u = ok[h] ? select_uniform(epoch, static_cast<uint32_t>(i), static_cast<uint32_t>(lane + 32 * h),
                                                  key0, key1)
                                 : 1.0;
          const bool hit = ok[h] && u < pr[h];
          const uint32_t bh = __ballot_sync(0xffffffffu, hit);
          const int rh = bh ? 32 * h + __ffs(bh) - 1 : kSelH * 32;
          if (ok[h] && lane + 32 * h <= rh) mm = fmin(mm, fabs(u - praw[h]) / fmax(praw[h], 0x1p-24));
          if (bh) { rs = rh; break; }
        }
        if (rs < kSelH * 32) {
          if (lane == 0) {
            J[i] = base + rs;
            tau_old[i] = tau[t + rs];
            admit[2 * na] = i;
            admit[2 * na + 1] = rs;
            dirty[i] = dtag;   // epoch tag of the admission (estimates pick tags newer than theirs)
          }
#pragma unroll
          for (int h = 0; h < kSelH; ++h)
            if (lane == (rs & 31) && h == (rs >> 5)) ok[h] = false;   // consumed
          ++na;
        } else if (s_ev[i]) {
          if (lane == 0) admit[2 * (nc + t) - 2 - 2 * nz] = i;
          ++nz;
        }
      }
    }
    if (lane == 0) { counts[0] = na; counts[1] = nz; }
    if (lane == 0 && cum) cum[0] += static_cast<unsigned long long>(na);
  }
  // per-epoch report row (A12): evictions (slots vacated this epoch, refilled or not)
  {
    int ne = 0;
    for (int i = threadIdx.x; i < t; i += blockDim.x) ne += s_ev[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
    __shared__ int s_ne[8];
    if ((threadIdx.x & 31) == 0) s_ne[threadIdx.x >> 5] = ne;
    __syncthreads();
    if (threadIdx.x == 0 && elog) {
      int tot = 0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) tot += s_ne[q];
      elog[0] = static_cast<double>(epoch);
      elog[1] = static_cast<double>(base + nc);
      elog[2] = static_cast<double>(counts[0]);
      elog[3] = static_cast<double>(tot);
      elog[4] = scal[SC_LAM];
      elog[5] = scal[SC_EK];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mm = fmin(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double me = INFINITY;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) me = fmin(me, s_red[q]);
    scal[SC_MINMARGIN] = fmin(scal[SC_MINMARGIN], me);
    if (elog) elog[6] = me;
  }
}

// C(:, slot) <- X(:, r) for admissions, C(:, slot) <- 0 for vacated slots.
// A7: basis slab C(:, slot) <- X(:, r) bit-exactly for every admission and C(:, slot) <- 0
// for vacated slots, in the row-tiled layout C_blk[tile][slot][RL] (RL = 128 bytes of rows;
// DESIGN.md section 6) that A9 streams with one TMA box per tile.  Each column is spread over
// the whole (small, persistent) grid, so the kernel never floods the block scheduler.
template <typename T>
__global__ void basis_copy_kernel(const T* __restrict__ X, int64_t ld, T* __restrict__ Cb, int64_t m_loc,
                                  const int* __restrict__ admit, const int* __restrict__ counts, int nc, int t) {
  constexpr int RL = 128 / sizeof(T);
  constexpr int V = 16 / sizeof(T);
  const int na = counts[0], nz = counts[1];
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = (m_loc % V == 0) && (ld % V == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  for (int a = 0; a < na + nz; ++a) {
    int slot, r = -1;
    if (a < na) { slot = admit[2 * a]; r = admit[2 * a + 1]; }
    else slot = admit[2 * (nc + t) - 2 - 2 * (a - na)];
    const T* src = r >= 0 ? X + static_cast<int64_t>(r) * ld : nullptr;
    if (vec) {
      // four independent 16-byte loads in flight per thread before their stores
      constexpr int U = 4;
      const int64_t nv = m_loc / V;
      int64_t v = tid;
      for (; v + (U - 1) * stride < nv; v += U * stride) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          x[u] = src ? __ldcs(reinterpret_cast<const uint4*>(src + (v + u * stride) * V)) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = (v + u * stride) * V;
          __stcs(reinterpret_cast<uint4*>(Cb + ((i / RL) * t + slot) * RL + (i % RL)), x[u]);
        }
      }
      for (; v < nv; v += stride) {
        const int64_t i = v * V;
        const uint4 x = src ? __ldcs(reinterpret_cast<const uint4*>(src + i)) : make_uint4(0u, 0u, 0u, 0u);
        __stcs(reinterpret_cast<uint4*>(Cb + ((i / RL) * t + slot) * RL + (i % RL)), x);
      }
    } else {
      for (int64_t i = tid; i < m_loc; i += stride) Cb[((i / RL) * t + slot) * RL + (i % RL)] = src ? src[i] : T(0);
    }
  }
}

// out (m_loc x t, column-major) <- the row-tiled basis C_blk (oid_finalize)
template <typename T>
__global__ void basis_untile_kernel(const T* __restrict__ Cb, int64_t m_loc, int t, T* __restrict__ out) {
  constexpr int RL = 128 / sizeof(T);
  const int64_t n = m_loc * t;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int slot = static_cast<int>(e / m_loc);
    const int64_t i = e - static_cast<int64_t>(slot) * m_loc;
    out[e] = Cb[((i / RL) * t + slot) * RL + (i % RL)];
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
  const double frob2 = scal[SC_FROB2_EST];    // ||A_obs||^2 of the estimated state (snapshot)
  const double e2 = frob2 - 2.0 * T + gpp;
  unsigned f = *flags;
  if (e2 < 0.0) f |= 4u;
  const double est = sqrt(fmax(e2, 0.0));
  out[0] = e2; out[1] = T; out[2] = gpp; out[3] = frob2; out[4] = est;
  out[5] = frob2 > 0.0 ? est / sqrt(frob2) : 0.0;
  out[6] = static_cast<double>(f);
  out[7] = scal[SC_KAPPA_EST];
}

// End-of-commit snapshot (epoch parity par) for an estimate that may overlap the next commit:
// J, the admission tags, ||A_obs||^2.
__global__ void commit_snapshot_kernel(const int64_t* __restrict__ J, const int* __restrict__ dirty, int t,
                                       int64_t* __restrict__ Jsnap, int* __restrict__ Dsnap, double* __restrict__ scal,
                                       int par) {
  for (int i = threadIdx.x; i < t; i += blockDim.x) { Jsnap[i] = J[i]; Dsnap[i] = dirty[i]; }
  if (threadIdx.x == 0) scal[SC_FROB2_SNAP + par] = scal[SC_FROB2];
}

// Scalars of the estimated epoch (parity par) for hutch_final_kernel: ||A_obs||^2 of the
// snapshot (protected by ev_snap_free until the estimate ends) ...
__global__ void est_scalars_kernel(double* __restrict__ scal, int par) {
  scal[SC_FROB2_EST] = scal[SC_FROB2_SNAP + par];
}
// ... and kappa(S_J) of that epoch's Alg 4, taken in estimate_begin BEFORE ev_sj_free releases the
// parity: the A8 chain of the commit two epochs later rewrites SC_KAPPA_SNAP + par after that event
__global__ void est_kappa_kernel(double* __restrict__ scal, int par) {
  scal[SC_KAPPA_EST] = scal[SC_KAPPA_SNAP + par];
}

// Slots admitted after the last estimate (admission tags > last_tag), compacted in slot order;
// counts[2] = number of such (dirty) slots.  Tags are never cleared (no race with the next commit).
__global__ void dirty_compact_kernel(const int* __restrict__ dtag, int t, int last_tag, int* __restrict__ list,
                                     int* __restrict__ counts, unsigned long long* __restrict__ cum) {
  if (threadIdx.x != 0) return;
  int c = 0;
  for (int i = 0; i < t; ++i)
    if (dtag[i] > last_tag) list[c++] = i;
  counts[2] = c;
  if (cum) { cum[1] += static_cast<unsigned long long>(c); cum[2] += 1ull; }
}

// per-estimate report row (A12): [epoch, e2, T, gpp, frob2, est_rel, flags, kappa] from est[8] =
// [e2, T, gpp, frob2, est_abs, est_rel, flags, kappa]
__global__ void est_log_kernel(const double* __restrict__ est, double epoch, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    dst[0] = epoch;
    dst[1] = est[0]; dst[2] = est[1]; dst[3] = est[2]; dst[4] = est[3];
    dst[5] = est[5]; dst[6] = est[6]; dst[7] = est[7];
  }
}

// copies a scalar of the state into a report row (the kappa of an epoch's S_J, once A8 has run)
__global__ void log_scalar_kernel(const double* __restrict__ src, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *dst = *src;
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

// Two-level fixed-order sum of the per-chunk A9 partials over the dirty rows q < counts[2]:
// pass 1 (grid.y = nseg segments of the chunk range) writes seg[y](q, j); pass 2 (nseg = 1 view)
// sums the segments into out(q, j).  Layout of every partial: t x t column-major.
__global__ void sum_dirty_chunks_kernel(const double* __restrict__ part, int nchunks, int t, const int* __restrict__ counts,
                                        double* __restrict__ out) {
  const int nd = counts[2];
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(nd) * t) return;
  const int q = static_cast<int>(idx % nd), j = static_cast<int>(idx / nd);
  const int64_t e = q + static_cast<int64_t>(j) * t;
  const int64_t n = static_cast<int64_t>(t) * t;
  const int per = (nchunks + gridDim.y - 1) / gridDim.y;
  const int c0 = blockIdx.y * per, c1 = min(nchunks, c0 + per);
  double s = 0.0;
  for (int c = c0; c < c1; ++c) s += part[static_cast<int64_t>(c) * n + e];
  out[static_cast<int64_t>(blockIdx.y) * n + e] = s;
}

// gate[0] = a, gate[1] = b
__global__ void set_flag_kernel(int* __restrict__ gate, int a, int b) {
  gate[0] = a;
  gate[1] = b;
}

}  // namespace oid
