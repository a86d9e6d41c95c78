// A9 exact basis Gram on the fp64 tensor cores, fed by TMA (sm_100a).
//
// Dpart[cta](q, j) = sum_{rows r of the CTA's chunk} C(r, d_q) C(r, j) for the dirty slots d_q
// (slots admitted since the last estimate) and every slot j.  The
// basis slab C (m_loc x t, column-major) is streamed once per group of 32 dirty slots.
//
// CTA = 1 producer warp + CW compute warps, one CTA per SM over a contiguous row chunk:
//   producer   cp.async.bulk.tensor 2D boxes {128 bytes of rows, <= 256 columns} with the
//              128-byte swizzle into an nstage-deep ring (full/empty mbarriers);
//   compute    warp w owns the 8-column blocks nb = w + CW i (i < 4): mma.sync m8n8k4 f64
//              (DMMA) with the 32 dirty slots as M (4 blocks of 8) and the rows as K.
// The K order is permuted so that each lane reads two consecutive rows (one 16-byte load per
// two DMMA k-steps) for both operands; the column order inside an 8-column block is permuted
// so that the lanes of one shared-memory phase hit distinct swizzled 16-byte chunks
// (conflict-free B loads).  The sum over rows is a dot product, so the order only changes
// rounding; per-CTA partials are reduced in a fixed order afterwards (deterministic).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "k1_tc.cuh"

namespace oid {
namespace bgtc {

constexpr int kMaxStages = 8;
constexpr int kNbw = 4;   // 8-column blocks per compute warp

// rows per 128-byte line, and the lane -> column permutation inside an 8-column block
template <typename T> struct Fmt;
template <> struct Fmt<double> {
  static constexpr int RL = 16;
  // a quarter-warp phase holds g4 in {2p, 2p+1}: their lines must differ in bit 2
  __device__ static int perm(int g) { return (g >> 1) | ((g & 1) << 2); }
};
template <> struct Fmt<float> {
  static constexpr int RL = 32;
  // a half-warp phase holds g4 in {0..3} or {4..7}: their lines must differ in bits 1-2
  __device__ static int perm(int g) { return ((g & 3) << 1) | (g >> 2); }
};

// two consecutive rows (k-pair u, lane quad i4) of line j of a stage, as fp64
template <typename T>
__device__ __forceinline__ double2 ld_pair(const uint8_t* stage, int j, int u, int i4);
template <>
__device__ __forceinline__ double2 ld_pair<double>(const uint8_t* stage, int j, int u, int i4) {
  const int jj = j & 255;
  const uint8_t* line = stage + (static_cast<size_t>(j >> 8) << 15) + (jj << 7);
  return *reinterpret_cast<const double2*>(line + ((((u << 2) | i4) ^ (jj & 7)) << 4));
}
template <>
__device__ __forceinline__ double2 ld_pair<float>(const uint8_t* stage, int j, int u, int i4) {
  const int jj = j & 255;
  const uint8_t* line = stage + (static_cast<size_t>(j >> 8) << 15) + (jj << 7);
  const float2 v = *reinterpret_cast<const float2*>(line + (((((u << 1) | (i4 >> 1)) ^ (jj & 7)) << 4) | ((i4 & 1) << 3)));
  return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  // not volatile: the compiler may interleave independent accumulators (DMMA latency)
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
    basis_gram_tc_kernel(const __grid_constant__ CUtensorMap map, int64_t m_loc, int t, int64_t rows_per_cta,
                         int nstage, int stage_bytes, int nbox, const int* __restrict__ list,
                         const int* __restrict__ counts, double* __restrict__ part) {
  using namespace k1tc;
  constexpr int RL = Fmt<T>::RL;
  constexpr int KP = RL / 8;   // k-pairs (two DMMA k-steps of 4 rows) per line
  extern __shared__ unsigned char bg_raw[];
  // 1024-byte aligned ring (128B swizzle atoms); pointer arithmetic keeps the shared space
  uint8_t* ring = bg_raw + ((1024u - (smem_u32(bg_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ int dl[32];
  const int nd = counts[2];
  if (nd == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g4 = lane >> 2, i4 = lane & 3;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(m_loc, r0 + rows_per_cta);
  const int ntile = r1 > r0 ? static_cast<int>((r1 - r0 + RL - 1) / RL) : 0;
  double* out = part + static_cast<int64_t>(blockIdx.x) * t * t;
  if (tid == 0) {
    for (int s = 0; s < nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int g = 0;   // tiles streamed by this CTA so far (ring position)
  for (int q0 = 0; q0 < nd; q0 += 32) {
    if (tid < 32) dl[tid] = (q0 + tid < nd) ? list[q0 + tid] : -1;
    __syncthreads();
    if (warp == CW) {
      // ---------------- producer
      if (lane == 0) {
        for (int it = 0; it < ntile; ++it) {
          const int gi = g + it, s = gi % nstage, use = gi / nstage;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
          mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nbox) * static_cast<uint32_t>(min(t, 256)) * 128u);
          const int row = static_cast<int>(r0 + static_cast<int64_t>(it) * RL);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(ring + static_cast<size_t>(s) * stage_bytes + (static_cast<size_t>(b) << 15), &map, &full[s], row,
                        256 * b);
        }
      }
    } else {
      // ---------------- compute
      const int ndg = min(32, nd - q0);
      const int MB = (ndg + 7) >> 3;
      int dcol[4];
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) dcol[mm] = dl[8 * mm + g4];
      int jcol[kNbw];
      bool jok[kNbw];
#pragma unroll
      for (int b = 0; b < kNbw; ++b) {
        jcol[b] = 8 * (warp + CW * b) + Fmt<T>::perm(g4);
        jok[b] = jcol[b] < t;
      }
      const int nbw = min(kNbw, max(0, ((t + 7) / 8 - warp + CW - 1) / CW));   // blocks this warp owns
      double acc[4][kNbw][2];
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
#pragma unroll
        for (int b = 0; b < kNbw; ++b) { acc[mm][b][0] = 0.0; acc[mm][b][1] = 0.0; }
      for (int it = 0; it < ntile; ++it) {
        const int gi = g + it, s = gi % nstage, use = gi / nstage;
        mbar_wait(&full[s], use & 1);
        const uint8_t* st = ring + static_cast<size_t>(s) * stage_bytes;
#pragma unroll
        for (int u = 0; u < KP; ++u) {
          double2 a[4];
#pragma unroll
          for (int mm = 0; mm < 4; ++mm)
            a[mm] = (mm < MB && dcol[mm] >= 0) ? ld_pair<T>(st, dcol[mm], u, i4) : make_double2(0.0, 0.0);
          double2 bv[kNbw];
#pragma unroll
          for (int b = 0; b < kNbw; ++b)
            bv[b] = (b < nbw && jok[b]) ? ld_pair<T>(st, jcol[b], u, i4) : make_double2(0.0, 0.0);
          // first k-step of the pair for every accumulator, then the second: consecutive DMMAs
          // never depend on each other
#pragma unroll
          for (int b = 0; b < kNbw; ++b) {
            if (b >= nbw) break;   // warp-uniform
#pragma unroll
            for (int mm = 0; mm < 4; ++mm)
              if (mm < MB) dmma(acc[mm][b], a[mm].x, bv[b].x);   // warp-uniform
          }
#pragma unroll
          for (int b = 0; b < kNbw; ++b) {
            if (b >= nbw) break;
#pragma unroll
            for (int mm = 0; mm < 4; ++mm)
              if (mm < MB) dmma(acc[mm][b], a[mm].y, bv[b].y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // D fragment: row g4 of m-block mm, columns 2 i4 + h of the 8-column block
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const int q = 8 * mm + g4;
        if (q >= ndg) continue;
#pragma unroll
        for (int b = 0; b < kNbw; ++b) {
          if (b >= nbw) break;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (warp + CW * b) + Fmt<T>::perm(2 * i4 + h);
            if (j < t) out[(q0 + q) + static_cast<int64_t>(j) * t] = acc[mm][b][h];
          }
        }
      }
    }
    g += ntile;
    __syncthreads();
  }
}

}  // namespace bgtc
}  // namespace oid
