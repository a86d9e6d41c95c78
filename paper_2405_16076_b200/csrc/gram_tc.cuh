// A9 exact basis Gram on the fp64 tensor cores, fed by TMA (sm_100a).
//
// Dpart[cta](q, j) = sum_{rows r of the CTA's chunk} C(r, d_q) C(r, j) for the dirty slots d_q
// (slots admitted since the last estimate) and every slot j.
//
// Basis layout: row-tiled, C_blk[tile][slot][RL] with RL = 128 bytes of
// rows (16 fp64 / 32 fp32), so one tile of all t slots is one contiguous t x 128-byte block:
// the producer streams it with one 3-D TMA box {RL, t, 1} (128-byte swizzle), i.e. purely
// sequential HBM reads.  The basis copy (A7) writes this layout; oid_finalize un-tiles it.
//
// CTA = 1 producer warp + kCW compute warps, many short CTAs (each a contiguous run of tiles),
// so kernels of higher-priority streams are scheduled as CTAs retire:
//   producer   cp.async.bulk.tensor 3D, nstage-deep ring (full/empty mbarriers);
//   compute    warp = one m-block of D (8 dirty slots) x a contiguous range of n-blocks (8 slots
//              each), balanced over the 4 SM sub-partitions; mma.sync m8n8k4 f64 (DMMA) with the
//              basis rows as K.
// The K order is permuted so that each lane reads two consecutive rows (one 16-byte load per
// two DMMA k-steps) for both operands; the column order inside an 8-column block is permuted
// so that the lanes of one shared-memory phase hit distinct swizzled 16-byte chunks
// (conflict-free B loads).  The sum over rows is a dot product, so the order only changes
// rounding; per-CTA partials are reduced in a fixed order afterwards (deterministic).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"

namespace oid {
namespace bgtc {

constexpr int kMaxStages = 8;
constexpr int kCW = 8;        // compute warps
constexpr int kTpw = 16;      // max (m, n) tiles per compute warp: 4 m-blocks x 32 n-blocks / 8 (t <= 256);
                              // for t > 256 the dirty slots go in groups of 16 (2 m-blocks x 52 / 8 <= 13)

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
  // box b (slots 256 b ..) sits at 32 KB b, i.e. line j is at 128 j either way
  const uint8_t* line = stage + (j << 7);
  return *reinterpret_cast<const double2*>(line + ((((u << 2) | i4) ^ (j & 7)) << 4));
}
template <>
__device__ __forceinline__ double2 ld_pair<float>(const uint8_t* stage, int j, int u, int i4) {
  const uint8_t* line = stage + (j << 7);
  const float2 v = *reinterpret_cast<const float2*>(line + (((((u << 1) | (i4 >> 1)) ^ (j & 7)) << 4) | ((i4 & 1) << 3)));
  return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}

// not volatile: the compiler may interleave independent accumulators (DMMA latency)
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          k1tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(k1tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <typename T>
__global__ void __maxnreg__(224)
    basis_gram_tc_kernel(const __grid_constant__ CUtensorMap map, int64_t ntiles_total, int t, int64_t tiles_per_cta,
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
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * tiles_per_cta;
  const int64_t tile1 = ntiles_total < tile0 + tiles_per_cta ? ntiles_total : tile0 + tiles_per_cta;
  const int ntile = tile1 > tile0 ? static_cast<int>(tile1 - tile0) : 0;
  double* out = part + static_cast<int64_t>(blockIdx.x) * t * t;
  if (tid == 0) {
    for (int s = 0; s < nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t tx_bytes = static_cast<uint32_t>(nbox) * static_cast<uint32_t>(min(t, 256)) * 128u;
  const int NB = (t + 7) >> 3;                 // n-blocks of 8 slots
  // ring position carried across dirty groups: stage s_pos, phase bit ph
  int s_pos = 0;
  uint32_t ph = 0;
  const int gsz = t <= 256 ? 32 : 16;          // dirty slots per pass over the chunk
  for (int q0 = 0; q0 < nd; q0 += gsz) {
    if (tid < 32) dl[tid] = (tid < gsz && q0 + tid < nd) ? list[q0 + tid] : -1;
    __syncthreads();
    if (warp == kCW) {
      // ---------------- producer
      if (lane == 0) {
        int s = s_pos;
        uint32_t p = ph;
        for (int it = 0; it < ntile; ++it) {
          mbar_wait(&empty[s], p ^ 1u);          // first pass: fresh barrier, parity 1 completes at once
          mbar_arrive_expect_tx(&full[s], tx_bytes);
          const int tile = static_cast<int>(tile0 + it);
          for (int b = 0; b < nbox; ++b)
            tma_load_3d(ring + static_cast<size_t>(s) * stage_bytes + (static_cast<size_t>(b) << 15), &map, &full[s], 0,
                        256 * b, tile);
          if (++s == nstage) { s = 0; p ^= 1u; }
        }
      }
    } else {
      // ---------------- compute: warp -> one m-block (8 dirty slots) x a contiguous n-block range
      // (m-blocks padded to 1, 2 or 4 so that the kCW warps split evenly: every SM sub-partition
      // gets the same DMMA work; padded m-blocks multiply zeros)
      const int ndg = min(gsz, nd - q0);
      const int MB = (ndg + 7) >> 3;
      const int MBp = MB <= 1 ? 1 : (MB <= 2 ? 2 : 4);
      const int wpm = kCW / MBp;                       // warps per m-block
      const int mb = warp / wpm, part = warp - mb * wpm;
      const int nb_b = (part * NB) / wpm, nb_e = ((part + 1) * NB) / wpm;
      const int nt = nb_e - nb_b;                      // <= kTpw
      // rows of padded / absent dirty slots read line 0 (finite data, their D rows are dropped);
      // B lines j >= t (at most 7 past the box, inside the 1024-byte rounded stage) only feed D
      // columns that are never stored
      const int dA = mb < MB ? max(0, dl[8 * mb + g4]) : 0;
      const int jc0 = 8 * nb_b + Fmt<T>::perm(g4);
      double acc[kTpw][2];
#pragma unroll
      for (int i = 0; i < kTpw; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
      int s = s_pos;
      uint32_t p = ph;
      for (int it = 0; it < ntile; ++it) {
        mbar_wait(&full[s], p);
        const uint8_t* st = ring + static_cast<size_t>(s) * stage_bytes;
#pragma unroll
        for (int u = 0; u < KP; ++u) {
          const double2 a = ld_pair<T>(st, dA, u, i4);
#pragma unroll
          for (int h = 0; h < kTpw; h += 8) {
            if (h >= nt) break;                        // warp-uniform
            double2 bv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)   // warp-uniform guard: never read past this warp's n-blocks
              bv[k] = h + k < nt ? ld_pair<T>(st, jc0 + 8 * (h + k), u, i4) : make_double2(0.0, 0.0);
            // first k-step of the pair for these accumulators, then the second: consecutive DMMAs
            // never depend on each other
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (h + k < nt) dmma(acc[h + k], a.x, bv[k].x);   // warp-uniform predicates
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (h + k < nt) dmma(acc[h + k], a.y, bv[k].y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == nstage) { s = 0; p ^= 1u; }
      }
      // D fragment: row g4 of the m-block, columns 2 i4 + h of each n-block
      const int q = 8 * mb + g4;
      if (q < ndg) {
#pragma unroll
        for (int i = 0; i < kTpw; ++i) {
          if (i >= nt) break;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jj = 8 * (nb_b + i) + Fmt<T>::perm(2 * i4 + h);
            if (jj < t) out[(q0 + q) + static_cast<int64_t>(jj) * t] = acc[i][h];
          }
        }
      }
    }
    // advance the ring position by ntile for the next dirty group
    {
      const int adv = s_pos + ntile;
      ph ^= static_cast<uint32_t>((adv / nstage) & 1);
      s_pos = adv % nstage;
    }
    __syncthreads();
  }
}

}  // namespace bgtc
}  // namespace oid
