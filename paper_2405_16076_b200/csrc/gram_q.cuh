// A9Q: the basis Gram G(q, j) = A_J(:, d_q)^T A_J(:, j) for the dirty slots d_q on the
// int8 tensor cores, from a quantised copy of the basis written by A7 (K1F mode, k1_mode = 4).
//
// Quantised basis: every basis column is held a second time as four signed
// base-256 digit planes of v = round(x 2^F_s), |v| <= 2^30 (F_s per slot and shard, from the column's
// maximum exponent that K1F observed for the block the column came from), i.e. |x - x_q| <= 2^-28
// max|x|.  Layout: row tiles of 128 data rows; per tile one block of 4 t "rows" (row 4 s + p =
// plane p of slot s) x 128 bytes in 128-byte-swizzled K-major atoms (8 rows x 128 B, 16-byte chunk c
// of row r at ((c ^ (r & 7)) << 4)), so a tile of a slot chunk is one contiguous bulk copy and feeds
// tcgen05.mma directly as the B operand.  4 bytes per element: half the fp64 basis read.
//
// G(q, j) 2^(F_q + F_j) = sum_{p, p'} 256^(p + p') sum_rows d_p(row, d_q) d_p'(row, j): one int8 MMA
// D[(q, p), (j, p')] (M = 4 x 32 dirty slots, N = 4 x up to 128 slots, K = 128 rows per tile) with
// int32 accumulation (exact for <= 1024 tiles; then the accumulators are drained to fp64), combined
// in fp64 at the drain.  Output: the per-CTA partials part[cta][q + j t] of the fp64 A9
// (basis_gram_tc_kernel), reduced by the same fixed-order kernels.
//
// CTA (one per SM, 8 warps): warp 0 bulk-copy producer (B: one copy per tile), warp 1 TMEM allocator
// + MMA issuer, warps 4-7 gather the dirty slots' rows of the tile into the A stage (LDG from the
// quantised basis, re-swizzled) and drain TMEM (lane quarter = warp % 4).  CTA = (row-tile set,
// slot chunk of <= 128 slots); tiles dealt round-robin.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"

namespace oid {
namespace a9q {

using k1tc::smem_u32;

constexpr int kTR = 128;          // data rows per tile (K)
constexpr int kTc = 128;          // slots per chunk (N = 4 kTc = 512 TMEM columns)
constexpr int kNSB = 3;           // B stages (<= 4 kTc x 128 B = 64 KB)
constexpr int kNSA = 2;           // A stages (128 rows x 128 B = 16 KB)
constexpr int kThreads = 256;
constexpr int kEpochTiles = 1024; // int32 bound: 1024 x 128 rows x 128 x 128 = 2^31
constexpr int kGather0 = 4;       // first gather / drain warp

__host__ __device__ inline int64_t block_bytes(int t) { return static_cast<int64_t>((4 * t + 7) / 8) * 1024; }
__host__ __device__ inline int nchunks(int t) { return (t + kTc - 1) / kTc; }
// quantised-basis bytes for m_loc rows (+ one chunk of slack: the last chunk's copy may run past)
inline size_t qbasis_bytes(int64_t m_loc, int t) {
  const int64_t ntiles = (m_loc + kTR - 1) / kTR;
  return static_cast<size_t>(ntiles) * block_bytes(t) + 65536;
}
inline size_t smem_bytes() { return 1024 + kNSB * 65536 + kNSA * 16384; }

// UMMA shared-memory descriptor, K-major, 128-byte swizzle (SBO = 1024: 8-row atoms)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
  d |= static_cast<uint64_t>(1) << 46;                 // version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t swz(int r, int c) {   // byte offset of chunk c of row r in a block
  return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

#define A9Q_TMEM_LD32(taddr, r)                                                                                     \
  asm volatile(                                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "    \
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"                 \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),      \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),     \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                   \
      : "r"(taddr))

struct Shared {
  uint64_t b_full[kNSB], b_empty[kNSB], a_full[kNSA], a_empty[kNSA], d_full, d_empty;
  uint32_t tmem_base;
  int dl[32];
  int fq[32];     // F of the dirty slots of this pass
};

// part[cta][q + j t] (q < nd, j < t) for the CTA's tiles; grid = nranges x nchunks
__global__ void __launch_bounds__(kThreads, 1)
gram_q_kernel(const uint8_t* __restrict__ Cq, const int* __restrict__ Fq, int64_t ntiles_total, int t, int nranges,
              const int* __restrict__ list, const int* __restrict__ counts, double* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Shared sh;
  const int nd = counts[2];
  if (nd == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.x % nchunks(t), range = blockIdx.x / nchunks(t);
  const int s0 = chunk * kTc, tc = min(kTc, t - s0);
  const int nrow = (4 * tc + 15) / 16 * 16;                // N (B rows) of this chunk, padded to 16
  const int64_t bb = block_bytes(t);
  const uint32_t bcopy = static_cast<uint32_t>((nrow + 7) / 8 * 1024);
  const int ntiles = static_cast<int>((ntiles_total - range + nranges - 1) / nranges);
  if (ntiles <= 0) {            // no tiles (more CTAs than tiles): zero partial rows, nothing else
    double* o = part + static_cast<int64_t>(blockIdx.x) * t * t;
    for (int idx = threadIdx.x; idx < nd * t; idx += blockDim.x) o[(idx % nd) + static_cast<int64_t>(idx / nd) * t] = 0.0;
    return;
  }
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* bbuf = base;                                    // kNSB x 64 KB
  uint8_t* abuf = bbuf + kNSB * 65536;                     // kNSA x 16 KB
  double* out = part + static_cast<int64_t>(blockIdx.x) * t * t;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNSB; ++s) { k1tc::mbar_init(&sh.b_full[s], 1); k1tc::mbar_init(&sh.b_empty[s], 1); }
    for (int s = 0; s < kNSA; ++s) { k1tc::mbar_init(&sh.a_full[s], 4); k1tc::mbar_init(&sh.a_empty[s], 1); }
    k1tc::mbar_init(&sh.d_full, 1);
    k1tc::mbar_init(&sh.d_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) k1tc::tmem_alloc<1>(&sh.tmem_base, 512);
  k1tc::tc_fence_before();
  __syncthreads();
  k1tc::tc_fence_after();
  const uint32_t tmem = sh.tmem_base;
  int T0 = 0, ndrain = 0;
#pragma unroll 1
  for (int q0 = 0; q0 < nd; q0 += 32) {                    // dirty slots in passes of 32
    const int ndg = min(32, nd - q0);
    if (threadIdx.x < 32) {
      const int s = threadIdx.x < ndg ? list[q0 + threadIdx.x] : -1;
      sh.dl[threadIdx.x] = s;
      sh.fq[threadIdx.x] = s >= 0 ? Fq[s] : 0;
    }
    __syncthreads();
    if (warp == 0) {
      // ------------------------------------------------ producer: the chunk's rows of each tile
      for (int i = 0; i < ntiles; ++i) {
        const int T = T0 + i, s = T % kNSB;
        if (T >= kNSB) k1tc::mbar_wait(&sh.b_empty[s], ((T / kNSB) - 1) & 1);
        if (lane == 0) {
          const int64_t tile = range + static_cast<int64_t>(i) * nranges;
          k1tc::mbar_arrive_expect_tx(&sh.b_full[s], bcopy);
          k1tc::bulk_load(bbuf + s * 65536, Cq + tile * bb + static_cast<int64_t>(chunk) * 65536, bcopy, &sh.b_full[s]);
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      const uint32_t id0 = k1tc::idesc_i8m(128, nrow > 256 ? 256 : nrow, true);
      const uint32_t id1 = k1tc::idesc_i8m(128, nrow > 256 ? nrow - 256 : 16, true);
      bool first = true;
      for (int i = 0; i < ntiles; ++i) {
        const int T = T0 + i, sa = T % kNSA, sb = T % kNSB;
        k1tc::mbar_wait(&sh.a_full[sa], (T / kNSA) & 1);
        k1tc::mbar_wait(&sh.b_full[sb], (T / kNSB) & 1);
        k1tc::tc_fence_after();
        if (i > 0 && (i % kEpochTiles) == 0) {             // int32 bound: drain, restart
          k1tc::mma_commit_e(&sh.d_full);
          k1tc::mbar_wait(&sh.d_empty, ndrain & 1);
          ++ndrain;
          k1tc::tc_fence_after();
          first = true;
        }
        const uint32_t a0 = smem_u32(abuf + sa * 16384), b0 = smem_u32(bbuf + sb * 65536);
#pragma unroll
        for (int ks = 0; ks < kTR / 32; ++ks) {
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint64_t ad = desc_sw128(a0 + 32 * ks);
          k1tc::mma_i8_ss_e(tmem, ad, desc_sw128(b0 + 32 * ks), id0, acc);
          if (nrow > 256) k1tc::mma_i8_ss_e(tmem + 256, ad, desc_sw128(b0 + 32768 + 32 * ks), id1, acc);
        }
        first = false;
        k1tc::mma_commit_e(&sh.a_empty[sa]);
        k1tc::mma_commit_e(&sh.b_empty[sb]);
      }
      k1tc::mma_commit_e(&sh.d_full);
      ++ndrain;
    } else if (warp >= kGather0) {
      // ------------------------------------------------ A gather + drains
      const int gt = threadIdx.x - 32 * kGather0;          // 0..127
      const int quarter = warp & 3;
      bool first_drain = true;
      auto drain = [&]() {
        k1tc::mbar_wait(&sh.d_full, ndrain & 1);
        ++ndrain;
        k1tc::tc_fence_after();
        // lane l of quarter Q holds D rows 4 q + p, q = 8 Q + l / 4, p = l % 4
        const int q = 8 * quarter + (lane >> 2), p = lane & 3;
        const double wq = __longlong_as_double(static_cast<long long>(8 * p + 1023) << 52);   // 256^p
#pragma unroll 1
        for (int c0 = 0; c0 < nrow; c0 += 32) {           // 8 slots x 4 planes per load
          uint32_t v[32];
          A9Q_TMEM_LD32(tmem + (static_cast<uint32_t>(32 * quarter) << 16) + c0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          double g[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            // sum over p' in fp64 (exact integers scaled by powers of two, largest term last)
            double x = static_cast<double>(static_cast<int>(v[4 * jj])) +
                       static_cast<double>(static_cast<int>(v[4 * jj + 1])) * 256.0;
            x += static_cast<double>(static_cast<int>(v[4 * jj + 2])) * 65536.0;
            x += static_cast<double>(static_cast<int>(v[4 * jj + 3])) * 16777216.0;
            x *= wq;
            x += __shfl_xor_sync(0xffffffffu, x, 1);
            x += __shfl_xor_sync(0xffffffffu, x, 2);
            g[jj] = x;
          }
          if (q < ndg) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int j = s0 + c0 / 4 + jj;
              if ((jj & 3) == p && j < s0 + tc) {
                const int e = -(sh.fq[q] + Fq[j]);
                const double val = g[jj] * __longlong_as_double(static_cast<long long>(e + 1023) << 52);
                double* dst = out + (q0 + q) + static_cast<int64_t>(j) * t;
                *dst = first_drain ? val : *dst + val;
              }
            }
          }
        }
        if (first_drain) {
          // the fixed-order reduction sums whole partial rows: zero the columns of the other
          // slot chunks (computed by the other CTAs of this row-tile set)
          for (int idx = gt; idx < ndg * t; idx += 128) {
            const int qq = idx / t, j = idx - qq * t;
            if (j < s0 || j >= s0 + tc) out[(q0 + qq) + static_cast<int64_t>(j) * t] = 0.0;
          }
        }
        first_drain = false;
        k1tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.d_empty);
      };
      for (int i = 0; i < ntiles; ++i) {
        const int T = T0 + i, sa = T % kNSA;
        const int64_t tile = range + static_cast<int64_t>(i) * nranges;
        const uint8_t* blk = Cq + tile * bb;
        // 16-byte chunks of the dirty rows: idx = (q, p, c), q < ndg
        uint4 vals[8];
        int dsts[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = gt + 128 * k;                  // < 32 x 4 x 8 = 1024
          const int q = idx >> 5, p = (idx >> 3) & 3, c = idx & 7;
          dsts[k] = -1;
          if (q < ndg) {
            const int rs = 4 * sh.dl[q] + p, rd = 4 * q + p;
            vals[k] = __ldg(reinterpret_cast<const uint4*>(blk + swz(rs, c)));
            dsts[k] = static_cast<int>(swz(rd, c));
          }
        }
        if (T >= kNSA) k1tc::mbar_wait(&sh.a_empty[sa], ((T / kNSA) - 1) & 1);
        uint8_t* as = abuf + sa * 16384;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (dsts[k] >= 0) *reinterpret_cast<uint4*>(as + dsts[k]) = vals[k];
        k1tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.a_full[sa]);
        // the MMA issuer closes an epoch when it reaches tile i = k kEpochTiles (after this
        // tile's A stage is published), then waits for the drain
        if (i > 0 && (i % kEpochTiles) == 0) drain();
      }
      drain();
    }
    k1tc::tc_fence_before();
    __syncthreads();
    k1tc::tc_fence_after();
    T0 += ntiles;
  }
  k1tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    k1tc::tc_fence_after();
    k1tc::tmem_dealloc<1>(tmem, 512);
  }
}

// A7 for the quantised copy, step 1: per admission (or vacated slot) a = 0 .. na + nz - 1 of this
// commit, its slot, column r (-1: vacated) and C = (the column's maximum biased exponent over the
// K1F units that saw it) - 30, so |v| <= 2^29 for its largest element; F_s = kFbase - C -> Fq.
// One warp per admission.
__global__ void quant_adm_kernel(const int* __restrict__ admit, const int* __restrict__ counts, int nc, int t,
                                 const int* __restrict__ gE, int nunits, int nsg, int kFbase, int* __restrict__ Fq,
                                 int4* __restrict__ qadm) {
  const int na = counts[0], nz = counts[1];
  const int a = static_cast<int>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (a >= na + nz) return;
  int slot, r = -1;
  if (a < na) { slot = admit[2 * a]; r = admit[2 * a + 1]; }
  else slot = admit[2 * (nc + t) - 2 - 2 * (a - na)];
  int em = 0;
  if (r >= 0) {
    const int cg = r >> 5, jl = r & 31, ncg = (nc + 31) / 32;
    for (int u = ln; u < nunits; u += 32)
      if (((u / nsg) % ncg) == cg && (u % nsg) == 0) em = max(em, gE[u * 32 + jl]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) em = max(em, __shfl_xor_sync(0xffffffffu, em, o));
  }
  const int C = em - 30;
  if (ln == 0) {
    Fq[slot] = r >= 0 ? kFbase - C : 0;
    qadm[a] = make_int4(slot, r, C, 0);
  }
}

// A7 for the quantised copy, step 2: every admitted column is read once and written twice -
// bit-exactly into the row-tiled fp64 / fp32 basis (lines of RL rows)
// and as the digit planes of v = round(x 2^F_s) (zero lines and planes for vacated slots).  Work
// items are (admission, 512 rows); a warp takes items with a grid stride over all admissions (the
// grid fills the GPU whatever the device-side admission count) and loads the next item's rows into
// registers while it converts and stores the current one from its shared buffer.
template <typename T>
__global__ void __launch_bounds__(256, 3)
basis_quant_kernel(const T* __restrict__ X, int64_t ld, uint8_t* __restrict__ Cq, int64_t m_loc, int t,
                   const int* __restrict__ counts, const int4* __restrict__ qadm, T* __restrict__ Cb) {
  constexpr int RL = 128 / sizeof(T);
  constexpr bool kF64 = sizeof(T) == 8;
  constexpr int kQ = 16 * static_cast<int>(sizeof(T)) / 16;   // uint4 per 16-row run (8 / 4)
  constexpr int kE = 16 / static_cast<int>(sizeof(T));        // elements per uint4
  const int nadm = counts[0] + counts[1];
  const int64_t bb = block_bytes(t);
  const int64_t nchunk16 = (m_loc + 15) / 16;
  const int nwork = static_cast<int>((nchunk16 + 31) / 32);      // items per admission
  const int total = nadm * nwork;                                 // < 2^31 (m_loc < 2^31, nadm <= 2 b + t)
  __shared__ uint4 s_x[8][32 * kQ + 32];                        // +1 uint4 pad per run
  const int wl = threadIdx.x >> 5, ln = threadIdx.x & 31;
  uint4* sw = s_x[wl];
  const int wstride = static_cast<int>(gridDim.x) * (blockDim.x >> 5);
  uint4 nx[kQ];
  // coalesced loads of item wi's 512 rows (zeros past m_loc and for vacated slots)
  auto fetch = [&](int wi) {
    const int a = wi / nwork;
    const int64_t base_row = static_cast<int64_t>(wi - a * nwork) * 512;
    const int r = __ldg(&qadm[a].y);
    const T* col = r >= 0 ? X + static_cast<int64_t>(r) * ld : nullptr;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int64_t row = base_row + static_cast<int64_t>(q * 32 + ln) * kE;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (col && row + kE <= m_loc) v = __ldcs(reinterpret_cast<const uint4*>(col + row));
      else if (col && row < m_loc) {
        T tmp[kE];
#pragma unroll
        for (int e = 0; e < kE; ++e) tmp[e] = row + e < m_loc ? col[row + e] : T(0);
        v = *reinterpret_cast<uint4*>(tmp);
      }
      nx[q] = v;
    }
  };
  int w = static_cast<int>(blockIdx.x) * (blockDim.x >> 5) + wl;
  if (w < total) fetch(w);
  for (; w < total; w += wstride) {
    const int a = w / nwork;
    const int64_t wk = w - a * nwork;
    const int4 qa = __ldg(&qadm[a]);
    const int slot = qa.x, C = qa.z;
    const int64_t base_row = wk * 512;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int u = q * 32 + ln;
      sw[(u / kQ) * (kQ + 1) + (u % kQ)] = nx[q];                // run u / kQ, padded
    }
    __syncwarp();
    if (w + wstride < total) fetch(w + wstride);                   // in flight during the work below
    // exact copy: a run of 16 rows is one 128-byte basis line (f64, 8 lanes per line) or
    // half of one (f32, 4 lanes)
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int u = q * 32 + ln;
      const int run = u / kQ, part = u % kQ;
      const int64_t i0r = base_row + static_cast<int64_t>(run) * 16;
      if (i0r < m_loc) {
        T* dst = Cb + ((i0r / RL) * t + slot) * RL + (i0r % RL);
        __stcs(reinterpret_cast<uint4*>(dst) + part, sw[run * (kQ + 1) + part]);
      }
    }
    const int64_t ch = wk * 32 + ln;                               // this lane's run
    const bool valid = ch < nchunk16;
    const int64_t i0 = ch * 16;
    uint32_t wv[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      // one 16-byte shared load per kE elements (conflict-free: runs are 9 / 5 uint4 apart)
      uint32_t hi, lo;
      if constexpr (kF64) {
        const uint4 q4 = sw[ln * (kQ + 1) + e / 2];
        hi = (e & 1) ? q4.w : q4.y; lo = (e & 1) ? q4.z : q4.x;
      } else {
        const uint4 q4 = sw[ln * (kQ + 1) + e / 4];
        hi = (e & 3) == 0 ? q4.x : (e & 3) == 1 ? q4.y : (e & 3) == 2 ? q4.z : q4.w; lo = 0u;
      }
      const int E = static_cast<int>((hi << 1) >> (kF64 ? 21 : 24));
      const uint32_t pw = (E - C) < 0 || (E - C) > 31 ? 0u : (1u << (E - C));   // 2^(33 - k)
      const uint32_t tt = kF64 ? __funnelshift_r(lo, (hi & 0xFFFFFu) | 0x100000u, 21) : ((hi << 8) | 0x80000000u);
      const uint32_t u = __umulhi(tt, pw) + 1u;
      const int v = static_cast<int>(u >> 1);
      const int sg = static_cast<int>(hi) >> 31;
      wv[e] = static_cast<uint32_t>(v * (2 * sg + 1) + 0x808080);
    }
    __syncwarp();                                                  // the buffer is reused by the next item
    // 4x4 byte transposes -> plane words (rows i0 .. i0 + 15 of plane p)
    uint32_t P[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t x0 = __byte_perm(wv[4 * q], wv[4 * q + 1], 0x5140), x1 = __byte_perm(wv[4 * q], wv[4 * q + 1], 0x7362);
      const uint32_t y0 = __byte_perm(wv[4 * q + 2], wv[4 * q + 3], 0x5140), y1 = __byte_perm(wv[4 * q + 2], wv[4 * q + 3], 0x7362);
      P[0][q] = __byte_perm(x0, y0, 0x5410) ^ 0x80808080u;
      P[1][q] = __byte_perm(x0, y0, 0x7632) ^ 0x80808080u;
      P[2][q] = __byte_perm(x1, y1, 0x5410) ^ 0x80808080u;
      P[3][q] = __byte_perm(x1, y1, 0x7632);
    }
    const int64_t tile = i0 / kTR;
    const int c = static_cast<int>((i0 % kTR) / 16);
    uint8_t* blk = Cq + tile * bb;
    if (valid) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
        *reinterpret_cast<uint4*>(blk + swz(4 * slot + p, c)) = make_uint4(P[p][0], P[p][1], P[p][2], P[p][3]);
    }
  }
}

}  // namespace a9q
}  // namespace oid
