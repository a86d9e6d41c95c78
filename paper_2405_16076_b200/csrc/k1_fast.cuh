// K1F, the fast fused ingest for sm_100a (OID_K1_TC_FAST): Y_part = Z(:, rows) X_blk and the column
// norms n_j = ||x_j||^2 in one read of X (Alg 3 steps 10 and 13), with every snapshot
// value quantised to a 31-bit per-column fixed point (the north_star's "chosen to meet the stated
// tolerance"; DESIGN section 7 derives the error bound the parity tests check).
//
// Arithmetic.  The sketch entries are Gauss-16 half-integers L = q + 1/2 with q int8 (reading R2), so
// Z X = s (Q X + (1/2) 1 colsum(X)).  Each x is rounded to v = round(x 2^F_j), |v| <= 2^30, and v is
// cut into four SIGNED base-256 digits (v + 0x808080 has the digits + 128 in bytes 0..2 and the top
// digit in byte 3), so Q v = sum_p 256^p Q d_p runs on the tensor cores as tcgen05.mma kind::i8 with
// int32 accumulation in TMEM, exactly.  The only rounding is the quantisation of x (<= 2^-29 of the
// column's maximum per element, see kH / kShrink) and the final fp64 assembly.
//
// Shape of the contraction (B200-first): the four planes of the 32 block columns are stacked into the
// M = 128 rows of the A operand (row 32 (j / 8) + 8 p + j % 8 = plane p of column j), so one unit holds up to 512
// sketch rows in the 512 TMEM columns (D = 128 lanes x nu columns, two N = 256 MMAs per K step) and
// every X element is converted ONCE per launch when ell <= 512 (C3) instead of once per 256 sketch
// rows.  The sketch tile Z^T (nu x 64 rows of int8, K-major) is the B operand, generated straight into
// shared memory.  The digit conversion is integer-only and runs mostly on the FMA pipe (IMAD.HI as
// the right shift), because fp64 instructions stall while int8 MMAs run on the SM.
//
// CTA (one per SM, 16 warps, persistent over one unit = contiguous row range x 32 columns x nu
// sketch rows):
//   warp 0       TMA producer: one box per tile, every column one contiguous 528-byte line
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer (A and B from shared memory)
//   warps 4-7    digit slicer: 16 rows of one column per thread and tile; per-column exponent
//                check; the A operand (row 32 (j/8) + 8 p + j%8 = plane p of column j); int32 dp4a column
//                sums and norm terms; drains the accumulators at epoch ends (a warp reads TMEM lane
//                quarter warp % 4, where the four planes of 8 columns sit in adjacent lanes)
//   warps 8-15   sketch generator: Philox4x32-10 (rounds 1-2 and half of round 3 factored into a
//                row part and a group part), Gauss-16 nibbles -> int8 by PRMT, st.shared into B
// Exponents.  F_j starts from a guess (the unit's observed column maximum of the previous launch,
// kept in the workspace; the first tile + 8 bits when there is none).  A tile whose maximum exceeds
// the guess by more than kH bits raises F_j: the accumulators are drained to fp64 first
// ("accumulation epochs", also every kEpochTiles tiles against int32 overflow), so X is still read
// once.  A guess more than kH + kShrink bits above the unit's observed maximum (precision would be
// lost) makes the CTA run the unit again with the observed exponents (at most once).
#pragma once
#include <climits>
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
#include "sm100.cuh"

namespace oid {
namespace k1f {

using k1tc::smem_u32;

constexpr int kWarps = 18;
constexpr int kThreads = 32 * kWarps;
constexpr int kKT = 64;            // data rows per tile (K of one pipeline stage)
constexpr int kNSX = 6;            // X stages (~100 KB of fp64 in flight per SM)
constexpr int kNSA = 3;            // A stages (digit planes, 8 KB)
constexpr int kNSB = 3;            // B stages (sketch tile, 256 / 512 rows x 64 bytes)
constexpr int kSl0 = 2, kSlW = 8;  // slicer warps 2..9 (each TMEM lane quarter twice)
constexpr int kSlE = kKT / kSlW;   // rows per slicer thread and tile (16)
constexpr int kGen0 = 10, kGenW = 8;   // generator warps 10..17
constexpr int kEpochTiles = 2048;  // int32 bound: 2048 * 64 rows * 128 * 111 < 2^31
constexpr int kH = 1;              // exponent headroom over the guess (bits)
constexpr int kShrink = 1;         // tolerated excess of the guess over the observed maximum (bits)
constexpr int kHFirst = 8;         // headroom over the first tile when there is no guess
constexpr int kNoGuess = INT_MIN;
constexpr int kMaxUnits = 256;

struct Keys { uint32_t k0[10], k1[10]; };   // Philox key schedule (reading R1)

struct Geom {
  int nu;            // sketch rows per unit (multiple of 16, <= 512)
  int nsg, ncg;      // sketch-row groups, 32-column groups
  int nranges;       // CTAs sharing the tiles of one (column group, sketch group), round-robin
  int xline, x_bytes, b_bytes, smem;
  int brows;         // rows of a B stage (256 or 512; rows past nu are generated and ignored)
  // multipliers passed at run time so that ptxas keeps them as IMAD / IMAD.HI (FMA pipe)
  // instead of strength-reducing them to ALU shifts (the pipes are balanced by hand)
  uint32_t k2, k16, k256, k2048, k65536, k2p31;
  int nunits() const { return nranges * ncg * nsg; }
};

inline Geom make_geom(int ell, int ncols, int64_t m_loc, bool f64, int num_sms) {
  Geom g{};
  g.nsg = (ell + 511) / 512;
  g.nu = ((ell + g.nsg - 1) / g.nsg + 15) / 16 * 16;
  g.ncg = (ncols + 31) / 32;
  const int per_range_units = g.nsg * g.ncg;
  int nr = std::max(1, num_sms / per_range_units);
  const int64_t tiles = (m_loc + kKT - 1) / kKT;
  g.nranges = static_cast<int>(std::min<int64_t>(nr, tiles));   // CTAs per (column, sketch) group
  g.xline = kKT * (f64 ? 8 : 4) + 16;   // one column's tile rows + 16 B pad (conflict-free reads)
  g.x_bytes = 32 * g.xline;
  g.brows = g.nu > 256 ? 512 : 256;
  g.b_bytes = g.brows * kKT;
  g.k2 = 2; g.k16 = 16; g.k256 = 256; g.k2048 = 2048; g.k65536 = 65536; g.k2p31 = 0x80000000u;
  g.smem = 1024 + kNSX * g.x_bytes + kNSA * (128 * kKT) + kNSB * g.b_bytes;
  return g;
}

struct Shared {
  uint64_t x_full[kNSX], x_empty[kNSX];
  uint64_t a_full[kNSA], a_empty[kNSA];
  uint64_t b_full[kNSB], b_empty[kNSB];
  uint64_t d_full, d_empty;
  uint32_t tmem_base;
  int aflag[kNSA];
  int cold[32];           // C_j of the epoch being drained
  int tmx[kSlW][32];      // per slicer warp: tile maximum of E (raise path), then the observed max
  double cs[kSlW][32], nr[kSlW][32];
  int redo;
};

// mad.hi.u32 / mul.lo.u32 / mad.lo.s32 as written (the multiplier comes from a kernel parameter
// where the FMA pipe is wanted, see Geom)
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t mullo(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ int madlo_s(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int mulhi_s(int a, int b) {
  int d;
  asm("mul.hi.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t s) {   // a << s, 0 for s >= 32
  uint32_t d;
  asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(s));
  return d;
}

#define K1F_TMEM_LD32(taddr, r)                                                                                      \
  asm volatile(                                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "    \
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"                 \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),      \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),     \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                   \
      : "r"(taddr))

__device__ __forceinline__ double pow2(int e) {   // 2^e as a double, e in [-1022, 1023]
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// Per-element constants of the conversion (see convert16).
template <typename T> struct Fmt;
template <> struct Fmt<double> {
  static constexpr int kFbase = 1021;   // F = kFbase - C  (a = E - C = E + F - 1021)
  static constexpr int kEmax = 2047;
};
template <> struct Fmt<float> {
  static constexpr int kFbase = 125;    // a = E + F - 125
  static constexpr int kEmax = 255;
};

template <typename TD, int NROW>
__global__ void __launch_bounds__(kThreads, 1)
k1f_kernel(const __grid_constant__ CUtensorMap tmap, int ncols, const __grid_constant__ Keys keys, int64_t row_begin,
           int64_t m_loc, Geom g, uint32_t t0, uint32_t t1, double* __restrict__ part, double* __restrict__ npart,
           double* __restrict__ cpart, int* __restrict__ gE, unsigned* __restrict__ flags) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Shared sh;
  constexpr bool kF64 = sizeof(TD) == 8;
  constexpr int kFbase = Fmt<TD>::kFbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int sg = unit % g.nsg;
  const int cg = (unit / g.nsg) % g.ncg;
  const int range = unit / (g.nsg * g.ncg);
  // tiles are dealt round-robin (tile gt = range + k nranges): at any moment the whole grid reads
  // a narrow window of rows of each column (few 2 MB pages, DRAM row locality), instead of 148
  // distant row ranges x 32 columns
  const int64_t total_tiles = (m_loc + kKT - 1) / kKT;
  const int ntiles = static_cast<int>((total_tiles - range + g.nranges - 1) / g.nranges);
  const int nu = g.nu;
  const int nh = nu > 256 ? 2 : 1;                 // N halves of the unit (MMA N <= 256)
  static_assert(NROW == 1 || NROW == 2, "generator rows per thread");

  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* xbuf = base;                                    // kNSX x x_bytes: [column][xline]
  uint8_t* abuf = xbuf + kNSX * g.x_bytes;                 // kNSA x 8 KB
  uint8_t* bbuf = abuf + kNSA * 128 * kKT;                 // kNSB x b_bytes

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNSX; ++s) {
      k1tc::mbar_init(&sh.x_full[s], 1);
      k1tc::mbar_init(&sh.x_empty[s], kSlW);
    }
    for (int s = 0; s < kNSA; ++s) {
      k1tc::mbar_init(&sh.a_full[s], kSlW);
      k1tc::mbar_init(&sh.a_empty[s], 1);
    }
    for (int s = 0; s < kNSB; ++s) {
      k1tc::mbar_init(&sh.b_full[s], kGenW);
      k1tc::mbar_init(&sh.b_empty[s], 1);
    }
    k1tc::mbar_init(&sh.d_full, 1);
    k1tc::mbar_init(&sh.d_empty, kSlW);
    sh.redo = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) k1tc::tmem_alloc<1>(&sh.tmem_base, 512);
  k1tc::tc_fence_before();
  __syncthreads();
  k1tc::tc_fence_after();
  const uint32_t tmem = sh.tmem_base;

  // running counters across passes (pipeline phases continue)
  int T0 = 0;        // global tile index of this pass's first tile
  int ndrain = 0;    // drains so far (d_full / d_empty phase)
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (warp == 0) {
      // ------------------------------------------------------------ TMA producer
      // one 2-D box per tile: kKT + pad rows x 32 columns, no swizzle, so every column is one
      // contiguous line of xline bytes (512-byte lines stream at HBM speed; 128-byte lines cap
      // near 4.6 TB/s, scripts/micro/xstream.cu).  The pad rows (16 bytes, the next tile's first
      // rows, hit in L2) offset the lines so the slicer's reads are bank-conflict-free.  Rows past
      // m_loc and columns past ncols are zero-filled by the TMA unit.
      for (int t = 0; t < ntiles; ++t) {
        const int T = T0 + t, s = T % kNSX;
        if (T >= kNSX) k1tc::mbar_wait(&sh.x_empty[s], ((T / kNSX) - 1) & 1);
        k1tc::mbar_arrive_expect_tx_e(&sh.x_full[s], g.x_bytes);
        k1tc::tma_load_2d_e(xbuf + s * g.x_bytes, &tmap, &sh.x_full[s], static_cast<int>((range + int64_t(t) * g.nranges) * kKT),
                            32 * cg);
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t abase = smem_u32(abuf), bbase = smem_u32(bbuf);
      const uint32_t id0 = k1tc::idesc_i8m(128, nh == 2 ? 256 : nu, true);
      const uint32_t id1 = k1tc::idesc_i8m(128, nh == 2 ? nu - 256 : 16, true);
      const uint32_t bchunk = static_cast<uint32_t>(g.brows) * 16;   // bytes per 16-byte K chunk of B
      bool first = true;
      for (int t = 0; t < ntiles; ++t) {
        const int T = T0 + t, sa = T % kNSA, sb = T % kNSB;
        k1tc::mbar_wait(&sh.a_full[sa], (T / kNSA) & 1);
        k1tc::mbar_wait(&sh.b_full[sb], (T / kNSB) & 1);
        k1tc::tc_fence_after();
        if (sh.aflag[sa] && t > 0) {       // close the accumulation epoch: drain D first
          k1tc::mma_commit_e(&sh.d_full);
          k1tc::mbar_wait(&sh.d_empty, ndrain & 1);
          ++ndrain;
          k1tc::tc_fence_after();
          first = true;
        }
        const uint32_t a0 = abase + sa * (128 * kKT), b0 = bbase + sb * g.b_bytes;
#pragma unroll
        for (int ks = 0; ks < kKT / 32; ++ks) {
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint64_t ad = k1tc::umma_desc(a0 + ks * 2 * 2048, 2048, 128);
          k1tc::mma_i8_ss_e(tmem, ad, k1tc::umma_desc(b0 + ks * 2 * bchunk, bchunk, 128), id0, acc);
          if (nh == 2) k1tc::mma_i8_ss_e(tmem + 256, ad, k1tc::umma_desc(b0 + ks * 2 * bchunk + 4096, bchunk, 128), id1, acc);
        }
        first = false;
        k1tc::mma_commit_e(&sh.a_empty[sa]);
        k1tc::mma_commit_e(&sh.b_empty[sb]);
      }
      k1tc::mma_commit_e(&sh.d_full);      // final epoch
      ++ndrain;
    } else if (warp >= kSl0 && warp < kSl0 + kSlW) {
      // ------------------------------------------------------------ digit slicer + drains
      const int sw = warp - kSl0;          // 0 .. kSlW - 1
      const int rs = sw * kSlE;            // first tile row of this thread (rows rs .. rs + kSlE - 1)
      const int c = rs >> 4, h = (rs >> 3) & 1;   // K chunk (16 rows) and 8-row half of the rows
      const int j = lane;                  // column within the group
      const int quarter = warp & 3;        // TMEM lane quarter this warp may read
      constexpr int kDW = kSlW / 4;        // warps per TMEM lane quarter in a drain
      const int dpair = sw >> 2;           // which of them (column chunks dealt round-robin)
      constexpr int kBarSl = 1;
      constexpr int kSlT = 32 * kSlW;
      // exponent guess (first pass) or the observed maximum (second pass)
      int Cj = gE[unit * 32 + j];
      bool need_first = (Cj == kNoGuess);  // derive from the first tile
      if (!need_first) Cj = Cj - 31 + kH;  // guess = observed max E -> C
      int Cfirst = Cj;                     // C of the first epoch (the precision check)
      int obs = 0;                         // observed max E of this thread's elements
      int cs[4] = {0, 0, 0, 0};
      int nq[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // digit-pair sums D_pq = sum_i d_p d_q, p <= q
      double csf = 0.0, nrf = 0.0;
      bool first_drain = true;
      const uint32_t K2p31 = g.k2p31, K2 = g.k2, K256 = g.k256, K2048 = g.k2048;

      // int32 digit sums of the closing epoch -> fp64, with that epoch's F = kFbase - C
      auto flush = [&](int Cep) {
        const int F = kFbase - Cep;
        const long long csi = static_cast<long long>(cs[0]) + (static_cast<long long>(cs[1]) << 8) +
                              (static_cast<long long>(cs[2]) << 16) + (static_cast<long long>(cs[3]) << 24);
        csf += static_cast<double>(csi) * pow2(-F);
        // ||v||^2 = sum_p,q 256^(p+q) D_pq (exact integers; fp64 sum, largest terms first)
        double nn = static_cast<double>(nq[0]) * 0x1p48;                                      // (3,3)
        nn += 2.0 * static_cast<double>(nq[1]) * 0x1p40;                                     // (2,3)
        nn += static_cast<double>(nq[2]) * 0x1p32 + 2.0 * static_cast<double>(nq[3]) * 0x1p32;  // (2,2) (1,3)
        nn += 2.0 * static_cast<double>(nq[4]) * 0x1p24 + 2.0 * static_cast<double>(nq[5]) * 0x1p24;  // (1,2) (0,3)
        nn += static_cast<double>(nq[6]) * 0x1p16 + 2.0 * static_cast<double>(nq[7]) * 0x1p16;  // (1,1) (0,2)
        nn += 2.0 * static_cast<double>(nq[8]) * 0x1p8 + static_cast<double>(nq[9]);          // (0,1) (0,0)
        nrf += nn * pow2(-F) * pow2(-F);
#pragma unroll
        for (int p = 0; p < 4; ++p) cs[p] = 0;
#pragma unroll
        for (int q = 0; q < 10; ++q) nq[q] = 0;
      };
      // D (TMEM, int32; lane 32 (j / 8) + 8 p + j % 8 = plane p of column j) of the closing epoch -> fp64 partials
      // part[unit][r][j]: the four planes of a column sit in adjacent lanes of one warp, so they
      // are combined by two shuffles in a fixed order; column chunks alternate between the two
      // warps of a lane quarter.  sh.cold holds the epoch's C_j.
      auto drain = [&](int Cep) {
        if (sw < 1) sh.cold[j] = Cep;
        k1tc::named_bar(kBarSl, kSlT);
        k1tc::mbar_wait(&sh.d_full, ndrain & 1);
        ++ndrain;
        k1tc::tc_fence_after();
        const int jd = 8 * quarter + (lane & 7), pd = lane >> 3;
        const double wgt = pow2(8 * pd - (kFbase - sh.cold[jd]));
        double* dst = part + static_cast<int64_t>(unit) * nu * 32;
        const int nchunk = (nu + 31) / 32;
#pragma unroll 1
        for (int k = dpair; k < nchunk; k += kDW) {
          const int c0 = 32 * k;
          uint32_t v[32];
          K1F_TMEM_LD32(tmem + (static_cast<uint32_t>(32 * quarter) << 16) + c0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          double out[8];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            double x = static_cast<double>(static_cast<int>(v[i])) * wgt;
            x += __shfl_xor_sync(0xffffffffu, x, 8);
            x += __shfl_xor_sync(0xffffffffu, x, 16);
            if ((i >> 3) == pd) out[i & 7] = x;   // lane p keeps rows 8 p .. 8 p + 7 of the chunk
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = c0 + 8 * pd + i;
            if (r < nu) {
              double* q = dst + static_cast<int64_t>(r) * 32 + jd;
              *q = first_drain ? out[i] : *q + out[i];
            }
          }
        }
        first_drain = false;
        k1tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.d_empty);
        k1tc::named_bar(kBarSl, kSlT);     // sh.cold is reused by the next drain
      };

#pragma unroll 1
      for (int t = 0; t < ntiles; ++t) {
        const int T = T0 + t;
        const int sx = T % kNSX, sa = T % kNSA;
        k1tc::mbar_wait(&sh.x_full[sx], (T / kNSX) & 1);
        uint32_t hi[kSlE], lo[kSlE];
        {
          const uint8_t* ln = xbuf + sx * g.x_bytes + j * g.xline;
          if constexpr (kF64) {
#pragma unroll
            for (int q = 0; q < kSlE / 2; ++q) {
              const uint4 v = *reinterpret_cast<const uint4*>(ln + (rs + 2 * q) * 8);
              lo[2 * q] = v.x; hi[2 * q] = v.y; lo[2 * q + 1] = v.z; hi[2 * q + 1] = v.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < kSlE / 4; ++q) {
              const uint4 v = *reinterpret_cast<const uint4*>(ln + (rs + 4 * q) * 4);
              hi[4 * q] = v.x; hi[4 * q + 1] = v.y; hi[4 * q + 2] = v.z; hi[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int e = 0; e < kSlE; ++e) lo[e] = 0u;
          }
        }
        // biased exponents E (FMA pipe): e2 = bits << 1 drops the sign, E = e2 >> 21 (f64) / >> 24
        int Ee[kSlE];
        int emax = 0;
#pragma unroll
        for (int e = 0; e < kSlE; ++e) {
          // E = (bits << 1) >> 21 (f64) / >> 24 (f32) on the FMA pipe (IMAD, IMAD.HI): the ALU pipe
          // carries the generator's decode
          Ee[e] = static_cast<int>(madhi(mullo(hi[e], K2), kF64 ? K2048 : K256, 0u));
          emax = max(emax, Ee[e]);
        }
        obs = max(obs, emax);
        if (need_first) {                    // no guess: C from the first tile's maximum + kHFirst
          sh.tmx[sw][j] = emax;
          k1tc::named_bar(kBarSl, kSlT);
          int em = 0;
#pragma unroll
          for (int q = 0; q < kSlW; ++q) em = max(em, sh.tmx[q][j]);
          Cj = em - 31 + kHFirst;
          Cfirst = Cj;
          need_first = false;
          k1tc::named_bar(kBarSl, kSlT);
        }
        int newep = (t > 0 && (t % kEpochTiles) == 0) ? 1 : 0;
        if (newep && threadIdx.x == 32 * kSl0) atomicAdd(gE + kMaxUnits * 32 + 3, 1);
        const int Cold = Cj;                 // exponents of the epoch that may close here
        if (k1tc::named_bar_or(kBarSl, kSlT, (emax - Cj > 31) ? 1 : 0)) {
          // raise: C_j = (tile max E) - 31 + kH for the columns that overflow; a new epoch
          sh.tmx[sw][j] = emax;
          k1tc::named_bar(kBarSl, kSlT);
          int em = 0;
#pragma unroll
          for (int q = 0; q < kSlW; ++q) em = max(em, sh.tmx[q][j]);
          k1tc::named_bar(kBarSl, kSlT);
          if (em - Cj > 31) Cj = em - 31 + kH;
          if (t > 0) newep = 1;
          else Cfirst = Cj;
          if (threadIdx.x == 32 * kSl0) atomicAdd(gE + kMaxUnits * 32 + (t > 0 ? 1 : 0), 1);
        }
        if (newep) flush(Cold);              // before this tile's digits are added
        // ---- conversion: v = round(|x| 2^F) (31-bit), digits of v sg + 0x808080, 4x4 transposes
        uint32_t w[kSlE];
#pragma unroll
        for (int e = 0; e < kSlE; ++e) {
          const uint32_t a = static_cast<uint32_t>(Ee[e] - Cj);   // <= 31; negative -> p = 0
          const uint32_t p = shl_clamp(1u, a);                   // 2^(33 - k)
          uint32_t tt;
          // pipes balanced against the generator (ALU-heavy decode, FMA-heavy Philox): shifts on
          // the ALU, the variable right shift and the sign on the FMA pipe
          if constexpr (kF64) {
            // top 32 bits of the 53-bit mantissa: (1 << 31) | (mantissa 51..32 << 11) | (lo >> 21)
            tt = __funnelshift_r(lo[e], (hi[e] & 0xFFFFFu) | 0x100000u, 21);
          } else {
            tt = (hi[e] << 8) | 0x80000000u;
          }
          const uint32_t u = madhi(tt, p, 1u);                     // (t >> (k - 1)) + 1
          const int v = static_cast<int>(madhi(u, K2p31, 0u));     // round half up of t / 2^k
          const int sgn = madlo_s(mulhi_s(static_cast<int>(hi[e]), 2), 2, 1);   // -1 or +1 (FMA pipe)
          w[e] = static_cast<uint32_t>(madlo_s(v, sgn, 0x808080));
        }
        // the stage is released only once its values have been consumed (the loads' results are
        // in registers): an arrive right after issuing the loads let the next TMA load overwrite
        // the first lines before slow loads had read them
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.x_empty[sx]);
        uint32_t P[4][kSlE / 4];
#pragma unroll
        for (int q = 0; q < kSlE / 4; ++q) {
          const uint32_t x0 = k1tc::prmt(w[4 * q], w[4 * q + 1], 0x5140), x1 = k1tc::prmt(w[4 * q], w[4 * q + 1], 0x7362);
          const uint32_t y0 = k1tc::prmt(w[4 * q + 2], w[4 * q + 3], 0x5140), y1 = k1tc::prmt(w[4 * q + 2], w[4 * q + 3], 0x7362);
          P[0][q] = k1tc::prmt(x0, y0, 0x5410) ^ 0x80808080u;
          P[1][q] = k1tc::prmt(x0, y0, 0x7632) ^ 0x80808080u;
          P[2][q] = k1tc::prmt(x1, y1, 0x5410) ^ 0x80808080u;
          P[3][q] = k1tc::prmt(x1, y1, 0x7632);
        }
        // A stage free?  (the conversion above runs before the wait: see the generator)
#pragma unroll
        for (int q = 0; q < kSlE / 4; ++q) asm volatile("" ::"r"(P[0][q]), "r"(P[1][q]), "r"(P[2][q]), "r"(P[3][q]));
        if (T >= kNSA) k1tc::mbar_wait(&sh.a_empty[sa], ((T / kNSA) - 1) & 1);
        // A row 32 (j / 8) + 8 p + j % 8: the 8 lanes of a store phase hit 8 different 16-byte
        // bank groups, and the four planes of a column share a TMEM lane quarter (lanes l + 8 p)
        uint8_t* as = abuf + sa * (128 * kKT) + c * 2048 + (j >> 3) * 512 + (j & 7) * 16 + h * 8;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          if constexpr (kSlE == 16)
            *reinterpret_cast<uint4*>(as + p * 128) = make_uint4(P[p][0], P[p][1], P[p][2], P[p][3]);
          else
            *reinterpret_cast<uint2*>(as + p * 128) = make_uint2(P[p][0], P[p][1]);
        }
        k1tc::fence_proxy_async();
        if (sw == 0 && lane == 0) sh.aflag[sa] = newep;
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.a_full[sa]);
        // exact int32 column sums and norm terms of the digits (dp4a)
#pragma unroll
        for (int q = 0; q < kSlE / 4; ++q) {
#pragma unroll
          for (int p = 0; p < 4; ++p) cs[p] = __dp4a(static_cast<int>(P[p][q]), 0x01010101, cs[p]);
          nq[0] = __dp4a(static_cast<int>(P[3][q]), static_cast<int>(P[3][q]), nq[0]);
          nq[1] = __dp4a(static_cast<int>(P[2][q]), static_cast<int>(P[3][q]), nq[1]);
          nq[2] = __dp4a(static_cast<int>(P[2][q]), static_cast<int>(P[2][q]), nq[2]);
          nq[3] = __dp4a(static_cast<int>(P[1][q]), static_cast<int>(P[3][q]), nq[3]);
          nq[4] = __dp4a(static_cast<int>(P[1][q]), static_cast<int>(P[2][q]), nq[4]);
          nq[5] = __dp4a(static_cast<int>(P[0][q]), static_cast<int>(P[3][q]), nq[5]);
          nq[6] = __dp4a(static_cast<int>(P[1][q]), static_cast<int>(P[1][q]), nq[6]);
          nq[7] = __dp4a(static_cast<int>(P[0][q]), static_cast<int>(P[2][q]), nq[7]);
          nq[8] = __dp4a(static_cast<int>(P[0][q]), static_cast<int>(P[1][q]), nq[8]);
          nq[9] = __dp4a(static_cast<int>(P[0][q]), static_cast<int>(P[0][q]), nq[9]);
        }
        if (newep) drain(Cold);              // the MMA issuer commits the closed epoch at this tile
      }
      // final epoch of the pass
      flush(Cj);
      drain(Cj);
      // observed maxima, the precision check and the next launch's guess
      sh.tmx[sw][j] = obs;
      sh.cs[sw][j] = csf;
      sh.nr[sw][j] = nrf;
      k1tc::named_bar(kBarSl, kSlT);
      if (sw == 0) {
        int em = 0;
        double nsum = 0.0, csum = 0.0;
#pragma unroll
        for (int q = 0; q < kSlW; ++q) {
          em = max(em, sh.tmx[q][j]);
          nsum += sh.nr[q][j];
          csum += sh.cs[q][j];
        }
        gE[unit * 32 + j] = em;
        if (em >= Fmt<TD>::kEmax) atomicOr(flags, 1u);          // NaN / Inf in the block
        // the first epoch's C more than kH + kShrink above what the data needed: precision lost
        const bool lost = em > 0 && (em - Cfirst) < 31 - kH - kShrink;
        if (lost && pass == 0 && atomicOr(&sh.redo, 1) == 0) atomicAdd(gE + kMaxUnits * 32 + 2, 1);
        npart[unit * 32 + j] = nsum;
        cpart[unit * 32 + j] = csum;
      }
    } else if (warp >= kGen0) {
      // ------------------------------------------------------------ sketch generator
      const int gt = threadIdx.x - 32 * kGen0;    // 0..255
      // per-row parts of rounds 1-3 (counter (g, R, 0, 0), key (k0, k1), reading R2)
      uint32_t A2[2], R2[2];
      int rr[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        rr[q] = gt + 256 * q;
        const uint32_t R = static_cast<uint32_t>(sg * nu + rr[q]);
        uint32_t hi, lo;
        mulhilo32(0xD2511F53u, R ^ keys.k0[0], hi, lo);
        A2[q] = hi ^ keys.k1[1];
        R2[q] = lo;
      }
      const uint32_t bchunk = static_cast<uint32_t>(g.brows) * 16;
      const uint32_t boff[2] = {static_cast<uint32_t>((rr[0] >> 3) * 128 + (rr[0] & 7) * 16),
                                static_cast<uint32_t>((rr[1] >> 3) * 128 + (rr[1] & 7) * 16)};
      const uint32_t K16 = g.k16, K65536 = g.k65536;
      // the 32 sketch entries of each (row q, group gi) stream of tile t: Philox4x32-10 words
      auto philox = [&](int t, uint32_t (&c0)[4], uint32_t (&c1)[4], uint32_t (&c2)[4], uint32_t (&c3)[4]) {
        // group parts (uniform): rounds 1-3
        const uint32_t g0 = static_cast<uint32_t>((row_begin + (range + int64_t(t) * g.nranges) * kKT) >> 5);
        uint32_t G2[2], G3k[2], G5k[2], G5l[2];
#pragma unroll
        for (int gi = 0; gi < 2; ++gi) {
          uint32_t hh, l;
          mulhilo32(0xD2511F53u, g0 + gi, hh, l);
          const uint32_t G1 = hh ^ keys.k1[0];
          G2[gi] = l;
          uint32_t h2, l2;
          mulhilo32(0xCD9E8D57u, G1, h2, l2);
          const uint32_t G3 = h2 ^ keys.k0[1];
          const uint32_t G4 = l2;
          uint32_t h3, l3;
          mulhilo32(0xD2511F53u, G3, h3, l3);
          G3k[gi] = G4 ^ keys.k0[2];
          G5k[gi] = h3 ^ keys.k1[2];
          G5l[gi] = l3;
        }
#pragma unroll
        for (int q = 0; q < NROW; ++q)
#pragma unroll
          for (int gi = 0; gi < 2; ++gi) {
            const int ci = 2 * q + gi;
            const uint32_t x2 = A2[q] ^ G2[gi];      // c2 after round 2
            uint32_t h1, l1;
            mulhilo32(0xCD9E8D57u, x2, h1, l1);      // round 3
            c0[ci] = h1 ^ G3k[gi];
            c1[ci] = l1;
            c2[ci] = G5k[gi] ^ R2[q];
            c3[ci] = G5l[gi];
          }
#pragma unroll
        for (int rnd = 3; rnd < 10; ++rnd) {
#pragma unroll
          for (int ci = 0; ci < 2 * NROW; ++ci) {
            uint32_t hi0, lo0, hi1, lo1;
            mulhilo32(0xD2511F53u, c0[ci], hi0, lo0);
            mulhilo32(0xCD9E8D57u, c2[ci], hi1, lo1);
            const uint32_t n0 = hi1 ^ c1[ci] ^ keys.k0[rnd];
            const uint32_t n2 = hi0 ^ c3[ci] ^ keys.k1[rnd];
            c0[ci] = n0; c1[ci] = lo1; c2[ci] = n2; c3[ci] = lo0;
          }
        }
      };
      // software pipeline: the Philox rounds of tile t + 1 (FMA-heavy pipe) and the Gauss-16 decode
      // and stores of tile t (ALU pipe) are independent code in one block, so they interleave
      // one tile: wait for the stage, Philox of tile t + 1 into (n*), decode and store (c*) of tile t
      auto tile = [&](int t, const uint32_t (&c0)[4], const uint32_t (&c1)[4], const uint32_t (&c2)[4],
                      const uint32_t (&c3)[4], uint32_t (&n0)[4], uint32_t (&n1)[4], uint32_t (&n2)[4], uint32_t (&n3)[4]) {
        const int T = T0 + t, s = T % kNSB;
        if (T >= kNSB) {
          if (lane == 0) k1tc::mbar_wait(&sh.b_empty[s], ((T / kNSB) - 1) & 1);
          __syncwarp();
        }
        philox(t + 1, n0, n1, n2, n3);             // (past the last tile: unused)
        uint8_t* bs = bbuf + s * g.b_bytes;
#pragma unroll
        for (int ci = 0; ci < 2 * NROW; ++ci) {
          const int q = ci >> 1, gi = ci & 1;
          const uint32_t ws[4] = {c0[ci], c1[ci], c2[ci], c3[ci]};
          uint32_t pk[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // 8 nibbles n = (sign, v): q = m_v (sign 0) or ~m_v = -m_v - 1 (sign 1), 4 per PRMT
            const uint32_t wv = ws[k];
            const uint32_t wm = wv & 0x77777777u;
            const uint32_t w4 = mullo(wv, K16);
            const uint32_t mlo = k1tc::prmt(t0, t1, wm), mhi = k1tc::prmt(t0, t1, madhi(wm, K65536, 0u));
            const uint32_t slo = k1tc::prmt(wv, w4, 0x9D8Cu), shi = k1tc::prmt(wv, w4, 0xBFAEu);
            pk[2 * k] = mlo ^ slo;
            pk[2 * k + 1] = mhi ^ shi;
          }
          uint8_t* d0 = bs + (2 * gi) * bchunk + boff[q];
          *reinterpret_cast<uint4*>(d0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(d0 + bchunk) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        k1tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) k1tc::mbar_arrive(&sh.b_full[s]);
      };
      // software pipeline over ping-pong register buffers (no copies between tiles): the Philox
      // rounds of tile t + 1 (FMA-heavy pipe) and the decode / stores of tile t (ALU pipe) are
      // independent code in one block, so they interleave
      uint32_t a0[4], a1[4], a2[4], a3[4], b0[4], b1[4], b2[4], b3[4];
      philox(0, a0, a1, a2, a3);
      int t = 0;
      for (; t + 1 < ntiles; t += 2) {
        tile(t, a0, a1, a2, a3, b0, b1, b2, b3);
        tile(t + 1, b0, b1, b2, b3, a0, a1, a2, a3);
      }
      if (t < ntiles) tile(t, a0, a1, a2, a3, b0, b1, b2, b3);
    }
    // ---- end of pass: everyone learns whether the unit runs again
    k1tc::tc_fence_before();
    __syncthreads();
    k1tc::tc_fence_after();
    T0 += ntiles;   // (ndrain is tracked by the MMA warp and by the slicers; both advance alike)
    if (!sh.redo) break;
    __syncthreads();
    if (threadIdx.x == 0) sh.redo = 0;
    __syncthreads();
  }
  k1tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    k1tc::tc_fence_after();
    k1tc::tmem_dealloc<1>(tmem, 512);
  }
}

__global__ void fill_int_kernel(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// out = [scale (sum over ranges of part + colsum / 2) (ell x ncols, col-major); norms]
__global__ void k1f_reduce_kernel(const double* __restrict__ part, const double* __restrict__ npart,
                                  const double* __restrict__ cpart, Geom g, int ell, int ncols, double scale,
                                  double* __restrict__ out, unsigned* __restrict__ flags) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ny = static_cast<int64_t>(ell) * ncols;
  const int per_range = g.ncg * g.nsg;
  if (idx < ny) {
    const int j = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
    const int sgi = r / g.nu, rl = r % g.nu, cgi = j >> 5, jl = j & 31;
    double s = 0.0, c = 0.0;
#pragma unroll 8
    for (int rg = 0; rg < g.nranges; ++rg) {
      const int u = rg * per_range + cgi * g.nsg + sgi;
      s += part[(static_cast<int64_t>(u) * g.nu + rl) * 32 + jl];
      c += cpart[(rg * per_range + cgi * g.nsg) * 32 + jl];
    }
    out[idx] = scale * fma(0.5, c, s);
  } else if (idx < ny + ncols) {
    const int j = static_cast<int>(idx - ny);
    const int cgi = j >> 5, jl = j & 31;
    double s = 0.0;
#pragma unroll 8
    for (int rg = 0; rg < g.nranges; ++rg) s += npart[(rg * per_range + cgi * g.nsg) * 32 + jl];
    out[idx] = s;
    if (!isfinite(s)) atomicOr(flags, 1u);
  }
}

}  // namespace k1f

// ------------------------------------------------------------------ host side
// workspace: part (units x 512 x 32 fp64) | npart | cpart (units x 32 fp64); the exponent guesses
// (units x 32 int, kept across launches) live in a region of their own
inline size_t k1f_workspace_bytes() {
  return static_cast<size_t>(k1f::kMaxUnits) * 512 * 32 * sizeof(double) +
         2 * static_cast<size_t>(k1f::kMaxUnits) * 32 * sizeof(double);
}

inline bool k1f_call_ok(const K1TcArgs& a) {
  const int es = a.f64 ? 8 : 4;
  if (a.ncols < 1 || a.ncols > 64) return false;
  if (a.row_begin % 32 != 0) return false;
  if ((a.ld * es) % 16 != 0) return false;
  if (reinterpret_cast<uintptr_t>(a.X) % 16 != 0) return false;
  if (a.row_end - a.row_begin >= (int64_t(1) << 31)) return false;
  const k1f::Geom g = k1f::make_geom(a.ell, a.ncols, a.row_end - a.row_begin, a.f64, a.num_sms);
  if (g.nunits() > k1f::kMaxUnits) return false;
  if (g.smem > 227 * 1024) return false;
  return k1tc_encoder() != nullptr;
}

inline cudaError_t k1f_launch(const K1TcArgs& a, int* gE, cudaStream_t st, int* nlaunch) {
  *nlaunch = 0;
  const int64_t m_loc = a.row_end - a.row_begin;
  k1f::Geom g = k1f::make_geom(a.ell, a.ncols, m_loc, a.f64, a.num_sms);
  k1f::Keys keys;
  uint32_t k0 = a.key0, k1 = a.key1;
  for (int r = 0; r < 10; ++r) {
    keys.k0[r] = k0; keys.k1[r] = k1;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  double* part = reinterpret_cast<double*>(a.ws);
  double* npart = part + static_cast<size_t>(k1f::kMaxUnits) * 512 * 32;
  double* cpart = npart + static_cast<size_t>(k1f::kMaxUnits) * 32;
  CUtensorMap map;
  const int es = a.f64 ? 8 : 4;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m_loc), static_cast<cuuint64_t>(a.ncols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * es};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(g.xline / es), 32u};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = k1tc_encoder()(&map, a.f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                               const_cast<void*>(a.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  auto fn = a.f64 ? (g.brows == 512 ? k1f::k1f_kernel<double, 2> : k1f::k1f_kernel<double, 1>)
                  : (g.brows == 512 ? k1f::k1f_kernel<float, 2> : k1f::k1f_kernel<float, 1>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
  if (e == cudaSuccess)
    fn<<<g.nunits(), k1f::kThreads, g.smem, st>>>(map, a.ncols, keys, a.row_begin, m_loc, g, a.t0, a.t1, part, npart, cpart, gE,
                                                  a.flags);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return e;
  }
  *nlaunch += 1;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t nout = int64_t(a.ell) * a.ncols + a.ncols;
  k1f::k1f_reduce_kernel<<<static_cast<unsigned>((nout + 255) / 256), 256, 0, st>>>(part, npart, cpart, g, a.ell, a.ncols,
                                                                                  a.scale, a.out, a.flags);
  *nlaunch += 1;
  return cudaGetLastError();
}

}  // namespace oid
