// K1, tensor-core variant for sm_100a: Y_part = Z(:, slab) * X_blk and n_j = ||x_j||^2 in one
// read of X (Alg 3 steps 10 and 13), exact up to one rounding of each snapshot
// value to a per-column fixed point (56 bits for fp64 data, 48 bits for fp32 data).
//
// Why tensor cores and why exact: the sketch entries are Gauss-16 half-integers L = q + 1/2,
// q in [-111, 110] (reading R2), so Z = s (Q + 1/2) with Q int8 and
//     Z X = s (Q X + (1/2) 1 colsum(X)).
// Each value x of column j is cut into S two's-complement 8-bit digit planes of
// x_int = rint(x 2^F_j) (S = 7 for fp64, 6 for fp32; the column exponent F_j leaves kH bits of
// headroom above the first tile's maximum), and Q * X_digit runs on the 5th-generation tensor
// cores as tcgen05.mma kind::i8 with exact int32 accumulation in TMEM.  Y = s (sum_p 2^(8p-F_j)
// D_p + colsum_j / 2) is assembled in fp64.
//
// Work decomposition.  The rows of X are cut into slabs; a slab is processed by nh "units" of
// R = 128 TM NC sketch rows.  With NC = 2 a unit is a CTA pair (2-CTA cluster) running
// tcgen05.mma.cta_group::2 with M = 256: each CTA generates the sketch entries of its 128 rows
// of every M tile into its own TMEM (A operand) and converts only ITS half of the block's
// columns into digit planes (its half of the B operand, N split across the pair), so every
// value of X is loaded and converted exactly once per unit (ell = 512: once in total).
//
// CTA organisation (22 warps, one CTA per SM):
//   warp 0        TMA producer: cp.async.bulk.tensor 2D boxes (128 B of rows x BH columns,
//                 128-byte swizzle) of this CTA's columns into an NS-stage ring
//   warp 1        TMEM allocator; in the leader CTA the single-thread MMA issuer of the pair,
//                 which also sequences the accumulation epochs (below)
//   warps 2-9     sketch generator: Philox4x32-10 -> Gauss-16 nibbles -> int8 q by PRMT table
//                 lookups (levels held in 2 registers) -> tcgen05.st into TMEM (A operand);
//                 32 entries per Philox call
//   warps 10-17   digit slicer: X stage -> exponent check -> int8 digit planes (B operand), one
//                 tile at a time by all 256 threads; column norms and column sums in fp64
//   warps 18-21   epilogue: at the end of an accumulation epoch, tcgen05.ld of the int32
//                 accumulators -> fp64 partial sums (one warp per TMEM lane quarter)
// Accumulation epochs: a column's exponent is set by the first tile and raised (never lowered)
// when a later tile exceeds it; a raise in either CTA of the pair, or 1024 tiles (the int32
// bound: 65536 rows x 255 x 127 < 2^31), closes the epoch: the leader records the exponents in
// force, the accumulators are flushed to fp64 (exactly) by both CTAs' epilogues and
// accumulation restarts.  X is still read once.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
#include "sm100.cuh"
#include "k1_tc.cuh"

namespace oid {



namespace k1p {
using namespace k1tc;  // PTX helpers (sm100.cuh)
#ifndef K1P_WAIT
#define K1P_WAIT mbar_wait_nh
#endif

constexpr int kKTile = 128;         // data rows per pipeline stage (four 32-row Philox groups)
constexpr int kACols = kKTile / 4;  // TMEM columns of one M tile's sketch entries per stage
constexpr int kH = 6;               // exponent headroom bits over the first tile
constexpr int kEmin = -900;         // exponents are clamped here (data below 2^-900 lose bits)
constexpr int kNone = -100000;      // "no nonzero seen yet" exponent
constexpr int kMaxEpochTiles = 65536 / kKTile;   // int32 bound: 65536 rows x 255 x 127 < 2^31
constexpr int kMaxStages = 8;
constexpr int kMaxA = 4;
// Roles by warp id (24 warps; SMSP = id % 4, slot = id / 4): slot 0 epilogue, slots 1-2 generator
// (each role needs one warp per TMEM lane quarter = SMSP), slots 3-5 the slicer on SMSPs 0, 2, 3
// (8 warps), the TMA producer on SMSP 0 (slot 5) and the MMA issuer alone with the generator on
// SMSP 1 (slot 5): the issuer's dependent uniform-datapath sequences (elect / R2UR / UTCIMMA)
// would otherwise take the issue slots of the slicer warps sharing its SMSP, and every slicer warp
// must finish a tile before its B stage is complete.  The warp arbiter favours higher ids, so the
// issuer and the producer never wait behind the ALU-bound loops and the slicer sits above the
// generator (which runs up to four A stages ahead); the epilogue runs only at epoch ends.
constexpr int kEpiW = 4, kGenW = 8, kSlW = 8;
constexpr int kWarpsK1 = 24;
enum K1Role { kRoleEpi, kRoleGen, kRoleSlicer, kRoleTma, kRoleMma, kRoleIdle };
__device__ __forceinline__ int k1_role(int warp, int& idx) {
  const int sp = warp & 3, slot = warp >> 2;
  if (slot == 0) { idx = sp; return kRoleEpi; }
  if (slot <= 2) { idx = (slot - 1) * 4 + sp; return kRoleGen; }
  if (sp == 1) { idx = 0; return slot == 5 ? kRoleMma : kRoleIdle; }
  if (sp == 0) {
    if (slot == 5) { idx = 0; return kRoleTma; }
    idx = slot - 3; return kRoleSlicer;                      // 0, 1
  }
  idx = (sp == 2 ? 2 : 5) + (slot - 3); return kRoleSlicer;  // 2..4, 5..7
}
constexpr int kWMma = 21;           // k1_role(21) == kRoleMma (TMEM allocator in both CTAs)
constexpr int kMaxSlT = 32 * 8;     // slicer threads (maximum)
constexpr int kBarSl = 1;           // named barrier of the slicer warps
constexpr int kDbgTiles = 4096;
constexpr int kDbgRows = 12;
constexpr int kMaxSms = 160;

template <typename T> struct Fmt;
template <> struct Fmt<double> {
  static constexpr int kS = 6;      // digit planes: x_int in [-2^47, 2^47)
  static constexpr int kTop = 46;   // |x 2^F| < 2^46 whenever |x| < 2^e
};
template <> struct Fmt<float> {
  static constexpr int kS = 6;      // x_int in [-2^47, 2^47)
  static constexpr int kTop = 46;
};

// sum of the 4 byte products (signed a, unsigned b) + c
__device__ __forceinline__ int dp4a_su(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

struct Geom {
  int bpad;        // padded block width (16, 32, 64)
  int nc;          // CTAs per unit (1, or 2 = cta_group::2 pair)
  int TM;          // M tiles per unit (of 128 NC sketch rows)
  int R;           // sketch rows per unit
  int nh;          // units per slab
  int ellp;        // nh R (row stride of the partial sums)
  int nslabs;
  int64_t rows_per_slab;
  int ks;          // digit planes
  int nst;         // X / B pipeline stages
  int na;          // A (sketch entry) stages in TMEM
  int x_bytes, b_bytes;
  int smem;        // dynamic smem bytes
  long long* dbg;  // [kDbgRows][kDbgTiles] clock64 of CTA 0
  int exp;         // diagnostics only (OID_K1_EXP): bit 0 no Philox, bit 1 no conversion, bit 2 no TMEM store
};

inline Geom make_geom(int ell, int ncols, int64_t m_loc, bool f64, int num_sms) {
  Geom g{};
  g.bpad = ncols <= 16 ? 16 : (ncols <= 32 ? 32 : 64);
  g.ks = f64 ? Fmt<double>::kS : Fmt<float>::kS;
  const int ntot = g.bpad * g.ks;
  g.nc = (g.bpad >= 32 && ell > 128) ? 2 : 1;
  g.TM = (2 * ntot + 2 * 32 <= 512 && ell > 128 * g.nc) ? 2 : 1;
  g.R = 128 * g.TM * g.nc;
  g.nh = (ell + g.R - 1) / g.R;
  g.ellp = g.nh * g.R;
  g.na = std::min(kMaxA, (512 - g.TM * ntot) / (kACols * g.TM));
  const int bh = g.bpad / g.nc;
  g.x_bytes = kKTile * bh * (f64 ? 8 : 4);
  g.b_bytes = kKTile * g.ks * bh;
  g.nst = kMaxStages;
  while (g.nst > 2 && g.nst * (g.x_bytes + g.b_bytes) + 1024 > 200 * 1024) --g.nst;
  g.smem = g.nst * (g.x_bytes + g.b_bytes) + 1024;
  const int per_slab = g.nh * g.nc;
  g.nslabs = std::max(1, num_sms / per_slab);
  int64_t per = (m_loc + g.nslabs - 1) / g.nslabs;
  per = (per + kKTile - 1) / kKTile * kKTile;
  g.rows_per_slab = per;
  g.nslabs = static_cast<int>((m_loc + per - 1) / per);
  return g;
}

// Value bits of one element: the biased-exponent key and the bound e with |x| < 2^e (kNone = 0).
template <typename T> struct Bits;
template <> struct Bits<double> {
  static constexpr int kWords = 2;
  __device__ static __forceinline__ uint32_t key(const uint32_t* w) { return w[1] & 0x7FFFFFFFu; }
  __device__ static __forceinline__ int ebound(uint32_t k) {
    const int E = static_cast<int>(k >> 20);
    return E ? E - 1022 : (k ? -1021 : kNone);
  }
  __device__ static __forceinline__ double value(const uint32_t* w) {
    return __hiloint2double(static_cast<int>(w[1]), static_cast<int>(w[0]));
  }
};
template <> struct Bits<float> {
  static constexpr int kWords = 1;
  __device__ static __forceinline__ uint32_t key(const uint32_t* w) { return w[0] & 0x7FFFFFFFu; }
  __device__ static __forceinline__ int ebound(uint32_t k) {
    const int E = static_cast<int>(k >> 23);
    return E ? E - 126 : (k ? -125 : kNone);
  }
  __device__ static __forceinline__ double value(const uint32_t* w) { return static_cast<double>(__uint_as_float(w[0])); }
};

__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }

// 4x4 byte transpose: out[b] = byte b of w0..w3 (word k of out[b] holds byte b of w_k)
__device__ __forceinline__ void tr4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& b0, uint32_t& b1,
                                    uint32_t& b2, uint32_t& b3) {
  const uint32_t x0 = prmt(w0, w1, 0x5140), x1 = prmt(w0, w1, 0x7362);
  const uint32_t y0 = prmt(w2, w3, 0x5140), y1 = prmt(w2, w3, 0x7362);
  b0 = prmt(x0, y0, 0x5410);
  b1 = prmt(x0, y0, 0x7632);
  b2 = prmt(x1, y1, 0x5410);
  b3 = prmt(x1, y1, 0x7632);
}
__device__ __forceinline__ void tr4_lo3(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& b0, uint32_t& b1,
                                        uint32_t& b2) {
  const uint32_t x0 = prmt(w0, w1, 0x5140), y0 = prmt(w2, w3, 0x5140);
  const uint32_t x1 = prmt(w0, w1, 0x0062), y1 = prmt(w2, w3, 0x0062);
  b0 = prmt(x0, y0, 0x5410);
  b1 = prmt(x0, y0, 0x7632);
  b2 = prmt(x1, y1, 0x5410);
}
__device__ __forceinline__ void tr4_lo2(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& b0, uint32_t& b1) {
  const uint32_t x0 = prmt(w0, w1, 0x5140), y0 = prmt(w2, w3, 0x5140);
  b0 = prmt(x0, y0, 0x5410);
  b1 = prmt(x0, y0, 0x7632);
}

// Digit planes of 4 consecutive rows: out[p] = bytes p of x_int(row 0..3), x_int = rint(x 2^F).
// fp64 (7 planes): x 2^F = h 2^24 + l, h = rint(x 2^(F-24)), n = rint(l) in [-2^23, 2^23], all
// exact on the fp64 pipe (the 1.5 2^52 magic constant leaves the two's-complement integer in the
// low mantissa bits); x_int = (h + (n >> 24)) 2^24 + (n mod 2^24) = rint(x 2^F) exactly.
// fp32 (6 planes): one fma, |x_int| < 2^47 fits the 52-bit mantissa.
template <typename T>
__device__ __forceinline__ void digits4(const double (&x)[4], double p0, double phi, uint32_t (&out)[Fmt<T>::kS]) {
  constexpr double M = 6755399441055744.0;   // 1.5 2^52
  if constexpr (sizeof(T) == 8) {
    uint32_t nl[4], hh[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double t1 = __fma_rn(x[r], phi, M);
      const double hd = __dsub_rn(t1, M);
      const double v = __dmul_rn(x[r], p0);
      const double l = __fma_rn(hd, -16777216.0, v);
      const double t2 = __dadd_rn(l, M);
      const int n = __double2loint(t2);
      nl[r] = static_cast<uint32_t>(n);
      hh[r] = static_cast<uint32_t>(__double2loint(t1) + (n >> 31));
    }
    tr4_lo3(nl[0], nl[1], nl[2], nl[3], out[0], out[1], out[2]);
    tr4(hh[0], hh[1], hh[2], hh[3], out[3], out[4], out[5], out[6]);
  } else {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double t = __fma_rn(x[r], p0, M);
      lo[r] = static_cast<uint32_t>(__double2loint(t));
      hi[r] = static_cast<uint32_t>(__double2hiint(t));
    }
    tr4(lo[0], lo[1], lo[2], lo[3], out[0], out[1], out[2], out[3]);
    tr4_lo2(hi[0], hi[1], hi[2], hi[3], out[4], out[5]);
  }
}

struct Shared {
  uint64_t x_full[kMaxStages], x_empty[kMaxStages];
  uint64_t b_full[kMaxStages], b_empty[kMaxStages];
  uint64_t a_full[kMaxA], a_empty[kMaxA];
  uint64_t d_full, d_empty;
  uint32_t tmem_base;
  int estage[kMaxStages][64];   // leader: exponents of every column for the stage (a change = a raise)
  int erec[2][64];              // exponents of the epoch being flushed (by epoch parity)
  int elast[2];                 // 1: that flush is the last one
};

template <typename T, int BPAD, int TM, int NC>
__global__ void __launch_bounds__(32 * kWarpsK1, 1)
k1_tc_kernel(const __grid_constant__ CUtensorMap tmap, int ncols, int64_t row_begin, int64_t m_loc, int ell,
             uint32_t key0, uint32_t key1, uint32_t t0, uint32_t t1, Geom g, double* __restrict__ part,
             double* __restrict__ npart, double* __restrict__ cpart) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Shared sh;
  constexpr int KS = Fmt<T>::kS;
  constexpr int kTop = Fmt<T>::kTop;
  constexpr int BH = BPAD / NC;                     // columns converted by this CTA
  constexpr int NU = (KS - 1) * BH;                 // unsigned B rows per CTA
  constexpr int NB = KS * BH;                       // B rows per CTA
  constexpr int NTOT = KS * BPAD;                   // accumulator columns per M tile
  constexpr int NCH = (NC * NU + 255) / 256;        // unsigned MMAs per K step (N <= 256)
  constexpr int NUC = NU / NCH;                     // B rows per CTA per unsigned MMA
  static_assert(NU % NCH == 0 && NUC % 16 == 0, "unsigned MMA split");
  constexpr int MM = 128 * NC;                      // MMA M
  constexpr int ACOL0 = TM * NTOT;                  // first TMEM column of the A stages
  constexpr int R = 128 * TM * NC;
  constexpr int BOXR = 128 / sizeof(T);             // rows per 128-byte TMA line
  constexpr int NBOX = kKTile / BOXR;
  constexpr int RPT = kKTile * BH / (32 * kSlW);    // rows per slicer thread (4, 8, 16)
  constexpr int chB = NB * 16;                      // bytes per 16-byte K chunk of a B stage
  static_assert(RPT % 4 == 0 && (RPT <= 16 || RPT % 16 == 0), "slicer rows per thread");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int ridx = 0;
  const int role = k1_role(warp, ridx);
  const int h = NC == 2 ? static_cast<int>(cluster_rank()) : 0;
  const int unit_g = blockIdx.x / NC;
  const int slab = unit_g / g.nh, u = unit_g % g.nh;
  const int64_t r0 = static_cast<int64_t>(slab) * g.rows_per_slab;
  const int64_t r1 = min(m_loc, r0 + g.rows_per_slab);
  const int ntiles = static_cast<int>((r1 - r0 + kKTile - 1) / kKTile);
  const int NS = g.nst, NA = g.na;

  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* xbuf = base;
  uint8_t* bbuf = xbuf + NS * g.x_bytes;

  // leader-CTA addresses (shared::cluster) of the barriers and records the pair shares
  auto lead = [&](const void* p) -> uint32_t { return NC == 2 ? mapa(smem_u32(p), 0) : smem_u32(p); };
  auto peer = [&](const void* p) -> uint32_t { return mapa(smem_u32(p), static_cast<uint32_t>(h ^ 1)); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sh.x_full[s], 1);
      mbar_init(&sh.x_empty[s], kSlW);
      mbar_init(&sh.b_full[s], NC * kSlW);
      mbar_init(&sh.b_empty[s], 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(&sh.a_full[s], NC * kGenW);
      mbar_init(&sh.a_empty[s], 1);
    }
    mbar_init(&sh.d_full, h == 0 ? 1 + 32 : 2);
    mbar_init(&sh.d_empty, NC * kEpiW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWMma) tmem_alloc<NC>(&sh.tmem_base, 512);
  tc_fence_before();
  if constexpr (NC == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_base;

  if (role == kRoleTma) {
    // ---------------------------------------------------------------- TMA producer
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < ntiles; ++t) {
      if (t >= NS) K1P_WAIT(&sh.x_empty[s], ph ^ 1u);
      if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[4 * kDbgTiles + t] = clock64();
      if (g.exp & 512) { mbar_arrive_e(&sh.x_full[s]); if (++s == NS) { s = 0; ph ^= 1u; } continue; }
      mbar_arrive_expect_tx_e(&sh.x_full[s], g.x_bytes);
      uint8_t* dst = xbuf + s * g.x_bytes;
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        tma_load_2d_e(dst + bx * BH * 128, &tmap, &sh.x_full[s], static_cast<int>(r0 + int64_t(t) * kKTile + bx * BOXR),
                      h * BH);
      if (++s == NS) { s = 0; ph ^= 1u; }
    }
  } else if (role == kRoleMma) {
    if (h == 0) {
      // ---------------------------------------------------------------- MMA issuer of the unit
      const uint16_t mask = NC == 2 ? 3 : 1;
      const uint32_t bbase0 = smem_u32(bbuf);
      int cur0 = kNone, cur1 = kNone;      // exponents in force: columns lane, lane + 32
      int q = 0;
      // close accumulation epoch q: record the exponents in force (erec, elast) in both CTAs,
      // flush (both epilogues read D), wait until D is free again.  d_full of the leader: the MMA
      // commit + one arrival per issuer lane (after its local record stores); of the peer: the
      // commit + one arrive.expect_tx whose bytes the st.async record stores complete.
      auto close_epoch = [&](int last) {
        const int par = q & 1;
        sh.erec[par][lane] = cur0;
        if (BPAD > 32) sh.erec[par][lane + 32] = cur1;
        if (lane == 0) sh.elast[par] = last;
        mma_commit_mc<NC>(&sh.d_full, mask);
        if constexpr (NC == 2) {
          const uint32_t pbar = peer(&sh.d_full);
          st_async_u32(peer(&sh.erec[par][lane]), static_cast<uint32_t>(cur0), pbar);
          if (BPAD > 32) st_async_u32(peer(&sh.erec[par][lane + 32]), static_cast<uint32_t>(cur1), pbar);
          if (lane == 0) {
            st_async_u32(peer(&sh.elast[par]), static_cast<uint32_t>(last), pbar);
            mbar_arrive_expect_tx_remote(pbar, 4u * (BPAD > 32 ? 64 : 32) + 4u);
          }
        }
        mbar_arrive(&sh.d_full);
        K1P_WAIT(&sh.d_empty, par);                     // both epilogues have read D
        tc_fence_after();
        ++q;
      };
      int s = 0, sa = 0, ek = 0;
      uint32_t ph = 0, pha = 0;
      for (int t = 0; t < ntiles; ++t) {
        if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[9 * kDbgTiles + t] = clock64();
        K1P_WAIT(&sh.a_full[sa], pha);
        if (g.dbg && blockIdx.x == 0 && t < 2048 && lane == 0) g.dbg[9 * kDbgTiles + 2048 + t] = clock64();
        K1P_WAIT(&sh.b_full[s], ph);
        tc_fence_after();
        if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[2 * kDbgTiles + t] = clock64();
        // exponents of the stage (only ever raised): a change closes the accumulation epoch
        const int e0 = *reinterpret_cast<volatile int*>(&sh.estage[s][lane]);
        const int e1 = BPAD > 32 ? *reinterpret_cast<volatile int*>(&sh.estage[s][lane + 32]) : kNone;
        const bool chg = __any_sync(0xffffffffu, (lane < BPAD && e0 != cur0) || (BPAD > 32 && e1 != cur1));
        const bool newacc = chg || ek == 0;
        if (++ek == kMaxEpochTiles) ek = 0;
        if (newacc && t > 0) close_epoch(0);
        if (lane < BPAD) cur0 = e0;
        if (BPAD > 32) cur1 = e1;
        // one elected thread issues the tile's MMAs: descriptors are the stage's base descriptor
        // plus compile-time offsets (address field = byte address >> 4)
        if (!(g.exp & 256) && elect_one()) {
          const uint64_t bd0 = umma_desc(bbase0 + s * g.b_bytes, chB, 128);
          const uint32_t a0 = tmem + ACOL0 + sa * TM * kACols;
#pragma unroll
          for (int ks = 0; ks < kKTile / 32; ++ks) {
#pragma unroll
            for (int tm = 0; tm < TM; ++tm) {
              const uint32_t at = a0 + tm * kACols + ks * 8;
              const uint32_t acc = (newacc && ks == 0) ? 0u : 1u;
              const uint32_t dcol = tmem + tm * NTOT;
#pragma unroll
              for (int c = 0; c < NCH; ++c)
                mma_i8_ts_1<NC>(dcol + c * NC * NUC, at, bd0 + ((2 * ks * chB + (c * NUC / 8) * 128) >> 4),
                                idesc_i8m(MM, NC * NUC, false), acc);
              mma_i8_ts_1<NC>(dcol + NC * NU, at, bd0 + ((2 * ks * chB + (NU / 8) * 128) >> 4),
                              idesc_i8m(MM, NC * BH, true), acc);
            }
          }
        }
        __syncwarp();
        mma_commit_mc<NC>(&sh.a_empty[sa], mask);
        mma_commit_mc<NC>(&sh.b_empty[s], mask);
        if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[3 * kDbgTiles + t] = clock64();
        if (++s == NS) { s = 0; ph ^= 1u; }
        if (++sa == NA) { sa = 0; pha ^= 1u; }
      }
      close_epoch(1);
    }
  } else if (role == kRoleGen) {
    // ---------------------------------------------------------------- sketch generator
    // thread -> (sketch row, K chunks): TM = 2: row of M tile gw / 4, both 32-entry chunks;
    // TM = 1: chunk gw / 4 of the row.  TMEM lane quarter = warp % 4.
    const int gw = ridx;
    const int quarter = warp & 3;
    const int sl = gw >> 2;
    constexpr int NCALL = (kKTile / 32) * TM / 2;   // Philox calls (32 entries each) per thread per tile
    const int tm = TM == 2 ? sl : 0;
    const int kc0 = TM == 2 ? 0 : sl * NCALL;
    const int rl = tm * MM + h * 128 + quarter * 32 + lane;   // row within the unit
    const int r = u * R + rl;
    const bool warp_live = (u * R + tm * MM + h * 128 + quarter * 32) < ell;
    const uint64_t g32_0 = static_cast<uint64_t>((row_begin + r0) >> 5);
    const uint32_t a_bar = lead(&sh.a_full[0]);
    int sa = 0;
    uint32_t pha = 0;
    for (int t = 0; t < ntiles; ++t) {
      if (t >= NA) {
        K1P_WAIT(&sh.a_empty[sa], pha ^ 1u);
        tc_fence_after();
      }

      uint32_t pk[8 * NCALL];
      if (warp_live && !(g.exp & 1)) {
        uint32_t c0[NCALL], c1[NCALL], c2[NCALL], c3[NCALL];
#pragma unroll
        for (int ci = 0; ci < NCALL; ++ci) {
          c0[ci] = static_cast<uint32_t>(g32_0 + static_cast<uint64_t>(t) * (kKTile / 32) + kc0 + ci);
          c1[ci] = static_cast<uint32_t>(r);
          c2[ci] = 0u;
          c3[ci] = 0u;
        }
        uint32_t kk0 = key0, kk1 = key1;
#pragma unroll
        for (int rnd = 0; rnd < 10; ++rnd) {
#pragma unroll
          for (int ci = 0; ci < NCALL; ++ci) {
            uint32_t hi0, lo0, hi1, lo1;
            mulhilo32(0xD2511F53u, c0[ci], hi0, lo0);
            mulhilo32(0xCD9E8D57u, c2[ci], hi1, lo1);
            const uint32_t n0 = hi1 ^ c1[ci] ^ kk0;
            const uint32_t n2 = hi0 ^ c3[ci] ^ kk1;
            c0[ci] = n0; c1[ci] = lo1; c2[ci] = n2; c3[ci] = lo0;
          }
          kk0 += 0x9E3779B9u;
          kk1 += 0xBB67AE85u;
        }
#pragma unroll
        for (int ci = 0; ci < NCALL; ++ci) {
          const uint32_t ws[4] = {c0[ci], c1[ci], c2[ci], c3[ci]};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // 8 nibbles n = (sign, v): q = m_v (sign 0) or ~m_v = -m_v - 1 (sign 1), 4 per PRMT
            const uint32_t w = ws[k];
            const uint32_t wm = w & 0x77777777u;
            const uint32_t w4 = w * 16u;
            const uint32_t mlo = prmt(t0, t1, wm), mhi = prmt(t0, t1, __umulhi(wm, 0x10000u));
            const uint32_t slo = prmt(w, w4, 0x9D8Cu), shi = prmt(w, w4, 0xBFAEu);   // sign bytes 0x00/0xFF
            pk[8 * ci + 2 * k] = mlo ^ slo;
            pk[8 * ci + 2 * k + 1] = mhi ^ shi;
          }
        }
        if (r >= ell) {
#pragma unroll
          for (int k = 0; k < 8 * NCALL; ++k) pk[k] = 0u;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8 * NCALL; ++k) pk[k] = 0u;
      }
      const uint32_t ta = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + ACOL0 + (sa * TM + tm) * kACols + kc0 * 8;
      if (!(g.exp & 4)) {
        tmem_store<8 * NCALL>(ta, pk);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(a_bar + sa * 8);
      if (g.dbg && blockIdx.x == 0 && gw == 0 && lane == 0 && t < kDbgTiles) g.dbg[t] = clock64();
      // every generator warp of CTAs 0 and 1, first 512 tiles: rows 11 (CTA 0) and 9 (CTA 1)

      if (++sa == NA) { sa = 0; pha ^= 1u; }
    }
  } else if (role == kRoleSlicer) {
    // ---------------------------------------------------------------- digit slicer
    // No fp64 instruction on this path: on sm_100a DFMA/DADD stall while the tensor cores run
    // int8 MMAs (scripts/micro/mma_dfma.cu), so the digits, the column sums and the norms are all
    // formed with integer / IDP4A arithmetic (ALU and FMA pipes), and fp64 is used only when an
    // accumulator is flushed (exponent raise, every kFlushTiles tiles, end of the slab).
    // Warp w owns CPW columns of this CTA's half; lane -> (column c, rows rq RPT .. +RPT-1).
    constexpr int CPW = BH / kSlW;                  // columns per warp (2, 4, 8)
    constexpr int LPC = 32 / CPW;                   // lanes per column (16, 8, 4)
    const int sw = ridx;
    const int jc = sw * CPW + lane / LPC;            // column of this CTA's half
    const int rq = lane % LPC;                      // row group
    const int j = h * BH + jc;                      // column of the block
    const int row0 = rq * RPT;
    int ecur = kNone;                               // column exponent (|x| < 2^ecur), same in all its lanes
    double nrm64 = 0.0, cs64 = 0.0;                 // flushed sums (fp64)
    bool nonfinite = false;
    // integer accumulators in units of 2^-F (column sums) and 2^-2F (norms) of the current F
    int offk[11], diagk[7];                         // sum over rows of d_p d_q, p < q (k = p + q - 1), p = q (k = p)
    int csk[7];                                     // sum over rows of d_p (column sums of x_int by plane)
    uint32_t nE = 0, nH = 0;                        // nonzero count = nE - nH
#pragma unroll
    for (int k = 0; k < 11; ++k) offk[k] = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) { diagk[k] = 0; csk[k] = 0; }
    auto flush = [&](int e) {                       // e: exponent the accumulators were formed with
      if (e != kNone) {
        const int F = kTop - e;
        // exact integer combination (the plane terms cancel for negative values), then one
        // rounding: x_int^2 + x_int = x_int (x_int + 1) >= 0 summed, and sum x_int
        __int128 sq = 0, sm = 0;
#pragma unroll
        for (int p = 0; p < KS; ++p) {
          sq += static_cast<__int128>(diagk[p]) << (16 * p);
          sm += static_cast<__int128>(csk[p]) << (8 * p);
        }
#pragma unroll
        for (int k = 0; k < 2 * KS - 3; ++k) sq += static_cast<__int128>(offk[k]) << (8 * (k + 1) + 1);
        auto to_d = [](__int128 v) {
          const int64_t hi = static_cast<int64_t>(v >> 64);
          const uint64_t lo = static_cast<uint64_t>(v);
          return fma(static_cast<double>(hi), 18446744073709551616.0, static_cast<double>(lo));
        };
        if constexpr (sizeof(T) == 8) {
          // fp64 data: x_int = floor(x 2^F); norms and sums of x_int + 1/2 (unbiased)
          const double nnz = static_cast<double>(static_cast<int>(nE - nH));
          nrm64 += fma(0.25, nnz, to_d(sq + sm)) * pow2(-2 * F);
          cs64 += fma(0.5, nnz, to_d(sm)) * pow2(-F);
        } else {
          // fp32 data: x_int = trunc(x 2^F), exact for all but values 2^-15 below the bound
          nrm64 += to_d(sq) * pow2(-2 * F);
          cs64 += to_d(sm) * pow2(-F);
        }
      }
#pragma unroll
      for (int k = 0; k < 11; ++k) offk[k] = 0;
#pragma unroll
      for (int k = 0; k < 7; ++k) { diagk[k] = 0; csk[k] = 0; }
      nE = 0; nH = 0;
    };
    const uint32_t bfull_lead = lead(&sh.b_full[0]);
    const uint32_t estage_lead = lead(&sh.estage[0][j]);
    constexpr int NW = Bits<T>::kWords;
    constexpr int kFlushTiles = 256;
    // digits of x_int = floor(x 2^F) (fp64: ones' complement of the truncated magnitude for x < 0;
    // fp32: two's complement) with q = m >> r, m the 53-bit significand, r = 1075 - E - F >= 0;
    // accumulates the nonzero count, norms and column sums of the tile
    auto convert_acc = [&](const uint32_t (&vh)[RPT], const uint32_t (&vl)[RPT], const uint32_t (&ex)[RPT], int e,
                           uint32_t (&P)[RPT / 4][KS]) {
      const int cc = e == kNone ? 4096 : 1022 + e - (kTop - 53);
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        nE += ex[i];
        nH = __umulhi(ex[i], 0xFFFFFFFFu) + nH;                  // ex - 1 for ex >= 1, else 0
      }
#pragma unroll
      for (int q4 = 0; q4 < RPT / 4; ++q4) {
        uint32_t ql[4], qh[4];
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const int i = 4 * q4 + r4;
          const uint32_t r = min(static_cast<uint32_t>(cc - static_cast<int>(ex[i])), 63u);
          const uint32_t mh = (vh[i] & 0x000FFFFFu) | 0x00100000u;
          const uint64_t qm = ((static_cast<uint64_t>(mh) << 32) | vl[i]) >> r;   // two SHF (m < 2^53)
          const uint32_t lo2 = static_cast<uint32_t>(qm), hi1 = static_cast<uint32_t>(qm >> 32);
          const uint32_t sg = static_cast<uint32_t>(__mulhi(static_cast<int>(vh[i]), 2));   // x < 0 ? ~0 : 0
          if constexpr (sizeof(T) == 8) {
            ql[r4] = lo2 ^ sg;
            qh[r4] = hi1 ^ sg;
          } else {
            asm("sub.cc.u32 %0, %2, %4;\n\tsubc.u32 %1, %3, %4;"
                : "=r"(ql[r4]), "=r"(qh[r4]) : "r"(lo2 ^ sg), "r"(hi1 ^ sg), "r"(sg));
          }
        }
        tr4(ql[0], ql[1], ql[2], ql[3], P[q4][0], P[q4][1], P[q4][2], P[q4][3]);
        if constexpr (KS == 7) tr4_lo3(qh[0], qh[1], qh[2], qh[3], P[q4][4], P[q4][5], P[q4][6]);
        else tr4_lo2(qh[0], qh[1], qh[2], qh[3], P[q4][4], P[q4][5]);
        // norms: sum over the 4 rows of d_p d_q by IDP4A (planes 0..KS-2 unsigned, KS-1 signed)
        if (!(g.exp & 64))
#pragma unroll
        for (int p = 0; p < KS; ++p) {
#pragma unroll
          for (int qq = p; qq < KS; ++qq) {
            if (qq == p) {
              if (p == KS - 1) diagk[p] = __dp4a(static_cast<int>(P[q4][p]), static_cast<int>(P[q4][p]), diagk[p]);
              else diagk[p] = static_cast<int>(__dp4a(P[q4][p], P[q4][p], static_cast<unsigned>(diagk[p])));
            } else {
              int& acc = offk[p + qq - 1];
              if (qq == KS - 1) acc = dp4a_su(P[q4][qq], P[q4][p], acc);
              else acc = static_cast<int>(__dp4a(P[q4][p], P[q4][qq], static_cast<unsigned>(acc)));
            }
          }
          if (p == KS - 1) csk[p] = __dp4a(static_cast<int>(P[q4][p]), 0x01010101, csk[p]);
          else csk[p] = static_cast<int>(__dp4a(P[q4][p], 0x01010101u, static_cast<unsigned>(csk[p])));
        }
      }
    };
    int s = 0;
    uint32_t ph = 0;
    int since_flush = 0;
    // two tiles per iteration: the barrier waits, shared-memory loads and the proxy fence of the
    // pair overlap (a warp's work per tile is short; its latencies are not)
    constexpr int G = 1;
    for (int t = 0; t < ntiles; t += G) {
      const int cnt = min(G, ntiles - t);
      const bool dbgt = g.dbg && blockIdx.x == 0 && sw == (g.exp >> 12) && lane == 0 && t < kDbgTiles;
      if (dbgt) g.dbg[5 * kDbgTiles + t] = clock64();
      int sg_[G];
      uint32_t pg_[G];
      sg_[0] = s; pg_[0] = ph;
      if constexpr (G > 1) {
        sg_[1] = s + 1 == NS ? 0 : s + 1;
        pg_[1] = s + 1 == NS ? ph ^ 1u : ph;
      }
      uint32_t w[G][RPT * NW];
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (gi < cnt) {
          K1P_WAIT(&sh.x_full[sg_[gi]], pg_[gi]);
          // RPT rows of column jc from the 128B-swizzled boxes (16-byte chunks of 16 / sizeof(T) rows)
          const uint8_t* xs = xbuf + sg_[gi] * g.x_bytes + jc * 128;
#pragma unroll
          for (int c = 0; c < RPT * NW / 4; ++c) {
            const int rc = row0 + c * (16 / static_cast<int>(sizeof(T)));
            const int cl = (rc % BOXR) * static_cast<int>(sizeof(T)) / 16;
            const uint4 v = *reinterpret_cast<const uint4*>(xs + (rc / BOXR) * BH * 128 + ((cl ^ (jc & 7)) << 4));
            w[gi][4 * c + 0] = v.x; w[gi][4 * c + 1] = v.y; w[gi][4 * c + 2] = v.z; w[gi][4 * c + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int c = 0; c < RPT * NW; ++c) w[gi][c] = 0u;
        }
      }
      if (dbgt) g.dbg[6 * kDbgTiles + t] = clock64();
      // release the X stages only once the loads have landed in registers (the arrive depends on
      // their values through an opaque OR): otherwise the next TMA load can overwrite the stage
      // before the shared-memory loads read it (a WAR race across proxies, observed in K1F)
      uint32_t tok = 0u;
#pragma unroll
      for (int gi = 0; gi < G; ++gi)
#pragma unroll
        for (int c = 0; c < RPT * NW; ++c) tok |= w[gi][c];
      asm volatile("or.b32 %0, %0, 1;" : "+r"(tok));
      __syncwarp();
      if (lane == 0 && tok != 0u) {
#pragma unroll
        for (int gi = 0; gi < G; ++gi)
          if (gi < cnt) mbar_arrive(&sh.x_empty[sg_[gi]]);
      }
      // fp64-layout words (hi, lo), biased exponents, and the exponent check of each tile in order;
      // a raise at the pair's second tile flushes the accumulators only after the first tile
      uint32_t vh[G][RPT], vl[G][RPT], ex[G][RPT];
      int ecg[G];
      bool pending = false;
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        uint32_t emx = 0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          if constexpr (sizeof(T) == 8) {
            vh[gi][i] = w[gi][2 * i + 1];
            vl[gi][i] = w[gi][2 * i];
            ex[gi][i] = __umulhi(vh[gi][i] * 2u, 2048u);         // (hi >> 20) & 0x7ff (FMA pipe)
          } else {
            const uint32_t b = w[gi][i];
            const uint32_t e8 = __umulhi(b * 2u, 256u);          // fp32 biased exponent
            ex[gi][i] = e8 ? e8 + 896u : 0u;                     // as an fp64 exponent (0: zero / subnormal)
            vh[gi][i] = (b & 0x80000000u) | (ex[gi][i] << 20) | ((b >> 3) & 0xFFFFFu);
            vl[gi][i] = b << 29;
          }
          emx = max(emx, ex[gi][i]);
        }
        // exponent bound of this lane's values: |x| < 2^(emx - 1022); a column raise is warp-local
        const int eb = emx ? static_cast<int>(emx) - 1022 : kNone;
        const int viol = (eb != kNone) && (ecur == kNone || eb > ecur);
        if (__any_sync(0xffffffffu, viol)) {
          int em = eb;
#pragma unroll
          for (int o = LPC / 2; o > 0; o >>= 1) em = max(em, __shfl_xor_sync(0xffffffffu, em, o));
          if (em != kNone && (ecur == kNone || em > ecur)) {
            if (gi == 0) {
              flush(ecur);
              since_flush = 0;
            } else {
              pending = true;
            }
            if (g.dbg && blockIdx.x == 0 && (lane % LPC) == 0)
              atomicAdd(reinterpret_cast<unsigned long long*>(&g.dbg[10 * kDbgTiles + 4000 + sw]), 1ull);
            if (em >= 1025) nonfinite = true;                    // Inf / NaN (exponent 2047)
            ecur = max(kEmin, em + kH);
          }
        }
        ecg[gi] = ecur;
      }
      if (dbgt) g.dbg[10 * kDbgTiles + t] = clock64();
#pragma unroll
      for (int gi = 0; gi < G; ++gi)
        if (gi < cnt && t + gi >= NS) K1P_WAIT(&sh.b_empty[sg_[gi]], pg_[gi] ^ 1u);
      if (dbgt) g.dbg[7 * kDbgTiles + t] = clock64();
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (gi < cnt) {
          if (gi == 1 && pending) {
            flush(ecg[0]);
            since_flush = 0;
          }
          uint32_t P[RPT / 4][KS];
          if (g.exp & 128) {
#pragma unroll
            for (int q4 = 0; q4 < RPT / 4; ++q4)
#pragma unroll
              for (int p = 0; p < KS; ++p) P[q4][p] = vl[gi][q4] ^ vh[gi][p % RPT];
          } else {
            convert_acc(vh[gi], vl[gi], ex[gi], ecg[gi], P);
          }
#pragma unroll
          for (int p = 0; p < KS; ++p) {
            const int n = p * BH + jc;
            uint8_t* dst = bbuf + sg_[gi] * g.b_bytes + (row0 / 16) * chB + (n >> 3) * 128 + (n & 7) * 16 + (row0 % 16);
            if constexpr (RPT == 4) *reinterpret_cast<uint32_t*>(dst) = P[0][p];
            else if constexpr (RPT == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(P[0][p], P[1][p]);
            else {
#pragma unroll
              for (int c16 = 0; c16 < RPT / 16; ++c16)
                *reinterpret_cast<uint4*>(dst + c16 * chB) =
                    make_uint4(P[4 * c16][p], P[4 * c16 + 1][p], P[4 * c16 + 2][p], P[4 * c16 + 3][p]);
            }
          }
          // this column's exponent for the stage (CTA 1: st.async completing 4 transaction bytes on
          // the leader's b_full, whose expected bytes the leader's first slicer warp posts)
          if (rq == 0) {
            if (h == 0) sh.estage[sg_[gi]][j] = ecg[gi];
            else st_async_u32(estage_lead + sg_[gi] * 64 * 4, static_cast<uint32_t>(ecg[gi]), bfull_lead + sg_[gi] * 8);
          }
        }
      }
      since_flush += cnt;
      if (since_flush >= kFlushTiles) { flush(ecur); since_flush = 0; }
      if (dbgt) g.dbg[8 * kDbgTiles + t] = clock64();
      if (!(g.exp & 32)) fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int gi = 0; gi < G; ++gi) {
          if (gi < cnt) {
            if (NC == 2 && h == 0 && sw == 0) mbar_arrive_expect_tx(&sh.b_full[sg_[gi]], 4 * BH);
            else mbar_arrive_remote(bfull_lead + sg_[gi] * 8);
          }
        }
      }
      if (dbgt) g.dbg[1 * kDbgTiles + t] = clock64();
      if (g.dbg && blockIdx.x < 2 && lane == 0 && t < 256) g.dbg[11 * kDbgTiles + (blockIdx.x * 8 + sw) * 256 + t] = clock64();
      const int sl = sg_[cnt - 1];
      ph = sl + 1 == NS ? pg_[cnt - 1] ^ 1u : pg_[cnt - 1];
      s = sl + 1 == NS ? 0 : sl + 1;
    }
    flush(ecur);
    // norms and column sums: the lanes of column jc combine in a fixed butterfly order
#pragma unroll
    for (int o = LPC / 2; o > 0; o >>= 1) {
      nrm64 += __shfl_xor_sync(0xffffffffu, nrm64, o);
      cs64 += __shfl_xor_sync(0xffffffffu, cs64, o);
    }
    const bool nf = __any_sync(0xffffffffu, nonfinite) && nonfinite;
    if (u == 0 && rq == 0 && j < ncols) {
      npart[static_cast<int64_t>(slab) * BPAD + j] = nf ? __longlong_as_double(0x7ff8000000000000LL) : nrm64;
      cpart[static_cast<int64_t>(slab) * BPAD + j] = cs64;
    }
  } else if (role == kRoleEpi) {
    // ---------------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    const uint32_t dempty_lead = lead(&sh.d_empty);
    for (int qe = 0;; ++qe) {
      const int par = qe & 1;
      // one warp polls the barrier, the others sleep on a named barrier (no mbarrier polling)
      if (ridx == 0) K1P_WAIT(&sh.d_full, par);
      named_bar(2, 32 * kEpiW);
      tc_fence_after();
      const int last = *reinterpret_cast<volatile int*>(&sh.elast[par]);
#pragma unroll 1
      for (int tm = 0; tm < TM; ++tm) {
        const int r = u * R + tm * MM + h * 128 + quarter * 32 + lane;
#pragma unroll 1
        for (int jb = 0; jb < BPAD; jb += 16) {
          double acc[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) acc[k] = 0.0;
          const int hb = jb / BH, jcb = jb % BH;
#pragma unroll 1
          for (int p = KS - 1; p >= 0; --p) {
            int col;
            if (p < KS - 1) {
              const int n = p * BH + jcb;
              col = (n / NUC) * NC * NUC + hb * NUC + n % NUC;
            } else {
              col = NC * NU + hb * BH + jcb;
            }
            uint32_t v[16];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + tm * NTOT + col;
            OID_TMEM_LD16(taddr, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const double wgt = pow2(8 * p);
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] = fma(static_cast<double>(static_cast<int>(v[k])), wgt, acc[k]);
          }
          if (r < ell) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int jj = jb + k;
              if (jj >= ncols) continue;
              const int e = *reinterpret_cast<volatile int*>(&sh.erec[par][jj]);
              const double val = (e == kNone) ? 0.0 : acc[k] * pow2(e - kTop);
              double* dst = part + (static_cast<int64_t>(slab) * BPAD + jj) * g.ellp + r;
              *dst = (qe == 0) ? val : *dst + val;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(dempty_lead);
      if (last) break;
    }
  }
  tc_fence_before();
  if constexpr (NC == 2) cluster_sync(); else __syncthreads();
  if (warp == kWMma) {
    tc_fence_after();
    tmem_dealloc<NC>(tmem, 512);
  }
}

// out = [scale * (sum over slabs of part + colsum / 2) (ell x ncols, col-major); norms]
__global__ void k1_tc_reduce_kernel(const double* __restrict__ part, const double* __restrict__ npart,
                                    const double* __restrict__ cpart, Geom g, int ell, int ncols, double scale,
                                    double* __restrict__ out, unsigned* __restrict__ flags) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ny = static_cast<int64_t>(ell) * ncols;
  if (idx < ny) {
    const int j = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
    double s = 0.0, c = 0.0;
#pragma unroll 8   // the loads of several slabs in flight; the sums keep their fixed order
    for (int sl = 0; sl < g.nslabs; ++sl) {
      s += part[(static_cast<int64_t>(sl) * g.bpad + j) * g.ellp + r];
      c += cpart[static_cast<int64_t>(sl) * g.bpad + j];
    }
    out[idx] = scale * fma(0.5, c, s);
  } else if (idx < ny + ncols) {
    const int j = static_cast<int>(idx - ny);
    double s = 0.0;
#pragma unroll 8
    for (int sl = 0; sl < g.nslabs; ++sl) s += npart[static_cast<int64_t>(sl) * g.bpad + j];
    out[idx] = s;
    if (!isfinite(s)) atomicOr(flags, 1u);
  }
}

}  // namespace k1p

// ------------------------------------------------------------------ host side
inline size_t k1p_workspace_bytes(int /*ell*/, int /*b_max*/, int64_t /*m_loc*/, bool /*f64*/) {
  // partial sums: nslabs * bpad * ellp doubles with nslabs * nh * nc <= SMs and ellp = nh * 128 TM nc
  return static_cast<size_t>(k1p::kMaxSms) * 256 * 64 * sizeof(double) +
         2 * static_cast<size_t>(k1p::kMaxSms) * 64 * sizeof(double) + 1024;
}

inline bool k1p_supported(int ell, int b_max, bool /*f64*/) { return ell >= 1 && ell <= 1024 && b_max <= 64; }

// Whether this call can use the tensor-core kernel (alignment rules of TMA and the Philox groups).
inline bool k1p_call_ok(const K1TcArgs& a) {
  const int es = a.f64 ? 8 : 4;
  if (a.ncols < 1 || a.ncols > 64) return false;
  if (a.row_begin % 32 != 0) return false;        // Philox blocks of 32 rows (reading R2)
  if ((a.ld * es) % 16 != 0) return false;
  if (reinterpret_cast<uintptr_t>(a.X) % 16 != 0) return false;
  if (a.row_end - a.row_begin >= (int64_t(1) << 31)) return false;
  if (a.num_sms > k1p::kMaxSms) return false;
  // two stages of X and digit planes must fit beside the static shared state (f64, 33..64
  // columns on one CTA does not)
  if (k1p::make_geom(a.ell, a.ncols, a.row_end - a.row_begin, a.f64, a.num_sms).smem > 200 * 1024) return false;
  return k1tc_encoder() != nullptr;
}

template <typename T, int BPAD, int TM, int NC>
inline cudaError_t k1p_launch_t(const CUtensorMap& map, const K1TcArgs& a, const k1p::Geom& g, cudaStream_t st,
                                 double* part, double* npart, double* cpart) {
  auto fn = k1p::k1_tc_kernel<T, BPAD, TM, NC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();   // consumed here: a later call must not report it again
    return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(g.nslabs * g.nh * NC));
  cfg.blockDim = dim3(32 * k1p::kWarpsK1);
  cfg.dynamicSmemBytes = static_cast<size_t>(g.smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, map, a.ncols, a.row_begin, a.row_end - a.row_begin, a.ell, a.key0, a.key1, a.t0,
                            a.t1, g, part, npart, cpart);
}

template <typename T>
inline cudaError_t k1p_dispatch(const CUtensorMap& map, const K1TcArgs& a, const k1p::Geom& g, cudaStream_t st,
                                 double* part, double* npart, double* cpart) {
#define K1_CASE(BP, TMV, NCV) \
  if (g.bpad == BP && g.TM == TMV && g.nc == NCV) return k1p_launch_t<T, BP, TMV, NCV>(map, a, g, st, part, npart, cpart)
  K1_CASE(16, 1, 1);
  K1_CASE(16, 2, 1);
  K1_CASE(32, 1, 1);
  K1_CASE(32, 1, 2);
  K1_CASE(32, 2, 2);
  K1_CASE(64, 1, 1);
  K1_CASE(64, 1, 2);
#undef K1_CASE
  return cudaErrorInvalidConfiguration;
}

inline cudaError_t k1p_launch(const K1TcArgs& a, cudaStream_t st, int* nlaunch) {
  *nlaunch = 0;
  const int64_t m_loc = a.row_end - a.row_begin;
  k1p::Geom g = k1p::make_geom(a.ell, a.ncols, m_loc, a.f64, a.num_sms);
  g.dbg = a.dbg;
  g.exp = getenv("OID_K1_EXP") ? atoi(getenv("OID_K1_EXP")) : 0;
  CUtensorMap map;
  const int es = a.f64 ? 8 : 4;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m_loc), static_cast<cuuint64_t>(a.ncols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * es};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(g.bpad / g.nc)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = k1tc_encoder()(&map, a.f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                               const_cast<void*>(a.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  double* part = reinterpret_cast<double*>(a.ws);
  double* npart = part + static_cast<size_t>(k1p::kMaxSms) * 256 * 64;
  double* cpart = npart + static_cast<size_t>(k1p::kMaxSms) * 64;
  cudaError_t e = a.f64 ? k1p_dispatch<double>(map, a, g, st, part, npart, cpart)
                        : k1p_dispatch<float>(map, a, g, st, part, npart, cpart);
  *nlaunch += 1;
  if (e != cudaSuccess) return e;
  const int64_t nout = int64_t(a.ell) * a.ncols + a.ncols;
  k1p::k1_tc_reduce_kernel<<<static_cast<unsigned>((nout + 255) / 256), 256, 0, st>>>(part, npart, cpart, g, a.ell,
                                                                                     a.ncols, a.scale, a.out, a.flags);
  *nlaunch += 1;
  return cudaGetLastError();
}

}  // namespace oid
