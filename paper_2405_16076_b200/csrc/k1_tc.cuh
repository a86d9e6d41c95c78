// K1, tensor-core variant for sm_100a: Y_part = Z(:, slab) * X_blk and n_j = ||x_j||^2 in one
// read of X (Alg 3 steps 10 and 13), exact to fp64 rounding.
//
// Why exact: the sketch entries are Gauss-16 half-integers L = q + 1/2, q in [-111, 110]
// (reading R2), so Z = s (Q + 1/2) with Q int8 and Z X = s (Q X + (1/2) 1 colsum(X)).  Each snapshot value x is cut into S = 7 two's-complement 8-bit digit
// planes of a per-column fixed-point integer x_int = round(x * 2^F_j) (56-bit fixed point; the
// column exponent F_j leaves kHeadroom bits above the first tile's maximum), and Q * X_digit
// runs on the 5th-generation tensor cores as tcgen05.mma kind::i8 with exact int32 accumulation
// in TMEM.  Y = s * (sum_p 2^(8p - F_j) * D_p + colsum_j / 2) is assembled in fp64.
//
// CTA organisation (one CTA per SM, 14 warps; one work unit = row slab x 128*TM sketch rows):
//   warp 0        TMA producer: cp.async.bulk.tensor 2D boxes (128 B x BPAD, 128B swizzle) of X
//   warp 1        TMEM allocator + single-thread tcgen05.mma issuer (A from TMEM, B from smem)
//   warps 6-13    digit slicer: X stage -> per-column exponent check -> int8 digit planes (B op.),
//                 8 rows per thread, software-pipelined one tile ahead (the exponent decision
//                 for tile t+1 is made while tile t is converted); also the epilogue at
//                 accumulation-epoch ends (tcgen05.ld of the int32 accumulators, fp64 partials)
//   warps 2-5     sketch generator: Philox4x32-10 -> Gauss-16 nibbles -> int8 q by two PRMT
//                 table lookups per 4 entries (levels held in 2 registers) -> tcgen05.st into
//                 TMEM (A operand); 32 entries per Philox call
// Per-column exponents start from the first tile of the unit plus kHeadroom bits; if a later
// tile exceeds them, or 1024 tiles have accumulated (int32 overflow bound: 65536 rows x 255 x
// 127 < 2^31), the accumulators are flushed to fp64 (exactly) and accumulation restarts
// ("accumulation epochs"), so X is still read once.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
#include "sm100.cuh"

namespace oid {

struct K1TcArgs {
  const void* X;
  int64_t ld;
  int ncols;
  int64_t row_begin, row_end;
  int ell;
  uint32_t key0, key1;
  double scale;
  bool f64;
  char* ws;
  double* out;
  unsigned* flags;
  int num_sms;
  uint32_t t0, t1;   // Gauss-16 magnitudes m_0..m_3, m_4..m_7 as bytes (reading R2)
  long long* dbg;     // diagnostics (may be null): per-tile role timestamps of CTA 0
  const uint4* omega; // stored sketch entries (NEXT-3, may be null): the Philox words of every
                      // (32-row group g of the shard, sketch row r) at omega[g * ell + r]
};

namespace k1tc {

constexpr int kWarps = 14;
constexpr int kThreads = 32 * kWarps;
constexpr int kKTile = 64;          // data rows per pipeline stage
constexpr int kS = 7;               // digit planes (56-bit fixed point)
constexpr int kTop = 55;            // |x_int| < 2^55
constexpr int kHeadroom = 8;        // exponent headroom bits over the first tile
constexpr int kEmin = -900;         // exponents are clamped here (data below 2^-900 lose bits)
constexpr int kNone = -100000;      // "no nonzero seen yet" exponent
constexpr int kMaxEpochTiles = 1024;
constexpr int kMaxStages = 4;
// Roles by warp id.  The slicer is the critical path and the warp arbiter favours higher warp
// ids, so the slicer gets the top warps and the (run-ahead) generator the ones below.
constexpr int kGen0 = 2, kSlicer0 = 6;    // first warp of each role
constexpr int kSlW = 8;                   // slicer warps (6..13)
constexpr int kSlT = 32 * kSlW;           // slicer threads

struct Geom {
  int bpad;      // padded block width (16, 32, 64)
  int TM;        // M tiles (of 128 sketch rows) per CTA
  int rows;      // 128 * TM
  int ntot;      // bpad * kS accumulator columns per M tile
  int x_bytes, b_bytes;   // per stage
  int nst;       // pipeline stages of X / B
  int smem;      // dynamic smem bytes
  int nhalves;   // sketch-row slices
  int nslabs;
  int64_t rows_per_slab;
  long long* dbg;  // [5][kDbgTiles] clock64 of CTA 0: A ready, B ready, MMA start, MMA issued, TMA issue
  int exp;         // diagnostics only (OID_K1_EXP): 1 = skip the Philox generation, 2 = skip the digit conversion
  const uint4* omega;   // stored Philox words (NEXT-3) or null: generate in registers
  int64_t g0;           // first 32-row group of the shard
};
constexpr int kDbgTiles = 4096;
constexpr int kDbgRows = 10;

inline Geom make_geom(int ell, int ncols, int64_t m_loc, bool f64, int num_sms) {
  Geom g{};
  g.bpad = ncols <= 16 ? 16 : (ncols <= 32 ? 32 : 64);
  g.ntot = g.bpad * kS;
  // TMEM: TM accumulators of ntot columns + 2 A stages of TM x 16 columns <= 512
  g.TM = (ell > 128 && 2 * g.ntot + 64 <= 512) ? 2 : 1;
  g.rows = 128 * g.TM;
  g.x_bytes = kKTile * g.bpad * (f64 ? 8 : 4);
  g.b_bytes = g.ntot * kKTile;
  g.nst = kMaxStages;
  while (g.nst > 2 && g.nst * (g.x_bytes + g.b_bytes) + 1024 + 4096 > 225 * 1024) --g.nst;
  g.smem = g.nst * (g.x_bytes + g.b_bytes) + 1024;
  g.nhalves = (ell + g.rows - 1) / g.rows;
  g.nslabs = std::max(1, num_sms / g.nhalves);
  int64_t per = (m_loc + g.nslabs - 1) / g.nslabs;
  per = (per + kKTile - 1) / kKTile * kKTile;
  g.rows_per_slab = per;
  g.nslabs = static_cast<int>((m_loc + per - 1) / per);
  return g;
}

// Value bits of one element: x = (-1)^neg * m * 2^e2 (m < 2^53), plus the frexp-style exponent
// key (biased exponent field, 0 for zero).
template <typename T> struct Bits;
template <> struct Bits<double> {
  static constexpr int kPer16 = 8;   // 16-byte chunks per 16 rows
  __device__ static __forceinline__ uint32_t key(uint32_t hi) { return hi & 0x7FFFFFFFu; }
  // exponent bound e (|x| < 2^e) from the max key of a group; kNone if all zero
  __device__ static __forceinline__ int ebound(uint32_t k) {
    const int E = static_cast<int>(k >> 20);
    return E ? E - 1022 : (k ? -1021 : kNone);
  }
};
template <> struct Bits<float> {
  static constexpr int kPer16 = 4;
  __device__ static __forceinline__ uint32_t key(uint32_t b) { return b & 0x7FFFFFFFu; }
  __device__ static __forceinline__ int ebound(uint32_t k) {
    const int E = static_cast<int>(k >> 23);
    return E ? E - 126 : (k ? -125 : kNone);
  }
};

// x_int = round(x * 2^F) as a 64-bit two's-complement integer, for |x * 2^F| < 2^55, on the
// fp64 pipe: hi = floor(x 2^(F-32)) and lo = x 2^F - hi 2^32 in [0, 2^32) are exact; lo is
// rounded to nearest by the 2^52 magic add (a carry out of lo goes into hi).
// p32 = 2^(F-32), p0 = 2^F, both 0 for an all-zero column.
__device__ __forceinline__ void fixpt(double x, double p32, double p0, uint32_t& lo, uint32_t& hi, double& vout) {
  const double M = 6755399441055744.0;             // 1.5 * 2^52
  const double t1 = __fma_rd(x, p32, M);            // M + floor(x 2^(F-32))
  const double hd = t1 - M;                         // exact
  const double v = x * p0;                          // exact (power-of-two scaling)
  vout = v;
  const double l = fma(hd, -4294967296.0, v);       // exact, in [0, 2^32)
  const double t2 = l + 4503599627370496.0;         // 2^52 + rint(l)
  const uint32_t t2h = static_cast<uint32_t>(__double2hiint(t2));
  lo = static_cast<uint32_t>(__double2loint(t2));
  hi = static_cast<uint32_t>(__double2loint(t1)) + (t2h & 1u);
}

struct Shared {
  uint64_t x_full[kMaxStages], x_empty[kMaxStages];
  uint64_t b_full[kMaxStages], b_empty[kMaxStages];
  uint64_t a_full[2], a_empty[2];
  uint64_t d_full, d_empty;
  uint32_t tmem_base;
  int bflags[kMaxStages];
  int ecur[2][64];
  int ehist[4][64];
  uint64_t tok[2];
  int egen, qsh;
  int epi_done;      // epilogue warps finished (4 per accumulation epoch, in epoch order)
  int emax[2][4][2][64];
  double nrm[kSlT];
  double csum[kSlT];
};

// Load the 8 values (rows 16 c16 + 8 h .. +7) of column j from a 128B-swizzled X stage as raw
// bits (fp64: 16 words, fp32: 8 words).
template <typename T, int BPAD>
__device__ __forceinline__ void load_half(const uint8_t* xs, int j, int c16, int h, uint32_t (&w)[sizeof(T) == 8 ? 16 : 8]) {
  if constexpr (sizeof(T) == 8) {
    const uint8_t* base = xs + (c16 * BPAD + j) * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + (((4 * h + q) ^ (j & 7)) << 4));
      w[4 * q + 0] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  } else {
    const uint8_t* base = xs + ((c16 >> 1) * BPAD + j) * 128;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int qq = (c16 & 1) * 4 + 2 * h + q;
      const uint4 v = *reinterpret_cast<const uint4*>(base + ((qq ^ (j & 7)) << 4));
      w[4 * q + 0] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  }
}

template <typename T, int BPAD, int TM, bool OMEGA>
__global__ void __launch_bounds__(kThreads, 1)
k1_tc_kernel(const __grid_constant__ CUtensorMap tmap, int ncols, int64_t row_begin, int64_t m_loc, int ell,
             uint32_t key0, uint32_t key1, uint32_t t0, uint32_t t1, Geom g, double* __restrict__ part,
             double* __restrict__ npart, double* __restrict__ cpart) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Shared sh;
  constexpr bool kF64 = sizeof(T) == 8;
  constexpr int NTOT = BPAD * kS;
  constexpr int ROWS = 128 * TM;
  constexpr int ACOL0 = TM * NTOT;                 // first TMEM column of the A stages
  constexpr int BOX_ROWS = 128 / sizeof(T);
  constexpr int NBOX = kKTile / BOX_ROWS;
  constexpr int NHU = 8 * BPAD;                    // (column, 8-row half chunk) units per tile
  constexpr int HU = (NHU + kSlT - 1) / kSlT;      // half units per slicer thread
  constexpr int NWH = kF64 ? 16 : 8;               // 32-bit words per half unit
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int slab = unit / g.nhalves, half = unit % g.nhalves;
  const int64_t r0 = static_cast<int64_t>(slab) * g.rows_per_slab;
  const int64_t r1 = min(m_loc, r0 + g.rows_per_slab);
  const int ntiles = static_cast<int>((r1 - r0 + kKTile - 1) / kKTile);
  const int NS = g.nst;

  // dynamic smem: [X stages (1024-aligned, 128B-swizzled)] [B stages]
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* xbuf = base;
  uint8_t* bbuf = xbuf + NS * g.x_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sh.x_full[s], 1);
      mbar_init(&sh.x_empty[s], kSlW / 2);
      mbar_init(&sh.b_full[s], 1);
      mbar_init(&sh.b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sh.a_full[s], 4);
      mbar_init(&sh.a_empty[s], 1);
    }
    mbar_init(&sh.d_full, 2);
    mbar_init(&sh.d_empty, kSlW / 2);
    mbar_init(&sh.tok[0], 1);
    mbar_init(&sh.tok[1], 1);
    sh.egen = 0;
    sh.qsh = 0;
    sh.epi_done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (warp-uniform)
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < ntiles; ++t) {
      if (t >= NS) mbar_wait(&sh.x_empty[s], ph ^ 1);
      if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[4 * kDbgTiles + t] = clock64();
      mbar_arrive_expect_tx_e(&sh.x_full[s], g.x_bytes);
      uint8_t* dst = xbuf + s * g.x_bytes;
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        tma_load_2d_e(dst + bx * BPAD * 128, &tmap, &sh.x_full[s], static_cast<int>(r0 + int64_t(t) * kKTile + bx * BOX_ROWS), 0);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (warp-uniform, elected lane)
    constexpr int chB = NTOT / 8 * 128;      // bytes per 16-byte K chunk of the B stage
    constexpr int NU = (kS - 1) * BPAD;      // unsigned digit planes 0 .. S-2
    constexpr int NUC = NU > 256 ? NU / 2 : NU;
    int q = 0;
    bool first = true;
    int s = 0;
    uint32_t ph = 0;
    const uint32_t bbase0 = smem_u32(bbuf);
    for (int t = 0; t < ntiles; ++t) {
      const int sa = t & 1;
      mbar_wait(&sh.a_full[sa], (t >> 1) & 1);
      mbar_wait(&sh.b_full[s], ph);
      tc_fence_after();
      if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[2 * kDbgTiles + t] = clock64();
      if (sh.bflags[s] && t > 0) {           // close accumulation epoch q: flush D to fp64
        mma_commit_e(&sh.d_full);
        mbar_arrive_e(&sh.d_full);
        mbar_wait(&sh.d_empty, q & 1);
        tc_fence_after();
        ++q;
        first = true;
      }
      const uint32_t bbase = bbase0 + s * g.b_bytes;
#pragma unroll
      for (int ks = 0; ks < kKTile / 32; ++ks) {
#pragma unroll
        for (int tm = 0; tm < TM; ++tm) {
          const uint32_t at = tmem + ACOL0 + (sa * TM + tm) * 16 + ks * 8;
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint32_t dcol = tmem + tm * NTOT;
#pragma unroll
          for (int n0 = 0; n0 < NU; n0 += NUC) {
            const uint64_t bd = umma_desc(bbase + 2 * ks * chB + (n0 / 8) * 128, chB, 128);
            mma_i8_ta_e(dcol + n0, at, bd, idesc_i8(NUC, false), acc);
          }
          const uint64_t bd = umma_desc(bbase + 2 * ks * chB + (NU / 8) * 128, chB, 128);
          mma_i8_ta_e(dcol + NU, at, bd, idesc_i8(BPAD, true), acc);
        }
      }
      first = false;
      mma_commit_e(&sh.a_empty[sa]);
      mma_commit_e(&sh.b_empty[s]);
      if (g.dbg && blockIdx.x == 0 && t < kDbgTiles && lane == 0) g.dbg[3 * kDbgTiles + t] = clock64();
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    mma_commit_e(&sh.d_full);
    mbar_arrive_e(&sh.d_full);
  } else if (warp >= kSlicer0) {
    // ---------------------------------------------------------------- digit slicer (2 x 128 threads)
    // Two groups of 4 warps convert alternate tiles concurrently (group g: tiles t = g mod 2).
    // Shared per-tile bookkeeping (epoch index, exponent raises, b_full) is serialised in tile
    // order by a token passed between the groups (mbarriers tok[0..1]).
    constexpr int GT = 128;
    constexpr int GHU = (NHU + GT - 1) / GT;         // half units per thread per tile
    const int sw = warp - kSlicer0;                  // 0..7
    const int grp = sw >> 2;
    const int gt = threadIdx.x - 32 * (kSlicer0 + 4 * grp);   // 0..127
    const int st = threadIdx.x - 32 * kSlicer0;      // 0..255
    const int j = (gt >> 1) % BPAD;                  // this thread's column (all its half units)
    const int barg = 1 + grp;                        // group barrier
    constexpr int kBarAll = 3;
    constexpr int chB = NTOT / 8 * 128;
    const int quarter = warp & 3;                    // TMEM lane quarter this warp may access
    // epilogue of accumulation epoch qe: D (int32, TMEM) -> fp64 partial sums, one group
    // Epilogues run in epoch order.  Each group drains only the epochs its own tiles open, so it
    // may skip d_full phases; with the MMA two flushes behind, the parity of epoch qe would match
    // the completed phase qe - 2 and the drain would read D mid-accumulation.  Waiting for the
    // epilogue of epoch qe - 1 first (which itself waited for phase qe - 1) makes the parity wait
    // unambiguous and orders the read-modify-write of `part` after the previous epoch's stores.
    auto epilogue = [&](int qe) {
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&sh.epi_done) < 4 * qe) __nanosleep(32);
      __syncwarp();
      __threadfence_block();
      mbar_wait(&sh.d_full, qe & 1);
      tc_fence_after();
#pragma unroll
      for (int tm = 0; tm < TM; ++tm) {
        const int rl = tm * 128 + 32 * quarter + lane;
        const int r = half * ROWS + rl;
#pragma unroll 1
        for (int jb = 0; jb < BPAD; jb += 16) {
          double acc[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) acc[k] = 0.0;
#pragma unroll 1
          for (int p = kS - 1; p >= 0; --p) {
            uint32_t v[16];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + tm * NTOT + p * BPAD + jb;
            OID_TMEM_LD16(taddr, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const double wgt = __longlong_as_double(static_cast<long long>(8 * p + 1023) << 52);
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] = fma(static_cast<double>(static_cast<int>(v[k])), wgt, acc[k]);
          }
          if (r < ell) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int jj = jb + k;
              if (jj >= ncols) continue;
              const int e = sh.ehist[qe & 3][jj];
              const double val =
                  (e == kNone) ? 0.0 : acc[k] * __longlong_as_double(static_cast<long long>(e - kTop + 1023) << 52);
              double* dst = part + (static_cast<int64_t>(unit) * BPAD + jj) * ROWS + rl;
              *dst = (qe == 0) ? val : *dst + val;
            }
          }
        }
      }
      tc_fence_before();
      __threadfence_block();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sh.d_empty);
        atomicAdd(&sh.epi_done, 1);
      }
    };
    auto keymax = [&](const uint32_t (&w)[NWH]) -> uint32_t {
      uint32_t km = 0;
      if constexpr (kF64) {
#pragma unroll
        for (int e = 0; e < 8; ++e) km = max(km, Bits<double>::key(w[2 * e + 1]));
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) km = max(km, Bits<float>::key(w[e]));
      }
      return km;
    };
    auto load_tile = [&](int s, uint32_t (&w)[GHU][NWH]) {
      const uint8_t* xs = xbuf + s * g.x_bytes;
#pragma unroll
      for (int k = 0; k < GHU; ++k) {
        const int hu = gt + GT * k;
        if (hu < NHU) load_half<T, BPAD>(xs, j, (hu >> 1) / BPAD, hu & 1, w[k]);
      }
    };
    auto publish = [&](const uint32_t (&w)[GHU][NWH]) {
#pragma unroll
      for (int k = 0; k < GHU; ++k) {
        const int hu = gt + GT * k;
        if (hu < NHU) sh.emax[0][(hu >> 1) / BPAD][hu & 1][j] = Bits<T>::ebound(keymax(w[k]));
      }
    };
    // columns (threads gt < BPAD): first tile sets the exponents, later tiles only raise them
    auto set_ecur = [&](bool first) {
      if (gt >= BPAD) return;
      int eb = kNone;
#pragma unroll
      for (int c = 0; c < 4; ++c) eb = max(eb, max(sh.emax[0][c][0][gt], sh.emax[0][c][1][gt]));
      const int ep = sh.ecur[0][gt];
      if (first) sh.ecur[0][gt] = eb == kNone ? kNone : max(kEmin, eb + kHeadroom);
      else if (eb != kNone && (ep == kNone || eb > ep)) sh.ecur[0][gt] = max(kEmin, eb + kHeadroom);
    };
    double nacc = 0.0, cacc = 0.0;
    // exact fixed-point digits of x * 2^F_j -> K-major B operand of stage s; returns 1 when an
    // element of this thread exceeds its column's current exponent bound (needs a raise)
    auto convert = [&](const uint32_t (&wc)[GHU][NWH], int s, bool norms) -> int {
      const int e = sh.ecur[0][j];
      const bool zero_col = (e == kNone);
      const int F = zero_col ? 0 : kTop - e;
      const double p0 = zero_col ? 0.0 : __longlong_as_double(static_cast<long long>(F + 1023) << 52);
      const double p32 = zero_col ? 0.0 : __longlong_as_double(static_cast<long long>(F - 32 + 1023) << 52);
      uint8_t* bst = bbuf + s * g.b_bytes;
      int viol = 0;
#pragma unroll
      for (int k = 0; k < GHU; ++k) {
        const int hu = gt + GT * k;
        if (hu >= NHU) continue;
        const int u = hu >> 1, h = hu & 1, c16 = u / BPAD;
        const int eb = Bits<T>::ebound(keymax(wc[k]));
        viol |= (eb != kNone) && (zero_col || eb > e);
        uint32_t outw[kS][2];
#pragma unroll
        for (int w4 = 0; w4 < 2; ++w4) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int e8 = 4 * w4 + r;
            double x;
            if constexpr (kF64) x = __hiloint2double(static_cast<int>(wc[k][2 * e8 + 1]), static_cast<int>(wc[k][2 * e8]));
            else x = static_cast<double>(__uint_as_float(wc[k][e8]));
            if (norms) {
              nacc = fma(x, x, nacc);
              cacc += x;
            }
            double v;
            fixpt(x, p32, p0, lo[r], hi[r], v);
          }
          // 4x4 byte transposes: word w4 of digit plane p = byte p of rows 4w4 .. 4w4+3
          const uint32_t x0 = prmt(lo[0], lo[1], 0x5140), x1 = prmt(lo[0], lo[1], 0x7362);
          const uint32_t y0 = prmt(lo[2], lo[3], 0x5140), y1 = prmt(lo[2], lo[3], 0x7362);
          outw[0][w4] = prmt(x0, y0, 0x5410);
          outw[1][w4] = prmt(x0, y0, 0x7632);
          outw[2][w4] = prmt(x1, y1, 0x5410);
          outw[3][w4] = prmt(x1, y1, 0x7632);
          const uint32_t u0 = prmt(hi[0], hi[1], 0x5140), u1 = prmt(hi[0], hi[1], 0x7362);
          const uint32_t v0 = prmt(hi[2], hi[3], 0x5140), v1 = prmt(hi[2], hi[3], 0x7362);
          outw[4][w4] = prmt(u0, v0, 0x5410);
          outw[5][w4] = prmt(u0, v0, 0x7632);
          outw[6][w4] = prmt(u1, v1, 0x5410);
        }
#pragma unroll
        for (int p = 0; p < kS; ++p) {
          const int n = p * BPAD + j;
          uint2* dst = reinterpret_cast<uint2*>(bst + c16 * chB + (n >> 3) * 128 + (n & 7) * 16 + h * 8);
          *dst = make_uint2(outw[p][0], outw[p][1]);
        }
      }
      return viol;
    };
    // tile 0 sets the exponents (group 0 reads it, both groups synchronise)
    if (grp == 0 && ntiles > 0) {
      mbar_wait(&sh.x_full[0], 0);
      uint32_t w0[GHU][NWH];
      load_tile(0, w0);
      publish(w0);
    }
    named_bar(kBarAll, 2 * GT);
    if (grp == 0) set_ecur(true);
    named_bar(kBarAll, 2 * GT);
    int s = grp % NS;
    uint32_t ph = (grp / NS) & 1;
    int k = 0;
    int qlast = -1;
#pragma unroll 1
    for (int t = grp; t < ntiles; t += 2, ++k) {
      const bool dbgt = g.dbg && blockIdx.x == 0 && gt == 0 && t < kDbgTiles;
      if (dbgt) g.dbg[5 * kDbgTiles + t] = clock64();
      mbar_wait(&sh.x_full[s], ph);
      uint32_t wc[GHU][NWH];
      load_tile(s, wc);
      if (t >= NS) mbar_wait(&sh.b_empty[s], ph ^ 1u);
      if (dbgt) g.dbg[6 * kDbgTiles + t] = clock64();
      int egen = *reinterpret_cast<volatile int*>(&sh.egen);
      int viol = g.exp == 2 ? 0 : convert(wc, s, true);
      // release the X stage only after its values were consumed: an arrive right after issuing
      // the shared-memory loads lets the next TMA load overwrite them first (a WAR race across
      // the generic and async proxies, observed in K1F)
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.x_empty[s]);
      fence_proxy_async();
      int viol_any = named_bar_or(barg, GT, viol);
      if (dbgt) g.dbg[7 * kDbgTiles + t] = clock64();
      // ---- token: bookkeeping in tile order
      if (t > 0) mbar_wait(&sh.tok[grp], grp == 1 ? (k & 1) : ((k - 1) & 1));
      if (dbgt) g.dbg[8 * kDbgTiles + t] = clock64();
      int newacc = (t % kMaxEpochTiles) == 0;
      for (;;) {
        // (the token holder alone writes egen, so eg is uniform here; the snapshots egen taken
        // before the conversion may differ between threads, hence the reduction)
        const int eg = *reinterpret_cast<volatile int*>(&sh.egen);
        if (named_bar_or(barg, GT, eg != egen)) {  // exponents raised by the other group: redo
          egen = eg;
          viol = convert(wc, s, false);
          fence_proxy_async();
          viol_any = named_bar_or(barg, GT, viol);
        }
        if (!viol_any) break;
        publish(wc);                             // raise the exponents of the offending columns
        named_bar(barg, GT);
        set_ecur(false);
        named_bar(barg, GT);
        if (gt == 0) sh.egen = egen + 1;
        named_bar(barg, GT);
        newacc = 1;
      }
      const int q0 = *reinterpret_cast<volatile int*>(&sh.qsh);
      const int q = (newacc && t > 0) ? q0 + 1 : q0;
      if (newacc && gt < BPAD) sh.ehist[q & 3][gt] = sh.ecur[0][gt];
      named_bar(barg, GT);
      if (gt == 0) {
        sh.qsh = q;
        sh.bflags[s] = newacc;
        mbar_arrive(&sh.b_full[s]);
        if (g.dbg && blockIdx.x == 0 && t < kDbgTiles) g.dbg[1 * kDbgTiles + t] = clock64();
        mbar_arrive(&sh.tok[grp ^ 1]);           // hand the token to tile t + 1
      }
      if (dbgt) g.dbg[9 * kDbgTiles + t] = clock64();
      if (newacc && t > 0) epilogue(q - 1);
      qlast = q;
      s += 2;
      if (s >= NS) { s -= NS; ph ^= 1u; }
    }
    if (ntiles > 0 && ((ntiles - 1) & 1) == grp) epilogue(qlast);   // the last tile's group
    // norms and column sums: threads sharing column j combine in fixed order (half 0 units only)
    sh.nrm[st] = nacc;
    sh.csum[st] = cacc;
    named_bar(kBarAll, 2 * GT);
    if (half == 0 && st < BPAD && st < ncols) {
      double sum = 0.0, cs = 0.0;
      for (int kk = 0; kk < 2 * GT; ++kk) {
        const int gtk = kk % GT;
        if (((gtk >> 1) % BPAD) != st || gtk >= NHU) continue;
        sum += sh.nrm[kk];
        cs += sh.csum[kk];
      }
      npart[static_cast<int64_t>(slab) * BPAD + st] = sum;
      cpart[static_cast<int64_t>(slab) * BPAD + st] = cs;
    }
  } else {
    // ---------------------------------------------------------------- sketch generator (4 warps)
    // warp -> TMEM lane quarter; each thread owns sketch row rl (and rl + 128 when TM = 2) and
    // writes both 32-row K chunks of a tile (2 Philox calls per row) with one tcgen05.st each.
    const int gw = warp - kGen0;                     // 0..3
    const int quarter = warp & 3;
    const uint64_t g32_0 = static_cast<uint64_t>((row_begin + r0) >> 5);
    for (int t = 0; t < ntiles; ++t) {
      const int sa = t & 1;
      if (t >= 2) {
        if (lane == 0) mbar_wait(&sh.a_empty[sa], ((t >> 1) - 1) & 1);
        __syncwarp();
        tc_fence_after();
      }
      // all 2 TM Philox calls of this thread's rows run interleaved (independent streams, shared
      // key schedule): instruction-level parallelism instead of 2 TM dependent 10-round chains
      constexpr int NC = 2 * TM;
      uint32_t c0[NC], c1[NC], c2[NC], c3[NC];
#pragma unroll
      for (int tm = 0; tm < TM; ++tm)
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int ci = 2 * tm + kc;
          c0[ci] = static_cast<uint32_t>(g32_0 + static_cast<uint64_t>(t) * (kKTile / 32) + kc);
          c1[ci] = static_cast<uint32_t>(half * ROWS + tm * 128 + quarter * 32 + lane);
          c2[ci] = 0u;
          c3[ci] = 0u;
        }
      uint32_t kk0 = key0, kk1 = key1;
      asm volatile("" : "+r"(kk0), "+r"(kk1));   // keep the key schedule in-loop (register budget)
      const int nrnd = (g.exp == 1 || OMEGA) ? 0 : 10;
      if constexpr (OMEGA) {
        // stored sketch entries (NEXT-3): the same Philox words, streamed from HBM (one 16-byte
        // load per 32 entries, consecutive lanes = consecutive sketch rows)
#pragma unroll
        for (int ci = 0; ci < NC; ++ci) {
          // rows r >= ell (the padded half) read row ell - 1: their products are discarded
          const int64_t gi = static_cast<int64_t>(c0[ci]) - g.g0;
          c1[ci] = min(c1[ci], static_cast<uint32_t>(ell - 1));
          uint4 v;
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "l"(g.omega + gi * ell + c1[ci]));
          c0[ci] = v.x; c1[ci] = v.y; c2[ci] = v.z; c3[ci] = v.w;
        }
      }
#pragma unroll
      for (int rnd = 0; rnd < 10; ++rnd) {
        if (rnd >= nrnd) break;
#pragma unroll
        for (int ci = 0; ci < NC; ++ci) {
          uint32_t hi0, lo0, hi1, lo1;
          mulhilo32(0xD2511F53u, c0[ci], hi0, lo0);   // one IMAD.WIDE.U32 each
          mulhilo32(0xCD9E8D57u, c2[ci], hi1, lo1);
          const uint32_t n0 = hi1 ^ c1[ci] ^ kk0;
          const uint32_t n2 = hi0 ^ c3[ci] ^ kk1;
          c0[ci] = n0; c1[ci] = lo1; c2[ci] = n2; c3[ci] = lo0;
        }
        kk0 += 0x9E3779B9u;
        kk1 += 0xBB67AE85u;
      }
#pragma unroll
      for (int tm = 0; tm < TM; ++tm) {
        const int rl = tm * 128 + quarter * 32 + lane;
        const int r = half * ROWS + rl;
        uint32_t pk[16];
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int ci = 2 * tm + kc;
          const uint32_t ws[4] = {c0[ci], c1[ci], c2[ci], c3[ci]};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // 8 nibbles n = (sign, v): q = m_v (sign 0) or ~m_v = -m_v - 1 (sign 1), 4 per PRMT
            const uint32_t w = ws[k], w4 = w << 4;
            const uint32_t mlo = prmt(t0, t1, w & 0x7777u), mhi = prmt(t0, t1, (w >> 16) & 0x7777u);
            const uint32_t slo = prmt(w, w4, 0x9D8Cu), shi = prmt(w, w4, 0xBFAEu);   // sign bytes 0x00/0xFF
            pk[8 * kc + 2 * k] = mlo ^ slo;
            pk[8 * kc + 2 * k + 1] = mhi ^ shi;
          }
        }
        if (half * ROWS + tm * 128 + quarter * 32 + 31 >= ell && r >= ell) {   // warp-uniform test first
#pragma unroll
          for (int k = 0; k < 16; ++k) pk[k] = 0u;
        }
        tmem_st16(tmem + (static_cast<uint32_t>(32 * quarter) << 16) + ACOL0 + (sa * TM + tm) * 16, pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.a_full[sa]);
      if (g.dbg && blockIdx.x == 0 && gw == 0 && lane == 0 && t < kDbgTiles) g.dbg[t] = clock64();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// NEXT-3: store the Philox words of the shard's sketch entries, omega[g * ell + r] = Philox4x32-10
// at counter (g0 + g, r, 0, 0) (reading R2), so K1 streams them instead of generating them
__global__ void omega_fill_kernel(uint4* __restrict__ omega, int64_t ngroups, int64_t g0, int ell, uint32_t key0,
                                  uint32_t key1) {
  const int64_t n = ngroups * ell;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gq = i / ell;
    const int r = static_cast<int>(i - gq * ell);
    const U4 w = philox4x32_10(static_cast<uint32_t>(g0 + gq), static_cast<uint32_t>(r), 0u, 0u, key0, key1);
    omega[i] = make_uint4(w.x, w.y, w.z, w.w);
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
    const int h = r / g.rows, rl = r % g.rows;
    double s = 0.0, c = 0.0;
#pragma unroll 8   // the loads of several slabs in flight; the sums keep their fixed order
    for (int sl = 0; sl < g.nslabs; ++sl) {
      s += part[(static_cast<int64_t>(sl * g.nhalves + h) * g.bpad + j) * g.rows + rl];
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

}  // namespace k1tc

// ------------------------------------------------------------------ host side
constexpr int kTcMaxUnits = 256;

inline size_t k1tc_workspace_bytes(int /*ell*/, int /*b_max*/, int64_t /*m_loc*/, bool /*f64*/) {
  return static_cast<size_t>(kTcMaxUnits) * 64 * 256 * sizeof(double) +
         2 * static_cast<size_t>(kTcMaxUnits) * 64 * sizeof(double) + 1024;
}

inline bool k1tc_supported(int ell, int b_max, bool /*f64*/) { return ell >= 1 && ell <= 1024 && b_max <= 64; }

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled k1tc_encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// Whether this call can use the tensor-core kernel (alignment rules of TMA and the Philox groups).
inline bool k1tc_call_ok(const K1TcArgs& a) {
  const int es = a.f64 ? 8 : 4;
  if (a.ncols < 1 || a.ncols > 64) return false;
  if (a.row_begin % 32 != 0) return false;        // Philox blocks of 32 rows (reading R2)
  if ((a.ld * es) % 16 != 0) return false;
  if (reinterpret_cast<uintptr_t>(a.X) % 16 != 0) return false;
  if (a.row_end - a.row_begin >= (int64_t(1) << 31)) return false;
  const k1tc::Geom g = k1tc::make_geom(a.ell, a.ncols, a.row_end - a.row_begin, a.f64, a.num_sms);
  if (g.nslabs * g.nhalves > kTcMaxUnits) return false;
  return k1tc_encoder() != nullptr;
}

template <typename T, int BPAD, int TM>
inline cudaError_t k1tc_launch_t(const CUtensorMap& map, const K1TcArgs& a, const k1tc::Geom& g, cudaStream_t st,
                                 double* part, double* npart, double* cpart) {
  auto fn = g.omega ? k1tc::k1_tc_kernel<T, BPAD, TM, true> : k1tc::k1_tc_kernel<T, BPAD, TM, false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();   // consumed here: a later call must not report it again
    return e;
  }
  fn<<<g.nslabs * g.nhalves, k1tc::kThreads, g.smem, st>>>(map, a.ncols, a.row_begin, a.row_end - a.row_begin, a.ell,
                                                           a.key0, a.key1, a.t0, a.t1, g, part, npart, cpart);
  return cudaGetLastError();
}

template <typename T>
inline cudaError_t k1tc_dispatch(const CUtensorMap& map, const K1TcArgs& a, const k1tc::Geom& g, cudaStream_t st,
                                 double* part, double* npart, double* cpart) {
  if (g.bpad == 16) return g.TM == 2 ? k1tc_launch_t<T, 16, 2>(map, a, g, st, part, npart, cpart)
                                     : k1tc_launch_t<T, 16, 1>(map, a, g, st, part, npart, cpart);
  if (g.bpad == 32) return g.TM == 2 ? k1tc_launch_t<T, 32, 2>(map, a, g, st, part, npart, cpart)
                                     : k1tc_launch_t<T, 32, 1>(map, a, g, st, part, npart, cpart);
  return k1tc_launch_t<T, 64, 1>(map, a, g, st, part, npart, cpart);
}

inline cudaError_t k1tc_launch(const K1TcArgs& a, cudaStream_t st, int* nlaunch) {
  *nlaunch = 0;
  const int64_t m_loc = a.row_end - a.row_begin;
  k1tc::Geom g = k1tc::make_geom(a.ell, a.ncols, m_loc, a.f64, a.num_sms);
  g.dbg = a.dbg;
  g.omega = a.omega;
  g.g0 = a.row_begin / 32;
  g.exp = getenv("OID_K1_EXP") ? atoi(getenv("OID_K1_EXP")) : 0;
  CUtensorMap map;
  const int es = a.f64 ? 8 : 4;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m_loc), static_cast<cuuint64_t>(a.ncols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * es};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(g.bpad)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = k1tc_encoder()(&map, a.f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                               const_cast<void*>(a.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  double* part = reinterpret_cast<double*>(a.ws);
  double* npart = part + static_cast<size_t>(kTcMaxUnits) * 64 * 256;
  double* cpart = npart + static_cast<size_t>(kTcMaxUnits) * 64;
  cudaError_t e = a.f64 ? k1tc_dispatch<double>(map, a, g, st, part, npart, cpart)
                        : k1tc_dispatch<float>(map, a, g, st, part, npart, cpart);
  *nlaunch += 1;
  if (e != cudaSuccess) return e;
  const int64_t nout = int64_t(a.ell) * a.ncols + a.ncols;
  k1tc::k1_tc_reduce_kernel<<<static_cast<unsigned>((nout + 255) / 256), 256, 0, st>>>(part, npart, cpart, g, a.ell,
                                                                                     a.ncols, a.scale, a.out, a.flags);
  *nlaunch += 1;
  return cudaGetLastError();
}

}  // namespace oid
