// K1, tensor-core variant for sm_100a: Y_part = Z(:, slab) * X_blk and n_j = ||x_j||^2 in one
// read of X (Alg 3 steps 10 and 13), exactly.
//
// Why exact: the sketch entries are Gauss-256 integers q in [-127, 127] (reading R2), so
// Z = s * Q with Q int8.  Each snapshot value x is cut into S two's-complement 8-bit digits of a
// per-column fixed-point integer x_int = round(x * 2^F_j) (S = 8 digit planes, 64-bit fixed point),
// and Q * X_digit_s runs on the 5th-generation tensor cores as tcgen05.mma kind::i8 with exact
// int32 accumulation in TMEM.  Y = s * sum_s 2^(8 s - F_j) * D_s is assembled in fp64.
//
// CTA organisation (one CTA per SM, 16 warps, persistent over one work unit = row slab x
// slice of 128*T_M sketch rows):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D boxes of X (64 rows x b) into a ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-3   digit slicer: X stage -> per-column exponent check -> int8 digit planes (B op.)
//   warps 4-7   epilogue: tcgen05.ld of the int32 accumulators, fp64 assembly, partial out
//   warps 8-15  sketch generator: Philox4x32-10 -> Gauss-256 bytes -> A operand in smem
// Per-column exponents start from the first tile of the unit plus 16 bits of headroom; if a
// later tile exceeds them the accumulators are flushed to fp64 (exactly) and accumulation
// restarts with a larger exponent ("accumulation epochs"), so X is still read once.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"

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
};

__constant__ int8_t c_qtab_i8[256];

namespace k1tc {

constexpr int kThreads = 512;
constexpr int kKTile = 64;          // data rows per pipeline stage
constexpr int kNumStages = 3;
constexpr int kHeadroom = 16;       // exponent headroom bits
constexpr int kEmin = -900;         // exponents are clamped here (data below 2^-900 lose bits)
constexpr int kNone = -100000;      // "no nonzero seen yet" exponent

struct Geom {
  int bpad;      // padded block width (16, 32, 64)
  int S;         // digit planes (8 fp64, 6 fp32)
  int TM;        // M tiles (of 128 sketch rows) per CTA
  int rows;      // 128 * TM
  int ntot;      // bpad * S accumulator columns per M tile
  int tmem_cols; // allocation (power of two)
  int a_bytes, b_bytes, x_bytes;   // per stage
  int smem;      // dynamic smem bytes
  int nst;       // pipeline stages (2 or 3)
  int nhalves;   // sketch-row slices
  int nslabs;
  int64_t rows_per_slab;
};

inline Geom make_geom(int ell, int ncols, int64_t m_loc, bool f64, int num_sms) {
  Geom g{};
  g.bpad = ncols <= 16 ? 16 : (ncols <= 32 ? 32 : 64);
  g.S = 8;   // 64-bit fixed point for both fp64 and fp32 data
  g.ntot = g.bpad * g.S;
  g.TM = (2 * g.ntot <= 512) ? 2 : 1;
  g.rows = 128 * g.TM;
  const int need = g.TM * g.ntot;
  g.tmem_cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
  g.a_bytes = g.rows * kKTile;
  g.b_bytes = g.ntot * kKTile;
  g.x_bytes = kKTile * g.bpad * (f64 ? 8 : 4);
  g.nst = kNumStages;
  while (g.nst > 2 && g.nst * (g.a_bytes + g.b_bytes + g.x_bytes) + 256 * 32 * 4 + 4096 > 220 * 1024) --g.nst;
  g.smem = g.nst * (g.a_bytes + g.b_bytes + g.x_bytes) + 256 * 32 * 4 + 4096;
  g.nhalves = (ell + g.rows - 1) / g.rows;
  g.nslabs = std::max(1, num_sms / g.nhalves);
  int64_t per = (m_loc + g.nslabs - 1) / g.nslabs;
  per = (per + kKTile - 1) / kKTile * kKTile;
  g.rows_per_slab = per;
  g.nslabs = static_cast<int>((m_loc + per - 1) / per);
  return g;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes,
// LBO = byte distance of the two 16-byte K halves, SBO = distance of 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;   // version (sm_100)
  return d;                              // base offset 0, layout SWIZZLE_NONE (0)
}

// Instruction descriptor, kind::i8: D s32, A s8 (K-major), B u8/s8 (K-major), M=128, N.
__device__ __forceinline__ uint32_t idesc_i8(int n, bool b_signed) {
  uint32_t d = 0;
  d |= 2u << 4;                          // D format: S32
  d |= 1u << 7;                          // A format: signed 8-bit
  d |= (b_signed ? 1u : 0u) << 10;       // B format
  d |= static_cast<uint32_t>(n >> 3) << 17;
  d |= static_cast<uint32_t>(128 >> 4) << 24;
  return d;
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define OID_TMEM_LD32(taddr, r)                                                                                   \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, " \
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(taddr))

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// exponent e with |v| < 2^e for finite v > 0 (frexp exponent); kNone for v == 0
__device__ __forceinline__ int exp_bound(double v) {
  if (!(v > 0.0)) return kNone;
  const long long bits = __double_as_longlong(v);
  int e = static_cast<int>((bits >> 52) & 0x7ff);
  if (e == 0) return -1021;    // subnormal
  if (e == 0x7ff) return 1024; // inf/nan: force a (harmless) raise; the norm flags it
  return e - 1022;
}

struct Shared {
  uint64_t x_full[kNumStages], x_empty[kNumStages];
  uint64_t a_full[kNumStages], b_full[kNumStages], ab_empty[kNumStages];
  uint64_t d_full, d_empty;
  uint32_t tmem_base;
  int bflags[kNumStages];
  int flush_final[2];
  int ecur[64];
  int ehist[2][64];
  double colmax[128];
  double nrm[64][2];
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
k1_tc_kernel(const __grid_constant__ CUtensorMap tmap, int ncols, int64_t row_begin, int64_t m_loc, int ell,
             uint32_t key0, uint32_t key1, Geom g, double* __restrict__ part, double* __restrict__ npart) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ Shared sh;
  constexpr bool kF64 = sizeof(T) == 8;
  constexpr int S = 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int slab = unit / g.nhalves, half = unit % g.nhalves;
  const int64_t r0 = static_cast<int64_t>(slab) * g.rows_per_slab;
  const int64_t r1 = min(m_loc, r0 + g.rows_per_slab);
  const int ntiles = static_cast<int>((r1 - r0 + kKTile - 1) / kKTile);
  const int bpad = g.bpad;
  const int NS = g.nst;

  uint8_t* abuf = smem_raw;
  uint8_t* bbuf = abuf + NS * g.a_bytes;
  uint8_t* xbuf = bbuf + NS * g.b_bytes;
  uint32_t* qtab = reinterpret_cast<uint32_t*>(xbuf + NS * g.x_bytes);   // [256][32]

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sh.x_full[s], 1);
      mbar_init(&sh.x_empty[s], 2);
      mbar_init(&sh.a_full[s], 8);
      mbar_init(&sh.b_full[s], 1);
      mbar_init(&sh.ab_empty[s], 1);
    }
    mbar_init(&sh.d_full, 2);
    mbar_init(&sh.d_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 256 * 32; i += kThreads) qtab[i] = static_cast<uint32_t>(c_qtab_i8[i >> 5]) & 0xFFu;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(g.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % NS;
        if (t >= NS) mbar_wait(&sh.x_empty[s], ((t / NS) - 1) & 1);
        mbar_arrive_expect_tx(&sh.x_full[s], g.x_bytes);
        tma_load_2d(xbuf + s * g.x_bytes, &tmap, &sh.x_full[s], static_cast<int>(r0 + int64_t(t) * kKTile), 0);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const int chA = g.rows / 8 * 128;      // bytes per 16-byte K chunk of the A stage
      const int chB = g.ntot / 8 * 128;
      int q = 0;
      bool first = true;
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % NS;
        const uint32_t ph = (t / NS) & 1;
        mbar_wait(&sh.a_full[s], ph);
        mbar_wait(&sh.b_full[s], ph);
        tc_fence_after();
        if (sh.bflags[s] && t > 0) {           // close accumulation epoch q: flush D to fp64
          sh.flush_final[q & 1] = 0;
          mma_commit(&sh.d_full);
          mbar_arrive(&sh.d_full);
          mbar_wait(&sh.d_empty, q & 1);
          tc_fence_after();
          ++q;
          first = true;
        }
        const uint32_t abase = smem_u32(abuf + s * g.a_bytes);
        const uint32_t bbase = smem_u32(bbuf + s * g.b_bytes);
#pragma unroll
        for (int ks = 0; ks < kKTile / 32; ++ks) {
          for (int tm = 0; tm < g.TM; ++tm) {
            const uint64_t ad = umma_desc(abase + 2 * ks * chA + tm * 16 * 128, chA, 128);
            const uint32_t acc = (first && ks == 0) ? 0u : 1u;
            const uint32_t dcol = tmem + tm * g.ntot;
            // unsigned digit planes 0 .. S-2 (columns [0, (S-1) bpad)), chunks of <= 256
            const int nu = (S - 1) * bpad;
            for (int n0 = 0; n0 < nu; n0 += 256) {
              const int nn = min(256, nu - n0);
              const uint64_t bd = umma_desc(bbase + 2 * ks * chB + (n0 / 8) * 128, chB, 128);
              mma_i8(dcol + n0, ad, bd, idesc_i8(nn, false), acc);
            }
            // signed top plane
            const uint64_t bd = umma_desc(bbase + 2 * ks * chB + (nu / 8) * 128, chB, 128);
            mma_i8(dcol + nu, ad, bd, idesc_i8(bpad, true), acc);
          }
        }
        first = false;
        mma_commit(&sh.ab_empty[s]);
      }
      sh.flush_final[q & 1] = 1;
      mma_commit(&sh.d_full);
      mbar_arrive(&sh.d_full);
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------------- digit slicer (64 threads)
    const int st = threadIdx.x - 64;                 // 0..63
    const int per = 64 / bpad;                       // threads per column
    const int j = st % bpad;                         // this thread's column
    const int base = 62;                             // |x_int| < 2^62 for |x| < 2^E
    const int chB = g.ntot / 8 * 128;
    double nacc = 0.0;
    int q = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % NS;
      const uint32_t ph = (t / NS) & 1;
      mbar_wait(&sh.x_full[s], ph);
      const T* xs = reinterpret_cast<const T*>(xbuf + s * g.x_bytes);   // [col][64 rows]
      // pass 1: this thread's part of the column maximum
      double m = 0.0;
      for (int c = st / bpad; c < kKTile / 16; c += per) {
        const T* src = xs + j * kKTile + c * 16;
#pragma unroll
        for (int r = 0; r < 16; ++r) m = fmax(m, fabs(static_cast<double>(src[r])));
      }
      sh.colmax[st] = m;
      named_bar(1, 64);
      if (st < bpad) {
        double mm = 0.0;
        for (int k = 0; k < per; ++k) mm = fmax(mm, sh.colmax[st + k * bpad]);
        const int eb = exp_bound(mm);
        int raise = 0;
        if (t == 0) {
          sh.ecur[st] = eb == kNone ? kNone : max(kEmin, eb + kHeadroom);
        } else if (eb != kNone && (sh.ecur[st] == kNone || eb > sh.ecur[st])) {
          sh.ecur[st] = max(kEmin, eb + kHeadroom);
          raise = 1;
        }
        sh.colmax[64 + st] = raise;
      }
      named_bar(1, 64);
      int raise_any = 0;
      for (int k = 0; k < bpad; ++k) raise_any |= (sh.colmax[64 + k] != 0.0);
      const bool newacc = (t == 0) || raise_any;
      if (newacc && t > 0) {
        ++q;
        if (q >= 2) mbar_wait(&sh.d_empty, (q - 2) & 1);   // flush q-2 done: ehist[q & 1] is free
      }
      if (newacc && st < bpad) sh.ehist[q & 1][st] = sh.ecur[st];
      if (t >= NS) mbar_wait(&sh.ab_empty[s], ((t / NS) - 1) & 1);
      // pass 2: exact fixed-point digits of x * 2^F_j -> K-major B operand
      const int e = sh.ecur[j];
      const int F = base - e;
      const double scl = (e == kNone) ? 0.0 : __longlong_as_double(static_cast<long long>(F + 1023) << 52);
      uint8_t* bst = bbuf + s * g.b_bytes;
      for (int c = st / bpad; c < kKTile / 16; c += per) {
        const T* src = xs + j * kKTile + c * 16;
        uint32_t outw[S][4];
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double x = static_cast<double>(src[4 * w4 + k]);
            nacc = fma(x, x, nacc);
            const long long xi = __double2ll_rn(x * scl);
            lo[k] = static_cast<uint32_t>(xi);
            hi[k] = static_cast<uint32_t>(static_cast<unsigned long long>(xi) >> 32);
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
          if constexpr (S == 8) {
            outw[6][w4] = prmt(u1, v1, 0x5410);
            outw[7][w4] = prmt(u1, v1, 0x7632);
          }
        }
#pragma unroll
        for (int p = 0; p < S; ++p) {
          const int n = p * bpad + j;
          uint4* dst = reinterpret_cast<uint4*>(bst + c * chB + (n >> 3) * 128 + (n & 7) * 16);
          *dst = make_uint4(outw[p][0], outw[p][1], outw[p][2], outw[p][3]);
        }
      }
      fence_proxy_async();
      named_bar(1, 64);
      if (st == 0) {
        sh.bflags[s] = newacc ? 1 : 0;
        mbar_arrive(&sh.b_full[s]);
      }
      if (lane == 0) mbar_arrive(&sh.x_empty[s]);
    }
    // norms: threads sharing column j combine in fixed order (half 0 units only)
    sh.nrm[st][0] = nacc;
    named_bar(1, 64);
    if (half == 0 && st < bpad && st < ncols) {
      double sum = 0.0;
      for (int k = 0; k < per; ++k) sum += sh.nrm[st + k * bpad][0];
      npart[static_cast<int64_t>(slab) * bpad + st] = sum;
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- epilogue (4 warps)
    const int eq = warp - 4;
    const int base = 62;
    int q = 0;
    for (;;) {
      mbar_wait(&sh.d_full, q & 1);
      tc_fence_after();
      const int fin = sh.flush_final[q & 1];
      for (int tm = 0; tm < g.TM; ++tm) {
        const int rl = tm * 128 + 32 * eq + lane;
        const int r = half * g.rows + rl;
        for (int jb = 0; jb < bpad; jb += 32) {
          double acc[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) acc[k] = 0.0;
          for (int p = S - 1; p >= 0; --p) {
            uint32_t v[32];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * eq) << 16) + tm * g.ntot + p * bpad + jb;
            OID_TMEM_LD32(taddr, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const double w = __longlong_as_double(static_cast<long long>(8 * p + 1023) << 52);
#pragma unroll
            for (int k = 0; k < 32; ++k) acc[k] = fma(static_cast<double>(static_cast<int>(v[k])), w, acc[k]);
          }
          if (r < ell) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int jj = jb + k;
              if (jj >= ncols) continue;
              const int e = sh.ehist[q & 1][jj];
              const double val = (e == kNone) ? 0.0
                                              : acc[k] * __longlong_as_double(static_cast<long long>(e - base + 1023) << 52);
              double* dst = part + (static_cast<int64_t>(unit) * bpad + jj) * g.rows + rl;
              *dst = (q == 0) ? val : *dst + val;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.d_empty);
      if (fin) break;
      ++q;
    }
  } else {
    // ---------------------------------------------------------------- sketch generator (8 warps)
    const int rt = threadIdx.x - 256;
    const int parts = 256 / g.rows;
    const int rl = rt % g.rows, pidx = rt / g.rows;
    const int r = half * g.rows + rl;
    const int chA = g.rows / 8 * 128;
    const uint32_t* tl = qtab + lane;
    const uint64_t g16_0 = static_cast<uint64_t>((row_begin + r0) >> 4);
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % NS;
      if (t >= NS) mbar_wait(&sh.ab_empty[s], ((t / NS) - 1) & 1);
      uint8_t* ast = abuf + s * g.a_bytes;
      for (int c = pidx; c < kKTile / 16; c += parts) {
        uint4 o = make_uint4(0u, 0u, 0u, 0u);
        if (r < ell) {
          const uint32_t grp = static_cast<uint32_t>(g16_0 + static_cast<uint64_t>(t) * (kKTile / 16) + c);
          const U4 w = philox4x32_10(grp, static_cast<uint32_t>(r), 0u, 0u, key0, key1);
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
          uint32_t pk[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t a = ws[k];
            const uint32_t b0 = tl[(a & 0xFFu) << 5], b1 = tl[((a >> 8) & 0xFFu) << 5];
            const uint32_t b2 = tl[((a >> 16) & 0xFFu) << 5], b3 = tl[(a >> 24) << 5];
            pk[k] = prmt(prmt(b0, b1, 0x0040), prmt(b2, b3, 0x0040), 0x5410);
          }
          o = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        *reinterpret_cast<uint4*>(ast + c * chA + (rl >> 3) * 128 + (rl & 7) * 16) = o;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.a_full[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols));
  }
}

// out = [scale * sum over slabs of part (ell x ncols, col-major); sum of norm partials]
__global__ void k1_tc_reduce_kernel(const double* __restrict__ part, const double* __restrict__ npart, Geom g, int ell,
                                    int ncols, double scale, double* __restrict__ out, unsigned* __restrict__ flags) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ny = static_cast<int64_t>(ell) * ncols;
  if (idx < ny) {
    const int j = static_cast<int>(idx / ell), r = static_cast<int>(idx % ell);
    const int h = r / g.rows, rl = r % g.rows;
    double s = 0.0;
    for (int sl = 0; sl < g.nslabs; ++sl)
      s += part[(static_cast<int64_t>(sl * g.nhalves + h) * g.bpad + j) * g.rows + rl];
    out[idx] = scale * s;
  } else if (idx < ny + ncols) {
    const int j = static_cast<int>(idx - ny);
    double s = 0.0;
    for (int sl = 0; sl < g.nslabs; ++sl) s += npart[static_cast<int64_t>(sl) * g.bpad + j];
    out[idx] = s;
    if (!isfinite(s)) atomicOr(flags, 1u);
  }
}

}  // namespace k1tc

// ------------------------------------------------------------------ host side
constexpr int kTcMaxUnits = 256;

inline size_t k1tc_workspace_bytes(int /*ell*/, int /*b_max*/, int64_t /*m_loc*/, bool /*f64*/) {
  return static_cast<size_t>(kTcMaxUnits) * 64 * 256 * sizeof(double) + static_cast<size_t>(kTcMaxUnits) * 64 * sizeof(double) + 1024;
}

inline bool k1tc_supported(int ell, int b_max, bool /*f64*/) { return ell >= 1 && ell <= 1024 && b_max <= 64; }

inline cudaError_t k1tc_init_tables(const int32_t* q, cudaStream_t st) {
  int8_t q8[256];
  for (int i = 0; i < 256; ++i) q8[i] = static_cast<int8_t>(q[i]);
  return cudaMemcpyToSymbolAsync(c_qtab_i8, q8, sizeof(q8), 0, cudaMemcpyHostToDevice, st);
}

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
  if (a.row_begin % 16 != 0) return false;
  if ((a.ld * es) % 16 != 0) return false;
  if (reinterpret_cast<uintptr_t>(a.X) % 16 != 0) return false;
  if (a.row_end - a.row_begin >= (int64_t(1) << 31)) return false;
  const k1tc::Geom g = k1tc::make_geom(a.ell, a.ncols, a.row_end - a.row_begin, a.f64, a.num_sms);
  if (g.nslabs * g.nhalves > kTcMaxUnits) return false;
  return k1tc_encoder() != nullptr;
}

inline cudaError_t k1tc_launch(const K1TcArgs& a, cudaStream_t st, int* nlaunch) {
  *nlaunch = 0;
  const int64_t m_loc = a.row_end - a.row_begin;
  const k1tc::Geom g = k1tc::make_geom(a.ell, a.ncols, m_loc, a.f64, a.num_sms);
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m_loc), static_cast<cuuint64_t>(a.ncols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * (a.f64 ? 8 : 4)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(k1tc::kKTile), static_cast<cuuint32_t>(g.bpad)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = k1tc_encoder()(&map, a.f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                               const_cast<void*>(a.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  double* part = reinterpret_cast<double*>(a.ws);
  double* npart = part + static_cast<size_t>(kTcMaxUnits) * 64 * 256;
  const int units = g.nslabs * g.nhalves;
  cudaError_t e;
  if (a.f64) {
    e = cudaFuncSetAttribute(k1tc::k1_tc_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
    if (e != cudaSuccess) return e;
    k1tc::k1_tc_kernel<double><<<units, k1tc::kThreads, g.smem, st>>>(map, a.ncols, a.row_begin, m_loc, a.ell, a.key0,
                                                                      a.key1, g, part, npart);
  } else {
    e = cudaFuncSetAttribute(k1tc::k1_tc_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
    if (e != cudaSuccess) return e;
    k1tc::k1_tc_kernel<float><<<units, k1tc::kThreads, g.smem, st>>>(map, a.ncols, a.row_begin, m_loc, a.ell, a.key0,
                                                                     a.key1, g, part, npart);
  }
  *nlaunch += 1;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t nout = int64_t(a.ell) * a.ncols + a.ncols;
  k1tc::k1_tc_reduce_kernel<<<static_cast<unsigned>((nout + 255) / 256), 256, 0, st>>>(part, npart, g, a.ell, a.ncols,
                                                                                     a.scale, a.out, a.flags);
  *nlaunch += 1;
  return cudaGetLastError();
}

}  // namespace oid
