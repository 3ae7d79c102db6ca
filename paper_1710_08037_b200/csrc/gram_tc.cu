// K5: upper-triangle Hermitian Gram on the 5th-gen tensor cores (tcgen05 +
// TMEM + TMA), split precision fp16 x 3, with the fused PLV-family epilogue.
//
// Replaces the per-trial complex product of Appendix impl 3
// (`ndat(:,:,t) * ndat(:,:,t)'`) and SPEC plv_matrix /
// iplv / ciplv.  Z = Zr + i Zi is held as four fp16 planes
// (hi/lo of Re and Im, z = hi + lo to ~2^-24).  Per K-step of 16 samples the
// single MMA-issuing thread launches 12 UMMAs (K=16):
//   Re += Rh.Rh' + Rh.Rl' + Rl.Rh' + Ih.Ih' + Ih.Il' + Il.Ih'
//   Im += Ih.Rh' + Ih.Rl' + Il.Rh' - Rh.Ih' - Rh.Il' - Rl.Ih'
// (negation through the instruction descriptor's negate-A bit; the lo*lo
// terms, <= 2^-24, are dropped).
//
// Two variants share this file (template CG):
//   CG = 2 (default): a CTA pair (cluster of 2, tcgen05 cta_group::2) owns a
//     256 x 128 output tile; UMMA M = 256, N = 128.  Each CTA stages its own
//     128 rows of the I panel and half (64 rows) of the J panel; the rank-0
//     CTA issues the MMAs, both CTAs' TMEM hold their 128 rows.
//   CG = 1: one CTA per 128-row half of the tile (UMMA M = 128, N = 128).
//
// Accumulation accuracy.  The tensor core's fp32 accumulate is biased
// (measured on B200: relative error ~= n_accumulates * 2^-25, i.e. each UMMA
// truncates the running sum): accumulating all of T in TMEM would cost
// ~2e-5 at T = 2000 and ~8e-5 at T = 16384.  So the K loop is cut into chunks
// of kc_blocks * 32 samples; each chunk accumulates from zero in one of two
// TMEM buffers (ping-pong, 2 x (Re 128 + Im 128) = 512 columns) while the
// epilogue warps drain the other buffer into fp32 register sums
// (round-to-nearest).  With 128-sample chunks the error is ~1e-6.
//
// Warp roles (576 threads per CTA, one CTA per SM, persistent over items):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane; rank 0 only for CG=2)
//   warps 2..17 epilogue: warp w reads TMEM lane quadrant w%4, column quarter
//               (w-2)/4; drains chunks into 32 Re + 32 Im register sums and,
//               at the end of a round, emits PLV / iPLV / ciPLV.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdlib>

#include "epilogue.cuh"
#include "ps_internal.h"
#include "ptx.cuh"

namespace ps {
namespace {

constexpr int BMC = 128;       // rows per CTA (TMEM lanes)
constexpr int BN = kSplitBN;   // 128 columns (UMMA N)
constexpr int BK = kSplitBK;   // 32 samples per pipeline stage
constexpr uint32_t SWZ = (BK == 16) ? 6u : (BK == 32) ? 4u : 2u;  // 32B / 64B / 128B swizzle
constexpr uint32_t SBO = 8u * BK * 2u;                             // bytes per 8-row core group
constexpr int NEPI_WARPS = 16;
constexpr int NTHREADS = 64 + NEPI_WARPS * 32;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t BUF_COLS = 2 * BN;          // Re + Im of one accumulation buffer
constexpr int HALF = BN / (NEPI_WARPS / 4);    // columns per epilogue warp

// GS = true: the 3-multiplication (Gauss) complex Gram.  With a = Zr_i,
// b = Zi_i, c = Zr_j, d = Zi_j:  k1 = (a + b) c,  k2 = -a (c + d),
// k3 = b (c - d);  Re = k1 - k3,  Im = k1 + k2 -- 9 split UMMAs per K step
// instead of 12.  Planes 4..7 hold S = Zr + Zi and D = Zr - Zi (hi / lo);
// A stages {Zr, Zi, S} (planes 0-5), B stages {Zr} (planes 0-1) and {S, D}
// (planes 4-7).  The three accumulators of a 256 x 128 tile take 384 TMEM
// columns, so there is one accumulation buffer (the MMA waits while the
// epilogue drains a chunk, folding k1 - k3 and k1 + k2 into its Re / Im sums).
//
// CV = true (Gauss only, PS_GAUSS_CONV=1; measured slower, kept as an
// experiment): the S / D planes are not streamed.  TMA loads the
// four split planes {Zr, Zi} hi / lo of A and B (4 of the 6 smem slots, the
// same bytes per stage as the 4-product Gram) into each CTA's own full
// barrier; the epilogue warps -- idle between chunk drains -- rebuild
// S = Zr + Zi (A slots 4-5) and S, D (B slots 2-3, 4-5, over Zi) with the
// arithmetic of gauss_planes_kernel (bit-identical operands), fence the
// writes to the async proxy and arrive on rank 0's conv barrier, which the
// MMA issuer waits on instead of full.  Bit-identical to CV = false
// (tools/gauss_conv_check.py) but C5's Gram takes 88.5 ms against 52.3 ms:
// the conversion adds ~80 KB of LSU shared-memory traffic per stage against
// the 24 KB of TMA writes it saves, on an SM whose shared memory is already
// busy feeding 18 UMMAs per stage (profiles/r01_gauss_conv.txt).
// MK = true: the mask-count Gram (K7).  One E4M3 (fp8) plane per
// operand holds the unmasked indicator u(t) in {0, 1} (1 byte per sample);
// one kind::f8f6f4 UMMA (K = 32) per 32-sample stage accumulates
// T_ij = sum_t u_i(t) u_j(t) -- exact in fp32 for T < 2^24 (every partial sum
// is an integer below 2^24, so the accumulate never rounds) -- and the
// epilogue stores the per-pair counts (int32) the metric epilogue of the main
// Gram then reads instead of scanning the planes.  A stage holds 128 samples
// (128-byte operand rows, the 128B swizzle, 1024-byte 8-row groups; four K =
// 32 UMMAs per stage): TMA moves whole 128-byte row segments, 4x fewer row
// requests per sample than 32-sample stages.
template <int CG, bool GS = false, bool MK = false>
struct Geo {
  static constexpr int BNT = BN;                         // tile columns (UMMA N)
  static constexpr int H = BNT / (NEPI_WARPS / 4);       // columns per epilogue warp
  static constexpr int NACC = GS ? 3 : (MK ? 1 : 2);     // accumulators per buffer
  static constexpr int NBUF = GS ? 1 : 2;                // accumulation buffers (ping-pong when 2)
  static constexpr uint32_t BUF = NACC * BNT;            // TMEM columns per buffer
  static constexpr int NPL = GS ? 6 : (MK ? 1 : 4);      // planes staged per operand
  static constexpr int BNC = BNT / CG;                   // J-panel rows staged per CTA
  static constexpr int ES = MK ? 1 : 2;                  // operand bytes per sample
  static constexpr int KB = MK ? 4 * BK : BK;            // samples per pipeline stage
  static constexpr int A_PLANE = BMC * KB * ES;
  static constexpr int B_PLANE = BNC * KB * ES;
  static constexpr int A_BYTES = NPL * A_PLANE;
  static constexpr int B_BYTES = NPL * B_PLANE;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // per CTA
  // (GS, CG = 1: a 128-row J panel makes a 96 KB stage -- two fit the 227 KB)
  static constexpr int STAGES = MK ? 6 : GS ? (CG == 2 ? 3 : 2) : (CG == 2 ? 4 : 3);
  static_assert(STAGES * STAGE_BYTES + 1024 + 256 <= 227 * 1024, "stages must fit shared memory");
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int UMMA_M = BMC * CG;
  static_assert(NBUF * BUF <= TMEM_COLS, "the accumulation buffers must fit TMEM");
  static_assert(H % 16 == 0, "epilogue loads 16 columns at a time");
};

static_assert(2 * BUF_COLS <= TMEM_COLS, "two Re+Im buffers must fit TMEM");
static_assert(BK % 16 == 0 && BK * 2 <= 128, "BK must be a multiple of 16 within one swizzle row");
static_assert(HALF % 16 == 0, "epilogue loads 16 columns at a time");

__device__ __forceinline__ Item load_item(const Item* items, int i) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(items + i));
  return Item{v.x, v.y, v.z, v.w};
}

template <int H>
__device__ __forceinline__ void add_chunk(float (&s)[H], uint32_t taddr) {
  uint32_t v[16];
#pragma unroll
  for (int c = 0; c < H; c += 16) {
    ptx::tmem_ld_32x32b_x16(taddr + c, v);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 16; ++k) s[c + k] += __uint_as_float(v[k]);
  }
}

// Gauss drain: Re += k1 - k3, Im += k1 + k2 (accumulators at +0, +n, +2n);
// 4 columns per load keep the 2 x H register sums live without spilling
template <int H>
__device__ __forceinline__ void add_chunk_gauss(float (&re)[H], float (&im)[H], uint32_t taddr, uint32_t n) {
#pragma unroll
  for (int c = 0; c < H; c += 4) {
    uint32_t v1[4], v2[4], v3[4];
    ptx::tmem_ld_32x32b_x4(taddr + c, v1);
    ptx::tmem_ld_32x32b_x4(taddr + n + c, v2);
    ptx::tmem_ld_32x32b_x4(taddr + 2 * n + c, v3);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float k1 = __uint_as_float(v1[k]);
      re[c + k] += k1 - __uint_as_float(v3[k]);
      im[c + k] += k1 + __uint_as_float(v2[k]);
    }
  }
}

// S = Zr + Zi (and D = Zr - Zi) of 4 samples from their split hi / lo
// halves, re-split to hi / lo -- the arithmetic of gauss_planes_kernel
// (prep_kernels.cu), so the operands are bit-identical to the streamed planes
template <bool WITH_D>
__device__ __forceinline__ void gauss_split4(const uint2 rh, const uint2 rl, const uint2 ih, const uint2 il, uint2& sh,
                                             uint2& sl, uint2& dh, uint2& dl) {
  const __half* prh = reinterpret_cast<const __half*>(&rh);
  const __half* prl = reinterpret_cast<const __half*>(&rl);
  const __half* pih = reinterpret_cast<const __half*>(&ih);
  const __half* pil = reinterpret_cast<const __half*>(&il);
  __half* psh = reinterpret_cast<__half*>(&sh);
  __half* psl = reinterpret_cast<__half*>(&sl);
  __half* pdh = reinterpret_cast<__half*>(&dh);
  __half* pdl = reinterpret_cast<__half*>(&dl);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float zr = __fadd_rn(__half2float(prh[k]), __half2float(prl[k]));
    const float zi = __fadd_rn(__half2float(pih[k]), __half2float(pil[k]));
    const float S = __fadd_rn(zr, zi);
    psh[k] = __float2half_rn(S);
    psl[k] = __float2half_rn(__fsub_rn(S, __half2float(psh[k])));
    if (WITH_D) {
      const float D = __fsub_rn(zr, zi);
      pdh[k] = __float2half_rn(D);
      pdl[k] = __float2half_rn(__fsub_rn(D, __half2float(pdh[k])));
    }
  }
}

// CV feed: form the S (A) and S, D (B) slots of one landed stage in place;
// thread t of the 16 epilogue warps takes every 512th 8-byte position (the
// swizzle is the same in every plane, so the element-wise map is offset-wise)
template <class G>
__device__ __forceinline__ void gauss_convert_stage(uint8_t* sa, int t) {
  constexpr int NT = NEPI_WARPS * 32;
#pragma unroll 1
  for (int o = t * 8; o < G::A_PLANE; o += NT * 8) {
    const uint2 rh = *reinterpret_cast<const uint2*>(sa + o);
    const uint2 rl = *reinterpret_cast<const uint2*>(sa + G::A_PLANE + o);
    const uint2 ih = *reinterpret_cast<const uint2*>(sa + 2 * G::A_PLANE + o);
    const uint2 il = *reinterpret_cast<const uint2*>(sa + 3 * G::A_PLANE + o);
    uint2 sh, sl, dh, dl;
    gauss_split4<false>(rh, rl, ih, il, sh, sl, dh, dl);
    *reinterpret_cast<uint2*>(sa + 4 * G::A_PLANE + o) = sh;
    *reinterpret_cast<uint2*>(sa + 5 * G::A_PLANE + o) = sl;
  }
  uint8_t* sb = sa + G::A_BYTES;
#pragma unroll 1
  for (int o = t * 8; o < G::B_PLANE; o += NT * 8) {
    const uint2 rh = *reinterpret_cast<const uint2*>(sb + o);
    const uint2 rl = *reinterpret_cast<const uint2*>(sb + G::B_PLANE + o);
    const uint2 ih = *reinterpret_cast<const uint2*>(sb + 2 * G::B_PLANE + o);
    const uint2 il = *reinterpret_cast<const uint2*>(sb + 3 * G::B_PLANE + o);
    uint2 sh, sl, dh, dl;
    gauss_split4<true>(rh, rl, ih, il, sh, sl, dh, dl);
    *reinterpret_cast<uint2*>(sb + 2 * G::B_PLANE + o) = sh;  // over Zi (read above)
    *reinterpret_cast<uint2*>(sb + 3 * G::B_PLANE + o) = sl;
    *reinterpret_cast<uint2*>(sb + 4 * G::B_PLANE + o) = dh;
    *reinterpret_cast<uint2*>(sb + 5 * G::B_PLANE + o) = dl;
  }
}

template <int H>
__device__ __forceinline__ void store_sums(const float (&s)[H], uint32_t taddr) {
#pragma unroll
  for (int c = 0; c < H; c += 16) {
    uint32_t v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(s[c + k]);
    ptx::tmem_st_32x32b_x16(taddr + c, v);
  }
}

// Signed Re / Im outputs (cre, cim) of one interior warp slice: a second pass
// over the TMEM columns, only when requested.  inv(j) = 1 / T_ij.
template <int BN, int HALF, bool DIAG, typename InvF>
__device__ __forceinline__ void emit_signed_round(const GramParams& p, uint32_t ta, int jb, long long od, long long om,
                                                  InvF inv, bool first, bool direct, bool mirror, int div) {
  const long long N = p.N;
  const int l = threadIdx.x & 31;  // DIAG: this lane's own column in the block
#pragma unroll 1
  for (int g = 0; g < HALF; g += 4) {
    uint32_t vre[4], vim[4];
    ptx::tmem_ld_32x32b_x4(ta + g, vre);
    ptx::tmem_ld_32x32b_x4(ta + BN + g, vim);
    ptx::tmem_wait_ld();
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      float* o = static_cast<float*>(q == 0 ? p.out_cre : p.out_cim);
      if (!o) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = g + e;
        if (DIAG && c < l) continue;  // below the diagonal
        const float v = (DIAG && c == l) ? (q == 0 ? 1.0f : 0.0f)
                                         : __uint_as_float(q == 0 ? vre[e] : vim[e]) * inv(jb + c);
        const long long d = od + c;
        const float s = (first ? 0.0f : o[d]) + v;
        const float a = div == 1 ? s : mean_scale(s, div);
        if (direct) o[d] = a;
        if (mirror && (!DIAG || c > l)) o[om + (long long)c * N] = q == 1 ? -a : a;
      }
    }
  }
}

// Interior warp block of one finished round (every pair of the warp's 32
// rows x HALF columns strictly above the diagonal and inside; N % 4 == 0).
// Kept compact for the instruction cache: MASKED (per-pair counts from the K7
// Gram, p.cnt) is a template parameter, so the common unmasked loop carries
// no count code, and the ill-conditioned pairs of a column group are queued
// for refinement after the group from a bit mask (one copy of the queue code).
template <int BN, int HALF, bool MASKED, bool DIAG, bool SCALE>
__device__ __forceinline__ void emit_interior(const GramParams& p, const RoundInfo ri, uint32_t ta, int i, int jb,
                                           float inv_t) {
  // DIAG: the warp block sits on the diagonal (ib == jb): lane l's own column
  // is c == l (exact diagonal metrics), columns c < l lie below it
  const int l = threadIdx.x & 31;
  unsigned illc = 0, nind = 0;
  // ill-conditioning test of the general path, 1e-6 (|cim| are / d + 1) >
  // tol sqrt(d), multiplied through by d / 1e-6 (d > 0): no division
  const float kt = p.illcond_tol * 1e6f;
  const float tol = p.illcond_tol;
  auto inv_at = [&](int j) -> float {
    if (!MASKED || (DIAG && j <= i)) return inv_t;
    const long long cs = p.pool ? (long long)(ri.u0 / p.R) : (long long)ri.u0;
    const int te = p.cnt[cs * (long long)p.N * p.N + (long long)i * p.N + j];  // i < j
    if (te <= 0) {
      atomicOr(&p.status->flags, FLAG_EMPTY_WINDOW);
      return 0.0f;
    }
    return __frcp_rn(static_cast<float>(te));  // == 1.0f / te (correctly rounded)
  };
  // flags of one column group -> counters / refinement queue.  The group's
  // values are selected with compile-time indices (a runtime-indexed array
  // would live in local memory: every group would spill it)
  auto flush = [&](unsigned fl, int j0, const auto& m) {
    constexpr int n = sizeof(m) / sizeof(m[0]);
    while (fl) {
      const int e = __ffs(fl) - 1;
      fl &= fl - 1;
      float ci = m[0].ci;
#pragma unroll
      for (int q = 1; q < n; ++q) ci = (e == q) ? m[q].ci : ci;
      ++illc;
      if (p.refine) {
        const unsigned long long k = atomicAdd(&p.status->n_illcond, 1ull);
        if (k < (unsigned long long)p.refine_cap) {
          RefineEntry en;
          en.slot = (int)ri.slot;
          en.i = i;
          en.j = j0 + e;
          en.u0 = ri.u0;
          en.nu = ri.nu;
          en.approx = ci;
          p.refine[k] = en;
        }
      }
    }
  };
  // Element offsets of this warp slice's first direct entry (i, jb) and
  // first mirror entry (jb, i) in the slot, computed once per round: the
  // per-group addresses are 64-bit adds (the mirror column walks rows by N)
  const long long N = p.N;
  const long long soff = ri.slot * N * N;
  const long long od = soff + (long long)i * N + jb;
  const long long om = soff + (long long)jb * N + i;
  const bool mirror = ri.last && !p.slot_upper && !(p.debug_flags & 4);
  const bool direct = !(p.debug_flags & 8);
  // trial mean: the last round of a slot scales by 1 / R (mean_scale: a
  // reciprocal multiply, exact for a mean of 1; no division slow path here)
  const int div = (ri.last && p.mean_div != 1) ? p.mean_div : 1;
  const float fd = (float)div, rdv = 1.0f / fd;  // mean_scale_r operands (1, 1: identity)
  const InteriorPair dm = {1.0f, 0.0f, 0.0f, 1.0f, 0.0f, 1.0f, 0.0f, 0.0f};  // diagonal
  if (ri.first && (p.N & 7) == 0) {
    // first round of the slot: 8 columns per step, one 32-byte direct store
    // per metric (a full sector per lane) and lane-coalesced mirror stores
#pragma unroll 1
    for (int g = 0; g < HALF; g += 8) {
      uint32_t vre[8], vim[8];
      ptx::tmem_ld_32x32b_x8(ta + g, vre);
      ptx::tmem_ld_32x32b_x8(ta + BN + g, vim);
      ptx::tmem_wait_ld();
      InteriorPair m8[8];
      unsigned fl = 0;
      const int d0 = DIAG ? l - g : -1;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const InteriorPair& m = m8[e] = interior_pair(__uint_as_float(vre[e]), __uint_as_float(vim[e]), inv_at(jb + g + e));
        const bool up = !DIAG || e > d0;  // strictly above the diagonal
        nind += (up && m.d <= 0.0f && m.aim > tol) ? 1u : 0u;
        fl |= (up && m.d > 0.0f && m.aim * m.are + m.d > kt * m.d * m.d * m.rd) ? (1u << e) : 0u;
        if (DIAG && e == d0) m8[e] = dm;
      }
      if (fl) flush(fl, jb + g, m8);
      emit8_interior<DIAG, SCALE>(p, od + g, om + (long long)g * N, m8, direct, mirror, fd, rdv, d0);
    }
  } else {
#pragma unroll 1
    for (int g = 0; g < HALF; g += 4) {
      uint32_t vre[4], vim[4];
      ptx::tmem_ld_32x32b_x4(ta + g, vre);
      ptx::tmem_ld_32x32b_x4(ta + BN + g, vim);
      ptx::tmem_wait_ld();
      InteriorPair m4[4];
      unsigned fl = 0;
      const int d0 = DIAG ? l - g : -1;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const InteriorPair& m = m4[e] = interior_pair(__uint_as_float(vre[e]), __uint_as_float(vim[e]), inv_at(jb + g + e));
        const bool up = !DIAG || e > d0;
        nind += (up && m.d <= 0.0f && m.aim > tol) ? 1u : 0u;
        fl |= (up && m.d > 0.0f && m.aim * m.are + m.d > kt * m.d * m.d * m.rd) ? (1u << e) : 0u;
        if (DIAG && e == d0) m4[e] = dm;
      }
      if (fl) flush(fl, jb + g, m4);
      if (!DIAG || d0 < 4) emit4_interior<DIAG, SCALE>(p, od + g, om + (long long)g * N, m4, ri.first, direct, mirror, fd, rdv, d0);
    }
  }
  if (p.out_cre || p.out_cim)
    emit_signed_round<BN, HALF, DIAG>(p, ta, jb, od, om, inv_at, ri.first, direct, mirror, div);
  if (illc && !p.refine) atomicAdd(&p.status->n_illcond, (unsigned long long)illc);
  if (nind) atomicAdd(&p.status->n_indeterminate, (unsigned long long)nind);
}

// PLV-family epilogue of one finished round for row i and this warp's
// HALF-column slice; sums are read back 4 columns at a time from TMEM.
template <int BN, int HALF>
__device__ __forceinline__ void emit_round(const GramParams& p, const Item& w, int r, int r0, int r1, uint32_t ta,
                                           int i, int h, bool any_masked) {
  const RoundInfo ri = round_info(p, w, r, r0, r1);
  const long long Tobs = (long long)p.T * ri.nu;
  const float inv_t = 1.0f / static_cast<float>(Tobs);
  unsigned illc = 0;
  // |Re| rounded to 1 in fp32 with a clearly non-zero Im: the ciPLV
  // denominator is below the split arithmetic's resolution (reported 0,
  // counted so the caller knows to use fp64; ps_plv_result.n_indeterminate_ciplv)
  unsigned nind = 0;
  // Interior warp block: all 32 rows of this warp lie strictly above all
  // HALF columns of its slice and inside the matrix -- no per-pair diagonal /
  // bounds / mask logic (every tile off the diagonal band takes this path).
  const int lane = threadIdx.x & 31;
  const int ib = i - lane, jb = w.J * BN + h * HALF;
  // (masked samples: the interior path stays when the K7 count Gram supplied
  // per-pair counts -- one int load per pair instead of the plane scan)
  const bool interior = (!any_masked || p.cnt) && (p.N & 3) == 0 && ib + 31 < jb && jb + HALF <= p.N;
  auto inv_at = [&](int j) -> float {
    if (!any_masked) return inv_t;
    const long long te = effective_T<true>(p, ri.u0, ri.nu, i, j);
    if (te <= 0) {
      atomicOr(&p.status->flags, FLAG_EMPTY_WINDOW);
      return 0.0f;
    }
    return 1.0f / static_cast<float>(te);
  };
  // SCALE: the round that closes a trial mean divides (mean_scale); every
  // other round stores its values as they are (no per-element select)
  const bool scale = ri.last && p.mean_div != 1;
  if (interior) {
    if (any_masked) {
      if (scale) emit_interior<BN, HALF, true, false, true>(p, ri, ta, i, jb, inv_t);
      else emit_interior<BN, HALF, true, false, false>(p, ri, ta, i, jb, inv_t);
    } else {
      if (scale) emit_interior<BN, HALF, false, false, true>(p, ri, ta, i, jb, inv_t);
      else emit_interior<BN, HALF, false, false, false>(p, ri, ta, i, jb, inv_t);
    }
    return;
  }
  // every row of the block below every column: no pair i <= j to emit
  if (ib >= jb + HALF) return;
  // diagonal warp block (ib == jb) inside the matrix: the interior loops with
  // per-lane predicates (the general per-pair path below was measured to gate
  // the whole pipeline in short-K regimes: it holds its tile's accumulator
  // several times longer than an interior block, profiles/r02_session2/
  // emission_experiments.md)
  if (ib == jb && (!any_masked || p.cnt) && (p.N & 3) == 0 && jb + HALF <= p.N && !(p.debug_flags & 2048)) {
    if (any_masked) {
      if (scale) emit_interior<BN, HALF, true, true, true>(p, ri, ta, i, jb, inv_t);
      else emit_interior<BN, HALF, true, true, false>(p, ri, ta, i, jb, inv_t);
    } else {
      if (scale) emit_interior<BN, HALF, false, true, true>(p, ri, ta, i, jb, inv_t);
      else emit_interior<BN, HALF, false, true, false>(p, ri, ta, i, jb, inv_t);
    }
    return;
  }
#pragma unroll 1
  for (int g = 0; g < HALF; g += 4) {
    uint32_t vre[4], vim[4];
    ptx::tmem_ld_32x32b_x4(ta + g, vre);
    ptx::tmem_ld_32x32b_x4(ta + BN + g, vim);
    ptx::tmem_wait_ld();
    const int j0 = w.J * BN + h * HALF + g;
    // all four pairs strictly upper and inside: compute, then 16-byte RMW
    const bool vec = (p.N & 3) == 0 && i < p.N && j0 > i && j0 + 3 < p.N;
    PairMetrics<float> m4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + e;
      if (i >= p.N || j >= p.N || j < i) continue;
      PairMetrics<float>& m = m4[e];
      if (j == i) {
        m = diag_metrics<float>();
      } else {
        float it_ = inv_t;
        if (any_masked) {
          const long long te = effective_T<true>(p, ri.u0, ri.nu, i, j);
          if (te <= 0) {
            atomicOr(&p.status->flags, FLAG_EMPTY_WINDOW);
            it_ = 0.0f;
          } else {
            it_ = 1.0f / static_cast<float>(te);
          }
        }
        m = pair_metrics<float, true>(__uint_as_float(vre[e]), __uint_as_float(vim[e]), it_);
        const float are = fabsf(m.cre);
        const float d = (1.0f - are) * (1.0f + are);
        if (d <= 0.0f && m.iplv > p.illcond_tol) ++nind;
        // predicted ciPLV error for a ~1e-6 error in Re / Im: queue the pair
        // for exact FP64 recomputation (refine kernel) when it exceeds tol
        if (d > 0.0f && 1e-6f * (fabsf(m.cim) * are / d + 1.0f) > p.illcond_tol * sqrtf(d)) {
          ++illc;
          if (p.refine) {
            const unsigned long long k = atomicAdd(&p.status->n_illcond, 1ull);
            if (k < (unsigned long long)p.refine_cap) {
              RefineEntry en;
              en.slot = (int)ri.slot;
              en.i = i;
              en.j = j;
              en.u0 = ri.u0;
              en.nu = ri.nu;
              en.approx = m.ciplv;
              p.refine[k] = en;
            }
          }
        }
      }
      if (!vec) emit_all<float>(p, ri.slot, i, j, m, ri.first, ri.last);
    }
    if (vec) emit4_all(p, ri.slot, i, j0, m4, ri.first, ri.last);
  }
  if (illc && !p.refine) atomicAdd(&p.status->n_illcond, (unsigned long long)illc);
  if (nind) atomicAdd(&p.status->n_indeterminate, (unsigned long long)nind);
}

// 576 threads = 18 warps, one CTA per SM; with 5 warps on some SM sub-partition
// the register budget is 16384 / (5 * 32) -> 96 per thread.
//
// Items carry 256-row tiles (I indexes 256-row panels).  CG = 2: the pair
// covers all 256 rows.  CG = 1: item.g's high bit is unused; instead the host
// doubles the items and the low bit of I (after << 1) selects the half -- see
// launch_gram_split: for CG = 1 the host passes 128-row panel indices.
template <int CG, bool GS, bool CV, bool MK = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    gram_split_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmB2, const GramParams p) {
  using G = Geo<CG, GS, MK>;
  static_assert(!(MK && (GS || CV)), "the mask-count Gram is its own variant");
  static_assert(!CV || GS, "smem S / D conversion is a Gauss-Gram feed");
  // bytes TMA delivers per stage and CTA (CV: 4 planes of A and of B)
  constexpr int LOAD_BYTES = CV ? 4 * (G::A_PLANE + G::B_PLANE) : G::STAGE_BYTES;
  constexpr int BN = G::BNT;  // tile columns of this variant (shadows the 128-column default)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::STAGES * G::STAGE_BYTES);
  uint64_t* empty = full + G::STAGES;
  uint64_t* tfull = empty + G::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint64_t* conv = tempty + 2;          // [STAGES] (CV: operand slots complete, S / D formed)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(conv + G::STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  const int grp = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ngrp = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  int* tflag = &p.status->flags;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < G::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&conv[s], CG * NEPI_WARPS);  // one arrival per epilogue warp of the group
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], CG * NEPI_WARPS);  // one arrival per epilogue warp of the group
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    if (GS) ptx::tma_prefetch_desc(&tmB2);
  }
  if (warp == 1) {
    ptx::tmem_alloc_cg<CG>(tslot, TMEM_COLS);
    ptx::tmem_relinquish_cg<CG>();
  }
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;

  const int nk = (p.T + G::KB - 1) / G::KB;
  const int kcb = p.kc_blocks;
  const int nchunks = (nk + kcb - 1) / kcb;

  if (warp == 0) {
    // ===================== TMA producer (every CTA) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      long long w_empty = 0;
      const long long p_t0 = clock64();
      // lockstep bookkeeping (see GramParams::lock_cnt)
      const bool lock = p.lock_cnt != nullptr;
      const long long S = p.lock_group;
      const long long rk = (long long)p.lock_rounds * nk;                 // K blocks per item
      const int c_full = (p.n_items + ngrp - 1) / ngrp;                    // items of the busiest groups
      const int n_full = p.n_items - (c_full - 1) * ngrp;                  // groups with c_full items
      auto expected = [&](long long g) -> int {                            // producers that pass group g
        const long long e0 = g * S;
        if (e0 < (long long)(c_full - 1) * rk) return CG * ngrp;
        if (e0 < (long long)c_full * rk) return CG * n_full;
        return 0;
      };
      long long e = 0;  // K blocks issued by this producer
      bool pace = true;  // cleared after a pacing timeout (counters are still published)
      // next item loaded one iteration ahead (its latency off the per-item path)
      Item w_next = grp < p.n_items ? load_item(p.items, grp) : Item{0, 0, 0, 0};
      for (int it = grp; it < p.n_items; it += ngrp) {
        const Item w = w_next;
        if (it + ngrp < p.n_items) w_next = load_item(p.items, it + ngrp);
        const int r0 = p.pool ? 0 : w.g * p.Rg;
        const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
        // (debug_flags & 16: every item streams panel 0 -- operands L2-resident,
        // results meaningless; measures the kernel without DRAM operand traffic)
        const bool l2only = (p.debug_flags & 16) != 0;
        const int rowA = (l2only ? 0 : w.I * G::UMMA_M) + (int)rank * BMC;
        const int rowB = (l2only ? 0 : w.J * BN) + (int)rank * G::BNC;
        for (int r = r0; r < r1; ++r) {
          const int u = w.b * p.R + r;
          for (int kb = 0; kb < nk; ++kb) {
            if (lock && e > 0 && e % S == 0) {
              const long long g = e / S;
              atomicAdd(&p.lock_cnt[g - 1], 1);  // group g-1 fully issued
              if (pace && g - p.lock_lag >= 0) {
                const long long gw = g - p.lock_lag;
                const int need = expected(gw);
                const long long t0 = clock64();
                while (ptx::ld_acquire_gpu(&p.lock_cnt[gw]) < need) {
                  __nanosleep(256);
                  // pacing only, never a hang: if the others do not show up
                  // within ~0.2 s (CTAs not co-resident, e.g. the GPU is
                  // shared) this producer stops pacing for the rest of the launch
                  if (clock64() - t0 > 400000000LL) {
                    pace = false;
                    break;
                  }
                }
              }
            }
            ++e;
            if (p.prof) ptx::mbar_wait_prof(&empty[stage], phase ^ 1u, &w_empty);
            else ptx::mbar_wait(&empty[stage], phase ^ 1u, tflag);
            uint8_t* sa = smem + stage * G::STAGE_BYTES;
            if (p.debug_flags & 64) {
              // experiment (PS_DEBUG_EPI=64): no operand loads at all -- the
              // stage is released without TMA, so the kernel times the MMA /
              // epilogue pipeline alone (values meaningless)
              if (CG == 1 || rank == 0) ptx::mbar_arrive(&full[stage]);
            } else if (CV) {
              // each CTA counts its own 4 + 4 planes; its epilogue warps convert
              ptx::mbar_arrive_expect_tx(&full[stage], LOAD_BYTES);
              ptx::tma_load_4d(sa, &tmA, &full[stage], kb * G::KB, rowA, u, 0);
              ptx::tma_load_4d(sa + G::A_BYTES, &tmB, &full[stage], kb * G::KB, rowB, u, 0);
            } else if (CG == 1) {
              ptx::mbar_arrive_expect_tx(&full[stage], G::STAGE_BYTES);
              ptx::tma_load_4d(sa, &tmA, &full[stage], kb * G::KB, rowA, u, 0);
              ptx::tma_load_4d(sa + G::A_BYTES, &tmB, &full[stage], kb * G::KB, rowB, u, 0);
              if (GS) ptx::tma_load_4d(sa + G::A_BYTES + 2 * G::B_PLANE, &tmB2, &full[stage], kb * G::KB, rowB, u, 4);
            } else {
              // rank 0's full barrier counts the bytes of both CTAs
              if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * G::STAGE_BYTES);
              ptx::tma_load_4d_cg2(sa, &tmA, &full[stage], kb * G::KB, rowA, u, 0);
              ptx::tma_load_4d_cg2(sa + G::A_BYTES, &tmB, &full[stage], kb * G::KB, rowB, u, 0);
              if (GS)
                ptx::tma_load_4d_cg2(sa + G::A_BYTES + 2 * G::B_PLANE, &tmB2, &full[stage], kb * G::KB, rowB, u, 4);
            }
            if (p.prefetch_blocks > 0 && !(p.debug_flags & 64)) {
              const int kp = kb + p.prefetch_blocks;
              if (kp < nk) {
                ptx::tma_prefetch_4d(&tmA, kp * G::KB, rowA, u, 0);
                ptx::tma_prefetch_4d(&tmB, kp * G::KB, rowB, u, 0);
                if (GS && !CV) ptx::tma_prefetch_4d(&tmB2, kp * G::KB, rowB, u, 4);
              }
            }
            if (++stage == G::STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      if (lock && e > 0) atomicAdd(&p.lock_cnt[(e - 1) / S], 1);  // last (possibly partial) group
      if (p.prof) {
        atomicAdd(&p.prof[3], (unsigned long long)w_empty);
        atomicAdd(&p.prof[4], (unsigned long long)(clock64() - p_t0));
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (rank 0) =====================
    if (rank == 0) {  // whole warp: uniform descriptors, one elected lane issues
      // PS_DEBUG_EPI & 128: the 4-product K step as 12 separately elected
      // UMMAs (the previous issue form; experiments)
      const bool mma_split_issue = (p.debug_flags & 128) != 0;
      constexpr uint32_t idesc_pos = ptx::make_idesc_f16(G::UMMA_M, BN, false);
      constexpr uint32_t idesc_neg = ptx::make_idesc_f16(G::UMMA_M, BN, true);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t uses[2] = {0u, 0u};
      int buf = 0;
      long long w_full = 0, w_tempty = 0;
      const long long m_t0 = clock64();
      // next item loaded one iteration ahead (its latency off the per-item path)
      Item w_next = grp < p.n_items ? load_item(p.items, grp) : Item{0, 0, 0, 0};
      for (int it = grp; it < p.n_items; it += ngrp) {
        const Item w = w_next;
        if (it + ngrp < p.n_items) w_next = load_item(p.items, it + ngrp);
        const int r0 = p.pool ? 0 : w.g * p.Rg;
        const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
        for (int r = r0; r < r1; ++r) {
          for (int kb = 0; kb < nk; ++kb) {
            const bool chunk_start = (kb % kcb) == 0;
            const bool chunk_end = (kb % kcb) == kcb - 1 || kb == nk - 1;
            if (chunk_start) {
              if (p.prof) ptx::mbar_wait_prof(&tempty[buf], (uses[buf] & 1u) ^ 1u, &w_tempty);
              else ptx::mbar_wait(&tempty[buf], (uses[buf] & 1u) ^ 1u, tflag);
              ptx::tc_fence_after();
            }
            // __shfl_sync makes the operands provably warp-uniform, so ptxas
            // keeps them in uniform registers for UTCHMMA
            const uint32_t d_re = __shfl_sync(0xffffffffu, tmem + (uint32_t)buf * G::BUF, 0);
            const uint32_t d_im = d_re + BN;
            if (CV) ptx::mbar_wait_cluster(&conv[stage], phase);
            else if (p.prof) ptx::mbar_wait_prof(&full[stage], phase, &w_full);
            else ptx::mbar_wait(&full[stage], phase, tflag);
            ptx::tc_fence_after();
            // descriptor of the stage's A tile; planes / K sub-steps are
            // constant offsets added to the 14-bit start-address field
            // (smem addresses < 256 KB never carry out of it)
            const uint32_t sa_u = __shfl_sync(0xffffffffu, ptx::smem_u32(smem + stage * G::STAGE_BYTES), 0);
            const uint64_t dA = ptx::make_smem_desc(sa_u, SBO, SWZ);
            const uint64_t dB = dA + (uint64_t)(G::A_BYTES >> 4);
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks) {
              const uint64_t ko = (uint64_t)(ks * 32) >> 4;  // 16 fp16 = 32 bytes along K
              const uint64_t aRh = dA + ko + 0 * (G::A_PLANE >> 4);
              const uint64_t aRl = dA + ko + 1 * (G::A_PLANE >> 4);
              const uint64_t aIh = dA + ko + 2 * (G::A_PLANE >> 4);
              const uint64_t aIl = dA + ko + 3 * (G::A_PLANE >> 4);
              const uint64_t bRh = dB + ko + 0 * (G::B_PLANE >> 4);
              const uint64_t bRl = dB + ko + 1 * (G::B_PLANE >> 4);
              const uint64_t bIh = dB + ko + 2 * (G::B_PLANE >> 4);  // GS: S hi
              const uint64_t bIl = dB + ko + 3 * (G::B_PLANE >> 4);  // GS: S lo
              const uint32_t acc0 = (chunk_start && ks == 0) ? 0u : 1u;
              if constexpr (MK) {
                // T_ij += u_i . u_j over the stage's 128 samples: four fp8
                // UMMAs (K = 32), each 32 bytes further along the swizzled rows
                if (ks == 0) {
                  const uint64_t a8 = ptx::make_smem_desc(sa_u, 8u * G::KB, 2u);  // 128B swizzle
                  const uint64_t b8 = a8 + (uint64_t)(G::A_BYTES >> 4);
#pragma unroll
                  for (int k8 = 0; k8 < G::KB / 32; ++k8)
                    ptx::mma_f8_ss_warp<CG>(d_re, a8 + 2 * k8, b8 + 2 * k8, idesc_pos, (chunk_start && k8 == 0) ? 0u : 1u);
                }
              } else if constexpr (GS) {
               if (!mma_split_issue) {
                // one elected block per K step (9 UMMAs, see mma_gauss_step_warp)
                const uint32_t alo = (uint32_t)dA + (uint32_t)ko, blo = (uint32_t)dB + (uint32_t)ko;
                constexpr uint32_t AP = G::A_PLANE >> 4, BP = G::B_PLANE >> 4;
                const uint32_t av[6] = {alo, alo + AP, alo + 2 * AP, alo + 3 * AP, alo + 4 * AP, alo + 5 * AP};
                const uint32_t bv[6] = {blo, blo + BP, blo + 2 * BP, blo + 3 * BP, blo + 4 * BP, blo + 5 * BP};
                ptx::mma_gauss_step_warp<CG>(d_re, d_im, d_re + 2 * BN, av, bv, (uint32_t)(dA >> 32), idesc_pos,
                                             idesc_neg, acc0);
               } else {
                const uint64_t aSh = dA + ko + 4 * (G::A_PLANE >> 4);
                const uint64_t aSl = dA + ko + 5 * (G::A_PLANE >> 4);
                const uint64_t bDh = dB + ko + 4 * (G::B_PLANE >> 4);
                const uint64_t bDl = dB + ko + 5 * (G::B_PLANE >> 4);
                const uint32_t d_k3 = d_re + 2 * BN;
                // k1 = S_i . Zr_j   (accumulator 0)
                ptx::mma_f16_ss_warp<CG>(d_re, aSh, bRh, idesc_pos, acc0);
                ptx::mma_f16_ss_warp<CG>(d_re, aSh, bRl, idesc_pos, 1u);
                ptx::mma_f16_ss_warp<CG>(d_re, aSl, bRh, idesc_pos, 1u);
                // k2 = -Zr_i . S_j  (accumulator 1)
                ptx::mma_f16_ss_warp<CG>(d_im, aRh, bIh, idesc_neg, acc0);
                ptx::mma_f16_ss_warp<CG>(d_im, aRh, bIl, idesc_neg, 1u);
                ptx::mma_f16_ss_warp<CG>(d_im, aRl, bIh, idesc_neg, 1u);
                // k3 = Zi_i . D_j   (accumulator 2)
                ptx::mma_f16_ss_warp<CG>(d_k3, aIh, bDh, idesc_pos, acc0);
                ptx::mma_f16_ss_warp<CG>(d_k3, aIh, bDl, idesc_pos, 1u);
                ptx::mma_f16_ss_warp<CG>(d_k3, aIl, bDh, idesc_pos, 1u);
               }
              } else if (!mma_split_issue) {
                // one elected block per K step (12 UMMAs, see mma_4prod_step_warp)
                const uint32_t alo = (uint32_t)dA + (uint32_t)ko, blo = (uint32_t)dB + (uint32_t)ko;
                const uint32_t av[4] = {alo, alo + (G::A_PLANE >> 4), alo + 2 * (G::A_PLANE >> 4),
                                        alo + 3 * (G::A_PLANE >> 4)};
                const uint32_t bv[4] = {blo, blo + (G::B_PLANE >> 4), blo + 2 * (G::B_PLANE >> 4),
                                        blo + 3 * (G::B_PLANE >> 4)};
                ptx::mma_4prod_step_warp<CG>(d_re, d_im, av, bv, (uint32_t)(dA >> 32), idesc_pos, idesc_neg, acc0);
              } else {
                // Re = Zr Zr' + Zi Zi'
                ptx::mma_f16_ss_warp<CG>(d_re, aRh, bRh, idesc_pos, acc0);
                ptx::mma_f16_ss_warp<CG>(d_re, aRh, bRl, idesc_pos, 1u);
                ptx::mma_f16_ss_warp<CG>(d_re, aRl, bRh, idesc_pos, 1u);
                ptx::mma_f16_ss_warp<CG>(d_re, aIh, bIh, idesc_pos, 1u);
                ptx::mma_f16_ss_warp<CG>(d_re, aIh, bIl, idesc_pos, 1u);
#ifndef PS_EXPERIMENT_9MMA  // (timing experiment only: 9 of the 12 UMMAs, wrong values)
                ptx::mma_f16_ss_warp<CG>(d_re, aIl, bIh, idesc_pos, 1u);
#endif
                // Im = Zi Zr' - Zr Zi'
                ptx::mma_f16_ss_warp<CG>(d_im, aIh, bRh, idesc_pos, acc0);
                ptx::mma_f16_ss_warp<CG>(d_im, aIh, bRl, idesc_pos, 1u);
#ifndef PS_EXPERIMENT_9MMA
                ptx::mma_f16_ss_warp<CG>(d_im, aIl, bRh, idesc_pos, 1u);
#endif
                ptx::mma_f16_ss_warp<CG>(d_im, aRh, bIh, idesc_neg, 1u);
                ptx::mma_f16_ss_warp<CG>(d_im, aRh, bIl, idesc_neg, 1u);
#ifndef PS_EXPERIMENT_9MMA
                ptx::mma_f16_ss_warp<CG>(d_im, aRl, bIh, idesc_neg, 1u);
#endif
              }
            }
            ptx::mma_commit_warp<CG>(&empty[stage]);  // the group's smem slots free once these retire
            if (++stage == G::STAGES) {
              stage = 0;
              phase ^= 1u;
            }
            if (chunk_end) {
              ptx::mma_commit_warp<CG>(&tfull[buf]);  // chunk partial complete -> epilogues
              uses[buf]++;
              if (G::NBUF == 2) buf ^= 1;
            }
          }
        }
      }
      if (p.prof && lane == 0) {
        atomicAdd(&p.prof[0], (unsigned long long)w_full);
        atomicAdd(&p.prof[1], (unsigned long long)w_tempty);
        atomicAdd(&p.prof[2], (unsigned long long)(clock64() - m_t0));
      }
    }
  } else {
    // ===================== epilogue (warps 2..17, every CTA) =====================
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    const int h = (warp - 2) >> 2;    // column slice
    const int il = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t uses[2] = {0u, 0u};
    int buf = 0;
    int cst = 0;        // CV: stage / phase of the next stage to convert
    uint32_t cph = 0u;
    const int ct = (warp - 2) * 32 + lane;
    const bool any_masked = (p.status->flags & FLAG_ANY_MASKED) != 0;
    constexpr int H = G::H;
    // register sums of Re / Im (GS: folded from k1, k2, k3 at every drain)
    float sre[H], sim[H];
#pragma unroll
    for (int k = 0; k < H; ++k) sre[k] = sim[k] = 0.0f;
    long long e_wait = 0, e_emit = 0;  // PS_GRAM_PROF: cycles blocked on tfull / emitting
    const long long e_t0 = p.prof ? clock64() : 0;
    // next item loaded one iteration ahead (its latency off the per-item path)
    Item w_next = grp < p.n_items ? load_item(p.items, grp) : Item{0, 0, 0, 0};
    for (int it = grp; it < p.n_items; it += ngrp) {
      const Item w = w_next;
      if (it + ngrp < p.n_items) w_next = load_item(p.items, it + ngrp);
      const int r0 = p.pool ? 0 : w.g * p.Rg;
      const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
      const int i = w.I * G::UMMA_M + (int)rank * BMC + il;
      for (int r = r0; r < r1; ++r) {
        for (int c = 0; c < nchunks; ++c) {
          if constexpr (CV) {
            // form S / D of this chunk's stages as they land (the MMA issuer
            // waits on conv); the chunk's drain follows below
            const int kb1 = min(nk, (c + 1) * kcb);
            for (int kb = c * kcb; kb < kb1; ++kb) {
              ptx::mbar_wait(&full[cst], cph, tflag);
              gauss_convert_stage<G>(smem + cst * G::STAGE_BYTES, ct);
              ptx::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                if (CG == 2) ptx::mbar_arrive_rank0_cluster(&conv[cst]);
                else ptx::mbar_arrive(&conv[cst]);
              }
              if (++cst == G::STAGES) {
                cst = 0;
                cph ^= 1u;
              }
            }
          }
          if (p.prof) ptx::mbar_wait_prof(&tfull[buf], uses[buf] & 1u, &e_wait);
          else ptx::mbar_wait(&tfull[buf], uses[buf] & 1u, tflag);
          ptx::tc_fence_after();
          const uint32_t ta = tmem + lane_base + (uint32_t)buf * G::BUF + (uint32_t)(h * H);
          // single-chunk rounds (short K: over_trials, coherence, T <= 128):
          // the chunk accumulator already is the round's sum (0 + x = x), so
          // it is emitted in place -- no drain / park round trip through TMEM
          const bool direct = !GS && !MK && nchunks == 1 && !p.pool;
          if (!direct) {
            if constexpr (GS) {
              add_chunk_gauss<H>(sre, sim, ta, BN);
            } else if constexpr (MK) {
              add_chunk<H>(sre, ta);
            } else {
              add_chunk<H>(sre, ta);
              add_chunk<H>(sim, ta + BN);
            }
          }
          if (MK && c == nchunks - 1 && (!p.pool || r == r1 - 1)) {
            // per-pair observation counts of this round's unit (pool: of the
            // band) -> p.cnt[slot][i][j], every in-bounds pair of the tile
            if (i < p.N) {
              const long long cs = p.pool ? (long long)w.b : (long long)w.b * p.R + r;
              int* dst = p.cnt + cs * (long long)p.N * p.N + (long long)i * p.N;
              const int jb = w.J * BN + h * H;
              if ((p.N & 3) == 0 && jb + H <= p.N) {
#pragma unroll
                for (int k = 0; k < H; k += 4)
                  *reinterpret_cast<int4*>(dst + jb + k) =
                      make_int4((int)sre[k], (int)sre[k + 1], (int)sre[k + 2], (int)sre[k + 3]);
              } else {
#pragma unroll
                for (int k = 0; k < H; ++k)
                  if (jb + k < p.N) dst[jb + k] = (int)sre[k];
              }
            }
#pragma unroll
            for (int k = 0; k < H; ++k) sre[k] = 0.0f;
          } else if (!MK && c == nchunks - 1 && (!p.pool || r == r1 - 1)) {
            // Round complete: park the fp32 sums back in this (still owned)
            // TMEM buffer and emit from there with a compact loop, so the
            // register sums are dead during the store-heavy epilogue.
            if (!direct) {
              store_sums<H>(sre, ta);
              store_sums<H>(sim, ta + BN);
              ptx::tmem_wait_st();
            }
            const long long t_em = p.prof ? clock64() : 0;
            if (!(p.debug_flags & 1)) emit_round<BN, H>(p, w, r, r0, r1, ta, i, h, any_masked);
            if (p.prof) e_emit += clock64() - t_em;
#pragma unroll
            for (int k = 0; k < H; ++k) sre[k] = sim[k] = 0.0f;  // sums dead across the emission
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2) ptx::mbar_arrive_rank0(&tempty[buf]);
            else ptx::mbar_arrive(&tempty[buf]);
          }
          uses[buf]++;
          if (G::NBUF == 2) buf ^= 1;
        }
      }
      if (p.sb_cnt) {  // item emitted by this warp: count it towards its output sub-block
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          const int sb = p.item_sb[it];
          if (atomicAdd(&p.sb_cnt[sb], 1) == p.sb_need[sb] - 1) {
            __threadfence_system();
            p.sb_flag[sb] = 1;
          }
        }
      }
    }
    if (p.prof && lane == 0) {
      atomicAdd(&p.prof[5], (unsigned long long)e_wait);
      atomicAdd(&p.prof[6], (unsigned long long)e_emit);
      atomicAdd(&p.prof[7], (unsigned long long)(clock64() - e_t0));
    }
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // both CTAs done with TMEM and remote barriers
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg<CG>(tmem, TMEM_COLS);
  }
}

template <int CG, bool GS, bool CV = false, bool MK = false>
cudaError_t launch_cg(const void* tmapA, const void* tmapB, const void* tmapB2, const GramParams& p, int groups,
                      cudaStream_t st) {
  using G = Geo<CG, GS, MK>;
  cudaError_t e = cudaFuncSetAttribute(gram_split_kernel<CG, GS, CV, MK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       G::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (p.n_items <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * CG);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = G::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gram_split_kernel<CG, GS, CV, MK>, *static_cast<const CUtensorMap*>(tmapA),
                            *static_cast<const CUtensorMap*>(tmapB),
                            *static_cast<const CUtensorMap*>(tmapB2 ? tmapB2 : tmapB), p);
}

}  // namespace

bool gauss_smem_convert() {
  static const bool cv = [] {
    const char* s = std::getenv("PS_GAUSS_CONV");
    return s && std::atoi(s) != 0;
  }();
  return cv;
}

int split_cta_group() {
  static const int cg = [] {
    const char* s = std::getenv("PS_CTA_GROUP");
    return (s && std::atoi(s) == 1) ? 1 : 2;
  }();
  return cg;
}

int split_panel_rows() { return split_cta_group() * BMC; }

int split_b_box_rows() { return BN / split_cta_group(); }

int split_epi_arrivals() { return NEPI_WARPS * split_cta_group(); }

cudaError_t launch_gram_split(const void* tmapA, const void* tmapB, const void* tmapB2, bool gauss,
                              const GramParams& p, int groups, cudaStream_t st) {
  if (gauss && gauss_smem_convert())
    return split_cta_group() == 2 ? launch_cg<2, true, true>(tmapA, tmapB, nullptr, p, groups, st)
                                  : launch_cg<1, true, true>(tmapA, tmapB, nullptr, p, groups, st);
  if (gauss)
    return split_cta_group() == 2 ? launch_cg<2, true>(tmapA, tmapB, tmapB2, p, groups, st)
                                  : launch_cg<1, true>(tmapA, tmapB, tmapB2, p, groups, st);
  return split_cta_group() == 2 ? launch_cg<2, false>(tmapA, tmapB, nullptr, p, groups, st)
                                : launch_cg<1, false>(tmapA, tmapB, nullptr, p, groups, st);
}

cudaError_t launch_gram_count(const void* tmapA, const void* tmapB, const GramParams& p, int groups, cudaStream_t st) {
  return split_cta_group() == 2 ? launch_cg<2, false, false, true>(tmapA, tmapB, nullptr, p, groups, st)
                                : launch_cg<1, false, false, true>(tmapA, tmapB, nullptr, p, groups, st);
}

}  // namespace ps
