// Fused PLV / iPLV / ciPLV epilogue shared by the two Gram kernels.
//
// Given one Gram entry G_ij = sum_t z_i(t) conj(z_j(t)) (Eq 7)
// and the effective observation count T_ij, emit the requested
// metrics straight from the accumulator registers -- the complex N x N Gram
// never round-trips HBM (north star (3)).
//   PLV   = |G|/T                          Eq 7
//   iPLV  = |Im G|/T                       Eq 13  SPEC.md:198, abs per :258
//   ciPLV = |Im|/sqrt(1 - Re^2)            Eq 14  SPEC.md:207, singular -> 0 :259
// Diagonal: PLV = 1, iPLV = ciPLV = 0.
#pragma once
#include <cuda_fp16.h>
#include "ps_internal.h"

namespace ps {

template <typename S>
struct PairMetrics {
  S plv, iplv, ciplv, cre, cim;
};

// SPLIT: fp32 path. 1 - Re^2 is formed as (1-|Re|)(1+|Re|) (exact for
// |Re| >= 1/2), PLV and ciPLV are clamped to <= 1; the SPEC's
// 1e-12 singularity threshold is below fp32 resolution, so "singular" means
// 1 - |Re| rounds to <= 0.  FP64 path: the SPEC rule verbatim.
template <typename S, bool SPLIT>
__device__ __forceinline__ PairMetrics<S> pair_metrics(S gre, S gim, S inv_t) {
  PairMetrics<S> m;
  const S cre = gre * inv_t, cim = gim * inv_t;
  const S are = fabs(cre), aim = fabs(cim);
  S plv;
  S ci;
  if (SPLIT) {
    // MUFU.RSQ-based magnitude and ciPLV denominator: ~2 ulp, far below the
    // 1e-5 budget, and no IEEE sqrt / division sequences in the epilogue
    const S ss = cre * cre + cim * cim;
    plv = ss * rsqrtf(fmaxf(ss, S(1e-30)));  // < 1e-15 off below the clamp, exact 0 at 0
    plv = plv > S(1) ? S(1) : plv;
    const S d = (S(1) - are) * (S(1) + are);
    ci = d > S(0) ? aim * rsqrtf(d) : S(0);
    ci = ci > S(1) ? S(1) : ci;
  } else {
    plv = sqrt(cre * cre + cim * cim);
    ci = (are >= S(1) - S(1e-12)) ? S(0) : aim / sqrt(S(1) - cre * cre);
    // |Im|^2 <= 1 - Re^2 (Cauchy-Schwarz); near the singularity rounding can
    // still push the quotient past 1 -- keep the SPEC.md:150 bound
    ci = ci > S(1) ? S(1) : ci;
  }
  m.plv = plv;
  m.iplv = aim;
  m.ciplv = ci;
  m.cre = cre;
  m.cim = cim;
  return m;
}

template <typename S>
__device__ __forceinline__ PairMetrics<S> diag_metrics() {
  PairMetrics<S> m;
  m.plv = S(1);
  m.iplv = S(0);
  m.ciplv = S(0);
  m.cre = S(1);
  m.cim = S(0);
  return m;
}

// Is sample t of row `row` masked?  Masked samples are exactly 0 in every
// plane; an unmasked unit phasor has max(|re|,|im|) >= 1/sqrt(2), so its hi
// parts can never both be zero.
template <bool SPLIT>
__device__ __forceinline__ bool sample_masked(const void* planes, long long plane_stride, long long idx) {
  if (SPLIT) {
    const __half* h = static_cast<const __half*>(planes);
    return __half2float(h[idx]) == 0.0f && __half2float(h[2 * plane_stride + idx]) == 0.0f;
  } else {
    const double* d = static_cast<const double*>(planes);
    return d[idx] == 0.0 && d[plane_stride + idx] == 0.0;
  }
}

// Samples masked in both rows (only when both rows have masked samples).
template <bool SPLIT>
__device__ __noinline__ int masked_overlap(const void* planes, long long plane_stride, long long ri, long long rj,
                                           int T, int Tp) {
  int both = 0;
  for (int t = 0; t < T; ++t)
    both += (sample_masked<SPLIT>(planes, plane_stride, ri * Tp + t) &&
             sample_masked<SPLIT>(planes, plane_stride, rj * Tp + t))
                ? 1
                : 0;
  return both;
}

// Effective observation count of pair (i, j) over units [u0, u0 + nu)
// (SPEC.md:260): samples unmasked in both signals.  Only called when the
// fixup kernel reported masked samples.
template <bool SPLIT>
__device__ __forceinline__ long long effective_T(const GramParams& p, int u0, int nu, int i, int j) {
  if (p.cnt) {  // K7 count Gram ran: one load (pool: the band's slot already sums its units)
    const long long cs = p.pool ? (long long)(u0 / p.R) : (long long)u0;
    const int a = i < j ? i : j, b = i < j ? j : i;
    return p.cnt[cs * (long long)p.N * p.N + (long long)a * p.N + b];
  }
  long long tot = 0;
  for (int u = u0; u < u0 + nu; ++u) {
    const long long ri = (long long)u * p.N + i, rj = (long long)u * p.N + j;
    const int mi = p.maskcount[ri], mj = p.maskcount[rj];
    long long c = (long long)p.T - mi - mj;
    if (mi > 0 && mj > 0) c += masked_overlap<SPLIT>(p.planes, p.plane_stride, ri, rj, p.T, p.Tp);
    tot += c;
  }
  return tot;
}

// Trial-mean scaling at the last round of a slot: split (fp32) outputs are
// multiplied by the fp32 reciprocal 1 / R on every path that forms a mean
// (interior and general epilogues, trial-group reduce), so any two paths
// that sum the same terms produce bit-identical means; FP64 divides.
// A sum equal to the divisor is an exact mean of 1 (every diagonal entry of
// PLV / cre; SPEC.md:194 wants the self-pair PLV exactly 1) -- R * fl(1 / R)
// alone can round below 1 (fp32: R = 41, 47, 55, ...).
__device__ __forceinline__ float mean_scale(float acc, int div) {
  const float d = (float)div;
  return acc == d ? 1.0f : acc * (1.0f / d);
}
__device__ __forceinline__ double mean_scale(double acc, int div) { return acc / (double)div; }
// The same with fd = (float)div and rd = 1 / fd precomputed (fd = rd = 1: the
// identity), branch-free for the emission loops.
__device__ __forceinline__ float mean_scale_r(float acc, float fd, float rd) { return acc == fd ? 1.0f : acc * rd; }

// Accumulating store of one metric value into slot `base` at (i, j); the
// mirror (j, i) is written at the last round of the slot (negated for the
// antisymmetric signed imaginary part).
template <typename S>
__device__ __forceinline__ void emit(S* base, long long N, int i, int j, S v, bool first, bool last, int div,
                                     bool anti, bool mirror) {
  const long long idx = (long long)i * N + j;
  S acc = first ? v : base[idx] + v;
  if (last && div != 1) acc = mean_scale(acc, div);
  base[idx] = acc;
  if (mirror && last && i != j) base[(long long)j * N + i] = anti ? -acc : acc;
}

template <typename S>
__device__ __forceinline__ void emit_all(const GramParams& p, long long slot, int i, int j,
                                         const PairMetrics<S>& m, bool first, bool last) {
  const long long off = slot * (long long)p.N * p.N;
  const long long N = p.N;
  if (p.out_plv) emit<S>(static_cast<S*>(p.out_plv) + off, N, i, j, m.plv, first, last, p.mean_div, false, !p.slot_upper);
  if (p.out_iplv) emit<S>(static_cast<S*>(p.out_iplv) + off, N, i, j, m.iplv, first, last, p.mean_div, false, !p.slot_upper);
  if (p.out_ciplv)
    emit<S>(static_cast<S*>(p.out_ciplv) + off, N, i, j, m.ciplv, first, last, p.mean_div, false, !p.slot_upper);
  if (p.out_cre) emit<S>(static_cast<S*>(p.out_cre) + off, N, i, j, m.cre, first, last, p.mean_div, false, !p.slot_upper);
  if (p.out_cim) emit<S>(static_cast<S*>(p.out_cim) + off, N, i, j, m.cim, first, last, p.mean_div, true, !p.slot_upper);
}

// Four consecutive columns j0..j0+3 of row i, all strictly above the diagonal
// and inside the matrix (caller checks; needs N % 4 == 0 for 16-byte rows):
// one 16-byte read-modify-write per metric for the direct part, all reads
// issued before any write so their latencies overlap; mirror writes are
// coalesced across the warp's lanes (consecutive i).
__device__ __forceinline__ void emit4_all(const GramParams& p, long long slot, int i, int j0,
                                          const PairMetrics<float> (&m)[4], bool first, bool last) {
  const long long N = p.N;
  const long long off = slot * N * N;
  float* outs[5] = {static_cast<float*>(p.out_plv), static_cast<float*>(p.out_iplv),
                    static_cast<float*>(p.out_ciplv), static_cast<float*>(p.out_cre),
                    static_cast<float*>(p.out_cim)};
  float4 prev[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    prev[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (outs[q] && !first) prev[q] = *reinterpret_cast<const float4*>(outs[q] + off + (long long)i * N + j0);
  }
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    if (!outs[q]) continue;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = q == 0 ? m[e].plv : q == 1 ? m[e].iplv : q == 2 ? m[e].ciplv : q == 3 ? m[e].cre : m[e].cim;
    float4 a = make_float4(prev[q].x + v[0], prev[q].y + v[1], prev[q].z + v[2], prev[q].w + v[3]);
    if (last && p.mean_div != 1) {
      const int d = p.mean_div;
      a = make_float4(mean_scale(a.x, d), mean_scale(a.y, d), mean_scale(a.z, d), mean_scale(a.w, d));
    }
    float* base = outs[q] + off;
    if (!(p.debug_flags & 8)) *reinterpret_cast<float4*>(base + (long long)i * N + j0) = a;
    if (last && !p.slot_upper && !(p.debug_flags & 4)) {
      const float s = q == 4 ? -1.f : 1.f;
      base[(long long)(j0 + 0) * N + i] = s * a.x;
      base[(long long)(j0 + 1) * N + i] = s * a.y;
      base[(long long)(j0 + 2) * N + i] = s * a.z;
      base[(long long)(j0 + 3) * N + i] = s * a.w;
    }
  }
}

// 32-byte global accesses (STG.E.256 / LDG.E.256 on sm_100a)
__device__ __forceinline__ void st_v8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
// Interior warp blocks (every pair strictly above the diagonal and inside,
// no masks or K7 counts): the split metrics of one pair plus the quantities
// the ill-conditioning test reuses (one MUFU.RSQ of 1 - Re^2 serves both the
// ciPLV denominator and the test).  Same arithmetic as pair_metrics<float, true>.
struct InteriorPair {
  float plv, aim, ci, cre, cim;  // aim = iPLV
  float are, d, rd;              // |Re|, 1 - Re^2, rsqrt(1 - Re^2) (for the test)
};

__device__ __forceinline__ InteriorPair interior_pair(float gre, float gim, float inv_t) {
  InteriorPair m;
  m.cre = gre * inv_t;
  m.cim = gim * inv_t;
  m.are = fabsf(m.cre);
  m.aim = fabsf(m.cim);
  const float ss = m.cre * m.cre + m.cim * m.cim;
  const float plv = ss * rsqrtf(fmaxf(ss, 1e-30f));
  m.plv = plv > 1.0f ? 1.0f : plv;
  m.d = (1.0f - m.are) * (1.0f + m.are);
  m.rd = rsqrtf(m.d);
  const float ci = m.d > 0.0f ? m.aim * m.rd : 0.0f;
  m.ci = ci > 1.0f ? 1.0f : ci;
  return m;
}


// Eight consecutive columns of one row in the FIRST round of their slot
// (plain stores, nothing to accumulate; N % 8 == 0): element offsets od of
// the direct entry (i, j0) and om of the mirror entry (j0, i).  One 32-byte
// store per metric for the direct part (a full sector per lane), mirror
// stores coalesced across the warp's lanes (consecutive i), their addresses
// stepped by one row (N) per column.  fd / rd = the trial-mean divisor at
// the last round of a slot and its reciprocal (else 1 / 1; mean_scale_r).  PLV / iPLV / ciPLV only: the signed
// Re / Im outputs (rarely requested) go through emit_signed_round, outside
// the hot loop, so the loop body stays small enough for the instruction
// cache.  DIAG (a warp block on the diagonal): column e of the group is this
// lane's own column at e == d0; entries e < d0 lie below the diagonal (not
// written), the mirror is written for e > d0 only.
template <bool DIAG = false, bool SCALE = true>
__device__ __forceinline__ void emit8_interior(const GramParams& p, long long od, long long om,
                                               const InteriorPair (&m)[8], bool direct, bool mirror, float fd,
                                               float rd, int d0 = -1) {
  const long long N = p.N;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    float* o = static_cast<float*>(q == 0 ? p.out_plv : q == 1 ? p.out_iplv : p.out_ciplv);
    if (!o) continue;
    float a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = q == 0 ? m[e].plv : q == 1 ? m[e].aim : m[e].ci;
      a[e] = SCALE ? mean_scale_r(v, fd, rd) : v;
    }
    if (direct) {
      if (!DIAG || d0 <= 0) {
        st_v8(o + od, a);
      } else if (d0 < 8) {
#pragma unroll
        for (int e = 1; e < 8; ++e)
          if (e >= d0) o[od + e] = a[e];
      }
    }
    if (mirror) {
      float* mp = o + om;
#pragma unroll
      for (int e = 0; e < 8; ++e, mp += N)
        if (!DIAG || e > d0) *mp = a[e];
    }
  }
}

// Four consecutive columns of one row (N % 4 == 0), any round: one 16-byte
// read-modify-write per metric for the direct part, all reads issued before
// any write so their latencies overlap; mirror writes (last round) as in
// emit8_interior.  DIAG as there (entries below the diagonal are read with
// the row but never written).
template <bool DIAG = false, bool SCALE = true>
__device__ __forceinline__ void emit4_interior(const GramParams& p, long long od, long long om,
                                               const InteriorPair (&m)[4], bool first, bool direct, bool mirror,
                                               float fd, float rd, int d0 = -1) {
  const long long N = p.N;
  float* outs[3] = {static_cast<float*>(p.out_plv), static_cast<float*>(p.out_iplv),
                    static_cast<float*>(p.out_ciplv)};
  float4 prev[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    prev[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (outs[q] && !first && (!DIAG || d0 < 4)) prev[q] = *reinterpret_cast<const float4*>(outs[q] + od);
  }
  auto sc = [&](float x) { return SCALE ? mean_scale_r(x, fd, rd) : x; };
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (!outs[q]) continue;
    auto val = [&](int e) { return q == 0 ? m[e].plv : q == 1 ? m[e].aim : m[e].ci; };
    const float a[4] = {sc(prev[q].x + val(0)), sc(prev[q].y + val(1)), sc(prev[q].z + val(2)),
                        sc(prev[q].w + val(3))};
    if (direct) {
      if (!DIAG || d0 <= 0) {
        *reinterpret_cast<float4*>(outs[q] + od) = make_float4(a[0], a[1], a[2], a[3]);
      } else if (d0 < 4) {
#pragma unroll
        for (int e = 1; e < 4; ++e)
          if (e >= d0) outs[q][od + e] = a[e];
      }
    }
    if (mirror) {
      float* mp = outs[q] + om;
#pragma unroll
      for (int e = 0; e < 4; ++e, mp += N)
        if (!DIAG || e > d0) *mp = a[e];
    }
  }
}

// Round bookkeeping common to both kernels: which slot a (item, trial) round
// writes and whether it is the first / last contribution to that slot.
struct RoundInfo {
  long long slot;
  bool first, last;
  int u0, nu;  // units covered by the round's Gram
};

__device__ __forceinline__ RoundInfo round_info(const GramParams& p, const Item& w, int r, int r0, int r1) {
  RoundInfo ri;
  if (p.pool) {
    ri.slot = w.b;
    ri.first = ri.last = true;
    ri.u0 = w.b * p.R;
    ri.nu = p.R;
    return ri;
  }
  ri.u0 = w.b * p.R + r;
  ri.nu = 1;
  if (p.slot_mode == 0) {
    ri.slot = (long long)w.b * p.R + r;
    ri.first = ri.last = true;
  } else if (p.slot_mode == 1) {
    ri.slot = w.b;
    ri.first = (r == r0);
    ri.last = (r == r1 - 1);
  } else {
    ri.slot = (long long)w.b * p.G + w.g;
    ri.first = (r == r0);
    ri.last = (r == r1 - 1);
  }
  return ri;
}

}  // namespace ps
