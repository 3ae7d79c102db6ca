// Phasor preparation kernels: input packing for cuFFT, the one-sided Hilbert
// spectral mask (K2), normalisation to unit phasors with split-plane output
// (K4), the exact-median amplitude-floor fixup, and the trial-group reduce.
//
// Reference semantics: SPEC.md:76-93 (analytic_signal, normalize_phasors),
// design decisions SPEC.md:120-125, per-pair effective T SPEC.md:260.
// All of these are HBM-bound streaming kernels.
#include <cuda_fp16.h>
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "ps_internal.h"

namespace ps {

namespace {

constexpr int kNormThreads = 256;
constexpr int kNormPerThread = 4;
constexpr int kNormSamplesPerBlock = kNormThreads * kNormPerThread;

// Output formats of the normalisation stage.
enum OutFmt : int { OUT_SPLIT = 0, OUT_F64 = 1, OUT_COMPLEX = 2 };

__device__ __forceinline__ long long row_offset(const SrcDesc& s, long long r) {
  const long long n = r % s.N;
  const long long u = r / s.N;
  const long long t = u % s.R;
  const long long b = u / s.R;
  return b * s.s_band + t * s.s_trial + n * s.s_sig;
}

// Loads sample (r, t) of the source as a complex value in compute type S.
template <typename IT, typename S, int KIND>
__device__ __forceinline__ void load_a(const SrcDesc& s, long long roff, long long r, long long t, S& re,
                                       S& im) {
  if (KIND == 0) {
    re = static_cast<S>(static_cast<const IT*>(s.ptr)[roff + t * s.s_samp]);
    im = static_cast<const S*>(s.hbuf)[(r - s.h_row0) * s.h_ld + t];
    if (s.h_scale) im *= static_cast<const S*>(s.h_scale)[r - s.h_row0];
  } else {
    const IT* p = static_cast<const IT*>(s.ptr) + 2 * (roff + t * s.s_samp);
    re = static_cast<S>(p[0]);
    im = static_cast<S>(p[1]);
  }
}

template <typename S>
__device__ __forceinline__ S amp_of(S re, S im) {
  return sqrt(re * re + im * im);
}

// Writes z = (zr, zi) at element (row r, sample t) in the requested format.
template <typename S, int FMT>
__device__ __forceinline__ void store_z(void* out, long long plane_stride, long long idx, S zr, S zi) {
  if (FMT == OUT_SPLIT) {
    __half* p = static_cast<__half*>(out);
    const float fr = static_cast<float>(zr), fi = static_cast<float>(zi);
    const __half rh = __float2half_rn(fr);
    const __half ih = __float2half_rn(fi);
    // residuals from the full-precision value (exact for S = float; for
    // S = double the residual is rounded once to fp16)
    const __half rl = __float2half_rn(static_cast<float>(zr - static_cast<S>(__half2float(rh))));
    const __half il = __float2half_rn(static_cast<float>(zi - static_cast<S>(__half2float(ih))));
    p[idx] = rh;
    p[plane_stride + idx] = rl;
    p[2 * plane_stride + idx] = ih;
    p[3 * plane_stride + idx] = il;
  } else if (FMT == OUT_F64) {
    double* p = static_cast<double*>(out);
    p[idx] = static_cast<double>(zr);
    p[plane_stride + idx] = static_cast<double>(zi);
  } else {
    S* p = static_cast<S*>(out);
    p[2 * idx] = zr;
    p[2 * idx + 1] = zi;
  }
}

template <typename S, int FMT>
__device__ __forceinline__ void zero_z(void* out, long long plane_stride, long long idx) {
  store_z<S, FMT>(out, plane_stride, idx, S(0), S(0));
}

__device__ __forceinline__ unsigned long long key_of(double a) {
  return static_cast<unsigned long long>(__double_as_longlong(a));
}
__device__ __forceinline__ double val_of(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>(k));
}

// ---------------------------------------------------------------------------
// K4: z = a/|a| (or z = a for phasor input), split/planes output, row min/max
// of |a| for the amplitude-floor pre-check.  Each block handles 1024
// consecutive samples of one row; loads are warp-coalesced along samples.
// ---------------------------------------------------------------------------
template <typename IT, typename S, int KIND, int FMT>
__global__ void __launch_bounds__(kNormThreads) normalize_kernel(SrcDesc src, long long row0, int chunks,
                                                                 void* out, int pitch, long long plane_stride,
                                                                 unsigned long long* rowmin,
                                                                 unsigned long long* rowmax, DevStatus* st) {
  const long long rl = blockIdx.x / chunks;
  const int ch = blockIdx.x % chunks;
  const long long r = row0 + rl;
  const long long roff = row_offset(src, r);
  const long long T = src.T;
  S amin = sizeof(S) == 4 ? S(FLT_MAX) : S(DBL_MAX);
  S amax = S(0);
  bool bad = false;
  const long long obase = (FMT == OUT_COMPLEX ? (r - row0) : r) * pitch;
#pragma unroll
  for (int k = 0; k < kNormPerThread; ++k) {
    const long long t = (long long)ch * kNormSamplesPerBlock + k * kNormThreads + threadIdx.x;
    if (t < T) {
      S re, im;
      load_a<IT, S, KIND>(src, roff, r, t, re, im);
      const S a = amp_of(re, im);
      S zr = S(0), zi = S(0);
      if (KIND == 2) {
        zr = re;
        zi = im;
      } else if (a > S(0)) {
        zr = re / a;
        zi = im / a;
      }
      store_z<S, FMT>(out, plane_stride, obase + t, zr, zi);
      if (!(a <= (sizeof(S) == 4 ? S(FLT_MAX) : S(DBL_MAX)))) bad = true;
      amin = a < amin ? a : amin;
      amax = a > amax ? a : amax;
    } else if (t < pitch && FMT != OUT_COMPLEX) {
      zero_z<S, FMT>(out, plane_stride, obase + t);  // zero the pitch padding
    }
  }
  // block reduce min / max
  __shared__ double smin[kNormThreads / 32], smax[kNormThreads / 32];
  double dmin = static_cast<double>(amin), dmax = static_cast<double>(amax);
  for (int o = 16; o > 0; o >>= 1) {
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smin[w] = dmin;
    smax[w] = dmax;
  }
  if (bad) atomicOr(&st->flags, FLAG_NONFINITE);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kNormThreads / 32; ++i) {
      dmin = fmin(dmin, smin[i]);
      dmax = fmax(dmax, smax[i]);
    }
    dmin = fmin(smin[0], dmin);
    dmax = fmax(smax[0], dmax);
    atomicMin(&rowmin[r], key_of(dmin));
    atomicMax(&rowmax[r], key_of(dmax));
  }
}

// ---------------------------------------------------------------------------
// K4 fast path: fp32 source (real + H, or interleaved complex64), samples
// contiguous and 16-byte aligned rows, split fp16 planes.  Each thread moves
// 2 x 4 samples with 16-byte loads and 8-byte plane stores (HBM-bound:
// 16 B/sample algorithmic traffic).
// ---------------------------------------------------------------------------
constexpr int kVecPer = 2;                                     // 4-sample groups per thread
constexpr int kVecSamplesPerBlock = kNormThreads * 4 * kVecPer;

__device__ __forceinline__ uint32_t pack_half2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// 4 consecutive samples at t0 of row r (source offset roff): normalise, split,
// store the planes; folds |a| into amin / amax and non-finite into bad.
template <int KIND>
__device__ __forceinline__ void normalize_vec4(const SrcDesc& src, long long r, long long roff, long long t0, float hs,
                                               __half* out, long long obase, long long ps, float& amin, float& amax,
                                               bool& bad) {
    float re[4], im[4];
    if (KIND == 0) {
      const float4 x = *reinterpret_cast<const float4*>(static_cast<const float*>(src.ptr) + roff + t0);
      const float4 h = *reinterpret_cast<const float4*>(static_cast<const float*>(src.hbuf) +
                                                        (r - src.h_row0) * src.h_ld + t0);
      re[0] = x.x; re[1] = x.y; re[2] = x.z; re[3] = x.w;
      im[0] = h.x * hs; im[1] = h.y * hs; im[2] = h.z * hs; im[3] = h.w * hs;
    } else {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(src.ptr) + 2 * (roff + t0));
      const float4 a = p[0], b = p[1];
      re[0] = a.x; im[0] = a.y; re[1] = a.z; im[1] = a.w;
      re[2] = b.x; im[2] = b.y; re[3] = b.z; im[3] = b.w;
    }
    __half rh[4], rlo[4], ih[4], ilo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // one MUFU.RSQ instead of sqrt + two IEEE divisions: z is rounded to
      // the 22-bit hi/lo split anyway, and the row min/max only feed the
      // conservative amplitude-floor pre-check (the fixup recomputes |a|
      // exactly for any row it inspects)
      const float a2 = re[k] * re[k] + im[k] * im[k];
      const float inv = a2 > 0.0f ? rsqrtf(a2) : 0.0f;
      const float a = a2 * inv;
      float zr = 0.0f, zi = 0.0f;
      if (KIND == 2) {
        zr = re[k];
        zi = im[k];
      } else {
        zr = re[k] * inv;
        zi = im[k] * inv;
      }
      rh[k] = __float2half_rn(zr);
      ih[k] = __float2half_rn(zi);
      rlo[k] = __float2half_rn(zr - __half2float(rh[k]));
      ilo[k] = __float2half_rn(zi - __half2float(ih[k]));
      if (!(a <= FLT_MAX)) bad = true;
      amin = fminf(amin, a);
      amax = fmaxf(amax, a);
    }
    __half* o = out + obase + t0;
    *reinterpret_cast<uint2*>(o) = make_uint2(pack_half2(rh[0], rh[1]), pack_half2(rh[2], rh[3]));
    *reinterpret_cast<uint2*>(o + ps) = make_uint2(pack_half2(rlo[0], rlo[1]), pack_half2(rlo[2], rlo[3]));
    *reinterpret_cast<uint2*>(o + 2 * ps) = make_uint2(pack_half2(ih[0], ih[1]), pack_half2(ih[2], ih[3]));
    *reinterpret_cast<uint2*>(o + 3 * ps) = make_uint2(pack_half2(ilo[0], ilo[1]), pack_half2(ilo[2], ilo[3]));
    if (src.gauss_planes) {
      // Gauss-Gram operands S = Zr + Zi, D = Zr - Zi from the rounded split
      // values -- the arithmetic of gauss_planes_kernel, fused here so the
      // planes are not read back (16 B / sample saved)
      __half sh[4], sl[4], dh[4], dl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float zr = __half2float(rh[k]) + __half2float(rlo[k]);
        const float zi = __half2float(ih[k]) + __half2float(ilo[k]);
        const float S = zr + zi, D = zr - zi;
        sh[k] = __float2half_rn(S);
        sl[k] = __float2half_rn(S - __half2float(sh[k]));
        dh[k] = __float2half_rn(D);
        dl[k] = __float2half_rn(D - __half2float(dh[k]));
      }
      *reinterpret_cast<uint2*>(o + 4 * ps) = make_uint2(pack_half2(sh[0], sh[1]), pack_half2(sh[2], sh[3]));
      *reinterpret_cast<uint2*>(o + 5 * ps) = make_uint2(pack_half2(sl[0], sl[1]), pack_half2(sl[2], sl[3]));
      *reinterpret_cast<uint2*>(o + 6 * ps) = make_uint2(pack_half2(dh[0], dh[1]), pack_half2(dh[2], dh[3]));
      *reinterpret_cast<uint2*>(o + 7 * ps) = make_uint2(pack_half2(dl[0], dl[1]), pack_half2(dl[2], dl[3]));
    }
}

template <int KIND>
__global__ void __launch_bounds__(kNormThreads) normalize_vec_kernel(SrcDesc src, long long row0, int chunks,
                                                                     __half* out, int pitch, long long ps,
                                                                     unsigned long long* rowmin,
                                                                     unsigned long long* rowmax, DevStatus* st) {
  const long long rl = blockIdx.x / chunks;
  const int ch = blockIdx.x % chunks;
  const long long r = row0 + rl;
  const long long roff = row_offset(src, r);
  const long long T = src.T;
  float amin = FLT_MAX, amax = 0.0f;
  bool bad = false;
  const long long obase = r * pitch;
  const float hs = (KIND == 0 && src.h_scale) ? static_cast<const float*>(src.h_scale)[r - src.h_row0] : 1.0f;
#pragma unroll
  for (int g = 0; g < kVecPer; ++g) {
    const long long t0 = (long long)ch * kVecSamplesPerBlock + ((long long)g * kNormThreads + threadIdx.x) * 4;
    if (t0 < T) {
      normalize_vec4<KIND>(src, r, roff, t0, hs, out, obase, ps, amin, amax, bad);
    } else if (t0 < pitch) {  // T % 4 == 0: the pitch pad is one 4-sample group
      __half* o = out + obase + t0;
      const uint2 z = make_uint2(0u, 0u);
      const int np = src.gauss_planes ? 8 : 4;
      for (int pl = 0; pl < np; ++pl) *reinterpret_cast<uint2*>(o + pl * ps) = z;
    }
  }
  __shared__ float smin[kNormThreads / 32], smax[kNormThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    amin = fminf(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = amin;
    smax[threadIdx.x >> 5] = amax;
  }
  if (bad) atomicOr(&st->flags, FLAG_NONFINITE);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kNormThreads / 32; ++i) {
      amin = fminf(amin, smin[i]);
      amax = fmaxf(amax, smax[i]);
    }
    atomicMin(&rowmin[r], key_of((double)amin));
    atomicMax(&rowmax[r], key_of((double)amax));
  }
}

// The same for short rows (T % 128 == 0, T <= kVecSamplesPerBlock / 2): a block
// takes kVecSamplesPerBlock / T whole rows instead of leaving most of its
// threads idle on one (T = 256: 2.2x the time per sample of long rows).  A
// warp's 32 x 4 samples lie in one row, so row min / max are a warp reduction
// and one atomic pair per warp.
template <int KIND>
__global__ void __launch_bounds__(kNormThreads) normalize_vec_rows_kernel(SrcDesc src, long long row0, long long nrows,
                                                                          int rpb, __half* out, int pitch,
                                                                          long long ps, unsigned long long* rowmin,
                                                                          unsigned long long* rowmax, DevStatus* st) {
  const int T = (int)src.T;
  bool bad = false;
#pragma unroll
  for (int g = 0; g < kVecPer; ++g) {
    const int s4 = (g * kNormThreads + threadIdx.x) * 4;  // sample slot within the block's rows
    const long long rl = (long long)blockIdx.x * rpb + s4 / T;
    if (s4 / T < rpb && rl < nrows) {
      const long long r = row0 + rl;
      const long long t0 = s4 % T;
      const float hs = (KIND == 0 && src.h_scale) ? static_cast<const float*>(src.h_scale)[r - src.h_row0] : 1.0f;
      float amin = FLT_MAX, amax = 0.0f;
      normalize_vec4<KIND>(src, r, row_offset(src, r), t0, hs, out, r * pitch, ps, amin, amax, bad);
      // (whole warps take this branch together: 128 samples of one row)
      for (int o = 16; o > 0; o >>= 1) {
        amin = fminf(amin, __shfl_xor_sync(0xffffffffu, amin, o));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      }
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&rowmin[r], key_of((double)amin));
        atomicMax(&rowmax[r], key_of((double)amax));
      }
    }
  }
  if (bad) atomicOr(&st->flags, FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// Fused Hilbert + normalise for real fp32 rows of length T = 4096 (the
// short-T, many-trial regime of config C4): one CTA per pair of rows, the two
// rows packed as x_a + i x_b into one complex FFT (the Hilbert multiplier
// -i sgn(k) is real-linear, so IFFT(h . FFT(x_a + i x_b)) = H{x_a} + i H{x_b}).
// In-place radix-16 FFT in shared memory (3 passes each way, 256 threads x
// 16 values), the multiplier fused into the first inverse pass, and the
// normalisation / fp16 hi-lo split / row min-max fused into the epilogue.
// HBM traffic 12 B/sample (x in, planes out) versus ~40 B/sample for the
// cuFFT R2C -> K2 -> C2R -> K4 chain.  H is written to `hbuf` only for rows
// whose amplitude pre-check fails, so the exact-median fixup can run as usual.
// ---------------------------------------------------------------------------
constexpr int kFftT = 4096;
constexpr int kFftThreads = 256;  // kFftT / 16
__host__ __device__ constexpr int kFftPad(int i) { return i + (i >> 4); }  // breaks the stride-16 bank pattern
// twiddle tables per pass, laid out [r][k] (lanes read consecutive k):
//   pass NS=16 : W_256^(k r),  k < 16,  r = 1..15
//   pass NS=256: W_4096^(k r), k < 256, r = 1..15
constexpr int kTw16 = 0;
constexpr int kTw256 = 15 * 16;
constexpr int kTwCount = kTw256 + 15 * 256;
constexpr int kFftSmemBytes = (kFftPad(kFftT) + kTwCount) * 8;

// Complex arithmetic on sm_100's packed FP32 pipe (FADD2 / FMUL2 / FFMA2 work
// on an aligned register pair = one float2, with free per-operand swap
// (.LO_HI), per-half negation and scalar broadcast): a complex add is one
// instruction and a complex multiply two, half the scalar count.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(-a.y, a.x), make_float2(b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

template <bool INV>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 s0 = cadd(a0, a2), d0 = csub(a0, a2), s1 = cadd(a1, a3), d1 = csub(a1, a3);
  const float2 t = INV ? make_float2(-d1.y, d1.x) : make_float2(d1.y, -d1.x);  // d1 * (+-i)
  a0 = cadd(s0, s1);
  a2 = csub(s0, s1);
  a1 = cadd(d0, t);
  a3 = csub(d0, t);
}

// W16^m (forward sign) for compile-time m in [0, 9]
__device__ __forceinline__ float2 w16(int m) {
  const float c1 = 0.92387953251128674f, s1 = 0.38268343236508977f, c2 = 0.70710678118654752f;
  switch (m) {
    case 1: return make_float2(c1, -s1);
    case 2: return make_float2(c2, -c2);
    case 3: return make_float2(s1, -c1);
    case 4: return make_float2(0.f, -1.f);
    case 6: return make_float2(-c2, -c2);
    case 9: return make_float2(-c1, s1);
    default: return make_float2(1.f, 0.f);
  }
}

// Position of output k of dft16 in v[]: the result is left transposed
// (X[k1 + 4 k2] in v[4 k1 + k2]) and consumers index through this map.
__host__ __device__ constexpr int d16(int k) { return 4 * (k & 3) + (k >> 2); }

// In-register 16-point DFT (4 x 4 decomposition), sign per INV; output k in v[d16(k)].
template <bool INV>
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
  // n = 4 n1 + n2 ; first 4-point DFTs over n1
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] = A[n2][k1]; twiddle W16^(n2 k1)
#pragma unroll
  for (int k1 = 1; k1 < 4; ++k1)
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2) {
      const int m = n2 * k1;
      float2& x = v[4 * k1 + n2];
      const float c2 = 0.70710678118654752f;
      // W16^m with the trivial factors spelled out (the compiler may not fold
      // multiplications by 0 / +-1 under IEEE semantics)
      if (m == 4) {
        x = INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
      } else if (m == 2) {
        // (1 -+ i) x c2 : x + (-+ i) x, one packed add and one packed multiply
        x = __fmul2_rn(__fadd2_rn(x, INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x)), make_float2(c2, c2));
      } else if (m == 6) {
        // (-1 -+ i) x c2
        x = __fmul2_rn(__fadd2_rn(make_float2(-x.x, -x.y), INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x)),
                       make_float2(c2, c2));
      } else {
        float2 tw = w16(m);
        if (INV) tw.y = -tw.y;
        x = cmul(x, tw);
      }
    }
  // second 4-point DFTs over n2 -> X[k1 + 4 k2] lands in v[4 k1 + k2]
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1 + 0], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}

// In-place radix-16 passes over the 4096-point buffer: decimation in frequency
// forward (natural order in, digit-reversed out: frequency 256 k2 + 16 k1 + k0
// at position 256 k0 + 16 k1 + k2), decimation in time inverse (digit-reversed
// in, natural out).  Every thread reads and writes the SAME 16 positions in a
// pass, so a pass needs no barrier between its loads and its stores, and the
// exchanges between the stride-16 and stride-1 passes stay inside one aligned
// group of 16 threads (a 256-point block): __syncwarp instead of a CTA barrier.
// Position sets (pad(i) = i + i / 16; every access is a per-thread base plus
// a compile-time offset):
//   stride 256: pad(j + 256 r)          = pad(j) + 272 r
//   stride 16 : pad(256 b + o + 16 r)   = 272 b + o + 17 r   (b = j / 16, o = j % 16)
//   stride 1  : pad(16 j + r)           = 17 j + r
// Twiddles multiply DFT16 output r (forward, after the butterfly) or input r
// (inverse, before it) by W^(k r), k = j (stride 256, W_4096) or o (stride 16,
// W_256), conjugated for the inverse.
template <int STRIDE>
__device__ __forceinline__ int pass_base() {
  const int j = threadIdx.x;
  return STRIDE == 256 ? kFftPad(j) : STRIDE == 16 ? 272 * (j >> 4) + (j & 15) : 17 * j;
}
template <int STRIDE>
__host__ __device__ constexpr int pass_step() {
  return STRIDE == 256 ? 272 : STRIDE == 16 ? 17 : 1;
}
// v[r] = element r of this thread's set
template <int STRIDE>
__device__ __forceinline__ void load_set(float2 (&v)[16], const float2* buf) {
  const float2* p = buf + pass_base<STRIDE>();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = p[r * pass_step<STRIDE>()];
}
// element r of the set = DFT16 output r (held in v[d16(r)])
template <int STRIDE>
__device__ __forceinline__ void store_set(const float2 (&v)[16], float2* buf) {
  float2* p = buf + pass_base<STRIDE>();
#pragma unroll
  for (int r = 0; r < 16; ++r) p[r * pass_step<STRIDE>()] = v[d16(r)];
}
// OUT: the DFT16 outputs (v[d16(r)]) are twiddled, else the inputs (v[r])
template <bool INV, int STRIDE, bool OUT>
__device__ __forceinline__ void twiddle16(float2 (&v)[16], const float2* tw) {
  const float2* t = tw + (STRIDE == 16 ? kTw16 + (threadIdx.x & 15) : kTw256 + threadIdx.x);
  constexpr int NS = STRIDE == 16 ? 16 : 256;
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    float2 w = t[(r - 1) * NS];
    if (INV) w.y = -w.y;
    float2& x = v[OUT ? d16(r) : r];
    x = cmul(x, w);
  }
}

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

__device__ __forceinline__ float rsqrt_ftz(float a) {
  float d;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(a));
  return d;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// L2 prefetch of `bytes` (multiple of 16, 16-byte aligned) at p (TMA bulk,
// no registers or shared memory involved)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 2^(1 - e) with m = m' 2^e, m' in [0.5, 1) (frexpf convention), clamped to
// [2^-126, 2^126]: scales m into [1, 2).  0 / non-finite m -> 2 (e = 0).
// Exponent-field arithmetic; denormal m clamps to 2^126 as frexpf would.
__device__ __forceinline__ float pow2_scale(float m) {
  int e = 0;
  if (m > 0.f && m <= FLT_MAX) e = (int)((__float_as_uint(m) >> 23) & 0xffu) - 126;
  const int s = min(126, max(-126, 1 - e));
  return __uint_as_float((uint32_t)(127 + s) << 23);
}

// Normalises 4 consecutive samples (re = x * scale, im = H) into the four
// fp16 split planes at o (plane stride ps) -- and, with GS, the Gauss-Gram
// planes S = Zr + Zi, D = Zr - Zi (hi / lo) from the rounded split values,
// the arithmetic of gauss_planes_kernel; returns their min / max |a|.
template <bool GS>
__device__ __forceinline__ void emit4_split(const float (&zr)[4], const float (&zi)[4], __half* o, long long ps);

template <bool GS>
__device__ __forceinline__ void normalize4_split(const float (&re)[4], const float (&im)[4], __half* o,
                                                 long long ps, float& lo2, float& hi2) {
  float zr[4], zi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float a2 = re[k] * re[k] + im[k] * im[k];
    // |a|^2 clamped to FLT_MIN: a zero sample gives z = 0 (0 * finite); a
    // sample this small is below the amplitude floor of its row, which the
    // exact fixup then masks from H (its row min trips the pre-check)
    const float inv = rsqrtf(fmaxf(a2, FLT_MIN));
    zr[k] = re[k] * inv;
    zi[k] = im[k] * inv;
    lo2 = fminf(lo2, a2);
    hi2 = fmax_nan(hi2, a2);  // NaN-propagating: a non-finite sample surfaces in the row max
  }
  emit4_split<GS>(zr, zi, o, ps);
}

// The same for 4 consecutive samples of two rows at once, the rows riding the
// two halves of the packed FP32 instructions: re[k] = (x_a, x_b) scaled,
// h[k] = (H_a, H_b) as the packed inverse FFT left them.
template <bool GS>
__device__ __forceinline__ void normalize4_split_pair(const float2 (&re)[4], const float2 (&h)[4], __half* oa,
                                                      __half* ob, bool hasb, long long ps, float& lo_a, float& hi_a,
                                                      float& lo_b, float& hi_b) {
  float zra[4], zia[4], zrb[4], zib[4];
  float2 a2s[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 a2 = __ffma2_rn(re[k], re[k], __fmul2_rn(h[k], h[k]));
    // the argument is clamped to a normal number: the flush-to-zero form
    // (one MUFU, no denormal pre-scaling) returns the same value
    const float2 inv = make_float2(rsqrt_ftz(fmaxf(a2.x, FLT_MIN)), rsqrt_ftz(fmaxf(a2.y, FLT_MIN)));
    const float2 zr = __fmul2_rn(re[k], inv), zi = __fmul2_rn(h[k], inv);
    zra[k] = zr.x;
    zrb[k] = zr.y;
    zia[k] = zi.x;
    zib[k] = zi.y;
    a2s[k] = a2;
  }
  // 3-input min / max (FMNMX3): two instructions per row and statistic
  lo_a = fminf(fminf(fminf(lo_a, a2s[0].x), a2s[1].x), fminf(a2s[2].x, a2s[3].x));
  lo_b = fminf(fminf(fminf(lo_b, a2s[0].y), a2s[1].y), fminf(a2s[2].y, a2s[3].y));
  hi_a = fmax3_nan(fmax3_nan(hi_a, a2s[0].x, a2s[1].x), a2s[2].x, a2s[3].x);
  hi_b = fmax3_nan(fmax3_nan(hi_b, a2s[0].y, a2s[1].y), a2s[2].y, a2s[3].y);
  emit4_split<GS>(zra, zia, oa, ps);
  if (hasb) emit4_split<GS>(zrb, zib, ob, ps);
}

template <bool GS>
__device__ __forceinline__ void emit4_split(const float (&zr)[4], const float (&zi)[4], __half* o, long long ps) {
  // packed conversions (F2FP / HADD2.F32): the same round-to-nearest
  // values as per-element __float2half_rn, half the instructions
  uint32_t w[GS ? 8 : 4][2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const __half2 rh = __floats2half2_rn(zr[2 * q], zr[2 * q + 1]);
    const __half2 ih = __floats2half2_rn(zi[2 * q], zi[2 * q + 1]);
    const float2 rf = __half22float2(rh), jf = __half22float2(ih);
    const __half2 rl = __floats2half2_rn(zr[2 * q] - rf.x, zr[2 * q + 1] - rf.y);
    const __half2 il = __floats2half2_rn(zi[2 * q] - jf.x, zi[2 * q + 1] - jf.y);
    w[0][q] = *reinterpret_cast<const uint32_t*>(&rh);
    w[1][q] = *reinterpret_cast<const uint32_t*>(&rl);
    w[2][q] = *reinterpret_cast<const uint32_t*>(&ih);
    w[3][q] = *reinterpret_cast<const uint32_t*>(&il);
    if (GS) {
      const float2 rlf = __half22float2(rl), ilf = __half22float2(il);
      const float ar = rf.x + rlf.x, br = rf.y + rlf.y;  // rounded Zr of the two samples
      const float ai = jf.x + ilf.x, bi = jf.y + ilf.y;  // rounded Zi
      const float s0 = ar + ai, s1 = br + bi, d0 = ar - ai, d1 = br - bi;
      const __half2 sh = __floats2half2_rn(s0, s1), dh = __floats2half2_rn(d0, d1);
      const float2 shf = __half22float2(sh), dhf = __half22float2(dh);
      const __half2 sl = __floats2half2_rn(s0 - shf.x, s1 - shf.y), dl = __floats2half2_rn(d0 - dhf.x, d1 - dhf.y);
      w[4][q] = *reinterpret_cast<const uint32_t*>(&sh);
      w[5][q] = *reinterpret_cast<const uint32_t*>(&sl);
      w[6][q] = *reinterpret_cast<const uint32_t*>(&dh);
      w[7][q] = *reinterpret_cast<const uint32_t*>(&dl);
    }
  }
#pragma unroll
  for (int pl = 0; pl < (GS ? 8 : 4); ++pl) *reinterpret_cast<uint2*>(o + pl * ps) = make_uint2(w[pl][0], w[pl][1]);
}

template <bool GS>
__global__ void __launch_bounds__(kFftThreads, 3) hilbert_fused4096_kernel(
    SrcDesc src, long long row0, long long nrows, __half* out, int pitch, long long ps, unsigned long long* rowmin,
    unsigned long long* rowmax, float* hbuf, double amp_floor, DevStatus* st) {
  extern __shared__ float2 fsm[];
  float2* buf = fsm;
  float2* tw = fsm + kFftPad(kFftT);
  for (int m = threadIdx.x; m < kTwCount; m += kFftThreads) {
    int ns, kk, r;
    if (m < kTw256) {
      ns = 16;
      r = 1 + m / 16;
      kk = m % 16;
    } else {
      ns = 256;
      r = 1 + (m - kTw256) / 256;
      kk = (m - kTw256) % 256;
    }
    const int n = 16 * ns;  // sub-transform length after the pass
    float s, c;
    sincospif(-2.0f * (float)((kk * r) % n) / (float)n, &s, &c);
    tw[m] = make_float2(c, s);
  }
  __shared__ float red[4][kFftThreads / 32];
  __shared__ int need_flags[2];
  __syncthreads();
  const int j = threadIdx.x;
  const long long npairs = (nrows + 1) / 2;
  for (long long pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const long long ra = row0 + 2 * pr, rb = ra + 1;
    const bool hasb = 2 * pr + 1 < nrows;
    const long long oa = row_offset(src, ra), ob = hasb ? row_offset(src, rb) : 0;
    const float* x = static_cast<const float*>(src.ptr);  // s_samp == 1 (hilbert_fused_supported)
    const float* xpa = x + oa + j;
    const float* xpb = x + ob + j;
    if (j == 0 && pr + gridDim.x < npairs) {
      // the CTA's next pair into L2 while this one computes: its first loads
      // (a full DRAM round trip ahead of the first barrier) then hit L2
      const long long nra = row0 + 2 * (pr + gridDim.x);
      bulk_prefetch_l2(x + row_offset(src, nra), kFftT * sizeof(float));
      if (2 * (pr + gridDim.x) + 1 < nrows) bulk_prefetch_l2(x + row_offset(src, nra + 1), kFftT * sizeof(float));
    }
    float2 v[16];
    float ma = 0.f, mb = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      v[q] = make_float2(__ldg(xpa + q * kFftThreads), hasb ? __ldg(xpb + q * kFftThreads) : 0.0f);
      ma = fmaxf(ma, fabsf(v[q].x));
      mb = fmaxf(mb, fabsf(v[q].y));
    }
    // Scale each row by a power of two to max |x| in [1, 2) before packing:
    // the FFT's rounding error scales with the larger row of the pair, so
    // rows of very different magnitude would otherwise leak error into the
    // smaller one.  Exact (power of two) and z = a / |a| is scale-free.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    }
    if ((j & 31) == 0) {
      red[0][j >> 5] = ma;
      red[1][j >> 5] = mb;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kFftThreads / 32; ++w) {
      ma = fmaxf(ma, red[0][w]);
      mb = fmaxf(mb, red[1][w]);
    }
    const float sa = pow2_scale(ma), sb = pow2_scale(mb);
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __fmul2_rn(v[q], make_float2(sa, sb));
    // forward FFT, decimation in frequency.  buf is free: every thread of the
    // previous pair passed that pair's last barrier after its last read.
    dft16<false>(v);
    twiddle16<false, 256, true>(v, tw);
    store_set<256>(v, buf);
    __syncthreads();
    load_set<16>(v, buf);
    dft16<false>(v);
    twiddle16<false, 16, true>(v, tw);
    store_set<16>(v, buf);
    __syncwarp();
    load_set<1>(v, buf);
    dft16<false>(v);
    // v[d16(r)] = X[256 r + 16 k1 + k0] with 16 k0 + k1 = j: the register index
    // is the top digit of the frequency, so the Hilbert multiplier -i sgn(k)
    // is -i for r < 8 and +i for r >= 8, with DC and Nyquist (0 there) in
    // thread 0's r = 0 and r = 8.  The inverse's first pass runs on the same
    // registers.  Its 1/T is folded into the epilogue (x scaled by T instead:
    // exact, power of two).
    float2 u[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const float2 z = v[d16(r)];
      u[r] = r < 8 ? make_float2(z.y, -z.x) : make_float2(-z.y, z.x);
    }
    if (j == 0) {
      u[0] = make_float2(0.f, 0.f);
      u[8] = make_float2(0.f, 0.f);
    }
    // inverse FFT, decimation in time -> T (H_a sa + i H_b sb) at t in natural
    // order in buf
    dft16<true>(u);
    store_set<1>(u, buf);
    __syncwarp();
    load_set<16>(u, buf);
    twiddle16<true, 16, false>(u, tw);
    dft16<true>(u);
    store_set<16>(u, buf);
    __syncthreads();
    load_set<256>(u, buf);
    twiddle16<true, 256, false>(u, tw);
    dft16<true>(u);
    store_set<256>(u, buf);
    __syncthreads();
    // normalise both rows from (x, H in smem): 4 consecutive samples per
    // thread and step (16-byte x loads -- L2 hits, software-pipelined one
    // step ahead -- and 8-byte plane stores); row min / max of |a|^2
    const float soa = sa * (float)kFftT, sob = sb * (float)kFftT;
    float amin_a = FLT_MAX, amax_a = 0.f, amin_b = FLT_MAX, amax_b = 0.f;
    const float2* hb = buf + kFftPad(4 * j);
    __half* opa = out + ra * pitch + 4 * j;
    __half* opb = out + rb * pitch + 4 * j;
    const float4* xa4 = reinterpret_cast<const float4*>(x + oa) + j;
    const float4* xb4 = reinterpret_cast<const float4*>(x + ob) + j;
    float4 na = xa4[0], nb = hasb ? xb4[0] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int g = 0; g < kFftT / (4 * kFftThreads); ++g) {
      const int off = g * 4 * kFftThreads;  // samples
      const float4 ca = na, cb = nb;
      if (g + 1 < kFftT / (4 * kFftThreads)) {
        na = xa4[(g + 1) * kFftThreads];
        if (hasb) nb = xb4[(g + 1) * kFftThreads];
      }
      float2 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = hb[kFftPad(off) + k];
      const float2 re[4] = {make_float2(ca.x * soa, cb.x * sob), make_float2(ca.y * soa, cb.y * sob),
                            make_float2(ca.z * soa, cb.z * sob), make_float2(ca.w * soa, cb.w * sob)};
      normalize4_split_pair<GS>(re, h, opa + off, opb + off, hasb, ps, amin_a, amax_a, amin_b, amax_b);
    }
    // block min / max of both rows (the CTA owns them: plain stores)
    float vals[4] = {amin_a, amax_a, amin_b, amax_b};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vals[0] = fminf(vals[0], __shfl_xor_sync(0xffffffffu, vals[0], o));
      vals[1] = fmax_nan(vals[1], __shfl_xor_sync(0xffffffffu, vals[1], o));
      vals[2] = fminf(vals[2], __shfl_xor_sync(0xffffffffu, vals[2], o));
      vals[3] = fmax_nan(vals[3], __shfl_xor_sync(0xffffffffu, vals[3], o));
    }
    if ((j & 31) == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[q][j >> 5] = vals[q];
    __syncthreads();
    // thread 0 closes row a, thread 32 (another warp) row b
    if (j == 0 || j == 32) {
      const int q0 = j == 0 ? 0 : 2;
      float lo = red[q0][0], hi = red[q0 + 1][0];
      for (int w = 1; w < kFftThreads / 32; ++w) {
        lo = fminf(lo, red[q0][w]);
        hi = fmax_nan(hi, red[q0 + 1][w]);
      }
      int need = 0;
      if (j == 0 || hasb) {
        // a non-finite |a| anywhere in a row leaves its max non-finite (NaN
        // propagates, inf is the max)
        if (!(hi <= FLT_MAX)) atomicOr(&st->flags, FLAG_NONFINITE);
        lo = sqrtf(lo);  // |a|^2 -> |a|
        hi = sqrtf(hi);
        // back to input units: 1 / (scale T) is a power of two, built from the
        // exponent of the scale (exact; no double-precision division)
        const float sc = j == 0 ? sa : sb;
        const int e = (int)((__float_as_uint(sc) >> 23) & 0xffu) - 127 + 12;  // scale T = 2^e, T = 2^12
        const double rs = __hiloint2double((1023 - e) << 20, 0);
        const long long rr = j == 0 ? ra : rb;
        rowmin[rr] = key_of((double)lo * rs);
        rowmax[rr] = key_of((double)hi * rs);
        // the fixup decides on the min / max ratio, which the scaling leaves unchanged
        need = (lo == 0.0f) || ((double)lo < amp_floor * (double)hi * (1.0 + 1e-5));
      }
      need_flags[j == 0 ? 0 : 1] = need;
    }
    __syncthreads();
    // rare: keep H (input units) of a row the exact-median fixup will inspect
    if (need_flags[0] || need_flags[1]) {
      const float ua = 1.0f / soa, ub = 1.0f / sob;
      for (int t = j; t < kFftT; t += kFftThreads) {
        const float2 hv = buf[kFftPad(t)];
        if (need_flags[0]) hbuf[(ra - src.h_row0) * src.h_ld + t] = hv.x * ua;
        if (need_flags[1]) hbuf[(rb - src.h_row0) * src.h_ld + t] = hv.y * ub;
      }
    }
    // the next pair's first stores come after its row-max barrier
  }
}

// ---------------------------------------------------------------------------
// The same kernel for rows of T = 2048 or 1024 samples (NP = 4096 / T = 2 or 4
// row pairs per CTA iteration, side by side in the 4096-point buffer).  Only
// the outer pass changes: the stride-256 pass becomes NP independent radix-RQ
// butterflies per thread (RQ = 16 / NP: 8 or 4, twiddles W_T^(j s)); the
// stride-16 and stride-1 passes work inside 256-point blocks and do not care
// which transform a block belongs to.  In pass C the register index is still
// the top digit of the frequency (weight T / 16), so the Hilbert multiplier
// keeps its r < 8 rule; DC and Nyquist of pair q sit in thread q * 256 / NP.
// ---------------------------------------------------------------------------
// 8-point DFT of v[b .. b + 7] in place; output k lands in v[b + d8(k)]
__host__ __device__ constexpr int d8(int k) { return (k & 1) * 4 + (k >> 1); }
template <bool INV>
__device__ __forceinline__ void dft8(float2 (&v)[16], int b) {
  const float c2 = 0.70710678118654752f;
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    const float2 a = v[b + n], c = v[b + n + 4];
    v[b + n] = cadd(a, c);
    float2 d = csub(a, c);
    const float2 rot = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);  // d * (-+ i)
    if (n == 1) d = __fmul2_rn(__fadd2_rn(d, rot), make_float2(c2, c2));                            // W8^1
    else if (n == 2) d = rot;                                                                       // W8^2
    else if (n == 3) d = __fmul2_rn(__fadd2_rn(make_float2(-d.x, -d.y), rot), make_float2(c2, c2));  // W8^3
    v[b + n + 4] = d;
  }
  dft4<INV>(v[b + 0], v[b + 1], v[b + 2], v[b + 3]);  // X0 X2 X4 X6
  dft4<INV>(v[b + 4], v[b + 5], v[b + 6], v[b + 7]);  // X1 X3 X5 X7
}
// radix-RQ butterfly of v[b .. b + RQ - 1]; output k in v[b + dq<RQ>(k)]
template <int RQ>
__host__ __device__ constexpr int dq(int k) { return RQ == 16 ? d16(k) : RQ == 8 ? d8(k) : k; }
template <bool INV, int RQ>
__device__ __forceinline__ void dftq(float2 (&v)[16], int b) {
  if (RQ == 16) dft16<INV>(v);
  else if (RQ == 8) dft8<INV>(v, b);
  else dft4<INV>(v[b + 0], v[b + 1], v[b + 2], v[b + 3]);
}

template <bool GS, int NP>
__global__ void __launch_bounds__(kFftThreads, 3) hilbert_fused_short_kernel(
    SrcDesc src, long long row0, long long nrows, __half* out, int pitch, long long ps, unsigned long long* rowmin,
    unsigned long long* rowmax, float* hbuf, double amp_floor, DevStatus* st) {
  constexpr int RQ = 16 / NP;        // radix of the outer pass
  constexpr int TT = kFftT / NP;     // row length
  constexpr int NR = 2 * NP;         // rows per CTA iteration
  extern __shared__ float2 fsm[];
  float2* buf = fsm;
  float2* tw = fsm + kFftPad(kFftT);
  // tw[kTw16 + (r-1) 16 + o] = W_256^(o r); tw[kTw256 + (s-1) 256 + j] = W_TT^(j s), s < RQ
  for (int m = threadIdx.x; m < kTw256 + (RQ - 1) * 256; m += kFftThreads) {
    int n, kk, r;
    if (m < kTw256) {
      n = 256;
      r = 1 + m / 16;
      kk = m % 16;
    } else {
      n = TT;
      r = 1 + (m - kTw256) / 256;
      kk = (m - kTw256) % 256;
    }
    float sn, cs;
    sincospif(-2.0f * (float)((kk * r) % n) / (float)n, &sn, &cs);
    tw[m] = make_float2(cs, sn);
  }
  __shared__ float red[2 * NR][kFftThreads / 32];
  __shared__ int need_flags[NR];
  __syncthreads();
  const int j = threadIdx.x;
  const float* x = static_cast<const float*>(src.ptr);  // s_samp == 1 (hilbert_fused_supported)
  const long long ngroups = (nrows + NR - 1) / NR;
  for (long long gr = blockIdx.x; gr < ngroups; gr += gridDim.x) {
    long long rrow[NR], roff[NR];
    bool has[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      has[i] = NR * gr + i < nrows;
      rrow[i] = row0 + NR * gr + (has[i] ? i : 0);
      roff[i] = row_offset(src, rrow[i]);
    }
    if (j < NR && gr + gridDim.x < ngroups && NR * (gr + gridDim.x) + j < nrows)
      bulk_prefetch_l2(x + row_offset(src, row0 + NR * (gr + gridDim.x) + j), TT * sizeof(float));
    // v[RQ q + r] = (x_a, x_b)[j + 256 r] of pair q
    float2 v[16];
    float mx[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) mx[i] = 0.f;
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        const float xa = has[2 * q] ? __ldg(x + roff[2 * q] + j + 256 * r) : 0.0f;
        const float xb = has[2 * q + 1] ? __ldg(x + roff[2 * q + 1] + j + 256 * r) : 0.0f;
        v[RQ * q + r] = make_float2(xa, xb);
        mx[2 * q] = fmaxf(mx[2 * q], fabsf(xa));
        mx[2 * q + 1] = fmaxf(mx[2 * q + 1], fabsf(xb));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < NR; ++i) mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
    if ((j & 31) == 0)
#pragma unroll
      for (int i = 0; i < NR; ++i) red[i][j >> 5] = mx[i];
    __syncthreads();
    float sc[NR];  // per-row power-of-two scale (see the T = 4096 kernel)
#pragma unroll
    for (int i = 0; i < NR; ++i) {
#pragma unroll
      for (int w = 0; w < kFftThreads / 32; ++w) mx[i] = fmaxf(mx[i], red[i][w]);
      sc[i] = pow2_scale(mx[i]);
    }
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
      for (int r = 0; r < RQ; ++r) v[RQ * q + r] = __fmul2_rn(v[RQ * q + r], make_float2(sc[2 * q], sc[2 * q + 1]));
    // outer pass (decimation in frequency): NP radix-RQ butterflies, output s
    // of pair q times W_TT^(j s) to position 256 (RQ q + s) + j
    {
      const float2* t = tw + kTw256 + j;
      float2* pb = buf + kFftPad(j);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        dftq<false, RQ>(v, RQ * q);
#pragma unroll
        for (int sI = 0; sI < RQ; ++sI) {
          float2 y = v[RQ * q + dq<RQ>(sI)];
          if (sI > 0) y = cmul(y, t[(sI - 1) * 256]);
          pb[(RQ * q + sI) * 272] = y;
        }
      }
    }
    __syncthreads();
    load_set<16>(v, buf);
    dft16<false>(v);
    twiddle16<false, 16, true>(v, tw);
    store_set<16>(v, buf);
    __syncwarp();
    load_set<1>(v, buf);
    dft16<false>(v);
    float2 u[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const float2 z = v[d16(r)];
      u[r] = r < 8 ? make_float2(z.y, -z.x) : make_float2(-z.y, z.x);
    }
    if (j % (256 / NP) == 0) {  // DC and Nyquist of pair j / (256 / NP)
      u[0] = make_float2(0.f, 0.f);
      u[8] = make_float2(0.f, 0.f);
    }
    dft16<true>(u);
    store_set<1>(u, buf);
    __syncwarp();
    load_set<16>(u, buf);
    twiddle16<true, 16, false>(u, tw);
    dft16<true>(u);
    store_set<16>(u, buf);
    __syncthreads();
    // outer pass of the inverse (decimation in time): input s of pair q from
    // position 256 (RQ q + s) + j times conj W_TT^(j s); output r back in place
    {
      const float2* t = tw + kTw256 + j;
      float2* pb = buf + kFftPad(j);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
#pragma unroll
        for (int sI = 0; sI < RQ; ++sI) {
          float2 y = pb[(RQ * q + sI) * 272];
          if (sI > 0) {
            float2 w = t[(sI - 1) * 256];
            w.y = -w.y;
            y = cmul(y, w);
          }
          u[RQ * q + sI] = y;
        }
        dftq<true, RQ>(u, RQ * q);
      }
#pragma unroll
      for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < RQ; ++r) pb[(RQ * q + r) * 272] = u[RQ * q + dq<RQ>(r)];
    }
    __syncthreads();
    // epilogue: positions [1024 g, 1024 g + 1024) belong to pair q = 1024 g / TT
    float so[NR], amin[NR], amax[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      so[i] = sc[i] * (float)TT;
      amin[i] = FLT_MAX;
      amax[i] = 0.f;
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int q = (1024 * g) / TT;
      const int t0 = (1024 * g) % TT + 4 * j;  // sample within the row
      const int ia = 2 * q, ib = 2 * q + 1;
      if (!has[ia]) continue;  // (rows are dealt in order: pair q absent means nothing follows)
      const float4 ca = *reinterpret_cast<const float4*>(x + roff[ia] + t0);
      const float4 cb = has[ib] ? *reinterpret_cast<const float4*>(x + roff[ib] + t0) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float2* hb = buf + kFftPad(1024 * g + 4 * j);
      float2 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = hb[k];
      const float2 re[4] = {make_float2(ca.x * so[ia], cb.x * so[ib]), make_float2(ca.y * so[ia], cb.y * so[ib]),
                            make_float2(ca.z * so[ia], cb.z * so[ib]), make_float2(ca.w * so[ia], cb.w * so[ib])};
      normalize4_split_pair<GS>(re, h, out + rrow[ia] * pitch + t0, out + rrow[ib] * pitch + t0, has[ib], ps,
                                amin[ia], amax[ia], amin[ib], amax[ib]);
    }
    // row statistics: thread 32 i closes row i
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        amin[i] = fminf(amin[i], __shfl_xor_sync(0xffffffffu, amin[i], o));
        amax[i] = fmax_nan(amax[i], __shfl_xor_sync(0xffffffffu, amax[i], o));
      }
    if ((j & 31) == 0)
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        red[2 * i][j >> 5] = amin[i];
        red[2 * i + 1][j >> 5] = amax[i];
      }
    __syncthreads();
    if ((j & 31) == 0 && (j >> 5) < NR) {
      const int i = j >> 5;
      float lo = red[2 * i][0], hi = red[2 * i + 1][0];
      for (int w = 1; w < kFftThreads / 32; ++w) {
        lo = fminf(lo, red[2 * i][w]);
        hi = fmax_nan(hi, red[2 * i + 1][w]);
      }
      int need = 0;
      bool present = false;
      float scale = 1.f;
      long long rr = 0;
#pragma unroll
      for (int i2 = 0; i2 < NR; ++i2)
        if (i2 == i) {
          present = has[i2];
          scale = sc[i2];
          rr = rrow[i2];
        }
      if (present) {
        if (!(hi <= FLT_MAX)) atomicOr(&st->flags, FLAG_NONFINITE);
        lo = sqrtf(lo);
        hi = sqrtf(hi);
        int lg = 0;
        while ((1 << lg) < TT) ++lg;
        const int e = (int)((__float_as_uint(scale) >> 23) & 0xffu) - 127 + lg;  // scale TT = 2^e
        const double rs = __hiloint2double((1023 - e) << 20, 0);
        rowmin[rr] = key_of((double)lo * rs);
        rowmax[rr] = key_of((double)hi * rs);
        need = (lo == 0.0f) || ((double)lo < amp_floor * (double)hi * (1.0 + 1e-5));
      }
      need_flags[i] = need;
    }
    __syncthreads();
    // rare: keep H (input units) of a row the exact-median fixup will inspect
    bool any_need = false;
#pragma unroll
    for (int i = 0; i < NR; ++i) any_need = any_need || need_flags[i] != 0;
    if (any_need) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (!need_flags[i]) continue;
        const float un = 1.0f / so[i];
        const int q = i / 2;
        for (int t = j; t < TT; t += kFftThreads) {
          const float2 hv = buf[kFftPad(q * TT + t)];
          hbuf[(rrow[i] - src.h_row0) * src.h_ld + t] = ((i & 1) ? hv.y : hv.x) * un;
        }
      }
    }
    // the next group's first stores come after its row-max barrier
  }
}

// ---------------------------------------------------------------------------
// Exact amplitude-floor fixup.  For each row: if the cheap
// bound min|a| >= floor * max|a| holds, no sample can fall below
// floor * median and the row is untouched (the common case: Rayleigh
// amplitudes never get near 1e-6 of the median).  Otherwise the exact median
// (numpy semantics: mean of the two middle values) is found by a 64-bit radix
// select over the order-preserving bit patterns of |a|, and samples with
// |a| < floor*median or |a| == 0 are zeroed (masked).
// ---------------------------------------------------------------------------
constexpr int kFixThreads = 256;
constexpr int kFixBatch = 32;  // rows pre-checked per CTA iteration

template <typename IT, typename S, int KIND>
__device__ double row_amp(const SrcDesc& src, long long roff, long long r, long long t) {
  S re, im;
  load_a<IT, S, KIND>(src, roff, r, t, re, im);
  return static_cast<double>(amp_of(re, im));
}

template <typename IT, typename S, int KIND, int FMT>
__global__ void __launch_bounds__(kFixThreads) fixup_kernel(SrcDesc src, long long row0, long long nrows,
                                                            void* out, int pitch, long long plane_stride,
                                                            const unsigned long long* rowmin,
                                                            const unsigned long long* rowmax, int* maskcount,
                                                            double amp_floor, DevStatus* st, int batch) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long sh_prefix;
  __shared__ long long sh_k;
  __shared__ unsigned long long red_u[kFixThreads / 32];
  __shared__ long long red_c[kFixThreads / 32];
  __shared__ int need_list[kFixBatch];
  __shared__ int n_need;
  const long long T = src.T;
  // Rows are pre-checked `batch` (<= kFixBatch) at a time, one row per lane of warp 0 (the
  // common case -- no row needs the median -- is one pass of two loads per
  // row instead of a CTA-wide iteration per row); the rows that fail the
  // check are then taken one at a time by the whole CTA.
  for (long long base = (long long)blockIdx.x * batch; base < nrows; base += (long long)gridDim.x * batch) {
    if (threadIdx.x == 0) n_need = 0;
    __syncthreads();
    if (threadIdx.x < batch && base + threadIdx.x < nrows) {
      const long long r = row0 + base + threadIdx.x;
      const double amin = val_of(rowmin[r]);
      const double amax = val_of(rowmax[r]);
      // (1 + 1e-5) margin: the vectorised normaliser's min/max come from a
      // rsqrt-based |a| (a few ulp); the exact path below recomputes |a|.
      const bool need = (amin == 0.0) || (amin < amp_floor * amax * (1.0 + 1e-5));
      if (!need) maskcount[r] = 0;
      else need_list[atomicAdd(&n_need, 1)] = threadIdx.x;
    }
    __syncthreads();
    const int n_rows_needed = n_need;
   for (int q = 0; q < n_rows_needed; ++q) {
    const long long rl = base + need_list[q];
    const long long r = row0 + rl;
    const long long roff = row_offset(src, r);
    // ---- radix select of the k-th smallest key -------------------------
    auto select_kth = [&](long long k) -> unsigned long long {
      unsigned long long prefix = 0, hmask = 0;
      for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (long long t = threadIdx.x; t < T; t += blockDim.x) {
          const unsigned long long key = key_of(row_amp<IT, S, KIND>(src, roff, r, t));
          if ((key & hmask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          long long cum = 0;
          int sel = 255;
          for (int d = 0; d < 256; ++d) {
            if (cum + (long long)hist[d] > k) {
              sel = d;
              break;
            }
            cum += hist[d];
          }
          sh_k = k - cum;
          sh_prefix = prefix | ((unsigned long long)sel << shift);
        }
        __syncthreads();
        prefix = sh_prefix;
        k = sh_k;
        hmask |= 0xFFull << shift;
        __syncthreads();
      }
      return prefix;
    };
    // PhasorEpochs (KIND 2, plv_matrix input): masked
    // samples are the exact zeros -- no amplitude floor, no
    // median (the oracle's phasors_from_unit); the selection is skipped
    const long long k1 = (T % 2 == 0) ? (T / 2 - 1) : (T / 2);
    const unsigned long long v1 = KIND == 2 ? 0ull : select_kth(k1);
    unsigned long long v2 = v1;
    if (KIND != 2 && T % 2 == 0) {
      // count of keys <= v1 and the smallest key > v1
      unsigned long long mgt = ~0ull;
      long long cle = 0;
      for (long long t = threadIdx.x; t < T; t += blockDim.x) {
        const unsigned long long key = key_of(row_amp<IT, S, KIND>(src, roff, r, t));
        if (key <= v1) ++cle;
        else mgt = key < mgt ? key : mgt;
      }
      for (int o = 16; o > 0; o >>= 1) {
        cle += __shfl_xor_sync(0xffffffffu, cle, o);
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mgt, o);
        mgt = m2 < mgt ? m2 : mgt;
      }
      if ((threadIdx.x & 31) == 0) {
        red_u[threadIdx.x >> 5] = mgt;
        red_c[threadIdx.x >> 5] = cle;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 1; i < kFixThreads / 32; ++i) {
          cle += red_c[i];
          mgt = red_u[i] < mgt ? red_u[i] : mgt;
        }
        red_c[0] = cle;
        red_u[0] = mgt;
      }
      __syncthreads();
      cle = red_c[0];
      mgt = red_u[0];
      v2 = (cle >= k1 + 2) ? v1 : mgt;
      __syncthreads();
    }
    const double median = 0.5 * (val_of(v1) + val_of(v2));
    const double thr = KIND == 2 ? 0.0 : amp_floor * median;
    // ---- masking pass ---------------------------------------------------
    long long cnt = 0;
    const long long obase = (FMT == OUT_COMPLEX ? rl : r) * pitch;
    for (long long t = threadIdx.x; t < T; t += blockDim.x) {
      const double a = row_amp<IT, S, KIND>(src, roff, r, t);
      if (a < thr || a == 0.0) {
        zero_z<S, FMT>(out, plane_stride, obase + t);
        if (FMT == OUT_SPLIT && src.gauss_planes) {  // S, D planes written by the normaliser
          __half* hp = static_cast<__half*>(out);
#pragma unroll
          for (int pl = 4; pl < 8; ++pl) hp[pl * plane_stride + obase + t] = __float2half_rn(0.0f);
        }
        ++cnt;
      }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) red_c[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < kFixThreads / 32; ++i) cnt += red_c[i];
      maskcount[r] = static_cast<int>(cnt);
      atomicAdd(&st->n_fix_rows, 1);
      if (cnt > 0) {
        atomicOr(&st->flags, FLAG_ANY_MASKED);
        atomicAdd(&st->n_masked, static_cast<unsigned long long>(cnt));
      }
      if (cnt == T) atomicOr(&st->flags, FLAG_ALL_MASKED);
    }
    __syncthreads();
   }
  }
}

// PhasorEpochs (KIND 2): masked samples are the exact zeros, which the
// normaliser already wrote as z = 0; rows whose minimum |z| is 0 only need
// their zeros counted.  One warp per row, coalesced along samples (the
// general fixup's block-per-row median machinery is not needed).
template <typename IT>
__global__ void phasor_zero_count_kernel(SrcDesc src, long long row0, long long nrows,
                                         const unsigned long long* rowmin, int* maskcount, DevStatus* st) {
  const int lane = threadIdx.x & 31;
  const long long wpb = blockDim.x >> 5;
  const long long T = src.T;
  for (long long rl = (long long)blockIdx.x * wpb + (threadIdx.x >> 5); rl < nrows; rl += (long long)gridDim.x * wpb) {
    const long long r = row0 + rl;
    if (val_of(rowmin[r]) != 0.0) {
      if (lane == 0) maskcount[r] = 0;
      continue;
    }
    const long long roff = row_offset(src, r);
    long long cnt = 0;
    for (long long t = lane; t < T; t += 32) {
      const IT* q = static_cast<const IT*>(src.ptr) + 2 * (roff + t * src.s_samp);
      cnt += (q[0] == IT(0) && q[1] == IT(0)) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      maskcount[r] = static_cast<int>(cnt);
      atomicAdd(&st->n_fix_rows, 1);
      if (cnt > 0) {
        atomicOr(&st->flags, FLAG_ANY_MASKED);
        atomicAdd(&st->n_masked, static_cast<unsigned long long>(cnt));
      }
      if (cnt == T) atomicOr(&st->flags, FLAG_ALL_MASKED);
    }
  }
}

// ---------------------------------------------------------------------------
// Pack rows of a real input into a dense [nrows][T] buffer of type OT (cuFFT
// input when the caller's layout / dtype is not directly usable).
// ---------------------------------------------------------------------------
template <typename IT, typename OT>
__global__ void pack_real_kernel(SrcDesc src, long long row0, long long nrows, OT* dst) {
  const long long T = src.T;
  const long long total = nrows * T;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long rl = e / T, t = e % T;
    const long long roff = row_offset(src, row0 + rl);
    dst[e] = static_cast<OT>(static_cast<const IT*>(src.ptr)[roff + t * src.s_samp]);
  }
}

// Packing copy with per-row power-of-two scaling (max |x| -> [1, 2)), for
// lengths at which cuFFT's R2C pairs two rows of a batch into one complex
// transform (odd T): without it the rounding error of a large row leaks into
// its partner.  inv_scale[rl] = 1 / scale, applied to H downstream (SrcDesc::
// h_scale); exact, since the factors are powers of two.  One block per row.
template <typename IT, typename OT>
__global__ void __launch_bounds__(256) pack_real_scaled_kernel(SrcDesc src, long long row0, long long nrows, OT* dst,
                                                               OT* inv_scale) {
  __shared__ double red[8];
  const long long T = src.T;
  for (long long rl = blockIdx.x; rl < nrows; rl += gridDim.x) {
    const IT* x = static_cast<const IT*>(src.ptr) + row_offset(src, row0 + rl);
    double m = 0.0;
    for (long long t = threadIdx.x; t < T; t += blockDim.x) m = fmax(m, fabs((double)x[t * src.s_samp]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    for (int w = 0; w < 8; ++w) m = fmax(m, red[w]);
    __syncthreads();
    int e = 0;
    if (m > 0.0 && m <= DBL_MAX) frexp(m, &e);
    const int lim = sizeof(OT) == 4 ? 126 : 1000;
    const int sh = min(lim, max(-lim, 1 - e));
    const OT s = (OT)ldexp(1.0, sh);
    for (long long t = threadIdx.x; t < T; t += blockDim.x) dst[rl * T + t] = static_cast<OT>(x[t * src.s_samp]) * s;
    if (threadIdx.x == 0) inv_scale[rl] = (OT)ldexp(1.0, -sh);
  }
}

// In-place per-row power-of-two scaling of y[rl][0..L) (row stride ld):
// undo == 0: scale max |y| into [1, 2) and store the inverse factor;
// undo == 1: multiply by the stored inverse factor (exact restore).
template <typename S>
__global__ void __launch_bounds__(256) scale_rows_kernel(S* y, long long nrows, long long L, long long ld, S* inv_scale,
                                                         int undo) {
  __shared__ double red[8];
  for (long long rl = blockIdx.x; rl < nrows; rl += gridDim.x) {
    S* row = y + rl * ld;
    if (undo) {
      const S f = inv_scale[rl];
      for (long long t = threadIdx.x; t < L; t += blockDim.x) row[t] *= f;
      continue;
    }
    double m = 0.0;
    for (long long t = threadIdx.x; t < L; t += blockDim.x) m = fmax(m, fabs((double)row[t]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    for (int w = 0; w < 8; ++w) m = fmax(m, red[w]);
    __syncthreads();
    int e = 0;
    if (m > 0.0 && m <= DBL_MAX) frexp(m, &e);
    const int lim = sizeof(S) == 4 ? 126 : 1000;
    const int sh = min(lim, max(-lim, 1 - e));
    const S s = (S)ldexp(1.0, sh);
    for (long long t = threadIdx.x; t < L; t += blockDim.x) row[t] *= s;
    if (threadIdx.x == 0) inv_scale[rl] = (S)ldexp(1.0, -sh);
  }
}

// K2: one-sided Hilbert multiplier on the half spectrum, scaled by 1/T so the
// C2R output is H{x} directly: Y_k = -i X_k / T for strictly positive bins,
// Y_0 = Y_{T/2} = 0.
template <typename C>
__global__ void hilbert_spectrum_kernel(C* spec, long long nrows, int T) {
  const int nb = T / 2 + 1;
  const long long total = nrows * nb;
  using S = decltype(spec->x);
  const S inv = S(1) / S(T);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(e % nb);
    C v = spec[e];
    C y;
    if (k == 0 || (T % 2 == 0 && k == T / 2)) {
      y.x = S(0);
      y.y = S(0);
    } else {
      y.x = v.y * inv;
      y.y = -v.x * inv;
    }
    spec[e] = y;
  }
}

// K2h: the Hilbert multiplier for real rows of EVEN length T transformed as
// complex sequences of half the length (M = T / 2, z[n] = x[2n] + i x[2n+1],
// i.e. the row itself re-read as complex).  With Z = FFT_M(z), the transform
// of the even / odd samples is E_k = (Z_k + conj Z_{M-k}) / 2 and
// O_k = (Z_k - conj Z_{M-k}) / 2i, the row's spectrum X_k = E_k + W_T^k O_k,
// the Hilbert spectrum Y_k = -i X_k (0 < k < M), Y_0 = Y_M = 0, and the packed
// output v[n] = H[2n] + i H[2n+1] has V_k = E'_k + i O'_k with
// E'_k = (Y_k + conj Y_{M-k}) / 2, O'_k = (Y_k - conj Y_{M-k}) / (2 W_T^k).
// Substituting, everything collapses to
//   V_k = i sin(2 pi k / T) Z_k + cos(2 pi k / T) conj Z_{M-k}   (0 < k < M),  V_0 = 0,
// so R2C's split pass, the -i sgn(k) pass and C2R's merge pass become this one
// in-place pass between two C2C transforms of length M (8 instead of 24 bytes
// per sample).  The 1/M of the unnormalised inverse is folded in.
template <typename C>
__global__ void __launch_bounds__(256) hilbert_halfspec_kernel(C* spec, long long nrows, int M, int tpr) {
  using S = decltype(spec->x);
  // blockIdx.x tiles k = 0 .. M/2 (thread k handles the bins k and M - k),
  // blockIdx.y strides the rows: the twiddle is computed once per thread.
  // Short rows (M/2 + 1 < 256): tpr (a power of two) threads per row and
  // 256 / tpr rows per block, so few lanes idle.
  const int k = blockIdx.x * tpr + (threadIdx.x & (tpr - 1));
  const int rsub = threadIdx.x / tpr, rpb = 256 / tpr;
  if (k > M / 2) return;
  const int m = M - k;
  S sn, cs;
  if (sizeof(S) == 4) {
    float sf, cf;
    sincospif((float)k / (float)M, &sf, &cf);  // 2 pi k / T = pi k / M
    sn = sf;
    cs = cf;
  } else {
    double sd, cd;
    sincospi((double)k / (double)M, &sd, &cd);
    sn = sd;
    cs = cd;
  }
  const S inv = S(1) / S(M);
  sn *= inv;
  cs *= inv;
  for (long long row = (long long)blockIdx.y * rpb + rsub; row < nrows; row += (long long)gridDim.y * rpb) {
    C* z = spec + row * M;
    if (k == 0) {
      C v;
      v.x = S(0);
      v.y = S(0);
      z[0] = v;
    } else if (m == k) {  // M even, k = M / 2: cos = 0
      const C a = z[k];
      C v;
      v.x = -sn * a.y;
      v.y = sn * a.x;
      z[k] = v;
    } else {
      const C a = z[k], b = z[m];
      C vk, vm;
      vk.x = cs * b.x - sn * a.y;
      vk.y = sn * a.x - cs * b.y;
      vm.x = -sn * b.y - cs * a.x;
      vm.y = sn * b.x + cs * a.y;
      z[k] = vk;
      z[m] = vm;
    }
  }
}

// analytic output: out[rl][t] = (x, H) -- Re taken from x unchanged.
template <typename IT, typename S>
__global__ void analytic_out_kernel(SrcDesc src, long long row0, long long nrows, S* out) {
  const long long T = src.T;
  const long long total = nrows * T;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long rl = e / T, t = e % T;
    const long long r = row0 + rl;
    const long long roff = row_offset(src, r);
    S re, im;
    load_a<IT, S, 0>(src, roff, r, t, re, im);
    out[2 * e] = re;
    out[2 * e + 1] = im;
  }
}

// out_m[i] = sum_g ws_m[g][i] / R  (deterministic fixed-order trial-group sum; fp32:
// times the fp32 reciprocal, as every split-path mean)
template <typename S>
__global__ void group_reduce_kernel(const S* ws, int G, long long slot_elems, long long elems, int R,
                                    S* out, long long upper_n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < elems;
       e += (long long)gridDim.x * blockDim.x) {
    // slot layout of ws: [band][G][N*N]; elems = B*N*N, slot_elems = N*N
    const long long b = e / slot_elems, i = e % slot_elems;
    if (upper_n && i / upper_n > i % upper_n) continue;  // PS_LAYOUT_UPPER: lower triangle untouched
    const S* p = ws + (b * G) * slot_elems + i;
    S acc = p[0];
    for (int g = 1; g < G; ++g) acc += p[g * slot_elems];
    out[e] = sizeof(S) == 4 ? (acc == S(R) ? S(1) : acc * (S(1) / S(R))) : acc / S(R);  // = epilogue.cuh mean_scale
  }
}

// Time-resolved mode (Eq 8): re-key the phasor planes so the
// Gram's K axis runs over trials.  src [P][B*R][N][Tp] -> dst [P][B*T][N][Rp]
// (P = 4 fp16 planes or 2 f64 planes), trial padding zeroed; maskcount_dst
// [(b*T + t)*N + n] = number of masked trials (masked samples are exactly 0 in
// every plane).
// One block per (band, signal, 32-sample tile): the [R][32] slab of every
// plane goes through shared memory in 32 x 32 tiles, so reads run along t and
// writes along r (both coalesced); a trial is masked at sample t when all its
// planes are zero there (warp ballot per written row).
constexpr int kTrTile = 32;
template <typename E, int P>
__global__ void __launch_bounds__(kTrTile * 8) transpose_trials_kernel(
    const E* __restrict__ src, long long sps, int Tp, E* __restrict__ dst, long long dps, int Rp, int B, int R, int N,
    int T, int* __restrict__ maskcount_dst) {
  __shared__ E tile[P][kTrTile][kTrTile + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int ntt = (T + kTrTile - 1) / kTrTile;
  const long long blk = blockIdx.x;
  const int tt = (int)(blk % ntt);
  const long long bn = blk / ntt;
  const int n = (int)(bn % N);
  const int b = (int)(bn / N);
  const int t0 = tt * kTrTile;
  int masked = 0;  // per written row t = t0 + ty + k*8, accumulated by lane 0 of the warp
  int mk[kTrTile / 8] = {};
  for (int r0 = 0; r0 < Rp; r0 += kTrTile) {
#pragma unroll
    for (int k = 0; k < kTrTile / 8; ++k) {
      const int r = r0 + ty + 8 * k, t = t0 + tx;
      const long long sidx = ((long long)(b * R + r) * N + n) * Tp + t;
#pragma unroll
      for (int pl = 0; pl < P; ++pl) tile[pl][ty + 8 * k][tx] = (r < R && t < T) ? src[pl * sps + sidx] : E(0.0f);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTrTile / 8; ++k) {
      const int t = t0 + ty + 8 * k, r = r0 + tx;
      bool zero = true;
      E v[P];
#pragma unroll
      for (int pl = 0; pl < P; ++pl) {
        v[pl] = tile[pl][tx][ty + 8 * k];
        zero = zero && (static_cast<float>(v[pl]) == 0.0f);
      }
      if (t < T && r < Rp) {
        const long long didx = ((long long)(b * T + t) * N + n) * Rp + r;
#pragma unroll
        for (int pl = 0; pl < P; ++pl) dst[pl * dps + didx] = v[pl];
      }
      mk[k] += __popc(__ballot_sync(0xffffffffu, zero && r < R));
    }
    __syncthreads();
  }
  (void)masked;
  if (tx == 0) {
#pragma unroll
    for (int k = 0; k < kTrTile / 8; ++k) {
      const int t = t0 + ty + 8 * k;
      if (t < T) maskcount_dst[(long long)(b * T + t) * N + n] = mk[k];
    }
  }
}

int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148LL * 16) g = 148LL * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// Band-pass front end (DESIGN.md section 8(f) #1).
// The two-pass zero-phase FIR is evaluated spectrally on FFT length Lf >=
// L + n_taps - 1 (L = T + 2 pad): linear convolution without wrap-around,
// the first pass truncated to L samples exactly as the time-domain filter
// with zero initial state leaves it.
// ---------------------------------------------------------------------------
// xp[rl][i] = reflect-padded x (numpy 'reflect') for i < L, 0 for L <= i < Lf
template <typename IT, typename S>
__global__ void reflect_pad_kernel(SrcDesc src, long long row0, long long nrows, long long pad, long long L,
                                   long long Lf, S* xp) {
  const long long total = nrows * Lf;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long rl = e / Lf, i = e % Lf;
    S v = S(0);
    if (i < L) {
      long long j = i - pad;
      if (j < 0) j = -j;
      if (j >= src.T) j = 2 * (src.T - 1) - j;
      const long long roff = row_offset(src, row0 + rl);
      v = static_cast<S>(static_cast<const IT*>(src.ptr)[roff + j * src.s_samp]);
    }
    xp[e] = v;
  }
}

// spec[rl][k] *= (conj ? conj(Hf[k]) : Hf[k]) * scale
template <typename C>
__global__ void spectrum_mul_kernel(C* spec, long long nrows, long long nb, const double2* Hf, int conj,
                                    double scale) {
  using S = decltype(spec->x);
  const long long total = nrows * nb;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const double2 h = Hf[e % nb];
    const S hr = static_cast<S>(h.x * scale), hi = static_cast<S>((conj ? -h.y : h.y) * scale);
    const C v = spec[e];
    C y;
    y.x = v.x * hr - v.y * hi;
    y.y = v.x * hi + v.y * hr;
    spec[e] = y;
  }
}

// y[rl][i] = 0 for L <= i < Lf (first-pass truncation)
template <typename S>
__global__ void zero_tail_kernel(S* y, long long nrows, long long L, long long Lf) {
  const long long w = Lf - L;
  const long long total = nrows * w;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    y[(e / w) * Lf + L + e % w] = S(0);
}

// ---------------------------------------------------------------------------
// Welch coherence front end (DESIGN.md 8(f) #3)
// ---------------------------------------------------------------------------
// seg[(row * S + s) * W + t] = x[row][s * hop + t] * win[t]
template <typename IT, typename S>
__global__ void welch_segments_kernel(SrcDesc src, long long rows, int nseg, int W, int hop, const double* win,
                                      S* seg) {
  const long long per = (long long)nseg * W;
  const long long total = rows * per;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / per, rem = e % per;
    const long long s = rem / W, t = rem % W;
    const IT v = static_cast<const IT*>(src.ptr)[row_offset(src, row) + (s * hop + t) * src.s_samp];
    seg[e] = static_cast<S>(static_cast<double>(v) * win[t]);
  }
}

// One warp per (band b, bin kb, signal n): the spectra X_n,q(k0 + kb) over the
// K = R * S segments (q = r * S + s), scaled by sqrt(K / sum_q |X|^2) so the
// Gram over q divided by K is the normalised cross-spectrum; written as the
// Gram operand row ((b * nb + kb) * N + n) of K samples (pitch Kp, zero pad).
template <typename C, bool SPLIT>
__global__ void coherence_planes_kernel(const C* __restrict__ spec, int nbW, long long B, long long R, long long N,
                                        int nseg, int k0, int nb, int K, int Kp, void* planes, long long ps) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= B * nb * N) return;
  const long long n = w % N, kb = (w / N) % nb, b = w / (N * nb);
  auto at = [&](int q) -> C {
    const long long r = q / nseg, s = q % nseg;
    return spec[(((b * R + r) * N + n) * nseg + s) * nbW + k0 + kb];
  };
  double sum = 0.0;
  for (int q = lane; q < K; q += 32) {
    const C x = at(q);
    sum += (double)x.x * (double)x.x + (double)x.y * (double)x.y;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double scale = sum > 0.0 ? sqrt((double)K / sum) : 0.0;
  const long long row = (b * nb + kb) * N + n;
  for (int q = lane; q < Kp; q += 32) {
    double re = 0.0, im = 0.0;
    if (q < K) {
      const C x = at(q);
      re = (double)x.x * scale;
      im = (double)x.y * scale;
    }
    const long long idx = row * Kp + q;
    if (SPLIT) {
      __half* p = static_cast<__half*>(planes);
      const __half rh = __float2half_rn((float)re), ih = __float2half_rn((float)im);
      p[idx] = rh;
      p[ps + idx] = __float2half_rn((float)(re - (double)__half2float(rh)));
      p[2 * ps + idx] = ih;
      p[3 * ps + idx] = __float2half_rn((float)(im - (double)__half2float(ih)));
    } else {
      double* p = static_cast<double*>(planes);
      p[idx] = re;
      p[ps + idx] = im;
    }
  }
}

// out[b][e] = max_kb ws[b * nb + kb][e]
template <typename S>
__global__ void band_max_kernel(const S* ws, long long B, long long nb, long long nn, S* out, long long upper_n) {
  const long long total = B * nn;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / nn, i = e % nn;
    if (upper_n && i / upper_n > i % upper_n) continue;  // PS_LAYOUT_UPPER
    S m = ws[(b * nb) * nn + i];
    for (long long kb = 1; kb < nb; ++kb) {
      const S v = ws[(b * nb + kb) * nn + i];
      m = v > m ? v : m;
    }
    out[e] = m;
  }
}

// out[rl][t] = y[rl][pad + t] (dense trimmed rows)
template <typename S>
__global__ void trim_rows_kernel(const S* y, long long nrows, long long ld, long long pad, long long T, S* out) {
  const long long total = nrows * T;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = y[(e / T) * ld + pad + e % T];
}

}  // namespace

cudaError_t launch_reflect_pad(const SrcDesc& src, long long row0, long long nrows, long long pad, long long L,
                               long long Lf, void* xp, int dst_double, cudaStream_t st) {
  const int g = grid_for(nrows * Lf, 256);
  if (src.is_double) {
    if (!dst_double) return cudaErrorInvalidValue;
    reflect_pad_kernel<double, double><<<g, 256, 0, st>>>(src, row0, nrows, pad, L, Lf, (double*)xp);
  } else if (dst_double) {
    reflect_pad_kernel<float, double><<<g, 256, 0, st>>>(src, row0, nrows, pad, L, Lf, (double*)xp);
  } else {
    reflect_pad_kernel<float, float><<<g, 256, 0, st>>>(src, row0, nrows, pad, L, Lf, (float*)xp);
  }
  return cudaGetLastError();
}

// *dst = *src by one thread: dst may be mapped pinned host memory, so a
// counter reaches the host without a copy-engine transfer (which would queue
// behind bulk D2H copies of other streams)
__global__ void copy_u64_kernel(const unsigned long long* src, volatile unsigned long long* dst) {
  *dst = *src;
  __threadfence_system();
}

cudaError_t launch_copy_u64(const unsigned long long* src, unsigned long long* dst, cudaStream_t st) {
  copy_u64_kernel<<<1, 1, 0, st>>>(src, dst);
  return cudaGetLastError();
}

cudaError_t launch_welch_segments(const SrcDesc& src, long long rows, int nseg, int W, int hop, const double* win,
                                  void* seg, int dst_double, cudaStream_t st) {
  const int g = grid_for(rows * nseg * (long long)W, 256);
  if (src.is_double) {
    if (!dst_double) return cudaErrorInvalidValue;
    welch_segments_kernel<double, double><<<g, 256, 0, st>>>(src, rows, nseg, W, hop, win, (double*)seg);
  } else if (dst_double) {
    welch_segments_kernel<float, double><<<g, 256, 0, st>>>(src, rows, nseg, W, hop, win, (double*)seg);
  } else {
    welch_segments_kernel<float, float><<<g, 256, 0, st>>>(src, rows, nseg, W, hop, win, (float*)seg);
  }
  return cudaGetLastError();
}

cudaError_t launch_coherence_planes(const void* spec, int spec_double, int nbW, long long B, long long R, long long N,
                                    int nseg, int k0, int nb, int K, int Kp, void* planes, long long ps, int split,
                                    cudaStream_t st) {
  const long long warps = B * nb * N;
  const long long blocks = (warps * 32 + 255) / 256;
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned g = (unsigned)blocks;
  if (spec_double) {
    if (split)
      coherence_planes_kernel<double2, true><<<g, 256, 0, st>>>((const double2*)spec, nbW, B, R, N, nseg, k0, nb, K,
                                                                 Kp, planes, ps);
    else
      coherence_planes_kernel<double2, false><<<g, 256, 0, st>>>((const double2*)spec, nbW, B, R, N, nseg, k0, nb, K,
                                                                  Kp, planes, ps);
  } else {
    if (split)
      coherence_planes_kernel<float2, true><<<g, 256, 0, st>>>((const float2*)spec, nbW, B, R, N, nseg, k0, nb, K, Kp,
                                                                planes, ps);
    else
      coherence_planes_kernel<float2, false><<<g, 256, 0, st>>>((const float2*)spec, nbW, B, R, N, nseg, k0, nb, K,
                                                                 Kp, planes, ps);
  }
  return cudaGetLastError();
}

cudaError_t launch_band_max(const void* ws, long long B, long long nb, long long nn, void* out, int is_double,
                            cudaStream_t st, long long upper_n) {
  const int g = grid_for(B * nn, 256);
  if (is_double) band_max_kernel<double><<<g, 256, 0, st>>>((const double*)ws, B, nb, nn, (double*)out, upper_n);
  else band_max_kernel<float><<<g, 256, 0, st>>>((const float*)ws, B, nb, nn, (float*)out, upper_n);
  return cudaGetLastError();
}

cudaError_t launch_spectrum_mul(void* spec, long long nrows, long long nb, const void* Hf, int conj, double scale,
                                int is_double, cudaStream_t st) {
  const int g = grid_for(nrows * nb, 256);
  if (is_double)
    spectrum_mul_kernel<double2><<<g, 256, 0, st>>>((double2*)spec, nrows, nb, (const double2*)Hf, conj, scale);
  else
    spectrum_mul_kernel<float2><<<g, 256, 0, st>>>((float2*)spec, nrows, nb, (const double2*)Hf, conj, scale);
  return cudaGetLastError();
}

cudaError_t launch_zero_tail(void* y, long long nrows, long long L, long long Lf, int is_double, cudaStream_t st) {
  if (Lf <= L) return cudaSuccess;
  const int g = grid_for(nrows * (Lf - L), 256);
  if (is_double) zero_tail_kernel<double><<<g, 256, 0, st>>>((double*)y, nrows, L, Lf);
  else zero_tail_kernel<float><<<g, 256, 0, st>>>((float*)y, nrows, L, Lf);
  return cudaGetLastError();
}

cudaError_t launch_trim_rows(const void* y, long long nrows, long long ld, long long pad, long long T, void* out,
                             int is_double, cudaStream_t st) {
  const int g = grid_for(nrows * T, 256);
  if (is_double) trim_rows_kernel<double><<<g, 256, 0, st>>>((const double*)y, nrows, ld, pad, T, (double*)out);
  else trim_rows_kernel<float><<<g, 256, 0, st>>>((const float*)y, nrows, ld, pad, T, (float*)out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_pack_real(const SrcDesc& src, long long row0, long long nrows, void* dst, int dst_double,
                             cudaStream_t st) {
  const int g = grid_for(nrows * src.T, 256);
  if (src.is_double) {
    if (dst_double) pack_real_kernel<double, double><<<g, 256, 0, st>>>(src, row0, nrows, (double*)dst);
    else return cudaErrorInvalidValue;
  } else {
    if (dst_double) pack_real_kernel<float, double><<<g, 256, 0, st>>>(src, row0, nrows, (double*)dst);
    else pack_real_kernel<float, float><<<g, 256, 0, st>>>(src, row0, nrows, (float*)dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_real_scaled(const SrcDesc& src, long long row0, long long nrows, void* dst, void* inv_scale,
                                    int dst_double, cudaStream_t st) {
  const unsigned g = (unsigned)(nrows < 148 * 16 ? nrows : 148 * 16);
  if (nrows <= 0) return cudaSuccess;
  if (src.is_double) {
    if (!dst_double) return cudaErrorInvalidValue;
    pack_real_scaled_kernel<double, double><<<g, 256, 0, st>>>(src, row0, nrows, (double*)dst, (double*)inv_scale);
  } else if (dst_double) {
    pack_real_scaled_kernel<float, double><<<g, 256, 0, st>>>(src, row0, nrows, (double*)dst, (double*)inv_scale);
  } else {
    pack_real_scaled_kernel<float, float><<<g, 256, 0, st>>>(src, row0, nrows, (float*)dst, (float*)inv_scale);
  }
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(void* y, long long nrows, long long L, long long ld, void* inv_scale, int undo,
                              int is_double, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  const unsigned g = (unsigned)(nrows < 148 * 16 ? nrows : 148 * 16);
  if (is_double) scale_rows_kernel<double><<<g, 256, 0, st>>>((double*)y, nrows, L, ld, (double*)inv_scale, undo);
  else scale_rows_kernel<float><<<g, 256, 0, st>>>((float*)y, nrows, L, ld, (float*)inv_scale, undo);
  return cudaGetLastError();
}

cudaError_t launch_hilbert_spectrum(void* spec, long long nrows, int T, int is_double, cudaStream_t st) {
  const int g = grid_for(nrows * (T / 2 + 1), 256);
  if (is_double) hilbert_spectrum_kernel<double2><<<g, 256, 0, st>>>((double2*)spec, nrows, T);
  else hilbert_spectrum_kernel<float2><<<g, 256, 0, st>>>((float2*)spec, nrows, T);
  return cudaGetLastError();
}

cudaError_t launch_hilbert_halfspec(void* spec, long long nrows, int T, int is_double, cudaStream_t st) {
  const int M = T / 2;
  const int per_row = M / 2 + 1;
  int tpr = 256;  // threads per row: the smallest power of two covering the row, at most 256
  while (tpr / 2 >= per_row && tpr > 1) tpr /= 2;
  const int rpb = 256 / tpr;
  const int kb = (per_row + tpr - 1) / tpr;
  // enough row-strided blocks to fill the GPU a few times over; every thread
  // keeps its twiddle across its rows
  long long ry = (148LL * 16 + kb - 1) / kb;
  ry = std::max(1LL, std::min(ry, std::min((nrows + rpb - 1) / rpb, 65535LL)));
  const dim3 g((unsigned)kb, (unsigned)ry);
  if (is_double) hilbert_halfspec_kernel<double2><<<g, 256, 0, st>>>((double2*)spec, nrows, M, tpr);
  else hilbert_halfspec_kernel<float2><<<g, 256, 0, st>>>((float2*)spec, nrows, M, tpr);
  return cudaGetLastError();
}

bool hilbert_fused_supported(const SrcDesc& src, int fmt, int cdouble, int pitch) {
  const bool aligned = (reinterpret_cast<uintptr_t>(src.ptr) & 15u) == 0 && src.s_samp == 1 && src.s_sig % 4 == 0 &&
                       (src.R == 1 || src.s_trial % 4 == 0) && (src.B == 1 || src.s_band % 4 == 0);
  const bool len_ok = (src.T == kFftT || src.T == kFftT / 2 || src.T == kFftT / 4) && pitch == src.T;
  return src.kind == 0 && !src.is_double && !cdouble && fmt == OUT_SPLIT && len_ok && aligned;
}

template <bool GS, int NP>
cudaError_t launch_hilbert_fused_short_t(const SrcDesc& src, long long row0, long long nrows, __half* out, int pitch,
                                         long long plane_stride, unsigned long long* rowstat, long long rows_total,
                                         double amp_floor, DevStatus* status, cudaStream_t st) {
  auto kern = hilbert_fused_short_kernel<GS, NP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kFftSmemBytes);
  if (e != cudaSuccess) return e;
  int dev = 0, n_sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFftThreads, kFftSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long groups = (nrows + 2 * NP - 1) / (2 * NP);
  const long long cap = (long long)per_sm * n_sms;
  const unsigned grid = (unsigned)(groups < cap ? groups : cap);
  kern<<<grid, kFftThreads, kFftSmemBytes, st>>>(src, row0, nrows, out, pitch, plane_stride, rowstat,
                                                 rowstat + rows_total,
                                                 static_cast<float*>(const_cast<void*>(src.hbuf)), amp_floor, status);
  return cudaGetLastError();
}

template <bool GS>
cudaError_t launch_hilbert_fused_t(const SrcDesc& src, long long row0, long long nrows, __half* out, int pitch,
                                   long long plane_stride, unsigned long long* rowstat, long long rows_total,
                                   double amp_floor, DevStatus* status, cudaStream_t st) {
  // the attribute is per device: set it on every launch (cheap), so a process
  // driving several GPUs gets it on each
  cudaError_t e = cudaFuncSetAttribute(hilbert_fused4096_kernel<GS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kFftSmemBytes);
  if (e != cudaSuccess) return e;
  int dev = 0, n_sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hilbert_fused4096_kernel<GS>, kFftThreads,
                                                    kFftSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long npairs = (nrows + 1) / 2;
  const long long cap = (long long)per_sm * n_sms;
  const unsigned grid = (unsigned)(npairs < cap ? npairs : cap);
  hilbert_fused4096_kernel<GS><<<grid, kFftThreads, kFftSmemBytes, st>>>(
      src, row0, nrows, out, pitch, plane_stride, rowstat, rowstat + rows_total,
      static_cast<float*>(const_cast<void*>(src.hbuf)), amp_floor, status);
  return cudaGetLastError();
}

// With src.gauss_planes the kernel also writes the Gauss-Gram S / D planes
// (planes 4..7); *gauss_done reports it.
cudaError_t launch_hilbert_fused(const SrcDesc& src, long long row0, long long nrows, void* out, int pitch,
                                 long long plane_stride, unsigned long long* rowstat, long long rows_total,
                                 double amp_floor, DevStatus* status, cudaStream_t st, int* gauss_done) {
  if (gauss_done) *gauss_done = src.gauss_planes ? 1 : 0;
  if (nrows <= 0) return cudaSuccess;
  __half* o = static_cast<__half*>(out);
  static const bool unified = std::getenv("PS_HILBERT_UNIFIED") != nullptr;  // experiment: NP = 1 of the short kernel
  if (src.T == kFftT && unified)
    return src.gauss_planes ? launch_hilbert_fused_short_t<true, 1>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                    rows_total, amp_floor, status, st)
                            : launch_hilbert_fused_short_t<false, 1>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                     rows_total, amp_floor, status, st);
  if (src.T == kFftT / 2)
    return src.gauss_planes ? launch_hilbert_fused_short_t<true, 2>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                    rows_total, amp_floor, status, st)
                            : launch_hilbert_fused_short_t<false, 2>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                     rows_total, amp_floor, status, st);
  if (src.T == kFftT / 4)
    return src.gauss_planes ? launch_hilbert_fused_short_t<true, 4>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                    rows_total, amp_floor, status, st)
                            : launch_hilbert_fused_short_t<false, 4>(src, row0, nrows, o, pitch, plane_stride, rowstat,
                                                                     rows_total, amp_floor, status, st);
  return src.gauss_planes
             ? launch_hilbert_fused_t<true>(src, row0, nrows, o, pitch, plane_stride, rowstat, rows_total, amp_floor,
                                            status, st)
             : launch_hilbert_fused_t<false>(src, row0, nrows, o, pitch, plane_stride, rowstat, rows_total,
                                             amp_floor, status, st);
}

// Gauss-Gram operand planes: S = Zr + Zi and D = Zr - Zi from the split
// planes {Re hi, Re lo, Im hi, Im lo} of the same samples, as hi / lo fp16
// pairs in planes 4..7 (flat element range [e0, e1) of every plane, 8-aligned).
__global__ void gauss_planes_kernel(__half* planes, long long ps, long long e0, long long e1) {
  const long long n8 = (e1 - e0) / 8;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n8; v += (long long)gridDim.x * blockDim.x) {
    const long long e = e0 + 8 * v;
    const uint4 rh = *reinterpret_cast<const uint4*>(planes + e);
    const uint4 rl = *reinterpret_cast<const uint4*>(planes + ps + e);
    const uint4 ih = *reinterpret_cast<const uint4*>(planes + 2 * ps + e);
    const uint4 il = *reinterpret_cast<const uint4*>(planes + 3 * ps + e);
    const __half* prh = reinterpret_cast<const __half*>(&rh);
    const __half* prl = reinterpret_cast<const __half*>(&rl);
    const __half* pih = reinterpret_cast<const __half*>(&ih);
    const __half* pil = reinterpret_cast<const __half*>(&il);
    __align__(16) __half sh[8], sl[8], dh[8], dl[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float zr = __half2float(prh[k]) + __half2float(prl[k]);
      const float zi = __half2float(pih[k]) + __half2float(pil[k]);
      const float S = zr + zi, D = zr - zi;
      sh[k] = __float2half_rn(S);
      sl[k] = __float2half_rn(S - __half2float(sh[k]));
      dh[k] = __float2half_rn(D);
      dl[k] = __float2half_rn(D - __half2float(dh[k]));
    }
    *reinterpret_cast<uint4*>(planes + 4 * ps + e) = *reinterpret_cast<const uint4*>(sh);
    *reinterpret_cast<uint4*>(planes + 5 * ps + e) = *reinterpret_cast<const uint4*>(sl);
    *reinterpret_cast<uint4*>(planes + 6 * ps + e) = *reinterpret_cast<const uint4*>(dh);
    *reinterpret_cast<uint4*>(planes + 7 * ps + e) = *reinterpret_cast<const uint4*>(dl);
  }
}

cudaError_t launch_gauss_planes(void* planes, long long plane_stride, long long e0, long long e1, cudaStream_t st) {
  if (e1 <= e0) return cudaSuccess;
  const long long n8 = (e1 - e0) / 8;
  const unsigned grid = (unsigned)std::min<long long>((n8 + 255) / 256, 148LL * 16);
  gauss_planes_kernel<<<grid, 256, 0, st>>>(static_cast<__half*>(planes), plane_stride, e0, e1);
  return cudaGetLastError();
}

// fmt: 0 split fp16 planes, 1 f64 planes, 2 complex interleaved (of compute type)
#define PS_NORM_DISPATCH(KIND, FMT)                                                                  \
  do {                                                                                               \
    if (src.is_double)                                                                               \
      normalize_kernel<double, double, KIND, FMT>                                                    \
          <<<grid, kNormThreads, 0, st>>>(src, row0, chunks, out, pitch, plane_stride, rowmin, rowmax, \
                                          status);                                                   \
    else if (cdouble)                                                                                \
      normalize_kernel<float, double, KIND, FMT>                                                     \
          <<<grid, kNormThreads, 0, st>>>(src, row0, chunks, out, pitch, plane_stride, rowmin, rowmax, \
                                          status);                                                   \
    else                                                                                             \
      normalize_kernel<float, float, KIND, FMT>                                                      \
          <<<grid, kNormThreads, 0, st>>>(src, row0, chunks, out, pitch, plane_stride, rowmin, rowmax, \
                                          status);                                                   \
  } while (0)

cudaError_t launch_normalize_fmt(const SrcDesc& src, long long row0, long long nrows, void* out, int fmt,
                                 int cdouble, int pitch, long long plane_stride, unsigned long long* rowstat,
                                 long long rows_total, DevStatus* status, cudaStream_t st, int* gauss_done) {
  if (gauss_done) *gauss_done = 0;
  // vectorised fast path: fp32 source, split planes, contiguous 16B-aligned rows
  {
    const bool aligned_base = (reinterpret_cast<uintptr_t>(src.ptr) & 15u) == 0 &&
                              (src.kind != 0 || ((reinterpret_cast<uintptr_t>(src.hbuf) & 15u) == 0 &&
                                                 src.h_ld % 4 == 0));
    const long long q = src.kind == 0 ? 4 : 2;  // row offsets must be 16-byte multiples
    const bool strides_ok = (src.s_sig % q == 0) && (src.R == 1 || src.s_trial % q == 0) &&
                            (src.B == 1 || src.s_band % q == 0);
    if (fmt == OUT_SPLIT && !cdouble && !src.is_double && src.s_samp == 1 && src.T % 4 == 0 && aligned_base &&
        strides_ok) {
      const int vchunks = static_cast<int>((src.T + kVecSamplesPerBlock - 1) / kVecSamplesPerBlock);
      const long long vblk = nrows * vchunks;
      if (vblk <= 0) return cudaSuccess;
      if (vblk > 0x7fffffffLL) return cudaErrorInvalidValue;
      __half* o = static_cast<__half*>(out);
      unsigned long long* rmin = rowstat;
      unsigned long long* rmax = rowstat + rows_total;
      if (gauss_done) *gauss_done = src.gauss_planes ? 1 : 0;
      if (src.T % 128 == 0 && src.T * 2 <= kVecSamplesPerBlock && pitch == src.T) {  // short rows: several per block
        const int rpb = (int)(kVecSamplesPerBlock / src.T);
        const long long blocks = (nrows + rpb - 1) / rpb;
        if (src.kind == 0)
          normalize_vec_rows_kernel<0><<<(unsigned)blocks, kNormThreads, 0, st>>>(src, row0, nrows, rpb, o, pitch,
                                                                                plane_stride, rmin, rmax, status);
        else if (src.kind == 1)
          normalize_vec_rows_kernel<1><<<(unsigned)blocks, kNormThreads, 0, st>>>(src, row0, nrows, rpb, o, pitch,
                                                                                plane_stride, rmin, rmax, status);
        else
          normalize_vec_rows_kernel<2><<<(unsigned)blocks, kNormThreads, 0, st>>>(src, row0, nrows, rpb, o, pitch,
                                                                                plane_stride, rmin, rmax, status);
        return cudaGetLastError();
      }
      if (src.kind == 0)
        normalize_vec_kernel<0><<<(unsigned)vblk, kNormThreads, 0, st>>>(src, row0, vchunks, o, pitch, plane_stride,
                                                                         rmin, rmax, status);
      else if (src.kind == 1)
        normalize_vec_kernel<1><<<(unsigned)vblk, kNormThreads, 0, st>>>(src, row0, vchunks, o, pitch, plane_stride,
                                                                         rmin, rmax, status);
      else
        normalize_vec_kernel<2><<<(unsigned)vblk, kNormThreads, 0, st>>>(src, row0, vchunks, o, pitch, plane_stride,
                                                                         rmin, rmax, status);
      return cudaGetLastError();
    }
  }
  const int chunks = static_cast<int>((src.T + kNormSamplesPerBlock - 1) / kNormSamplesPerBlock);
  const long long nblk = nrows * chunks;
  if (nblk <= 0) return cudaSuccess;
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned grid = static_cast<unsigned>(nblk);
  unsigned long long* rowmin = rowstat;
  unsigned long long* rowmax = rowstat + rows_total;
  // real input with a float source but double compute keeps H in double
  if (src.kind == 0) {
    if (fmt == OUT_SPLIT) PS_NORM_DISPATCH(0, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_NORM_DISPATCH(0, OUT_F64);
    else PS_NORM_DISPATCH(0, OUT_COMPLEX);
  } else if (src.kind == 1) {
    if (fmt == OUT_SPLIT) PS_NORM_DISPATCH(1, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_NORM_DISPATCH(1, OUT_F64);
    else PS_NORM_DISPATCH(1, OUT_COMPLEX);
  } else {
    if (fmt == OUT_SPLIT) PS_NORM_DISPATCH(2, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_NORM_DISPATCH(2, OUT_F64);
    else PS_NORM_DISPATCH(2, OUT_COMPLEX);
  }
  return cudaGetLastError();
}
#undef PS_NORM_DISPATCH

#define PS_FIX_DISPATCH(KIND, FMT)                                                                    \
  do {                                                                                              \
    if (src.is_double)                                                                              \
      fixup_kernel<double, double, KIND, FMT><<<grid, kFixThreads, 0, st>>>(                        \
          src, row0, nrows, out, pitch, plane_stride, rowmin, rowmax, maskcount, amp_floor, status, batch); \
    else if (cdouble)                                                                               \
      fixup_kernel<float, double, KIND, FMT><<<grid, kFixThreads, 0, st>>>(                         \
          src, row0, nrows, out, pitch, plane_stride, rowmin, rowmax, maskcount, amp_floor, status, batch); \
    else                                                                                            \
      fixup_kernel<float, float, KIND, FMT><<<grid, kFixThreads, 0, st>>>(                          \
          src, row0, nrows, out, pitch, plane_stride, rowmin, rowmax, maskcount, amp_floor, status, batch); \
  } while (0)

cudaError_t launch_fixup_fmt(const SrcDesc& src, long long row0, long long nrows, void* out, int fmt,
                             int cdouble, int pitch, long long plane_stride, const unsigned long long* rowstat,
                             long long rows_total, int* maskcount, double amp_floor, DevStatus* status,
                             cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  // rows per pre-check batch: as many as keep 148 * 8 CTAs busy when every
  // row needs the exact pass, at most one per lane of a warp
  const int batch = (int)std::max(1LL, std::min<long long>(kFixBatch, nrows / (148 * 8)));
  const long long batches = (nrows + batch - 1) / batch;
  const unsigned grid = static_cast<unsigned>(batches < 148 * 8 ? batches : 148 * 8);
  const unsigned long long* rowmin = rowstat;
  const unsigned long long* rowmax = rowstat + rows_total;
  if (src.kind == 2) {  // phasors: count the exact zeros (no median)
    const unsigned g = static_cast<unsigned>(std::min<long long>((nrows + 7) / 8, 148LL * 16));
    if (src.is_double)
      phasor_zero_count_kernel<double><<<g, 256, 0, st>>>(src, row0, nrows, rowmin, maskcount, status);
    else
      phasor_zero_count_kernel<float><<<g, 256, 0, st>>>(src, row0, nrows, rowmin, maskcount, status);
    return cudaGetLastError();
  }
  if (src.kind == 0) {
    if (fmt == OUT_SPLIT) PS_FIX_DISPATCH(0, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_FIX_DISPATCH(0, OUT_F64);
    else PS_FIX_DISPATCH(0, OUT_COMPLEX);
  } else if (src.kind == 1) {
    if (fmt == OUT_SPLIT) PS_FIX_DISPATCH(1, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_FIX_DISPATCH(1, OUT_F64);
    else PS_FIX_DISPATCH(1, OUT_COMPLEX);
  } else {
    if (fmt == OUT_SPLIT) PS_FIX_DISPATCH(2, OUT_SPLIT);
    else if (fmt == OUT_F64) PS_FIX_DISPATCH(2, OUT_F64);
    else PS_FIX_DISPATCH(2, OUT_COMPLEX);
  }
  return cudaGetLastError();
}
#undef PS_FIX_DISPATCH

cudaError_t launch_analytic_out(const SrcDesc& src, long long row0, long long nrows, void* out,
                                cudaStream_t st) {
  const int g = grid_for(nrows * src.T, 256);
  // hbuf type decides the output precision: f64 input -> c128, else c64
  if (src.is_double) analytic_out_kernel<double, double><<<g, 256, 0, st>>>(src, row0, nrows, (double*)out);
  else analytic_out_kernel<float, float><<<g, 256, 0, st>>>(src, row0, nrows, (float*)out);
  return cudaGetLastError();
}

cudaError_t launch_transpose_trials(const void* src, long long sps, int Tp, void* dst, long long dps, int Rp, int B,
                                    int R, int N, int T, int split, int* maskcount_dst, cudaStream_t st) {
  const long long blocks = (long long)B * N * ((T + kTrTile - 1) / kTrTile);
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned g = (unsigned)blocks;
  if (split)
    transpose_trials_kernel<__half, 4><<<g, kTrTile * 8, 0, st>>>(static_cast<const __half*>(src), sps, Tp,
                                                                  static_cast<__half*>(dst), dps, Rp, B, R, N, T,
                                                                  maskcount_dst);
  else
    transpose_trials_kernel<double, 2><<<g, kTrTile * 8, 0, st>>>(static_cast<const double*>(src), sps, Tp,
                                                                  static_cast<double*>(dst), dps, Rp, B, R, N, T,
                                                                  maskcount_dst);
  return cudaGetLastError();
}

// K7 operand: u(t) = 1 where a sample is unmasked (masked samples are exactly
// 0 in every plane; an unmasked unit phasor never has both hi parts 0), 0 where
// masked or in the row padding -- as E4M3 bytes (1.0 = 0x38).  One thread per
// 16-sample chunk, 16-byte store.
__device__ __forceinline__ bool is_zero_el(__half v) { return __half2float(v) == 0.0f; }
__device__ __forceinline__ bool is_zero_el(double v) { return v == 0.0; }

template <typename E, int IM_PLANE>
__global__ void indicator_plane_kernel(const E* __restrict__ planes, long long ps, long long rows, int Tp, int T,
                                       uint8_t* __restrict__ ind, int ip) {
  const long long cpr = ip / 16;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cpr;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cpr;
    const int t0 = (int)(e % cpr) * 16;
    __align__(16) uint8_t v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int t = t0 + k;
      bool u = false;
      if (t < T) {
        const long long idx = r * Tp + t;
        u = !(is_zero_el(planes[idx]) && is_zero_el(planes[IM_PLANE * ps + idx]));
      }
      v[k] = u ? 0x38 : 0x00;  // E4M3 1.0 / 0.0
    }
    *reinterpret_cast<uint4*>(ind + r * ip + t0) = *reinterpret_cast<const uint4*>(v);
  }
}

cudaError_t launch_indicator_plane(const void* planes, long long plane_stride, int split, long long rows, int Tp,
                                   int T, void* ind, int ind_pitch, cudaStream_t st) {
  const int g = grid_for(rows * (ind_pitch / 16), 256);
  if (split)
    indicator_plane_kernel<__half, 2><<<g, 256, 0, st>>>((const __half*)planes, plane_stride, rows, Tp, T,
                                                          (uint8_t*)ind, ind_pitch);
  else
    indicator_plane_kernel<double, 1><<<g, 256, 0, st>>>((const double*)planes, plane_stride, rows, Tp, T,
                                                          (uint8_t*)ind, ind_pitch);
  return cudaGetLastError();
}

// Full layout from upper-triangle slots: one 32 x 32 tile (I <= J) per block;
// the block sums its upper entries over the G slots (coalesced rows), writes
// them, and writes the mirror tile (J, I) from shared memory so those stores
// are coalesced too.  Sum order per entry as group_reduce_kernel (g = 0 ..
// G-1), so both triangles equal what mirrored slots would give.
template <typename S>
__global__ void __launch_bounds__(256) group_reduce_sym_kernel(const S* __restrict__ ws, int G, int N, int nt, int R,
                                                               S* __restrict__ out, bool anti) {
  __shared__ S tile[32][33];
  // blockIdx.x -> (I, J), I <= J, row-major over the upper tile triangle
  int t = blockIdx.x, I = 0;
  while (t >= nt - I) {
    t -= nt - I;
    ++I;
  }
  const int J = I + t;
  const long long nn = (long long)N * N;
  const S* wb = ws + (long long)blockIdx.y * G * nn;
  S* ob = out + (long long)blockIdx.y * nn;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int j = J * 32 + tx;
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = ty + 8 * rr, i = I * 32 + r;
    if (i < N && j < N && (I < J || r <= tx)) {
      const S* p = wb + (long long)i * N + j;
      S acc = p[0];
      for (int g = 1; g < G; ++g) acc += p[g * nn];
      acc = sizeof(S) == 4 ? (acc == S(R) ? S(1) : acc * (S(1) / S(R))) : acc / S(R);  // = epilogue.cuh mean_scale
      ob[(long long)i * N + j] = acc;
      tile[r][tx] = acc;
    }
  }
  __syncthreads();
  const int ii = I * 32 + tx;  // output column of the mirror tile
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = ty + 8 * rr, jj = J * 32 + r;  // output row
    if (jj < N && ii < N && (I < J || tx < r)) {
      const S v = tile[tx][r];
      ob[(long long)jj * N + ii] = anti ? -v : v;
    }
  }
}

// The same for fp32 with N % 4 == 0: one row of the tile per thread group of
// 8, 16-byte loads of the G slots and 16-byte stores of both triangles (a
// quarter of the memory instructions; same sums in the same order).
__global__ void __launch_bounds__(256) group_reduce_sym4_kernel(const float* __restrict__ ws, int G, int N, int nt,
                                                                int R, float* __restrict__ out, bool anti) {
  __shared__ float tile[32][33];
  int t = blockIdx.x, I = 0;
  while (t >= nt - I) {
    t -= nt - I;
    ++I;
  }
  const int J = I + t;
  const long long nn = (long long)N * N;
  const float* wb = ws + (long long)blockIdx.y * G * nn;
  float* ob = out + (long long)blockIdx.y * nn;
  const int c4 = (threadIdx.x & 7) * 4, r = threadIdx.x >> 3;  // 4 columns of row r
  {
    const int i = I * 32 + r, j = J * 32 + c4;
    // a diagonal tile keeps column c of row r when r <= c: the float4 is
    // loaded whole when any of its columns is kept (the slots hold finite
    // values or zeros below the diagonal) and masked on the way out
    if (i < N && j < N && (I < J || r <= c4 + 3)) {
      const float4* p = reinterpret_cast<const float4*>(wb + (long long)i * N + j);
      const long long step = nn / 4;
      float4 acc = __ldg(p);
      for (int g = 1; g < G; ++g) {
        const float4 v = __ldg(p + g * step);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      const float rR = 1.0f / (float)R, fR = (float)R;  // = epilogue.cuh mean_scale
      acc.x = acc.x == fR ? 1.0f : acc.x * rR;
      acc.y = acc.y == fR ? 1.0f : acc.y * rR;
      acc.z = acc.z == fR ? 1.0f : acc.z * rR;
      acc.w = acc.w == fR ? 1.0f : acc.w * rR;
      tile[r][c4 + 0] = acc.x;
      tile[r][c4 + 1] = acc.y;
      tile[r][c4 + 2] = acc.z;
      tile[r][c4 + 3] = acc.w;
      float* o = ob + (long long)i * N + j;
      if (I < J || r <= c4) {
        *reinterpret_cast<float4*>(o) = acc;  // (N % 4 == 0: j + 3 < N)
      } else {  // the diagonal crosses this float4: keep columns >= r
        if (r <= c4 + 1) o[1] = acc.y;
        if (r <= c4 + 2) o[2] = acc.z;
        o[3] = acc.w;
      }
    }
  }
  __syncthreads();
  {
    // mirror tile (J, I): output row jj = J*32 + r, columns ii = I*32 + c4 ..
    const int jj = J * 32 + r, ii = I * 32 + c4;
    if (jj < N && ii < N && (I < J || c4 < r)) {
      float4 v = make_float4(tile[c4][r], tile[c4 + 1][r], tile[c4 + 2][r], tile[c4 + 3][r]);
      if (anti) v = make_float4(-v.x, -v.y, -v.z, -v.w);
      float* o = ob + (long long)jj * N + ii;
      if (I < J || c4 + 3 < r) {
        *reinterpret_cast<float4*>(o) = v;
      } else {  // diagonal tile: keep columns < r
        o[0] = v.x;
        if (c4 + 1 < r) o[1] = v.y;
        if (c4 + 2 < r) o[2] = v.z;
      }
    }
  }
}

cudaError_t launch_group_reduce(const void* ws, int G, int N, int B, int n_outputs, void* const* outs, int R,
                                int is_double, cudaStream_t st, int upper) {
  // ws holds n_outputs consecutive blocks of [B][G][N*N]
  const long long nn = (long long)N * N;
  const long long elems = (long long)B * nn;
  const long long ws_block = elems * G;
  const int nt = (N + 31) / 32;
  const long long tiles = (long long)nt * (nt + 1) / 2;
  if (!upper && (tiles > 0x7fffffffLL || B > 65535)) return cudaErrorInvalidValue;
  for (int m = 0; m < n_outputs; ++m) {
    if (!outs[m]) continue;
    if (upper) {
      const int g = grid_for(elems, 256);
      if (is_double)
        group_reduce_kernel<double><<<g, 256, 0, st>>>((const double*)ws + m * ws_block, G, nn, elems, R,
                                                        (double*)outs[m], N);
      else
        group_reduce_kernel<float><<<g, 256, 0, st>>>((const float*)ws + m * ws_block, G, nn, elems, R,
                                                       (float*)outs[m], N);
    } else {
      const dim3 grid((unsigned)tiles, (unsigned)B), block(32, 8);
      if (is_double)
        group_reduce_sym_kernel<double><<<grid, block, 0, st>>>((const double*)ws + m * ws_block, G, N, nt, R,
                                                                 (double*)outs[m], m == 4);
      else if (N % 4 == 0 && (reinterpret_cast<uintptr_t>(ws) & 15u) == 0 &&
               (reinterpret_cast<uintptr_t>(outs[m]) & 15u) == 0)
        group_reduce_sym4_kernel<<<grid, 256, 0, st>>>((const float*)ws + m * ws_block, G, N, nt, R,
                                                       (float*)outs[m], m == 4);
      else
        group_reduce_sym_kernel<float><<<grid, block, 0, st>>>((const float*)ws + m * ws_block, G, N, nt, R,
                                                                (float*)outs[m], m == 4);
    }
  }
  return cudaGetLastError();
}

}  // namespace ps
