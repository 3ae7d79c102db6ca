// Exact FP64 recomputation of ill-conditioned ciPLV pairs of the split path.
//
// ciPLV = |Im| / sqrt(1 - Re^2) (Eq 14) amplifies an error e in
// Re by |Im||Re| / (1 - Re^2)^1.5: for strongly zero-lag-coupled pairs
// (volume conduction, config C2) a 1e-6 Gram error becomes > 1e-5.  The split
// Gram epilogue queues such pairs; these kernels recompute G_ij for them in
// double precision straight from the fp16 hi/lo planes (z = hi + lo to
// 2^-24 per sample; the average over T samples brings that to ~1e-9) and
// correct the emitted ciPLV.
//   refine_exact_kernel: one warp per queued (pair, round); 16-byte plane
//     loads, fixed-order warp reduction.
//   refine_apply_kernel: one thread per output location; the host sorted the
//     queue, so corrections are summed in trial order (deterministic).
#include <cuda_fp16.h>

#include "epilogue.cuh"
#include "ps_internal.h"

namespace ps {
namespace {

__device__ __forceinline__ void h8(const uint4& v, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = __half22float2(h[k]);
    f[2 * k] = x.x;
    f[2 * k + 1] = x.y;
  }
}

__global__ void refine_exact_kernel(const GramParams p, const RefineEntry* __restrict__ e, int n,
                                    double* __restrict__ exact) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const RefineEntry en = e[w];
  const __half* pl = static_cast<const __half*>(p.planes);
  const long long ps = p.plane_stride;
  double gre = 0.0, gim = 0.0;
  for (int u = en.u0; u < en.u0 + en.nu; ++u) {
    const long long ri = ((long long)u * p.N + en.i) * p.Tp;
    const long long rj = ((long long)u * p.N + en.j) * p.Tp;
    // Tp is a multiple of 8 and the pitch padding is zero: whole 8-sample
    // chunks up to Tp are safe to read and contribute nothing past T
    for (int t = lane * 8; t < p.Tp; t += 256) {
      float arh[8], arl[8], aih[8], ail[8], brh[8], brl[8], bih[8], bil[8];
      h8(*reinterpret_cast<const uint4*>(pl + ri + t), arh);
      h8(*reinterpret_cast<const uint4*>(pl + ps + ri + t), arl);
      h8(*reinterpret_cast<const uint4*>(pl + 2 * ps + ri + t), aih);
      h8(*reinterpret_cast<const uint4*>(pl + 3 * ps + ri + t), ail);
      h8(*reinterpret_cast<const uint4*>(pl + rj + t), brh);
      h8(*reinterpret_cast<const uint4*>(pl + ps + rj + t), brl);
      h8(*reinterpret_cast<const uint4*>(pl + 2 * ps + rj + t), bih);
      h8(*reinterpret_cast<const uint4*>(pl + 3 * ps + rj + t), bil);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double ar = (double)arh[k] + (double)arl[k], ai = (double)aih[k] + (double)ail[k];
        const double br = (double)brh[k] + (double)brl[k], bi = (double)bih[k] + (double)bil[k];
        gre += ar * br + ai * bi;
        gim += ai * br - ar * bi;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    gre += __shfl_xor_sync(0xffffffffu, gre, o);
    gim += __shfl_xor_sync(0xffffffffu, gim, o);
  }
  if (lane == 0) {
    long long te = (long long)p.T * en.nu;
    if (p.status->flags & FLAG_ANY_MASKED) te = effective_T<true>(p, en.u0, en.nu, en.i, en.j);
    const double inv = te > 0 ? 1.0 / (double)te : 0.0;
    const PairMetrics<double> m = pair_metrics<double, false>(gre, gim, inv);
    exact[w] = m.ciplv > 1.0 ? 1.0 : m.ciplv;
  }
}

__global__ void refine_apply_kernel(const GramParams p, const RefineEntry* __restrict__ e,
                                    const double* __restrict__ exact, const int* __restrict__ groups, int n_groups,
                                    int overwrite, int div) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups || !p.out_ciplv) return;
  const int k0 = groups[g], k1 = groups[g + 1];
  double corr = 0.0, sum = 0.0;
  for (int k = k0; k < k1; ++k) {
    corr += exact[k] - (double)e[k].approx;
    sum += exact[k];
  }
  const RefineEntry& e0 = e[k0];
  float* o = static_cast<float*>(p.out_ciplv) + (long long)e0.slot * p.N * p.N;
  const long long a = (long long)e0.i * p.N + e0.j, b = (long long)e0.j * p.N + e0.i;
  // every round of the slot refined: take the exact mean outright (keeps
  // exact zeros of the singularity rule exact); otherwise correct the mean
  const float v = overwrite ? (float)exact[k1 - 1]
                  : (k1 - k0 == div) ? (float)(sum / (double)div)
                                     : (float)((double)o[a] + corr / (double)div);
  o[a] = v;
  o[b] = v;
}

}  // namespace

cudaError_t launch_refine(const GramParams& p, const RefineEntry* entries, const int* groups, int n_groups,
                          int n_entries, double* exact, int overwrite, int div, cudaStream_t st) {
  if (n_groups <= 0) return cudaSuccess;
  const int threads = 256;
  refine_exact_kernel<<<(n_entries * 32 + threads - 1) / threads, threads, 0, st>>>(p, entries, n_entries, exact);
  refine_apply_kernel<<<(n_groups + threads - 1) / threads, threads, 0, st>>>(p, entries, exact, groups, n_groups,
                                                                              overwrite, div);
  return cudaGetLastError();
}

}  // namespace ps
