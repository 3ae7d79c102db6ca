// Exact FP64 recomputation of ill-conditioned ciPLV pairs of the split path.
//
// ciPLV = |Im| / sqrt(1 - Re^2) (Eq 14) amplifies an error e in
// Re by |Im||Re| / (1 - Re^2)^1.5: for strongly zero-lag-coupled pairs
// (volume conduction, config C2) a 1e-6 Gram error becomes > 1e-5.  The split
// Gram epilogue queues such pairs; this kernel recomputes G_ij for them in
// double precision straight from the fp16 hi/lo planes (z = hi + lo to
// 2^-24 per sample; the average over T samples brings that to ~1e-9) and
// corrects the emitted ciPLV.  One warp per output location; entries of one
// location are processed in trial order and the warp reduction order is fixed,
// so the result is deterministic.
#include <cuda_fp16.h>

#include "epilogue.cuh"
#include "ps_internal.h"

namespace ps {
namespace {

__global__ void refine_kernel(const GramParams p, const RefineEntry* __restrict__ e, const int* __restrict__ groups,
                              int n_groups, int overwrite, int div) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_groups) return;
  const __half* pl = static_cast<const __half*>(p.planes);
  const long long ps = p.plane_stride;
  double corr = 0.0, exact_last = 0.0;
  const RefineEntry& e0 = e[groups[warp]];
  for (int k = groups[warp]; k < groups[warp + 1]; ++k) {
    const RefineEntry en = e[k];
    double gre = 0.0, gim = 0.0;
    for (int u = en.u0; u < en.u0 + en.nu; ++u) {
      const long long ri = ((long long)u * p.N + en.i) * p.Tp;
      const long long rj = ((long long)u * p.N + en.j) * p.Tp;
      for (int t = lane; t < p.T; t += 32) {
        const double ar = (double)__half2float(pl[ri + t]) + (double)__half2float(pl[ps + ri + t]);
        const double ai = (double)__half2float(pl[2 * ps + ri + t]) + (double)__half2float(pl[3 * ps + ri + t]);
        const double br = (double)__half2float(pl[rj + t]) + (double)__half2float(pl[ps + rj + t]);
        const double bi = (double)__half2float(pl[2 * ps + rj + t]) + (double)__half2float(pl[3 * ps + rj + t]);
        gre += ar * br + ai * bi;
        gim += ai * br - ar * bi;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      gre += __shfl_xor_sync(0xffffffffu, gre, o);
      gim += __shfl_xor_sync(0xffffffffu, gim, o);
    }
    long long te = (long long)p.T * en.nu;
    if (p.status->flags & FLAG_ANY_MASKED) te = effective_T<true>(p, en.u0, en.nu, en.i, en.j);
    const double inv = te > 0 ? 1.0 / (double)te : 0.0;
    const PairMetrics<double> m = pair_metrics<double, false>(gre, gim, inv);
    double ci = m.ciplv > 1.0 ? 1.0 : m.ciplv;
    exact_last = ci;
    corr += ci - (double)en.approx;
  }
  if (lane == 0 && p.out_ciplv) {
    float* o = static_cast<float*>(p.out_ciplv) + (long long)e0.slot * p.N * p.N;
    const long long a = (long long)e0.i * p.N + e0.j, b = (long long)e0.j * p.N + e0.i;
    float v;
    if (overwrite) v = (float)exact_last;
    else v = (float)((double)o[a] + corr / (double)div);
    o[a] = v;
    o[b] = v;
  }
}

}  // namespace

cudaError_t launch_refine(const GramParams& p, const RefineEntry* entries, const int* groups, int n_groups,
                          int overwrite, int div, cudaStream_t st) {
  if (n_groups <= 0) return cudaSuccess;
  const int threads = 256;
  const int blocks = (n_groups * 32 + threads - 1) / threads;
  refine_kernel<<<blocks, threads, 0, st>>>(p, entries, groups, n_groups, overwrite, div);
  return cudaGetLastError();
}

}  // namespace ps
