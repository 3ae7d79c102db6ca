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

#include <algorithm>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

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
    // The planes hold z to 2^-24 per component, so even this FP64 sum carries
    // ~3 * 2^-24 * sqrt(2 / T) in Re and Im (rounding errors averaged over T).
    // ciPLV amplifies an error e in Re by ciPLV |Re| / (1 - Re^2) and one in Im
    // by 1 / sqrt(1 - Re^2): when that exceeds the 1e-5 budget the value is
    // indeterminate in split precision -- counted, so the caller is told to
    // use fp64 (ps_plv_result.n_indeterminate_ciplv)
    const double are = fabs(m.cre), d = 1.0 - m.cre * m.cre;
    const double dz = 3.0 * 5.9604644775390625e-8 * sqrt(2.0 / (double)(te > 0 ? te : 1));
    // (Im exactly 0 from the planes: identical rows, whose plane errors cancel
    // in Im exactly as well -- ciPLV = 0 is exact there)
    const double e_im = m.cim != 0.0 ? dz / sqrt(d > 0.0 ? d : 1.0) : 0.0;
    if (d > 0.0 && m.ciplv * are * dz / d + e_im > 1e-5) atomicAdd(&p.status->n_indeterminate, 1ull);
  }
}

__global__ void refine_apply_kernel(const GramParams p, const RefineEntry* __restrict__ e,
                                    const double* __restrict__ exact, const int* __restrict__ groups, int n_groups,
                                    const int* __restrict__ d_n_groups, int overwrite, int div) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_n_groups) n_groups = *d_n_groups;
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
  // exact zeros of the singularity rule exact); otherwise correct the mean.
  // div = R rounds per slot (trial mean: / R); div = -R: trial SUM (no division)
  const int nr = div < 0 ? -div : div;
  const double dv = div < 0 ? 1.0 : (double)div;
  const float v = overwrite ? (float)exact[k1 - 1]
                  : (k1 - k0 == nr) ? (float)(sum / dv)
                                    : (float)((double)o[a] + corr / dv);
  o[a] = v;
  if (!p.upper_only) o[b] = v;
}

// ---- device-side ordering of the refinement queue ---------------------------
// Entries arrive in atomicAdd order; corrections must be applied per output
// location in trial order (deterministic).  Sort on the device: a stable LSD
// radix sort by u0, then by the packed (slot, i, j) key, then group starts by
// flagging key changes -- no host round trip (the host sort dominated calls
// with ~1e5-1e6 leakage-coupled pairs).
__global__ void refine_keys_kernel(RefineEntry* __restrict__ e, int n, int slot_div, uint32_t* __restrict__ ku0,
                                   int* __restrict__ idx) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  RefineEntry en = e[q];
  if (slot_div > 1) {
    en.slot /= slot_div;  // workspace slot b*G+g -> final output slot b
    e[q].slot = en.slot;
  }
  ku0[q] = (uint32_t)en.u0;
  idx[q] = q;
}

__device__ __forceinline__ unsigned long long pos_key(const RefineEntry& en, int ib) {
  return ((unsigned long long)en.slot << (2 * ib)) | ((unsigned long long)en.i << ib) | (unsigned long long)en.j;
}

__global__ void refine_poskey_kernel(const RefineEntry* __restrict__ e, const int* __restrict__ idx1, int n, int ib,
                                     unsigned long long* __restrict__ kpos) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) kpos[q] = pos_key(e[idx1[q]], ib);
}

__global__ void refine_gather_kernel(const RefineEntry* __restrict__ e, const int* __restrict__ idx2,
                                     const unsigned long long* __restrict__ kpos2, int n,
                                     RefineEntry* __restrict__ sorted, uint8_t* __restrict__ flags) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  sorted[q] = e[idx2[q]];
  flags[q] = (q == 0 || kpos2[q] != kpos2[q - 1]) ? 1 : 0;
}

__global__ void refine_terminate_kernel(int* groups, const int* d_n_groups, int n) { groups[*d_n_groups] = n; }

}  // namespace

cudaError_t launch_refine(const GramParams& p, const RefineEntry* entries, const int* groups, int n_groups,
                          int n_entries, double* exact, int overwrite, int div, cudaStream_t st) {
  if (n_groups <= 0) return cudaSuccess;
  const int threads = 256;
  refine_exact_kernel<<<(n_entries * 32 + threads - 1) / threads, threads, 0, st>>>(p, entries, n_entries, exact);
  refine_apply_kernel<<<(n_groups + threads - 1) / threads, threads, 0, st>>>(p, entries, exact, groups, n_groups,
                                                                              nullptr, overwrite, div);
  return cudaGetLastError();
}

size_t refine_sort_ws_bytes(int n) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, n);
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, n);
  cub::DeviceSelect::Flagged(nullptr, c, thrust::counting_iterator<int>(0), (const uint8_t*)nullptr, (int*)nullptr,
                             (int*)nullptr, n);
  const size_t cubb = std::max(a, std::max(b, c));
  // ku0, ku0s (4 n) + idx, idx1, idx2 (4 n) + kpos, kpos2 (8 n) + flags (n) + n_groups + cub
  // (each of the 9 carve-outs is rounded up to 256 bytes)
  return (size_t)n * (4 * 2 + 4 * 3 + 8 * 2 + 1) + 10 * 256 + 256 + cubb;
}

cudaError_t launch_refine_sorted(const GramParams& p, RefineEntry* entries, int n, int slot_div, int ib, int key_bits,
                                 void* ws,
                                 size_t ws_bytes, RefineEntry* sorted, double* exact, int* groups, int overwrite,
                                 int div, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  char* w = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = w;
    w += (bytes + 255) & ~size_t(255);
    return r;
  };
  uint32_t* ku0 = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
  uint32_t* ku0s = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
  int* idx = reinterpret_cast<int*>(take((size_t)n * 4));
  int* idx1 = reinterpret_cast<int*>(take((size_t)n * 4));
  int* idx2 = reinterpret_cast<int*>(take((size_t)n * 4));
  unsigned long long* kpos = reinterpret_cast<unsigned long long*>(take((size_t)n * 8));
  unsigned long long* kpos2 = reinterpret_cast<unsigned long long*>(take((size_t)n * 8));
  uint8_t* flags = reinterpret_cast<uint8_t*>(take((size_t)n));
  int* d_ng = reinterpret_cast<int*>(take(64));
  const size_t used = (size_t)(w - static_cast<char*>(ws));
  if (used > ws_bytes) return cudaErrorInvalidValue;
  size_t cub_bytes = ws_bytes - used;
  void* cub_ws = w;
  const int threads = 256, blocks = (n + threads - 1) / threads;
  refine_keys_kernel<<<blocks, threads, 0, st>>>(entries, n, slot_div, ku0, idx);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, ku0, ku0s, idx, idx1, n, 0, 32, st);
  if (e != cudaSuccess) return e;
  refine_poskey_kernel<<<blocks, threads, 0, st>>>(entries, idx1, n, ib, kpos);
  cub_bytes = ws_bytes - used;
  // only the bits a (slot, i, j) key can occupy: 8-bit passes saved for small N
  e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, kpos, kpos2, idx1, idx2, n, 0, key_bits, st);
  if (e != cudaSuccess) return e;
  refine_gather_kernel<<<blocks, threads, 0, st>>>(entries, idx2, kpos2, n, sorted, flags);
  cub_bytes = ws_bytes - used;
  e = cub::DeviceSelect::Flagged(cub_ws, cub_bytes, thrust::counting_iterator<int>(0), flags, groups, d_ng, n, st);
  if (e != cudaSuccess) return e;
  refine_terminate_kernel<<<1, 1, 0, st>>>(groups, d_ng, n);
  refine_exact_kernel<<<(n * 32 + threads - 1) / threads, threads, 0, st>>>(p, sorted, n, exact);
  refine_apply_kernel<<<blocks, threads, 0, st>>>(p, sorted, exact, groups, n, d_ng, overwrite, div);
  return cudaGetLastError();
}

// Streamed copy-out of the pipelined host path: the final (refined) ciPLV
// value at every queued entry, packed with its flat output index, so the host
// can patch the blocks it already received without shipping them again.
__global__ void refine_pick_kernel(const RefineEntry* __restrict__ e, int n, const float* __restrict__ out,
                                   long long N, long long* __restrict__ idx, float* __restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const RefineEntry en = e[q];
  const long long at = ((long long)en.slot * N + en.i) * N + en.j;
  idx[q] = at;
  val[q] = out[at];
}

cudaError_t launch_refine_pick(const RefineEntry* entries, int n, const float* out, long long N, long long* idx,
                               float* val, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  refine_pick_kernel<<<(n + 255) / 256, 256, 0, st>>>(entries, n, out, N, idx, val);
  return cudaGetLastError();
}

}  // namespace ps
