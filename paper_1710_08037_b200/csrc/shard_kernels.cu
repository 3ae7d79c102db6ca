// Multi-GPU combine / gather kernels.
//
//  * reduce_partials: the fixed-order combination of the per-rank partial
//    metric sums of a (band, trial)-sharded call (PS_TRIALS_SUM)
//    ("deterministic tree order"): out = (p_0 + p_1 + ... + p_{P-1}) / div,
//    summed left to right, so the result is bit-identical run to run and
//    independent of the collective's internal order.
//  * shard_pack / shard_unpack: move the upper-triangle output tiles one
//    shard owns between a [N][N] matrix and a dense packed buffer, so the
//    optional gather is an all-gather of owned tiles (1/P of the output per
//    rank) instead of an all-reduce of zero-filled dense matrices.
#include <cuda_runtime.h>

#include <cstdint>

#include "ps_internal.h"

namespace ps {
namespace {

template <typename S>
__global__ void reduce_partials_kernel(const S* __restrict__ parts, int P, long long stride, long long n, S div,
                                       S* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    S acc = parts[e];
    for (int p = 1; p < P; ++p) acc += parts[p * stride + e];
    out[e] = acc / div;
  }
}

// 16-byte lanes (4 floats / 2 doubles) when every part and the output are aligned
template <typename S, typename V>
__global__ void reduce_partials_vec_kernel(const V* __restrict__ parts, int P, long long vstride, long long nv, S div,
                                           V* __restrict__ out) {
  constexpr int L = sizeof(V) / sizeof(S);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nv; e += (long long)gridDim.x * blockDim.x) {
    V a = parts[e];
    S* pa = reinterpret_cast<S*>(&a);
    for (int p = 1; p < P; ++p) {
      V b = parts[p * vstride + e];
      const S* pb = reinterpret_cast<const S*>(&b);
#pragma unroll
      for (int k = 0; k < L; ++k) pa[k] += pb[k];
    }
#pragma unroll
    for (int k = 0; k < L; ++k) pa[k] = pa[k] / div;
    out[e] = a;
  }
}

// one block per packed tile; threads run along the tile's columns (coalesced
// rows of the matrix); entries outside the matrix are packed as 0
template <typename S>
__global__ void shard_pack_kernel(const S* __restrict__ M, long long N, const int2* __restrict__ tiles, int bm, int bn,
                                  S* __restrict__ packed) {
  const int2 t = tiles[blockIdx.x];
  S* dst = packed + (long long)blockIdx.x * bm * bn;
  const long long i0 = (long long)t.x * bm, j0 = (long long)t.y * bn;
  for (int e = threadIdx.x; e < bm * bn; e += blockDim.x) {
    const int r = e / bn, c = e % bn;
    const long long i = i0 + r, j = j0 + c;
    dst[e] = (i < N && j < N) ? M[i * N + j] : S(0);
  }
}

// owned entries (i <= j, inside the matrix) of a packed tile -> M, plus the
// mirror (j, i) when mirror != 0 (negated when mirror < 0)
template <typename S>
__global__ void shard_unpack_kernel(const S* __restrict__ packed, long long N, const int2* __restrict__ tiles, int bm,
                                    int bn, S* __restrict__ M, int mirror) {
  const int2 t = tiles[blockIdx.x];
  const S* src = packed + (long long)blockIdx.x * bm * bn;
  const long long i0 = (long long)t.x * bm, j0 = (long long)t.y * bn;
  for (int e = threadIdx.x; e < bm * bn; e += blockDim.x) {
    const int r = e / bn, c = e % bn;
    const long long i = i0 + r, j = j0 + c;
    if (i >= N || j >= N || i > j) continue;
    const S v = src[e];
    M[i * N + j] = v;
    if (mirror && i != j) M[j * N + i] = mirror < 0 ? -v : v;
  }
}

int grid_cap(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148LL * 32) g = 148LL * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_reduce_partials(const void* parts, int P, long long stride, long long n, double div, int is_double,
                                   void* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int L = is_double ? 2 : 4;
  const bool vec = (n % L) == 0 && (stride % L) == 0 && ((uintptr_t)parts % 16) == 0 && ((uintptr_t)out % 16) == 0;
  if (vec) {
    const int g = grid_cap(n / L, 256);
    if (is_double)
      reduce_partials_vec_kernel<double, double2><<<g, 256, 0, st>>>((const double2*)parts, P, stride / L, n / L,
                                                                      div, (double2*)out);
    else
      reduce_partials_vec_kernel<float, float4><<<g, 256, 0, st>>>((const float4*)parts, P, stride / L, n / L,
                                                                    (float)div, (float4*)out);
  } else {
    const int g = grid_cap(n, 256);
    if (is_double)
      reduce_partials_kernel<double><<<g, 256, 0, st>>>((const double*)parts, P, stride, n, div, (double*)out);
    else
      reduce_partials_kernel<float><<<g, 256, 0, st>>>((const float*)parts, P, stride, n, (float)div, (float*)out);
  }
  return cudaGetLastError();
}

cudaError_t launch_shard_pack(const void* M, long long N, const void* tiles, int n_tiles, int bm, int bn, int is_double,
                              void* packed, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  if (is_double)
    shard_pack_kernel<double><<<n_tiles, 256, 0, st>>>((const double*)M, N, (const int2*)tiles, bm, bn,
                                                       (double*)packed);
  else
    shard_pack_kernel<float><<<n_tiles, 256, 0, st>>>((const float*)M, N, (const int2*)tiles, bm, bn, (float*)packed);
  return cudaGetLastError();
}

cudaError_t launch_shard_unpack(const void* packed, long long N, const void* tiles, int n_tiles, int bm, int bn,
                                int is_double, void* M, int mirror, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  if (is_double)
    shard_unpack_kernel<double><<<n_tiles, 256, 0, st>>>((const double*)packed, N, (const int2*)tiles, bm, bn,
                                                         (double*)M, mirror);
  else
    shard_unpack_kernel<float><<<n_tiles, 256, 0, st>>>((const float*)packed, N, (const int2*)tiles, bm, bn,
                                                        (float*)M, mirror);
  return cudaGetLastError();
}

}  // namespace ps
