// K6: FP64 accuracy mode of the upper-triangle Hermitian Gram + fused
// PLV-family epilogue on the FP64 tensor path (DMMA, mma.sync m8n8k4 f64).
//
// Same contract as gram_tc.cu (Appendix impl 3
// PAPER.md:282-287) with double operands and double accumulation
// ("all phasor sums accumulate in double precision"), target
// parity 1e-12 against the fp64 oracle.
//   CTA tile 64 x 64, 8 warps (2 x 4), warp tile 32 x 16 = 4 x 2 m8n8 tiles,
//   K staged 16 samples at a time in shared memory with cp.async double
//   buffering (rows padded to 20 doubles: conflict-free fragment loads).
#include <algorithm>
#include <cstdint>

#include "epilogue.cuh"
#include "ps_internal.h"

namespace ps {
namespace {

constexpr int BM = kF64BM;
constexpr int BN = kF64BN;
constexpr int BK = 16;
constexpr int LD = BK + 4;  // padded row stride (doubles)
constexpr int NTHREADS = 256;
constexpr int TILE_D = 64 * LD;            // doubles per [64][LD] tile
constexpr int STAGE_D = 4 * TILE_D;        // Are, Aim, Bre, Bim
constexpr int SMEM_BYTES = 2 * STAGE_D * 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Stage one K block (16 samples) of the four operand tiles: 4 x 64 rows x
// 16 doubles = 512 16-byte chunks, two per thread.
__device__ __forceinline__ void load_stage(double* st, const double* planes, long long pstride, int Tp,
                                           long long rowA0, long long rowB0, int nA, int nB, int kb) {
  for (int c = threadIdx.x; c < 4 * 64 * (BK / 2); c += NTHREADS) {
    const int tile = c / (64 * (BK / 2));
    const int rem = c % (64 * (BK / 2));
    const int row = rem / (BK / 2);
    const int col = (rem % (BK / 2)) * 2;
    const bool isA = tile < 2;
    const int plane = tile & 1;  // 0 re, 1 im
    const int nvalid = isA ? nA : nB;
    const long long grow = (isA ? rowA0 : rowB0) + (row < nvalid ? row : 0);
    const double* src = planes + plane * pstride + grow * Tp + (long long)kb * BK + col;
    cp_async16(st + tile * TILE_D + row * LD + col, src, row < nvalid);
  }
}

__global__ void __launch_bounds__(NTHREADS) gram_f64_kernel(const GramParams p) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int gid = lane >> 2, tig = lane & 3;
  const double* planes = static_cast<const double*>(p.planes);
  const int nk = p.Tp / BK;  // Tp is a multiple of 16 for the f64 planes (zero padded)
  const bool any_masked = (p.status->flags & FLAG_ANY_MASKED) != 0;

  for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
    const Item w = p.items[it];
    const int r0 = p.pool ? 0 : w.g * p.Rg;
    const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
    const int I0 = w.I * BM, J0 = w.J * BN;
    const int nA = min(BM, p.N - I0), nB = min(BN, p.N - J0);
    double acc_re[4][2][2], acc_im[4][2][2];
    for (int r = r0; r < r1; ++r) {
      const int u = w.b * p.R + r;
      if (!p.pool || r == r0) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) acc_re[a][b][0] = acc_re[a][b][1] = acc_im[a][b][0] = acc_im[a][b][1] = 0.0;
      }
      const long long rowA0 = (long long)u * p.N + I0, rowB0 = (long long)u * p.N + J0;
      load_stage(sm, planes, p.plane_stride, p.Tp, rowA0, rowB0, nA, nB, 0);
      cp_async_commit();
      for (int kb = 0; kb < nk; ++kb) {
        double* cur = sm + (kb & 1) * STAGE_D;
        if (kb + 1 < nk) {
          load_stage(sm + ((kb + 1) & 1) * STAGE_D, planes, p.plane_stride, p.Tp, rowA0, rowB0, nA, nB, kb + 1);
          cp_async_commit();
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* Are = cur;
        const double* Aim = cur + TILE_D;
        const double* Bre = cur + 2 * TILE_D;
        const double* Bim = cur + 3 * TILE_D;
#pragma unroll
        for (int k4 = 0; k4 < BK / 4; ++k4) {
          const int kk = k4 * 4 + tig;
          double br[2], bi[2];
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int row = wn * 16 + b * 8 + gid;
            br[b] = Bre[row * LD + kk];
            bi[b] = Bim[row * LD + kk];
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int row = wm * 32 + a * 8 + gid;
            const double ar = Are[row * LD + kk];
            const double ai = Aim[row * LD + kk];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              dmma(acc_re[a][b], ar, br[b]);   // Re += Zr Zr'
              dmma(acc_re[a][b], ai, bi[b]);   //    + Zi Zi'
              dmma(acc_im[a][b], ai, br[b]);   // Im += Zi Zr'
              dmma(acc_im[a][b], -ar, bi[b]);  //    - Zr Zi'
            }
          }
        }
        __syncthreads();
      }
      if (p.pool && r != r1 - 1) continue;
      // ---- fused epilogue ----
      const RoundInfo ri = round_info(p, w, r, r0, r1);
      const long long Tobs = (long long)p.T * ri.nu;
      const double inv_t = 1.0 / static_cast<double>(Tobs);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = I0 + wm * 32 + a * 8 + gid;
            const int j = J0 + wn * 16 + b * 8 + 2 * tig + e;
            if (i >= p.N || j >= p.N || j < i) continue;
            PairMetrics<double> m;
            if (i == j) {
              m = diag_metrics<double>();
            } else {
              double it_ = inv_t;
              if (any_masked) {
                const long long te = effective_T<false>(p, ri.u0, ri.nu, i, j);
                if (te <= 0) {
                  atomicOr(&p.status->flags, FLAG_EMPTY_WINDOW);
                  it_ = 0.0;
                } else {
                  it_ = 1.0 / static_cast<double>(te);
                }
              }
              m = pair_metrics<double, false>(acc_re[a][b][e], acc_im[a][b][e], it_);
            }
            emit_all<double>(p, ri.slot, i, j, m, ri.first, ri.last);
          }
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_gram_f64(const GramParams& p, int grid, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(gram_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (p.n_items <= 0) return cudaSuccess;
  // `grid` is one CTA per SM; fill every resident slot (2 CTAs / SM: 80 KB of
  // shared memory each) so the DMMA pipeline has 16 warps per SM to hide
  // its latency
  static int per_sm = 0;
  if (per_sm == 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_f64_kernel, NTHREADS, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    per_sm = per_sm < 1 ? 1 : per_sm;
  }
  const long long g = std::min<long long>((long long)grid * per_sm, p.n_items);
  gram_f64_kernel<<<(unsigned)g, NTHREADS, SMEM_BYTES, st>>>(p);
  return cudaGetLastError();
}

}  // namespace ps
