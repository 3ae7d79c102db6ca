// K5: upper-triangle Hermitian Gram on the 5th-gen tensor cores (tcgen05 +
// TMEM + TMA), split precision fp16 x 3, with the fused PLV-family epilogue.
//
// Replaces the per-trial complex product of Appendix impl 3
// (`ndat(:,:,t) * ndat(:,:,t)'`) and SPEC plv_matrix /
// iplv / ciplv.  Z = Zr + i Zi is held as four fp16 planes
// (hi/lo of Re and Im, z = hi + lo to ~2^-24).  Per K-step of 16 samples the
// single MMA-issuing thread launches 12 UMMAs (M=128, N=256, K=16):
//   Re += Rh.Rh' + Rh.Rl' + Rl.Rh' + Ih.Ih' + Ih.Il' + Il.Ih'
//   Im += Ih.Rh' + Ih.Rl' + Il.Rh' - Rh.Ih' - Rh.Il' - Rl.Ih'
// (negation through the instruction descriptor's negate-A bit; the lo*lo
// terms, <= 2^-24, are dropped).  Re and Im accumulate in fp32 in TMEM
// (2 x 256 columns = all 512).  Only tiles touching the upper triangle are
// computed; each pair (i <= j) is emitted by exactly one tile.
//
// Warp roles (192 threads, one CTA per SM, persistent over work items):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue: tcgen05.ld -> metrics -> global stores
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "epilogue.cuh"
#include "ps_internal.h"
#include "ptx.cuh"

namespace ps {
namespace {

constexpr int BM = kSplitBM;   // 128 rows of panel I  (UMMA M)
constexpr int BN = kSplitBN;   // 256 rows of panel J  (UMMA N)
constexpr int BK = kSplitBK;   // 32 samples per pipeline stage
constexpr int STAGES = 2;
constexpr int A_PLANE = BM * BK * 2;
constexpr int B_PLANE = BN * BK * 2;
constexpr int A_BYTES = 4 * A_PLANE;
constexpr int B_BYTES = 4 * B_PLANE;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t SWZ = (BK == 16) ? 6u : (BK == 32) ? 4u : 2u;  // 32B / 64B / 128B swizzle
constexpr uint32_t SBO = 8u * BK * 2u;                             // bytes per 8-row core group
constexpr int NTHREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;

static_assert(2 * BN <= (int)TMEM_COLS, "Re + Im accumulators must fit TMEM");
static_assert(BK % 16 == 0 && BK * 2 <= 128, "BK must be a multiple of 16 within one swizzle row");

__global__ void __launch_bounds__(NTHREADS, 1)
    gram_split_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GramParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* tflag = &p.status->flags;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, 128);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    ptx::tmem_alloc(tslot, TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;

  const int nk = (p.T + BK - 1) / BK;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const Item w = p.items[it];
        const int r0 = p.pool ? 0 : w.g * p.Rg;
        const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
        for (int r = r0; r < r1; ++r) {
          const int u = w.b * p.R + r;
          for (int kb = 0; kb < nk; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1u, tflag);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            ptx::tma_load_4d(sa, &tmA, &full[stage], kb * BK, w.I * BM, u, 0);
            ptx::tma_load_4d(sa + A_BYTES, &tmB, &full[stage], kb * BK, w.J * BN, u, 0);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc_pos = ptx::make_idesc_f16(BM, BN, false);
      constexpr uint32_t idesc_neg = ptx::make_idesc_f16(BM, BN, true);
      const uint32_t d_re = tmem;
      const uint32_t d_im = tmem + BN;
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const Item w = p.items[it];
        const int r0 = p.pool ? 0 : w.g * p.Rg;
        const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
        for (int r = r0; r < r1; ++r) {
          const bool start_acc = !p.pool || r == r0;
          if (start_acc) {
            ptx::mbar_wait(tempty, acc_phase ^ 1u, tflag);
            ptx::tc_fence_after();
          }
          for (int kb = 0; kb < nk; ++kb) {
            ptx::mbar_wait(&full[stage], phase, tflag);
            ptx::tc_fence_after();
            const uint32_t sa = ptx::smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks) {
              const uint32_t ko = ks * 32;  // 16 fp16 = 32 bytes along K inside the swizzle row
              const uint64_t aRh = ptx::make_smem_desc(sa + 0 * A_PLANE + ko, SBO, SWZ);
              const uint64_t aRl = ptx::make_smem_desc(sa + 1 * A_PLANE + ko, SBO, SWZ);
              const uint64_t aIh = ptx::make_smem_desc(sa + 2 * A_PLANE + ko, SBO, SWZ);
              const uint64_t aIl = ptx::make_smem_desc(sa + 3 * A_PLANE + ko, SBO, SWZ);
              const uint64_t bRh = ptx::make_smem_desc(sb + 0 * B_PLANE + ko, SBO, SWZ);
              const uint64_t bRl = ptx::make_smem_desc(sb + 1 * B_PLANE + ko, SBO, SWZ);
              const uint64_t bIh = ptx::make_smem_desc(sb + 2 * B_PLANE + ko, SBO, SWZ);
              const uint64_t bIl = ptx::make_smem_desc(sb + 3 * B_PLANE + ko, SBO, SWZ);
              const uint32_t acc0 = (start_acc && kb == 0 && ks == 0) ? 0u : 1u;
              // Re = Zr Zr' + Zi Zi'
              ptx::mma_f16_ss(d_re, aRh, bRh, idesc_pos, acc0);
              ptx::mma_f16_ss(d_re, aRh, bRl, idesc_pos, 1u);
              ptx::mma_f16_ss(d_re, aRl, bRh, idesc_pos, 1u);
              ptx::mma_f16_ss(d_re, aIh, bIh, idesc_pos, 1u);
              ptx::mma_f16_ss(d_re, aIh, bIl, idesc_pos, 1u);
              ptx::mma_f16_ss(d_re, aIl, bIh, idesc_pos, 1u);
              // Im = Zi Zr' - Zr Zi'
              ptx::mma_f16_ss(d_im, aIh, bRh, idesc_pos, acc0);
              ptx::mma_f16_ss(d_im, aIh, bRl, idesc_pos, 1u);
              ptx::mma_f16_ss(d_im, aIl, bRh, idesc_pos, 1u);
              ptx::mma_f16_ss(d_im, aRh, bIh, idesc_neg, 1u);
              ptx::mma_f16_ss(d_im, aRh, bIl, idesc_neg, 1u);
              ptx::mma_f16_ss(d_im, aRl, bIh, idesc_neg, 1u);
            }
            ptx::mma_commit(&empty[stage]);  // smem slot free once these MMAs retire
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          const bool end_acc = !p.pool || r == r1 - 1;
          if (end_acc) {
            ptx::mma_commit(tfull);  // accumulators complete -> epilogue
            acc_phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int il = q * 32 + lane;
    uint32_t acc_phase = 0;
    const bool any_masked = (p.status->flags & FLAG_ANY_MASKED) != 0;
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item w = p.items[it];
      const int r0 = p.pool ? 0 : w.g * p.Rg;
      const int r1 = p.pool ? p.R : min(p.R, r0 + p.Rg);
      for (int r = r0; r < r1; ++r) {
        if (p.pool && r != r1 - 1) continue;
        const RoundInfo ri = round_info(p, w, r, r0, r1);
        ptx::mbar_wait(tfull, acc_phase, tflag);
        ptx::tc_fence_after();
        const int i = w.I * BM + il;
        const long long Tobs = (long long)p.T * ri.nu;
        const float inv_t = 1.0f / static_cast<float>(Tobs);
        unsigned illc = 0;
        for (int c = 0; c < BN; c += 32) {
          uint32_t vre[32], vim[32];
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c;
          ptx::tmem_ld_32x32b_x32(ta, vre);
          ptx::tmem_ld_32x32b_x32(ta + BN, vim);
          ptx::tmem_wait_ld();
          if (i < p.N) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int j = w.J * BN + c + k;
              if (j >= p.N || j < i) continue;
              PairMetrics<float> m;
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
                m = pair_metrics<float, true>(__uint_as_float(vre[k]), __uint_as_float(vim[k]), it_);
                const float are = fabsf(m.cre);
                const float d = (1.0f - are) * (1.0f + are);
                // predicted ciPLV error from an fp32-accumulation error of
                // ~4e-7 in Re: |Im| |Re| / d^1.5 * 4e-7
                if (d > 0.0f && fabsf(m.cim) * are * 4e-7f > p.illcond_tol * d * sqrtf(d)) ++illc;
              }
              emit_all<float>(p, ri.slot, i, j, m, ri.first, ri.last);
            }
          }
        }
        if (illc) atomicAdd(&p.status->n_illcond, (unsigned long long)illc);
        ptx::tc_fence_before();
        ptx::mbar_arrive(tempty);
        acc_phase ^= 1u;
      }
    }
  }

  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace

cudaError_t launch_gram_split(const void* tmapA, const void* tmapB, const GramParams& p, int grid,
                              cudaStream_t st) {
  cudaError_t e =
      cudaFuncSetAttribute(gram_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (p.n_items <= 0) return cudaSuccess;
  gram_split_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(*static_cast<const CUtensorMap*>(tmapA),
                                                          *static_cast<const CUtensorMap*>(tmapB), p);
  return cudaGetLastError();
}

}  // namespace ps
