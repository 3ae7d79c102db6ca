// Thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05 (UMMA / TMEM).
// Descriptor bit layouts follow the PTX ISA "tcgen05 matrix descriptors" and
// "instruction descriptor" tables (cross-checked against the CUTLASS 4.5
// cute/arch/mma_sm100_desc.hpp bitfields shipped in the venv).
#pragma once
#include <cstdint>

namespace ps {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// ---- mbarrier --------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar_addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug must not hang the GPU (gpurun strike rule).
// After ~8 s of spinning the kernel traps (the launch then fails with an
// error the host reports instead of hanging).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int* /*unused*/) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > 16000000000LL) asm volatile("trap;");
  }
}

// mbar_wait that adds the cycles it spent blocked to *acc (profiling builds of
// the pipeline: PS_GRAM_PROF)
__device__ __forceinline__ void mbar_wait_prof(uint64_t* bar, uint32_t parity, long long* acc) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > 16000000000LL) asm volatile("trap;");
  }
  *acc += clock64() - t0;
}

// ---- TMA ------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// L2 prefetch of a TMA box (no shared memory, no barrier): pulls the operand
// slice a later tma_load_4d will read from DRAM into L2 ahead of time
__device__ __forceinline__ void tma_prefetch_4d(const void* tmap, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---- clusters (CTA pairs for cta_group::2) ----------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem object in CTA rank 0 of the pair
// (the peer rank lives in bit 24 of the cluster shared window).
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
__device__ __forceinline__ void mbar_arrive_rank0(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerBitMask) : "memory");
}
// cluster-scope release arrive on rank 0's copy of `bar` (own CTA's when rank 0)
__device__ __forceinline__ void mbar_arrive_rank0_cluster(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerBitMask)
               : "memory");
}
// bounded cluster-scope acquire wait (arrivals from the peer CTA's threads)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  const long long t0 = clock64();
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > 16000000000LL) asm volatile("trap;");
  }
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operands)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 2-CTA TMA: data lands in this CTA's smem, transaction bytes are counted on
// rank 0's mbarrier.
__device__ __forceinline__ void tma_load_4d_cg2(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                                int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---- tcgen05 ----------------------------------------------------------------
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* dst_smem, uint32_t ncols) {
  if (CG == 1)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
  else
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_relinquish_cg() {
  if (CG == 1) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  else asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
  else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_f16_ss_cg(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-collective forms: the whole warp executes the call with warp-uniform
// operands (so they live in uniform registers) and one elected lane issues.
// Issuing from a lone `if (lane == 0)` thread instead makes ptxas re-broadcast
// every descriptor to uniform registers per instruction (R2UR chains), which
// measurably starved the tensor pipe.
template <int CG>
__device__ __forceinline__ void mma_f16_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// One K = 16 step of the 4-product split Gram as a single warp-collective
// block: one elect.sync for all 12 UMMAs; the descriptors are the stage's
// 32-bit start-address words (lo, per plane) paired with the common high
// word in registers (mov.b64), so per UMMA only the MMA itself issues.
//   Re += Rh.Rh' + Rh.Rl' + Rl.Rh' + Ih.Ih' + Ih.Il' + Il.Ih'
//   Im += Ih.Rh' + Ih.Rl' + Il.Rh' - Rh.Ih' - Rh.Il' - Rl.Ih'
// a[0..3] / b[0..3] = {Rh, Rl, Ih, Il} low words; acc = 0 starts both sums.
template <int CG>
__device__ __forceinline__ void mma_4prod_step_warp(uint32_t d_re, uint32_t d_im, const uint32_t (&a)[4],
                                                    const uint32_t (&b)[4], uint32_t hi, uint32_t ipos,
                                                    uint32_t ineg, uint32_t acc) {
#define PS_MMA4(CGS)                                                                                 \
  asm volatile(                                                                                        \
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 ar, al, ai, aj, br, bl, bi, bj;\n\t"                   \
      "elect.sync _|e, 0xffffffff;\n\t"                                                              \
      "setp.ne.b32 p, %13, 0;\n\tsetp.eq.b32 t, %13, %13;\n\t"                                       \
      "mov.b64 ar, {%2, %10};\n\tmov.b64 al, {%3, %10};\n\tmov.b64 ai, {%4, %10};\n\t"             \
      "mov.b64 aj, {%5, %10};\n\tmov.b64 br, {%6, %10};\n\tmov.b64 bl, {%7, %10};\n\t"             \
      "mov.b64 bi, {%8, %10};\n\tmov.b64 bj, {%9, %10};\n\t"                                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ar, br, %11, p;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ar, bl, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], al, br, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ai, bi, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ai, bj, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], aj, bi, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], ai, br, %11, p;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], ai, bl, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], aj, br, %11, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], ar, bi, %12, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], ar, bj, %12, t;\n\t"                         \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], al, bi, %12, t;\n\t}"                        \
      ::"r"(d_re), "r"(d_im), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), \
      "r"(b[3]), "r"(hi), "r"(ipos), "r"(ineg), "r"(acc)                                              \
      : "memory")
  if (CG == 1) PS_MMA4("1");
  else PS_MMA4("2");
#undef PS_MMA4
}

// One K = 16 step of the Gauss 3-product split Gram as a single
// warp-collective block (see mma_4prod_step_warp):
//   k1 += S_i Zr_j   (Sh.Rh' + Sh.Rl' + Sl.Rh')      -> d1
//   k2 -= Zr_i S_j   (Rh.Sh' + Rh.Sl' + Rl.Sh')      -> d2 (negated A)
//   k3 += Zi_i D_j   (Ih.Dh' + Ih.Dl' + Il.Dh')      -> d3
// a = {Rh, Rl, Ih, Il, Sh, Sl} and b = {Rh, Rl, Sh, Sl, Dh, Dl} low words.
template <int CG>
__device__ __forceinline__ void mma_gauss_step_warp(uint32_t d1, uint32_t d2, uint32_t d3, const uint32_t (&a)[6],
                                                    const uint32_t (&b)[6], uint32_t hi, uint32_t ipos,
                                                    uint32_t ineg, uint32_t acc) {
#define PS_MMAG(CGS)                                                                                 \
  asm volatile(                                                                                        \
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 arh, arl, aih, ail, ash, asl, brh, brl, bsh, bsl, bdh, bdl;\n\t" \
      "elect.sync _|e, 0xffffffff;\n\t"                                                              \
      "setp.ne.b32 p, %20, 0;\n\tsetp.eq.b32 t, %20, %20;\n\t"                                       \
      "mov.b64 arh, {%3, %15};\n\tmov.b64 arl, {%4, %15};\n\tmov.b64 aih, {%5, %15};\n\t"          \
      "mov.b64 ail, {%6, %15};\n\tmov.b64 ash, {%7, %15};\n\tmov.b64 asl, {%8, %15};\n\t"          \
      "mov.b64 brh, {%9, %15};\n\tmov.b64 brl, {%10, %15};\n\tmov.b64 bsh, {%11, %15};\n\t"        \
      "mov.b64 bsl, {%12, %15};\n\tmov.b64 bdh, {%13, %15};\n\tmov.b64 bdl, {%14, %15};\n\t"       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ash, brh, %16, p;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], ash, brl, %16, t;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%0], asl, brh, %16, t;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], arh, bsh, %17, p;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], arh, bsl, %17, t;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%1], arl, bsh, %17, t;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%2], aih, bdh, %16, p;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%2], aih, bdl, %16, t;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CGS ".kind::f16 [%2], ail, bdh, %16, t;\n\t}"                      \
      ::"r"(d1), "r"(d2), "r"(d3), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(b[0]), \
      "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(hi), "r"(ipos), "r"(ineg), "r"(0u), "r"(0u), \
      "r"(acc)                                                                                          \
      : "memory")
  if (CG == 1) PS_MMAG("1");
  else PS_MMAG("2");
#undef PS_MMAG
}

// kind::f8f6f4 (E4M3 A / B, fp32 D; the instruction descriptor's format
// fields are 0 for E4M3 exactly as for F16, so make_idesc_f16 applies): the
// K7 mask-count Gram's 0 / 1 indicator operands, K = 32 per instruction
template <int CG>
__device__ __forceinline__ void mma_f8_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
            "r"(smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

// Commit: arrive (once) on `bar` when this thread's prior MMAs retire; for
// CG = 2 the arrival is multicast to the barrier at the same offset in both
// CTAs of the pair.
template <int CG>
__device__ __forceinline__ void mma_commit_cg(uint64_t* bar) {
  if (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  else
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16 inputs, fp32 accumulate).
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread
// have completed (implicitly fences before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit: thread (lane) l of the warp gets row
// (quadrant*32 + l), registers v[k] = column (col0 + k).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): K-major
// operand, swizzle mode `layout` (2 = 128B, 4 = 64B, 6 = 32B), SBO = bytes
// between consecutive 8-row core-matrix groups, LBO unused for swizzled
// K-major (set to 1), version 1 (sm_100), base offset 0 (tiles are aligned to
// the swizzle repeat).
__device__ __forceinline__ uint64_t make_smem_desc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                              // LBO (ignored)
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;     // SBO
  d |= (uint64_t)1u << 46;                              // version
  d |= (uint64_t)(layout & 7u) << 61;                    // swizzle / layout type
  return d;
}

// Instruction descriptor for kind::f16: fp16 A/B, fp32 D, both K-major.
__host__ __device__ constexpr uint32_t make_idesc_f16(int M, int N, bool negate_a) {
  return (1u << 4)                       // D format F32
         | (0u << 7) | (0u << 10)        // A, B format F16
         | ((negate_a ? 1u : 0u) << 13)  // negate A
         | (0u << 15) | (0u << 16)       // A, B K-major
         | ((uint32_t)(N >> 3) << 17)    // N >> 3
         | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

}  // namespace ptx
}  // namespace ps
