// TMEM read latency with and without UMMAs in flight on the same SM
// (diagnostic for the short-K Gram, profiles/r02_session2/emission_experiments.md).
//
// One CTA per SM (cta_group::1), 512 TMEM columns.  Warp 1 (elected lane)
// issues `n_mma` kind::f16 UMMAs (M = 128, N = 128, K = 16) into columns
// [256, 384) from a zero-filled shared-memory operand, committing to an
// mbarrier every 16; warps 2..5 (the four TMEM lane quadrants) meanwhile run
// `n_ld` rounds of tcgen05.ld.32x32b.x32 + wait::ld of columns [0, 32) and time
// each round with clock64.  mode 0: no UMMAs (the reads alone); mode 1: UMMAs
// issued concurrently.  Prints the mean read-round cycles per mode and the
// UMMA stream's cycles.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1710_08037_b200/csrc \
//        tools/tmem_read_probe.cu -o gpurun_out/tmem_read_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "ptx.cuh"

using namespace ps;

__global__ void __launch_bounds__(192, 1) probe(int mode, int n_mma, int n_ld, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t opnd[2 * 128 * 32];  // A and B: 128 rows x 16 fp16 (32 B), no swizzle
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < (int)sizeof(opnd) / 4; k += blockDim.x) reinterpret_cast<uint32_t*>(opnd)[k] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    ptx::tmem_alloc(&tbase, 512);
    ptx::tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    if (mode == 1) {
      const uint32_t idesc = ptx::make_idesc_f16(128, 128, false);
      // no-swizzle K-major: 8-row core groups of 8 x 16 B; SBO = 8 rows x 16 B... (values are zeros: any
      // legal layout gives the same work)
      const uint64_t da = ptx::make_smem_desc(ptx::smem_u32(opnd), 128, 0);
      const uint64_t db = ptx::make_smem_desc(ptx::smem_u32(opnd + 128 * 32), 128, 0);
      const long long t0 = clock64();
      uint32_t ph = 0;
      for (int m = 0; m < n_mma; ++m) {
        ptx::mma_f16_ss_warp<1>(tmem + 256, da, db, idesc, m == 0 ? 0u : 1u);
        if ((m & 15) == 15) {
          ptx::mma_commit_warp<1>(&bar);
          ptx::mbar_wait(&bar, ph, nullptr);
          ph ^= 1u;
        }
      }
      if (lane == 0) out[blockIdx.x * 8 + 5] = (unsigned long long)(clock64() - t0);
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t v[32];
    unsigned long long sum = 0, mx = 0, x = 0;
    for (int r = 0; r < n_ld; ++r) {
      const long long t0 = clock64();
      ptx::tmem_ld_32x32b_x32(ta, v);
      ptx::tmem_wait_ld();
      const unsigned long long dt = (unsigned long long)(clock64() - t0);
      sum += dt;
      mx = dt > mx ? dt : mx;
#pragma unroll
      for (int k = 0; k < 32; ++k) x ^= v[k];
    }
    if (lane == 0) {
      out[blockIdx.x * 8 + q] = sum;
      if (q == 0) out[blockIdx.x * 8 + 4] = mx;
    }
    if (x == 0x12345) out[blockIdx.x * 8 + 6] = x;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  int n_sms = 0;
  cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d = nullptr;
  cudaMalloc(&d, (size_t)n_sms * 8 * sizeof(unsigned long long));
  const int n_mma = 200000, n_ld = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, (size_t)n_sms * 8 * sizeof(unsigned long long));
    probe<<<n_sms, 192>>>(mode, n_mma, n_ld, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);  // SM 0's counters
    const double rd = (double)(h[0] + h[1] + h[2] + h[3]) / (4.0 * n_ld);
    std::printf("{\"mode\": \"%s\", \"tmem_ld_x32_round_cycles_mean\": %.1f, \"max\": %llu, \"mma_stream_cycles\": %llu, "
                "\"mma_cycles_per_umma\": %.1f}\n",
                mode ? "UMMAs in flight" : "reads alone", rd, h[4], h[5], mode ? (double)h[5] / n_mma : 0.0);
  }
  return 0;
}
