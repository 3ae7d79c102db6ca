// Device->host copy-out probe for the pipelined host path (GPU box only):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/d2h_probe.cu -o /tmp/d2h_probe && /tmp/d2h_probe
// Moves the upper triangle of an N x N fp32 matrix (row bands x column
// stages, the streamed copy-out's block shapes) into pinned host memory:
//   dma2d  cudaMemcpy2DAsync per block (copy engine)
//   dma1d  one contiguous copy of the same byte count (link ceiling)
//   sm     a copy kernel writing the blocks straight into mapped host memory
//          (16-byte loads / stores, one warp per row segment)
// and the same three while a compute-heavy kernel occupies the SMs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

struct Blk {
  long long r0, r1, c0, c1;
};

__global__ void sm_copy(const float* __restrict__ src, float* dst, long long N, const Blk* blks, int nb) {
  // grid-stride over (block, row); one warp per row segment, float4 when aligned
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  long long total = 0;
  for (int b = 0; b < nb; ++b) total += blks[b].r1 - blks[b].r0;
  for (long long w = warp; w < total; w += nw) {
    long long x = w;
    int b = 0;
    while (x >= blks[b].r1 - blks[b].r0) x -= blks[b].r1 - blks[b].r0, ++b;
    const long long r = blks[b].r0 + x;
    const long long c0 = blks[b].c0, c1 = blks[b].c1;
    const float* s = src + r * N;
    float* d = dst + r * N;
    long long c = c0;
    for (; c < c1 && (c & 3); ++c)
      if (c - c0 == lane) d[c] = s[c];
    const long long a0 = c, a1 = c1 & ~3LL;
    for (long long q = a0 + 4 * lane; q < a1; q += 128)
      *reinterpret_cast<float4*>(d + q) = __ldg(reinterpret_cast<const float4*>(s + q));
    for (long long q = a1 + lane; q < c1; q += 32) d[q] = s[q];
  }
}

// HBM-heavy load: streaming reads of a large buffer (like the Gram's operand traffic)
__global__ void busy_mem(const float4* __restrict__ x, long long n, int reps, float* sink) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
      const float4 v = __ldcs(x + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void busy(float* x, int iters) {
  float a = x[threadIdx.x], b = 1.0001f;
  for (int i = 0; i < iters; ++i) a = a * b + 1e-7f;
  if (a == 12345.f) x[threadIdx.x] = a;
}

int main() {
  const long long N = 20000;
  std::vector<Blk> blks;
  // column stages as the host path builds them; row bands of 3072
  std::vector<long long> cols;
  long long w = 1024, wmax = 3584;
  for (long long x = 0; x < N; x += w, w = std::min(wmax, w + 512)) cols.push_back(x);
  cols.push_back(N);
  for (size_t s = 0; s + 1 < cols.size(); ++s)
    for (long long r0 = 0; r0 < cols[s + 1]; r0 += 3072) {
      const long long r1 = std::min(r0 + 3072, cols[s + 1]);
      const long long top = std::min(r1, cols[s]);
      if (top > r0) blks.push_back({r0, top, cols[s], cols[s + 1]});
      for (long long a = std::max(r0, cols[s]); a < r1; a += 256)
        blks.push_back({a, std::min(a + 256, r1), a, cols[s + 1]});
    }
  double bytes = 0;
  for (auto& b : blks) bytes += 4.0 * (b.r1 - b.r0) * (b.c1 - b.c0);
  // three matrices, as the three metrics of the host path
  float *dm[3], *hm[3], *hdm[3];
  for (int m = 0; m < 3; ++m) {
    cudaMalloc(&dm[m], N * N * 4);
    cudaMemset(dm[m], 0, N * N * 4);
    cudaHostAlloc(&hm[m], N * N * 4, cudaHostAllocMapped | cudaHostAllocPortable);
    memset(hm[m], 0, N * N * 4);
    cudaHostGetDevicePointer((void**)&hdm[m], hm[m], 0);
  }
  float *d = dm[0], *h = hm[0], *hd = hdm[0];
  const long long nmem = (4LL << 30) / 16;
  float4* mem;
  cudaMalloc(&mem, nmem * 16);
  cudaMemset(mem, 0, nmem * 16);
  Blk* dblk;
  cudaMalloc(&dblk, blks.size() * sizeof(Blk));
  cudaMemcpy(dblk, blks.data(), blks.size() * sizeof(Blk), cudaMemcpyHostToDevice);
  float* bx;
  cudaMalloc(&bx, 1024 * 4);
  cudaMemset(bx, 0, 1024 * 4);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](int mode, int loaded, int grid) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      if (loaded == 1) busy<<<nsm, 576, 0, s1>>>(bx, 20000000);
      if (loaded == 2) busy_mem<<<nsm, 576, 0, s1>>>(mem, nmem, 60, bx);
      cudaEventRecord(e0, s0);
      if (mode == 0) {
        for (auto& b : blks)
          cudaMemcpy2DAsync(h + b.r0 * N + b.c0, N * 4, d + b.r0 * N + b.c0, N * 4, (b.c1 - b.c0) * 4, b.r1 - b.r0,
                            cudaMemcpyDeviceToHost, s0);
      } else if (mode == 3) {  // three matrices, metric-interleaved per block (the host path's order)
        for (auto& b : blks)
          for (int m = 0; m < 3; ++m)
            cudaMemcpy2DAsync(hm[m] + b.r0 * N + b.c0, N * 4, dm[m] + b.r0 * N + b.c0, N * 4, (b.c1 - b.c0) * 4,
                              b.r1 - b.r0, cudaMemcpyDeviceToHost, s0);
      } else if (mode == 1) {
        cudaMemcpyAsync(h, d, (size_t)bytes, cudaMemcpyDeviceToHost, s0);
      } else {
        sm_copy<<<grid, 256, 0, s0>>>(d, hd, N, dblk, (int)blks.size());
      }
      cudaEventRecord(e1, s0);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
      cudaDeviceSynchronize();
    }
    return best;
  };
  const char* names[4] = {"dma2d", "dma1d", "sm", "dma2d_3mat"};
  const char* loads[3] = {"", "_alu", "_hbm"};
  printf("{\"blocks\": %zu, \"bytes\": %.0f", blks.size(), bytes);
  for (int loaded = 0; loaded < 3; ++loaded)
    for (int mode = 0; mode < 4; ++mode) {
      if (mode == 3) {
        const float ms = run(mode, loaded, 0);
        printf(", \"%s%s_GBps\": %.1f", names[mode], loads[loaded], 3 * bytes / ms / 1e6);
      } else if (mode == 2) {
        for (int grid : {nsm / 4, nsm, nsm * 4}) {
          const float ms = run(mode, loaded, grid);
          printf(", \"%s%s_g%d_GBps\": %.1f", names[mode], loads[loaded], grid, bytes / ms / 1e6);
        }
      } else {
        const float ms = run(mode, loaded, 0);
        printf(", \"%s%s_GBps\": %.1f", names[mode], loads[loaded], bytes / ms / 1e6);
      }
    }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
