// HBM copy-throughput probes: stream count, per-thread ILP, cache hints,
// block size — which load/store shape reaches the measured copy peak
// (tools only: informs the K4 optimizer kernel's access pattern)
#include <cstdio>
#include <cuda_runtime.h>
template <int NR, int NW, int U, int HINT>
__global__ void kstreams(float4* const* __restrict__ in, float4* const* __restrict__ out, long n4) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long i0 = (long)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n4; i0 += stride) {
    float4 v[NR][U];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const long i = i0 + (long)u * blockDim.x;
        v[r][u] = i < n4 ? (HINT == 0 ? __ldcs(in[r] + i) : HINT == 1 ? __ldg(in[r] + i) : __ldlu(in[r] + i))
                         : make_float4(0, 0, 0, 0);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + (long)u * blockDim.x;
      if (i >= n4) continue;
      float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
      for (int r = 0; r < NR; ++r) { acc.x += v[r][u].x; acc.y += v[r][u].y; acc.z += v[r][u].z; acc.w += v[r][u].w; }
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        if (HINT == 0) __stcs(out[w] + i, acc); else out[w][i] = acc;
      }
    }
  }
}
// persistent grid, each block streams one contiguous chunk (instead of a grid stride)
template <int NR, int NW>
__global__ void kchunk(float4* const* __restrict__ in, float4* const* __restrict__ out, long n4) {
  const long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long b0 = blockIdx.x * per, b1 = b0 + per < n4 ? b0 + per : n4;
  for (long i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < NR; ++r) { const float4 v = __ldcs(in[r] + i); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
#pragma unroll
    for (int w = 0; w < NW; ++w) __stcs(out[w] + i, acc);
  }
}
template <int NR, int NW>
void run_chunk(long total_bytes, int threads) {
  long n4 = total_bytes / 16 / (NR + NW);
  float4 *hi[8], *ho[8];
  for (int r = 0; r < NR; ++r) { cudaMalloc(&hi[r], n4 * 16); cudaMemset(hi[r], 0, n4 * 16); }
  for (int w = 0; w < NW; ++w) cudaMalloc(&ho[w], n4 * 16);
  float4 **di, **dout;
  cudaMalloc(&di, sizeof(hi)); cudaMalloc(&dout, sizeof(ho));
  cudaMemcpy(di, hi, sizeof(hi), cudaMemcpyHostToDevice); cudaMemcpy(dout, ho, sizeof(ho), cudaMemcpyHostToDevice);
  int blocks; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kchunk<NR, NW>, threads, 0);
  int grid = blocks * 148;
  for (int i = 0; i < 3; ++i) kchunk<NR, NW><<<grid, threads>>>(di, dout, n4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) kchunk<NR, NW><<<grid, threads>>>(di, dout, n4);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
  printf("chunked persistent r%d w%d thr%d: %.0f GB/s\n", NR, NW, threads, n4 * 16.0 * (NR + NW) / ms / 1e6);
  for (int r = 0; r < NR; ++r) cudaFree(hi[r]);
  for (int w = 0; w < NW; ++w) cudaFree(ho[w]);
  cudaFree(di); cudaFree(dout);
}
template <int NR, int NW, int U, int HINT>
void run(long total_bytes, int threads, int waves) {
  long n4 = total_bytes / 16 / (NR + NW);
  float4 *hi[8], *ho[8];
  for (int r = 0; r < NR; ++r) { cudaMalloc(&hi[r], n4 * 16); cudaMemset(hi[r], 0, n4 * 16); }
  for (int w = 0; w < NW; ++w) cudaMalloc(&ho[w], n4 * 16);
  float4 **di, **dout;
  cudaMalloc(&di, sizeof(hi)); cudaMalloc(&dout, sizeof(ho));
  cudaMemcpy(di, hi, sizeof(hi), cudaMemcpyHostToDevice); cudaMemcpy(dout, ho, sizeof(ho), cudaMemcpyHostToDevice);
  int blocks; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kstreams<NR, NW, U, HINT>, threads, 0);
  int grid = blocks * 148 * waves;
  for (int i = 0; i < 3; ++i) kstreams<NR, NW, U, HINT><<<grid, threads>>>(di, dout, n4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) kstreams<NR, NW, U, HINT><<<grid, threads>>>(di, dout, n4);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
  printf("r%d w%d U%d hint%d thr%d waves%d (blocks/SM %d): %.0f GB/s\n", NR, NW, U, HINT, threads, waves, blocks,
         n4 * 16.0 * (NR + NW) / ms / 1e6);
  for (int r = 0; r < NR; ++r) cudaFree(hi[r]);
  for (int w = 0; w < NW; ++w) cudaFree(ho[w]);
  cudaFree(di); cudaFree(dout);
}
int main() {
  const long T = 2400L << 20;
  run<1, 1, 1, 0>(T, 256, 1);
  run<1, 1, 2, 0>(T, 256, 1);
  run<1, 1, 4, 0>(T, 256, 1);
  run<1, 1, 4, 1>(T, 256, 1);
  run<1, 1, 4, 2>(T, 256, 1);
  run<1, 1, 1, 0>(T, 256, 8);
  run<1, 1, 4, 0>(T, 512, 1);
  run<1, 1, 8, 0>(T, 256, 1);
  run<4, 4, 2, 0>(T, 256, 1);
  run<4, 4, 2, 1>(T, 256, 1);
  run<4, 4, 1, 0>(T, 256, 4);
  run_chunk<1, 1>(T, 256);
  run_chunk<3, 1>(T, 256);
  run_chunk<4, 4>(T, 256);
  run<3, 1, 1, 0>(T, 256, 1);
  run<3, 1, 1, 0>(T, 256, 8);
  // torch-style copy for reference: cudaMemcpy D2D
  {
    long n = T / 2;
    void *x, *y; cudaMalloc(&x, n); cudaMalloc(&y, n);
    cudaMemcpy(y, x, n, cudaMemcpyDeviceToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) cudaMemcpyAsync(y, x, n, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
    printf("cudaMemcpy D2D: %.0f GB/s\n", 2.0 * n / ms / 1e6);
  }
  return 0;
}
