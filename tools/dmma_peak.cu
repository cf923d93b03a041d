// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput vs DFMA, B200.
// Independent accumulator tiles per warp, full occupancy; prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int T>
__global__ void dmma_chains(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) c[t][0] = c[t][1] = t * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int T>
double run(int sms, int threads, int bpsm, double* out) {
  const int iters = 1 << 12, blocks = sms * bpsm;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  dmma_chains<T><<<blocks, threads>>>(out, 64);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(t0);
    dmma_chains<T><<<blocks, threads>>>(out, iters);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 256 * T * (double)iters * (threads / 32) * blocks;
  return flops / best / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  printf("{\"dmma_tflops\": {\"T4_w8\": %.2f, \"T8_w8\": %.2f, \"T8_w16\": %.2f, \"T4_w32\": %.2f, \"T2_w4\": %.2f}}\n",
         run<4>(sms, 256, 1, out), run<8>(sms, 256, 1, out), run<8>(sms, 256, 2, out), run<4>(sms, 256, 4, out),
         run<2>(sms, 128, 1, out));
  return 0;
}
