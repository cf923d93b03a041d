// FP64 peak microbenchmark for the roofline denominator (SURVEY §8d asks for
// a measured DFMA rate; MEASURED_PEAKS.json only has HBM and bf16).
// Independent DFMA chains per thread, full occupancy; prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int iters = 1 << 14, threads = 256, blocks = sms * 8;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  dfma_chains<8><<<blocks, threads>>>(out, 256, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(t0);
    dfma_chains<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * (double)iters * threads * blocks;
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
  return 0;
}
