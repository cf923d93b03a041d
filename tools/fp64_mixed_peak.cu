// Do the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) and the FP64 vector
// path (DFMA) share throughput on B200?  One kernel, warps split between
// DMMA chains and DFMA chains (warp-uniform role), same duration each;
// prints the DMMA-only, DFMA-only and mixed aggregate TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

// role per warp: 0 = DMMA, 1 = DFMA; dmma_frac of the warps run DMMA
__global__ void mixed(double* out, int dmma_iters, int dfma_iters, int dmma_warps_per_8) {
  const int w = threadIdx.x >> 5;
  const bool tc = (w % 8) < dmma_warps_per_8;
  double s = 0.0;
  if (tc) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = t * 1e-3;
    for (int i = 0; i < dmma_iters; ++i) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a), "d"(b));
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  } else {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-7 + c;
    for (int i = 0; i < dfma_iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 0.999999, 1e-9);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

static float time_it(int blocks, int threads, int di, int fi, int dw, double* out) {
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  mixed<<<blocks, threads>>>(out, 16, 64, dw);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(t0);
    mixed<<<blocks, threads>>>(out, di, fi, dw);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int threads = 256, blocks = sms * 4;
  const int di = 1 << 11, fi = 1 << 14;  // equal flops per warp in either role
  // flops per warp: DMMA 8 tiles x 256 FMA x 2 per iteration; DFMA 8 chains x 32 lanes x 2
  const double per_dmma_warp = 2.0 * 256 * 8 * di, per_dfma_warp = 2.0 * 8 * 32 * fi;
  const double warps = (threads / 32.0) * blocks;
  const float t_d = time_it(blocks, threads, di, fi, 8, out);  // all DMMA
  const float t_f = time_it(blocks, threads, di, fi, 0, out);  // all DFMA
  const float t_m = time_it(blocks, threads, di, fi, 4, out);  // half / half
  const double tf_d = per_dmma_warp * warps / t_d / 1e9, tf_f = per_dfma_warp * warps / t_f / 1e9;
  const double tf_m = (per_dmma_warp + per_dfma_warp) * warps / 2 / t_m / 1e9;
  printf("{\"dmma_only_tflops\": %.2f, \"dfma_only_tflops\": %.2f, \"mixed_half_half_tflops\": %.2f, "
         "\"mixed_ms\": %.3f, \"dmma_ms\": %.3f, \"dfma_ms\": %.3f}\n",
         tf_d, tf_f, tf_m, t_m, t_d, t_f);
  return 0;
}
