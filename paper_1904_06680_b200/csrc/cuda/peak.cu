// peak.cu -- FP32 FFMA throughput probe: the roofline denominator of the
// rollout kernel (MEASURED_PEAKS.json carries only HBM and bf16 figures).
// 8 independent FMA chains per thread, 2 flop per FMA, every SM saturated.
#include <cuda_runtime.h>

#include "device_api.h"

namespace ppdev {

__global__ void __launch_bounds__(256) ffma_loop(float* out, int iters, float seed,
                                                  long long* cycles) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
  const float m = 0.999999f, c = 1e-7f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
      a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
  }
  const long long t1 = clock64();
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chains alive
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

int measure_ffma(int device, double* tflops, double* sm_mhz) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  long long* cyc = nullptr;
  cudaMalloc(&out, 1024 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  ffma_loop<<<blocks, threads>>>(out, 64, 1.f, cyc);  // warm-up / clock ramp
  ffma_loop<<<blocks, threads>>>(out, iters, 1.f, cyc);
  double best = 0.0, mhz = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    ffma_loop<<<blocks, threads>>>(out, iters, 1.f, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    long long cycles = 0;
    cudaMemcpy(&cycles, cyc, sizeof(cycles), cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 8.0 * 16.0 * iters * static_cast<double>(blocks) * threads;
    const double tf = flop / (ms * 1e-3) / 1e12;
    if (tf > best) {
      best = tf;
      mhz = static_cast<double>(cycles) / (ms * 1e-3) / 1e6;
    }
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  cudaFree(cyc);
  *tflops = best;
  *sm_mhz = mhz;
  return e;
}

}  // namespace ppdev
