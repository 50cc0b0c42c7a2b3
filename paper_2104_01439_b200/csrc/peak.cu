// FP64 FMA throughput microbenchmark (hh_fp64_peak): the denominator of the
// factorisation's TFLOP/s fractions ("measure FP64 FMA peak with
// a microbenchmark before quoting fractions").
//
// Every thread runs CH independent DFMA chains (enough to cover the FP64 pipe
// latency) for `iters` iterations; the grid is a multiple of the SM count with
// several CTAs per SM.  One DFMA = 2 flops.  The result is the best of `reps`
// launches timed with CUDA events.
#include <algorithm>
#include "hh_internal.cuh"

namespace {
constexpr int CH = 8;

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;   // keeps the chains live; never true in practice
}
// FP64 tensor-core MMA (mma.sync m8n8k4 f64, the instruction of the FD coarse
// solve's GEMMs, fd.cu): 4 independent accumulators per warp; 512 flops per MMA
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
}
}  // namespace

extern "C" hh_status hh_fp64_mma_peak(int32_t device, double* tflops) {
  if (!tflops) { hh_set_error("NULL argument"); return HH_E_ARG; }
  HH_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  HH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = nullptr;
  HH_CUDA_TRY(cudaMalloc(&out, sizeof(double)));
  cudaEvent_t e0, e1;
  HH_CUDA_TRY(cudaEventCreate(&e0));
  HH_CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256, iters = 1 << 13;
  k_dmma<<<blocks, threads>>>(out, 256);   // warm-up
  HH_CUDA_TRY(cudaGetLastError());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    HH_CUDA_TRY(cudaEventRecord(e0));
    k_dmma<<<blocks, threads>>>(out, iters);
    HH_CUDA_TRY(cudaEventRecord(e1));
    HH_CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    HH_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 512.0 * 4 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  return HH_OK;
}

extern "C" hh_status hh_fp64_peak(int32_t device, double* tflops, double* sm_mhz) {
  if (!tflops) { hh_set_error("NULL argument"); return HH_E_ARG; }
  HH_CUDA_TRY(cudaSetDevice(device));
  int sms = 0, clk_khz = 0;
  HH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, device);
  double* out = nullptr;
  HH_CUDA_TRY(cudaMalloc(&out, sizeof(double)));
  cudaEvent_t e0, e1;
  HH_CUDA_TRY(cudaEventCreate(&e0));
  HH_CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  k_dfma<<<blocks, threads>>>(out, 256, 0.999999, 1e-9);   // warm-up (clocks up)
  HH_CUDA_TRY(cudaGetLastError());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    HH_CUDA_TRY(cudaEventRecord(e0));
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    HH_CUDA_TRY(cudaEventRecord(e1));
    HH_CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    HH_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * CH * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (sm_mhz) *sm_mhz = clk_khz / 1e3;
  return HH_OK;
}
