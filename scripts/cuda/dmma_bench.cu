// FP64 throughput probe: DFMA chains vs warp-level FP64 MMA (mma.sync f64) on
// this GPU (is the FP64 tensor path worth using for the coarse factorisation's
// rank-nb updates?).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double x[8];
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 0.999999, 1e-9);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

// m8n8k4: per thread a: 1, b: 1, c/d: 2 doubles; 4 independent accumulators
__global__ void k_mma884(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[4][2];
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
}

// m16n8k16 (sm_90+): a: 8, b: 4, c/d: 4 doubles
__global__ void k_mma16816(double* out, int iters) {
  double a[8], b[4], c[2][4];
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-6 + k;
  for (int k = 0; k < 4; ++k) b[k] = 0.999 - k * 1e-3;
  for (int k = 0; k < 2; ++k) for (int q = 0; q < 4; ++q) c[k][q] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
  for (int k = 0; k < 2; ++k) for (int q = 0; q < 4; ++q) s += c[k][q];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters / 8);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 13;
  const double warps = (double)blocks * threads / 32;
  float ms = timeit(k_dfma, blocks, threads, iters, out);
  printf("{\"dfma_tflops\": %.2f, ", 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12);
  ms = timeit(k_mma884, blocks, threads, iters, out);
  printf("\"mma_m8n8k4_tflops\": %.2f, ", 2.0 * 256 * 4 * iters * warps / (ms * 1e-3) / 1e12);
  ms = timeit(k_mma16816, blocks, threads, iters, out);
  printf("\"mma_m16n8k16_tflops\": %.2f, ", 2.0 * 2048 * 2 * iters * warps / (ms * 1e-3) / 1e12);
  cudaError_t e = cudaGetLastError();
  printf("\"error\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
