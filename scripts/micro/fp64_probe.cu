// Probe: DFMA latency / throughput, rsqrt(double), smem load latency on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dfma(double* out, double a, double b, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}
__global__ void tput_dfma(double* out, double a, double b, int iters) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void tput_ffma(float* out, float a, float b, int iters) {
  float x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = fmaf(x0, b, a); x1 = fmaf(x1, b, a); x2 = fmaf(x2, b, a); x3 = fmaf(x3, b, a);
    x4 = fmaf(x4, b, a); x5 = fmaf(x5, b, a); x6 = fmaf(x6, b, a); x7 = fmaf(x7, b, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lat_rsqrt(double* out, double a, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}
__global__ void lat_div(double* out, double a, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / x + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}
// DMMA (mma.sync m8n8k4 f64) throughput: 8 independent accumulators per warp
__global__ void tput_dmma(double* out, double a, double b, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = a + threadIdx.x + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// DFMA throughput with W warps per SM (occupancy sweep)
int main() {
  double* d; long long* c; float* f;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64); cudaMalloc(&f, 1 << 24);
  long long h;
  const int it = 10000;
  lat_dfma<<<1, 32>>>(d, 1.0, 0.5, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * it));
  lat_rsqrt<<<1, 32>>>(d, 2.0, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt(double)+add latency: %.2f cycles\n", (double)h / it);
  lat_div<<<1, 32>>>(d, 2.0, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1/x (double)+add latency: %.2f cycles\n", (double)h / it);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    tput_dfma<<<148 * 4, 512>>>(d, 1.0, 0.999, 4000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * 4000 * 148.0 * 4 * 512 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    tput_ffma<<<148 * 4, 512>>>(f, 1.0f, 0.999f, 4000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * 4000 * 148.0 * 4 * 512 / (ms * 1e-3) / 1e12);
    for (int thr : {64, 128, 256, 512}) {
      cudaEventRecord(e0);
      tput_dmma<<<148, thr>>>(d, 1.0, 0.999, 4000);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("DMMA throughput (%d warps/SM): %.1f TFLOP/s\n", thr / 32,
             2.0 * 256 * 8 * 4000 * 148.0 * (thr / 32) / (ms * 1e-3) / 1e12);
      cudaEventRecord(e0);
      tput_dfma<<<148, thr>>>(d, 1.0, 0.999, 4000);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("DFMA throughput (%d warps/SM): %.1f TFLOP/s\n", thr / 32,
             2.0 * 8 * 4000 * 148.0 * thr / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
