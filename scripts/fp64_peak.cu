// fp64_peak.cu — measured FP64 ceilings on this GPU (roofline denominators).
//   dfma   : register-only DFMA chains (8 independent accumulators per thread)
//   dmma   : mma.sync.aligned.m8n8k4.row.col.f64 (register operands)
//   dmma16 : mma.sync.aligned.m16n8k4 / m16n8k8 / m16n8k16 .f64 (sm_90+ shapes)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak scripts/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 0.5, b = 1.0001;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0001 + i;
  double c[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// mixed: even warps run DFMA chains, odd warps m8n8k4 DMMA, concurrently — does the FP64
// vector pipe add to the tensor pipe, or do they share one ceiling?
__global__ void mixed_kernel(double* out, int iters_f, int iters_m) {
  const int warp = threadIdx.x >> 5;
  if (warp & 1) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters_m; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  double* d;
  CK(cudaMalloc(&d, 8));
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  float ms;
  // warm up
  dfma_kernel<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("{\"kernel\": \"dfma\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma884_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 4.0 * iters * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m8n8k4\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma1684_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 4 * 4.0 * iters * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m16n8k4\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma16816_kernel<<<blocks, threads>>>(d, iters / 4);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 16 * 2.0 * (iters / 4) * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m16n8k16\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
  }
  // mixed: iteration counts chosen so each half alone would take about the same time
  for (int ratio = 0; ratio < 3; ++ratio) {
    const int itf = iters, itm = iters * (ratio == 0 ? 1 : ratio == 1 ? 2 : 4) / 2;
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(d, itf, itm);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps_half = (double)blocks * (threads / 64);
    const double fl_f = 2.0 * 8 * itf * warps_half * 32, fl_m = 2.0 * 8 * 8 * 4 * 4.0 * itm * warps_half;
    printf("{\"kernel\": \"mixed dfma+dmma\", \"tflops\": %.2f, \"dfma_tf\": %.2f, \"dmma_tf\": %.2f, \"ms\": %.3f}\n",
           (fl_f + fl_m) / ms / 1e9, fl_f / ms / 1e9, fl_m / ms / 1e9, ms);
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
