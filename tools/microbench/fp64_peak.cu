// fp64 peak microbenchmark for B200 (sm_100a): DFMA pipe and DMMA (mma.sync f64).
// Used once to fix the fp64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 - i * 1e-5;
  double c[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  auto run = [&](const char* name, auto launch, double flop_per_launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"tflops\": %.3f}\n", name, best, flop_per_launch / best / 1e9);
  };
  const int it = 4096;
  run("dfma_acc8", [&] { k_dfma<8><<<blocks, threads>>>(d, it, 0.999999, 1e-7); }, 2.0 * 8 * it * (double)threads * blocks);
  run("dfma_acc16", [&] { k_dfma<16><<<blocks, threads>>>(d, it, 0.999999, 1e-7); }, 2.0 * 16 * it * (double)threads * blocks);
  run("dmma_m8n8k4", [&] { k_dmma_m8n8k4<<<blocks, threads>>>(d, it); }, 2.0 * 8 * 8 * 4 * 4 * it * (double)(threads / 32) * blocks);
  run("dmma_m16n8k16", [&] { k_dmma_m16n8k16<<<blocks, threads>>>(d, it / 4); }, 2.0 * 16 * 8 * 16 * 2 * (it / 4) * (double)(threads / 32) * blocks);
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(err));
  return 0;
}
