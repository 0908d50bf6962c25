// fp64 latency / per-SMSP throughput microbenchmark (sm_100a): sizes the dual-kernel design.
//   dependent DFMA chain, dependent DMMA m8n8k4 chain, double shuffle, rsqrt, DMMA rate vs warps/SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(long long* out, double* sink, int iters) {
  double x = threadIdx.x * 1e-3 + 1.0, y = 0.999999, z = 1e-9;
  long long t0, t1;
  // DFMA
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, z);
  t1 = clock64();
  out[0] = t1 - t0;
  // DMMA m8n8k4 dependent on C
  double c0 = x, c1 = x * 0.5, a = y, b = z;
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  t1 = clock64();
  out[1] = t1 - t0;
  // DMMA with A depending on previous D (full dependence)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(c1), "d"(b));
  }
  t1 = clock64();
  out[2] = t1 - t0;
  // shfl double
  double s = c0 + c1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1e-300;
  t1 = clock64();
  out[3] = t1 - t0;
  // rsqrt
  double r = s * s + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) r = rsqrt(r) + 1.0;
  t1 = clock64();
  out[4] = t1 - t0;
  // smem load-use
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = r;
  __syncwarp();
  int idx = threadIdx.x & 31;
  double v = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    v = sh[idx];
    idx = ((int)v & 31) ^ (threadIdx.x & 31);
  }
  t1 = clock64();
  out[5] = t1 - t0;
  // div
  double d = r + 3.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = 1.0 / d + 1.0;
  t1 = clock64();
  out[6] = t1 - t0;
  // exp
  double e = d * 1e-3;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) e = exp(e) * 1e-3;
  t1 = clock64();
  out[7] = t1 - t0;
  // log
  double lg = e + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) lg = log(lg) + 2.0;
  t1 = clock64();
  out[8] = t1 - t0;
  sink[threadIdx.x] = x + c0 + c1 + s + r + v + d + e + lg;
}

__global__ void k_dmma_rate(double* sink, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = 0; c[j][1] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) sink[0] = s;
}

__global__ void k_dfma_rate(double* sink, int iters, long long* cyc) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], 0.999999, 1e-7);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) sink[0] = s;
}

int main() {
  long long* d_out;
  double* sink;
  cudaMalloc(&d_out, 4096 * 8);
  cudaMalloc(&sink, 4096 * 8);
  const int iters = 1024;
  k_lat<<<1, 32>>>(d_out, sink, iters);
  long long h[16];
  cudaMemcpy(h, d_out, 9 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dmma_c_dep", "dmma_full_dep", "shfl_f64", "rsqrt_f64", "smem_ld_use", "div_f64", "exp_f64", "log_f64"};
  for (int i = 0; i < 9; ++i) printf("{\"lat\": \"%s\", \"clk\": %.2f}\n", nm[i], (double)h[i] / iters);
  // per-SM rate with w warps in one CTA (one CTA on one SM)
  for (int w = 1; w <= 16; w *= 2) {
    k_dmma_rate<<<1, 32 * w>>>(sink, iters, d_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    // FMA per clk per SM: w warps * 4 dmma * 256 FMA * iters / cycles
    printf("{\"rate\": \"dmma_m8n8k4\", \"warps\": %d, \"fma_per_clk_sm\": %.2f}\n", w, (double)w * 4 * 256 * iters / h[0]);
    k_dfma_rate<<<1, 32 * w>>>(sink, iters, d_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("{\"rate\": \"dfma_acc8\", \"warps\": %d, \"fma_per_clk_sm\": %.2f}\n", w, (double)w * 32 * 8 * iters / h[0]);
  }
  return 0;
}
