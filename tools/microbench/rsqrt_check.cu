#include <cstdio>
#include <cmath>
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // one Newton step: y (1.5 - 0.5 x y^2)
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}
__global__ void k(const double* x, double* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { o[2*i] = rsqrt_fast(x[i]); o[2*i+1] = rsqrt(x[i]); }
}
int main() {
  const int n = 1 << 20;
  double *x, *o; cudaMallocManaged(&x, n * 8); cudaMallocManaged(&o, 2 * n * 8);
  for (int i = 0; i < n; ++i) x[i] = std::exp(((i * 2654435761u) % 100000) / 100000.0 * 60 - 30);
  k<<<n / 256, 256>>>(x, o, n); cudaDeviceSynchronize();
  double mx = 0, mx2 = 0;
  for (int i = 0; i < n; ++i) { double ref = 1.0 / std::sqrt(x[i]); mx = fmax(mx, fabs(o[2*i] - ref) / ref); mx2 = fmax(mx2, fabs(o[2*i+1]-ref)/ref); }
  printf("{\"rsqrt_fast_maxrel\": %.3e, \"rsqrt_maxrel\": %.3e}\n", mx, mx2);
}
