// Do independent IEEE divisions overlap?  One warp: a chain of steps, each with
// 1 or 5 independent __ddiv_rn (the TWA's five divisions by one total).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a) {
  double x = a, y[5] = {a, a * 1.1, a * 1.2, a * 1.3, a * 1.4};
  long long t0 = clock64();
  for (int i = 0; i < 200; ++i) x = __ddiv_rn(x + 3.0, x + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < 200; ++i) {
    const double d = y[0] + 1.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) y[j] = __ddiv_rn(y[j] + 3.0, d);
  }
  long long t2 = clock64();
  out[threadIdx.x] = x + y[0] + y[1] + y[2] + y[3] + y[4];
  if (threadIdx.x == 0) cyc[0] = t1 - t0, cyc[1] = t2 - t1;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize(); }
  printf("one division per step: %.0f cycles; five independent divisions per step: %.0f cycles\n", c[0] / 200.0, c[1] / 200.0);
}
