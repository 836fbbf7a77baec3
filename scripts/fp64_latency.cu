// FP64 dependent-chain latencies on one warp (diagnostic): DADD, DMUL, DFMA, __ddiv_rn, glibc exp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2604_28175_b200/csrc/strait_device.cuh"

__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = x + b;
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) x = x * b;
  long long t2 = clock64();
  for (int i = 0; i < 1000; ++i) x = __fma_rn(x, b, a);
  long long t3 = clock64();
  for (int i = 0; i < 200; ++i) x = __ddiv_rn(a, x + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < 200; ++i) x = strait::dexp(x * 1e-3);
  long long t5 = clock64();
  volatile __shared__ double sh[32];
  sh[threadIdx.x] = x;
  for (int i = 0; i < 1000; ++i) x = sh[(int)(x) & 31] + b;
  long long t6 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999); cudaDeviceSynchronize();
  printf("cycles per dependent op: DADD %.1f DMUL %.1f DFMA %.1f DDIV %.1f dexp %.1f LDS+DADD %.1f\n", c[0] / 1000.0,
         c[1] / 1000.0, c[2] / 1000.0, c[3] / 200.0, c[4] / 200.0, c[5] / 1000.0);
}
