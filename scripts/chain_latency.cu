// Latency of the replay engine's projection chain in isolation (diagnostic):
// one warp repeats check_violate's per-co-runner projection — operands from
// shared memory, pressure_exponent, kernel_effect (glibc-exact exp), the
// projected completion vs the deadline — as a dependent chain, with one
// effect per step (Pred::effect) and with two interleaved (Pred::effect2).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -prec-div=true -std=c++17 \
//        -Iinclude scripts/chain_latency.cu -o /tmp/chain && /tmp/chain
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2604_28175_b200/csrc/strait_device.cuh"

using namespace strait;

__global__ void k(const double* P, double* out, long long* cyc) {
  __shared__ double aex[5][64], x0[64], st[64], rb[64], dl[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 64; i += 32) {
    for (int m = 0; m < 5; ++m) aex[m][i] = 0.1 + 0.01 * m + 0.001 * i;
    x0[i] = 0.05;
    st[i] = 100.0;
    rb[i] = 3.0 + 0.01 * i;
    dl[i] = 104.0;
  }
  __syncwarp();
  Pred<5> pr;
  pr.load(P, 50.0);
  double c[5] = {0.2, 0.1, 0.3, 0.05, 0.15};
  int s = lane, acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < 1000; ++it) {  // one projection per step; the next slot depends on the result
    double x = x0[s];
#pragma unroll
    for (int i = 0; i < 5; ++i) x += pr.w[i] * (aex[i][s] + c[i]);
    bool sat;
    const double e = pr.effect(x, sat);
    const bool late = st[s] + rb[s] * (1.0 + e * pr.coeff[1]) > dl[s];
    acc += late;
    s = (s + 1 + late) & 63;
  }
  long long t1 = clock64();
  for (int it = 0; it < 1000; ++it) {  // two projections per step, interleaved
    double xa = x0[s], xb = x0[(s + 7) & 63];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      xa += pr.w[i] * (aex[i][s] + c[i]);
      xb += pr.w[i] * (aex[i][(s + 7) & 63] + c[i]);
    }
    double ea, eb;
    pr.effect2(xa, xb, ea, eb);
    const bool la = st[s] + rb[s] * (1.0 + ea * pr.coeff[1]) > dl[s];
    const bool lb = st[s] + rb[s] * (1.0 + eb * pr.coeff[1]) > dl[s];
    acc += la + lb;
    s = (s + 1 + la + lb) & 63;
  }
  long long t2 = clock64();
  out[lane] = acc;
  if (lane == 0) cyc[0] = t1 - t0, cyc[1] = t2 - t1;
}

int main() {
  double hP[12] = {0.5, 2.718281828, 0.0, 0.3, 0.3, 0.3, 0.3, 0.3, 0.2, 0.2, 0.5, 1.0};
  double *P, *o;
  long long* c;
  cudaMalloc(&P, sizeof hP);
  cudaMemcpy(P, hP, sizeof hP, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 256);
  cudaMallocManaged(&c, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(P, o, c);
    cudaDeviceSynchronize();
  }
  printf("projection chain: %.0f cycles per step (one effect), %.0f per step of two interleaved\n", c[0] / 1000.0,
         c[1] / 1000.0);
}
