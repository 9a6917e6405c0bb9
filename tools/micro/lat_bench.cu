// Dependent-chain latencies on B200: DFMA, DADD(rn), DMUL+DADD, LDS.64, SHFL(f64), bar.sync
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = out[threadIdx.x], b = 1.0000001, c2 = 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c2);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, c2);
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // DMUL then DADD chain (exact mode madd)
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(__dmul_rn(a, b), c2);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // LDS chain (pointer chasing through smem index)
  int idx = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = s[idx]; idx = ((int)v) & 7; a += v * 1e-30; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // SHFL f64 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + c2;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = b / a;
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a) + c2;
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  out[threadIdx.x] = a + idx;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8 * 1024); cudaMemset(d, 0, 8 * 1024); cudaMalloc(&c, 64);
  const char* nm[] = {"DFMA", "DADD", "DMUL+DADD", "LDS.64(+conv)", "SHFL.f64+DADD", "bar.sync(256)", "DDIV", "DSQRT+DADD"};
  for (int T : {32, 256}) {
    k<<<1, T>>>(d, c, 1000); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("T=%3d %-16s %7.1f cycles/op\n", T, nm[i], h[i] / 1000.0);
  }
  return 0;
}
