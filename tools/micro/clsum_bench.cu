// Latency of one multi-value cluster all-reduce (cl_sum) and of primitives.
#include <cstdio>
#include "../../paper_2209_06916_b200/csrc/mgb_cluster.cuh"
using namespace mgb;

// pull variant: partials written locally, one barrier, peers read remotely
template <int N>
__device__ __forceinline__ void cl_sum_pull(ClCtx& c, cg::cluster_group& cl, double (&v)[N], int cnt) {
  cl_sum_a<N>(c, v, cnt);
  double* mine = c.cred + c.parity * (CL_MAXC * N);  // my CTA total per value
  if (c.t < cnt) {
    double s = 0.0;
    for (int w = 0; w < c.nw; ++w) s += c.wred[w * N + c.t];
    mine[c.t] = s;
  }
  cluster_barrier();
  if (c.t < cnt) {
    double s = 0.0;
    for (int r = 0; r < c.C; ++r) s += cl.map_shared_rank(mine, r)[c.t];
    c.tot[c.t] = s;
  }
  __syncthreads();
  for (int i = 0; i < N; ++i) if (i < cnt) v[i] = c.tot[i];
  c.parity ^= 1;
}

template <int N>
__global__ void bench(int iters, int cnt, int mode, double* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  double* sm = reinterpret_cast<double*>(smem_raw);
  ClCtx c;
  c.C = cl.num_blocks(); c.rank = cl.block_rank(); c.t = threadIdx.x; c.lane = c.t & 31; c.warp = c.t >> 5;
  c.nw = blockDim.x >> 5; c.wred = sm; c.cred = sm + 8 * 32; c.tot = c.cred + 2 * 16 * 32;
  c.parity = 0;
  cluster_barrier();
  double v[N];
  for (int i = 0; i < N; ++i) v[i] = c.t + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) cl_sum<N>(c, v, cnt);
    else if (mode == 1) cluster_barrier();
    else if (mode == 2) __syncthreads();
    else if (mode == 3) { cl_sum_a<N>(c, v, cnt); }
    else { cl_sum_pull<N>(c, cl, v, cnt); }
    v[0] *= 1e-3;
  }
  long long t1 = clock64();
  if (c.t == 0 && c.rank == 0) { *cyc = (t1 - t0) / iters; *out = v[0]; }
  cluster_barrier();
}

int main() {
  double* d; long long* cy; cudaMalloc(&d, 8); cudaMalloc(&cy, 8);
  for (int C : {8, 16}) for (int T : {128, 256}) for (int mode : {0, 1, 2, 4}) for (int cnt : {1, 21}) {
    
    auto fn = bench<21>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(T); cfg.dynamicSmemBytes = 40 * 1024;
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = C; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    int iters = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, fn, 10, cnt, mode, d, cy);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, fn, iters, cnt, mode, d, cy);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h; cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
    const char* nm[] = {"cl_sum", "cluster_barrier", "syncthreads", "cl_sum_a(warp+sync)", "cl_sum_pull"};
    printf("C=%2d T=%3d %-22s cnt=%2d : %7.0f cycles  %6.3f us/op (%s)\n", C, T, nm[mode], cnt, (double)h, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
