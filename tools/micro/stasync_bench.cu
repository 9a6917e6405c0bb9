// Latency of a cluster all-reduce of cnt values: DSMEM push + barrier.cluster
// (release) versus st.async + mbarrier complete_tx (no release fence).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void bench(int iters, int cnt, int mode, double* out, long long* cyc) {
  __shared__ __align__(16) double buf[2][16][32];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), rank = cl.block_rank(), t = threadIdx.x;
  if (t == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cbar();
  double v = t * 1e-3;
  uint32_t ph[2] = {0, 0};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int p = it & 1;
    if (mode == 0) {  // push + cluster barrier
      if (t < cnt) for (int r = 0; r < C; ++r)
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(mapa(su32(&buf[p][rank][t]), r)), "d"(v) : "memory");
      cbar();
    } else {  // st.async + mbarrier
      if (t == 0) mbar_expect(&bar[p], (uint32_t)(C * cnt * 8));
      if (t < cnt) for (int r = 0; r < C; ++r)
        st_async(mapa(su32(&buf[p][rank][t]), r), v, mapa(su32(&bar[p]), r));
      mbar_wait(&bar[p], ph[p]);
      ph[p] ^= 1;
    }
    double s = 0.0;
    if (t < cnt) for (int r = 0; r < C; ++r) s += buf[p][r][t];
    v = s * 1e-3 + 1.0;
  }
  long long t1 = clock64();
  if (t == 0 && rank == 0) { *cyc = (t1 - t0) / iters; *out = v; }
  cbar();
}

int main() {
  double* d; long long* cy; cudaMalloc(&d, 8); cudaMalloc(&cy, 8);
  for (int C : {4, 8, 16}) for (int mode : {0, 1}) for (int cnt : {1, 22, 44}) {
    if (cnt > 32) continue;
    cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = C; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, bench, 2000, cnt, mode, d, cy);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
    printf("C=%2d %-22s cnt=%2d : %6lld cycles (%s)\n", C, mode ? "st.async+mbarrier" : "push+cluster barrier", cnt, h,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
