// Feasibility + latency micro: (1) a cooperative launch with a 2-CTA cluster dimension; (2) the
// cost of one "EP max" step — every warp publishes a value, barrier, every warp reads all — with
// 16 warps in one CTA (bar.sync) vs 8 warps in each of 2 CTAs of a cluster (barrier.cluster +
// DSMEM reads via mapa/ld.shared::cluster).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void cta16(int iters, uint64_t *out, int64_t *sink) {
  __shared__ int64_t xm[2][16][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t m = lane + w;
  uint64_t t0 = gt();
  for (int it = 0; it < iters; ++it) {
    xm[it & 1][w][lane] = m;
    __syncthreads();
    int64_t v = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) v = max(v, xm[it & 1][q][lane]);
    m = v + 1;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (gt() - t0) / iters;
  sink[blockIdx.x * 512 + threadIdx.x] = m;
}

__global__ void __cluster_dims__(2, 1, 1) cl2x8(int iters, uint64_t *out, int64_t *sink) {
  __shared__ int64_t xm[2][8][32];
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned other = cl.block_rank() ^ 1u;
  int64_t m = lane + w;
  uint64_t t0 = gt();
  for (int it = 0; it < iters; ++it) {
    xm[it & 1][w][lane] = m;
    cl.sync();
    int64_t v = 0;
    int64_t(*rem)[8][32] = cl.map_shared_rank(xm, other);
#pragma unroll
    for (int q = 0; q < 8; ++q) v = max(v, max(xm[it & 1][q][lane], rem[it & 1][q][lane]));
    m = v + 1;
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (gt() - t0) / iters;
  sink[blockIdx.x * 256 + threadIdx.x] = m;
}

int main() {
  uint64_t *out; int64_t *sink;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&sink, 4096 * 512 * 8);
  const int iters = 20000;
  uint64_t h = 0;
  cta16<<<1, 512>>>(iters, out, sink);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("16 warps, one CTA, bar.sync:            %6.1f ns per step (%s)\n", (double)h, cudaGetErrorString(cudaGetLastError()));
  cl2x8<<<2, 256>>>(iters, out, sink);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("2 x 8 warps, cluster of 2, DSMEM:       %6.1f ns per step (%s)\n", (double)h, cudaGetErrorString(cudaGetLastError()));
  // cooperative launch of the cluster kernel over 128 CTAs (64 clusters)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(128); cfg.blockDim = dim3(256);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension; at[1].val.clusterDim.x = 2; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, cl2x8, iters, out, sink);
  cudaError_t e2 = cudaDeviceSynchronize();
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("cooperative + cluster launch, 128 CTAs: launch %s, sync %s, %6.1f ns per step\n", cudaGetErrorString(e), cudaGetErrorString(e2), (double)h);
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, (void *)cl2x8, &cfg);
  printf("max active clusters of 2 x 256 threads: %d\n", ncl);
}
