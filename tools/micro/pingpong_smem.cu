// Microbenchmark: handoff latency between two warps of ONE CTA through shared memory (volatile
// polling, value-as-flag) vs through global memory (.gpu and .cta scope), vs two CTAs through L2.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void st_gpu(int64_t *p, int64_t v) { asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ int64_t ld_gpu(const int64_t *p) { int64_t v; asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_cta(int64_t *p, int64_t v) { asm volatile("st.relaxed.cta.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ int64_t ld_cta(const int64_t *p) { int64_t v; asm volatile("ld.relaxed.cta.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

template <int MODE>  // 0 smem, 1 global .gpu, 2 global .cta (both warps in one CTA)
__global__ void pp_cta(int64_t *gflags, int iters, uint64_t *out) {
  __shared__ volatile int64_t sf[64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < 64) sf[threadIdx.x] = 0;
  __syncthreads();
  int64_t *gm = gflags + w * 32, *go = gflags + (1 - w) * 32;
  uint64_t t0 = gt();
  for (int it = 1; it <= iters; ++it) {
    auto put = [&]() {
      if (MODE == 0) sf[w * 32 + lane] = it;
      else if (MODE == 1) st_gpu(gm + lane, it);
      else st_cta(gm + lane, it);
    };
    auto get = [&]() -> int64_t {
      if (MODE == 0) return sf[(1 - w) * 32 + lane];
      else if (MODE == 1) return ld_gpu(go + lane);
      else return ld_cta(go + lane);
    };
    if (w == 0) {
      put();
      while (__any_sync(~0u, get() < it)) {}
    } else {
      while (__any_sync(~0u, get() < it)) {}
      put();
    }
  }
  if (w == 0 && lane == 0) out[0] = (gt() - t0) / iters;
}

__global__ void pp_grid(int64_t *flags, int iters, uint64_t *out) {
  const int lane = threadIdx.x & 31;
  int64_t *mine = flags + blockIdx.x * 32, *other = flags + (1 - blockIdx.x) * 32;
  uint64_t t0 = gt();
  for (int it = 1; it <= iters; ++it) {
    if (blockIdx.x == 0) {
      st_gpu(mine + lane, it);
      while (__any_sync(~0u, ld_gpu(other + lane) < it)) {}
    } else {
      while (__any_sync(~0u, ld_gpu(other + lane) < it)) {}
      st_gpu(mine + lane, it);
    }
  }
  if (blockIdx.x == 0 && lane == 0) out[0] = (gt() - t0) / iters;
}

int main() {
  int64_t *flags; uint64_t *out, h = 0;
  cudaMalloc(&flags, 64 * 8); cudaMalloc(&out, 8);
  const int iters = 20000;
  const char *names[3] = {"one CTA, shared memory", "one CTA, global .gpu", "one CTA, global .cta"};
  for (int m = 0; m < 3; ++m) {
    cudaMemset(flags, 0, 64 * 8);
    if (m == 0) pp_cta<0><<<1, 64>>>(flags, iters, out);
    if (m == 1) pp_cta<1><<<1, 64>>>(flags, iters, out);
    if (m == 2) pp_cta<2><<<1, 64>>>(flags, iters, out);
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-26s round trip %7.1f ns  %s\n", names[m], (double)h, cudaGetErrorString(cudaGetLastError()));
  }
  cudaMemset(flags, 0, 64 * 8);
  pp_grid<<<2, 32>>>(flags, iters, out);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-26s round trip %7.1f ns  %s\n", "two CTAs, L2 (.gpu)", (double)h, cudaGetErrorString(cudaGetLastError()));
}
