// Microbenchmark: handoff latency between two warps on different SMs through global memory
// (st.relaxed.gpu / ld.relaxed.gpu, value-as-flag), optionally with background store traffic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_rel(int64_t *p, int64_t v) { asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ int64_t ld_rel(const int64_t *p) { int64_t v; asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void pingpong(int64_t *flags, int iters, int sleep_ns, uint64_t *out, int64_t *junk, int64_t junk_n) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x >= 2) {  // background store traffic
    int64_t v = blockIdx.x;
    for (int it = 0; it < iters * 8; ++it)
      for (int64_t i = (int64_t)blockIdx.x * 32 * 64 + lane; i < junk_n; i += (int64_t)gridDim.x * 32 * 64)
        junk[i] = v + it;
    return;
  }
  int64_t *mine = flags + blockIdx.x * 32, *other = flags + (1 - blockIdx.x) * 32;
  uint64_t t0 = gt();
  for (int it = 1; it <= iters; ++it) {
    if (blockIdx.x == 0) {
      st_rel(mine + lane, it);
      while (__any_sync(~0u, ld_rel(other + lane) < it)) if (sleep_ns) __nanosleep(sleep_ns);
    } else {
      while (__any_sync(~0u, ld_rel(other + lane) < it)) if (sleep_ns) __nanosleep(sleep_ns);
      st_rel(mine + lane, it);
    }
  }
  if (blockIdx.x == 0 && lane == 0) out[0] = (gt() - t0) / iters;
}

int main() {
  int64_t *flags, *junk; uint64_t *out;
  const int64_t junk_n = 1ll << 28;  // 2 GB
  cudaMalloc(&flags, 64 * 8); cudaMalloc(&out, 8); cudaMalloc(&junk, junk_n * 8);
  for (int bg : {0, 1}) for (int sl : {0, 32, 256, 1024}) {
    cudaMemset(flags, 0, 64 * 8);
    pingpong<<<bg ? 148 * 8 : 2, 32>>>(flags, 2000, sl, out, junk, junk_n);
    uint64_t h = 0; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("background=%d sleep=%4d ns: round trip %.2f us (one-way %.2f us)  %s\n", bg, sl, h / 1e3, h / 2e3, cudaGetErrorString(cudaGetLastError()));
  }
}
