// memory.cu — row a9: per-rank peak memory ("max_memory_allocated").
//
// Events per op: +alloc at its start, -free at its finish, ordered by (time, per-rank event
// index). On a single-stream rank the event times are non-decreasing in program order (start_i >=
// finish_{i-1} >= start_{i-1}), so that order IS program order (Z6) and the peak
// does not depend on the scenario: peak_r = static + max(0, max_i (R_i + alloc_i)) where R_i is
// the exclusive prefix sum of (alloc - free) — the running total right after op i's allocation.
// One warp per rank: 32 ops per step, 64-bit warp inclusive scan with shuffles, the running
// maximum kept per lane (one warp reduction per rank); HBM read-bound
// (16 B per node: alloc + free), 8 B per rank written.
#include <cuda_runtime.h>

#include "graph.h"

namespace prism {

namespace {

__global__ void __launch_bounds__(256) peak_kernel(DevGraph g, int64_t *__restrict__ peak) {
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < g.W; r += warps) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
    // the rank's memory deltas: its stage template's (L2-resident), or per-node overrides
    const int64_t *al = g.node_alloc ? g.node_alloc + rb : g.t_alloc + g.t_op0[g.rank_stage[r]];
    const int64_t *fr = g.node_free ? g.node_free + rb : g.t_free + g.t_op0[g.rank_stage[r]];
    int64_t carry = 0, best = 0;  // best: this lane's max of R_i + alloc_i (warp max at the end)
    for (int32_t base = rb; base < re; base += 32) {
      const int32_t i = base + lane;
      int64_t a = 0, f = 0;
      if (i < re) {
        a = al[i - rb];
        f = fr[i - rb];
      }
      int64_t x = a - f;  // inclusive scan of (alloc - free)
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (i < re) best = max(best, carry + x - (a - f) + a);  // R_i + alloc_i
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) best = max(best, (int64_t)__shfl_xor_sync(0xffffffffu, best, off));
    if (lane == 0) peak[r] = g.static_mem[g.rank_stage[r]] + best;
  }
}

}  // namespace

cudaError_t preload_peak_kernel() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void *)peak_kernel);
}

cudaError_t launch_peak(const DevGraph &g, int64_t *peak, cudaStream_t st) {
  if (g.W == 0) return cudaSuccess;
  int blocks = (g.W + 7) / 8;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  peak_kernel<<<blocks, 256, 0, st>>>(g, peak);
  return cudaGetLastError();
}

}  // namespace prism
