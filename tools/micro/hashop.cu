// Microbenchmark: cycles per compute-span op of the cell kernel's inner loop (8 ranks x one
// perturbed duration per lane, fin stores optional) for a lone warp / W warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_15617_b200/csrc/graph.h"
using namespace prism;
constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL, K_MIX = 0xBF58476D1CE4E5B9ULL;

// V1: the same function with the 64-bit steps spelled out on 32-bit halves
__device__ __forceinline__ int64_t perturb_v1(int64_t d, uint64_t x, const ScenParams &p) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  const uint64_t y = z ^ (z >> 27);
  const uint32_t lo = (uint32_t)y, hi = (uint32_t)(y >> 32);
  const uint32_t h = __umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu;
  const uint32_t v = h >> 8;
  int32_t r = (int32_t)(v - __umulhi(v, p.mod_m32) * (uint32_t)p.mod);
  if (r < 0) r += p.mod;
  return (d * (int64_t)((uint32_t)r + (uint32_t)(65536 - p.amp))) >> 16;
}

// V2: the C hashes of one op written step by step across the ranks (structure of arrays), so the
// independent chains are interleaved in program order
template <int C>
__device__ __forceinline__ void perturb_soa(int64_t (&t)[C], int64_t d, uint64_t sx, const uint64_t (&rk)[C], uint64_t ix,
                                            const ScenParams &p) {
  uint64_t z[C];
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = (sx ^ (rk[r] + ix)) + 0x9E3779B97F4A7C15ULL;
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = (z[r] ^ (z[r] >> 30)) * 0xBF58476D1CE4E5B9ULL;
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = (z[r] ^ (z[r] >> 27));
  uint32_t v[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t lo = (uint32_t)z[r], hi = (uint32_t)(z[r] >> 32);
    v[r] = (__umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu) >> 8;
  }
  int32_t m[C];
#pragma unroll
  for (int r = 0; r < C; ++r) m[r] = (int32_t)(v[r] - __umulhi(v[r], p.mod_m32) * (uint32_t)p.mod);
#pragma unroll
  for (int r = 0; r < C; ++r) m[r] += m[r] < 0 ? p.mod : 0;
#pragma unroll
  for (int r = 0; r < C; ++r) t[r] += (d * (int64_t)((uint32_t)m[r] + (uint32_t)(65536 - p.amp))) >> 16;
}

// V3: compute spans only — rk[r] = (rank << 32) * K_MIX has a zero low word, so x's low word and
// the carry of x + G are the same for every rank of the op; the mod correction without a branch
template <int C>
__device__ __forceinline__ void perturb_soa3(int64_t (&t)[C], int64_t d, uint64_t sx, const uint32_t (&rkhi)[C],
                                             uint64_t ix, const ScenParams &p) {
  const uint32_t xlo = (uint32_t)sx ^ (uint32_t)ix;
  const uint32_t zlo = xlo + 0x7F4A7C15u;
  const uint32_t cg = 0x9E3779B9u + (zlo < xlo ? 1u : 0u);
  const uint32_t sxh = (uint32_t)(sx >> 32), ixh = (uint32_t)(ix >> 32);
  const uint32_t zlo30 = zlo >> 30;
  uint64_t z[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t zh = (sxh ^ (ixh + rkhi[r])) + cg;
    const uint32_t lo = zlo ^ (zlo30 | (zh << 2)), hi = zh ^ (zh >> 30);
    z[r] = ((uint64_t)hi << 32 | lo) * 0xBF58476D1CE4E5B9ULL;
  }
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = z[r] ^ (z[r] >> 27);
  uint32_t v[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t lo = (uint32_t)z[r], hi = (uint32_t)(z[r] >> 32);
    v[r] = (__umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu) >> 8;
  }
  int32_t m[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    m[r] = (int32_t)(v[r] - __umulhi(v[r], p.mod_m32) * (uint32_t)p.mod);
    m[r] += (int32_t)((uint32_t)m[r] >> 31) * p.mod;
  }
  const int64_t dc = d * (int64_t)(uint32_t)(65536 - p.amp);
#pragma unroll
  for (int r = 0; r < C; ++r) t[r] += (d * (int64_t)(uint32_t)m[r] + dc) >> 16;
}

template <int V, bool REC>
__global__ void bench(ScenParams p, int ops, int64_t *fin, int64_t Sp, long long *out, int64_t *sink) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x;
  uint64_t rk[8]; int64_t t[8]; uint32_t rkhi[8];
  for (int r = 0; r < 8; ++r) { rk[r] = ((uint64_t)(w * 8 + r) << 32) * K_MIX; t[r] = 0; rkhi[r] = (uint32_t)(rk[r] >> 32); }
  const uint64_t sx = p.seed ^ ((uint64_t)(lane + 1) * K_GOLD);
  const int64_t d = 1000000 + w;
  long long c0 = clock64();
  for (int i = 0; i < ops; ++i) {
    const uint64_t ix = (uint64_t)i * K_MIX;
    if (V == 2) {
      perturb_soa<8>(t, d, sx, rk, ix, p);
    } else if (V == 3) {
      perturb_soa3<8>(t, d, sx, rkhi, ix, p);
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) t[r] += V == 0 ? perturb_x(d, sx ^ (rk[r] + ix), p) : perturb_v1(d, sx ^ (rk[r] + ix), p);
    }
    if (REC) {
#pragma unroll
      for (int r = 0; r < 8; ++r) fin[((int64_t)(w * 8 + r) * ops + i) * Sp + lane] = t[r];
    }
  }
  long long c1 = clock64();
  int64_t s = 0;
  for (int r = 0; r < 8; ++r) s += t[r];
  sink[w * 32 + lane] = s;
  if (lane == 0) out[w] = c1 - c0;
}

int main() {
  ScenParams p{};
  p.S = 32; p.amp = 6554; p.seed = 0x5EED; p.mask = 7; p.mod = 2 * 6554 + 1;
  p.mod_m32 = (uint32_t)((((uint64_t)1 << 32) + p.mod - 1) / p.mod);
  const int ops = 2000;
  int64_t *fin, *sink; long long *out;
  const int maxw = 148 * 16;
  cudaMalloc(&fin, (size_t)maxw * 8 * ops * 32 * 8);
  cudaMalloc(&sink, maxw * 32 * 8); cudaMalloc(&out, maxw * 8);
  long long h[maxw];
  for (int nw : {1, 148 * 4, 148 * 14}) {
    for (int v = 0; v < 8; ++v) {
      auto k = v == 0 ? bench<0, false> : v == 1 ? bench<1, false> : v == 2 ? bench<0, true> : v == 3 ? bench<1, true> : v == 4 ? bench<2, false> : v == 5 ? bench<2, true> : v == 6 ? bench<3, false> : bench<3, true>;
      for (int rep = 0; rep < 2; ++rep) k<<<nw, 32>>>(p, ops, fin, 32, out, sink);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0); k<<<nw, 32>>>(p, ops, fin, 32, out, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, out, nw * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < nw; ++i) avg += h[i]; avg /= nw;
      static int64_t hs[maxw * 32]; cudaMemcpy(hs, sink, nw * 32 * 8, cudaMemcpyDeviceToHost);
      long long cks = 0; for (int i = 0; i < nw * 32; ++i) cks = cks * 31 + hs[i];
      printf("  checksum %lld\n", cks);
      printf("warps=%5d variant=%s rec=%d: %.0f cycles/op per warp, kernel %.3f ms  %s\n", nw, v >= 6 ? "v3" : v >= 4 ? "v2" : (v & 1) ? "v1" : "v0", v >= 4 ? (v & 1) : v >> 1,
             avg / ops, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
