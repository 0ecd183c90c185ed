// Microbenchmark: L1 throughput of warp gathers with different widths / patterns
// (informs the stage-2 term layout; not part of the library).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W>  // bytes per lane: 4, 16, 32
__device__ __forceinline__ uint32_t ld(const uint8_t *p) {
  if constexpr (W == 32) {
    uint32_t a,b,c,d,e,f,g,h;
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(p));
    return a^b^c^d^e^f^g^h;
  } else if constexpr (W == 16) {
    uint32_t a,b,c,d;
    asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(p));
    return a^b^c^d;
  } else {
    uint32_t a;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(a) : "l"(p));
    return a;
  }
}

// pattern: lane offset in bytes = (lane * stride) % window, plus iteration shift
template <int W>
__global__ void k(const uint8_t *buf, int stride, int iters, uint32_t *out) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  const uint32_t off = (lane * stride) & 8191;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= ld<W>(buf + ((off + ((it * 8 + u) & 7) * 8192) & 65535));
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int W>
double run(const uint8_t *buf, int stride, uint32_t *out) {
  int blocks = 148 * 8, iters = 400;
  k<W><<<blocks, 256>>>(buf, stride, 10, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<W><<<blocks, 256>>>(buf, stride, iters, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double reqs = (double)blocks * 8 * iters * 8;  // warp-level requests
  return reqs / (ms * 1e-3) / 148 / 1.965e9;   // requests per SM-clock
}

int main() {
  uint8_t *buf; uint32_t *out;
  cudaMalloc(&buf, 1 << 20); cudaMalloc(&out, 64); cudaMemset(buf, 1, 1 << 20);
  int strides[] = {4, 16, 32, 64, 128, 256};
  printf("requests per SM-clock (warp-wide loads), L1-resident 64 KB window\n");
  for (int s : strides) printf("W=4  stride=%4d  %.3f\n", s, run<4>(buf, s, out));
  for (int s : strides) if (s >= 16) printf("W=16 stride=%4d  %.3f\n", s, run<16>(buf, s, out));
  for (int s : strides) if (s >= 32) printf("W=32 stride=%4d  %.3f\n", s, run<32>(buf, s, out));
  return 0;
}
