// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM on B200 (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_bw tmem_bw.cu -I../../paper_2604_12798_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace vfa;

template <int MODE>  // 0: ld x32, 1: ld x16, 2: st x16, 3: ld x32 without per-load wait (4 in flight)
__global__ void kern(long long* out, int iters, float* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 32;
  const uint32_t ta = base + lane_off + col;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      float v[32];
      tmem_ld32(ta, v);
      tmem_wait_ld();
      reg_fence32(v);
      acc += v[0] + v[31];
    } else if (MODE == 1) {
      float v[16];
      tmem_ld16(ta, v);
      tmem_wait_ld();
      reg_fence16(v);
      acc += v[0] + v[15];
    } else if (MODE == 2) {
      uint32_t u[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) u[e] = i + e;
      tmem_st16(ta, u);
      tmem_wait_st();
    } else {
      float v[4][32];
#pragma unroll
      for (int k = 0; k < 4; ++k) tmem_ld32(base + lane_off + ((col + 128 * k) & 511), v[k]);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        reg_fence32(v[k]);
        acc += v[k][0] + v[k][31];
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}

template <int MODE>
void run(int warps, const char* name, double bytes_per_iter_warp) {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sink, 4 * 1024);
  const int iters = 20000;
  kern<MODE><<<148, warps * 32>>>(d, 100, sink);
  kern<MODE><<<148, warps * 32>>>(d, iters, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148;
  double bytes = bytes_per_iter_warp * warps * iters;
  printf("%-28s warps=%2d  %8.1f cycles/iter  %7.1f B/clk/SM  (%s)\n", name, warps, cyc / iters, bytes / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) run<0>(w, "ld 32x32b.x32 + wait", 32 * 32 * 4);
  for (int w : {4, 8, 16}) run<1>(w, "ld 32x32b.x16 + wait", 32 * 16 * 4);
  for (int w : {4, 8, 16}) run<2>(w, "st 32x32b.x16 + wait", 32 * 16 * 4);
  for (int w : {4, 8, 16}) run<3>(w, "4x ld x32, one wait", 4 * 32 * 32 * 4);
  return 0;
}
