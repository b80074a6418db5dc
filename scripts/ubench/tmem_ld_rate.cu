// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM -- how fast the softmax warps can
// read S (fp32) out of tensor memory. W warps per sub-partition each load 32 columns of their
// lane quarter per step (4 KB per warp-load) and wait; reports bytes per SM-cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_ld_rate tmem_ld_rate.cu -I../../paper_2604_12798_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "vfa_kernel.cuh"
using namespace vfa;

template <int LOADS>  // loads in flight per wait
__global__ void __launch_bounds__(512, 1) kern(long long* out, float* sink, int iters) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t col0 = ((warp >> 2) * 64) & 511;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // independent chains: the loads, not the adds, bound
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[32 * LOADS];
#pragma unroll
    for (int l = 0; l < LOADS; ++l) tmem_ld32(tb + lane_off + ((col0 + l * 32 + (it & 3) * 128) & 480), v + 32 * l);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32 * LOADS; ++e) acc[e & 7] += v[e];
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int LOADS>
void run(int warps) {
  const int iters = 4000, blocks = 148;
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, blocks * sizeof(long long));
  cudaMalloc(&sink, blocks * 512 * sizeof(float));
  kern<LOADS><<<blocks, warps * 32>>>(d_out, sink, 10);
  kern<LOADS><<<blocks, warps * 32>>>(d_out, sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double bytes = static_cast<double>(warps) * 32 * 4 * 32 * LOADS * iters;  // per SM
  std::printf("warps/SM %2d  loads in flight %d: %7.1f B per SM-cycle  (%s)\n", warps, LOADS, bytes / avg,
              cudaGetErrorString(e));
  cudaFree(d_out);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<1>(w);
    run<2>(w);
  }
  return 0;
}
