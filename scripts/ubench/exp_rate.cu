// Microbenchmark: the softmax inner loop of the attention kernels in isolation -- per element
// x = s*c - m (FFMA2), p = exp2(x) on MUFU.EX2 (or the FMA-pipe polynomial for EMU pairs of
// every 8), bf16 pack (F2FP), row sum (FADD2) -- with W warps per sub-partition, each thread
// owning CP columns of a row, optionally storing P to TMEM (tcgen05.st + wait::st) per 32
// columns as the kernels do. Reports cycles per block and the XU (MUFU) utilisation
// (16 exp2 per SM-cycle peak).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o exp_rate exp_rate.cu -I../../paper_2604_12798_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "vfa_kernel.cuh"
using namespace vfa;

template <int CP, int EMU, bool TST>
__global__ void __launch_bounds__(512, 1) kern(long long* out, float* sink, int iters, float seed) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (TST && warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = TST ? tbase_s : 0u;
  float v[CP];
#pragma unroll
  for (int e = 0; e < CP; ++e) v[e] = seed * (threadIdx.x + e) * 1e-3f - 8.0f;
  const float2 cs2 = make_float2(1.0f, 1.0f);
  float l = 0.f;
  uint32_t xs = 0;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t tcol = tb + lane_off + ((warp >> 2) & 7) * 32;  // distinct columns per warp
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float nm = -0.25f * (it & 3);
    const float2 nmu2 = make_float2(nm, nm);
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < CP / 32; ++c) {
      uint32_t u[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float2 x = __ffma2_rn(make_float2(v[c * 32 + e], v[c * 32 + e + 1]), cs2, nmu2);
        float2 p;
        if (((e >> 1) & 7) >= 8 - EMU) {
          p = ex2_poly3(x);
        } else {
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
        }
        acc[(e >> 1) & 1] = add_ftz2(acc[(e >> 1) & 1], p);
        u[e >> 1] = pack_bf16x2(p.x, p.y);
      }
      if constexpr (TST) {
        tmem_st16(tcol + (c & 1) * 16, u);
        tmem_wait_st();
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) xs ^= u[e];
      }
    }
    l += acc[0].x + acc[0].y + acc[1].x + acc[1].y;
#pragma unroll
    for (int e = 0; e < CP; ++e) v[e] = v[e] + 1e-7f;  // keep the loads live
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l + __uint_as_float(xs);
  tc_fence_before();
  __syncthreads();
  if (TST && warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int CP, int EMU, bool TST>
void run(int warps_per_smsp, const char* name) {
  const int threads = warps_per_smsp * 4 * 32, iters = 2000, blocks = 148;
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, blocks * sizeof(long long));
  cudaMalloc(&sink, blocks * 512 * sizeof(float));
  kern<CP, EMU, TST><<<blocks, threads>>>(d_out, sink, 10, 1.0f);
  kern<CP, EMU, TST><<<blocks, threads>>>(d_out, sink, iters, 1.0f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  // MUFU work per iteration per SMSP: warps * CP * (8-EMU)/8 exp2 of 32 lanes at 4 lanes/clk
  const double xu = warps_per_smsp * CP * (8.0 - EMU) / 8.0 * 8.0;
  const double cyc = avg / iters;
  std::printf("%-22s W=%d CP=%3d EMU=%d: %7.1f cycles/iter  XU busy %5.1f %%  (%s)\n", name, warps_per_smsp, CP, EMU, cyc,
              100.0 * xu / cyc, cudaGetErrorString(e));
  cudaFree(d_out);
  cudaFree(sink);
}

int main() {
  run<128, 0, false>(1, "regs only");
  run<128, 1, false>(1, "regs only");
  run<128, 2, false>(1, "regs only");
  run<64, 0, false>(2, "regs only");
  run<64, 1, false>(2, "regs only");
  run<64, 2, false>(2, "regs only");
  run<64, 3, false>(2, "regs only");
  run<32, 0, false>(4, "regs only");
  run<32, 2, false>(4, "regs only");
  run<128, 0, true>(1, "tmem st");
  run<128, 1, true>(1, "tmem st");
  run<64, 0, true>(2, "tmem st");
  run<64, 1, true>(2, "tmem st");
  run<64, 2, true>(2, "tmem st");
  run<32, 0, true>(4, "tmem st");
  run<32, 1, true>(4, "tmem st");
  // one thread per row with two independent warps per sub-partition (two softmax groups)
  run<128, 0, true>(2, "tmem st");
  run<128, 1, true>(2, "tmem st");
  return 0;
}
