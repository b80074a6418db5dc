// Microbenchmark: tcgen05.mma issue rate per SM for the attention kernel's operand modes
// (one CTA per SM, back-to-back MMAs of K = 16 into one accumulator, no other smem traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu -I../../paper_2604_12798_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace vfa;

// MODE 0: SS, A and B K-major (the QK^T of the kernel), N = NN
// MODE 1: TS, A from TMEM, B K-major (QK^T with Q resident in TMEM), N = NN
// MODE 2: TS, A from TMEM, B MN-major (the PV of the kernel), N = NN
// BG: background traffic from warps 1-8 while warp 0 issues: 0 none, 1 tcgen05.ld x32 loops
// (softmax S reads), 2 tcgen05.st x16 loops (P writes), 3 shared-memory reads (ld.shared.v4),
// 4 bulk async copies global -> smem (32 KB each, back to back: TMA-like write traffic)
template <int MODE, int NN, int BG = 0>
__global__ void __launch_bounds__(288, 1) kern(long long* out, int iters, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar;
  const int warp = threadIdx.x >> 5;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cbar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp == 1 && BG == 4) {
    uint32_t ph = 0;
    int n = 0;
    while (!done) {
      if ((threadIdx.x & 31) == 0) {
        mbar_arrive_expect_tx(&cbar, 32768);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(base + 65536)),
                     "l"(gsrc + (n & 63) * 32768), "r"(32768), "r"(smem_u32(&cbar))
                     : "memory");
      }
      __syncwarp();
      mbar_wait(&cbar, ph);
      ph ^= 1;
      ++n;
    }
    if (threadIdx.x == 32) out[148 + blockIdx.x] = n;
  } else if (warp > 0 && BG != 0 && BG != 4) {
    const uint32_t ta = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 384 + ((warp - 1) >> 2) * 32;
    float acc = 0.f;
    uint32_t u[16];
    for (int e = 0; e < 16; ++e) u[e] = e;
    const uint4* sp = reinterpret_cast<const uint4*>(base) + (threadIdx.x & 255);
    while (!done) {
      if (BG == 1) {
        float v[32];
        tmem_ld32(ta, v);
        tmem_wait_ld();
        reg_fence32(v);
        acc += v[0];
      } else if (BG == 2) {
        tmem_st16(ta, u);
        tmem_wait_st();
      } else {
        uint4 x = sp[0];
        uint4 y = sp[256];
        acc += __uint_as_float(x.x ^ y.w);
      }
    }
    if (acc == 12345.f) out[0] = 1;
  }
  if (warp == 0) {
    constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
    const uint32_t a_lo = (smem_u32(base) >> 4) | (1u << 16);
    const uint32_t b_lo_k = (smem_u32(base + 32768) >> 4) | (1u << 16);
    const uint32_t b_lo_mn = (smem_u32(base + 32768) >> 4) | (static_cast<uint32_t>((128 * 128) >> 4) << 16);
    constexpr uint32_t idesc_k = make_idesc_bf16(128, NN, false, false);
    constexpr uint32_t idesc_mn = make_idesc_bf16(128, NN, false, true);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t oa = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
        const uint32_t ob = ((kk >> 2) * (NN * 128) + (kk & 3) * 32) >> 4;
        if (elect_one()) {
          if (MODE == 0)
            mma_ss(tbase, (static_cast<uint64_t>(kHi) << 32) | (a_lo + oa), (static_cast<uint64_t>(kHi) << 32) | (b_lo_k + ob),
                   idesc_k, (it | kk) ? 1u : 0u);
          else if (MODE == 1)
            mma_ts(tbase, tbase + 256 + kk * 8, (static_cast<uint64_t>(kHi) << 32) | (b_lo_k + ob), idesc_k,
                   (it | kk) ? 1u : 0u);
          else
            mma_ts(tbase, tbase + 256 + kk * 8, (static_cast<uint64_t>(kHi) << 32) | (b_lo_mn + kk * (2048 >> 4)),
                   idesc_mn, (it | kk) ? 1u : 0u);
        }
        __syncwarp();
      }
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 0) done = 1;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int MODE, int NN, int BG = 0>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8 * 296);
  uint8_t* g;
  cudaMalloc(&g, 64 * 32768);
  cudaMemset(g, 0, 64 * 32768);
  auto k = kern<MODE, NN, BG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4000;
  k<<<148, 288, 100 * 1024>>>(d, 10, g);
  k<<<148, 288, 100 * 1024>>>(d, iters, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long nc[148];
  cudaMemcpy(nc, d + 148, sizeof(nc), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148;
  const double per = cyc / (iters * 8.0);
  const double floor = 128.0 * NN / 256.0;
  printf("%-34s BG=%d N=%3d  %7.1f cycles/MMA  (floor %5.1f, %5.1f%%)  smem operand %6.1f B/clk", name, BG, NN, per,
         floor, 100.0 * floor / per, (MODE == 0 ? (128 * 32.0 + NN * 32.0) : NN * 32.0) / per);
  if (BG == 4) printf("  bulk-copy writes %6.1f B/clk", nc[0] * 32768.0 / cyc);
  printf("  (%s)\n", cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(g);
}

int main() {
  run<0, 128>("SS  (QK^T, Q and K in smem)");
  run<1, 128>("TS  (QK^T, Q in TMEM)");
  run<2, 128>("TS  (PV, P in TMEM, V MN-major)");
  run<0, 64>("SS  (QK^T, Q and K in smem)");
  run<1, 64>("TS  (QK^T, Q in TMEM)");
  for (int i = 0; i < 1; ++i) {
    run<0, 128, 1>("SS  (QK^T) + TMEM loads");
    run<1, 128, 1>("TS  (QK^T) + TMEM loads");
    run<2, 128, 1>("TS  (PV) + TMEM loads");
    run<0, 128, 2>("SS  (QK^T) + TMEM stores");
    run<2, 128, 2>("TS  (PV) + TMEM stores");
    run<0, 128, 3>("SS  (QK^T) + smem reads");
    run<1, 128, 3>("TS  (QK^T) + smem reads");
    run<0, 128, 4>("SS  (QK^T) + bulk copies");
    run<1, 128, 4>("TS  (QK^T) + bulk copies");
    run<2, 128, 4>("TS  (PV) + bulk copies");
  }
  return 0;
}
