// Semantics check of the CTA-pair (cta_group::2) tcgen05 MMAs used by the paired attention
// kernel: S = Q K^T with each CTA holding its own 128 query rows (A) and half of the key rows
// (B, N split), and O = P V with P in each CTA's TMEM (A) and half of V's columns per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o mma2sm_test mma2sm_test.cu -I../../paper_2604_12798_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace vfa;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_ss2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts2(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
// byte offset of (row, col) in a K-major SW128 tile of R rows (64-col chunks of R x 128 B)
__host__ __device__ inline uint32_t sw128_kmajor(int row, int col, int R) {
  const int chunk = col / 64, c = col % 64;
  return chunk * R * 128 + row * 128 + ((((c * 2) / 16) ^ (row & 7)) * 16) + ((c * 2) % 16);
}

// q: [2][128][128] (tile per CTA), k: [128][128], v: [128][128], outputs s: [2][128][128] f32, o: [2][128][128] f32
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    test_kernel(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v, float* s_out, float* o_out) {
  extern __shared__ uint8_t dyn[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;                    // 32 KB: this CTA's 128 query rows
  uint8_t* sK = sQ + 128 * 128 * 2;      // 16 KB: this CTA's 64 key rows
  uint8_t* sV = sK + 64 * 128 * 2;       // 16 KB: this CTA's 64 value columns (MN-major)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const uint32_t rank = cluster_rank();
  const int tid = threadIdx.x, warp = tid >> 5;
  // fill smem
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sQ + sw128_kmajor(r, c, 128)) = q[rank * 128 * 128 + i];
  }
  for (int i = tid; i < 64 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sK + sw128_kmajor(r, c, 64)) = k[(rank * 64 + r) * 128 + c];
  }
  for (int i = tid; i < 128 * 64; i += 128) {  // V[key j][col n] for n in this CTA's half; MN-major: row = key
    const int j = i / 64, n = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sV + sw128_kmajor(j, n, 128)) = v[j * 128 + rank * 64 + n];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
  if (rank == 0 && warp == 0) {
    const uint32_t idesc = make_idesc_bf16(256, 128, false, false);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t oq = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
      const uint32_t ok = ((kk >> 2) * (64 * 128) + (kk & 3) * 32) >> 4;
      if (elect_one())
        mma_ss2(tbase, (uint64_t(kHi) << 32) | ((smem_u32(sQ) >> 4) + (1u << 16) + oq),
                (uint64_t(kHi) << 32) | ((smem_u32(sK) >> 4) + (1u << 16) + ok), idesc, kk > 0);
      __syncwarp();
    }
    if (elect_one()) commit2(&bar);
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // read S (128 cols) from TMEM: thread = row
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  float sv[128];
  for (int c = 0; c < 4; ++c) {
    tmem_ld32(tbase + lane_off + c * 32, sv + c * 32);
    tmem_wait_ld();
  }
  for (int c = 0; c < 128; ++c) s_out[(rank * 128 + tid) * 128 + c] = sv[c];
  // P = bf16(S / 16) into TMEM columns [128, 192) (packed pairs), then O = P V at columns 256..383
  uint32_t u[64];
  for (int e = 0; e < 128; e += 2) u[e / 2] = pack_bf16x2(sv[e] / 16.f, sv[e + 1] / 16.f);
  for (int c = 0; c < 4; ++c) tmem_st16(tbase + lane_off + 128 + c * 16, u + c * 16);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 0) {
    const uint32_t idesc = make_idesc_bf16(256, 128, false, true);
    for (int kk = 0; kk < 8; ++kk) {
      if (elect_one())
        mma_ts2(tbase + 256, tbase + 128 + kk * 8, (uint64_t(kHi) << 32) | ((smem_u32(sV) >> 4) + kk * (2048 >> 4)),
                idesc, kk > 0);
      __syncwarp();
    }
    if (elect_one()) commit2(&bar);
    __syncwarp();
  }
  mbar_wait(&bar, 1);
  tc_fence_after();
  float ov[128];
  for (int c = 0; c < 4; ++c) {
    tmem_ld32(tbase + lane_off + 256 + c * 32, ov + c * 32);
    tmem_wait_ld();
  }
  for (int c = 0; c < 128; ++c) o_out[(rank * 128 + tid) * 128 + c] = ov[c];
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

int main() {
  const int n = 128 * 128;
  std::vector<__nv_bfloat16> hq(2 * n), hk(n), hv(n);
  std::vector<float> fq(2 * n), fk(n), fv(n);
  srand(1);
  auto rnd = [] { return (rand() / (float)RAND_MAX - 0.5f) * 2.f; };
  for (int i = 0; i < 2 * n; ++i) { hq[i] = __float2bfloat16(rnd()); fq[i] = __bfloat162float(hq[i]); }
  for (int i = 0; i < n; ++i) { hk[i] = __float2bfloat16(rnd()); fk[i] = __bfloat162float(hk[i]); }
  for (int i = 0; i < n; ++i) { hv[i] = __float2bfloat16(rnd()); fv[i] = __bfloat162float(hv[i]); }
  __nv_bfloat16 *dq, *dk, *dv;
  float *ds, *dout;
  cudaMalloc(&dq, 2 * n * 2); cudaMalloc(&dk, n * 2); cudaMalloc(&dv, n * 2);
  cudaMalloc(&ds, 2 * n * 4); cudaMalloc(&dout, 2 * n * 4);
  cudaMemcpy(dq, hq.data(), 2 * n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, hk.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), n * 2, cudaMemcpyHostToDevice);
  const int smem = 1024 + 128 * 128 * 2 + 2 * 64 * 128 * 2;
  cudaFuncSetAttribute(test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  test_kernel<<<2, 128, smem>>>(dq, dk, dv, ds, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> s(2 * n), o(2 * n);
  cudaMemcpy(s.data(), ds, 2 * n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data(), dout, 2 * n * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int t = 0; t < 2; ++t)
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        double ref = 0;
        for (int x = 0; x < 128; ++x) ref += fq[t * n + r * 128 + x] * fk[c * 128 + x];
        es = fmax(es, fabs(ref - s[t * n + r * 128 + c]));
      }
  for (int t = 0; t < 2; ++t)
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        double ref = 0;
        for (int j = 0; j < 128; ++j) ref += (double)__bfloat162float(__float2bfloat16(s[t * n + r * 128 + j] / 16.f)) * fv[j * 128 + c];
        eo = fmax(eo, fabs(ref - o[t * n + r * 128 + c]));
      }
  printf("S max err %.3e, O max err %.3e\n", es, eo);
  return 0;
}
