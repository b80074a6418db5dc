// Host-side launch templates for vfa_fwd_kernel, included by the per-variant TUs
// (fwd_<variant>.cu). Each TU instantiates one MODE for every head dim / key block /
// query-tiles-per-CTA / softmax split.
#pragma once
#include <atomic>
#include <string>

#include "vfa_internal.h"
#include "vfa_kernel.cuh"

namespace vfa_host {

template <int D, int BC, int NQ, int MODE, int SPLIT, int PAIR = 1>
int launch_fwd(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
               const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t stream) {
  using C = vfa::Cfg<D, BC, NQ, SPLIT, MODE, PAIR>;
  auto kern = vfa::vfa_fwd_kernel<D, BC, NQ, MODE, SPLIT, PAIR>;
  // cudaFuncSetAttribute applies to the current device only: one flag bit per device, set
  // after the attribute is in place (a racing second setter is harmless)
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return vfa_host::fail(VFA_ERR_CUDA, "cudaGetDevice failed");
  const unsigned long long bit = 1ull << dev;
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return vfa_host::fail(VFA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return vfa_host::fail(VFA_ERR_CUDA, std::string("cudaFuncGetAttributes: ") + cudaGetErrorString(e));
    if (C::kRegBudget > fa.numRegs * C::kThreads)
      return vfa_host::fail(VFA_ERR_CUDA, "setmaxnreg budget " + std::to_string(C::kRegBudget) + " exceeds the launch allocation " +
                                    std::to_string(fa.numRegs * C::kThreads) + " (would deadlock)");
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  const long long units = static_cast<long long>(args.B) * args.Hkv * args.units_per_kvh;
  if (units <= 0) return VFA_OK;
  cudaError_t e;
  if constexpr (PAIR == 2) {
    // one cluster of two CTAs per unit (the unit's two query heads, one per CTA)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mr, args);
    if (e == cudaSuccess) e = cudaGetLastError();
  } else {
    kern<<<static_cast<unsigned>(units), C::kThreads, C::kSmem, stream>>>(mq, mk, mv, mr, args);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return vfa_host::fail(VFA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

// Softmax column split per variant (params.softmax_split = 0), measured best on B200
// (profiles/ab_r01_split.txt): VFA's frozen blocks need no cross-thread exchange, so all
// warps serving both tiles wins; FA / VSA exchange a row max on every block, which per-tile
// warp sets overlap with the other tile's work. One query tile per CTA: always 4.
constexpr int default_split(int mode) {
  return mode == vfa::kVFA ? VFA_SPLIT_VFA : (mode == vfa::kFA ? VFA_SPLIT_FA : VFA_SPLIT_VSA);
}

template <int D, int BC, int NQ, int MODE>
int dispatch_split(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                   const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st) {
  const int split = p->softmax_split ? p->softmax_split : default_split(MODE);
  if constexpr (BC == 32) {
    // 32-column S tiles: a part needs >= 16 columns, so 2 threads per row (two query tiles) or
    // one thread per row; a requested split of 4 runs as 2
    if (NQ == 2 && split != 1) return launch_fwd<D, BC, NQ, MODE, 2>(p, mq, mk, mv, mr, args, st);
    return launch_fwd<D, BC, NQ, MODE, 1>(p, mq, mk, mv, mr, args, st);
  } else {
    if (split == 1) return launch_fwd<D, BC, NQ, MODE, 1>(p, mq, mk, mv, mr, args, st);
    if (NQ == 2 && split == 2) return launch_fwd<D, BC, NQ, MODE, 2>(p, mq, mk, mv, mr, args, st);
    return launch_fwd<D, BC, NQ, MODE, 4>(p, mq, mk, mv, mr, args, st);
  }
}

template <int MODE>
int launch_mode(const VfaParams* p, int nq, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                const CUtensorMap& mr, const vfa::FwdArgs& a, cudaStream_t st) {
  // head_dim 32 runs on the D = 64 kernels: TMA zero-fills columns 32..63 of every Q / K / V
  // tile (exact: zero columns add nothing to QK^T, and PV's extra O columns are not stored)
  const int D = p->head_dim <= 64 ? 64 : 128, BC = p->k_block;
  if (a.pair == 2) {  // CTA pairs (d = 128): K/V shared by M = 256 MMAs; 2 or 1 query tiles per CTA
    if (p->softmax_split == 1) {  // one thread per row
      if (a.heads_per_unit == 4) {
        if (BC == 128) return launch_fwd<128, 128, 2, MODE, 1, 2>(p, mq, mk, mv, mr, a, st);
        return launch_fwd<128, 64, 2, MODE, 1, 2>(p, mq, mk, mv, mr, a, st);
      }
      if (BC == 128) return launch_fwd<128, 128, 1, MODE, 1, 2>(p, mq, mk, mv, mr, a, st);
      return launch_fwd<128, 64, 1, MODE, 1, 2>(p, mq, mk, mv, mr, a, st);
    }
    if (a.heads_per_unit == 4) {
      if (BC == 128) return launch_fwd<128, 128, 2, MODE, 4, 2>(p, mq, mk, mv, mr, a, st);
      return launch_fwd<128, 64, 2, MODE, 4, 2>(p, mq, mk, mv, mr, a, st);
    }
    if (BC == 128) return launch_fwd<128, 128, 1, MODE, 4, 2>(p, mq, mk, mv, mr, a, st);
    return launch_fwd<128, 64, 1, MODE, 4, 2>(p, mq, mk, mv, mr, a, st);
  }
#define VFA_NQ(DD, BB)                                                                          \
  return nq == 2 ? dispatch_split<DD, BB, 2, MODE>(p, mq, mk, mv, mr, a, st)                    \
                 : dispatch_split<DD, BB, 1, MODE>(p, mq, mk, mv, mr, a, st)
  if (D == 128 && BC == 128) VFA_NQ(128, 128);
  if (D == 128 && BC == 64) VFA_NQ(128, 64);
  if (D == 128 && BC == 32) VFA_NQ(128, 32);
  if (D == 64 && BC == 128) VFA_NQ(64, 128);
  if (D == 64 && BC == 32) VFA_NQ(64, 32);
  VFA_NQ(64, 64);
#undef VFA_NQ
}

}  // namespace vfa_host
