// vfa_ws_kernel instantiations (warp-specialised kernel for d = 128, Bc = 128, two query
// tiles per CTA; see ws_kernel.cuh) and its host launcher.
#include <atomic>
#include <string>

#include "vfa_internal.h"
#include "ws_kernel.cuh"
#include "ws1_kernel.cuh"

namespace vfa_host {

template <int MODE>
static int launch_ws_mode(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mr,
                          const vfa::FwdArgs& args, cudaStream_t stream) {
  using C = vfa::WsCfg;
  auto kern = vfa::vfa_ws_kernel<MODE>;
  static std::atomic<unsigned long long> attr_set{0};  // per device (see fwd_dispatch.cuh)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return fail(VFA_ERR_CUDA, "cudaGetDevice failed");
  const unsigned long long bit = 1ull << dev;
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncGetAttributes: ") + cudaGetErrorString(e));
    constexpr int kBudget = C::kRegBudget;
    if (kBudget > fa.numRegs * C::kThreads)
      return fail(VFA_ERR_CUDA, "setmaxnreg budget " + std::to_string(kBudget) + " exceeds the launch allocation " +
                                    std::to_string(fa.numRegs * C::kThreads) + " (would deadlock)");
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  const long long units = static_cast<long long>(args.B) * args.Hkv * args.units_per_kvh;
  if (units <= 0) return VFA_OK;
  kern<<<static_cast<unsigned>(units), C::kThreads, C::kSmem, stream>>>(mq, mk, mv, mr, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

template <int MODE>
static int launch_ws1_mode(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mr,
                           const vfa::FwdArgs& args, cudaStream_t stream) {
  using C = vfa::Ws1Cfg;
  auto kern = vfa::vfa_ws1_kernel<MODE>;
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return fail(VFA_ERR_CUDA, "cudaGetDevice failed");
  const unsigned long long bit = 1ull << dev;
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncGetAttributes: ") + cudaGetErrorString(e));
    if (C::kRegBudget > fa.numRegs * C::kThreads)
      return fail(VFA_ERR_CUDA, "setmaxnreg budget " + std::to_string(C::kRegBudget) + " exceeds the launch allocation " +
                                    std::to_string(fa.numRegs * C::kThreads) + " (would deadlock)");
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  const long long units = static_cast<long long>(args.B) * args.Hkv * args.units_per_kvh;
  if (units <= 0) return VFA_OK;
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mr, args);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

// Kernel per variant: the frozen-max variants (VFA, VSA) run the decoupled one-tile kernel
// (ws1_kernel.cuh: its two softmax groups only synchronise on exact-update blocks, the few
// sink / local ones); FA, where every block is an exact update that would serialise those
// groups, runs the ping-pong kernel (ws_kernel.cuh). profiles/ab_r02_ws1.txt.

int launch_ws(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mr, const vfa::FwdArgs& a, cudaStream_t st) {
  if (ws_uses_ws1(p)) {
    switch (p->variant) {
      case VFA_VARIANT_FA:
        return launch_ws1_mode<vfa::kFA>(mq, mk, mv, mr, a, st);
      case VFA_VARIANT_VFA:
        return launch_ws1_mode<vfa::kVFA>(mq, mk, mv, mr, a, st);
      case VFA_VARIANT_VSA:
        return launch_ws1_mode<vfa::kVSA>(mq, mk, mv, mr, a, st);
      default:
        return fail(VFA_ERR_CONFIG, "warp-specialised kernel: unsupported variant");
    }
  }
  switch (p->variant) {
    case VFA_VARIANT_FA:
      return launch_ws_mode<vfa::kFA>(mq, mk, mv, mr, a, st);
    case VFA_VARIANT_VFA:
      return launch_ws_mode<vfa::kVFA>(mq, mk, mv, mr, a, st);
    case VFA_VARIANT_VSA:
      return launch_ws_mode<vfa::kVSA>(mq, mk, mv, mr, a, st);
    default:
      return fail(VFA_ERR_CONFIG, "warp-specialised kernel: unsupported variant");
  }
}

}  // namespace vfa_host
