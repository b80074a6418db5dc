// vfa_ws_kernel instantiations (warp-specialised kernel for d = 128, Bc = 128, two query
// tiles per CTA; see ws_kernel.cuh) and its host launcher.
#include <atomic>
#include <string>

#include "vfa_internal.h"
#include "ws_kernel.cuh"

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

int launch_ws(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mr, const vfa::FwdArgs& a, cudaStream_t st) {
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
