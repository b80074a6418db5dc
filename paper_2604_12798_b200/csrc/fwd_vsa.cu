// vfa_fwd_kernel instantiations for variant vsa (vfa::kVSA); see vfa_kernel.cuh.
#include "fwd_dispatch.cuh"

namespace vfa_host {
int launch_vsa(const VfaParams* p, int nq, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mr, const vfa::FwdArgs& a, cudaStream_t st) {
  return launch_mode<vfa::kVSA>(p, nq, mq, mk, mv, mr, a, st);
}
}  // namespace vfa_host
