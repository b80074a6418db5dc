// vfa_fwd_kernel instantiations for variant vfa (vfa::kVFA); see vfa_kernel.cuh.
#include "fwd_dispatch.cuh"

namespace vfa_host {
int launch_vfa(const VfaParams* p, int nq, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mr, const vfa::FwdArgs& a, cudaStream_t st) {
  return launch_mode<vfa::kVFA>(p, nq, mq, mk, mv, mr, a, st);
}
}  // namespace vfa_host
