// Declarations shared by the host translation units of libvfa_b200.so (not part of the
// C ABI): the error channel and the per-variant kernel launchers (one TU each, so the
// kernel instantiations compile in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/vfa_b200.h"

namespace vfa {
struct FwdArgs;
}

namespace vfa_host {

// Sets the thread-local message returned by vfa_last_error() and returns `code`.
int fail(int code, const std::string& msg);

// Launches vfa_fwd_kernel for one variant (params.variant), dispatching head dim, key
// block, query tiles per CTA (nq) and the softmax split. Defined in fwd_<variant>.cu.
using LaunchFn = int (*)(const VfaParams* p, int nq, const CUtensorMap& mq, const CUtensorMap& mk,
                         const CUtensorMap& mv, const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st);
int launch_fa(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
              const vfa::FwdArgs&, cudaStream_t);
int launch_vfa(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
               const vfa::FwdArgs&, cudaStream_t);
int launch_vsa(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
               const vfa::FwdArgs&, cudaStream_t);
int launch_blasst(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                  const CUtensorMap&, const vfa::FwdArgs&, cudaStream_t);
int launch_blasst_fa4(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                      const CUtensorMap&, const vfa::FwdArgs&, cudaStream_t);
int launch_blasst_rowskip(const VfaParams*, int, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                          const CUtensorMap&, const vfa::FwdArgs&, cudaStream_t);
// Warp-specialised kernels (ws_kernel.cuh, ws1_kernel.cuh) for d = 128, k_block = q_block = 128,
// two query tiles per CTA / cluster; variants FA / VFA / VSA. Defined in fwd_ws.cu.
#ifndef VFA_WS_KIND
#define VFA_WS_KIND -1  // -1: FA on the ping-pong kernel, VFA / VSA on the decoupled one; 0 / 1: all on one
#endif
#ifndef VFA_WS1_PAIR
#define VFA_WS1_PAIR 0  // decoupled kernel with pair MMAs (cta_group::2): each CTA holds half of every K / V tile
#endif
inline bool ws_uses_ws1(const VfaParams* p) { return VFA_WS_KIND >= 0 ? VFA_WS_KIND == 1 : p->variant != VFA_VARIANT_FA; }
int launch_ws(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st);

}  // namespace vfa_host
