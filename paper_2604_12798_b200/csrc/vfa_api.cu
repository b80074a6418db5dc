// C ABI of libvfa_b200.so (include/vfa_b200.h): validation, tensor maps, the key-block
// representation kernel launch, per-variant dispatch of the attention kernel, and the
// host-resident pipelined forward. Device code lives in vfa_kernel.cuh.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "vfa_internal.h"
#include "vfa_kernel.cuh"


// ====================================================================================
// Host side
// ====================================================================================
namespace vfa_host {
namespace {
thread_local std::string g_last_error;
}  // namespace

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace vfa_host

namespace {
using vfa_host::fail;
long long* g_debug_trace = nullptr;  // debug only: set by vfa_debug_trace()

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 4-D bf16 tensor [B, H, L, D] (innermost D) with element strides; box {64, box_rows, 1, 1}.
bool make_map(CUtensorMap* map, const void* base, int64_t B, int64_t H, int64_t L, int64_t D, int64_t sb,
              int64_t sh, int64_t sr, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(B)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(sr * 2), static_cast<cuuint64_t>(sh * 2),
                           static_cast<cuuint64_t>(sb * 2)};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int64_t n_key_blocks(const VfaParams* p) { return p->seq_k / p->k_block; }
int64_t n_reprs(const VfaParams* p) {
  int64_t tc = n_key_blocks(p);
  return (p->tc1 > 0 && p->tc1 < tc) ? p->tc1 : tc;
}

// Block representations of `rows`-row blocks of x [B, H, L, D] (strides sb, sh, sr) for blocks
// [jb0, nblk): out [B, H, nblk, D] bf16 contiguous.
int launch_block_repr(const void* x, int64_t B, int64_t H, const int64_t* strides, int D, int rows, int nblk,
                      int kind, void* out, int jb0, cudaStream_t st) {
  if (nblk <= jb0) return VFA_OK;
  dim3 grid((nblk - jb0 + 3) / 4, static_cast<unsigned>(H), static_cast<unsigned>(B));
  const auto* xp = static_cast<const __nv_bfloat16*>(x);
  auto* op = static_cast<__nv_bfloat16*>(out);
  if (D == 128)
    vfa::krepr_kernel<128><<<grid, 128, 0, st>>>(xp, strides[0], strides[1], strides[2], static_cast<int>(H), rows,
                                                nblk, kind, op, jb0);
  else if (D == 64)
    vfa::krepr_kernel<64><<<grid, 128, 0, st>>>(xp, strides[0], strides[1], strides[2], static_cast<int>(H), rows,
                                               nblk, kind, op, jb0);
  else
    vfa::krepr_kernel<32><<<grid, 128, 0, st>>>(xp, strides[0], strides[1], strides[2], static_cast<int>(H), rows,
                                               nblk, kind, op, jb0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("krepr launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

int launch_krepr(const VfaParams* p, const void* k, void* out, cudaStream_t st, int jb0 = 0) {
  return launch_block_repr(k, p->batch, p->heads_kv, p->k_stride, static_cast<int>(p->head_dim), p->k_block,
                           static_cast<int>(n_reprs(p)), p->kind, out, jb0, st);
}

// block-wise qkind (src/vfa.py:69-76): the query tile's representation kind as a block_repr kind
int qkind_as_block_kind(int qkind) {
  return qkind == 1 ? VFA_KREPR_K_ABSMAX_UNSIGNED : (qkind == 2 ? VFA_KREPR_SABSMAX : VFA_KREPR_K_MEAN);
}

// workspace layout: [key representations][query representations][per-tile seeds] (the last two
// only for the block-wise query representations)
size_t ws_krepr_bytes(const VfaParams* p) {
  return static_cast<size_t>(p->batch * p->heads_kv * n_reprs(p) * p->head_dim * 2 + 255) / 256 * 256;
}
size_t ws_qrepr_bytes(const VfaParams* p) {
  return static_cast<size_t>(p->batch * p->heads_q * (p->seq_q / p->q_block) * p->head_dim * 2 + 255) / 256 * 256;
}
size_t ws_m0_bytes(const VfaParams* p) { return static_cast<size_t>(p->batch * p->heads_q * (p->seq_q / p->q_block) * 4); }

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

#ifndef VFA_WS_ENABLE
#define VFA_WS_ENABLE 1  // 0: every shape on vfa_fwd_kernel (experiments)
#endif
#ifndef VFA_PAIR_NQ2
#define VFA_PAIR_NQ2 1
#endif
// CTA pairs off by default: measured slower than one CTA per unit (profiles/ab_r01_pair.txt);
// cta_pair = 2 selects them per call
#ifndef VFA_PAIR_DEFAULT
#define VFA_PAIR_DEFAULT 0
#endif
// Shapes the warp-specialised kernel (ws_kernel.cuh) serves when a CTA holds two query tiles:
// d = 128, 128-row query / key blocks, default softmax layout, FA / VFA / VSA without the
// monitor. (Debug outputs -- state trace, row rebase, timeline -- also route to vfa_fwd_kernel.)
bool ws_eligible(const VfaParams* p) {
  return VFA_WS_ENABLE && p->head_dim == 128 && p->k_block == 128 && p->q_block == 128 && p->softmax_split == 0 &&
         !p->monitor && p->cta_pair != 2 && p->variant <= VFA_VARIANT_VSA;
}

bool default_pair(int variant) { return VFA_PAIR_DEFAULT != 0 && variant >= 0; }

void reset_counters(long long* stats, unsigned int* status, cudaStream_t st) {
  if (stats) cudaMemsetAsync(stats, 0, sizeof(long long) * VFA_STAT_COUNT, st);
  if (status) {
    cudaMemsetAsync(status, 0, sizeof(unsigned) * VFA_STATUS_COUNT, st);
    cudaMemsetAsync(status + VFA_STATUS_UNDERFLOW_ROW, 0xff, sizeof(unsigned) * 2, st);
  }
}

int forward_impl(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                 unsigned char* skip_trace, int* stab_block, cudaStream_t st, bool zero_counters,
                 long long row_base, void* seed_ws = nullptr, const float* row_bias = nullptr,
                 float* m_trace = nullptr);

}  // namespace

extern "C" {

int vfa_check_params(const VfaParams* p) {
  if (!p) return fail(VFA_ERR_CONFIG, "params is NULL");
  if (p->variant < VFA_VARIANT_FA || p->variant > VFA_VARIANT_BLASST_ROWSKIP)
    return fail(VFA_ERR_CONFIG, "variant must be 0 (fa), 1 (vfa), 2 (vsa), 3 (blasst), 4 (blasst_fa4) or 5 (blasst_rowskip)");
  if (p->kind < VFA_KREPR_SABSMAX || p->kind > VFA_KREPR_K_ABSMAX_UNSIGNED)
    return fail(VFA_ERR_CONFIG, "unknown key representation");
  if (p->qkind < 0 || p->qkind > 3) return fail(VFA_ERR_CONFIG, "unknown query representation");
  // a 128-row tcgen05 tile holds one reference query block; q_block < 128 leaves rows idle
  // (same schedule / statistics as the reference at that block size, 128 / q_block x the work)
  if (p->q_block != 128 && p->q_block != 64 && p->q_block != 32 && p->q_block != 16)
    return fail(VFA_ERR_CONFIG, "q_block must be 16, 32, 64 or 128 (tcgen05 M = 128 tiles)");
  if (p->k_block != 32 && p->k_block != 64 && p->k_block != 128)
    return fail(VFA_ERR_CONFIG, "k_block must be 32, 64 or 128");
  if (p->head_dim != 32 && p->head_dim != 64 && p->head_dim != 128)
    return fail(VFA_ERR_CONFIG, "head_dim must be 32, 64 or 128");
  if (p->n_sink < 0 || p->n_local < 0) return fail(VFA_ERR_CONFIG, "n_sink and n_local must be >= 0");
  if (p->softmax_split != 0 && p->softmax_split != 1 && p->softmax_split != 2 && p->softmax_split != 4)
    return fail(VFA_ERR_CONFIG, "softmax_split must be 0 (auto), 1, 2 or 4");
  if (p->cta_pair < 0 || p->cta_pair > 2) return fail(VFA_ERR_CONFIG, "cta_pair must be 0 (auto), 1 (off) or 2 (on)");
  if (p->variant >= VFA_VARIANT_VSA && p->lam > 1.0) return fail(VFA_ERR_CONFIG, "lambda must be in (0, 1]");
  if (!(p->tau >= 0.0)) return fail(VFA_ERR_CONFIG, "tau must be >= 0");  // src/sparse.py:52-53 (NaN rejected)
  // 0 selects 1/sqrt(d); the kernels fold the scale in after the row max, which needs scale > 0
  if (!(p->scale >= 0.0) || std::isinf(p->scale))
    return fail(VFA_ERR_CONFIG, "scale must be a positive finite number (0 = 1/sqrt(head_dim))");
  if (p->batch < 1 || p->heads_q < 1 || p->heads_kv < 1 || p->seq_q < 1 || p->seq_k < 1)
    return fail(VFA_ERR_DATA, "all dimensions must be >= 1");
  if (p->heads_q % p->heads_kv) return fail(VFA_ERR_DATA, "heads_q must be a multiple of heads_kv");
  if (p->seq_q % p->q_block)
    return fail(VFA_ERR_DATA, "seq_len_q=" + std::to_string(p->seq_q) + " not divisible by q_block=" +
                                  std::to_string(p->q_block));
  if (p->seq_k % p->k_block)
    return fail(VFA_ERR_DATA, "seq_len_k=" + std::to_string(p->seq_k) + " not divisible by k_block=" +
                                  std::to_string(p->k_block));
  if (p->causal && p->seq_q != p->seq_k) return fail(VFA_ERR_DATA, "causal masking requires N_q == N_k");
  if (p->tc1 < 0 || p->tc1 > n_key_blocks(p))
    return fail(VFA_ERR_CONFIG, "tc1 must be in 1..T_c (0 = all)");
  const int64_t* strides[4] = {p->q_stride, p->k_stride, p->v_stride, p->o_stride};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 3; ++j)
      if (strides[i][j] % 8 != 0 || strides[i][j] < 0)
        return fail(VFA_ERR_DATA, "strides must be non-negative multiples of 8 elements (16 bytes)");
  if (p->seq_q * p->heads_q * p->batch >= 0xffffffffLL) return fail(VFA_ERR_DATA, "too many rows");
  return VFA_OK;
}

size_t vfa_workspace_bytes(const VfaParams* p) {
  if (!p || vfa_check_params(p) != VFA_OK) return 0;
  size_t n = ws_krepr_bytes(p) + 256;
  if (p->qkind != 0) n += ws_qrepr_bytes(p) + ws_m0_bytes(p);
  return n;
}

int vfa_krepr_range(const VfaParams* p, const void* k, void* out, int first_block, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!k || !out) return fail(VFA_ERR_DATA, "NULL pointer");
  if (first_block < 0 || first_block > n_reprs(p)) return fail(VFA_ERR_CONFIG, "first_block out of range");
  return launch_krepr(p, k, out, static_cast<cudaStream_t>(stream), first_block);
}

int vfa_krepr(const VfaParams* p, const void* k, void* out, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!k || !out) return fail(VFA_ERR_DATA, "NULL pointer");
  return launch_krepr(p, k, out, static_cast<cudaStream_t>(stream));
}

int vfa_fwd(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
            void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
            unsigned char* skip_trace, int* stab_block, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q || !k || !v || !o) return fail(VFA_ERR_DATA, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(VFA_ERR_DATA, "tensors must be 16-byte aligned");
  return forward_impl(p, q, k, v, o, lse, workspace, workspace_bytes, stats, status, skip_trace, stab_block,
                      static_cast<cudaStream_t>(stream), true, 0);
}

int vfa_fwd_rebased(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                    void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                    const float* row_bias, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q || !k || !v || !o || !row_bias) return fail(VFA_ERR_DATA, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(VFA_ERR_DATA, "tensors must be 16-byte aligned");
  return forward_impl(p, q, k, v, o, lse, workspace, workspace_bytes, stats, status, nullptr, nullptr,
                      static_cast<cudaStream_t>(stream), true, 0, nullptr, row_bias);
}

int vfa_fwd_state_trace(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                        void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                        int* stab_block, float* m_trace, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q || !k || !v || !o || !m_trace) return fail(VFA_ERR_DATA, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(VFA_ERR_DATA, "tensors must be 16-byte aligned");
  return forward_impl(p, q, k, v, o, lse, workspace, workspace_bytes, stats, status, nullptr, stab_block,
                      static_cast<cudaStream_t>(stream), true, 0, nullptr, nullptr, m_trace);
}

}  // extern "C"

namespace {
// The forward on device buffers. zero_counters: reset stats/status first (false when a
// caller accumulates several launches into one status word, e.g. vfa_fwd_host's chunks).
int forward_impl(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                 unsigned char* skip_trace, int* stab_block, cudaStream_t st, bool zero_counters,
                 long long row_base, void* seed_ws, const float* row_bias, float* m_trace) {
  int rc = VFA_OK;
  // m-initialisation belongs to the frozen-max variants; FA and the BLASST family start at -inf
  const bool minit = (p->variant == VFA_VARIANT_VFA || p->variant == VFA_VARIANT_VSA) && p->use_m_init;
  const int64_t nrep = n_reprs(p);
  if (minit) {
    if (!workspace || workspace_bytes < vfa_workspace_bytes(p) || !aligned16(workspace))
      return fail(VFA_ERR_DATA, "workspace too small or misaligned");
  }
  const int D = static_cast<int>(p->head_dim), BC = p->k_block;
  const int group = static_cast<int>(p->heads_q / p->heads_kv);
#ifndef VFA_FORCE_NQ1
#define VFA_FORCE_NQ1 0  // experiments: one query tile per CTA even for even GQA groups
#endif
  const int nq = (group % 2 == 0 && !VFA_FORCE_NQ1) ? 2 : 1;
  // CTA pairs (cta_pair = 2, or auto): the unit's two query heads on two SMs sharing each K/V
  // tile through M = 256 MMAs; needs an even GQA group and d = 128
  const bool pair_ok = nq == 2 && D == 128 && p->q_block == 128 && BC >= 64;
  const int pair = (pair_ok && (p->cta_pair == 2 || (p->cta_pair == 0 && default_pair(p->variant)))) ? 2 : 1;
  // a pair holds two query tiles per CTA (four heads per cluster, the tiles ping-pong on the
  // tensor pipe as in the single-CTA kernel) when the GQA group allows, else one
  const int pair_nq = (VFA_PAIR_NQ2 && group % 4 == 0) ? 2 : 1;

  // warp-specialised kernels (d = Bc = 128, two query tiles per unit); the decoupled kernel's
  // pair-MMA build splits K-like tiles by rows between the two CTAs
  const bool ws_path = ws_eligible(p) && nq == 2 && pair == 1 && !m_trace && !row_bias;
  const int kbox = (ws_path && VFA_WS1_PAIR && vfa_host::ws_uses_ws1(p)) ? BC / 2 : BC / pair;
  CUtensorMap mq, mk, mv, mr;
  if (!make_map(&mq, q, p->batch, p->heads_q, p->seq_q, D, p->q_stride[0], p->q_stride[1], p->q_stride[2], 128) ||
      !make_map(&mk, k, p->batch, p->heads_kv, p->seq_k, D, p->k_stride[0], p->k_stride[1], p->k_stride[2], kbox) ||
      !make_map(&mv, v, p->batch, p->heads_kv, p->seq_k, D, p->v_stride[0], p->v_stride[1], p->v_stride[2], BC))
    return fail(VFA_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (minit) {
    if (!make_map(&mr, workspace, p->batch, p->heads_kv, nrep, D, p->heads_kv * nrep * D, nrep * D, D, kbox))
      return fail(VFA_ERR_CUDA, "cuTensorMapEncodeTiled failed (krepr)");
    if (!p->krepr_precomputed) {
      rc = launch_krepr(p, k, workspace, st);
      if (rc) return rc;
    }
  } else {
    mr = mk;
  }
  const float* m0_tile = nullptr;
  if (minit && p->qkind != 0) {
    // block-wise query representation: per query tile, seed = max_j qrepr . krepr_j
    // (seed_ws: a per-call seed area, so launches sharing one K/V workspace on different
    // streams do not overwrite each other's query representations and seeds)
    uint8_t* qrep = seed_ws ? static_cast<uint8_t*>(seed_ws) : static_cast<uint8_t*>(workspace) + ws_krepr_bytes(p);
    float* m0 = reinterpret_cast<float*>(qrep + ws_qrepr_bytes(p));
    const int tr = static_cast<int>(p->seq_q / p->q_block);
    rc = launch_block_repr(q, p->batch, p->heads_q, p->q_stride, D, p->q_block, tr, qkind_as_block_kind(p->qkind), qrep, 0,
                           st);
    if (rc) return rc;
    dim3 grid((tr + 3) / 4, static_cast<unsigned>(p->heads_q), static_cast<unsigned>(p->batch));
    const auto* qr = reinterpret_cast<const __nv_bfloat16*>(qrep);
    const auto* kr = static_cast<const __nv_bfloat16*>(workspace);
    const int tc = static_cast<int>(n_key_blocks(p));
    if (D == 128)
      vfa::minit_block_kernel<128><<<grid, 128, 0, st>>>(qr, kr, static_cast<int>(p->heads_q),
                                                         static_cast<int>(p->heads_kv), tr, p->q_block,
                                                         static_cast<int>(nrep), BC, tc, p->causal ? 1 : 0, m0);
    else if (D == 64)
      vfa::minit_block_kernel<64><<<grid, 128, 0, st>>>(qr, kr, static_cast<int>(p->heads_q),
                                                        static_cast<int>(p->heads_kv), tr, p->q_block,
                                                        static_cast<int>(nrep), BC, tc, p->causal ? 1 : 0, m0);
    else
      vfa::minit_block_kernel<32><<<grid, 128, 0, st>>>(qr, kr, static_cast<int>(p->heads_q),
                                                        static_cast<int>(p->heads_kv), tr, p->q_block,
                                                        static_cast<int>(nrep), BC, tc, p->causal ? 1 : 0, m0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("m-init seed launch: ") + cudaGetErrorString(e));
    m0_tile = m0;
  }
  if (zero_counters) reset_counters(stats, status, st);
  if (skip_trace)
    cudaMemsetAsync(skip_trace, 0,
                    static_cast<size_t>(p->batch * p->heads_q * (p->seq_q / p->q_block) * n_key_blocks(p)), st);

  vfa::FwdArgs a;
  a.B = static_cast<int>(p->batch);
  a.Hq = static_cast<int>(p->heads_q);
  a.Hkv = static_cast<int>(p->heads_kv);
  a.Lq = static_cast<int>(p->seq_q);
  a.Lk = static_cast<int>(p->seq_k);
  a.group = group;
  a.Tr = static_cast<int>(p->seq_q / p->q_block);
  a.qrows = p->q_block;
  a.Tc = static_cast<int>(n_key_blocks(p));
  a.heads_per_unit = pair == 2 ? 2 * pair_nq : nq;
  a.pair = pair;
  a.units_per_kvh = a.Tr * (group / a.heads_per_unit);
  const double scale = p->scale > 0 ? p->scale : 1.0 / std::sqrt(static_cast<double>(D));
  a.c_scale = static_cast<float>(scale * 1.4426950408889634);
  a.log2_lambda = (p->variant >= VFA_VARIANT_VSA && p->lam > 0) ? static_cast<float>(std::log2(p->lam)) : -INFINITY;
  a.tau = static_cast<float>(p->tau);  // log2 units: (m_new - m) * log2(e) <= tau <=> m_new - m <= tau * ln 2
  a.causal = p->causal ? 1 : 0;
  a.reorder = p->reorder ? 1 : 0;
  a.use_m_init = minit ? 1 : 0;
  a.nrep_cap = static_cast<int>(nrep);
  const bool blasst = p->variant >= VFA_VARIANT_BLASST;  // reference schedule: 1 sink + 1 local
  a.n_sink = blasst ? 1 : p->n_sink;
  a.n_local = blasst ? 1 : p->n_local;
  a.monitor = p->monitor ? 1 : 0;
  a.o = static_cast<__nv_bfloat16*>(o);
  a.o_sb = p->o_stride[0];
  a.o_sh = p->o_stride[1];
  a.o_sr = p->o_stride[2];
  a.lse = lse;
  a.stats = reinterpret_cast<unsigned long long*>(stats);
  a.status = status;
  a.skip_trace = skip_trace;
  a.stab = stab_block;
  a.m_trace = m_trace;
  a.m0_tile = m0_tile;
  a.row_bias = row_bias;
  a.dv = D;  // head_dim 32 runs on a D = 64 kernel: only the first 32 O columns are stored
  a.row_base = row_base;
  a.trace = g_debug_trace;

  // the warp-specialised kernel serves the headline shape (default layout, no debug outputs)
  if (ws_path) return vfa_host::launch_ws(p, mq, mk, mv, mr, a, st);
  static const vfa_host::LaunchFn kLaunch[] = {vfa_host::launch_fa,     vfa_host::launch_vfa,
                                               vfa_host::launch_vsa,    vfa_host::launch_blasst,
                                               vfa_host::launch_blasst_fa4, vfa_host::launch_blasst_rowskip};
  return kLaunch[p->variant](p, nq, mq, mk, mv, mr, a, st);
}

// ---------------------------------------------------------------- host-resident pipeline
// vfa_fwd_host: the problem is cut into K/V groups (one batch, `ck` KV heads) and each group
// into query sub-chunks (`nqs` consecutive query heads of the group). A group's K and V are
// copied host->device once into one of two K/V slots (and its key-block representations
// computed there); each sub-chunk's Q is copied into one of three Q/O
// slots, computed on compute stream c % 2 (one sub-chunk's causal tail overlaps the next
// one's head) and its O / LSE copied back on the D2H stream. PCIe transfers in both
// directions overlap the attention kernels; small sub-chunks keep the exposed head (first
// copy) and tail (last kernel + last copy-back) of the pipeline short.
constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct HostPlan {
  int64_t ck = 0, nqs = 0, subs = 0, groups = 0, chunks = 0, kv_slots = 0, q_slots = 0;
  size_t q_bytes = 0, kv_bytes = 0, lse_bytes = 0, ws_bytes = 0, kv_slot_bytes = 0, q_slot_bytes = 0;
  size_t seed_bytes = 0;  // block-wise qkind: query representations + per-tile seeds, per Q slot
  bool minit = false;
  VfaParams cp{};  // the per-sub-chunk problem (dense device layout)
};

// chunk_q_heads = 0: all query heads of the group; otherwise it must divide the GQA group
// and requires chunk_kv_heads == 1 (the sub-chunk's query heads are then contiguous).
bool host_plan(const VfaParams* p, int chunk_kv_heads, int chunk_q_heads, HostPlan* out) {
  if (chunk_kv_heads < 1 || p->heads_kv % chunk_kv_heads || chunk_q_heads < 0) return false;
  const int64_t group = p->heads_q / p->heads_kv;
  HostPlan g;
  g.ck = chunk_kv_heads;
  if (chunk_q_heads == 0 || chunk_q_heads >= group) {
    g.nqs = g.ck * group;
  } else {
    if (group % chunk_q_heads || g.ck != 1) return false;
    g.nqs = chunk_q_heads;
  }
  g.subs = g.ck * group / g.nqs;
  g.groups = p->batch * (p->heads_kv / g.ck);
  g.chunks = g.groups * g.subs;
  // enough slots that the copy stream never waits on a slot in steady state (the copy-in
  // runs ahead of the kernels by up to ~2 groups; HBM is plentiful, PCIe is the bottleneck)
  g.kv_slots = g.groups < 4 ? g.groups : 4;
  g.q_slots = g.chunks < 8 ? g.chunks : 8;
  g.minit = (p->variant == VFA_VARIANT_VFA || p->variant == VFA_VARIANT_VSA) && p->use_m_init;
  g.cp = *p;
  g.cp.batch = 1;
  g.cp.heads_q = g.nqs;
  g.cp.heads_kv = g.ck;
  g.cp.krepr_precomputed = g.minit ? 1 : 0;  // computed once per K/V group on the copy stream
  const int64_t D = p->head_dim;
  const int64_t qs[3] = {g.nqs * p->seq_q * D, p->seq_q * D, D};
  const int64_t ks[3] = {g.ck * p->seq_k * D, p->seq_k * D, D};
  for (int i = 0; i < 3; ++i) {
    g.cp.q_stride[i] = g.cp.o_stride[i] = qs[i];
    g.cp.k_stride[i] = g.cp.v_stride[i] = ks[i];
  }
  g.q_bytes = static_cast<size_t>(g.nqs * p->seq_q * D * 2);
  g.kv_bytes = static_cast<size_t>(g.ck * p->seq_k * D * 2);
  g.lse_bytes = static_cast<size_t>(g.nqs * p->seq_q * 4);
  g.ws_bytes = vfa_workspace_bytes(&g.cp);
  g.kv_slot_bytes = 2 * align_up(g.kv_bytes) + align_up(g.ws_bytes);
  if (g.minit && p->qkind != 0) g.seed_bytes = align_up(ws_qrepr_bytes(&g.cp) + ws_m0_bytes(&g.cp));
  g.q_slot_bytes = 2 * align_up(g.q_bytes) + align_up(g.lse_bytes) + g.seed_bytes;
  *out = g;
  return true;
}

struct HostStreams {
  int device = -1;
  cudaStream_t h2d = nullptr, d2h = nullptr, comp[2] = {nullptr, nullptr};
};

// per-thread, per-device streams of the pipeline (created once, non-blocking)
int host_streams(HostStreams** out) {
  thread_local HostStreams cache[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 16) return fail(VFA_ERR_CUDA, "cudaGetDevice failed");
  HostStreams& s = cache[dev];
  if (s.device != dev) {
    cudaStream_t* all[4] = {&s.h2d, &s.d2h, &s.comp[0], &s.comp[1]};
    for (cudaStream_t* x : all)
      if (cudaStreamCreateWithFlags(x, cudaStreamNonBlocking) != cudaSuccess)
        return fail(VFA_ERR_CUDA, "cudaStreamCreateWithFlags failed");
    s.device = dev;
  }
  *out = &s;
  return VFA_OK;
}
}  // namespace

extern "C" {

size_t vfa_host_scratch_bytes(const VfaParams* p, int chunk_kv_heads, int chunk_q_heads) {
  HostPlan g;
  if (!p || vfa_check_params(p) != VFA_OK || !host_plan(p, chunk_kv_heads, chunk_q_heads, &g)) return 0;
  return static_cast<size_t>(g.kv_slots) * g.kv_slot_bytes + static_cast<size_t>(g.q_slots) * g.q_slot_bytes + kAlign;
}

int vfa_fwd_host(const VfaParams* p, const void* q_host, const void* k_host, const void* v_host, void* o_host,
                 float* lse_host, void* scratch, size_t scratch_bytes, long long* stats, unsigned int* status,
                 int chunk_kv_heads, int chunk_q_heads, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q_host || !k_host || !v_host || !o_host) return fail(VFA_ERR_DATA, "NULL host pointer");
  HostPlan g;
  if (!host_plan(p, chunk_kv_heads, chunk_q_heads, &g))
    return fail(VFA_ERR_CONFIG,
                "chunk_kv_heads must divide heads_kv; chunk_q_heads must be 0 or divide the GQA group "
                "(with chunk_kv_heads = 1)");
  if (p->krepr_precomputed) return fail(VFA_ERR_CONFIG, "vfa_fwd_host computes the representations itself");
  const size_t need = vfa_host_scratch_bytes(p, chunk_kv_heads, chunk_q_heads);
  if (!scratch || scratch_bytes < need) return fail(VFA_ERR_DATA, "scratch too small (vfa_host_scratch_bytes)");
  HostStreams* hs = nullptr;
  rc = host_streams(&hs);
  if (rc) return rc;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(scratch) + kAlign - 1) & ~uintptr_t(kAlign - 1));
  uint8_t* kv_base = base;
  uint8_t* q_base = base + g.kv_slots * g.kv_slot_bytes;

  // debug: VFA_HOST_TIMELINE=1 records timing events along the pipeline and prints them
  // (ms from entry) to stderr, synchronizing at the end (scripts/host_timeline.py)
  const bool timeline = std::getenv("VFA_HOST_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  auto mark = [&](const std::string& what, cudaStream_t s) {
    if (!timeline) return;
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    marks.emplace_back(what, e);
  };
  std::vector<cudaEvent_t> ev;
  auto new_event = [&]() -> cudaEvent_t {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    ev.push_back(e);
    return e;
  };
  auto cleanup = [&]() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);  // released once their work completes
  };
  // error after work was enqueued: wait for every in-flight copy / kernel of the pipeline before
  // returning, since they reference caller-owned host buffers and scratch the caller may reuse
  auto abort_pipeline = [&](int code) {
    cudaStream_t all[4] = {hs->h2d, hs->d2h, hs->comp[0], hs->comp[1]};
    for (cudaStream_t x : all) cudaStreamSynchronize(x);
    cleanup();
    return code;
  };
  // counters accumulate over chunks; scratch reuse is ordered after the caller's prior work
  reset_counters(stats, status, caller);
  cudaEvent_t entry = new_event();
  if (!entry) return cleanup(), fail(VFA_ERR_CUDA, "cudaEventCreate failed");
  cudaEventRecord(entry, caller);
  cudaStreamWaitEvent(hs->h2d, entry, 0);
  cudaStreamWaitEvent(hs->comp[0], entry, 0);
  cudaStreamWaitEvent(hs->comp[1], entry, 0);
  mark("entry", hs->h2d);

  const int64_t D = p->head_dim, group = p->heads_q / p->heads_kv;
  const int64_t per_b = p->heads_kv / g.ck;
  std::vector<cudaEvent_t> kv_free(static_cast<size_t>(g.kv_slots), nullptr);
  std::vector<cudaEvent_t> q_free(static_cast<size_t>(g.q_slots), nullptr);
  int64_t c = 0;  // global sub-chunk counter
  for (int64_t gi = 0; gi < g.groups; ++gi) {
    const int64_t b = gi / per_b, kv0 = (gi % per_b) * g.ck;
    uint8_t* kvs = kv_base + (gi % g.kv_slots) * g.kv_slot_bytes;
    uint8_t* dk = kvs;
    uint8_t* dv = dk + align_up(g.kv_bytes);
    uint8_t* dws = dv + align_up(g.kv_bytes);
    const size_t koff = static_cast<size_t>((b * p->heads_kv + kv0) * p->seq_k * D) * 2;
    // K/V of the group (after every sub-chunk that used this slot has been copied out)
    if (kv_free[gi % g.kv_slots]) cudaStreamWaitEvent(hs->h2d, kv_free[gi % g.kv_slots], 0);
    cudaMemcpyAsync(dk, static_cast<const uint8_t*>(k_host) + koff, g.kv_bytes, cudaMemcpyHostToDevice, hs->h2d);
    cudaMemcpyAsync(dv, static_cast<const uint8_t*>(v_host) + koff, g.kv_bytes, cudaMemcpyHostToDevice, hs->h2d);
    cudaEvent_t kv_in = new_event();
    if (!kv_in) return abort_pipeline(fail(VFA_ERR_CUDA, "cudaEventCreate failed"));
    cudaEventRecord(kv_in, hs->h2d);
    mark("kv_in " + std::to_string(gi), hs->h2d);
    if (g.minit) {
      // representations once per group, on the compute stream of its first sub-chunk (a kernel
      // on the copy stream would stall the copies behind the running attention kernels)
      cudaStream_t cs0 = hs->comp[c & 1];
      cudaStreamWaitEvent(cs0, kv_in, 0);
      rc = launch_krepr(&g.cp, dk, dws, cs0);
      if (rc) return abort_pipeline(rc);
      kv_in = new_event();
      if (!kv_in) return abort_pipeline(fail(VFA_ERR_CUDA, "cudaEventCreate failed"));
      cudaEventRecord(kv_in, cs0);
    }
    // The first and last K/V groups run in half-size query sub-chunks: the pipeline's fill (the
    // first copies before any kernel) and drain (the last kernel and its copy-back, after the
    // last H2D) shrink. Only where the smaller sub-chunk
    // computes bit-identically (an even head count, or VFA's 4-threads-per-row layout, which a
    // single-tile CTA also uses).
    const bool same_bits = (g.nqs / 2) % 2 == 0 ||
                           (p->variant == VFA_VARIANT_VFA && (p->softmax_split == 4 ||
                                                              (p->softmax_split == 0 && !ws_eligible(p))));
    const bool tail = (gi == g.groups - 1 || gi == 0) && g.ck == 1 && g.nqs >= 2 && g.nqs % 2 == 0 && g.groups > 1 && same_bits;
    const int64_t nq_g = tail ? g.nqs / 2 : g.nqs;
    VfaParams cpg = g.cp;
    cpg.heads_q = nq_g;
    const size_t q_bytes_g = static_cast<size_t>(nq_g * p->seq_q * D * 2);
    const size_t lse_bytes_g = static_cast<size_t>(nq_g * p->seq_q * 4);
    const int64_t subs_g = g.subs * (g.nqs / nq_g);
    for (int64_t si = 0; si < subs_g; ++si, ++c) {
      const int64_t h0 = kv0 * group + si * nq_g;
      uint8_t* qsl = q_base + (c % g.q_slots) * g.q_slot_bytes;
      uint8_t* dq = qsl;
      uint8_t* dout = dq + align_up(g.q_bytes);
      float* dlse = reinterpret_cast<float*>(dout + align_up(g.q_bytes));
      void* dseed = g.seed_bytes ? reinterpret_cast<uint8_t*>(dlse) + align_up(g.lse_bytes) : nullptr;
      const size_t qoff = static_cast<size_t>((b * p->heads_q + h0) * p->seq_q * D) * 2;
      const size_t loff = static_cast<size_t>((b * p->heads_q + h0) * p->seq_q);
      if (q_free[c % g.q_slots]) cudaStreamWaitEvent(hs->h2d, q_free[c % g.q_slots], 0);
      cudaMemcpyAsync(dq, static_cast<const uint8_t*>(q_host) + qoff, q_bytes_g, cudaMemcpyHostToDevice, hs->h2d);
      cudaEvent_t q_in = new_event(), done = new_event(), out = new_event();
      if (!q_in || !done || !out) return abort_pipeline(fail(VFA_ERR_CUDA, "cudaEventCreate failed"));
      cudaEventRecord(q_in, hs->h2d);
      mark("q_in " + std::to_string(c), hs->h2d);
      cudaStream_t cs = hs->comp[c & 1];
      cudaStreamWaitEvent(cs, kv_in, 0);
      cudaStreamWaitEvent(cs, q_in, 0);
      mark("k_start " + std::to_string(c), cs);
      rc = forward_impl(&cpg, dq, dk, dv, dout, dlse, dws, g.ws_bytes, stats, status, nullptr, nullptr, cs,
                        false, static_cast<long long>(loff), dseed);
      if (rc) return abort_pipeline(rc);
      cudaEventRecord(done, cs);
      mark("k_end " + std::to_string(c), cs);
      cudaStreamWaitEvent(hs->d2h, done, 0);
      cudaMemcpyAsync(static_cast<uint8_t*>(o_host) + qoff, dout, q_bytes_g, cudaMemcpyDeviceToHost, hs->d2h);
      if (lse_host) cudaMemcpyAsync(lse_host + loff, dlse, lse_bytes_g, cudaMemcpyDeviceToHost, hs->d2h);
      cudaEventRecord(out, hs->d2h);
      mark("out " + std::to_string(c), hs->d2h);
      q_free[c % g.q_slots] = out;
      // the D2H stream has waited for every sub-chunk's kernel of this group by now
      if (si + 1 == subs_g) kv_free[gi % g.kv_slots] = out;
    }
  }
  cudaEvent_t exit_ev = new_event();
  if (!exit_ev) return abort_pipeline(fail(VFA_ERR_CUDA, "cudaEventCreate failed"));
  cudaEventRecord(exit_ev, hs->d2h);
  cudaStreamWaitEvent(caller, exit_ev, 0);
  if (timeline && !marks.empty()) {
    cudaError_t se = cudaEventSynchronize(exit_ev);
    for (auto& m : marks) {
      float ms = -1.f;
      cudaError_t ee = cudaEventElapsedTime(&ms, marks.front().second, m.second);
      std::fprintf(stderr, "vfa_host_timeline %s %.4f %s %s\n", m.first.c_str(), ms, cudaGetErrorName(se),
                   cudaGetErrorName(ee));
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
  cleanup();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("vfa_fwd_host: ") + cudaGetErrorString(e));
  return VFA_OK;
}

int vfa_schedule(int i, int q_block, int k_block, int t_c, int causal, int n_sink, int n_local, int reorder,
                 int variant, int* order_out, unsigned char* special_out, int cap) {
  if (i < 1 || q_block < 1 || k_block < 1 || t_c < 1) return -VFA_ERR_CONFIG;
  // the device's unit_schedule: FA / BLASST-FA4 / rowskip ascending; BLASST may reorder
  // (1 sink + 1 local); every block of the FA-like variants is exact
  const bool seq = variant == VFA_VARIANT_FA || variant == VFA_VARIANT_BLASST_FA4 || variant == VFA_VARIANT_BLASST_ROWSKIP;
  const bool all_exact = seq || variant == VFA_VARIANT_BLASST;
  if (variant >= VFA_VARIANT_BLASST) n_sink = n_local = 1;
  vfa::TileSchedule s = vfa::make_schedule(i, q_block, k_block, t_c, causal != 0, n_sink, n_local,
                                           !seq && reorder != 0, seq);
  for (int pos = 0; pos < s.vmax && pos < cap; ++pos) {
    int j = vfa::sched_block(s, pos);
    if (order_out) order_out[pos] = j;
    if (special_out) special_out[pos] = (all_exact || vfa::sched_is_special(s, j)) ? 1 : 0;
  }
  return s.vmax;
}

int vfa_status_code(const unsigned int* status_host) {
  if (!status_host) return fail(VFA_ERR_CONFIG, "status is NULL");
  if (status_host[VFA_STATUS_FLAGS] & 3u) {
    if (status_host[VFA_STATUS_FLAGS] & 1u)
      return fail(VFA_ERR_NUMERICAL, "query row " + std::to_string(status_host[VFA_STATUS_MASKED_ROW]) +
                                         " is fully masked; cannot normalize");
    return fail(VFA_ERR_NUMERICAL,
                "normalizer underflow at query row " + std::to_string(status_host[VFA_STATUS_UNDERFLOW_ROW]));
  }
  return VFA_OK;
}

const char* vfa_last_error(void) { return vfa_host::g_last_error.c_str(); }

int vfa_debug_trace(long long* device_buffer) {
#ifdef VFA_TRACE
  g_debug_trace = device_buffer;
  return VFA_OK;
#else
  (void)device_buffer;
  return fail(VFA_ERR_CONFIG, "library built without -DVFA_TRACE (scripts/trace_timeline.py builds the trace variant)");
#endif
}

const char* vfa_version(void) { return "vfa_b200 0.1.0 (sm_100a, tcgen05/TMEM/TMA)"; }

}  // extern "C"
