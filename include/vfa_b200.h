/*
 * vfa_b200.h — C ABI of the B200 (sm_100a) VFA / VSA / FA attention forward pass.
 *
 * This is the drop-in boundary for the reference's attention entry points
 * (/root/reference/pkg/src/vfa_lab):
 *   fa_forward(p, order_hook=None)                       src/fa.py:28
 *   vfa_forward(p, kind, reorder, use_m_init, qkind,
 *               tc1, monitor)                             src/vfa.py:156-164
 *   vsa_forward(p, cfg: SkipConfig, kind, qkind, tc1,
 *               monitor)                                  src/sparse.py:256-263
 *   AttentionProblem(q, k, v, blocks, scale, causal)     src/reference.py:20-46
 *   BlockSpec(seq_len_q, seq_len_k, head_dim,
 *             q_block, k_block)                          src/tensor.py:19-52
 *   precompute_kreprs(p, kind, tc1)                      src/vfa.py:79-88
 *   build_schedule(i, vmax, local, reorder)              src/vfa.py:146-153
 *   variant dispatch _execute(cfg, p)                    src/cli.py:243-286
 * The reference is Python; its "FFI" is the in-process call. The Python host
 * package paper_2604_12798_b200 binds these symbols with ctypes (see
 * INTEGRATION.md). No C++ or torch types cross this boundary: plain pointers,
 * sizes and a cudaStream_t passed as void*.
 *
 * Ownership: all pointers are non-owning device pointers allocated by the caller.
 * Inputs are const; outputs are written in stream order. The library keeps no
 * per-call state except a thread-local error string.
 *
 * Return codes mirror the reference CLI exit codes (src/cli.py:69-72):
 *   0 ok, 2 invalid configuration, 3 shape / stride / alignment (data) error,
 *   4 numerical (only from vfa_status_code on a read-back status word),
 *   5 CUDA launch or runtime error.
 */
#ifndef VFA_B200_H_
#define VFA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* the library is built with hidden visibility; only these entry points are exported */
#if defined(__GNUC__)
#define VFA_API __attribute__((visibility("default")))
#else
#define VFA_API
#endif

#define VFA_OK 0
#define VFA_ERR_CONFIG 2
#define VFA_ERR_DATA 3
#define VFA_ERR_NUMERICAL 4
#define VFA_ERR_CUDA 5

/* variant: src/cli.py:243-286 names */
#define VFA_VARIANT_FA 0  /* fa_forward: rescale every block, ascending order */
#define VFA_VARIANT_VFA 1 /* vfa_forward: m-init + sink/local reorder + frozen max */
#define VFA_VARIANT_VSA 2 /* vsa_forward: VFA + BLASST block skip */
/* the BLASST family, src/sparse.py:112-253 (m0 = -inf, every block exact, no m-init) */
#define VFA_VARIANT_BLASST 3         /* blasst_forward: order = reorder ? sink_local : sequential */
#define VFA_VARIANT_BLASST_FA4 4     /* blasst_fa4_forward: + rescale elision (params.tau) */
#define VFA_VARIANT_BLASST_ROWSKIP 5 /* blasst_rowskip_forward: row-granular threshold */

/* key representation kind: KEY_REPRS, src/vfa.py:39 */
#define VFA_KREPR_SABSMAX 0
#define VFA_KREPR_K_MAX 1
#define VFA_KREPR_K_MEAN 2
#define VFA_KREPR_K_ABSMAX_UNSIGNED 3

/* stats[] slots (int64, device; zeroed by vfa_fwd when non-NULL) */
#define VFA_STAT_VISITED 0        /* SkipStats.blocks_visited */
#define VFA_STAT_SKIPPED 1        /* SkipStats.blocks_skipped */
#define VFA_STAT_SPECIAL 2        /* processed with rowmax + rescale */
#define VFA_STAT_FROZEN 3         /* processed with the frozen max */
#define VFA_STAT_OVER_F32 4       /* monitor: exp args > 88.7228 (OverflowMonitor) */
#define VFA_STAT_OVER_F16 5       /* monitor: exp args > ln(65504) */
#define VFA_STAT_ELIDED 6         /* BLASST-FA4: SkipStats.rescales_elided */
#define VFA_STAT_ROWS_MASKED 7    /* BLASST rowskip: SkipStats.rows_masked */
/* monitor = 1 only (OverflowMonitor.exp_arg_max / calibration_gap, src/vfa.py:109-135). Float
 * statistics in log2 units of the scaled scores (natural units = value * ln 2), stored as
 * order-preserving keys: key = bits ^ (bits >> 31 ? 0xffffffff : 0x80000000), 0 = no value. */
#define VFA_STAT_EXP_ARG_MAX 8    /* key of the largest finite exp argument (processed blocks) */
#define VFA_STAT_GAP_NEG_MIN 9    /* key of -min over rows of (m seed - exact global row max) */
#define VFA_STAT_GAP_MAX 10       /* key of max over rows of the same gap */
#define VFA_STAT_GAP_SUM 11       /* double: sum of the gaps */
#define VFA_STAT_GAP_BELOW 12     /* rows with gap < 0 (seed below the exact max) */
#define VFA_STAT_GAP_ROWS 13      /* rows with a seed (m-init on); 0 = no gap recorded */
#define VFA_STAT_COUNT 14

/* status[] slots (uint32, device; initialised by vfa_fwd when non-NULL) */
#define VFA_STATUS_FLAGS 0          /* bit0 fully-masked row, bit1 normalizer underflow, bit2 non-finite O */
#define VFA_STATUS_UNDERFLOW_ROW 1  /* min linear row ((b*Hq+h)*Lq+r) with l==0, finite m; 0xffffffff none */
#define VFA_STATUS_MASKED_ROW 2     /* min linear row with l==0 and m==-inf; 0xffffffff none */
#define VFA_STATUS_NONFINITE_ROWS 3 /* number of rows with a non-finite output */
#define VFA_STATUS_COUNT 4

typedef struct VfaParams {
  /* geometry: q [B, Hq, Lq, D], k/v [B, Hkv, Lk, D], o like q; bf16, last dim contiguous */
  int64_t batch, heads_q, heads_kv, seq_q, seq_k, head_dim;
  /* element strides for (batch, head, row); all must be multiples of 8 (16 bytes) */
  int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3];
  /* lse is a contiguous float32 [B, Hq, Lq] */
  double scale;         /* softmax scale > 0; 0 selects 1/sqrt(D) (src/reference.py:45-46); negative,
                           infinite or NaN is rejected (VFA_ERR_CONFIG): the kernels fold the scale in
                           after the row max, which needs max(s) * scale == max(s * scale) */
  int32_t causal;       /* entrywise causal mask (requires Lq == Lk, src/reference.py:43-44) */
  int32_t q_block;      /* BlockSpec.q_block: 16, 32, 64 or 128 (one reference query block per
                           128-row tcgen05 tile; below 128 the remaining rows run idle) */
  int32_t k_block;      /* BlockSpec.k_block: 64 or 128 */
  int32_t variant;      /* VFA_VARIANT_* */
  int32_t kind;         /* VFA_KREPR_* */
  int32_t qkind;        /* QUERY_REPRS (src/vfa.py:40): 0 row_wise, 1 q_absmax, 2 q_sabsmax, 3 q_mean */
  int32_t reorder;      /* vfa_forward(reorder=...); BLASST: 1 = order 'sink_local' */
  int32_t use_m_init;   /* vfa_forward(use_m_init=...) */
  int32_t tc1;          /* representations for key blocks 1..tc1; 0 = all (src/vfa.py:79-88) */
  int32_t n_sink;       /* sink blocks taking the exact update (reference: 1) */
  int32_t n_local;      /* local blocks ending at the diagonal (reference: 1) */
  int32_t monitor;      /* count exp-argument overflows (OverflowMonitor, src/vfa.py:109-128) */
  double lam;           /* VSA threshold lambda in (0, 1]; <= 0 disables skipping (SkipConfig.lam=None) */
  int32_t krepr_precomputed; /* 1: workspace already holds vfa_krepr() output for this K; skip recomputing */
  int32_t softmax_split; /* 0 = default kernel choice: at d = 128 with 128-row blocks and an even
                           GQA group the warp-specialised kernels (two threads per row; VFA / VSA
                           the decoupled one-tile kernel, FA the ping-pong kernel), elsewhere the
                           general kernel's per-variant layout. An explicit layout runs the general
                           kernel: 1 = a softmax warpgroup per query tile (one thread per row),
                           2 = per-tile warp sets, 4 = all softmax warps serve both tiles */
  double tau;           /* BLASST-FA4 rescale elision: max increase <= tau * ln 2 (SkipConfig.tau) */
  int32_t cta_pair;     /* 0 = default, 1 = one CTA per unit, 2 = CTA pairs (even GQA group, d = 128):
                           the unit's two query heads on two SMs sharing K/V through M = 256 MMAs */
  int32_t reserved;
} VfaParams;

/* Host-only validation (no GPU needed). Returns VFA_OK or VFA_ERR_CONFIG / VFA_ERR_DATA. */
VFA_API int vfa_check_params(const VfaParams* p);

/* Bytes of device workspace vfa_fwd needs (key-block representations). */
VFA_API size_t vfa_workspace_bytes(const VfaParams* p);

/* The attention forward. q,k,v: bf16 device; o: bf16 device; lse: float32 device
 * [B,Hq,Lq] (nullable). workspace: >= vfa_workspace_bytes. stats: int64[VFA_STAT_COUNT]
 * (nullable). status: uint32[VFA_STATUS_COUNT] (nullable). skip_trace: uint8
 * [B, Hq, Lq/128, Lk/k_block] (nullable): per visit position, 1 = processed,
 * 2 = skipped, 0 = not visited. stab_block: int32 [B, Hq, Lq] (nullable): the StateTrace
 * stabilization position of every row (src/analysis.py:39-78) -- the 1-based key block of
 * the visit after which the running max equals its final value. stream: cudaStream_t
 * (NULL = legacy default). */
VFA_API int vfa_fwd(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                    void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                    unsigned char* skip_trace, int* stab_block, void* stream);

/* vfa_fwd with a per-row exponent rebase: row_bias float32 [B, Hq, Lq] (device, log2 units of
 * the scaled scores) multiplies the row's exponentials and normalizer by 2^bias, which leaves
 * O = PV / l unchanged and is subtracted from the LSE. Recovery path for the fp32 normalizer
 * underflow: a VFA row whose frozen max exceeds every score by more than fp32's exp range
 * (~87 nats) gets l == 0 on the device (vfa_fwd flags it like NormalizerUnderflowError and
 * writes the frozen max, natural units, into its LSE slot) although the float64 reference
 * normalizes it (src/core.py:101-109) as long as the gap stays below ~745 nats; re-running with
 * bias = (frozen max - exact row max) * log2(e) on those rows (0 elsewhere: bitwise vfa_fwd)
 * computes them exactly. The Python layer does this automatically (api.attention_forward). */
VFA_API int vfa_fwd_rebased(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                            void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                            const float* row_bias, void* stream);

/* vfa_fwd recording the reference's StateTrace (src/core.py:35-54, src/vfa.py:197,216): m_trace
 * float32 [B, Hq, Lq, Lk/k_block] (device) receives, per query row and visit position (the
 * schedule's order, vfa_schedule), the running max after that visit in natural units (entries
 * past the row's visible blocks are left untouched); stab_block as in vfa_fwd (nullable).
 * A debug output: one extra store per row and visit. */
VFA_API int vfa_fwd_state_trace(const VfaParams* p, const void* q, const void* k, const void* v, void* o,
                                float* lse, void* workspace, size_t workspace_bytes, long long* stats,
                                unsigned int* status, int* stab_block, float* m_trace, void* stream);

/* Bytes of device scratch vfa_fwd_host needs (up to four K/V group slots and eight query
 * sub-chunk slots), or 0 if the parameters or the chunking are invalid. */
VFA_API size_t vfa_host_scratch_bytes(const VfaParams* p, int chunk_kv_heads, int chunk_q_heads);

/* End-to-end forward from HOST memory (the reference's own calling convention: arrays in,
 * arrays out). q/k/v/o are dense host bf16 [B,H,L,D] (strides in *p are ignored), lse a
 * dense host float32 [B,Hq,Lq] (nullable); page-locked host memory gives full overlap.
 * The problem is pipelined in K/V groups (one batch, chunk_kv_heads KV heads, copied once)
 * and query sub-chunks (chunk_q_heads consecutive query heads of a group; 0 = the whole
 * group; a value below the GQA group requires chunk_kv_heads = 1): H2D copies, attention
 * kernels and D2H copies of consecutive sub-chunks overlap on library-owned streams.
 * stats/status are device buffers (nullable) accumulated over all chunks with whole-problem
 * row indices. `stream` is made to wait for the last copy, so a synchronize on it means
 * o/lse are in host memory. krepr_precomputed must be 0. */
VFA_API int vfa_fwd_host(const VfaParams* p, const void* q_host, const void* k_host, const void* v_host,
                         void* o_host, float* lse_host, void* scratch, size_t scratch_bytes,
                         long long* stats, unsigned int* status, int chunk_kv_heads, int chunk_q_heads,
                         void* stream);

/* Key-block representations only (precompute_kreprs): k bf16 [B,Hkv,Lk,D] ->
 * out bf16 contiguous [B, Hkv, n_blocks, D], n_blocks = tc1 or Lk/k_block. */
VFA_API int vfa_krepr(const VfaParams* p, const void* k, void* out, void* stream);

/* Incremental representations for an append-only K cache:
 * recomputes only key blocks [first_block, n_blocks) of `out` (layout of vfa_krepr), e.g. the
 * blocks that new tokens filled or extended; blocks before first_block are left untouched. */
VFA_API int vfa_krepr_range(const VfaParams* p, const void* k, void* out, int first_block, void* stream);

/* Host mirror of the device tile scheduler (build_schedule, src/vfa.py:146-153,
 * generalised to n_sink/n_local). i is the 1-based query block. Writes up to `cap`
 * visited key blocks (1-based) in visit order to order_out and their special
 * flag to special_out; returns the number visited (vmax) or a negative error. */
VFA_API int vfa_schedule(int i, int q_block, int k_block, int t_c, int causal, int n_sink, int n_local,
                 int reorder, int variant, int* order_out, unsigned char* special_out, int cap);

/* Maps a host copy of the status word to VFA_OK / VFA_ERR_NUMERICAL. */
VFA_API int vfa_status_code(const unsigned int* status_host);

/* Message for the last non-zero return on this thread. */
VFA_API const char* vfa_last_error(void);

/* Debug only (trace builds, -DVFA_TRACE): when non-NULL, subsequent vfa_fwd calls record
 * clock64() timestamps into device_buffer (long long[Tc * 32 + units * 4]: per visited block
 * of the first CTA 32 event slots -- softmax tile 0/1 "S ready"/"P done", MMA tile 0/1
 * "P observed"/"next QK issued", ... (scripts/trace_timeline.py) -- then per CTA its entry /
 * first S / last P / exit). NULL disables. */
VFA_API int vfa_debug_trace(long long* device_buffer);

/* Library version string. */
VFA_API const char* vfa_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VFA_B200_H_ */
