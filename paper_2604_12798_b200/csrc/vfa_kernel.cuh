// B200 (sm_100a) VFA / VSA / FA attention forward.
//
// One CTA = one work unit = (batch b, KV head, NQ query heads of that KV head's
// GQA group, one 128-row query tile). The NQ query tiles share every K/V tile
// loaded into shared memory and share the tile schedule (same rows => same
// causal extent, same sink/local blocks).
//
// Warp roles (20 warps, 640 threads):
//   warps 0-15  softmax: 4 warpgroups; each row of a query tile is shared by SPLIT
//               threads (TMEM lane r of SPLIT warpgroups). SPLIT 2: warpgroups 2t, 2t+1
//               serve tile t; SPLIT 4: all four serve both tiles in turn. The softmax also
//               rescales its part of O in TMEM on exact-update blocks (O is quiescent then).
//   warp 16     MMA issuer (converged warp, elect.sync), TMEM allocator
//   warp 17     TMA producer (one lane)
//   warps 18-19 idle (complete the last warpgroup for setmaxnreg)
// TMEM (512 columns): S_t at t*128 (P_t bf16 packed over the first half of each part's
// columns), O_t at NQ*128 + t*D.
// Modes (C-ABI variant codes): FA, VFA, VSA and the BLASST family (src/sparse.py:112-253):
// BL (threshold skip on the baseline recurrence, sequential or sink/local order), BL4
// (plus rescale elision when no row max rises by more than tau*ln2), BLR (row-granular
// threshold: suppressed rows contribute zero mass).
//
// Reference algorithm (src/X.py = /root/reference/pkg/src/vfa_lab/X.py):
//   precompute_kreprs / block_repr / sabsmax   src/vfa.py:47-88     -> krepr_kernel
//   m_init (row_wise)                          src/vfa.py:91-106    -> m-init prologue (tcgen05 Q.Krepr^T)
//   build_schedule / visible / local blocks    src/vfa.py:146-153, src/core.py:112-122 -> schedule.h
//   special-block update (rowmax + rescale)    src/vfa.py:202-208, src/core.py:76-92
//   frozen-block update (no rowmax/rescale)    src/vfa.py:209-215, src/core.py:95-98
//   BLASST skip (all rows m~ - m_new < ln l)   src/sparse.py:99-109, 296-304
//   fa_forward (rescale every block)           src/fa.py:28-61
//   finalize (O / l, l == 0 errors)            src/core.py:101-109
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vfa_b200.h"
#include "ptx.cuh"
#include "schedule.h"

namespace vfa {

constexpr int kBR = 128;          // query rows per tile (tcgen05 M)
// Warp layout (Cfg::kSoftmaxWarps ...): SPLIT 2 / 4: warps 0-15 are four softmax warpgroups
// (2 or 4 threads per row); SPLIT 1: one softmax warpgroup per query tile (one thread per row).
// Then the MMA issuer (all query tiles, strictly alternating) + TMEM allocator, the TMA
// producer, and two warps completing the last warpgroup. (One issuer per tile was measured
// slower: the tiles drift into phase and contend for the softmax issue slots.)
#ifndef VFA_REGS_SPLIT1
#define VFA_REGS_SPLIT1 216
#endif
constexpr int kMaxSmem = 227 * 1024;
constexpr float kLn2 = 0.6931471805599453f;

// kernel modes = C-ABI variant codes (include/vfa_b200.h)
enum Mode { kFA = 0, kVFA = 1, kVSA = 2, kBL = 3, kBL4 = 4, kBLR = 5 };
// every visited block takes the exact (rowmax + rescale) update
constexpr bool all_exact(int m) { return m == kFA || m == kBL || m == kBL4 || m == kBLR; }
// the block-skip test runs on every visited block
constexpr bool skips(int m) { return m == kVSA || m == kBL || m == kBL4 || m == kBLR; }

struct FwdArgs {
  int B, Hq, Hkv, Lq, Lk, group, Tr, Tc;
  int units_per_kvh, heads_per_unit;
  int qrows;          // query rows per reference block (q_block | 128): a 128-row MMA tile holds
                      // query block qt's qrows rows; the rest are idle lanes (never stored)
  float c_scale;      // softmax scale * log2(e)
  float log2_lambda;  // skip threshold in log2 units (-inf: no skipping)
  float tau;          // BLASST-FA4 elision threshold: max increase tau*ln2 (natural) = tau (log2)
  int causal, reorder, use_m_init, nrep_cap, n_sink, n_local, monitor;
  __nv_bfloat16* o;
  long long o_sb, o_sh, o_sr;
  float* lse;
  unsigned long long* stats;
  unsigned int* status;
  unsigned char* skip_trace;
  int* stab;  // per row: key block (1-based) of the visit where the running max last rose
  float* m_trace;  // StateTrace snapshots (src/core.py:35-54): per row and visit position, the running
                   // max after the visit (natural units), [B, Hq, Lq, Tc]; or null
  const float* m0_tile;  // block-wise qkind m-init: raw max_j qrepr_i . krepr_j per query tile, or null
  int dv;                 // head_dim (<= the kernel's D; 32 on a D = 64 kernel, zero-padded tiles)
  const float* row_bias;  // per-row exponent rebase (log2 units, [B, Hq, Lq]) or null: P and l of the
                          // row are scaled by 2^bias (O = PV / l unchanged), LSE corrected; used to
                          // recover rows whose fp32 normalizer underflowed (vfa_fwd_rebased)
  int pair;            // host: 2 = launched as CTA pairs (clusters of two CTAs), else 1
  long long row_base;  // linear-row offset of this launch's (b=0, h=0, r=0) in the status word
  long long* trace;  // debug: per-visit clock64 events of CTA 0 (vfa_debug_trace), or null
};

#ifndef VFA_S2_ALL
#define VFA_S2_ALL 0
#endif
#ifndef VFA_S1_SPLIT34
#define VFA_S1_SPLIT34 1
#endif
#ifndef VFA_POLY_S1
#define VFA_POLY_S1 0  // one thread per row: exp2 pairs (of 8) on the FMA pipe in columns 32-95
#endif
#ifndef VFA_SB_MAX
#define VFA_SB_MAX 2  // S buffers per tile (tuning experiments: 1 disables double buffering)
#endif
#ifndef VFA_Q_TMEM
#define VFA_Q_TMEM 1
#endif
#ifndef VFA_SB_NQ1
#define VFA_SB_NQ1 1  // double-buffer S for every mode when a CTA serves one query tile
#endif

// debug timeline slots per visited block (CTA 0 only, builds with -DVFA_TRACE): softmax t:
// S ready, P done; MMA t: P observed, next QK issued
constexpr int kTraceSlots = 32;
#ifdef VFA_TRACE
#define VFA_TRACE_EVENT(args, pos, slot)                                                     \
  do {                                                                                       \
    if ((args).trace != nullptr && blockIdx.x == 0) (args).trace[(pos) * kTraceSlots + (slot)] = clock64(); \
  } while (0)
// per-CTA phase stamps after CTA 0's per-visit slots: entry, first S seen, last P done, exit
#define VFA_TRACE_UNIT(args, slot)                                                           \
  do {                                                                                       \
    if ((args).trace != nullptr)                                                             \
      (args).trace[(args).Tc * kTraceSlots + blockIdx.x * 4 + (slot)] = clock64();           \
  } while (0)
#else
#define VFA_TRACE_EVENT(args, pos, slot) \
  do {                                   \
  } while (0)
#define VFA_TRACE_UNIT(args, slot) \
  do {                             \
  } while (0)
#endif

// PAIR == 2: a CTA pair (cluster of 2) shares every K/V tile through M = 256 tcgen05 MMAs
// (cta_group::2) over the same local tile index of both CTAs: each CTA holds NQ query tiles
// (its own heads), half of each K tile's rows and half of each V tile's columns, so a K/V stage
// is half as large.
template <int D, int BC, int NQ, int SPLIT, int MODE, int PAIR = 1>
struct Cfg {
  static constexpr int kQBytes = kBR * D * 2;
  static constexpr int kKVBytes = BC * D * 2 / PAIR;
  static constexpr int kDCh = D / 64;  // 64-column (128-byte) swizzle chunks
  // softmax column split: each row of a tile is shared by SPLIT threads (one per warpgroup)
  static constexpr int kCP = BC / SPLIT;             // S columns per part
  static constexpr int kOP = D / SPLIT;              // O columns rescaled / stored per part
  static constexpr int kNCH = kCP >= 32 ? 2 : 1;     // P hand-off chunks per block
  static constexpr int kCW = kCP / kNCH;             // columns per P chunk (16 or 32)
  // PV K-steps (16 P columns each) released by the first P hand-off. One thread per row with
  // 128-column rows (VFA_S1_SPLIT34): the first hand-off comes after 3/4 of the row, so only
  // 2 K-steps of PV remain after the softmax finishes (a shorter P -> PV -> QK -> S chain).
  static constexpr bool kS1Split = SPLIT == 1 && PAIR == 1 && kCP == 128 && VFA_S1_SPLIT34;
  static constexpr int kKS0 = kS1Split ? 6 : kCW / 16;
  static constexpr int kWarpsPerTile = SPLIT * 4;    // softmax warps covering one tile
  // SPLIT 2 with VFA_S2_ALL (and two query tiles): 8 softmax warps, 2 threads per row, all of them
  // serving both tiles in turn like SPLIT 4 (half the softmax warps per sub-partition)
  static constexpr bool kAllTiles = SPLIT == 4 || (SPLIT == 2 && VFA_S2_ALL && NQ == 2);
  static constexpr int kSoftmaxWarps = SPLIT == 1 ? 4 * NQ : (SPLIT == 2 && kAllTiles ? 8 : 16);
  static constexpr int kMmaWarp = kSoftmaxWarps;
  static constexpr int kLoadWarp = kSoftmaxWarps + 1;
  static constexpr int kThreads = (kSoftmaxWarps + 4) * 32;
  // setmaxnreg budgets. The CTA's register pool is what the launch allocated (threads x
  // compiled registers/thread, e.g. 640 x 96 = 61440); asking for more than the pool blocks
  // setmaxnreg.inc forever, so the host checks this budget before launching.
  static constexpr int kRegsSoftmax = (SPLIT == 1 || kSoftmaxWarps == 8) ? VFA_REGS_SPLIT1 : 104;
  static constexpr int kRegsOther = 56;
  static constexpr int kRegBudget = kSoftmaxWarps * 32 * kRegsSoftmax + (kThreads - kSoftmaxWarps * 32) * kRegsOther;
  static constexpr int kCtlBytes = 16384;
  static constexpr int kAvail = kMaxSmem - 1024 - kCtlBytes - NQ * kQBytes;
  static constexpr int kStagesRaw = kAvail / kKVBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmem = 1024 + NQ * kQBytes + kStages * kKVBytes + kCtlBytes;
  // TMEM: S buffers (BC fp32 columns each; P aliased as packed bf16 inside each part's
  // region), then O_t. Two S buffers per tile when they fit (BC = 64, or one query tile):
  // QK of block n+2 is then issued before the softmax of block n+1 starts, so the softmax
  // never waits on the PV -> QK latency of the previous block. Used for the all-exact modes
  // only: measured faster for FA at BC = 64, slower for VFA / VSA (profiles/ab_r01_sb.txt).
  // One query tile per CTA (VFA_SB_NQ1 >= 3): as many S buffers as TMEM holds next to O, up to
  // VFA_SB_NQ1 (3 at d = Bc = 128): QK^T then runs up to two blocks ahead of the softmax.
  static constexpr int kSBNQ1 = (512 - D) / BC < VFA_SB_NQ1 ? (512 - D) / BC : VFA_SB_NQ1;
  static constexpr int kSB =
      (NQ == 1 && VFA_SB_NQ1 >= 3 && VFA_SB_MAX >= 2 && PAIR == 1)
          ? kSBNQ1
          : ((NQ * 2 * BC + NQ * D <= 512 && VFA_SB_MAX >= 2 && (all_exact(MODE) || (NQ == 1 && VFA_SB_NQ1))) ? 2 : 1);
  static __host__ __device__ constexpr uint32_t s_off(int t, int b) {
    return static_cast<uint32_t>((t * kSB + b) * BC);
  }
  static constexpr int kOBase = NQ * kSB * BC;
  static constexpr int kColsUsed0 = kOBase + NQ * D;
  // Q resident in TMEM (D/2 columns per tile, bf16 pairs) where it fits, for BC = 64: QK^T then
  // runs A-from-TMEM, reading only K from shared memory. With both operands in shared memory an
  // N = 64 MMA is shared-memory bound (48 instead of 32 cycles, profiles/ubench_mma_rate_r01.txt);
  // at N = 128 both modes run at the 64-cycle floor (VFA_Q_TMEM=2 also moves Q for Bc = 128:
  // measured slower at d = 64, profiles/ab_r01_chain.txt).
  static constexpr bool kQT = PAIR == 1 && (BC == 64 || VFA_Q_TMEM == 2) && VFA_Q_TMEM && kColsUsed0 + NQ * D / 2 <= 512;
  static constexpr int kQBase = kColsUsed0;
  static constexpr int kColsUsed = kColsUsed0 + (kQT ? NQ * D / 2 : 0);
  static constexpr uint32_t kTmemCols = kColsUsed <= 256 ? 256 : 512;
  static_assert(kColsUsed <= 512, "TMEM over-subscribed");
  static_assert(kStages >= 3, "not enough shared memory for a K/V ring");
  static_assert(kCW % 16 == 0 && kOP % 16 == 0, "parts must be whole 16-column chunks");
  static_assert(SPLIT == 1 || SPLIT == 2 || SPLIT == 4,
                "SPLIT is 1 (a warpgroup per tile, a thread per row), 2 (per-tile warp sets) or 4 (all warps, both tiles)");
};

template <int NS, int NQ, int SB>
struct __align__(16) Ctl {
  uint32_t skip2[NQ][SB][2];   // CTA pair: each CTA's skip decision, gathered in the leader
  uint64_t q_full[NQ];
  uint64_t kv_full[NS];
  uint64_t kv_empty[NS];
  uint64_t s_full[NQ][SB];     // MMA -> softmax: S of sequence element g ready (buffer g % SB)
  uint64_t s_free[NQ][SB];     // softmax -> MMA: m-init chunk read
  uint64_t p_full[NQ][SB][2];  // softmax -> MMA: P chunk c (CW columns of every part) ready /
                               // skip decided; PV of chunk 0 overlaps the softmax of chunk 1
  uint64_t pv_done[NQ];        // MMA -> softmax (SB 2): PV before the next exact block done
  uint64_t o_final[NQ];    // MMA -> epilogue: last PV completed
  uint32_t tmem_base;
  uint32_t skip[NQ][SB];
  float xmax[NQ][2][4][kBR];    // [tile][parity][quarter][row]: quarter-row maxima exchange
  float xl[NQ][4][kBR];         // [tile][quarter][row]: final quarter-row sums
  uint8_t xfin[NQ][4][kBR];     // [tile][quarter][row]: output finite flags
};

struct Unit {
  int b, kvh, h0, qt;
};

__device__ __forceinline__ Unit decode_unit(const FwdArgs& a, int u) {
  Unit w;
  int bk = u / a.units_per_kvh;
  int r = u - bk * a.units_per_kvh;
  int pairs = a.group / a.heads_per_unit;
  w.qt = a.Tr - 1 - r / pairs;  // longest causal tiles first within each KV head
  int pair = r - (r / pairs) * pairs;
  w.b = bk / a.Hkv;
  w.kvh = bk - w.b * a.Hkv;
  w.h0 = w.kvh * a.group + pair * a.heads_per_unit;
  return w;
}

template <int MODE>
__device__ __forceinline__ TileSchedule unit_schedule(const FwdArgs& a, int qt, int BC) {
  // FA / BLASST-FA4 / rowskip: ascending, all exact; BLASST: the VFA visit order when
  // reorder (order='sink_local', src/sparse.py:133) but every block exact
  constexpr bool kSeq = MODE == kFA || MODE == kBL4 || MODE == kBLR;
  return make_schedule(qt + 1, a.qrows, BC, a.Tc, a.causal != 0, a.n_sink, a.n_local, kSeq ? false : (a.reorder != 0),
                       kSeq);
}

// number of m-init chunks (BC representations per chunk)
template <int MODE>
__device__ __forceinline__ int minit_chunks(const FwdArgs& a, const TileSchedule& s, int BC, int* nrep) {
  if ((MODE != kVFA && MODE != kVSA) || !a.use_m_init || a.m0_tile != nullptr) {
    *nrep = 0;
    return 0;
  }
  int n = s.vmax < a.nrep_cap ? s.vmax : a.nrep_cap;
  *nrep = n;
  return (n + BC - 1) / BC;
}


#ifndef VFA_MMA_SPIN
#define VFA_MMA_SPIN 0  // 1: the MMA issuer spins on test_wait instead of (suspending) try_wait
#endif
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t parity) {
  if constexpr (VFA_MMA_SPIN) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);
}
#ifndef VFA_POLY_SMSP0
// exp2 pairs (of 8) on the FMA pipe for the softmax warps of sub-partition 0 only, which also hosts
// the MMA issuer: fewer MUFU there leaves room in that sub-partition's MIO queue for the issuer's
// tcgen05.mma / mbarrier instructions
#define VFA_POLY_SMSP0 0
#endif
#ifndef VFA_SM_SPIN
#define VFA_SM_SPIN 0  // 1: the softmax warps spin on test_wait for S
#endif

// tcgen05.commit from one elected lane of the (converged) MMA warp.
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  if (elect_one()) mma_commit(bar);
  __syncwarp();
}

// Two threads per S row (the warp-specialised kernels): the thread owning half hf of a row
// (keys 64*hf .. 64*hf + 63) stores its packed-bf16 P over the first 32 of its own 64 S
// columns, which it has already loaded -- never over the other half's columns, which that
// thread may still be loading. TMEM column (relative to the S buffer) of PV K-step kk's P:
__host__ __device__ constexpr uint32_t p_col(int kk) { return static_cast<uint32_t>((kk >> 2) * 64 + (kk & 3) * 8); }

// ------------------------------------------------------------------------------------
// Softmax element math. x = s * (scale*log2 e) - m2 in packed pairs (FFMA2); P = exp2(x)
// on MUFU.EX2 for most pairs and on the FMA pipe (degree-4 polynomial, |rel err| < 3e-6)
// for kPoly of every 8 pairs, so that neither the XU nor the FMA pipe limits the
// tensor core; row sums accumulate in packed FADD2; P is packed to bf16 pairs.
#ifdef VFA_POLY_PAIRS
constexpr int kPolyOverride = VFA_POLY_PAIRS;  // tuning experiments (scripts/ab.py)
#else
constexpr int kPolyOverride = -1;
#endif
// Element pairs (of every 8) whose exp2 runs on the FMA pipe (degree-4 polynomial) instead
// of MUFU.EX2. Under the B200's 1 kW power cap the 13-instruction polynomial costs more
// energy (lower clocks) than it saves in MUFU time at head dim 128: measured best is 0 for
// both softmax splits (profiles/ab_r01_poly.txt). Kept identical for every split and mode so
// P (hence O) does not depend on the split or the variant.
// At head dim 64 (half the MMA work per exponential; the GPU is not power-capped) one pair
// in eight on the FMA pipe is measured +4 % at Bc 128 (profiles/ab_r01_poly.txt).
__host__ __device__ constexpr int poly_pairs(int d, int bc, int split) {
  return kPolyOverride >= 0 ? kPolyOverride : (d == 64 && bc == 128 ? 1 : 0);
}
#ifndef VFA_LATE_ROWSUM
#define VFA_LATE_ROWSUM 0  // 1: row sums after the P hand-off for every split, 2: split 1 only
#endif
__host__ __device__ constexpr bool late_rowsum_on(int split) {
  return VFA_LATE_ROWSUM == 1 || (VFA_LATE_ROWSUM == 2 && split == 1);
}
// softmax column split per mode (see the softmax role): measured best per variant
#ifndef VFA_SPLIT_FA
#define VFA_SPLIT_FA 2
#endif
#ifndef VFA_SPLIT_VFA
#define VFA_SPLIT_VFA 4
#endif
#ifndef VFA_SPLIT_VSA
#define VFA_SPLIT_VSA 2
#endif

__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  // clamp to [-127, 128]: x <= -127 (incl. masked -inf) gives exactly +0 (the exponent add
  // wraps 1.0 * 2^-127 to 0x00000000, matching MUFU.EX2.FTZ), x >= 128 gives +inf like MUFU
  x.x = fminf(fmaxf(x.x, -127.f), 128.f);
  x.y = fminf(fmaxf(x.y, -127.f), 128.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23: round to integer
  const float2 r = __fadd2_rn(x, magic);
  const float2 jf = __fadd2_rn(r, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-jf.x, -jf.y));  // f in [-0.5, 0.5]
  float2 p = __ffma2_rn(make_float2(0.009582853876054287f, 0.009582853876054287f), f,
                        make_float2(0.05590642988681793f, 0.05590642988681793f));
  p = __ffma2_rn(p, f, make_float2(0.24024099111557007f, 0.24024099111557007f));
  p = __ffma2_rn(p, f, make_float2(0.6931241750717163f, 0.6931241750717163f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  // scale by 2^j: add j to the exponent field (the low bits of r hold j)
  float2 y;
  y.x = __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(r.x) << 23));
  y.y = __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(r.y) << 23));
  return y;
}

// Degree-3 FMA-pipe exp2 with a floor split (x = j + f, f in [0, 1)): 2^f by a polynomial
// fitted here for minimax relative error (8.6e-5, far inside the bf16 rounding of P),
// 2^j by an exponent add. 12 instructions per element pair (2 FMNMX clamps per element, one
// FADD2 with round-down to extract floor(x), 2 FADD2, 3 FFMA2, 2 shift-adds) against 2 MUFU.EX2
// (16 XU cycles). Clamped to [-127, 128] like MUFU.EX2.FTZ: x <= -127 and -inf give +0, x >= 128
// gives +inf; x in (-127, -126) gives a denormal, which the flush-to-zero row sum drops.
__device__ __forceinline__ float2 add_rm2(float2 a, float2 b) {
  uint64_t r;
  asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "add.rm.ftz.f32x2 %0, ra, rb;\n\t}"
      : "=l"(r) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return make_float2(__uint_as_float(static_cast<uint32_t>(r)), __uint_as_float(static_cast<uint32_t>(r >> 32)));
}
__device__ __forceinline__ float2 add_ftz2(float2 a, float2 b) {
  uint64_t r;
  asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "add.rn.ftz.f32x2 %0, ra, rb;\n\t}"
      : "=l"(r) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return make_float2(__uint_as_float(static_cast<uint32_t>(r)), __uint_as_float(static_cast<uint32_t>(r >> 32)));
}
__device__ __forceinline__ float2 ex2_poly3(float2 x) {
  x.x = fminf(fmaxf(x.x, -127.f), 128.f);
  x.y = fminf(fmaxf(x.y, -127.f), 128.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 r = add_rm2(x, magic);                          // floor(x) in the low mantissa bits
  const float2 j = __fadd2_rn(r, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));    // exact, in [0, 1)
  float2 p = __ffma2_rn(make_float2(0.07706704f, 0.07706704f), f, make_float2(0.22764499f, 0.22764499f));
  p = __ffma2_rn(p, f, make_float2(0.69511676f, 0.69511676f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  float2 y;
  y.x = __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(r.x) << 23));
  y.y = __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(r.y) << 23));
  return y;
}
#ifndef VFA_POLY3
#define VFA_POLY3 1  // the FMA-pipe exp2 is the degree-3 floor form (0: degree-4, round to nearest)
#endif

// order-preserving key of a float (include/vfa_b200.h, VFA_STAT_EXP_ARG_MAX): larger float,
// larger unsigned key
__device__ __forceinline__ unsigned float_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <bool MON>
__device__ __forceinline__ void count_over(float2 x, uint32_t& o32, uint32_t& o16, float& xmax) {
  if (MON) {
    // OverflowMonitor (src/vfa.py:122-128) thresholds, in log2 units; exp_arg_max over the
    // finite arguments (masked entries are -inf and never raise the max)
    o32 += (x.x > 128.0f) + (x.y > 128.0f);
    o16 += (x.x > 15.999295f) + (x.y > 15.999295f);
    xmax = fmax3(xmax, x.x, x.y);
  }
}

// Max of N (a multiple of 8) consecutive values: four independent FMNMX3 chains (max is exact
// in any order, so the result does not depend on the reduction shape).
template <int N>
__device__ __forceinline__ float part_max(const float* v) {
  float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
  for (int e = 0; e < N; e += 8) {
    m0 = fmax3(m0, v[e], v[e + 1]);
    m1 = fmax3(m1, v[e + 2], v[e + 3]);
    m2 = fmax3(m2, v[e + 4], v[e + 5]);
    m3 = fmax3(m3, v[e + 6], v[e + 7]);
  }
  return fmax3(fmaxf(m0, m1), m2, m3);
}

// W consecutive columns (masked entries already -inf): P = exp2(s*cs - m2) -> W/2 packed
// bf16x2 words. LATE: P stays in v (fp32) for a row sum after the hand-off (off the
// S -> P -> PV chain); otherwise row sums go into two independent packed accumulators.
template <int W, bool MON, int kPoly, bool LATE>
__device__ __forceinline__ void p_chunk(float* v, float2 cs2, float2 nmu2, uint32_t* u, float2 (&acc)[2],
                                        uint32_t& o32, uint32_t& o16, float& xmax) {
#pragma unroll
  for (int e = 0; e < W; e += 2) {
    const float2 x = __ffma2_rn(make_float2(v[e], v[e + 1]), cs2, nmu2);
    count_over<MON>(x, o32, o16, xmax);
    float2 p;
    if (((e >> 1) & 7) < kPoly) {
      p = VFA_POLY3 ? ex2_poly3(x) : ex2_poly2(x);
    } else {
      p.x = ex2_approx(x.x);
      p.y = ex2_approx(x.y);
    }
    if constexpr (LATE) {
      v[e] = p.x;
      v[e + 1] = p.y;
    } else {
      acc[(e >> 1) & 1] = add_ftz2(acc[(e >> 1) & 1], p);
    }
    u[e >> 1] = pack_bf16x2(p.x, p.y);
  }
}

// row sum of W exponentials left in v by a LATE p_chunk
template <int W>
__device__ __forceinline__ void late_rowsum(const float* v, float2 (&acc)[2]) {
#pragma unroll
  for (int e = 0; e < W; e += 2) acc[(e >> 1) & 1] = add_ftz2(acc[(e >> 1) & 1], make_float2(v[e], v[e + 1]));
}

// ------------------------------------------------------------------------------------
template <int D, int BC, int NQ, int MODE, int SPLIT, int PAIR>
__global__ void __launch_bounds__(Cfg<D, BC, NQ, SPLIT, MODE, PAIR>::kThreads, 1)
    vfa_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmR,
                   const FwdArgs a) {
  using C = Cfg<D, BC, NQ, SPLIT, MODE, PAIR>;
  static_assert(PAIR == 1 || ((SPLIT == 4 || SPLIT == 1) && D == 128), "CTA pairs: d = 128, split 4 or 1");
  constexpr int NS = C::kStages;
  constexpr int CP = C::kCP;
  constexpr int OP = C::kOP;
  constexpr int NCH = C::kNCH;
  constexpr int CW = C::kCW;
  constexpr int kPoly = poly_pairs(D, BC, SPLIT);
  constexpr bool kLate = late_rowsum_on(SPLIT);
  constexpr int SB = C::kSB;
  using CtlT = Ctl<NS, NQ, SB>;
  static_assert(sizeof(CtlT) <= C::kCtlBytes, "control block too large");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + NQ * C::kQBytes;
  CtlT* ctl = reinterpret_cast<CtlT*>(sKV + NS * C::kKVBytes);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t crank = PAIR == 2 ? cluster_ctarank() : 0;  // CTA rank in the pair (0 = leader)

  if (tid == 0) {
    VFA_TRACE_UNIT(a, 0);
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&ctl->q_full[t], 1);
      for (int b = 0; b < SB; ++b) {
        mbar_init(&ctl->s_full[t][b], 1);
        // a pair's leader barriers count the softmax warps of both CTAs
        mbar_init(&ctl->s_free[t][b], C::kWarpsPerTile * PAIR);
        mbar_init(&ctl->p_full[t][b][0], C::kWarpsPerTile * PAIR);
        mbar_init(&ctl->p_full[t][b][1], C::kWarpsPerTile * PAIR);
      }
      mbar_init(&ctl->pv_done[t], 1);
      mbar_init(&ctl->o_final[t], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&ctl->kv_full[s], 1);
      mbar_init(&ctl->kv_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == C::kLoadWarp && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmR);
  }
  if (warp == C::kMmaWarp) {
    if constexpr (PAIR == 2)
      tmem_alloc_pair<C::kTmemCols>(&ctl->tmem_base);
    else
      tmem_alloc<C::kTmemCols>(&ctl->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR == 2) cluster_sync_all();  // peer barriers initialised before any remote op
  tc_fence_after();
  // the query head of local tile t (a pair's CTAs each hold one of the unit's two heads)
  auto head_of = [&](const Unit& u, int t) { return u.h0 + (PAIR == 2 ? static_cast<int>(crank) * NQ + t : t); };
  (void)head_of;
  // softmax -> MMA hand-offs arrive on the MMA-issuing CTA's barrier (the leader of a pair).
  // The TMEM data they publish is ordered by tcgen05.fence::* around the barrier, so the
  // follower's remote arrive is relaxed; only the arrive that also publishes a generic store
  // (the skip flag, `release_store`) pays a cluster-scope release.
  auto arrive_mma = [&](uint64_t* bar, bool release_store = false) {
    if constexpr (PAIR == 2) {
      if (crank == 0)
        mbar_arrive(bar);
      else if (release_store)
        mbar_arrive_cluster(mapa_shared(bar, 0));
      else
        mbar_arrive_cluster_relaxed(mapa_shared(bar, 0));
    } else {
      (void)release_store;
      mbar_arrive(bar);
    }
  };
  (void)arrive_mma;
  // Each role re-derives its work description after its setmaxnreg so that nothing
  // computed before the role split has to stay live (or spill) across it.
  // Sequence g = 0 .. G-1: nchunks m-init chunks (S = Q . Krepr^T), then the N visited
  // key blocks in schedule order (S = Q . K^T).
#define VFA_ROLE_SETUP()                                                       \
  const uint32_t tbase = ctl->tmem_base;                                       \
  const Unit unit = decode_unit(a, PAIR == 2 ? (blockIdx.x >> 1) : blockIdx.x); \
  const TileSchedule sched = unit_schedule<MODE>(a, unit.qt, BC);              \
  const int N = sched.vmax;                                                    \
  int nrep = 0;                                                                \
  const int nchunks = minit_chunks<MODE>(a, sched, BC, &nrep);                 \
  const int G = nchunks + N;                                                   \
  (void)tbase; (void)nrep; (void)nchunks; (void)N; (void)G

  if (warp >= C::kSoftmaxWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kRegsOther));
    if (warp == C::kLoadWarp) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        VFA_ROLE_SETUP();
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        for (int t = 0; t < NQ; ++t) {
          if constexpr (PAIR == 2) {
            // both CTAs' Q tiles count on the leader's barrier (the pair MMA reads both)
            if (crank == 0) mbar_arrive_expect_tx(&ctl->q_full[t], 2 * C::kQBytes);
#pragma unroll
            for (int c = 0; c < C::kDCh; ++c)
              tma_load_4d_pair(sQ + t * C::kQBytes + c * kBR * 128, &tmQ, &ctl->q_full[t], c * 64, unit.qt * a.qrows,
                               head_of(unit, t), unit.b, pol_q);
          } else {
            mbar_arrive_expect_tx(&ctl->q_full[t], C::kQBytes);
#pragma unroll
            for (int c = 0; c < C::kDCh; ++c)
              tma_load_4d(sQ + t * C::kQBytes + c * kBR * 128, &tmQ, &ctl->q_full[t], c * 64, unit.qt * a.qrows,
                          head_of(unit, t), unit.b, pol_q);
          }
        }
        int stage = 0;
        uint32_t phase = 0;
        // K-like tiles (keys, key representations): all D columns of BC / PAIR rows; a pair's
        // CTA r loads rows [r*BC/2, (r+1)*BC/2). V tiles: all BC rows of D / PAIR columns.
        auto load_tile = [&](const CUtensorMap* map, int row, bool is_v) {
          mbar_wait(&ctl->kv_empty[stage], phase ^ 1);
          uint8_t* dst = sKV + stage * C::kKVBytes;
          if constexpr (PAIR == 2) {
            if (crank == 0) mbar_arrive_expect_tx(&ctl->kv_full[stage], 2 * C::kKVBytes);
            if (is_v) {
              tma_load_4d_pair(dst, map, &ctl->kv_full[stage], static_cast<int>(crank) * 64, row, unit.kvh, unit.b,
                               pol_kv);
            } else {
#pragma unroll
              for (int c = 0; c < C::kDCh; ++c)
                tma_load_4d_pair(dst + c * (BC / 2) * 128, map, &ctl->kv_full[stage], c * 64,
                                 row + static_cast<int>(crank) * (BC / 2), unit.kvh, unit.b, pol_kv);
            }
          } else {
            (void)is_v;
            mbar_arrive_expect_tx(&ctl->kv_full[stage], C::kKVBytes);
#pragma unroll
            for (int c = 0; c < C::kDCh; ++c)
              tma_load_4d(dst + c * BC * 128, map, &ctl->kv_full[stage], c * 64, row, unit.kvh, unit.b, pol_kv);
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        };
        // the MMA warp's consumption order: op(0 .. SB-1); per g: [V(g)], op(g+SB)
        auto load_s_operand = [&](int g) {
          if (g < nchunks)
            load_tile(&tmR, g * BC, false);
          else
            load_tile(&tmK, (sched_block(sched, g - nchunks) - 1) * BC, false);
        };
        for (int g = 0; g < SB && g < G; ++g) load_s_operand(g);
        for (int g = 0; g < G; ++g) {
          if (g >= nchunks) {
            load_tile(&tmV, (sched_block(sched, g - nchunks) - 1) * BC, true);
            VFA_TRACE_EVENT(a, g - nchunks, 15);
          }
          if (g + SB < G) {
            load_s_operand(g + SB);
            if (g >= nchunks) VFA_TRACE_EVENT(a, g - nchunks, 16);
          }
        }
      }
    } else if (warp == C::kMmaWarp && (PAIR == 1 || crank == 0)) {
      // ============================ MMA issuer ============================
      // (a CTA pair's MMAs are all issued by the leader, M = 256 over both CTAs' tiles)
      // The whole warp runs the issue loop (warp-uniform state in uniform registers); one
      // elected lane issues each tcgen05 instruction. Per element g and query tile t:
      // PV_t(g) then QK_t(g+1), so each tile's next S is issued as soon as its own P is
      // consumed and the two query tiles ping-pong (anti-phase) on the tensor pipe.
      VFA_ROLE_SETUP();
      constexpr uint32_t kIdescQK = make_idesc_bf16(128 * PAIR, BC, false, false);
      constexpr uint32_t kIdescPV = make_idesc_bf16(128 * PAIR, D, false, true);
      // pair: commits arrive on both CTAs' barriers (same offset)
      auto commit = [&](uint64_t* bar) {
        if constexpr (PAIR == 2) {
          if (elect_one()) mma_commit_pair(bar);
          __syncwarp();
        } else {
          commit_elect(bar);
        }
      };
      // UMMA smem descriptors: hi word constant (SBO = 1024 B, version 1, SWIZZLE_128B),
      // lo word = (address >> 4) | LBO << 16. Addresses < 256 KiB so the start field never carries.
      constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t kLboK = 1u << 16;                                      // K-major: LBO unused
      constexpr uint32_t kLboV = static_cast<uint32_t>((BC * 128) >> 4) << 16;  // V: next 64-col chunk
      const uint32_t q_lo = smem_u32(sQ) >> 4;
      const uint32_t kv_lo = smem_u32(sKV) >> 4;
      for (int t = 0; t < NQ; ++t) mbar_wait(&ctl->q_full[t], 0);
      tc_fence_after();
      if constexpr (C::kQT) {
        // Q_t -> TMEM (lane = row, 8 columns per 16-element K-step); executes ahead of the MMAs
        // issued after it by this thread (in-order tcgen05 pipe)
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < NQ; ++t)
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t oq = ((kk >> 2) * (kBR * 128) + (kk & 3) * 32) >> 4;
              const uint64_t da = (static_cast<uint64_t>(kHi) << 32) | (q_lo + t * (C::kQBytes >> 4) + kLboK + oq);
              tmem_cp_128x256b(tbase + C::kQBase + t * (D / 2) + kk * 8, da);
            }
        }
        __syncwarp();
      }
      int stage = 0;
      uint32_t phase = 0;
      auto acquire = [&]() -> int {
        mma_wait(&ctl->kv_full[stage], phase);
        tc_fence_after();
        int st = stage;
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
        return st;
      };
      // One elected lane issues a whole batch of MMAs straight-line (electing per instruction
      // costs an ELECT, uniform-register broadcasts and a reconvergence per MMA: the issue of
      // a QK^T then took longer than its 512-cycle execution, profiles/trace_r02b.txt).
      auto issue_qk = [&](int t, int b, int st) {
        const uint32_t a_lo = q_lo + t * (C::kQBytes >> 4) + kLboK;
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboK;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oq = ((kk >> 2) * (kBR * 128) + (kk & 3) * 32) >> 4;
            const uint32_t ok = ((kk >> 2) * ((BC / PAIR) * 128) + (kk & 3) * 32) >> 4;
            const uint64_t da = (static_cast<uint64_t>(kHi) << 32) | (a_lo + oq);
            const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + ok);
            if constexpr (PAIR == 2)
              mma_ss_pair(tbase + C::s_off(t, b), da, db, kIdescQK, kk > 0 ? 1u : 0u);
            else if constexpr (C::kQT)
              mma_ts(tbase + C::s_off(t, b), tbase + C::kQBase + t * (D / 2) + kk * 8, db, kIdescQK, kk > 0 ? 1u : 0u);
            else
              mma_ss(tbase + C::s_off(t, b), da, db, kIdescQK, kk > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      // P of part pp occupies TMEM columns [pp*CP, pp*CP + CP/2) of S_t (packed bf16 pairs).
      // PV chunk c: the K-steps over P columns [c*CW, c*CW + CW) of every part.
      auto issue_pv_chunk = [&](int t, int b, int st, int c, bool& first) {
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboV;
        const int k_lo = c == 0 ? 0 : C::kKS0, k_hi = c == 0 ? C::kKS0 : CP / 16;  // this chunk's K-steps
        if (elect_one()) {
          bool acc = !first;
#pragma unroll
          for (int pp = 0; pp < SPLIT; ++pp) {
#pragma unroll
            for (int k2 = k_lo; k2 < k_hi; ++k2) {
              const int kk = pp * (CP / 16) + k2;  // K-step (16 key rows of V)
              const uint32_t pcol = pp * CP + k2 * 8;
              const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + kk * (2048 >> 4));
              if constexpr (PAIR == 2)
                mma_ts_pair(tbase + C::kOBase + t * D, tbase + C::s_off(t, b) + pcol, db, kIdescPV, acc ? 1u : 0u);
              else
                mma_ts(tbase + C::kOBase + t * D, tbase + C::s_off(t, b) + pcol, db, kIdescPV, acc ? 1u : 0u);
              acc = true;
            }
          }
        }
        __syncwarp();
        first = false;
      };
      uint32_t o_init = 0, p_ph = 0;  // p_ph bit t*SB+b: p_full[t][b] phase (visited blocks only)
      auto issue_s_tile = [&](int g, int t, int st) {
        // the buffer's previous occupant g - SB: an m-init chunk must have been read (s_free);
        // a visited block's P was consumed by its PV, issued before this QK
        const int b = g % SB;
        if (g >= SB && g - SB < nchunks) {
          mbar_wait(&ctl->s_free[t][b], ((g - SB) / SB) & 1);
          tc_fence_after();
        }
        issue_qk(t, b, st);
        commit(&ctl->s_full[t][b]);
      };
      for (int g = 0; g < SB && g < G; ++g) {
        const int st = acquire();
        for (int t = 0; t < NQ; ++t) issue_s_tile(g, t, st);
        commit(&ctl->kv_empty[st]);
      }
      for (int g = 0; g < G; ++g) {
        const bool main_blk = g >= nchunks;
        const int pos = g - nchunks;
        const int b = g % SB;
        const bool next_s = g + SB < G;
        // SB 2: the softmax of the next exact-update block rescales O, so it waits for this PV
        const bool signal_pv = SB >= 2 && main_blk && pos + 1 < N &&
                               (all_exact(MODE) || sched_is_special(sched, sched_block(sched, pos + 1)));
        const int vs = main_blk ? acquire() : -1;
        if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 17);
        int ks = -1;
        for (int t = 0; t < NQ; ++t) {
          if (main_blk) {
            bool first = ((o_init >> t) & 1u) == 0;  // first PV of this tile initialises O
            bool skip = false;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              if constexpr (PAIR == 2 && skips(MODE))  // pairs with the follower's release
                mbar_wait_cluster(&ctl->p_full[t][b][c], (p_ph >> (t * SB + b)) & 1u);
              else
                mma_wait(&ctl->p_full[t][b][c], (p_ph >> (t * SB + b)) & 1u);
              tc_fence_after();
              if (c == 0) {
                if (lane == 0) VFA_TRACE_EVENT(a, pos, 4 + 2 * t);
                if constexpr (PAIR == 2)  // the pair's PV is skipped only if both tiles skip
                  skip = skips(MODE) && ctl->skip2[t][b][0] != 0 && ctl->skip2[t][b][1] != 0;
                else
                  skip = skips(MODE) && (ctl->skip[t][b] != 0);
              }
              if (c == NCH - 1 && lane == 0) VFA_TRACE_EVENT(a, pos, 8 + 2 * t);
              if (!skip) issue_pv_chunk(t, b, vs, c, first);
            }
            if (lane == 0) VFA_TRACE_EVENT(a, pos, 9 + 2 * t);
            p_ph ^= 1u << (t * SB + b);
            if (!skip) o_init |= 1u << t;
            if (signal_pv) commit(&ctl->pv_done[t]);
            if (t == NQ - 1) commit(&ctl->kv_empty[vs]);
          }
          if (next_s) {
            if (t == 0) ks = acquire();
            if (main_blk && t == 0 && lane == 0) VFA_TRACE_EVENT(a, pos, 12);
            issue_s_tile(g + SB, t, ks);
            if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 5 + 2 * t);
          }
        }
        if (ks >= 0) commit(&ctl->kv_empty[ks]);
      }
      for (int t = 0; t < NQ; ++t) commit(&ctl->o_final[t]);
    }
  } else {
    // ============================ softmax WGs ============================
    // Each row of a query tile is shared by SPLIT threads (TMEM lane r of SPLIT warpgroups),
    // each owning CP = BC/SPLIT S columns and OP = D/SPLIT O columns.
    //   SPLIT == 2: warpgroups 2t, 2t+1 serve query tile t only (two independent warp sets
    //               that run in anti-phase, each hiding under the other tile's MMA window);
    //   SPLIT == 4: all four warpgroups serve both tiles in turn (tile 0 then tile 1 of each
    //               key block): half the per-thread work per tile-block, one shared issue stream;
    //   SPLIT == 1: one warpgroup per tile, one thread per row (no row-max exchange).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kRegsSoftmax));
    constexpr int NT = C::kAllTiles ? NQ : 1;  // query tiles this thread serves
    const int part = C::kAllTiles ? (warp >> 2) : (SPLIT == 2 ? ((warp >> 2) & 1) : 0);
    const int tile0 = C::kAllTiles ? 0 : warp / (4 * SPLIT);
    if (tile0 < NQ) {
      const int r = tid & 127;
      VFA_ROLE_SETUP();
      const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const int R = unit.qt * a.qrows + r;  // absolute query row
      // rows past the reference block (q_block < 128) compute on the next block's queries and are
      // discarded: they vote "skippable" / "elidable", count nothing and store nothing
      const bool live = r < a.qrows;
      const float cs = a.c_scale;
      float m2[NT], l[NT];  // running max (log2 units of scaled scores; identical in all parts)
      uint32_t xpar[NT];    // and this part's share of the normalizer, per served tile
      // StateTrace stabilization (src/analysis.py:39-78): the block of the visit after which
      // the running max equals its final value = the last visit that raised it (or the first
      // visit when nothing raised it); the first record's block otherwise
      int stab[NT];
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) {
        m2[ti] = -INFINITY;
        l[ti] = 0.f;
        xpar[ti] = 0;
        stab[ti] = sched_block(sched, 0);
      }
      uint32_t over32 = 0, over16 = 0;
      float argmax = -INFINITY;  // monitor: largest exp argument (log2 units)
      uint32_t pv_ph = 0;  // bit ti: pv_done phase (SB 2)
      auto tS = [&](int t, int b) { return tbase + C::s_off(t, b) + part * CP + lane_off; };
      auto tO = [&](int t) { return tbase + C::kOBase + t * D + part * OP + lane_off; };
      // row-max exchange across the SPLIT parts of a row (named barrier 1 + t)
      auto exchange_max = [&](int ti, int t, float mine) -> float {
        if constexpr (SPLIT == 1) return mine;  // one thread holds the whole row
        ctl->xmax[t][xpar[ti]][part][r] = mine;
        named_bar_sync(1 + t, SPLIT * kBR);
        const float* x = ctl->xmax[t][xpar[ti]][0];
        float m = fmaxf(x[r], x[kBR + r]);
        if constexpr (SPLIT == 4) m = fmaxf(m, fmaxf(x[2 * kBR + r], x[3 * kBR + r]));
        xpar[ti] ^= 1;
        return m;
      };
      // sequence element g (m-init chunks, then visited blocks) lives in S buffer g % SB
      auto wait_s = [&](int t, int g) {
        if constexpr (VFA_SM_SPIN) mbar_wait_spin(&ctl->s_full[t][g % SB], (g / SB) & 1);
        else mbar_wait(&ctl->s_full[t][g % SB], (g / SB) & 1);
        tc_fence_after();
      };
      auto load_part = [&](int t, int b, float* v) {
        if constexpr (CP >= 32) {
#pragma unroll
          for (int c = 0; c < CP / 32; ++c) tmem_ld32(tS(t, b) + c * 32, v + c * 32);
        } else {
          tmem_ld16(tS(t, b), v);
        }
        tmem_wait_ld();
        if constexpr (CP >= 32) {
#pragma unroll
          for (int c = 0; c < CP / 32; ++c) reg_fence32(v + c * 32);
        } else {
          reg_fence16(v);
        }
      };

      // ---- m-init: m0 = max_j scale * q . krepr_j over visible j <= tc1 (src/vfa.py:91-106)
      if (nchunks > 0) {
        float mx[NT];
#pragma unroll
        for (int ti = 0; ti < NT; ++ti) mx[ti] = -INFINITY;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int valid = nrep - ch * BC - part * CP;
#pragma unroll
          for (int ti = 0; ti < NT; ++ti) {
            const int t = tile0 + ti;
            wait_s(t, ch);
            float v[CP];
            load_part(t, ch % SB, v);
#pragma unroll
            for (int e = 0; e < CP; ++e)
              if (e < valid) mx[ti] = fmaxf(mx[ti], v[e]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_mma(&ctl->s_free[t][ch % SB]);
          }
        }
#pragma unroll
        for (int ti = 0; ti < NT; ++ti) m2[ti] = exchange_max(ti, tile0 + ti, mx[ti]) * cs;
      }
      if ((MODE == kVFA || MODE == kVSA) && a.use_m_init && a.m0_tile != nullptr) {
        // block-wise query representation (src/vfa.py:104-106): one seed for the whole tile
#pragma unroll
        for (int ti = 0; ti < NT; ++ti)
          m2[ti] = a.m0_tile[(static_cast<size_t>(unit.b) * a.Hq + head_of(unit, tile0 + ti)) * a.Tr + unit.qt] * cs;
      }

      // monitor: the m-init seed and the exact row max over every visited block (calibration
      // gap, src/vfa.py:129-135); this thread's part of the row until the epilogue combines it
      float seed2[NT], emax[NT];
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) {
        seed2[ti] = m2[ti];
        emax[ti] = -INFINITY;
      }
      float rbias[NT];
#pragma unroll
      for (int ti = 0; ti < NT; ++ti)
        rbias[ti] = (a.row_bias != nullptr && live)
                        ? a.row_bias[(static_cast<size_t>(unit.b) * a.Hq + head_of(unit, tile0 + ti)) * a.Lq + R]
                        : 0.f;
      const float2 cs2 = make_float2(cs, cs);
      // block-class counts beyond the closed form (skip / elision / row-mask variants only)
      int n_skipped = 0, n_skipped_special = 0, n_elided = 0, n_rows_masked = 0;
      for (int pos = 0; pos < N; ++pos) {
        const int j = sched_block(sched, pos);
        const bool special = all_exact(MODE) || sched_is_special(sched, j);
        const bool mask = sched_needs_mask(unit.qt + 1, j, a.qrows, BC, a.causal != 0);
        const int lim = R - (j - 1) * BC - part * CP;  // this part's columns > lim are masked
#pragma unroll
        for (int ti = 0; ti < NT; ++ti) {
          const int t = tile0 + ti;
          const int g = nchunks + pos;
          const int b = g % SB;
          if (r == 0 && part == 0) VFA_TRACE_EVENT(a, pos, 13 + t);
          wait_s(t, g);
          if (r == 0 && part == 0) VFA_TRACE_EVENT(a, pos, 2 * t);
          if (r == 0 && part == 0 && t == 0 && pos == 0) VFA_TRACE_UNIT(a, 1);
          float v[CP];
          load_part(t, b, v);
          if (mask) {  // entrywise causal mask (src/reference.py:93-96): exact zeros after exp2
#pragma unroll
            for (int e = 0; e < CP; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
          }
          // monitor only: the frozen block's part max for the exact global row max
          if (MODE == kVFA && !special && a.monitor) emax[ti] = fmaxf(emax[ti], part_max<CP>(v) * cs);
          bool skipped = false;
          bool rescale = false;  // this block rescales O by f (exact update, not skipped / elided)
          float f = 1.0f;
          if (MODE == kVSA && !special) {
            // ---- VSA frozen block: only the skip test (src/sparse.py:296-304). A row is below
            //      the threshold iff every part's maximum is (m~ = max over parts, and a part
            //      holding m~ > m fails the test), so one CTA-wide AND over the part maxima
            //      decides without exchanging row maxima; the frozen max is not updated.
            const float pm = part_max<CP>(v);
            const float pm2 = pm * cs;
            if (a.monitor) emax[ti] = fmaxf(emax[ti], pm2);
            const bool below = (pm2 - fmaxf(m2[ti], pm2) < a.log2_lambda) ||
                               (pm2 == -INFINITY && m2[ti] == -INFINITY && a.log2_lambda != -INFINITY) || !live;
            skipped = named_bar_and(1 + t, SPLIT * kBR, below);
            if (skipped) ++n_skipped;
          } else if (MODE != kVFA || special) {
            // ---- exact-update / skip-test block: rowmax over the full row (all parts,
            //      src/vfa.py:202-208, src/sparse.py:296-300), then rescale
            const float mt = exchange_max(ti, t, part_max<CP>(v));
            const float mt2 = mt * cs;
            if (a.monitor) emax[ti] = fmaxf(emax[ti], mt2);
            const float m2n = fmaxf(m2[ti], mt2);
            bool keep = true;  // rowskip: this row takes part in the update
            if (MODE == kBLR) {
              // row-granular threshold (src/sparse.py:223-227): NaN (dead row) is not kept
              keep = live && ((a.log2_lambda == -INFINITY) || (mt2 - m2n >= a.log2_lambda));
              skipped = named_bar_and(1 + t, SPLIT * kBR, !keep);
            } else if (skips(MODE)) {
              const bool below = (mt2 - m2n < a.log2_lambda) ||
                                 (mt2 == -INFINITY && m2n == -INFINITY && a.log2_lambda != -INFINITY) || !live;
              skipped = named_bar_and(1 + t, SPLIT * kBR, below);
            }
            bool elide = false;
            if (MODE == kBL4 && !skipped) {
              // rescale elision (src/sparse.py:187-193): every row had a finite max and none rose
              // by more than tau*ln2 -> keep the old max, factor exactly 1
              elide = named_bar_and(1 + t, SPLIT * kBR, (m2[ti] != -INFINITY && m2n - m2[ti] <= a.tau) || !live);
              n_elided += elide ? 1 : 0;
            }
            if (MODE == kBLR && live) n_rows_masked += (skipped || !keep) ? 1 : 0;
            if (skipped) {
              ++n_skipped;
              n_skipped_special += special ? 1 : 0;
            } else if (special && !elide) {
              // (warp-uniform branch: skipped / elide are CTA-wide decisions) rowskip: a
              // suppressed row keeps factor 1 and its max, and adds zero mass (src/sparse.py:241-247)
              const bool upd = (MODE != kBLR) || keep;
              f = (!upd || m2n == -INFINITY) ? 1.0f : ex2_approx(m2[ti] - m2n);
              if (upd && m2n > m2[ti]) stab[ti] = j;
              if (upd) m2[ti] = m2n;
              if (!upd) {
#pragma unroll
                for (int e = 0; e < CP; ++e) v[e] = -INFINITY;
              }
              l[ti] = __fmul_rn(l[ti], f);  // no FMA contraction: identical l-recurrence in every mode
              rescale = pos > 0 && ((MODE == kFA) || !__all_sync(0xffffffffu, f == 1.0f));
            }
          }
          // rescale this part of O in TMEM (src/core.py:91) before PV(pos) accumulates into it
          auto rescale_o = [&]() {
            const float2 f2 = make_float2(f, f);
#pragma unroll(SPLIT == 4 ? 2 : 1)
            for (int c = 0; c < OP / 16; ++c) {
              float o[16];
              tmem_ld16(tO(t) + c * 16, o);
              tmem_wait_ld();
              reg_fence16(o);
              uint32_t u[16];
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                const float2 x = __fmul2_rn(make_float2(o[e], o[e + 1]), f2);
                u[e] = __float_as_uint(x.x);
                u[e + 1] = __float_as_uint(x.y);
              }
              tmem_st16(tO(t) + c * 16, u);
            }
          };
          // SB 1: O is quiescent here (PV(pos-1) completed before S(pos): in-order tensor pipe).
          // SB 2: S(pos) was computed before PV(pos-1) was issued, so an exact block waits for
          // PV(pos-1) (pv_done, committed by the MMA warp ahead of every exact block) and hands
          // its P over only after the rescale.
          const bool defer = SB >= 2 && special && pos > 0;
          if (SB == 1 && rescale) rescale_o();
          // ---- frozen blocks (src/vfa.py:209-215) skip all of the above: no rowmax, no rescale
          if (r == 0 && part == 0) {
            if (skips(MODE)) {
              if constexpr (PAIR == 2)  // the leader's MMA warp needs both CTAs' decisions
                st_cluster_u32(mapa_shared(&ctl->skip2[t][b][crank], 0), skipped ? 1u : 0u);
              else
                ctl->skip[t][b] = skipped ? 1u : 0u;
            }
            if (a.skip_trace) {
              const size_t idx =
                  ((static_cast<size_t>(unit.b) * a.Hq + head_of(unit, t)) * a.Tr + unit.qt) * a.Tc + pos;
              a.skip_trace[idx] = skipped ? 2 : 1;
            }
          }
          if (!skipped) {
            // P = exp2(S*c - m2) in CW-column chunks; each chunk is handed to the MMA warp as
            // soon as it is in TMEM (PV of chunk 0 overlaps the softmax of chunk 1)
            const float nm = (m2[ti] == -INFINITY ? 0.f : -m2[ti]) + rbias[ti];
            const float2 nmu2 = make_float2(nm, nm);
            float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            if constexpr (C::kS1Split) {
              // 32-column sub-chunks; hand-off after 96 columns (PV K-steps 0-5) and after 128
#pragma unroll
              for (int sc = 0; sc < 4; ++sc) {
                uint32_t u[16];
                constexpr int kP1 = VFA_POLY_S1;
                if (a.monitor)
                  p_chunk<32, true, 0, kLate>(v + sc * 32, cs2, nmu2, u, acc, over32, over16, argmax);
                else if (sc == 1 || sc == 2)
                  p_chunk<32, false, kP1, kLate>(v + sc * 32, cs2, nmu2, u, acc, over32, over16, argmax);
                else
                  p_chunk<32, false, 0, kLate>(v + sc * 32, cs2, nmu2, u, acc, over32, over16, argmax);
                tmem_st16(tS(t, b) + sc * 16, u);
                if (!defer && (sc == 2 || sc == 3)) {
                  tmem_wait_st();
                  tc_fence_before();
                  __syncwarp();
                  const int c = sc == 2 ? 0 : 1;
                  if (lane == 0) arrive_mma(&ctl->p_full[t][b][c], skips(MODE) && (warp & 3) == 0 && part == 0 && c == 0);
                }
              }
            } else {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              uint32_t u[CW / 2];
              if (a.monitor)
                p_chunk<CW, true, kPoly, kLate>(v + c * CW, cs2, nmu2, u, acc, over32, over16, argmax);
              else if (VFA_POLY_SMSP0 > 0 && (warp & 3) == 0)  // the MMA issuer's sub-partition
                p_chunk<CW, false, VFA_POLY_SMSP0, kLate>(v + c * CW, cs2, nmu2, u, acc, over32, over16, argmax);
              else
                p_chunk<CW, false, kPoly, kLate>(v + c * CW, cs2, nmu2, u, acc, over32, over16, argmax);
              if constexpr (CW == 64) tmem_st32(tS(t, b) + c * 32, u);
              else if constexpr (CW == 32) tmem_st16(tS(t, b) + c * 16, u);
              else tmem_st8(tS(t, b) + c * 8, u);
              if (!defer) {
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_mma(&ctl->p_full[t][b][c], skips(MODE) && (warp & 3) == 0 && part == 0 && c == 0);
              }
            }
            }
            if constexpr (kLate) late_rowsum<NCH * CW>(v, acc);
            l[ti] = __fadd_rn(l[ti], __fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)));
          }
          if (defer) {
            mbar_wait(&ctl->pv_done[t], (pv_ph >> ti) & 1u);
            pv_ph ^= 1u << ti;
            tc_fence_after();
            if (rescale) rescale_o();
          }
          if constexpr (PAIR == 2) {
            if (skipped) {  // the pair's PV still runs if the other tile keeps the block: P = 0
              uint32_t z[CW / 2];
#pragma unroll
              for (int e = 0; e < CW / 2; ++e) z[e] = 0u;
#pragma unroll
              for (int c = 0; c < NCH; ++c) {
                if constexpr (CW == 32) tmem_st16(tS(t, b) + c * 16, z);
                else tmem_st8(tS(t, b) + c * 8, z);
              }
            }
          }
          if (skipped || defer) {
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
              for (int c = 0; c < NCH; ++c) arrive_mma(&ctl->p_full[t][b][c], skips(MODE) && (warp & 3) == 0 && part == 0 && c == 0);
          }
          if (a.m_trace != nullptr && part == 0 && live)  // (debug output: one store per row and visit)
            a.m_trace[((static_cast<size_t>(unit.b) * a.Hq + head_of(unit, t)) * a.Lq + R) * a.Tc + pos] = m2[ti] * kLn2;
          if (r == 0 && part == 0) VFA_TRACE_EVENT(a, pos, 2 * t + 1);
          if (r == 0 && part == 0 && pos == N - 1 && t == NQ - 1) VFA_TRACE_UNIT(a, 2);
        }
      }
      const int n_exact = all_exact(MODE) ? N : sched.n_spec;  // exact-update blocks per tile
      const int n_special = NT * n_exact - n_skipped_special - n_elided;
      const int n_frozen = NT * (N - n_exact) - (n_skipped - n_skipped_special) + n_elided;

      // ---- epilogue: O / l (src/core.py:101-109), LSE = m + ln l; l = sum over the parts
      bool any_nonfinite = false;
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) {
        const int t = tile0 + ti;
        const int h = head_of(unit, t);
        if (a.monitor && a.stats && (MODE == kVFA || MODE == kVSA) && a.use_m_init) {
          // OverflowMonitor.record_gap (src/vfa.py:129-135): m seed - exact global row max
          const float ex = exchange_max(ti, t, emax[ti]);
          if (part == 0) {
            const float gap = seed2[ti] - ex;
            const unsigned gmax = __reduce_max_sync(0xffffffffu, live ? float_key(gap) : 0u);
            const unsigned gneg = __reduce_max_sync(0xffffffffu, live ? float_key(-gap) : 0u);
            const unsigned below = __popc(__ballot_sync(0xffffffffu, live && gap < 0.f));
            const unsigned rows = __popc(__ballot_sync(0xffffffffu, live));
            float gsum = live ? gap : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
            if (lane == 0 && rows) {
              atomicMax(&a.stats[VFA_STAT_GAP_MAX], static_cast<unsigned long long>(gmax));
              atomicMax(&a.stats[VFA_STAT_GAP_NEG_MIN], static_cast<unsigned long long>(gneg));
              atomicAdd(reinterpret_cast<double*>(&a.stats[VFA_STAT_GAP_SUM]), static_cast<double>(gsum));
              atomicAdd(&a.stats[VFA_STAT_GAP_BELOW], static_cast<unsigned long long>(below));
              atomicAdd(&a.stats[VFA_STAT_GAP_ROWS], static_cast<unsigned long long>(rows));
            }
          }
        }
        float lsum = l[ti];
        if constexpr (SPLIT > 1) {
          ctl->xl[t][part][r] = l[ti];
          named_bar_sync(1 + t, SPLIT * kBR);
          lsum = __fadd_rn(ctl->xl[t][0][r], ctl->xl[t][1][r]);
          if constexpr (SPLIT == 4) lsum = __fadd_rn(lsum, __fadd_rn(ctl->xl[t][2][r], ctl->xl[t][3][r]));
        }
        mbar_wait(&ctl->o_final[t], 0);
        tc_fence_after();
        const float inv = 1.0f / lsum;
        __nv_bfloat16* orow =
            a.o + unit.b * a.o_sb + h * a.o_sh + static_cast<long long>(R) * a.o_sr + part * OP;
        bool finite = true;
#pragma unroll
        for (int c = 0; c < OP / 16; ++c) {
          float v[16];
          tmem_ld16(tO(t) + c * 16, v);
          tmem_wait_ld();
          reg_fence16(v);
          uint32_t u[8];
#pragma unroll
          const bool col_ok = part * OP + c * 16 < a.dv;  // (head_dim 32: padded columns are not O)
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float o0 = v[e] * inv, o1 = v[e + 1] * inv;
            finite = finite && (!col_ok || (isfinite(o0) && isfinite(o1)));
            u[e >> 1] = pack_bf16x2(o0, o1);
          }
          if (live && col_ok) {  // (the TMEM load above is warp-collective: idle lanes take part)
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
            dst[0] = make_uint4(u[0], u[1], u[2], u[3]);
            dst[1] = make_uint4(u[4], u[5], u[6], u[7]);
          }
        }
        const size_t lrow = (static_cast<size_t>(unit.b) * a.Hq + h) * a.Lq + R;
        const unsigned srow = static_cast<unsigned>(lrow + a.row_base);  // whole-problem row for the status
        finite = finite || !live;
        // (a row whose fp32 normalizer underflowed, l == 0 with a finite max, reports that max
        // instead, for the host's rebase, src/core.py:101-109 / vfa_fwd_rebased)
        if (part == 0 && live && a.lse)
          a.lse[lrow] = (lsum == 0.f && m2[ti] != -INFINITY) ? m2[ti] * kLn2 : (m2[ti] - rbias[ti] + __log2f(lsum)) * kLn2;
        if (part == 0 && live && a.stab) a.stab[lrow] = stab[ti];
        if (a.status) {
          if (part == 0 && live && lsum == 0.f) {
            if (m2[ti] == -INFINITY) {
              atomicOr(&a.status[VFA_STATUS_FLAGS], 1u);
              atomicMin(&a.status[VFA_STATUS_MASKED_ROW], srow);
            } else {
              atomicOr(&a.status[VFA_STATUS_FLAGS], 2u);
              atomicMin(&a.status[VFA_STATUS_UNDERFLOW_ROW], srow);
            }
          }
          // a row is non-finite if any part is: combine through smem, count it once
          bool row_ok = finite;
          if constexpr (SPLIT > 1) {
            ctl->xfin[t][part][r] = finite ? 1 : 0;
            named_bar_sync(1 + t, SPLIT * kBR);
            row_ok = ctl->xfin[t][0][r] && ctl->xfin[t][1][r];
            if constexpr (SPLIT == 4) row_ok = row_ok && ctl->xfin[t][2][r] && ctl->xfin[t][3][r];
          }
          if (part == 0 && !row_ok) any_nonfinite = true, atomicAdd(&a.status[VFA_STATUS_NONFINITE_ROWS], 1u);
        }
      }
      if (any_nonfinite) atomicOr(&a.status[VFA_STATUS_FLAGS], 4u);
      if (a.stats) {
        if (a.monitor) {
          if (live) {
            atomicAdd(&a.stats[VFA_STAT_OVER_F32], static_cast<unsigned long long>(over32));
            atomicAdd(&a.stats[VFA_STAT_OVER_F16], static_cast<unsigned long long>(over16));
          }
          const unsigned km = __reduce_max_sync(0xffffffffu, (live && argmax > -INFINITY) ? float_key(argmax) : 0u);
          if (lane == 0 && km) atomicMax(&a.stats[VFA_STAT_EXP_ARG_MAX], static_cast<unsigned long long>(km));
        }
        if (MODE == kBLR && part == 0) {
          const unsigned masked = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(n_rows_masked));
          if (lane == 0) atomicAdd(&a.stats[VFA_STAT_ROWS_MASKED], static_cast<unsigned long long>(masked));
        }
        if (r == 0 && part == 0) {
          if (MODE == kBL4) atomicAdd(&a.stats[VFA_STAT_ELIDED], static_cast<unsigned long long>(n_elided));
          atomicAdd(&a.stats[VFA_STAT_VISITED], static_cast<unsigned long long>(NT * N));
          atomicAdd(&a.stats[VFA_STAT_SKIPPED], static_cast<unsigned long long>(n_skipped));
          atomicAdd(&a.stats[VFA_STAT_SPECIAL], static_cast<unsigned long long>(n_special));
          atomicAdd(&a.stats[VFA_STAT_FROZEN], static_cast<unsigned long long>(n_frozen));
        }
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR == 2) cluster_sync_all();  // the peer may still be reading our smem / TMEM
  if (tid == 0) VFA_TRACE_UNIT(a, 3);
  if (warp == C::kMmaWarp) {
    tc_fence_after();
    if constexpr (PAIR == 2)
      tmem_dealloc_pair<C::kTmemCols>(ctl->tmem_base);
    else
      tmem_dealloc<C::kTmemCols>(ctl->tmem_base);
  }
}

// ------------------------------------------------------------------------------------
// Key-block representations (src/vfa.py:47-88): one warp per key block, lane owns
// D/32 consecutive columns; sabsmax keeps the first row on ties (strict >).
// Also computes the block-wise query representations (src/vfa.py:69-76) over 128-row query
// tiles (q_sabsmax = sabsmax, q_absmax = k_absmax_unsigned, q_mean = k_mean), and, with
// jb0 > 0, refreshes only blocks [jb0, nblk) (append-only K cache).
template <int D>
__global__ void __launch_bounds__(128) krepr_kernel(const __nv_bfloat16* __restrict__ k, long long sb, long long sh,
                                                    long long sr, int Hkv, int BC, int nblk, int kind,
                                                    __nv_bfloat16* __restrict__ out, int jb0 = 0) {
  constexpr int CPL = D / 32;  // columns per lane (1, 2 or 4)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jb = jb0 + blockIdx.x * 4 + warp;
  const int kvh = blockIdx.y, b = blockIdx.z;
  if (jb >= nblk) return;
  const __nv_bfloat16* base = k + b * sb + kvh * sh + static_cast<long long>(jb) * BC * sr + lane * CPL;
  float best[CPL], val[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    best[c] = kind == VFA_KREPR_K_MEAN ? 0.f : -INFINITY;
    val[c] = 0.f;
  }
#pragma unroll 8
  for (int row = 0; row < BC; ++row) {
    float x[CPL];
    if constexpr (CPL == 4) {
      const uint2 raw = *reinterpret_cast<const uint2*>(base + row * sr);
      const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
      const __nv_bfloat162 p1 = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
      x[0] = __low2float(p0);
      x[1] = __high2float(p0);
      x[2] = __low2float(p1);
      x[3] = __high2float(p1);
    } else if constexpr (CPL == 2) {
      const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(base + row * sr);
      x[0] = __low2float(p0);
      x[1] = __high2float(p0);
    } else {
      x[0] = __bfloat162float(base[row * sr]);
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      switch (kind) {
        case VFA_KREPR_SABSMAX:
          if (fabsf(x[c]) > best[c]) {
            best[c] = fabsf(x[c]);
            val[c] = x[c];
          }
          break;
        case VFA_KREPR_K_MAX:
          best[c] = fmaxf(best[c], x[c]);
          break;
        case VFA_KREPR_K_MEAN:
          best[c] += x[c];
          break;
        default:
          best[c] = fmaxf(best[c], fabsf(x[c]));
          break;
      }
    }
  }
  __nv_bfloat16* dst = out + ((static_cast<long long>(b) * Hkv + kvh) * nblk + jb) * D + lane * CPL;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    float r = kind == VFA_KREPR_SABSMAX ? val[c] : (kind == VFA_KREPR_K_MEAN ? best[c] / BC : best[c]);
    dst[c] = __float2bfloat16_rn(r);
  }
}

// Block-wise m-init seed (src/vfa.py:104-106): per query tile i, max over the visible key
// representations j <= min(vmax_i, nrep) of qrepr_i . krepr_j (raw, unscaled; fp32 dot).
// One warp per (batch, query head, tile); lane owns D/32 dimensions.
template <int D>
__global__ void __launch_bounds__(128) minit_block_kernel(const __nv_bfloat16* __restrict__ qrep,
                                                          const __nv_bfloat16* __restrict__ krep, int Hq, int Hkv,
                                                          int Tr, int QR, int nrep, int BC, int Tc, int causal,
                                                          float* __restrict__ m0) {
  constexpr int CPL = D / 32;
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z;
  if (w >= Tr) return;
  const int i = w + 1;  // 1-based query tile
  const int vmax = causal ? min((i * QR - 1) / BC + 1, Tc) : Tc;  // QR = q_block
  const int cap = vmax < nrep ? vmax : nrep;
  const int kvh = h / (Hq / Hkv);
  float qv[CPL];
  const __nv_bfloat16* qp = qrep + ((static_cast<size_t>(b) * Hq + h) * Tr + w) * D + lane * CPL;
#pragma unroll
  for (int c = 0; c < CPL; ++c) qv[c] = __bfloat162float(qp[c]);
  const __nv_bfloat16* kp = krep + (static_cast<size_t>(b) * Hkv + kvh) * nrep * D + lane * CPL;
  float best = -INFINITY;
  for (int j = 0; j < cap; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc = fmaf(qv[c], __bfloat162float(kp[static_cast<size_t>(j) * D + c]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    best = fmaxf(best, acc);
  }
  if (lane == 0) m0[(static_cast<size_t>(b) * Hq + h) * Tr + w] = best;
}

}  // namespace vfa
