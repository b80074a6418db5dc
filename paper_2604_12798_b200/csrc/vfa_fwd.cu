// B200 (sm_100a) VFA / VSA / FA attention forward.
//
// One CTA = one work unit = (batch b, KV head, NQ query heads of that KV head's
// GQA group, one 128-row query tile). The NQ query tiles share every K/V tile
// loaded into shared memory and share the tile schedule (same rows => same
// causal extent, same sink/local blocks).
//
// Warp roles (16 warps):
//   warps 0-3   softmax WG for query tile 0   (thread r owns row r, TMEM lane r)
//   warps 4-7   softmax WG for query tile 1
//   warps 8-11  correction WG: O rescale in TMEM on exact-update blocks only
//   warp 12     MMA issuer (one thread), TMEM allocator
//   warp 13     TMA producer (one thread)
//   warps 14-15 idle
// TMEM (512 columns): S_t at t*128 (P_t bf16 aliased over its first BC/2 columns),
// O_t at 256 + t*D.
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
// warps 0-15: four softmax warpgroups (2 query tiles x 2 column halves); warp 16: MMA
// issuer (both query tiles, strictly alternating) + TMEM allocator; warp 17: TMA producer;
// warps 18-19 complete the last warpgroup. (One issuer per tile was measured slower: the
// tiles drift into phase and contend for the softmax issue slots.)
constexpr int kSoftmaxWarps = 16;
constexpr int kMmaWarp = 16;
constexpr int kLoadWarp = 17;
constexpr int kThreads = 640;
// setmaxnreg budgets. The CTA's register pool is what the launch allocated
// (threads x compiled registers/thread, 640 x 96 = 61440); asking for more than the pool
// blocks setmaxnreg.inc forever, so the host checks this budget before launching.
constexpr int kRegsSoftmax = 104;
constexpr int kRegsOther = 56;
constexpr int kRegBudget = kSoftmaxWarps * 32 * kRegsSoftmax + (kThreads - kSoftmaxWarps * 32) * kRegsOther;
constexpr int kMaxSmem = 227 * 1024;
constexpr float kLn2 = 0.6931471805599453f;

enum Mode { kFA = 0, kVFA = 1, kVSA = 2 };

struct FwdArgs {
  int B, Hq, Hkv, Lq, Lk, group, Tr, Tc;
  int units_per_kvh, heads_per_unit;
  float c_scale;      // softmax scale * log2(e)
  float log2_lambda;  // skip threshold in log2 units (-inf: no skipping)
  int causal, reorder, use_m_init, nrep_cap, n_sink, n_local, monitor;
  __nv_bfloat16* o;
  long long o_sb, o_sh, o_sr;
  float* lse;
  unsigned long long* stats;
  unsigned int* status;
  unsigned char* skip_trace;
  long long row_base;  // linear-row offset of this launch's (b=0, h=0, r=0) in the status word
  long long* trace;  // debug: per-visit clock64 events of CTA 0 (vfa_debug_trace), or null
};

// debug timeline slots per visited block (CTA 0 only, builds with -DVFA_TRACE): softmax t:
// S ready, P done; MMA t: P observed, next QK issued
constexpr int kTraceSlots = 16;
#ifdef VFA_TRACE
#define VFA_TRACE_EVENT(args, pos, slot)                                                     \
  do {                                                                                       \
    if ((args).trace != nullptr && blockIdx.x == 0) (args).trace[(pos) * kTraceSlots + (slot)] = clock64(); \
  } while (0)
#else
#define VFA_TRACE_EVENT(args, pos, slot) \
  do {                                   \
  } while (0)
#endif

template <int D, int BC, int NQ, int SPLIT>
struct Cfg {
  static constexpr int kQBytes = kBR * D * 2;
  static constexpr int kKVBytes = BC * D * 2;
  static constexpr int kDCh = D / 64;  // 64-column (128-byte) swizzle chunks
  // softmax column split: each row of a tile is shared by SPLIT threads (one per warpgroup)
  static constexpr int kCP = BC / SPLIT;             // S columns per part
  static constexpr int kOP = D / SPLIT;              // O columns rescaled / stored per part
  static constexpr int kNCH = kCP >= 32 ? 2 : 1;     // P hand-off chunks per block
  static constexpr int kCW = kCP / kNCH;             // columns per P chunk (16 or 32)
  static constexpr int kWarpsPerTile = SPLIT * 4;    // softmax warps covering one tile
  static constexpr int kCtlBytes = 16384;
  static constexpr int kAvail = kMaxSmem - 1024 - kCtlBytes - NQ * kQBytes;
  static constexpr int kStagesRaw = kAvail / kKVBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmem = 1024 + NQ * kQBytes + kStages * kKVBytes + kCtlBytes;
  // TMEM: S_t (BC fp32 columns; P_t aliased as packed bf16 inside each half's region), O_t.
  static __host__ __device__ constexpr uint32_t s_off(int t) { return static_cast<uint32_t>(t * 128); }
  static constexpr int kOBase = NQ * 128;
  static constexpr int kColsUsed = kOBase + NQ * D;
  static constexpr uint32_t kTmemCols = kColsUsed <= 256 ? 256 : 512;
  static_assert(kColsUsed <= 512, "TMEM over-subscribed");
  static_assert(kStages >= 3, "not enough shared memory for a K/V ring");
  static_assert(kCW % 16 == 0 && kOP % 16 == 0, "parts must be whole 16-column chunks");
  static_assert(SPLIT == 2 || SPLIT == 4, "SPLIT is 2 (per-tile warp sets) or 4 (all warps, both tiles)");
};

template <int NS, int NQ>
struct __align__(16) Ctl {
  uint64_t q_full[NQ];
  uint64_t kv_full[NS];
  uint64_t kv_empty[NS];
  uint64_t s_full[NQ];     // MMA -> softmax: S of sequence element g ready
  uint64_t s_free[NQ];     // softmax -> MMA: m-init chunk read (16 warps)
  uint64_t p_full[NQ][2];  // softmax -> MMA: P chunk c (16 columns of each quarter = one PV
                           // K-step per quarter) ready / skip decided (16 warps)
  uint64_t o_final[NQ];    // MMA -> epilogue: last PV completed
  uint32_t tmem_base;
  uint32_t skip[NQ];
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
  return make_schedule(qt + 1, kBR, BC, a.Tc, a.causal != 0, a.n_sink, a.n_local,
                       MODE == kFA ? false : (a.reorder != 0), MODE == kFA);
}

// number of m-init chunks (BC representations per chunk)
template <int MODE>
__device__ __forceinline__ int minit_chunks(const FwdArgs& a, const TileSchedule& s, int BC, int* nrep) {
  if (MODE == kFA || !a.use_m_init) {
    *nrep = 0;
    return 0;
  }
  int n = s.vmax < a.nrep_cap ? s.vmax : a.nrep_cap;
  *nrep = n;
  return (n + BC - 1) / BC;
}


// tcgen05.commit from one elected lane of the (converged) MMA warp.
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  if (elect_one()) mma_commit(bar);
  __syncwarp();
}

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
// energy (lower clocks) than it saves in MUFU time: measured best is 0 for both softmax
// splits (profiles/ab_r01_poly.txt); the polynomial stays as a tuning knob. Kept identical
// for every split so P (hence O) does not depend on the split.
__host__ __device__ constexpr int poly_pairs() { return kPolyOverride >= 0 ? kPolyOverride : 0; }
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

template <bool MON>
__device__ __forceinline__ void count_over(float2 x, uint32_t& o32, uint32_t& o16) {
  if (MON) {
    // OverflowMonitor (src/vfa.py:122-128) thresholds, in log2 units
    o32 += (x.x > 128.0f) + (x.y > 128.0f);
    o16 += (x.x > 15.999295f) + (x.y > 15.999295f);
  }
}

// W consecutive columns (masked entries already -inf): P = exp2(s*cs - m2) -> W/2 packed
// bf16x2 words; row sums into two independent packed accumulators (halves the FADD2 chain).
template <int W, bool MON, int kPoly>
__device__ __forceinline__ void p_chunk(const float* v, float2 cs2, float2 nmu2, uint32_t* u, float2 (&acc)[2],
                                        uint32_t& o32, uint32_t& o16) {
#pragma unroll
  for (int e = 0; e < W; e += 2) {
    const float2 x = __ffma2_rn(make_float2(v[e], v[e + 1]), cs2, nmu2);
    count_over<MON>(x, o32, o16);
    float2 p;
    if (((e >> 1) & 7) < kPoly) {
      p = ex2_poly2(x);
    } else {
      p.x = ex2_approx(x.x);
      p.y = ex2_approx(x.y);
    }
    acc[(e >> 1) & 1] = __fadd2_rn(acc[(e >> 1) & 1], p);
    u[e >> 1] = pack_bf16x2(p.x, p.y);
  }
}

// ------------------------------------------------------------------------------------
template <int D, int BC, int NQ, int MODE, int SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    vfa_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmR,
                   const FwdArgs a) {
  using C = Cfg<D, BC, NQ, SPLIT>;
  constexpr int NS = C::kStages;
  constexpr int CP = C::kCP;
  constexpr int OP = C::kOP;
  constexpr int NCH = C::kNCH;
  constexpr int CW = C::kCW;
  constexpr int kPoly = poly_pairs();
  using CtlT = Ctl<NS, NQ>;
  static_assert(sizeof(CtlT) <= C::kCtlBytes, "control block too large");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + NQ * C::kQBytes;
  CtlT* ctl = reinterpret_cast<CtlT*>(sKV + NS * C::kKVBytes);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&ctl->q_full[t], 1);
      mbar_init(&ctl->s_full[t], 1);
      mbar_init(&ctl->s_free[t], C::kWarpsPerTile);
      mbar_init(&ctl->p_full[t][0], C::kWarpsPerTile);
      mbar_init(&ctl->p_full[t][1], C::kWarpsPerTile);
      mbar_init(&ctl->o_final[t], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&ctl->kv_full[s], 1);
      mbar_init(&ctl->kv_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == kLoadWarp && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmR);
  }
  if (warp == kMmaWarp) tmem_alloc<C::kTmemCols>(&ctl->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Each role re-derives its work description after its setmaxnreg so that nothing
  // computed before the role split has to stay live (or spill) across it.
  // Sequence g = 0 .. G-1: nchunks m-init chunks (S = Q . Krepr^T), then the N visited
  // key blocks in schedule order (S = Q . K^T).
#define VFA_ROLE_SETUP()                                                       \
  const uint32_t tbase = ctl->tmem_base;                                       \
  const Unit unit = decode_unit(a, blockIdx.x);                                \
  const TileSchedule sched = unit_schedule<MODE>(a, unit.qt, BC);              \
  const int N = sched.vmax;                                                    \
  int nrep = 0;                                                                \
  const int nchunks = minit_chunks<MODE>(a, sched, BC, &nrep);                 \
  const int G = nchunks + N;                                                   \
  (void)tbase; (void)nrep; (void)nchunks; (void)N; (void)G

  if (warp >= kSoftmaxWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsOther));
    if (warp == kLoadWarp) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        VFA_ROLE_SETUP();
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        for (int t = 0; t < NQ; ++t) {
          mbar_arrive_expect_tx(&ctl->q_full[t], C::kQBytes);
#pragma unroll
          for (int c = 0; c < C::kDCh; ++c)
            tma_load_4d(sQ + t * C::kQBytes + c * kBR * 128, &tmQ, &ctl->q_full[t], c * 64, unit.qt * kBR,
                        unit.h0 + t, unit.b, pol_q);
        }
        int stage = 0;
        uint32_t phase = 0;
        auto load_tile = [&](const CUtensorMap* map, int row) {
          mbar_wait(&ctl->kv_empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&ctl->kv_full[stage], C::kKVBytes);
          uint8_t* dst = sKV + stage * C::kKVBytes;
#pragma unroll
          for (int c = 0; c < C::kDCh; ++c)
            tma_load_4d(dst + c * BC * 128, map, &ctl->kv_full[stage], c * 64, row, unit.kvh, unit.b, pol_kv);
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        };
        // the MMA warp's consumption order: op(0); per g: [V(g)], op(g+1)
        auto load_s_operand = [&](int g) {
          if (g < nchunks)
            load_tile(&tmR, g * BC);
          else
            load_tile(&tmK, (sched_block(sched, g - nchunks) - 1) * BC);
        };
        load_s_operand(0);
        for (int g = 0; g < G; ++g) {
          if (g >= nchunks) load_tile(&tmV, (sched_block(sched, g - nchunks) - 1) * BC);
          if (g + 1 < G) load_s_operand(g + 1);
        }
      }
    } else if (warp == kMmaWarp) {
      // ============================ MMA issuer ============================
      // The whole warp runs the issue loop (warp-uniform state in uniform registers); one
      // elected lane issues each tcgen05 instruction. Per element g and query tile t:
      // PV_t(g) then QK_t(g+1), so each tile's next S is issued as soon as its own P is
      // consumed and the two query tiles ping-pong (anti-phase) on the tensor pipe.
      VFA_ROLE_SETUP();
      constexpr uint32_t kIdescQK = make_idesc_bf16(128, BC, false, false);
      constexpr uint32_t kIdescPV = make_idesc_bf16(128, D, false, true);
      // UMMA smem descriptors: hi word constant (SBO = 1024 B, version 1, SWIZZLE_128B),
      // lo word = (address >> 4) | LBO << 16. Addresses < 256 KiB so the start field never carries.
      constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t kLboK = 1u << 16;                                      // K-major: LBO unused
      constexpr uint32_t kLboV = static_cast<uint32_t>((BC * 128) >> 4) << 16;  // V: next 64-col chunk
      const uint32_t q_lo = smem_u32(sQ) >> 4;
      const uint32_t kv_lo = smem_u32(sKV) >> 4;
      for (int t = 0; t < NQ; ++t) mbar_wait(&ctl->q_full[t], 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      auto acquire = [&]() -> int {
        mbar_wait(&ctl->kv_full[stage], phase);
        tc_fence_after();
        int st = stage;
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
        return st;
      };
      auto issue_qk = [&](int t, int st) {
        const uint32_t a_lo = q_lo + t * (C::kQBytes >> 4) + kLboK;
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboK;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oq = ((kk >> 2) * (kBR * 128) + (kk & 3) * 32) >> 4;
          const uint32_t ok = ((kk >> 2) * (BC * 128) + (kk & 3) * 32) >> 4;
          if (elect_one())
            mma_ss(tbase + C::s_off(t), (static_cast<uint64_t>(kHi) << 32) | (a_lo + oq),
                   (static_cast<uint64_t>(kHi) << 32) | (b_lo + ok), kIdescQK, kk > 0 ? 1u : 0u);
          __syncwarp();
        }
      };
      // P of part pp occupies TMEM columns [pp*CP, pp*CP + CP/2) of S_t (packed bf16 pairs).
      // PV chunk c: the K-steps over P columns [c*CW, c*CW + CW) of every part.
      auto issue_pv_chunk = [&](int t, int st, int c, bool& first) {
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboV;
#pragma unroll
        for (int pp = 0; pp < SPLIT; ++pp) {
#pragma unroll
          for (int k2 = 0; k2 < CW / 16; ++k2) {
            const int kk = pp * (CP / 16) + c * (CW / 16) + k2;  // K-step (16 key rows of V)
            const uint32_t pcol = pp * CP + c * (CW / 2) + k2 * 8;
            if (elect_one())
              mma_ts(tbase + C::kOBase + t * D, tbase + C::s_off(t) + pcol,
                     (static_cast<uint64_t>(kHi) << 32) | (b_lo + kk * (2048 >> 4)), kIdescPV, first ? 0u : 1u);
            __syncwarp();
            first = false;
          }
        }
      };
      uint32_t sfree_ph = 0, p_ph = 0, o_init = 0;
      auto issue_s_tile = [&](int g, int t, int st) {
        // S_t's previous occupant g - 1: an m-init chunk must have been read (s_free);
        // a visited block's P was consumed by its PV, issued before this QK
        if (g >= 1 && g - 1 < nchunks) {
          mbar_wait(&ctl->s_free[t], (sfree_ph >> t) & 1u);
          sfree_ph ^= 1u << t;
          tc_fence_after();
        }
        issue_qk(t, st);
        commit_elect(&ctl->s_full[t]);
      };
      {
        const int st = acquire();
        for (int t = 0; t < NQ; ++t) issue_s_tile(0, t, st);
        commit_elect(&ctl->kv_empty[st]);
      }
      for (int g = 0; g < G; ++g) {
        const bool main_blk = g >= nchunks;
        const int pos = g - nchunks;
        const bool next_s = g + 1 < G;
        const int vs = main_blk ? acquire() : -1;
        int ks = -1;
        for (int t = 0; t < NQ; ++t) {
          if (main_blk) {
            bool first = ((o_init >> t) & 1u) == 0;  // first PV of this tile initialises O
            bool skip = false;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              mbar_wait(&ctl->p_full[t][c], (p_ph >> t) & 1u);
              tc_fence_after();
              if (c == 0) {
                if (lane == 0) VFA_TRACE_EVENT(a, pos, 4 + 2 * t);
                skip = (MODE == kVSA) && (ctl->skip[t] != 0);
              }
              if (!skip) issue_pv_chunk(t, vs, c, first);
            }
            p_ph ^= 1u << t;
            if (!skip) o_init |= 1u << t;
            if (t == NQ - 1) commit_elect(&ctl->kv_empty[vs]);
          }
          if (next_s) {
            if (t == 0) ks = acquire();
            issue_s_tile(g + 1, t, ks);
            if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 5 + 2 * t);
          }
        }
        if (ks >= 0) commit_elect(&ctl->kv_empty[ks]);
      }
      for (int t = 0; t < NQ; ++t) commit_elect(&ctl->o_final[t]);
    }
  } else {
    // ============================ softmax WGs ============================
    // Each row of a query tile is shared by SPLIT threads (TMEM lane r of SPLIT warpgroups),
    // each owning CP = BC/SPLIT S columns and OP = D/SPLIT O columns.
    //   SPLIT == 2: warpgroups 2t, 2t+1 serve query tile t only (two independent warp sets
    //               that run in anti-phase, each hiding under the other tile's MMA window);
    //   SPLIT == 4: all four warpgroups serve both tiles in turn (tile 0 then tile 1 of each
    //               key block): half the per-thread work per tile-block, one shared issue stream.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    constexpr int NT = (SPLIT == 4) ? NQ : 1;  // query tiles this thread serves
    const int part = (SPLIT == 4) ? (warp >> 2) : ((warp >> 2) & 1);
    const int tile0 = (SPLIT == 4) ? 0 : (warp >> 3);
    if (tile0 < NQ) {
      const int r = tid & 127;
      VFA_ROLE_SETUP();
      const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const int R = unit.qt * kBR + r;  // absolute query row
      const float cs = a.c_scale;
      float m2[NT], l[NT];  // running max (log2 units of scaled scores; identical in all parts)
      uint32_t xpar[NT];    // and this part's share of the normalizer, per served tile
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) {
        m2[ti] = -INFINITY;
        l[ti] = 0.f;
        xpar[ti] = 0;
      }
      uint32_t s_ph = 0;  // bit ti: s_full phase
      uint32_t over32 = 0, over16 = 0;
      auto tS = [&](int t) { return tbase + C::s_off(t) + part * CP + lane_off; };
      auto tO = [&](int t) { return tbase + C::kOBase + t * D + part * OP + lane_off; };
      // row-max exchange across the SPLIT parts of a row (named barrier 1 + t)
      auto exchange_max = [&](int ti, int t, float mine) -> float {
        ctl->xmax[t][xpar[ti]][part][r] = mine;
        named_bar_sync(1 + t, SPLIT * kBR);
        const float* x = ctl->xmax[t][xpar[ti]][0];
        float m = fmaxf(x[r], x[kBR + r]);
        if constexpr (SPLIT == 4) m = fmaxf(m, fmaxf(x[2 * kBR + r], x[3 * kBR + r]));
        xpar[ti] ^= 1;
        return m;
      };
      auto wait_s = [&](int ti, int t) {
        mbar_wait(&ctl->s_full[t], (s_ph >> ti) & 1u);
        s_ph ^= 1u << ti;
        tc_fence_after();
      };
      auto load_part = [&](int t, float* v) {
        if constexpr (CP >= 32) {
#pragma unroll
          for (int c = 0; c < CP / 32; ++c) tmem_ld32(tS(t) + c * 32, v + c * 32);
        } else {
          tmem_ld16(tS(t), v);
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
            wait_s(ti, t);
            float v[CP];
            load_part(t, v);
#pragma unroll
            for (int e = 0; e < CP; ++e)
              if (e < valid) mx[ti] = fmaxf(mx[ti], v[e]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl->s_free[t]);
          }
        }
#pragma unroll
        for (int ti = 0; ti < NT; ++ti) m2[ti] = exchange_max(ti, tile0 + ti, mx[ti]) * cs;
      }

      const float2 cs2 = make_float2(cs, cs);
      int n_skipped = 0, n_skipped_special = 0;  // VSA only (FA/VFA counts are closed-form)
      for (int pos = 0; pos < N; ++pos) {
        const int j = sched_block(sched, pos);
        const bool special = (MODE == kFA) || sched_is_special(sched, j);
        const bool mask = sched_needs_mask(unit.qt + 1, j, kBR, BC, a.causal != 0);
        const int lim = R - (j - 1) * BC - part * CP;  // this part's columns > lim are masked
#pragma unroll
        for (int ti = 0; ti < NT; ++ti) {
          const int t = tile0 + ti;
          wait_s(ti, t);
          if (r == 0 && part == 0) VFA_TRACE_EVENT(a, pos, 2 * t);
          float v[CP];
          load_part(t, v);
          if (mask) {  // entrywise causal mask (src/reference.py:93-96): exact zeros after exp2
#pragma unroll
            for (int e = 0; e < CP; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
          }
          bool skipped = false;
          if (MODE == kFA || MODE == kVSA || special) {
            // ---- exact-update / skip-test block: rowmax over the full row (four quarters,
            //      src/vfa.py:202-208, src/sparse.py:296-300), then rescale
            float mt = -INFINITY;
#pragma unroll
            for (int e = 0; e < CP; e += 2) mt = fmax3(mt, v[e], v[e + 1]);
            mt = exchange_max(ti, t, mt);
            const float mt2 = mt * cs;
            const float m2n = fmaxf(m2[ti], mt2);
            if (MODE == kVSA) {
              const bool below = (mt2 - m2n < a.log2_lambda) ||
                                 (mt2 == -INFINITY && m2n == -INFINITY && a.log2_lambda != -INFINITY);
              skipped = named_bar_and(1 + t, SPLIT * kBR, below);
            }
            if (skipped) {
              ++n_skipped;
              n_skipped_special += special ? 1 : 0;
            } else if (special) {
              const float f = (m2n == -INFINITY) ? 1.0f : ex2_approx(m2[ti] - m2n);
              m2[ti] = m2n;
              l[ti] = __fmul_rn(l[ti], f);  // no FMA contraction: identical l-recurrence in every mode
              // rescale this part of O in TMEM (src/core.py:91). O is quiescent here: PV(pos-1)
              // completed before S(pos) (in-order tensor pipe), PV(pos) waits for p_full.
              const bool work = (pos > 0) && ((MODE == kFA) || !__all_sync(0xffffffffu, f == 1.0f));
              if (work) {
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
              }
            }
          }
          // ---- frozen blocks (src/vfa.py:209-215) skip all of the above: no rowmax, no rescale
          if (r == 0 && part == 0) {
            if (MODE == kVSA) ctl->skip[t] = skipped ? 1u : 0u;
            if (a.skip_trace) {
              const size_t idx =
                  ((static_cast<size_t>(unit.b) * a.Hq + unit.h0 + t) * a.Tr + unit.qt) * a.Tc + pos;
              a.skip_trace[idx] = skipped ? 2 : 1;
            }
          }
          if (!skipped) {
            // P = exp2(S*c - m2) in CW-column chunks; each chunk is handed to the MMA warp as
            // soon as it is in TMEM (PV of chunk 0 overlaps the softmax of chunk 1)
            const float nm = m2[ti] == -INFINITY ? 0.f : -m2[ti];
            const float2 nmu2 = make_float2(nm, nm);
            float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              uint32_t u[CW / 2];
              if (a.monitor)
                p_chunk<CW, true, kPoly>(v + c * CW, cs2, nmu2, u, acc, over32, over16);
              else
                p_chunk<CW, false, kPoly>(v + c * CW, cs2, nmu2, u, acc, over32, over16);
              if constexpr (CW == 32) tmem_st16(tS(t) + c * 16, u);
              else tmem_st8(tS(t) + c * 8, u);
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&ctl->p_full[t][c]);
            }
            l[ti] = __fadd_rn(l[ti], __fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)));
          } else {
            __syncwarp();
            if (lane == 0)
              for (int c = 0; c < NCH; ++c) mbar_arrive(&ctl->p_full[t][c]);
          }
          if (r == 0 && part == 0) VFA_TRACE_EVENT(a, pos, 2 * t + 1);
        }
      }
      const int n_special = NT * sched.n_spec - n_skipped_special;
      const int n_frozen = NT * (N - sched.n_spec) - (n_skipped - n_skipped_special);

      // ---- epilogue: O / l (src/core.py:101-109), LSE = m + ln l; l = sum over the parts
      bool any_nonfinite = false;
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) {
        const int t = tile0 + ti;
        const int h = unit.h0 + t;
        ctl->xl[t][part][r] = l[ti];
        named_bar_sync(1 + t, SPLIT * kBR);
        float lsum = __fadd_rn(ctl->xl[t][0][r], ctl->xl[t][1][r]);
        if constexpr (SPLIT == 4) lsum = __fadd_rn(lsum, __fadd_rn(ctl->xl[t][2][r], ctl->xl[t][3][r]));
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
          for (int e = 0; e < 16; e += 2) {
            const float o0 = v[e] * inv, o1 = v[e + 1] * inv;
            finite = finite && isfinite(o0) && isfinite(o1);
            u[e >> 1] = pack_bf16x2(o0, o1);
          }
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
          dst[0] = make_uint4(u[0], u[1], u[2], u[3]);
          dst[1] = make_uint4(u[4], u[5], u[6], u[7]);
        }
        const size_t lrow = (static_cast<size_t>(unit.b) * a.Hq + h) * a.Lq + R;
        const unsigned srow = static_cast<unsigned>(lrow + a.row_base);  // whole-problem row for the status
        if (part == 0 && a.lse) a.lse[lrow] = (m2[ti] + __log2f(lsum)) * kLn2;
        if (a.status) {
          if (part == 0 && lsum == 0.f) {
            if (m2[ti] == -INFINITY) {
              atomicOr(&a.status[VFA_STATUS_FLAGS], 1u);
              atomicMin(&a.status[VFA_STATUS_MASKED_ROW], srow);
            } else {
              atomicOr(&a.status[VFA_STATUS_FLAGS], 2u);
              atomicMin(&a.status[VFA_STATUS_UNDERFLOW_ROW], srow);
            }
          }
          // a row is non-finite if any part is: combine through smem, count it once
          ctl->xfin[t][part][r] = finite ? 1 : 0;
          named_bar_sync(1 + t, SPLIT * kBR);
          bool row_ok = ctl->xfin[t][0][r] && ctl->xfin[t][1][r];
          if constexpr (SPLIT == 4) row_ok = row_ok && ctl->xfin[t][2][r] && ctl->xfin[t][3][r];
          if (part == 0 && !row_ok) any_nonfinite = true, atomicAdd(&a.status[VFA_STATUS_NONFINITE_ROWS], 1u);
        }
      }
      if (any_nonfinite) atomicOr(&a.status[VFA_STATUS_FLAGS], 4u);
      if (a.stats) {
        if (a.monitor) {
          atomicAdd(&a.stats[VFA_STAT_OVER_F32], static_cast<unsigned long long>(over32));
          atomicAdd(&a.stats[VFA_STAT_OVER_F16], static_cast<unsigned long long>(over16));
        }
        if (r == 0 && part == 0) {
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
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(ctl->tmem_base);
  }
}

// ------------------------------------------------------------------------------------
// Key-block representations (src/vfa.py:47-88): one warp per key block, lane owns
// D/32 consecutive columns; sabsmax keeps the first row on ties (strict >).
template <int D>
__global__ void __launch_bounds__(128) krepr_kernel(const __nv_bfloat16* __restrict__ k, long long sb, long long sh,
                                                    long long sr, int Hkv, int BC, int nblk, int kind,
                                                    __nv_bfloat16* __restrict__ out) {
  constexpr int CPL = D / 32;  // columns per lane (2 or 4)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jb = blockIdx.x * 4 + warp;
  const int kvh = blockIdx.y, b = blockIdx.z;
  if (jb >= nblk) return;
  const __nv_bfloat16* base = k + b * sb + kvh * sh + static_cast<long long>(jb) * BC * sr + lane * CPL;
  float best[CPL], val[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    best[c] = kind == VFA_KREPR_K_MEAN ? 0.f : -INFINITY;
    val[c] = 0.f;
  }
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
    } else {
      const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(base + row * sr);
      x[0] = __low2float(p0);
      x[1] = __high2float(p0);
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

}  // namespace vfa

// ====================================================================================
// Host side
// ====================================================================================
namespace {

thread_local std::string g_last_error;
long long* g_debug_trace = nullptr;  // debug only: set by vfa_debug_trace()

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

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

template <int D, int BC, int NQ, int MODE, int SPLIT>
int launch_fwd(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
               const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t stream) {
  using C = vfa::Cfg<D, BC, NQ, SPLIT>;
  auto kern = vfa::vfa_fwd_kernel<D, BC, NQ, MODE, SPLIT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("cudaFuncGetAttributes: ") + cudaGetErrorString(e));
    if (vfa::kRegBudget > fa.numRegs * vfa::kThreads)
      return fail(VFA_ERR_CUDA, "setmaxnreg budget " + std::to_string(vfa::kRegBudget) + " exceeds the launch allocation " +
                                    std::to_string(fa.numRegs * vfa::kThreads) + " (would deadlock)");
    attr_set = true;
  }
  const long long units = static_cast<long long>(args.B) * args.Hkv * args.units_per_kvh;
  if (units <= 0) return VFA_OK;
  kern<<<static_cast<unsigned>(units), vfa::kThreads, C::kSmem, stream>>>(mq, mk, mv, mr, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

// Softmax column split per variant (params.softmax_split = 0), measured best on B200
// (profiles/ab_r01_split.txt): VFA's frozen blocks need no cross-thread exchange, so all
// warps serving both tiles wins; FA / VSA exchange a row max on every block, which per-tile
// warp sets overlap with the other tile's work. One query tile per CTA: always 4.
constexpr int default_split(int variant) {
  return variant == VFA_VARIANT_FA ? VFA_SPLIT_FA : (variant == VFA_VARIANT_VFA ? VFA_SPLIT_VFA : VFA_SPLIT_VSA);
}

template <int D, int BC, int NQ, int MODE>
int dispatch_split(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                   const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st) {
  const int split = p->softmax_split ? p->softmax_split : default_split(p->variant);
  if (NQ == 2 && split == 2) return launch_fwd<D, BC, NQ, MODE, 2>(p, mq, mk, mv, mr, args, st);
  return launch_fwd<D, BC, NQ, MODE, 4>(p, mq, mk, mv, mr, args, st);
}

template <int D, int BC, int NQ>
int dispatch_mode(const VfaParams* p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                  const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st) {
  switch (p->variant) {
    case VFA_VARIANT_FA:
      return dispatch_split<D, BC, NQ, vfa::kFA>(p, mq, mk, mv, mr, args, st);
    case VFA_VARIANT_VFA:
      return dispatch_split<D, BC, NQ, vfa::kVFA>(p, mq, mk, mv, mr, args, st);
    default:
      return dispatch_split<D, BC, NQ, vfa::kVSA>(p, mq, mk, mv, mr, args, st);
  }
}

template <int D, int BC>
int dispatch_nq(const VfaParams* p, int nq, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                const CUtensorMap& mr, const vfa::FwdArgs& args, cudaStream_t st) {
  return nq == 2 ? dispatch_mode<D, BC, 2>(p, mq, mk, mv, mr, args, st)
                 : dispatch_mode<D, BC, 1>(p, mq, mk, mv, mr, args, st);
}

int launch_krepr(const VfaParams* p, const void* k, void* out, cudaStream_t st) {
  const int nblk = static_cast<int>(n_reprs(p));
  dim3 grid((nblk + 3) / 4, static_cast<unsigned>(p->heads_kv), static_cast<unsigned>(p->batch));
  if (p->head_dim == 128)
    vfa::krepr_kernel<128><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(k), p->k_stride[0],
                                                p->k_stride[1], p->k_stride[2], static_cast<int>(p->heads_kv),
                                                p->k_block, nblk, p->kind, static_cast<__nv_bfloat16*>(out));
  else
    vfa::krepr_kernel<64><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(k), p->k_stride[0],
                                               p->k_stride[1], p->k_stride[2], static_cast<int>(p->heads_kv),
                                               p->k_block, nblk, p->kind, static_cast<__nv_bfloat16*>(out));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("krepr launch: ") + cudaGetErrorString(e));
  return VFA_OK;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

void reset_counters(long long* stats, unsigned int* status, cudaStream_t st) {
  if (stats) cudaMemsetAsync(stats, 0, sizeof(long long) * VFA_STAT_COUNT, st);
  if (status) {
    cudaMemsetAsync(status, 0, sizeof(unsigned) * VFA_STATUS_COUNT, st);
    cudaMemsetAsync(status + VFA_STATUS_UNDERFLOW_ROW, 0xff, sizeof(unsigned) * 2, st);
  }
}

int forward_impl(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                 unsigned char* skip_trace, cudaStream_t st, bool zero_counters, long long row_base);

}  // namespace

extern "C" {

int vfa_check_params(const VfaParams* p) {
  if (!p) return fail(VFA_ERR_CONFIG, "params is NULL");
  if (p->variant < VFA_VARIANT_FA || p->variant > VFA_VARIANT_VSA)
    return fail(VFA_ERR_CONFIG, "variant must be 0 (fa), 1 (vfa) or 2 (vsa)");
  if (p->kind < VFA_KREPR_SABSMAX || p->kind > VFA_KREPR_K_ABSMAX_UNSIGNED)
    return fail(VFA_ERR_CONFIG, "unknown key representation");
  if (p->qkind != 0) return fail(VFA_ERR_CONFIG, "only the row_wise query representation runs on the GPU path");
  if (p->q_block != 128) return fail(VFA_ERR_CONFIG, "q_block must be 128 (tcgen05 M = 128)");
  if (p->k_block != 64 && p->k_block != 128) return fail(VFA_ERR_CONFIG, "k_block must be 64 or 128");
  if (p->head_dim != 64 && p->head_dim != 128) return fail(VFA_ERR_CONFIG, "head_dim must be 64 or 128");
  if (p->n_sink < 0 || p->n_local < 0) return fail(VFA_ERR_CONFIG, "n_sink and n_local must be >= 0");
  if (p->softmax_split != 0 && p->softmax_split != 2 && p->softmax_split != 4)
    return fail(VFA_ERR_CONFIG, "softmax_split must be 0 (auto), 2 or 4");
  if (p->variant == VFA_VARIANT_VSA && p->lam > 1.0) return fail(VFA_ERR_CONFIG, "lambda must be in (0, 1]");
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
  return static_cast<size_t>(p->batch * p->heads_kv * n_reprs(p) * p->head_dim * 2) + 256;
}

int vfa_krepr(const VfaParams* p, const void* k, void* out, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!k || !out) return fail(VFA_ERR_DATA, "NULL pointer");
  return launch_krepr(p, k, out, static_cast<cudaStream_t>(stream));
}

int vfa_fwd(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
            void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
            unsigned char* skip_trace, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q || !k || !v || !o) return fail(VFA_ERR_DATA, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(VFA_ERR_DATA, "tensors must be 16-byte aligned");
  return forward_impl(p, q, k, v, o, lse, workspace, workspace_bytes, stats, status, skip_trace,
                      static_cast<cudaStream_t>(stream), true, 0);
}

}  // extern "C"

namespace {
// The forward on device buffers. zero_counters: reset stats/status first (false when a
// caller accumulates several launches into one status word, e.g. vfa_fwd_host's chunks).
int forward_impl(const VfaParams* p, const void* q, const void* k, const void* v, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, long long* stats, unsigned int* status,
                 unsigned char* skip_trace, cudaStream_t st, bool zero_counters, long long row_base) {
  int rc = VFA_OK;
  const bool minit = p->variant != VFA_VARIANT_FA && p->use_m_init;
  const int64_t nrep = n_reprs(p);
  if (minit) {
    if (!workspace || workspace_bytes < vfa_workspace_bytes(p) || !aligned16(workspace))
      return fail(VFA_ERR_DATA, "workspace too small or misaligned");
  }
  const int D = static_cast<int>(p->head_dim), BC = p->k_block;
  const int group = static_cast<int>(p->heads_q / p->heads_kv);
  const int nq = (group % 2 == 0) ? 2 : 1;

  CUtensorMap mq, mk, mv, mr;
  if (!make_map(&mq, q, p->batch, p->heads_q, p->seq_q, D, p->q_stride[0], p->q_stride[1], p->q_stride[2], 128) ||
      !make_map(&mk, k, p->batch, p->heads_kv, p->seq_k, D, p->k_stride[0], p->k_stride[1], p->k_stride[2], BC) ||
      !make_map(&mv, v, p->batch, p->heads_kv, p->seq_k, D, p->v_stride[0], p->v_stride[1], p->v_stride[2], BC))
    return fail(VFA_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (minit) {
    if (!make_map(&mr, workspace, p->batch, p->heads_kv, nrep, D, p->heads_kv * nrep * D, nrep * D, D, BC))
      return fail(VFA_ERR_CUDA, "cuTensorMapEncodeTiled failed (krepr)");
    if (!p->krepr_precomputed) {
      rc = launch_krepr(p, k, workspace, st);
      if (rc) return rc;
    }
  } else {
    mr = mk;
  }
  if (zero_counters) reset_counters(stats, status, st);
  if (skip_trace)
    cudaMemsetAsync(skip_trace, 0,
                    static_cast<size_t>(p->batch * p->heads_q * (p->seq_q / 128) * n_key_blocks(p)), st);

  vfa::FwdArgs a;
  a.B = static_cast<int>(p->batch);
  a.Hq = static_cast<int>(p->heads_q);
  a.Hkv = static_cast<int>(p->heads_kv);
  a.Lq = static_cast<int>(p->seq_q);
  a.Lk = static_cast<int>(p->seq_k);
  a.group = group;
  a.Tr = static_cast<int>(p->seq_q / 128);
  a.Tc = static_cast<int>(n_key_blocks(p));
  a.heads_per_unit = nq;
  a.units_per_kvh = a.Tr * (group / nq);
  const double scale = p->scale > 0 ? p->scale : 1.0 / std::sqrt(static_cast<double>(D));
  a.c_scale = static_cast<float>(scale * 1.4426950408889634);
  a.log2_lambda = (p->variant == VFA_VARIANT_VSA && p->lam > 0) ? static_cast<float>(std::log2(p->lam)) : -INFINITY;
  a.causal = p->causal ? 1 : 0;
  a.reorder = p->reorder ? 1 : 0;
  a.use_m_init = minit ? 1 : 0;
  a.nrep_cap = static_cast<int>(nrep);
  a.n_sink = p->n_sink;
  a.n_local = p->n_local;
  a.monitor = p->monitor ? 1 : 0;
  a.o = static_cast<__nv_bfloat16*>(o);
  a.o_sb = p->o_stride[0];
  a.o_sh = p->o_stride[1];
  a.o_sr = p->o_stride[2];
  a.lse = lse;
  a.stats = reinterpret_cast<unsigned long long*>(stats);
  a.status = status;
  a.skip_trace = skip_trace;
  a.row_base = row_base;
  a.trace = g_debug_trace;

  if (D == 128 && BC == 128) return dispatch_nq<128, 128>(p, nq, mq, mk, mv, mr, a, st);
  if (D == 128 && BC == 64) return dispatch_nq<128, 64>(p, nq, mq, mk, mv, mr, a, st);
  if (D == 64 && BC == 128) return dispatch_nq<64, 128>(p, nq, mq, mk, mv, mr, a, st);
  return dispatch_nq<64, 64>(p, nq, mq, mk, mv, mr, a, st);
}

// ---------------------------------------------------------------- host-resident pipeline
// vfa_fwd_host: the problem is cut into chunks of (one batch, `ck` KV heads with their GQA
// query heads). Chunk c is copied host->device on the H2D stream into scratch slot c % S,
// computed on compute stream c % 2 (so one chunk's causal tail overlaps the next chunk's
// head), and its O / LSE copied back on the D2H stream, so PCIe transfers in both
// directions overlap the attention kernels.
constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct ChunkGeom {
  int64_t ck, nq, chunks, slots;
  size_t q_bytes, kv_bytes, lse_bytes, ws_bytes, slot_bytes;
  VfaParams cp;  // the per-chunk problem (dense device layout)
};

ChunkGeom chunk_geom(const VfaParams* p, int chunk_kv_heads) {
  ChunkGeom g{};
  g.ck = chunk_kv_heads;
  const int64_t group = p->heads_q / p->heads_kv;
  g.nq = g.ck * group;
  g.chunks = p->batch * (p->heads_kv / g.ck);
  g.slots = g.chunks < 3 ? g.chunks : 3;
  g.cp = *p;
  g.cp.batch = 1;
  g.cp.heads_q = g.nq;
  g.cp.heads_kv = g.ck;
  const int64_t D = p->head_dim;
  const int64_t qs[3] = {g.nq * p->seq_q * D, p->seq_q * D, D};
  const int64_t ks[3] = {g.ck * p->seq_k * D, p->seq_k * D, D};
  for (int i = 0; i < 3; ++i) {
    g.cp.q_stride[i] = g.cp.o_stride[i] = qs[i];
    g.cp.k_stride[i] = g.cp.v_stride[i] = ks[i];
  }
  g.q_bytes = static_cast<size_t>(g.nq * p->seq_q * D * 2);
  g.kv_bytes = static_cast<size_t>(g.ck * p->seq_k * D * 2);
  g.lse_bytes = static_cast<size_t>(g.nq * p->seq_q * 4);
  g.ws_bytes = vfa_workspace_bytes(&g.cp);
  g.slot_bytes = 2 * align_up(g.q_bytes) + 2 * align_up(g.kv_bytes) + align_up(g.lse_bytes) + align_up(g.ws_bytes);
  return g;
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

size_t vfa_host_scratch_bytes(const VfaParams* p, int chunk_kv_heads) {
  if (!p || vfa_check_params(p) != VFA_OK || chunk_kv_heads < 1 || p->heads_kv % chunk_kv_heads) return 0;
  const ChunkGeom g = chunk_geom(p, chunk_kv_heads);
  return static_cast<size_t>(g.slots) * g.slot_bytes + kAlign;
}

int vfa_fwd_host(const VfaParams* p, const void* q_host, const void* k_host, const void* v_host, void* o_host,
                 float* lse_host, void* scratch, size_t scratch_bytes, long long* stats, unsigned int* status,
                 int chunk_kv_heads, void* stream) {
  int rc = vfa_check_params(p);
  if (rc) return rc;
  if (!q_host || !k_host || !v_host || !o_host) return fail(VFA_ERR_DATA, "NULL host pointer");
  if (chunk_kv_heads < 1 || p->heads_kv % chunk_kv_heads)
    return fail(VFA_ERR_CONFIG, "chunk_kv_heads must divide heads_kv");
  if (p->krepr_precomputed) return fail(VFA_ERR_CONFIG, "vfa_fwd_host computes the representations itself");
  const size_t need = vfa_host_scratch_bytes(p, chunk_kv_heads);
  if (!scratch || scratch_bytes < need) return fail(VFA_ERR_DATA, "scratch too small (vfa_host_scratch_bytes)");
  const ChunkGeom g = chunk_geom(p, chunk_kv_heads);
  HostStreams* hs = nullptr;
  rc = host_streams(&hs);
  if (rc) return rc;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(scratch) + kAlign - 1) & ~uintptr_t(kAlign - 1));

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
  // counters accumulate over chunks; scratch reuse is ordered after the caller's prior work
  reset_counters(stats, status, caller);
  cudaEvent_t entry = new_event();
  if (!entry) return cleanup(), fail(VFA_ERR_CUDA, "cudaEventCreate failed");
  cudaEventRecord(entry, caller);
  cudaStreamWaitEvent(hs->h2d, entry, 0);
  cudaStreamWaitEvent(hs->comp[0], entry, 0);
  cudaStreamWaitEvent(hs->comp[1], entry, 0);

  const int64_t D = p->head_dim, group = p->heads_q / p->heads_kv;
  const int64_t per_b = p->heads_kv / g.ck;
  std::vector<cudaEvent_t> slot_free(static_cast<size_t>(g.slots), nullptr);
  for (int64_t c = 0; c < g.chunks; ++c) {
    const int64_t b = c / per_b, kv0 = (c % per_b) * g.ck, h0 = kv0 * group;
    const int64_t s = c % g.slots;
    uint8_t* sl = base + s * g.slot_bytes;
    uint8_t* dq = sl;
    uint8_t* dk = dq + align_up(g.q_bytes);
    uint8_t* dv = dk + align_up(g.kv_bytes);
    uint8_t* dout = dv + align_up(g.kv_bytes);
    float* dlse = reinterpret_cast<float*>(dout + align_up(g.q_bytes));
    uint8_t* dws = reinterpret_cast<uint8_t*>(dlse) + align_up(g.lse_bytes);
    const size_t qoff = static_cast<size_t>((b * p->heads_q + h0) * p->seq_q * D) * 2;
    const size_t koff = static_cast<size_t>((b * p->heads_kv + kv0) * p->seq_k * D) * 2;
    const size_t loff = static_cast<size_t>((b * p->heads_q + h0) * p->seq_q);
    // H2D (after the slot's previous chunk has been copied out)
    if (slot_free[s]) cudaStreamWaitEvent(hs->h2d, slot_free[s], 0);
    cudaMemcpyAsync(dk, static_cast<const uint8_t*>(k_host) + koff, g.kv_bytes, cudaMemcpyHostToDevice, hs->h2d);
    cudaMemcpyAsync(dv, static_cast<const uint8_t*>(v_host) + koff, g.kv_bytes, cudaMemcpyHostToDevice, hs->h2d);
    cudaMemcpyAsync(dq, static_cast<const uint8_t*>(q_host) + qoff, g.q_bytes, cudaMemcpyHostToDevice, hs->h2d);
    cudaEvent_t in = new_event(), done = new_event(), out = new_event();
    if (!in || !done || !out) return cleanup(), fail(VFA_ERR_CUDA, "cudaEventCreate failed");
    cudaEventRecord(in, hs->h2d);
    // compute
    cudaStream_t cs = hs->comp[c & 1];
    cudaStreamWaitEvent(cs, in, 0);
    rc = forward_impl(&g.cp, dq, dk, dv, dout, dlse, dws, g.ws_bytes, stats, status, nullptr, cs, false,
                      static_cast<long long>(loff));
    if (rc) return cleanup(), rc;
    cudaEventRecord(done, cs);
    // D2H
    cudaStreamWaitEvent(hs->d2h, done, 0);
    cudaMemcpyAsync(static_cast<uint8_t*>(o_host) + qoff, dout, g.q_bytes, cudaMemcpyDeviceToHost, hs->d2h);
    if (lse_host)
      cudaMemcpyAsync(lse_host + loff, dlse, g.lse_bytes, cudaMemcpyDeviceToHost, hs->d2h);
    cudaEventRecord(out, hs->d2h);
    slot_free[s] = out;
  }
  cudaEvent_t exit_ev = new_event();
  if (!exit_ev) return cleanup(), fail(VFA_ERR_CUDA, "cudaEventCreate failed");
  cudaEventRecord(exit_ev, hs->d2h);
  cudaStreamWaitEvent(caller, exit_ev, 0);
  cleanup();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VFA_ERR_CUDA, std::string("vfa_fwd_host: ") + cudaGetErrorString(e));
  return VFA_OK;
}

int vfa_schedule(int i, int q_block, int k_block, int t_c, int causal, int n_sink, int n_local, int reorder,
                 int variant, int* order_out, unsigned char* special_out, int cap) {
  if (i < 1 || q_block < 1 || k_block < 1 || t_c < 1) return -VFA_ERR_CONFIG;
  vfa::TileSchedule s = vfa::make_schedule(i, q_block, k_block, t_c, causal != 0, n_sink, n_local,
                                           variant != VFA_VARIANT_FA && reorder != 0, variant == VFA_VARIANT_FA);
  for (int pos = 0; pos < s.vmax && pos < cap; ++pos) {
    int j = vfa::sched_block(s, pos);
    if (order_out) order_out[pos] = j;
    if (special_out) special_out[pos] = vfa::sched_is_special(s, j) ? 1 : 0;
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

const char* vfa_last_error(void) { return g_last_error.c_str(); }

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
