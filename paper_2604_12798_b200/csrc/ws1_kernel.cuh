// B200 (sm_100a) attention forward with a decoupled softmax: one 128-row query tile per CTA,
// three S buffers in TMEM, K/V shared by a 2-CTA cluster through TMA multicast.
//
// Shape: head_dim 128, 128-key blocks, 128-row query blocks, GQA group even. A cluster is one
// work unit of vfa_fwd_kernel (b, KV head, two query heads of its group, one query tile): CTA r
// of the pair computes query head h0 + r. Both CTAs visit the same key blocks in the same
// order (same rows, same schedule), so each loads half of every K / V tile and multicasts it to
// both: per-SM L2 -> smem traffic equals the two-tiles-per-CTA kernels', while each CTA has the
// TMEM for three S buffers.
//
// Per CTA (640 threads):
//   warps 0-7   softmax group 0: sequence elements g = 0, 2, 4, ...   (two threads per row,
//   warps 8-15  softmax group 1: sequence elements g = 1, 3, 5, ...    64 S columns each)
//   warp 16     QK^T issuer (converged, elect.sync), TMEM allocator
//   warp 17     TMA producer
//   warp 18     PV issuer
//   warp 19     idle (QK^T issuer of odd elements with VFA_WS1_QK2=1; warp 16 then even ones)
// TMEM: S buffers at 0 / 128 / 256 (P packed bf16 in columns 0-31 / 64-95 of its S buffer, see p_col),
// O at 384. The MMA issues QK for element g + 3 as soon as PV(g) is issued, so S is up to
// three blocks ahead and the two groups' exponentials run back to back: the softmax is never
// waiting on a P -> PV -> QK -> S round trip (the limit of the ping-pong kernels).
//
// Running max across the two groups (src/vfa.py:199-215, src/core.py:76-98): exact-update
// positions are processed in schedule order; the group that finishes one publishes the row max
// as a new "version" (a ring of kVer slots with one mbarrier each) and a group needing the max
// after the e-th exact position waits for version e. VFA's frozen blocks (all but sink / local)
// need the seed / frozen max only, so after the specials the groups never wait on each other.
// Each group keeps its part of the normalizer relative to the max it last saw; the parts are
// rescaled to the final max at the end. O is rescaled (src/core.py:91) by the group that raised
// the max, after PV of the previous position completed (pv_done) and before its own P hand-off.
#pragma once
#include "vfa_kernel.cuh"

namespace vfa {

#ifndef VFA_WS1_PAIR
#define VFA_WS1_PAIR 0
#endif
#ifndef VFA_WS1_STAGES
#define VFA_WS1_STAGES (VFA_WS1_PAIR ? 10 : 5)
#endif
#ifndef VFA_WS1_EMU
#define VFA_WS1_EMU 1  // element pairs (of 8) per 32-column chunk on the FMA-pipe exp2
#endif
#ifndef VFA_WS1_PREFETCH
#define VFA_WS1_PREFETCH 0  // 1: load the next element's first S columns before finishing this one (measured 7 % slower: spills)
#endif
#ifndef VFA_WS1_QK2
#define VFA_WS1_QK2 0  // 1: two QK issuer warps (16, 19) on alternate elements (measured 1-3 % slower)
#endif
#ifndef VFA_WS1_PV_SKIPFIRST
#define VFA_WS1_PV_SKIPFIRST 0  // (not with VFA_WS1_PAIR)  // 1: PV issuer frees a skipped element's buffer before its V lands (no gain, -3 % dense VSA)
#endif
#ifndef VFA_WS1_PIPE
#define VFA_WS1_PIPE 0  // 1: next position's schedule facts computed during this one's S load (spills; VFA 1244 vs 1301)
#endif
#ifndef VFA_WS1_VPREF
#define VFA_WS1_VPREF 0  // 1: L2 prefetch of V(g) when K(g) is loaded (dense same, skip mode -12 %)
#endif
#ifndef VFA_WS1_MC
#define VFA_WS1_MC 1  // 1: each CTA loads half of every K / V tile and multicasts it to the pair; 0: full tiles per CTA
#endif
#ifndef VFA_WS1_LA
#define VFA_WS1_LA 3  // K/V load sequence: S-op(0 .. LA-1), then per element V(g), S-op(g + LA)
#endif
#ifndef VFA_WS1_C0
#define VFA_WS1_C0 32  // columns (per thread) in the first P hand-off of an element: 32 or 16
#endif
#ifndef VFA_WS1_STAB
#define VFA_WS1_STAB 0  // 1: schedule facts per visit position tabulated in smem once per CTA (VFA -2 %, VSA / skip mode +1-2 %)
#endif
#ifndef VFA_WS1_NG
#define VFA_WS1_NG 2  // softmax groups (elements g with g % NG == group); 3: 24 softmax warps
#endif
#ifndef VFA_WS1_REGS_SOFTMAX
#define VFA_WS1_REGS_SOFTMAX (VFA_WS1_NG == 3 ? 80 : 104)
#endif
#ifndef VFA_WS1_REGS_OTHER
#define VFA_WS1_REGS_OTHER (VFA_WS1_NG == 3 ? 24 : 64)
#endif

struct Ws1Cfg {
  static constexpr int D = 128, BC = 128;
  static constexpr int kNG = VFA_WS1_NG;  // softmax groups of 8 warps
  static_assert(kNG == 2 || kNG == 3, "softmax groups");
  static constexpr int kThreads = 32 * (8 * kNG + 4);
  static constexpr int kMmaWarp = 8 * kNG;       // QK issuer, TMEM allocator
  static constexpr int kLoadWarp = 8 * kNG + 1;
  static constexpr int kPvWarp = 8 * kNG + 2;    // PV issuer
  static constexpr int kQk2Warp = 8 * kNG + 3;   // second QK issuer (VFA_WS1_QK2)
  static constexpr int kSB = 3;     // S buffers
  static constexpr int kVer = 6;    // running-max version ring
  static constexpr int kQBytes = kBR * D * 2;  // 32 KB
  static constexpr int kPair = VFA_WS1_PAIR ? 2 : 1;
  // per stage and CTA: a whole K / V tile (32 KB, each CTA loads half and multicasts it), or with
  // pair MMAs this CTA's half (K-like tiles: BC / 2 key rows; V tiles: D / 2 columns)
  static constexpr int kKVBytes = BC * D * 2 / kPair;
  static constexpr int kStages = VFA_WS1_STAGES;
  static constexpr int kSchedTab = VFA_WS1_STAB ? 2048 : 1;  // visit positions tabulated per CTA
  static constexpr int kCtlBytes = (kNG == 3 ? 24 : (VFA_WS1_STAB ? 20 : 16)) * 1024;
  static constexpr int kSmem = kCtlBytes + kQBytes + kStages * kKVBytes;
  static constexpr int kRegBudget = (2 * kNG * VFA_WS1_REGS_SOFTMAX + VFA_WS1_REGS_OTHER) * 128;
  static_assert(kSmem <= kMaxSmem, "shared memory");
  // setmaxnreg redistributes the launch allocation (65536 / kThreads, rounded down to 8)
  static_assert(kRegBudget <= kThreads * ((65536 / kThreads) & ~7), "register budget");
  static __device__ __forceinline__ uint32_t s_off(int b) { return static_cast<uint32_t>(b * 128); }
  static constexpr uint32_t kOOff = 384;
};

struct __align__(16) Ws1Ctl {
  uint64_t q_full;
  uint64_t kv_full[Ws1Cfg::kStages];
  uint64_t kv_empty[Ws1Cfg::kStages];  // both CTAs' MMAs consumed the stage (multicast commits)
  uint64_t s_full[Ws1Cfg::kSB];
  uint64_t p_full[Ws1Cfg::kSB][2];     // P chunk c of the element in buffer b (or S consumed)
  uint64_t pv_done[2];                 // [pos & 1]: PV of visit position pos completed
  uint64_t o_final;
  uint64_t pv_issued[Ws1Cfg::kSB];     // PV issuer -> QK issuer: PV of the element in buffer b enqueued
  uint64_t mver[Ws1Cfg::kVer];         // running-max version v published (slot v % kVer)
  uint32_t tmem_base;
  uint32_t skip[Ws1Cfg::kSB];
  uint32_t skip2[Ws1Cfg::kSB][2];      // pair: both CTAs' skip decisions (on the leader)
  float zero;
  float m_pub[Ws1Cfg::kVer][kBR];      // version's running max (log2 units), per row
  int stab_pub[Ws1Cfg::kVer][kBR];     // version's StateTrace stabilisation block, per row
  float xmax[Ws1Cfg::kNG][2][2][kBR];  // [group][exact parity][half][row]: row-max exchange
  float xinit[Ws1Cfg::kNG][2][kBR];    // [group][half][row]: m-init partial maxima
  float xl[Ws1Cfg::kNG][2][kBR];       // [group][half][row]: final partial row sums
  uint8_t xfin[4][kBR];                // [column quarter][row]: output finite flags
  uint16_t sinfo[Ws1Cfg::kSchedTab];   // per visit position: key block | exact << 14 | masked << 15
};
static_assert(sizeof(Ws1Ctl) <= Ws1Cfg::kCtlBytes, "control block");

// exact-update positions before visit position pos (schedule order, src/vfa.py:146-153)
template <int MODE>
__device__ __forceinline__ int exact_before(const TileSchedule& s, int pos) {
  if (all_exact(MODE)) return pos;
  if (s.reorder) return pos < s.n_spec ? pos : s.n_spec;
  int c = pos < s.a ? pos : s.a;
  if (s.b0 <= s.b1 && pos >= s.b0) c += (pos < s.b1 ? pos : s.b1) - s.b0 + 1;
  return c;
}

#ifndef VFA_WS1_FASTWAIT
#define VFA_WS1_FASTWAIT 0  // bit 0: issuer / producer waits, bit 1: softmax waits probe the phase first
#endif
// mbarrier wait that first probes the phase (test_wait never suspends): a try_wait costs ~90
// cycles even on a completed phase, which the MMA issuers pay on every element
template <int BIT>
__device__ __forceinline__ void ws1_wait(uint64_t* bar, uint32_t parity) {
  if ((VFA_WS1_FASTWAIT >> BIT) & 1) {
    if (mbar_test_wait(bar, parity)) return;
  }
  mbar_wait(bar, parity);
}
#define iwait ws1_wait<0>
#define swait ws1_wait<1>

template <int MODE>
__global__ void __launch_bounds__(Ws1Cfg::kThreads, 1)
    vfa_ws1_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmR,
                   const FwdArgs a) {
  using C = Ws1Cfg;
  constexpr int D = C::D, BC = C::BC, NS = C::kStages, SB = C::kSB, NV = C::kVer;
  constexpr bool PR = C::kPair == 2;  // pair MMAs: the leader (rank 0) issues every MMA for both CTAs
  constexpr int NG = C::kNG;
  constexpr int kAllBar = 1 + NG;  // named barrier of all softmax warps (1 .. NG: one per group)
  // three groups: the registers hold 32 S columns at a time (chunks loaded as they are consumed)
  constexpr bool kLowReg = NG == 3;
  // K tiles ahead of V(g) in the load sequence (SB: as many as S buffers; fewer lets V(g) take
  // an older ring stage, K(g + SB) a younger one)
  constexpr int LA = VFA_WS1_LA;
  static_assert(LA >= 1 && LA <= SB, "load look-ahead");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  Ws1Ctl* ctl = reinterpret_cast<Ws1Ctl*>(smem_raw);
  uint8_t* sQ = smem_raw + C::kCtlBytes;
  uint8_t* sKV = sQ + C::kQBytes;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t crank = cluster_ctarank();

  if (tid == 0) {
    VFA_TRACE_UNIT(a, 0);
    ctl->zero = 0.f;
    mbar_init(&ctl->q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&ctl->kv_full[s], 1);
      mbar_init(&ctl->kv_empty[s], (VFA_WS1_MC && !PR) ? 2 : 1);
    }
    for (int b = 0; b < SB; ++b) {
      mbar_init(&ctl->s_full[b], 1);
      mbar_init(&ctl->p_full[b][0], 8 * C::kPair);  // (a pair's leader counts both CTAs' warps)
      mbar_init(&ctl->p_full[b][1], 8 * C::kPair);
    }
    mbar_init(&ctl->pv_done[0], 1);
    mbar_init(&ctl->pv_done[1], 1);
    mbar_init(&ctl->o_final, 1);
    for (int b = 0; b < SB; ++b) mbar_init(&ctl->pv_issued[b], 1);
    for (int v = 0; v < NV; ++v) mbar_init(&ctl->mver[v], 8);
    fence_barrier_init();
  }
  if (warp == C::kLoadWarp && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmR);
  }
  if (warp == C::kMmaWarp) {
    if constexpr (PR)
      tmem_alloc_pair<512>(&ctl->tmem_base);
    else
      tmem_alloc<512>(&ctl->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's barriers are initialised before any multicast lands
  tc_fence_after();

#define VFA_WS1_SETUP()                                                  \
  const uint32_t tbase = ctl->tmem_base;                                 \
  const Unit unit = decode_unit(a, blockIdx.x >> 1);                     \
  const int head = unit.h0 + static_cast<int>(crank);                   \
  const TileSchedule sched = unit_schedule<MODE>(a, unit.qt, BC);        \
  const int N = sched.vmax;                                              \
  int nrep = 0;                                                          \
  const int nchunks = minit_chunks<MODE>(a, sched, BC, &nrep);           \
  const int G = nchunks + N;                                             \
  (void)tbase; (void)nrep; (void)G; (void)head

  if (warp >= C::kMmaWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(VFA_WS1_REGS_OTHER));
    if (warp == C::kLoadWarp) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        VFA_WS1_SETUP();
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        if constexpr (PR) {
          // both CTAs' Q tiles count on the leader's barrier (the pair MMAs read both)
          if (crank == 0) mbar_arrive_expect_tx(&ctl->q_full, 2 * C::kQBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d_pair(sQ + c * kBR * 128, &tmQ, &ctl->q_full, c * 64, unit.qt * kBR, head, unit.b, pol_q);
        } else {
          mbar_arrive_expect_tx(&ctl->q_full, C::kQBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d(sQ + c * kBR * 128, &tmQ, &ctl->q_full, c * 64, unit.qt * kBR, head, unit.b, pol_q);
        }
        int stage = 0;
        uint32_t phase = 0;
        // each CTA loads 64-column chunk `crank` of the tile (K: dims, V: head-dim columns) and
        // multicasts it to both CTAs; each CTA's kv_full counts both halves
#ifndef VFA_WS1_DBG_SKIP
#define VFA_WS1_DBG_SKIP 0  // timing experiments only (wrong results): 1 = no V transfers
#endif
        int nload = 0;
        auto load_tile = [&](const CUtensorMap* map, int row) {
          iwait(&ctl->kv_empty[stage], phase ^ 1);
          if (VFA_WS1_DBG_SKIP && nload++ >= 8 && map == &tmV) {
            mbar_arrive(&ctl->kv_full[stage]);
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
            return;
          }
          if constexpr (PR) {
            // this CTA's half, counted on the leader's barrier: K-like tiles rows
            // [crank * BC/2, +BC/2) (both 64-column chunks), V tiles columns [crank * 64, +64)
            uint8_t* dst = sKV + stage * C::kKVBytes;
            if (crank == 0) mbar_arrive_expect_tx(&ctl->kv_full[stage], 2 * C::kKVBytes);
            if (map == &tmV) {
              tma_load_4d_pair(dst, map, &ctl->kv_full[stage], static_cast<int>(crank) * 64, row, unit.kvh, unit.b,
                               pol_kv);
            } else {
#pragma unroll
              for (int c = 0; c < 2; ++c)
                tma_load_4d_pair(dst + c * (BC / 2) * 128, map, &ctl->kv_full[stage], c * 64,
                                 row + static_cast<int>(crank) * (BC / 2), unit.kvh, unit.b, pol_kv);
            }
          } else if (VFA_WS1_MC) {
            mbar_arrive_expect_tx(&ctl->kv_full[stage], C::kKVBytes);
            tma_load_4d_mc(sKV + stage * C::kKVBytes + crank * (BC * 128), map, &ctl->kv_full[stage],
                           static_cast<int>(crank) * 64, row, unit.kvh, unit.b, static_cast<uint16_t>(3), pol_kv);
          } else {
            mbar_arrive_expect_tx(&ctl->kv_full[stage], C::kKVBytes);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_4d(sKV + stage * C::kKVBytes + h * (BC * 128), map, &ctl->kv_full[stage], h * 64, row, unit.kvh,
                          unit.b, pol_kv);
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        };
        auto load_s_operand = [&](int g) {
          if (g < nchunks)
            load_tile(&tmR, g * BC);
          else
            load_tile(&tmK, (sched_block(sched, g - nchunks) - 1) * BC);
        };
        // the MMA warps' consumption order: S-op(0 .. LA-1); per g: [V(g)], S-op(g + LA)
        for (int g = 0; g < LA && g < G; ++g) load_s_operand(g);
        for (int g = 0; g < G; ++g) {
          if (g >= nchunks) {
            load_tile(&tmV, (sched_block(sched, g - nchunks) - 1) * BC);
            VFA_TRACE_EVENT(a, g - nchunks, 12);  // V(g) TMA issued
          }
          if (g + LA < G) {
            load_s_operand(g + LA);
            if (g + LA >= nchunks) {
              VFA_TRACE_EVENT(a, g + LA - nchunks, 11);  // K(g + LA) TMA issued
              // V(g + SB) enters the ring only when K(g + SB)'s MMAs are done (5 stages), then
              // its TMA latency is on the PV path: warm L2 with it now
              if (VFA_WS1_VPREF)
                tma_prefetch_4d(&tmV, static_cast<int>(crank) * 64, (sched_block(sched, g + LA - nchunks) - 1) * BC,
                                unit.kvh, unit.b);
            }
          }
        }
      }
    } else if ((!PR || crank == 0) &&
               (warp == C::kMmaWarp || warp == C::kPvWarp || (VFA_WS1_QK2 && warp == C::kQk2Warp))) {
      // ============================ MMA issuers ============================
      // warp 16 issues the QK^T MMAs, warp 18 the PV MMAs: each one's barrier waits (~90
      // cycles a TRYWAIT, even when the phase is complete) overlap the other's queued MMAs,
      // where a single issuer's serial waits let the short tcgen05 queue run dry. QK(g + SB)
      // overwrites the S / P buffer of element g, so the QK issuer enqueues it only after the
      // PV issuer enqueued PV(g) (pv_issued; the tensor pipe runs MMAs in enqueue order).
      VFA_WS1_SETUP();
      const bool is_qk = warp != C::kPvWarp;
      constexpr uint32_t kIdescQK = make_idesc_bf16(128 * C::kPair, BC, false, false);
      constexpr uint32_t kIdescPV = make_idesc_bf16(128 * C::kPair, D, false, true);
      // completion signal: this CTA's barrier, or (pair) the same barrier of both CTAs
      auto commit_to = [&](uint64_t* bar) {
        if constexpr (PR)
          mma_commit_pair(bar);
        else
          mma_commit(bar);
      };
      constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t kLboK = 1u << 16;
      constexpr uint32_t kLboV = static_cast<uint32_t>((BC * 128) >> 4) << 16;
      // UMMA descriptors take the 18-bit shared::cta offset (14 bits of 16-byte units); in a
      // cluster launch the shared window address also carries the CTA rank (bit 24), masked off
      const uint32_t q_lo = ((smem_u32(sQ) >> 4) & 0x3FFFu) + kLboK;
      const uint32_t kv_lo = (smem_u32(sKV) >> 4) & 0x3FFFu;
      const uint32_t tO = tbase + C::kOOff;
      // both issuers walk the producer's load sequence (S-op(0 .. LA-1); per g: [V(g)],
      // [S-op(g + LA)]) and consume only their own tiles
      int stage = 0;
      uint32_t phase = 0;
      auto skip_tile = [&]() {
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
      };
      auto acquire = [&]() -> int {
        iwait(&ctl->kv_full[stage], phase);
        const int st = stage;
        skip_tile();
        return st;
      };
      auto release = [&](int st) {  // this CTA's MMAs on the stage done -> both producers
        if (elect_one()) {
          if (PR)
            mma_commit_pair(&ctl->kv_empty[st]);
          else if (VFA_WS1_MC)
            mma_commit_mc(&ctl->kv_empty[st], static_cast<uint16_t>(3));
          else
            mma_commit(&ctl->kv_empty[st]);
        }
        __syncwarp();
      };
#ifndef VFA_WS1_DBG_NOMMA
#define VFA_WS1_DBG_NOMMA 0  // timing experiments only (wrong results): no MMAs, barriers only
#endif
      // QK MMAs k-steps [k0, k1) into S buffer b; the commit to s_full after the last
      auto issue_qk = [&](int b, int st, int k0, int k1) {
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboK;
        if (VFA_WS1_DBG_NOMMA) {
          if (k1 == D / 16 && elect_one()) commit_to(&ctl->s_full[b]);
          __syncwarp();
          return;
        }
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            if (kk < k0 || kk >= k1) continue;
            const uint32_t off = ((kk >> 2) * (kBR * 128) + (kk & 3) * 32) >> 4;
            const uint32_t offk = ((kk >> 2) * ((BC / C::kPair) * 128) + (kk & 3) * 32) >> 4;
            const uint64_t da = (static_cast<uint64_t>(kHi) << 32) | (q_lo + off);
            const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + offk);
            if constexpr (PR)
              mma_ss_pair(tbase + C::s_off(b), da, db, kIdescQK, kk > 0 ? 1u : 0u);
            else
              mma_ss(tbase + C::s_off(b), da, db, kIdescQK, kk > 0 ? 1u : 0u);
          }
          if (k1 == D / 16) commit_to(&ctl->s_full[b]);
        }
        __syncwarp();
      };
      // PV of P chunk c: K-steps [0, C0/16) (chunk 0) or [C0/16, 4) (chunk 1) of each half (+4)
      auto issue_pv = [&](int b, int st, int c, bool first) {
        if (VFA_WS1_DBG_NOMMA) return;
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboV;
        const uint32_t tP = tbase + C::s_off(b);
        constexpr int K0 = VFA_WS1_C0 / 16;
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int kk = (i >> 2) * 4 + (i & 3);
            if (c == 0 ? (i & 3) >= K0 : (i & 3) < K0) continue;
            const bool lead = c == 0 && (i & 3) == 0 && (i >> 2) == 0;  // the element's first K-step
            const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + kk * (2048 >> 4));
            if constexpr (PR)
              mma_ts_pair(tO, tP + p_col(kk), db, kIdescPV, (first && lead) ? 0u : 1u);
            else
              mma_ts(tO, tP + p_col(kk), db, kIdescPV, (first && lead) ? 0u : 1u);
          }
        }
        __syncwarp();
      };
      if (is_qk) {
        mbar_wait(&ctl->q_full, 0);
        tc_fence_after();
        // the V tile of the load sequence between S-op(g) and S-op(g + 1), if any
        auto skip_v = [&](int g) {
          if (g >= LA - 1 && g + 1 < G && g - (LA - 1) >= nchunks) skip_tile();
        };
        // VFA_WS1_QK2: warps 16 and 19 issue the QK MMAs of alternate elements, so one issuer's
        // barrier waits and stage release after its eight k-steps overlap the other's queued
        // MMAs (a single issuer lets the three-deep MMA queue drain there, which is the rate
        // limit when the softmax is fast, e.g. VSA skipping most blocks)
        const int qk_par = (VFA_WS1_QK2 && warp != C::kMmaWarp) ? 1 : 0;
        for (int g = 0; g < G; ++g) {
          if (VFA_WS1_QK2 && (g & 1) != qk_par) {  // the other issuer's element
            skip_tile();
            skip_v(g);
            continue;
          }
          if (g >= SB) {  // PV(g - SB) enqueued (element g - SB's S / P buffer consumed)
            iwait(&ctl->pv_issued[g % SB], ((g - SB) / SB) & 1);
          }
          if (g >= nchunks && lane == 0) VFA_TRACE_EVENT(a, g - nchunks, 14);  // buffer free
          const int st = acquire();
          skip_v(g);
          tc_fence_after();
          if (g >= nchunks && lane == 0) VFA_TRACE_EVENT(a, g - nchunks, 13);  // K acquired
          issue_qk(g % SB, st, 0, D / 16);
          if (g >= SB && g - SB >= nchunks && lane == 0) VFA_TRACE_EVENT(a, g - SB - nchunks, 5);
          release(st);
        }
      } else {
        bool o_init = false;
        // the load sequence starts with min(LA, G) S operands
        for (int i = 0; i < LA && i < G; ++i) skip_tile();
        for (int g = 0; g < G; ++g) {
          const int b = g % SB;
          const uint32_t ph = (g / SB) & 1;
          const bool main_blk = g >= nchunks;
          const int pos = g - nchunks;
          if (VFA_WS1_PV_SKIPFIRST && skips(MODE) && main_blk) {
            // a skipped element frees its S / P buffer as soon as the softmax read S: tell the
            // QK issuer before waiting for the element's (unused) V tile
            iwait(&ctl->p_full[b][0], ph);
            if (ctl->skip[b] != 0) {
              if (lane == 0) VFA_TRACE_EVENT(a, pos, 4);
              iwait(&ctl->p_full[b][1], ph);
              if (g + SB < G) {
                if (elect_one()) mbar_arrive(&ctl->pv_issued[b]);
                __syncwarp();
              }
              const int vs = acquire();
              if (lane == 0) VFA_TRACE_EVENT(a, pos, 7);
              if (lane == 0) VFA_TRACE_EVENT(a, pos, 8);
              if (lane == 0) VFA_TRACE_EVENT(a, pos, 6);
              if (elect_one()) commit_to(&ctl->pv_done[pos & 1]);
              __syncwarp();
              release(vs);
              if (g + LA < G) skip_tile();
              continue;
            }
          }
          const int vs = main_blk ? acquire() : -1;
          if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 7);  // V acquired
          if constexpr (PR && skips(MODE))  // pairs with the follower's release (its skip flag)
            mbar_wait_cluster(&ctl->p_full[b][0], ph);
          else
            iwait(&ctl->p_full[b][0], ph);
          tc_fence_after();
          if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 4);  // MMA saw P chunk 0
          // (pair: the PV is one MMA for both CTAs; a CTA that skips hands over P = 0)
          const bool skip = skips(MODE) && (PR ? (ctl->skip2[b][0] != 0 && ctl->skip2[b][1] != 0) : ctl->skip[b] != 0);
          if (main_blk && !skip) issue_pv(b, vs, 0, !o_init);
          iwait(&ctl->p_full[b][1], ph);
          tc_fence_after();
          if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 8);  // MMA saw P chunk 1
          if (main_blk) {
            if (!skip) issue_pv(b, vs, 1, false);
            if (lane == 0) VFA_TRACE_EVENT(a, pos, 6);  // PV issued
            o_init = o_init || !skip;
            if (elect_one()) commit_to(&ctl->pv_done[pos & 1]);
            __syncwarp();
            release(vs);
          }
          if (g + SB < G) {  // QK(g + SB) may now overwrite this buffer
            if (elect_one()) mbar_arrive(&ctl->pv_issued[b]);
            __syncwarp();
          }
          if (g + LA < G) skip_tile();  // S-op(g + LA) in the load sequence
        }
        if (elect_one()) commit_to(&ctl->o_final);
        __syncwarp();
      }
    }
  } else {
    // ============================ softmax groups ============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(VFA_WS1_REGS_SOFTMAX));
    VFA_WS1_SETUP();
    const int gi = warp >> 3;         // group: elements g with g % NG == gi
    const int hf = (warp >> 2) & 1;   // half of every S row (64 columns)
    const int r = tid & 127;
    constexpr int CP = 64;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tbase + C::kOOff + hf * CP + lane_off;
    const int R = unit.qt * kBR + r;
    const float cs = a.c_scale;
    const float2 cs2 = make_float2(cs, cs);
    auto tS = [&](int b) { return tbase + C::s_off(b) + lane_off; };
    auto wait_s = [&](int g) {
      swait(&ctl->s_full[g % SB], (g / SB) & 1);
      tc_fence_after();
    };
    // P hand-offs arrive on the MMA-issuing CTA's barrier (a pair's leader); the TMEM data is
    // ordered by tcgen05 fences, so a follower's remote arrive is relaxed except for the one
    // that also publishes the skip flag (lane 0 of warps 0 / 8: cluster-scope release)
    auto arrive_p = [&](uint64_t* bar, bool flag) {
      if constexpr (PR) {
        if (crank == 0)
          mbar_arrive(bar);
        else if (flag)
          mbar_arrive_cluster(mapa_shared(bar, 0));
        else
          mbar_arrive_cluster_relaxed(mapa_shared(bar, 0));
      } else {
        (void)flag;
        mbar_arrive(bar);
      }
    };
    const bool flag_writer = skips(MODE) && (warp & 7) == 0;  // lane 0 of it writes the skip flag
    auto consumed = [&](int g) {  // S of element g read (m-init chunk) or handed over as P
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        arrive_p(&ctl->p_full[g % SB][0], flag_writer);
        arrive_p(&ctl->p_full[g % SB][1], false);
      }
    };
    // ---- m-init: m0 = max_j scale * q . krepr_j over visible j <= tc1 (src/vfa.py:91-106)
    // the schedule facts of every visit position, computed once by all softmax threads (the
    // per-element integer chains of sched_block & co. otherwise sit on each group's critical path)
    const bool use_tab = VFA_WS1_STAB && N <= C::kSchedTab;
    if (use_tab) {
      for (int p = tid; p < N; p += 256 * NG) {
        const int jj = sched_block(sched, p);
        const bool sp = all_exact(MODE) || sched_is_special(sched, jj);
        const bool mk = sched_needs_mask(unit.qt + 1, jj, kBR, BC, a.causal != 0);
        ctl->sinfo[p] = static_cast<uint16_t>(jj | (sp ? 1 << 14 : 0) | (mk ? 1 << 15 : 0));
      }
      named_bar_sync(kAllBar, 256 * NG);
    }
    const bool strace = a.skip_trace != nullptr && r == 0 && hf == 0;
    float m2 = -INFINITY;  // running max this group's normalizer part is relative to (log2 units)
    if (nchunks > 0) {
      float mx = -INFINITY;
      for (int g = gi; g < nchunks; g += NG) {
        wait_s(g);
        const int valid = nrep - g * BC - hf * CP;
        if constexpr (kLowReg) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            float v[32];
            tmem_ld32(tS(g % SB) + hf * CP + c * 32, v);
            tmem_wait_ld();
            reg_fence32(v);
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e < valid) mx = fmaxf(mx, v[e]);
          }
        } else {
          float v[CP];
          tmem_ld32(tS(g % SB) + hf * CP, v);
          tmem_ld32(tS(g % SB) + hf * CP + 32, v + 32);
          tmem_wait_ld();
          reg_fence32(v);
          reg_fence32(v + 32);
#pragma unroll
          for (int e = 0; e < CP; ++e)
            if (e < valid) mx = fmaxf(mx, v[e]);
        }
        consumed(g);
      }
      ctl->xinit[gi][hf][r] = mx;
      named_bar_sync(kAllBar, 256 * NG);
      float mi = -INFINITY;
#pragma unroll
      for (int q = 0; q < NG; ++q) mi = fmaxf(mi, fmaxf(ctl->xinit[q][0][r], ctl->xinit[q][1][r]));
      m2 = mi * cs;
    }
    if ((MODE == kVFA || MODE == kVSA) && a.use_m_init && a.m0_tile != nullptr)
      m2 = a.m0_tile[(static_cast<size_t>(unit.b) * a.Hq + head) * a.Tr + unit.qt] * cs;

    float l = 0.f;
    int stab = sched_block(sched, 0);
    int ver = 0;   // running-max versions (exact positions) this group has incorporated
    int n_ex = 0;  // exact positions this group processed (row-max exchange buffer parity)
    int n_visit = 0, n_skipped = 0, n_skipped_special = 0;
    // bring m2 / l / stab up to version v (published by the other group)
    auto catch_up = [&](int v) {
      if (v <= ver) return;
      const int slot = (v - 1) % NV;
      swait(&ctl->mver[slot], ((v - 1) / NV) & 1);
      const float mn = ctl->m_pub[slot][r];
      stab = ctl->stab_pub[slot][r];
      if (mn != m2) {
        l = __fmul_rn(l, ex2_approx(m2 - mn));  // (m2 = -inf: l is 0, the factor 0)
        m2 = mn;
      }
      ver = v;
    };
    // S of the group's next element is usually ready long before this one is done (QK runs up
    // to three elements ahead): its first 32 columns are loaded right after this element's last
    // P hand-off, so the TMEM load latency overlaps the tail of this element and the loop
    float v[kLowReg ? 32 : CP];
    bool prefetched = false;  // chunk 0 of element g is already loading into v[0 .. 31]
    // per-position schedule facts (key block, exact / masked, exact positions before it); with
    // VFA_WS1_PIPE the next position's are computed while this position's S loads from TMEM, so
    // the integer chains of the schedule are off the group's per-block critical path
    struct Step {
      int j, E;
      bool special, mask;
    };
    auto step_at = [&](int pos) {
      Step st;
      st.j = sched_block(sched, pos);
      st.special = all_exact(MODE) || sched_is_special(sched, st.j);
      st.mask = sched_needs_mask(unit.qt + 1, st.j, kBR, BC, a.causal != 0);
      st.E = exact_before<MODE>(sched, pos);
      return st;
    };
    const int g_first = nchunks + (((gi - nchunks) % NG) + NG) % NG;
    Step nxt = step_at(g_first - nchunks);
    for (int g = g_first; g < G; g += NG) {
      const int pos = g - nchunks;
      const int b = g % SB;
      Step cur;
      if (use_tab) {
        const uint32_t info = ctl->sinfo[pos];
        cur.j = static_cast<int>(info & 0x3FFFu);
        cur.special = (info >> 14) & 1u;
        cur.mask = (info >> 15) & 1u;
        cur.E = exact_before<MODE>(sched, pos);
      } else {
        cur = VFA_WS1_PIPE ? nxt : step_at(pos);
      }
      const int j = cur.j;
      const bool special = cur.special;
      const bool mask = cur.mask;
      const int E = cur.E;
      ++n_visit;
      catch_up(E);  // the running max after every exact position before this one
      if (!prefetched) {
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 3);  // (ws1 slots: see scripts/trace_timeline.py --ws1)
        wait_s(g);
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 0);
        tmem_ld32(tS(b) + hf * CP, v);
      }
      if (VFA_WS1_PIPE && g + 2 < G) nxt = step_at(pos + 2);
      if (r == 0 && hf == 0 && pos == 0) VFA_TRACE_UNIT(a, 1);
      const bool split = MODE == kVFA && !special;  // no row statistic before the exponentials
      const int lim = R - (j - 1) * BC - hf * CP;
      // kLowReg: the 64-column row max of a non-split element (VSA test / exact update), taken
      // over two sequential 32-column loads; its exponentials then reload chunk 0
      float pmax_all = -INFINITY;
      if constexpr (kLowReg) {
        tmem_wait_ld();
        reg_fence32(v);
        if (mask) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
        }
        if (!split) {
          const float pm0 = part_max<32>(v);
          tmem_ld32(tS(b) + hf * CP + 32, v);
          tmem_wait_ld();
          reg_fence32(v);
          if (mask) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = (e + 32 > lim) ? -INFINITY : v[e];
          }
          pmax_all = fmaxf(pm0, part_max<32>(v));
        }
      } else {
        if (split) {
          tmem_wait_ld();
          reg_fence32(v);
          tmem_ld32(tS(b) + hf * CP + 32, v + 32);
        } else {
          tmem_ld32(tS(b) + hf * CP + 32, v + 32);
          tmem_wait_ld();
          reg_fence32(v);
          reg_fence32(v + 32);
        }
        if (mask) {  // entrywise causal mask (src/reference.py:93-96)
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
          if (!split) {
#pragma unroll
            for (int e = 32; e < CP; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
          }
        }
      }
      if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 15);  // S (first chunk) in registers
      bool skipped = false;
      bool rescale = false;
      float f = 1.0f;
      if (MODE == kVSA && !special) {
        // VSA frozen block: the skip test only (src/sparse.py:296-304), against the frozen max
        const float pm2 = (kLowReg ? pmax_all : part_max<CP>(v)) * cs;
        const bool below = (pm2 - fmaxf(m2, pm2) < a.log2_lambda) ||
                           (pm2 == -INFINITY && m2 == -INFINITY && a.log2_lambda != -INFINITY);
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 9);  // S in registers, max taken
        skipped = named_bar_and(1 + gi, 256, below);
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 10);  // skip decided
        if (skipped) ++n_skipped;
      } else if (special) {
        // exact update (src/vfa.py:202-208): row max over both halves, then publish version E+1
        const int xp = n_ex & 1;
        ctl->xmax[gi][xp][hf][r] = kLowReg ? pmax_all : part_max<CP>(v);
        named_bar_sync(1 + gi, 256);
        const float mt2 = fmaxf(ctl->xmax[gi][xp][0][r], ctl->xmax[gi][xp][1][r]) * cs;
        ++n_ex;
        const float m2n = fmaxf(m2, mt2);
        if (skips(MODE)) {
          const bool below = (mt2 - m2n < a.log2_lambda) ||
                             (mt2 == -INFINITY && m2n == -INFINITY && a.log2_lambda != -INFINITY);
          skipped = named_bar_and(1 + gi, 256, below);
        }
        if (skipped) {
          ++n_skipped;
          ++n_skipped_special;
        } else {
          f = (m2n == -INFINITY) ? 1.0f : ex2_approx(m2 - m2n);
          if (m2n > m2) stab = j;
          m2 = m2n;
          l = __fmul_rn(l, f);
          rescale = pos > 0 && !__all_sync(0xffffffffu, f == 1.0f);
        }
        const int slot = E % NV;
        if (hf == 0) {
          ctl->m_pub[slot][r] = m2;
          ctl->stab_pub[slot][r] = stab;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->mver[slot]);
        ver = E + 1;
      }
      if (skips(MODE) && r == 0 && hf == 0) {
        if constexpr (PR)  // the leader's PV issuer needs both CTAs' decisions
          st_cluster_u32(mapa_shared(&ctl->skip2[b][crank], 0), skipped ? 1u : 0u);
        else
          ctl->skip[b] = skipped ? 1u : 0u;
      }
      if (strace)
        a.skip_trace[((static_cast<size_t>(unit.b) * a.Hq + head) * a.Tr + unit.qt) * a.Tc + pos] = skipped ? 2 : 1;
      if (rescale) {
        // O holds PV of every earlier position once PV(pos-1) completed (S(pos) ready implies
        // PV(pos-3) did, and PV(pos) waits for this group's P, so pv_done[(pos-1) & 1] is in or
        // just past phase (pos-1) >> 1): wait for it, then rescale this half of the row
        swait(&ctl->pv_done[(pos - 1) & 1], ((pos - 1) >> 1) & 1);
        tc_fence_after();
        const float2 f2 = make_float2(f, f);
#pragma unroll 1
        for (int c = 0; c < CP / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
          tmem_wait_ld();
          reg_fence16(o);
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 x = __fmul2_rn(make_float2(o[e], o[e + 1]), f2);
            o[e] = x.x;
            o[e + 1] = x.y;
          }
          tmem_st16(tO + c * 16, reinterpret_cast<const uint32_t*>(o));
        }
        tmem_wait_st();
      }
      if (!skipped) {
        const float nm = (m2 == -INFINITY ? 0.f : -m2);
        // row sum (src/tensor.py:81-89) in two packed accumulators, pairs in column order
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // chunk 0 = columns [0, C0), chunk 1 = [C0, 64): a smaller first chunk hands P to the
        // PV issuer earlier (VFA_WS1_C0)
        constexpr int C0 = VFA_WS1_C0;
        static_assert(C0 == 16 || C0 == 32, "first P chunk");
        static_assert(!kLowReg || C0 == 32, "three groups: 32-column chunks");
        uint32_t u[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float nmc = nm;
          if (c > 0) {  // ordered after chunk 0's hand-off (see ws_kernel.cuh)
            float z;
            asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(z) : "r"(smem_u32(&ctl->zero)) : "memory");
            nmc = nm + z;
          }
          if (kLowReg && (c == 1 || !split)) {  // this chunk's 32 columns into the registers
            tmem_ld32(tS(b) + hf * CP + c * 32, v);
            tmem_wait_ld();
            reg_fence32(v);
            if (mask) {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = (e + c * 32 > lim) ? -INFINITY : v[e];
            }
          }
          const float2 nmu2 = make_float2(nmc, nmc);
#pragma unroll
          for (int e = 0; e < CP; e += 2) {
            if (c == 0 ? e >= C0 : e < C0) continue;
            if (!kLowReg && c == 1 && e == 32 && split) {  // the second 32 columns' TMEM load
              tmem_wait_ld();
              reg_fence32(v + 32);
              if (mask) {
#pragma unroll
                for (int e2 = 32; e2 < CP; ++e2) v[e2] = (e2 > lim) ? -INFINITY : v[e2];
              }
            }
            const int ev = kLowReg ? e - c * 32 : e;
            const float2 x = __ffma2_rn(make_float2(v[ev], v[ev + 1]), cs2, nmu2);
            float2 p;
            if (((e >> 1) & 7) >= 8 - VFA_WS1_EMU) {
              p = ex2_poly2(x);  // degree 4, |rel err| < 3e-6
            } else {
              p.x = ex2_approx(x.x);
              p.y = ex2_approx(x.y);
            }
            acc[(e >> 1) & 1] = add_ftz2(acc[(e >> 1) & 1], p);
            u[e >> 1] = pack_bf16x2(p.x, p.y);
          }
          if (C0 == 32) {
            tmem_st16(tS(b) + hf * CP + c * 16, u + c * 16);
          } else if (c == 0) {
            tmem_st8(tS(b) + hf * CP, u);
          } else {
            tmem_st8(tS(b) + hf * CP + 8, u + 8);
            tmem_st16(tS(b) + hf * CP + 16, u + 16);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_p(&ctl->p_full[b][c], flag_writer && c == 0);
          if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, c == 0 ? 2 : 1);
        }
        l = __fadd_rn(l, __fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)));
      } else {
        if (split) tmem_wait_ld();
        if constexpr (PR) {
          // the pair's PV runs unless both CTAs skip: this CTA's P of the block must be zero
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
          tmem_st16(tS(b) + hf * CP, z);
          tmem_st16(tS(b) + hf * CP + 16, z);
          tmem_wait_st();
        }
        consumed(g);
        if (r == 0 && hf == 0) {
          VFA_TRACE_EVENT(a, pos, 2);
          VFA_TRACE_EVENT(a, pos, 1);
        }
      }
      // start loading the group's next element (v is free: the row sum was taken on the fly)
      prefetched = VFA_WS1_PREFETCH && g + 2 < G;
      if (prefetched) {
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos + 2, 3);
        wait_s(g + 2);
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos + 2, 0);
        tmem_ld32(tS((g + 2) % SB) + hf * CP, v);
      }
    }
    if (r == 0 && hf == 0 && gi == 1) VFA_TRACE_UNIT(a, 2);
    // ---- finalize (src/core.py:101-109): both groups' parts relative to the final max
    catch_up(exact_before<MODE>(sched, N));
    ctl->xl[gi][hf][r] = l;
    named_bar_sync(kAllBar, 256 * NG);
    float lsum = __fadd_rn(__fadd_rn(ctl->xl[0][0][r], ctl->xl[0][1][r]), __fadd_rn(ctl->xl[1][0][r], ctl->xl[1][1][r]));
#pragma unroll
    for (int q = 2; q < NG; ++q) lsum = __fadd_rn(lsum, __fadd_rn(ctl->xl[q][0][r], ctl->xl[q][1][r]));
    const int qq = warp >> 2;  // this thread's 32-column quarter of the O row (warps 0-15)
    const size_t lrow = (static_cast<size_t>(unit.b) * a.Hq + head) * a.Lq + R;
    const unsigned srow = static_cast<unsigned>(lrow + a.row_base);
    if (qq == 0) {
      if (a.lse) a.lse[lrow] = (lsum == 0.f && m2 != -INFINITY) ? m2 * kLn2 : (m2 + __log2f(lsum)) * kLn2;
      if (a.stab) a.stab[lrow] = stab;
      if (a.status && lsum == 0.f) {
        if (m2 == -INFINITY) {
          atomicOr(&a.status[VFA_STATUS_FLAGS], 1u);
          atomicMin(&a.status[VFA_STATUS_MASKED_ROW], srow);
        } else {
          atomicOr(&a.status[VFA_STATUS_FLAGS], 2u);
          atomicMin(&a.status[VFA_STATUS_UNDERFLOW_ROW], srow);
        }
      }
    }
    mbar_wait(&ctl->o_final, 0);
    tc_fence_after();
    const float inv = 1.0f / lsum;
    __nv_bfloat16* orow = a.o + unit.b * a.o_sb + head * a.o_sh + static_cast<long long>(R) * a.o_sr + qq * 32;
    bool finite = true;
    if (qq < 4) {
      float o[32];
      tmem_ld32(tbase + C::kOOff + qq * 32 + lane_off, o);
      tmem_wait_ld();
      reg_fence32(o);
      uint32_t u[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float o0 = o[e] * inv, o1 = o[e + 1] * inv;
        finite = finite && isfinite(o0) && isfinite(o1);
        u[e >> 1] = pack_bf16x2(o0, o1);
      }
      uint4* dst = reinterpret_cast<uint4*>(orow);
      dst[0] = make_uint4(u[0], u[1], u[2], u[3]);
      dst[1] = make_uint4(u[4], u[5], u[6], u[7]);
      dst[2] = make_uint4(u[8], u[9], u[10], u[11]);
      dst[3] = make_uint4(u[12], u[13], u[14], u[15]);
    }
    if (a.status) {
      if (qq < 4) ctl->xfin[qq][r] = finite ? 1 : 0;
      named_bar_sync(kAllBar, 256 * NG);
      if (qq == 0 && !(ctl->xfin[0][r] && ctl->xfin[1][r] && ctl->xfin[2][r] && ctl->xfin[3][r])) {
        atomicAdd(&a.status[VFA_STATUS_NONFINITE_ROWS], 1u);
        atomicOr(&a.status[VFA_STATUS_FLAGS], 4u);
      }
    }
    if (a.stats && r == 0 && hf == 0) {
      const int n_exact = all_exact(MODE) ? N : sched.n_spec;
      if (gi == 0) {
        atomicAdd(&a.stats[VFA_STAT_VISITED], static_cast<unsigned long long>(N));
        atomicAdd(&a.stats[VFA_STAT_SPECIAL], static_cast<unsigned long long>(n_exact));
        atomicAdd(&a.stats[VFA_STAT_FROZEN], static_cast<unsigned long long>(N - n_exact));
      }
      if (n_skipped) {
        atomicAdd(&a.stats[VFA_STAT_SKIPPED], static_cast<unsigned long long>(n_skipped));
        // skipped blocks leave their class (counted once per tile, as in vfa_fwd_kernel)
        atomicAdd(&a.stats[VFA_STAT_SPECIAL], static_cast<unsigned long long>(-n_skipped_special));
        atomicAdd(&a.stats[VFA_STAT_FROZEN], static_cast<unsigned long long>(-(n_skipped - n_skipped_special)));
      }
    }
    (void)n_visit;
  }
#undef VFA_WS1_SETUP
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer may still multicast into / commit onto this CTA's shared memory
  if (tid == 0) VFA_TRACE_UNIT(a, 3);
  if (warp == C::kMmaWarp) {
    tc_fence_after();
    if constexpr (PR)
      tmem_dealloc_pair<512>(ctl->tmem_base);
    else
      tmem_dealloc<512>(ctl->tmem_base);
  }
}

#undef iwait
#undef swait

}  // namespace vfa
