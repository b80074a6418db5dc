// B200 (sm_100a) warp-specialised attention forward for the headline shape: head_dim 128,
// 128-key blocks, 128-row query blocks, two query heads of one GQA group per CTA.
//
// Same work unit, schedule, m-init prologue and per-block math as vfa_fwd_kernel
// (vfa_kernel.cuh; reference map there), with the roles arranged so that no role waits on
// another's latency:
//   warps 0-7   softmax of query tile 0: two warps per sub-partition, two threads per row
//               (TMEM lane = row, 64 S columns each); they also rescale O on exact-update
//               blocks (src/core.py:91) and run the epilogue (O / l, LSE, src/core.py:101-109)
//   warps 8-15  softmax of query tile 1
//   warps 16-17 MMA issuers, one per query tile (converged warps, elect.sync), taking turns;
//               16 allocates TMEM
//   warp 18     TMA producer
//   warp 19     idle (completes the last warpgroup)
// TMEM (512 columns): S_t at t*128 (P_t packed bf16 in its columns 0-31 / 64-95, see p_col), O_t at
// 256 + t*128. Per key block and tile the tensor pipe runs PV_t, QK_t(next); the issuers'
// turn-taking keeps the order PV_0 QK_0 PV_1 QK_1, so each tile's softmax runs under the other
// tile's MMAs.
// Exponentials: exp2 on MUFU.EX2 for most element pairs and a degree-3 polynomial on the FMA
// pipe for VFA_WS_EMU of every 8 pairs, so the XU (16 exp2 per SM-cycle = exactly the tensor
// pipe's rate at d = 128) is not the bound. Row sums are taken after the P hand-off (off the
// S -> P -> PV chain).
#pragma once
#include "vfa_kernel.cuh"

namespace vfa {

#ifndef VFA_WS_EMU
#define VFA_WS_EMU 1  // element pairs (of 8) on the FMA-pipe exp2 in the chunks VFA_WS_EMU_CHUNKS
#endif
#ifndef VFA_WS_EMU_CHUNKS
#define VFA_WS_EMU_CHUNKS 0x3  // bit c: a thread's 32-column chunk c uses the FMA-pipe exp2
#endif
#ifndef VFA_WS_ACQ_FENCE
#define VFA_WS_ACQ_FENCE 1  // tcgen05 fence after the K/V full wait (experiments: 0)
#endif
#ifndef VFA_WS_NCH
#define VFA_WS_NCH 2  // P hand-off chunks per thread (2: 32 columns each, 4: 16 columns each)
#endif
constexpr int kNCH = VFA_WS_NCH;
constexpr int kCW = 64 / kNCH;  // columns per P chunk
static_assert(kNCH == 2 || kNCH == 4, "P hand-off in 2 or 4 chunks");
#ifndef VFA_WS_POLY3
#define VFA_WS_POLY3 0  // 1: degree-3 FMA-pipe exp2 (fewer instructions, 8.6e-5 relative error)
#endif
#ifndef VFA_WS_TOKEN
#define VFA_WS_TOKEN 1  // MMA issuers take turns (0: free-running, the tiles drift into phase)
#endif
#ifndef VFA_WS_REGS_SOFTMAX
#define VFA_WS_REGS_SOFTMAX 104
#endif
#ifndef VFA_WS_REGS_OTHER
#define VFA_WS_REGS_OTHER 64
#endif

struct WsCfg {
  static constexpr int D = 128, BC = 128, NQ = 2;
  static constexpr int kThreads = 640;  // 16 softmax warps + 2 MMA issuers + TMA + 1 idle
  static constexpr int kMmaWarp = 16;   // and 17: one MMA issuer per query tile
  static constexpr int kLoadWarp = 18;
  static constexpr int kQBytes = kBR * D * 2;    // 32 KB
  static constexpr int kKVBytes = BC * D * 2;    // 32 KB
#ifndef VFA_WS_STAGES
#define VFA_WS_STAGES 4
#endif
  // K/V ring: the MMA issuers hold V(g) and K(g+1); the other stages are loads in flight
  static constexpr int kStages = VFA_WS_STAGES;
  static constexpr int kCtlBytes = 8192;  // control block after the tiles
  static constexpr int kSmem = kCtlBytes + NQ * kQBytes + kStages * kKVBytes;
  static __device__ __forceinline__ uint32_t s_off(int t) { return static_cast<uint32_t>(t * 128); }
  static __device__ __forceinline__ uint32_t o_off(int t) { return static_cast<uint32_t>(256 + t * 128); }
  static_assert(kSmem <= kMaxSmem, "shared memory");
  // setmaxnreg pool = the launch allocation (640 threads x 96 registers)
  static constexpr int kRegBudget = (4 * VFA_WS_REGS_SOFTMAX + VFA_WS_REGS_OTHER) * 128;
  static_assert(kRegBudget <= 640 * 96, "register budget");
};

struct __align__(16) WsCtl {
  uint64_t q_full[2];
  uint64_t kv_full[WsCfg::kStages];
  uint64_t kv_empty[WsCfg::kStages];
  uint64_t s_full[2];     // MMA -> softmax t: S_t of sequence element g ready (parity g & 1)
  uint64_t s_free[2];     // softmax t -> MMA: m-init chunk read, S_t may be overwritten
  uint64_t p_full[2][4];  // softmax t -> MMA: P chunk c in TMEM (or the block skipped)
  uint64_t o_final[2];    // MMA -> correction: last PV_t complete
  uint64_t tok[2];        // MMA issuer 1-t -> issuer t: your turn to enqueue (keeps the tiles in anti-phase)
  uint32_t tmem_base;
  uint32_t skip[2];
  float zero;             // 0.0f: read back (volatile) to order softmax chunks, see chunk_bias
  float xmax[2][2][kBR];  // [tile][half][row]: row-max exchange between the two halves of a row
  float xl[2][2][kBR];    // [tile][half][row]: final partial row sums
  uint8_t xfin[2][2][kBR];  // [tile][half][row]: output finite flags
};
static_assert(sizeof(WsCtl) <= WsCfg::kCtlBytes, "control block");

// named barriers (0 = __syncthreads): 1+t rescale hand-off, 3+t final sums (256 threads:
// softmax t + correction), 5+t softmax t's CTA-wide votes (128 threads)
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(WsCfg::kThreads, 1)
    vfa_ws_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmR,
                  const FwdArgs a) {
  using C = WsCfg;
  constexpr int D = C::D, BC = C::BC, NS = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the dynamic shared window starts 1 KB aligned (no static shared memory): control block,
  // then the SWIZZLE_128B tiles at a 1 KB boundary
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  // SWIZZLE_128B tiles from the (1 KB aligned) start of the window, control block after them
  uint8_t* sQ = smem_raw;
  uint8_t* sKV = sQ + 2 * C::kQBytes;
  WsCtl* ctl = reinterpret_cast<WsCtl*>(sKV + NS * C::kKVBytes);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    VFA_TRACE_UNIT(a, 0);
    ctl->zero = 0.f;
    for (int t = 0; t < 2; ++t) {
      mbar_init(&ctl->q_full[t], 1);
      mbar_init(&ctl->s_full[t], 1);
      mbar_init(&ctl->s_free[t], 8);
      for (int c = 0; c < 4; ++c) mbar_init(&ctl->p_full[t][c], 8);
      mbar_init(&ctl->o_final[t], 1);
      mbar_init(&ctl->tok[t], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&ctl->kv_full[s], 1);
      mbar_init(&ctl->kv_empty[s], 2);  // released by both MMA issuers
    }
    fence_barrier_init();
  }
  if (warp == C::kLoadWarp && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmR);
  }
  if (warp == C::kMmaWarp) tmem_alloc<512>(&ctl->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

#define VFA_WS_SETUP()                                                   \
  const uint32_t tbase = ctl->tmem_base;                                 \
  const Unit unit = decode_unit(a, blockIdx.x);                          \
  const TileSchedule sched = unit_schedule<MODE>(a, unit.qt, BC);        \
  const int N = sched.vmax;                                              \
  int nrep = 0;                                                          \
  const int nchunks = minit_chunks<MODE>(a, sched, BC, &nrep);           \
  const int G = nchunks + N;                                             \
  (void)tbase; (void)nrep; (void)G
  // exact (rowmax + rescale) update at visit position pos
  auto exact_at = [&](const TileSchedule& s, int pos) {
    return all_exact(MODE) || sched_is_special(s, sched_block(s, pos));
  };

  if (warp >= C::kMmaWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(VFA_WS_REGS_OTHER));
    if (warp == C::kLoadWarp) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        VFA_WS_SETUP();
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        for (int t = 0; t < 2; ++t) {
          mbar_arrive_expect_tx(&ctl->q_full[t], C::kQBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d(sQ + t * C::kQBytes + c * kBR * 128, &tmQ, &ctl->q_full[t], c * 64, unit.qt * kBR,
                        unit.h0 + t, unit.b, pol_q);
        }
        int stage = 0;
        uint32_t phase = 0;
#ifndef VFA_WS_DBG_SKIP
#define VFA_WS_DBG_SKIP 0  // timing experiments only (wrong results): 1 = no V transfers, 2 = no K transfers
#endif
        int nload = 0;
        auto load_tile = [&](const CUtensorMap* map, int row) {
          mbar_wait(&ctl->kv_empty[stage], phase ^ 1);
          uint8_t* dst = sKV + stage * C::kKVBytes;
          if (VFA_WS_DBG_SKIP && nload++ >= 8 &&
              ((VFA_WS_DBG_SKIP == 1 && map == &tmV) || (VFA_WS_DBG_SKIP == 2 && map == &tmK))) {
            mbar_arrive(&ctl->kv_full[stage]);
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
            return;
          }
          mbar_arrive_expect_tx(&ctl->kv_full[stage], C::kKVBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d(dst + c * BC * 128, map, &ctl->kv_full[stage], c * 64, row, unit.kvh, unit.b, pol_kv);
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
        // the MMA warp's consumption order: S-op(0); per g: [V(g)], S-op(g+1)
        load_s_operand(0);
        for (int g = 0; g < G; ++g) {
          if (g >= nchunks) {
            load_tile(&tmV, (sched_block(sched, g - nchunks) - 1) * BC);
            VFA_TRACE_EVENT(a, g - nchunks, 15);
          }
          if (g + 1 < G) {
            load_s_operand(g + 1);
            if (g >= nchunks) VFA_TRACE_EVENT(a, g - nchunks, 16);
          }
        }
      }
    } else if (warp <= C::kMmaWarp + 1) {
      // ============================ MMA issuers (one per query tile) ============================
      // Warp 12 + t issues tile t's MMAs: QK_t(0); per sequence element g: PV_t(g) (after the
      // softmax's P hand-off), QK_t(g+1). Two issuers let one tile's barrier waits (a TRYWAIT costs
      // ~90 cycles even when the phase is complete) overlap the other tile's issue, so the short
      // tcgen05 queue does not drain between MMA groups. Both consume the same K/V ring stages;
      // a stage is released when both issuers' MMAs on it complete (kv_empty counts 2 commits).
      VFA_WS_SETUP();
      const int t = warp - C::kMmaWarp;
      constexpr uint32_t kIdescQK = make_idesc_bf16(128, BC, false, false);
      constexpr uint32_t kIdescPV = make_idesc_bf16(128, D, false, true);
      constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t kLboK = 1u << 16;
      constexpr uint32_t kLboV = static_cast<uint32_t>((BC * 128) >> 4) << 16;
      const uint32_t q_lo = (smem_u32(sQ) >> 4) + t * (C::kQBytes >> 4) + kLboK;
      const uint32_t kv_lo = smem_u32(sKV) >> 4;
      const uint32_t tS = tbase + C::s_off(t), tO = tbase + C::o_off(t);
      int stage = 0;
      uint32_t phase = 0;
      auto acquire = [&]() -> int {
        mbar_wait(&ctl->kv_full[stage], phase);
        if (VFA_WS_ACQ_FENCE) tc_fence_after();
        const int st = stage;
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
        return st;
      };
      auto release = [&](int st) {
        if (elect_one()) mma_commit(&ctl->kv_empty[st]);
        __syncwarp();
      };
      auto issue_qk = [&](int st) {
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboK;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * (kBR * 128) + (kk & 3) * 32) >> 4;
            const uint64_t da = (static_cast<uint64_t>(kHi) << 32) | (q_lo + off);
            const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + off);
            mma_ss(tS, da, db, kIdescQK, kk > 0 ? 1u : 0u);
          }
          mma_commit(&ctl->s_full[t]);
        }
        __syncwarp();
      };
      // PV of P chunk c: each half's chunk c = K-steps 4*hf + c*kCW/16 .. + kCW/16 (16 keys per
      // K-step; P K-step k in TMEM columns [8k, 8k + 8))
      auto issue_pv = [&](int st, int c, bool first) {
        const uint32_t b_lo = kv_lo + st * (C::kKVBytes >> 4) + kLboV;
        constexpr int kKS = kCW / 16;  // K-steps per half and chunk
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 2 * kKS; ++i) {
            const int kk = (i / kKS) * 4 + c * kKS + (i % kKS);
            const uint64_t db = (static_cast<uint64_t>(kHi) << 32) | (b_lo + kk * (2048 >> 4));
            mma_ts(tO, tS + p_col(kk), db, kIdescPV, (first && i == 0) ? 0u : 1u);
          }
        }
        __syncwarp();
      };
      // turn-taking: the tensor pipe sees PV_0(g) QK_0(g+1) PV_1(g) QK_1(g+1) ... as with one
      // issuer (tile 1's MMAs run under tile 0's softmax and vice versa), but each issuer's
      // barrier waits happen while the other issuer's MMAs fill the queue
      uint32_t tok_ph = 0;
      auto take_turn = [&]() {
        if (VFA_WS_TOKEN) {
          mbar_wait(&ctl->tok[t], tok_ph);
          tok_ph ^= 1u;
        }
      };
      auto pass_turn = [&]() {
        if (VFA_WS_TOKEN) {
          if (elect_one()) mbar_arrive(&ctl->tok[1 - t]);
          __syncwarp();
        }
      };
      mbar_wait(&ctl->q_full[t], 0);
      tc_fence_after();
      {
        const int st = acquire();
        if (t == 1) take_turn();
        issue_qk(st);
        pass_turn();
        release(st);
      }
      bool o_init = false;
      uint32_t p_ph = 0;
      for (int g = 0; g < G; ++g) {
        const bool main_blk = g >= nchunks;
        const int pos = g - nchunks;
        if (main_blk) {
          const int vs = acquire();
          if (t == 0 && lane == 0) VFA_TRACE_EVENT(a, pos, 17);
          mbar_wait(&ctl->p_full[t][0], p_ph);
          tc_fence_after();
          if (lane == 0) VFA_TRACE_EVENT(a, pos, 4 + 2 * t);
          const bool skip = skips(MODE) && ctl->skip[t] != 0;
          take_turn();
          if (!skip) issue_pv(vs, 0, !o_init);
#pragma unroll
          for (int c = 1; c < kNCH; ++c) {
            mbar_wait(&ctl->p_full[t][c], p_ph);
            tc_fence_after();
            if (c == kNCH - 1 && lane == 0) VFA_TRACE_EVENT(a, pos, 8 + 2 * t);
            if (!skip) issue_pv(vs, c, false);
          }
          if (lane == 0) VFA_TRACE_EVENT(a, pos, 9 + 2 * t);
          p_ph ^= 1u;
          o_init = o_init || !skip;
          if (g + 1 == G) pass_turn();  // the last element has no QK: hand the turn over here
          release(vs);
        }
        if (g + 1 < G) {
          const int ks = acquire();
          if (main_blk && t == 0 && lane == 0) VFA_TRACE_EVENT(a, pos, 12);
          if (g < nchunks) {  // the softmax must have read m-init chunk g out of S_t
            mbar_wait(&ctl->s_free[t], g & 1);
            tc_fence_after();
            take_turn();
          }
          issue_qk(ks);
          if (main_blk && lane == 0) VFA_TRACE_EVENT(a, pos, 5 + 2 * t);
          pass_turn();
          release(ks);
          if (main_blk && t == 1 && lane == 0) VFA_TRACE_EVENT(a, pos, 20);
        }
      }
      if (elect_one()) mma_commit(&ctl->o_final[t]);
      __syncwarp();
    }
  } else {
    // ============================ softmax: 8 warps per query tile ============================
    // warps 8t .. 8t+7 serve tile t; warp w handles TMEM lanes 32*(w&3) .. +31 (rows) and half
    // hf = (w>>2)&1 of every S row (64 columns), so each sub-partition runs two warps per tile:
    // one warp's dependency stalls are covered by the other's MUFU / FMA work. Both halves see
    // the same running max (exchanged through shared memory on exact-update blocks, which are
    // the only ones that need it); each keeps its part of the normalizer.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(VFA_WS_REGS_SOFTMAX));
    VFA_WS_SETUP();
    const int t = warp >> 3;
    const int hf = (warp >> 2) & 1;
    const int r = tid & 127;
    const int h = unit.h0 + t;
    constexpr int CP = 64;  // S columns per thread
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tbase + C::s_off(t) + lane_off;
    const uint32_t tO = tbase + C::o_off(t) + hf * CP + lane_off;
    const int R = unit.qt * kBR + r;
    const float cs = a.c_scale;
    float m2 = -INFINITY, l = 0.f;
    int stab = sched_block(sched, 0);
    auto wait_s = [&](int g) {
      mbar_wait(&ctl->s_full[t], g & 1);
      tc_fence_after();
    };
    auto load_s = [&](float* v) {
      tmem_ld32(tS + hf * CP, v);
      tmem_ld32(tS + hf * CP + 32, v + 32);
      tmem_wait_ld();
      reg_fence32(v);
      reg_fence32(v + 32);
    };
    // row max over both halves (named barrier 1 + t over the tile's 256 threads); single-buffered:
    // a half rewrites its slot only after S of a later block, i.e. after the MMA consumed both
    // halves' P of this block, which they hand over after reading the exchanged value
    auto row_max = [&](float mine) -> float {
      ctl->xmax[t][hf][r] = mine;
      named_bar_sync(1 + t, 256);
      return fmaxf(ctl->xmax[t][0][r], ctl->xmax[t][1][r]);
    };
    // ---- m-init: m0 = max_j scale * q . krepr_j over visible j <= tc1 (src/vfa.py:91-106)
    if (nchunks > 0) {
      float mx = -INFINITY;
      for (int ch = 0; ch < nchunks; ++ch) {
        wait_s(ch);
        float v[CP];
        load_s(v);
        const int valid = nrep - ch * BC - hf * CP;
#pragma unroll
        for (int e = 0; e < CP; ++e)
          if (e < valid) mx = fmaxf(mx, v[e]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->s_free[t]);
      }
      m2 = row_max(mx) * cs;
    }
    if ((MODE == kVFA || MODE == kVSA) && a.use_m_init && a.m0_tile != nullptr)
      m2 = a.m0_tile[(static_cast<size_t>(unit.b) * a.Hq + h) * a.Tr + unit.qt] * cs;

    int n_skipped = 0, n_skipped_special = 0;
    const float2 cs2 = make_float2(cs, cs);
    for (int pos = 0; pos < N; ++pos) {
      const int j = sched_block(sched, pos);
      const bool special = all_exact(MODE) || sched_is_special(sched, j);
      const bool mask = sched_needs_mask(unit.qt + 1, j, kBR, BC, a.causal != 0);
      if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 13 + t);
      wait_s(nchunks + pos);
      if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 2 * t);
      if (r == 0 && hf == 0 && t == 0 && pos == 0) VFA_TRACE_UNIT(a, 1);
      float v[CP];
      // VFA frozen blocks need no row statistic before the exponentials: load the first 32
      // columns, start the second load, and let chunk 0's P go out while it lands
      const bool split = MODE == kVFA && !special;
      if (split) {
        tmem_ld32(tS + hf * CP, v);
        tmem_wait_ld();
        reg_fence32(v);
        tmem_ld32(tS + hf * CP + 32, v + 32);
      } else {
        load_s(v);
      }
      if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 21 + 4 * t);
      const int lim = R - (j - 1) * BC - hf * CP;  // this half's columns > lim are masked
      if (mask) {  // entrywise causal mask (src/reference.py:93-96): exact zeros after exp2
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
        if (!split) {
#pragma unroll
          for (int e = 32; e < CP; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
        }
      }
      bool skipped = false;
      float f = 1.0f;
      bool rescale = false;
      if (MODE == kVSA && !special) {
        // VSA frozen block: only the skip test (src/sparse.py:296-304). A row is below the
        // threshold iff both halves' maxima are, so one AND over the tile decides without
        // exchanging maxima; the frozen max is not updated.
        const float pm2 = part_max<CP>(v) * cs;
        const bool below = (pm2 - fmaxf(m2, pm2) < a.log2_lambda) ||
                           (pm2 == -INFINITY && m2 == -INFINITY && a.log2_lambda != -INFINITY);
        skipped = named_bar_and(1 + t, 256, below);
        if (skipped) ++n_skipped;
      } else if (special) {
        // exact update: rowmax (src/vfa.py:202-208), threshold test for the skip variants
        const float mt2 = row_max(part_max<CP>(v)) * cs;
        const float m2n = fmaxf(m2, mt2);
        if (skips(MODE)) {
          const bool below = (mt2 - m2n < a.log2_lambda) ||
                             (mt2 == -INFINITY && m2n == -INFINITY && a.log2_lambda != -INFINITY);
          skipped = named_bar_and(1 + t, 256, below);
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
      }
      if (skips(MODE) && r == 0 && hf == 0) ctl->skip[t] = skipped ? 1u : 0u;
      if (a.skip_trace && r == 0 && hf == 0)
        a.skip_trace[((static_cast<size_t>(unit.b) * a.Hq + h) * a.Tr + unit.qt) * a.Tc + pos] = skipped ? 2 : 1;
      if (rescale) {
        // O_t is quiescent (S_t(pos) complete => PV_t(pos-1) complete): rescale this half of the
        // row before PV(pos) accumulates into it (src/core.py:91)
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
      }
#ifndef VFA_WS_DBG_FASTSM
#define VFA_WS_DBG_FASTSM 0  // timing experiment only (wrong results): no exponentials, P hand-off at once
#endif
      if (VFA_WS_DBG_FASTSM) {
        l += v[0] + v[CP - 1];
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          for (int c = 0; c < kNCH; ++c) mbar_arrive(&ctl->p_full[t][c]);
      } else if (!skipped) {
        const float nm = (m2 == -INFINITY ? 0.f : -m2);
#pragma unroll
        for (int c = 0; c < kNCH; ++c) {
          // chunk c > 0 starts after chunk c-1's hand-off: its bias goes through a volatile
          // shared-memory read issued after that hand-off, so the compiler cannot hoist its
          // exponentials above the earlier chunk's P store (which would delay the hand-off)
          float nmc = nm;
          if (c > 0) {
            float z;
            asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(z) : "r"(smem_u32(&ctl->zero)) : "memory");
            nmc = nm + z;
            if (split && c * kCW == 32) {  // the second 32-column load has landed by now
              tmem_wait_ld();
              reg_fence32(v + 32);
              if (mask) {
#pragma unroll
                for (int e = 32; e < CP; ++e) v[e] = (e > lim) ? -INFINITY : v[e];
              }
            }
          }
          const float2 nmu2 = make_float2(nmc, nmc);
          uint32_t u[kCW / 2];
#pragma unroll
          for (int e = 0; e < kCW; e += 2) {
            const float2 x = __ffma2_rn(make_float2(v[c * kCW + e], v[c * kCW + e + 1]), cs2, nmu2);
            float2 p;
            if (((VFA_WS_EMU_CHUNKS >> c) & 1) && ((e >> 1) & 7) >= 8 - VFA_WS_EMU) {
              // degree-4 polynomial (|rel err| < 3e-6): the degree-3 form's 8.6e-5 showed up as
              // ~4e-5 in LSE on rows dominated by one emulated element
              p = VFA_WS_POLY3 ? ex2_poly3(x) : ex2_poly2(x);
            } else {
              p.x = ex2_approx(x.x);
              p.y = ex2_approx(x.y);
            }
            v[c * kCW + e] = p.x;
            v[c * kCW + e + 1] = p.y;
            u[e >> 1] = pack_bf16x2(p.x, p.y);
          }
          // P of this half's chunk c (packed bf16, kCW/2 TMEM columns): PV K-steps
          // 4*hf + c*kCW/16 .. +kCW/16
          if constexpr (kCW == 32)
            tmem_st16(tS + hf * CP + c * (kCW / 2), u);
          else
            tmem_st8(tS + hf * CP + c * (kCW / 2), u);
          if (r == 0 && hf == 0 && c == 0) VFA_TRACE_EVENT(a, pos, 22 + 4 * t);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctl->p_full[t][c]);
          if (r == 0 && hf == 0) {
            if (c == 0) VFA_TRACE_EVENT(a, pos, 18 + t);
            if (c == kNCH - 1) VFA_TRACE_EVENT(a, pos, 2 * t + 1);
          }
        }
        // row sum after the hand-off (src/tensor.py:81-89), two packed accumulators
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int e = 0; e < CP; e += 2) acc[(e >> 1) & 1] = add_ftz2(acc[(e >> 1) & 1], make_float2(v[e], v[e + 1]));
        l = __fadd_rn(l, __fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)));
        if (r == 0 && hf == 0) VFA_TRACE_EVENT(a, pos, 23 + 4 * t);
      } else {
        if (rescale) tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          for (int c = 0; c < kNCH; ++c) mbar_arrive(&ctl->p_full[t][c]);
      }
    }
    if (r == 0 && hf == 0 && t == 1) VFA_TRACE_UNIT(a, 2);
    // ---- finalize (src/core.py:101-109): l = half 0 + half 1, O / l, LSE, status
    ctl->xl[t][hf][r] = l;
    named_bar_sync(1 + t, 256);
    const float lsum = __fadd_rn(ctl->xl[t][0][r], ctl->xl[t][1][r]);
    const size_t lrow = (static_cast<size_t>(unit.b) * a.Hq + h) * a.Lq + R;
    const unsigned srow = static_cast<unsigned>(lrow + a.row_base);
    if (hf == 0) {
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
    mbar_wait(&ctl->o_final[t], 0);
    tc_fence_after();
    const float inv = 1.0f / lsum;
    __nv_bfloat16* orow = a.o + unit.b * a.o_sb + h * a.o_sh + static_cast<long long>(R) * a.o_sr + hf * CP;
    bool finite = true;
#pragma unroll
    for (int c = 0; c < CP / 32; ++c) {
      float o[32];
      tmem_ld32(tO + c * 32, o);
      tmem_wait_ld();
      reg_fence32(o);
      uint32_t u[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float o0 = o[e] * inv, o1 = o[e + 1] * inv;
        finite = finite && isfinite(o0) && isfinite(o1);
        u[e >> 1] = pack_bf16x2(o0, o1);
      }
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
      dst[0] = make_uint4(u[0], u[1], u[2], u[3]);
      dst[1] = make_uint4(u[4], u[5], u[6], u[7]);
      dst[2] = make_uint4(u[8], u[9], u[10], u[11]);
      dst[3] = make_uint4(u[12], u[13], u[14], u[15]);
    }
    if (a.status) {
      // a row is non-finite if either half is: combine through shared memory, count it once
      ctl->xfin[t][hf][r] = finite ? 1 : 0;
      named_bar_sync(1 + t, 256);
      if (hf == 0 && !(ctl->xfin[t][0][r] && ctl->xfin[t][1][r])) {
        atomicAdd(&a.status[VFA_STATUS_NONFINITE_ROWS], 1u);
        atomicOr(&a.status[VFA_STATUS_FLAGS], 4u);
      }
    }
    if (a.stats && r == 0 && hf == 0) {
      const int n_exact = all_exact(MODE) ? N : sched.n_spec;
      atomicAdd(&a.stats[VFA_STAT_VISITED], static_cast<unsigned long long>(N));
      atomicAdd(&a.stats[VFA_STAT_SKIPPED], static_cast<unsigned long long>(n_skipped));
      atomicAdd(&a.stats[VFA_STAT_SPECIAL], static_cast<unsigned long long>(n_exact - n_skipped_special));
      atomicAdd(&a.stats[VFA_STAT_FROZEN],
                static_cast<unsigned long long>((N - n_exact) - (n_skipped - n_skipped_special)));
    }
  }
#undef VFA_WS_SETUP
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) VFA_TRACE_UNIT(a, 3);
  if (warp == C::kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(ctl->tmem_base);
  }
}

}  // namespace vfa
