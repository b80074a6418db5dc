// Per-query-tile key-block schedule, shared verbatim by the host C-ABI
// (vfa_schedule, used by the CPU tests) and every device role of the kernel.
//
// Reference semantics (1-based blocks):
//   visible_key_blocks / local_key_block   src/core.py:112-122
//   build_schedule (order + special set)   src/vfa.py:146-153
// generalised to n_sink sink blocks and the n_local blocks ending at `local`;
// (n_sink, n_local) = (1, 1) reproduces the reference exactly.
#pragma once

#ifdef __CUDACC__
#define VFA_HD __host__ __device__ __forceinline__
#else
#define VFA_HD inline
#endif

namespace vfa {

struct TileSchedule {
  int vmax;      // number of visible key blocks (1..vmax)
  int local;     // local (diagonal) key block
  int a;         // specials part 1: blocks [1, a]   (a may be 0)
  int b0, b1;    // specials part 2: blocks [b0, b1] (empty when b0 > b1)
  int n_spec;    // |special set|
  bool reorder;  // specials first, then the rest ascending
  bool all_special;  // FA baseline: every visited block takes the exact update
};

// i: 1-based query block; br/bc block sizes; t_c number of key blocks.
VFA_HD TileSchedule make_schedule(int i, int br, int bc, int t_c, bool causal, int n_sink, int n_local,
                                  bool reorder, bool all_special) {
  TileSchedule s;
  int last_aligned = (i * br - 1) / bc + 1;
  s.local = last_aligned < t_c ? last_aligned : t_c;
  s.vmax = causal ? s.local : t_c;
  s.all_special = all_special;
  if (all_special) {
    s.a = s.vmax;
    s.b0 = 1;
    s.b1 = 0;
    s.n_spec = s.vmax;
    s.reorder = false;
    return s;
  }
  s.reorder = reorder;
  s.a = n_sink < s.vmax ? n_sink : s.vmax;
  if (s.a < 0) s.a = 0;
  int lo = s.local - n_local + 1;
  s.b0 = lo > 1 ? lo : 1;
  s.b1 = s.local < s.vmax ? s.local : s.vmax;
  if (n_local <= 0) s.b1 = s.b0 - 1;
  if (s.b0 <= s.b1 && s.b0 <= s.a + 1) {  // the two intervals touch: merge
    if (s.b1 > s.a) s.a = s.b1;
    s.b0 = 1;
    s.b1 = 0;
  }
  s.n_spec = s.a + (s.b0 <= s.b1 ? s.b1 - s.b0 + 1 : 0);
  return s;
}

VFA_HD bool sched_is_special(const TileSchedule& s, int j) {
  return j <= s.a || (j >= s.b0 && j <= s.b1);
}

// Key block (1-based) visited at position pos in [0, vmax).
VFA_HD int sched_block(const TileSchedule& s, int pos) {
  if (!s.reorder) return pos + 1;
  if (pos < s.n_spec) {
    if (pos < s.a) return pos + 1;
    return s.b0 + (pos - s.a);
  }
  int k = pos - s.n_spec;  // k-th element of [1, vmax] minus the special set
  if (s.b0 > s.b1) return s.a + 1 + k;
  int gap = s.b0 - s.a - 1;  // blocks strictly between the two intervals
  if (k < gap) return s.a + 1 + k;
  return s.b1 + 1 + (k - gap);
}

// Does tile (query block i, key block j) need the entrywise causal mask?
VFA_HD bool sched_needs_mask(int i, int j, int br, int bc, bool causal) {
  return causal && (j * bc - 1 > (i - 1) * br);
}

}  // namespace vfa
