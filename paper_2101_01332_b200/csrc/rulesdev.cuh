// Device descriptors shared by the exploration kernels.
#pragma once
#include "engine.cuh"

struct RuleDev {
  int nsrc, nslots, same_canon, allow_self, efficient, max_req, max_kids;
  u32 nmatch[MAX_SRC];
  const u32* mcls[MAX_SRC];
  const u32* mbind[MAX_SRC];
  int nb[MAX_SRC];
  int bind_slot[MAX_SRC][MAX_VARS];
  int tgt_off[MAX_SRC], tgt_len[MAX_SRC];
  int leaf_off[MAX_SRC], leaf_len[MAX_SRC];
  const Instr* instr;
  const int* leaf;
  int vanilla;                     // filter_mode "vanilla": stop before the cycle gate
  unsigned long long vanilla_go;   // ... except at this position (apply it)
  u32* rej_log;                    // efficient-mode reject positions (on_reject), or null
  u32 rej_cap;
  unsigned long long deadline_ns;  // time limit on the device clock (%globaltimer), 0 = none
};

__device__ __forceinline__ unsigned long long dev_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Efficient-mode pre-filter: reaches(a, b) over the iteration-start snapshot
// (reference cycles.py:52-57, 151-169), dense class indices via cls_index.
// mode 0: the descendants bitset (word-major, bits[w * n + i] = word w of class
//         i's descendant set), while it fits the memory budget;
// mode 1: no closure: the Kahn peel levels of the same class graph
//         (level = height, TSAT_NONE = on or above a cycle) answer almost every
//         query -- a reaches b needs level(a) > level(b), and nothing peeled
//         reaches an unpeeled class -- and the survivors are decided by a search
//         from a pruned to classes above level(b).  Parallel callers search with
//         a small private budget and get REACH_UNKNOWN beyond it (the combo then
//         takes the exact path); the exact path (one thread) searches with the
//         epoch-stamped marks in ``visit``.
#define REACH_NO 0
#define REACH_YES 1
#define REACH_UNKNOWN 2
struct ReachDev {
  const u32* bits;
  u32 words, n;
  const u32* cls_index;
  u32 n_alloc;
  int valid;
  int mode;
  const u32* level;
  const u32* eoff;
  const u32* edst;
  u32* visit;   // [n] epoch marks (exact search)
  u32* stack;   // [n]
  u32* epoch;   // [1]
  int steps;    // private search budget (classes expanded) of parallel callers
};

__device__ __forceinline__ bool reach_prune(const ReachDev& r, u32 j, u32 lb) {
  u32 lj = r.level[j];
  return lb == TSAT_NONE ? lj != TSAT_NONE : (lj != TSAT_NONE && lj <= lb);
}

// bounded private search: REACH_UNKNOWN when it outgrows its budget
#define RQ_STACK 24
#define RQ_SEEN 48
static __device__ __noinline__ int reach_search_bounded(const ReachDev& r, u32 ia, u32 ib, u32 lb) {
  u32 stk[RQ_STACK], seen[RQ_SEEN];
  int sp = 0, ns = 0, steps = 0;
  stk[sp++] = ia;
  seen[ns++] = ia;
  while (sp) {
    u32 v = stk[--sp];
    if (++steps > r.steps) return REACH_UNKNOWN;
    for (u32 e = r.eoff[v], e1 = r.eoff[v + 1]; e < e1; e++) {
      u32 j = r.edst[e];
      if (j == ib) return REACH_YES;
      if (reach_prune(r, j, lb)) continue;
      bool dup = false;
      for (int q = 0; q < ns && !dup; q++) dup = seen[q] == j;
      if (dup) continue;
      if (ns == RQ_SEEN || sp == RQ_STACK) return REACH_UNKNOWN;
      seen[ns++] = j;
      stk[sp++] = j;
    }
  }
  return REACH_NO;
}

// exact search: one thread at a time (k_seq_rule)
static __device__ __noinline__ int reach_search_exact(const ReachDev& r, u32 ia, u32 ib, u32 lb) {
  u32 ep = ++*r.epoch;
  if (ep == 0) {  // marks wrapped: clear them
    for (u32 i = 0; i < r.n; i++) r.visit[i] = 0;
    ep = *r.epoch = 1;
  }
  u32 sp = 0;
  r.stack[sp++] = ia;
  r.visit[ia] = ep;
  while (sp) {
    u32 v = r.stack[--sp];
    for (u32 e = r.eoff[v], e1 = r.eoff[v + 1]; e < e1; e++) {
      u32 j = r.edst[e];
      if (j == ib) return REACH_YES;
      if (reach_prune(r, j, lb) || r.visit[j] == ep) continue;
      r.visit[j] = ep;
      r.stack[sp++] = j;
    }
  }
  return REACH_NO;
}

// reaches(a, b) for class ids a, b (already canonical): REACH_NO / REACH_YES,
// or REACH_UNKNOWN (mode 1, parallel callers only)
__device__ __forceinline__ int reach_query(const ReachDev& r, u32 a, u32 b, bool exact = false) {
  if (!r.valid) return REACH_NO;
  u32 ia = a < r.n_alloc ? r.cls_index[a] : TSAT_NONE;
  u32 ib = b < r.n_alloc ? r.cls_index[b] : TSAT_NONE;
  if (ia == TSAT_NONE || ib == TSAT_NONE) return REACH_NO;
  if (r.mode == 0) return (r.bits[(u64)(ib >> 5) * r.n + ia] >> (ib & 31)) & 1u ? REACH_YES : REACH_NO;
  u32 la = r.level[ia], lb = r.level[ib];
  if (lb == TSAT_NONE ? la != TSAT_NONE : (la != TSAT_NONE && la <= lb)) return REACH_NO;
  return exact ? reach_search_exact(r, ia, ib, lb) : reach_search_bounded(r, ia, ib, lb);
}

// decode product position -> per-source match indices (itertools.product order)
__device__ __forceinline__ void decode_pos(const RuleDev& R, unsigned long long p, u32* idx) {
  for (int i = R.nsrc - 1; i >= 0; i--) {
    idx[i] = (u32)(p % R.nmatch[i]);
    p /= R.nmatch[i];
  }
}

// eval_pattern of one target under env (reference rules.py:126-138).
// Variables are referenced in place (node-table analyses); only the results of
// the target's App nodes are materialised, in ``scratch`` (MAX_STACK entries).
// *outp points at the target's value (a node-table entry for a bare variable).
static __device__ int eval_target(const G& g, const Instr* ins, int len, const u32* env, Val* scratch,
                                  const Val*& outp) {
  const Val* st[MAX_STACK];
  int sp = 0, nr = 0;
  for (int k = 0; k < len; k++) {
    const Instr& in = ins[k];
    if (in.kind == I_VAR) {
      st[sp++] = &g.val[uf_find_ro(g.parent, env[in.arg])];
    } else {
      int na = in.arg;
      sp -= na;
      Val& r = scratch[nr++];
      int s = val_make(in.atom, ValRefs{st + sp}, na, r, g.atoms, g.tt);
      if (s != AS_OK) return s;
      st[sp++] = &r;
    }
  }
  outp = st[0];
  return AS_OK;
}
