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
};

struct ReachDev {
  const u32* bits;  // word-major: bits[w * n + i] = word w of class i's descendants
  u32 words, n;
  const u32* cls_index;
  u32 n_alloc;
  int valid;
};

__device__ __forceinline__ bool reach_query(const ReachDev& r, u32 a, u32 b) {
  if (!r.valid) return false;
  u32 ia = a < r.n_alloc ? r.cls_index[a] : TSAT_NONE;
  u32 ib = b < r.n_alloc ? r.cls_index[b] : TSAT_NONE;
  if (ia == TSAT_NONE || ib == TSAT_NONE) return false;
  return (r.bits[(u64)(ib >> 5) * r.n + ia] >> (ib & 31)) & 1u;
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
