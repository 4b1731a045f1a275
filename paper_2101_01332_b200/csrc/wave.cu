// Parallel wave apply: the bulk path of run_rule/_apply_combo
// (reference: pkg/src/tensorsat/explorer.py:146-163, 227-262).
//
// A wave takes the remaining product positions of one rule and evaluates all
// of them against the e-graph state at wave start:
//   1. join      compatible combos (multi-pattern: hash join on the shared
//                variables' canonical classes, emitted in itertools.product
//                order; single-pattern: every match)
//   2. gates     combined subst, shape check (target programs on the Value
//                analysis) and the efficient cycle pre-filter, fused
//   3. resolve   target terms become node requests, resolved level by level:
//                a key with only existing children is looked up in the
//                hashcons; otherwise it goes to a wave-local key table where
//                the first request in sequential order (min global position)
//                is the one that allocates -- exactly the hash-cons hits the
//                sequential loop would see.
//   4. hazards   conditions under which later combos would observe this
//                combo's effects differently from the wave-start state:
//                a union of two pre-existing classes (changes find()), a
//                union that grows a class's split origins, a request that
//                re-uses a node created as an earlier target root (its class
//                is the merged class), analysis errors.
//   5. commit    all combos before the first hazard (and before the node-limit
//                cutoff) are committed in bulk: ids by prefix sum in
//                sequential order, node records, fresh-root unions, hashcons
//                inserts.  The hazard combo itself runs on the exact
//                sequential path (k_seq_rule) and the next wave starts after it.
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "rulesdev.cuh"

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

#define FRESH 0x80000000u
#define MAX_REQ 32
#define WAVE_MAX_CAND (1u << 22)

RuleDev make_rule_dev(Engine& e, int ri, int filter_mode, int allow_self);
ReachDev make_reach_dev(Engine& e);

struct WaveState {
  u32 nacc, ncommit_cand, ncommit_acc, nwin, nk, base, kbase, stop, hazard, why, any_applied, sa_hit;
  unsigned long long p_end;
};

struct ReqT {        // request template (one App instruction of a target)
  u32 atom;
  int32_t nargs;
  int32_t kid[8];    // >= 0: request index within the combo; < 0: var slot -(s+1)
  int32_t depth;
  int32_t tgt;
  int32_t is_root;
};

struct WaveRule {
  int R;                 // requests per combo
  int ntgt;
  int root_req[MAX_SRC]; // request index of each target's root, -1 for a bare variable target
  int root_var[MAX_SRC]; // slot of a bare-variable target
  int nshared;
  int shpos[2][8];       // binding positions of the shared slots in sources 0 / 1
  const ReqT* tmpl;
};

struct WaveTab {  // wave-local key table; every tag carries the wave's epoch
  unsigned long long* minpos;  // (~epoch << 32) | min request position
  u32* wid;       // assigned node id of the winner
  u32* wroot;     // == epoch: winner is a target root
  Val* val;
  u32 mask;
  u32* wold;      // matched (old) class of a root winner's target
  u32 epoch;
  unsigned long long* tag;  // (epoch << 32) | key-hash high word per slot
  u32* own;                 // request that claimed the slot
};

// ---------------------------------------------------------------- join

__device__ __forceinline__ u64 shared_hash(const G& g, const u32* bind, int nb, u64 row, const int* pos, int ns) {
  u64 h = 0x9ae16a3b2f90404fULL;
  for (int s = 0; s < ns; s++) h = hash_mix(h, uf_find_ro(g.parent, bind[row * nb + pos[s]]));
  return h;
}

__global__ void k_hash_rows(G g, const u32* bind, int nb, u32 n, WaveRule W, int side, u64* out, u32* idx) {
  GRID_STRIDE(i, n) {
    out[i] = shared_hash(g, bind, nb, i, W.shpos[side], W.nshared);
    idx[i] = (u32)i;
  }
}

// Compatible positions for rows i >= i0, one warp per row: lanes test 32
// candidates of the equal-hash range at a time, a ballot keeps the emitted
// positions in j order (itertools.product order).  count pass: cnt[row];
// emit pass: out[off[row] + k] (capped at cap).
__global__ void k_join(G g, RuleDev R, WaveRule W, const u64* hA, u32 i0, const u64* hBs, const u32* iBs,
                       unsigned long long p_start, int skip_self, const u32* off, u32* cnt,
                       unsigned long long* out, u32 cap) {
  u32 lane = threadIdx.x & 31;
  u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
  u32 nB = R.nmatch[1];
  for (u64 t = warp; t < (u64)(R.nmatch[0] - i0); t += nw) {
    u32 i = i0 + (u32)t;
    u64 h = hA[t];
    u32 lo = 0, hi = nB;
    while (lo < hi) {
      u32 mid = (lo + hi) >> 1;
      if (hBs[mid] < h) lo = mid + 1;
      else hi = mid;
    }
    u32 ahead[8];
    for (int s = 0; s < W.nshared; s++)
      ahead[s] = uf_find_ro(g.parent, R.mbind[0][(u64)i * R.nb[0] + W.shpos[0][s]]);
    u32 c = 0;
    u32 o = off ? off[t] : 0;
    for (u32 k0 = lo; k0 < nB; k0 += 32) {
      u32 k = k0 + lane;
      bool inr = k < nB && hBs[k] == h;
      bool ok = false;
      if (inr) {
        u32 j = iBs[k];
        unsigned long long p = (unsigned long long)i * nB + j;
        ok = p >= p_start && !(skip_self && i == j);
        for (int s = 0; s < W.nshared && ok; s++)
          ok = ahead[s] == uf_find_ro(g.parent, R.mbind[1][(u64)j * R.nb[1] + W.shpos[1][s]]);
      }
      u32 m = __ballot_sync(0xffffffffu, ok);
      if (ok && out) {
        u32 q = o + c + __popc(m & ((1u << lane) - 1));
        if (q < cap) out[q] = (unsigned long long)i * nB + iBs[k];
      }
      c += __popc(m);
      if (!__any_sync(0xffffffffu, inr)) break;
    }
    if (cnt && lane == 0) cnt[t] = c;
  }
}

// ---------------------------------------------------------------- phases
//
// Every wave phase is a __device__ function over an index range striped by
// (tid, nth).  The grid path wraps each one in its own kernel
// (tid = global thread, nth = grid size); the single-CTA path (k_wave_cta)
// runs them back to back inside one block with __syncthreads() between
// phases, so a small wave costs one block's worth of barriers instead of
// ~20 kernel launches.  Per-wave tables are epoch-tagged (no clearing).

#define TID_LOOP(i, n) for (u64 i = tid; i < (u64)(n); i += nth)

// union-find read that is safe inside a kernel that also writes parent[]
// (no read-only cache path)
__device__ __forceinline__ u32 uf_find_rw(const u32* parent, u32 x) {
  u32 p;
  while ((p = parent[x]) != x) x = p;
  return x;
}

__device__ __forceinline__ unsigned long long mp_tag(u32 epoch, u64 gpos) {
  return ((unsigned long long)(~epoch) << 32) | gpos;
}
__device__ __forceinline__ unsigned long long fw_tag(u32 epoch, u32 c) {
  return ((unsigned long long)(~epoch) << 32) | c;
}
__device__ __forceinline__ bool is_winner(const WaveTab& T, u32 s, u64 gpos) {
  return T.minpos[s] == mp_tag(T.epoch, gpos);
}
__device__ __forceinline__ bool is_wroot(const WaveTab& T, u32 s) { return T.wroot[s] == T.epoch; }

// status: 0 accept, 1 shape fail, 2 cycle reject; hazard flag for gate errors
__device__ __forceinline__ void d_gates(u64 tid, u64 nth, const G& g, const RuleDev& R, const ReachDev& RD,
                                        const unsigned long long* pos, u32 n, unsigned long long p_base, u8* status,
                                        u32* env_out, u32* old_out, u8* hazard) {
  TID_LOOP(c, n) {
    unsigned long long p = pos ? pos[c] : p_base + c;
    u32 idx[MAX_SRC];
    decode_pos(R, p, idx);
    u32 env[MAX_VARS];
    for (int v = 0; v < R.nslots; v++) env[v] = TSAT_NONE;
    for (int i = 0; i < R.nsrc; i++)
      for (int j = 0; j < R.nb[i]; j++)
        env[R.bind_slot[i][j]] = uf_find_rw(g.parent, R.mbind[i][(u64)idx[i] * R.nb[i] + j]);
    u32 olds[MAX_SRC];
    for (int t = 0; t < R.nsrc; t++) olds[t] = uf_find_rw(g.parent, R.mcls[t][idx[t]]);
    u8 st = 0, hz = 0;
    if (g.analysis) {
      Val scratch[MAX_STACK];
      for (int t = 0; t < R.nsrc && st == 0; t++) {
        const Val* out = nullptr;
        int s = eval_target(g, R.instr + R.tgt_off[t], R.tgt_len[t], env, scratch, out);
        if (s == AS_ORIGIN_OVERFLOW || s == AS_TREE_FULL) {
          hz = 1;
          break;
        }
        if (s != AS_OK || !val_same_data(*out, g.val[olds[t]])) st = 1;
      }
    }
    if (st == 0 && !hz && R.efficient) {
      int hit = REACH_NO;
      for (int t = 0; t < R.nsrc && hit != REACH_YES; t++)
        for (int l = 0; l < R.leaf_len[t]; l++) {
          u32 leaf = env[R.leaf[R.leaf_off[t] + l]];
          int q = leaf == olds[t] ? REACH_YES : reach_query(RD, leaf, olds[t]);
          if (q == REACH_YES) {
            hit = REACH_YES;
            break;
          }
          if (q == REACH_UNKNOWN) hit = REACH_UNKNOWN;  // a later leaf may still say yes
        }
      if (hit == REACH_YES) st = 2;
      else if (hit == REACH_UNKNOWN) hz = 1;  // undecided within the budget: exact path
    }
    status[c] = st;
    hazard[c] = hz;
    for (int v = 0; v < R.nslots; v++) env_out[(u64)c * MAX_VARS + v] = env[v];
    for (int t = 0; t < R.nsrc; t++) old_out[(u64)c * MAX_SRC + t] = olds[t];
  }
}

// ---------------------------------------------------------------- resolution

__device__ __forceinline__ u64 wkey_hash(u32 op, int n, const u32* k) {
  u64 h = hash_mix(0x7a3f1e2dULL ^ ((u64)n << 40), op);
  for (int i = 0; i < n; i++) h = hash_mix(h, k[i]);
  return h;
}

// A request level resolves in two passes instead of one fenced key insert:
//   claim   — a request whose key is not in the hashcons claims a slot by a
//             CAS of (epoch, key hash) (equal hashes share the slot; the CAS
//             winner records itself as the slot's owner);
//   verify  — after the barrier every sharer compares its key with the
//             owner's (recomputed from the owner's request), takes part in the
//             min-position election, and the owner stores the slot's analysis.
// No key is stored and no fence is needed: the barrier between the passes
// (kernel boundary on grid waves, __syncthreads in k_wave_cta) orders them.  A 64-bit hash collision between different keys marks the combo
// for the exact path.
__device__ __forceinline__ int req_key(const WaveRule& W, const u32* ident, const u32* env, u32 a, u32 c, int r,
                                       u32* kids) {
  const ReqT& q = W.tmpl[r];
  for (int j = 0; j < q.nargs; j++) {
    int k = q.kid[j];
    kids[j] = k >= 0 ? ident[(u64)a * W.R + k] : env[(u64)c * MAX_VARS + (-k - 1)];
  }
  return q.nargs;
}

__device__ __forceinline__ void d_resolve_claim(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                                const u32* acc, u32 nacc, const int* lvl_req, int nlvl,
                                                const u32* env, u32* ident, const u8* hazard) {
  TID_LOOP(t, (u64)nacc * nlvl) {
    u32 a = (u32)(t / nlvl);
    int r = lvl_req[t % nlvl];
    u32 c = acc[a];
    u64 gpos = (u64)a * W.R + r;
    if (hazard[c]) {
      ident[gpos] = TSAT_NONE;
      continue;
    }
    const ReqT& q = W.tmpl[r];
    u32 kids[8];
    int n = req_key(W, ident, env, a, c, r, kids);
    bool real = true;
    for (int j = 0; j < n; j++) real &= !(kids[j] & FRESH);
    if (real) {
      u32 hit = hc_lookup(g, q.atom, n, kids);
      if (hit != TSAT_NONE) {
        ident[gpos] = uf_find_rw(g.parent, hit);
        continue;
      }
    }
    u64 h = wkey_hash(q.atom, n, kids);
    unsigned long long mine = ((unsigned long long)T.epoch << 32) | (u32)(h >> 32);
    u32 slot = (u32)h & T.mask;
    while (true) {
      unsigned long long cur = T.tag[slot];
      if ((u32)(cur >> 32) != T.epoch) {
        unsigned long long prev = atomicCAS(&T.tag[slot], cur, mine);
        if (prev == cur) {
          T.own[slot] = (u32)gpos;
          break;
        }
        cur = prev;
      }
      if (cur == mine) break;
      slot = (slot + 1) & T.mask;
    }
    ident[gpos] = FRESH | slot;
  }
}

__device__ __forceinline__ void d_resolve_verify(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                                 const u32* acc, u32 nacc, const int* lvl_req, int nlvl,
                                                 const u32* env, const u32* ident, u8* hazard) {
  TID_LOOP(t, (u64)nacc * nlvl) {
    u32 a = (u32)(t / nlvl);
    int r = lvl_req[t % nlvl];
    u64 gpos = (u64)a * W.R + r;
    u32 id = ident[gpos];
    if (id == TSAT_NONE || !(id & FRESH)) continue;
    u32 s = id & ~FRESH, c = acc[a];
    const ReqT& q = W.tmpl[r];
    u32 kids[8];
    int n = req_key(W, ident, env, a, c, r, kids);
    u32 own = T.own[s];
    if (own != (u32)gpos) {
      u32 ao = own / (u32)W.R;
      int ro = (int)(own % (u32)W.R);
      const ReqT& qo = W.tmpl[ro];
      bool eq = qo.atom == q.atom && qo.nargs == q.nargs;
      if (eq) {
        u32 ko[8];
        req_key(W, ident, env, ao, acc[ao], ro, ko);
        for (int j = 0; j < n && eq; j++) eq = ko[j] == kids[j];
      }
      if (!eq) {
        hazard[c] = 2;  // hash collision: the exact path decides
        continue;
      }
    }
    atomicMin(&T.minpos[s], mp_tag(T.epoch, gpos));
    if (g.analysis) {
      const Val* kv[8];
      for (int j = 0; j < n; j++) kv[j] = (kids[j] & FRESH) ? &T.val[kids[j] & ~FRESH] : &g.val[kids[j]];
      Val v;
      int st = val_make(q.atom, ValRefs{kv}, n, v, g.atoms, g.tt);
      if (st != AS_OK) hazard[c] = 2;
      else if (own == (u32)gpos) val_copy(T.val[s], v);
    }
  }
}

__device__ __forceinline__ void d_mark_roots(u64 tid, u64 nth, const WaveRule& W, const WaveTab& T, const u32* acc,
                                             u32 nacc, const u32* ident, const u8* hazard, const u32* olds) {
  TID_LOOP(a, nacc) {
    if (hazard[acc[a]]) continue;
    for (int t = 0; t < W.ntgt; t++) {
      int r = W.root_req[t];
      if (r < 0) continue;
      u32 id = ident[(u64)a * W.R + r];
      if (!(id & FRESH)) continue;
      u32 s = id & ~FRESH;
      if (is_winner(T, s, (u64)a * W.R + r)) {
        T.wroot[s] = T.epoch;
        T.wold[s] = olds[(u64)acc[a] * MAX_SRC + t];
      }
    }
  }
}

// Union kinds per (combo, target): 0 none, 1 fresh root winner -> matched class,
// 2 union(matched, existing class X), 3 union(matched, fresh non-root node F).
#define UK_NONE 0
#define UK_FRESH_ROOT 1
#define UK_CLASS 2
#define UK_FRESH_NODE 3

// per accepted combo: allocations, union plan, type-a hazards (combo's own
// evaluation cannot be trusted) and its write set.
__device__ __forceinline__ void d_cand_check(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                             const u32* acc, u32 nacc, u32 ncand, const u32* ident, const u32* env,
                                             const u32* olds, int multi, u8* hazard, u32* alloc, u8* ukind,
                                             u32* uother, u8* grow, u8* stop_after, u32* akid) {
  TID_LOOP(a0, ncand) {
    u32 a = (u32)a0;
    if (a >= nacc) {
      alloc[a] = 0;
      akid[a] = 0;
      stop_after[a] = 0;
      continue;
    }
    u32 c = acc[a];
    u32 na = 0, nk = 0;
    bool hz = hazard[c] != 0, sa = false;
    u8 why = hazard[c];
    for (int t = 0; t < MAX_SRC; t++) {
      ukind[(u64)a * MAX_SRC + t] = UK_NONE;
      grow[(u64)a * MAX_SRC + t] = 0;
    }
    if (!hz) {
      for (int r = 0; r < W.R && !hz; r++) {
        u32 id = ident[(u64)a * W.R + r];
        if (!(id & FRESH)) continue;
        u32 s = id & ~FRESH;
        bool win = is_winner(T, s, (u64)a * W.R + r);
        if (win) {
          na++;
          nk += (u32)W.tmpl[r].nargs;
        } else if (is_wroot(T, s) && !W.tmpl[r].is_root) {
          hz = true;  // inner reuse of a merged root
          why = 3;
        }
      }
      for (int t = 0; t < W.ntgt && !hz; t++) {
        u32 old = olds[(u64)c * MAX_SRC + t];
        int r = W.root_req[t];
        u8 kind = UK_NONE;
        u32 other = 0;
        const Val* nv = nullptr;
        if (r < 0) {
          u32 x = env[(u64)c * MAX_VARS + W.root_var[t]];
          if (x != old) {
            kind = UK_CLASS;
            other = x;
            nv = &g.val[x];
          }
        } else {
          u32 id = ident[(u64)a * W.R + r];
          if (!(id & FRESH)) {
            if (id != old) {
              kind = UK_CLASS;
              other = id;
              nv = &g.val[id];
            }
          } else {
            u32 s = id & ~FRESH;
            bool win = is_winner(T, s, (u64)a * W.R + r);
            if (win) {
              kind = UK_FRESH_ROOT;
              other = id;
              nv = &T.val[s];
            } else if (is_wroot(T, s)) {
              u32 x = T.wold[s];  // the earlier root's node now lives in its matched class
              if (x != old) {
                kind = UK_CLASS;
                other = x;
                nv = &g.val[x];
              }
            } else {
              kind = UK_FRESH_NODE;
              other = id;
              nv = &T.val[s];
            }
          }
        }
        if (kind != UK_NONE && g.analysis) {
          const Val& ov = g.val[old];
          if (!val_same_data(ov, *nv)) {
            hz = true;  // AnalysisMergeError: exact path raises it
            why = 5;
          } else if (kind == UK_CLASS) {
            // the kept (smaller) root's analysis changes iff the dropped one adds origins
            bool keep_is_old = old < other;
            if (keep_is_old ? val_merge_grows(ov, *nv) : val_merge_grows(*nv, ov)) grow[(u64)a * MAX_SRC + t] = 1;
          } else if (val_merge_grows(ov, *nv)) {
            grow[(u64)a * MAX_SRC + t] = 1;
          }
        }
        // a union or analysis change in a non-final target would feed the
        // combo's own later targets: let the exact path handle it
        if (t < W.ntgt - 1 && (kind == UK_CLASS || kind == UK_FRESH_NODE || grow[(u64)a * MAX_SRC + t])) {
          hz = true;
          why = 4;
        }
        if (multi && (kind == UK_CLASS || kind == UK_FRESH_NODE)) sa = true;
        ukind[(u64)a * MAX_SRC + t] = kind;
        uother[(u64)a * MAX_SRC + t] = other;
      }
    }
    hazard[c] = hz ? (why ? why : 1) : 0;
    stop_after[a] = sa ? 1 : 0;
    alloc[a] = hz ? 0 : na;
    akid[a] = hz ? 0 : nk;
  }
}

// first writer of every identity (class id or FRESH slot) in the wave
__device__ __forceinline__ void d_first_writer(u64 tid, u64 nth, const WaveRule& W, u32 epoch, const u32* acc,
                                               u32 nacc, const u8* hazard, const u32* olds, const u8* ukind,
                                               const u32* uother, const u8* grow, unsigned long long* fw_cls,
                                               unsigned long long* fw_fresh) {
  TID_LOOP(a, nacc) {
    u32 c = acc[a];
    if (hazard[c]) continue;
    unsigned long long tag = fw_tag(epoch, c);
    for (int t = 0; t < W.ntgt; t++) {
      u8 k = ukind[(u64)a * MAX_SRC + t];
      u32 old = olds[(u64)c * MAX_SRC + t], x = uother[(u64)a * MAX_SRC + t];
      bool gr = grow[(u64)a * MAX_SRC + t] != 0;
      if (k == UK_CLASS) {
        // only the dropped root changes identity; the kept root changes only
        // when its analysis grows
        u32 keep = old < x ? old : x, drop = old < x ? x : old;
        atomicMin(&fw_cls[drop], tag);
        if (gr) atomicMin(&fw_cls[keep], tag);
      } else if (k == UK_FRESH_NODE) {
        atomicMin(&fw_fresh[x & ~FRESH], tag);
        if (gr) atomicMin(&fw_cls[old], tag);
      } else if (k == UK_FRESH_ROOT && gr) {
        atomicMin(&fw_cls[old], tag);
      }
    }
  }
}

__device__ __forceinline__ bool read_dirty(u32 id, u32 c, u32 epoch, const unsigned long long* fw_cls,
                                           const unsigned long long* fw_fresh) {
  unsigned long long v = (id & FRESH) ? fw_fresh[id & ~FRESH] : fw_cls[id];
  return (u32)(v >> 32) == ~epoch && (u32)v < c;
}

#ifdef WAVE_DBG
__device__ unsigned long long g_wdbg_first = ~0ull;
__device__ unsigned long long g_wdbg_cnt[32];
#define WDBG_CAT(k) \
  if (bad && !dbg_cat) dbg_cat = (k)
#define WDBG_SET(k) dbg_cat = (k)
#else
#define WDBG_CAT(k)
#define WDBG_SET(k)
#endif

// class of a wave-start root at candidate c's turn: follow the drops of the
// earlier first writers (each identity has at most one writer before the
// first conflict, so the chain is exact up to there).  *grown: the root's
// analysis was extended earlier in the wave.  TSAT_NONE if the chain is long.
__device__ __forceinline__ u32 soft_find(u32 id, u32 c, u32 ep, const WaveRule& W, const unsigned long long* fw_cls,
                                         const u32* accpre, const u32* olds, const u8* ukind, const u32* uother,
                                         bool* grown) {
  *grown = false;
  for (int hop = 0; hop < 32; hop++) {
    unsigned long long v = fw_cls[id];
    if ((u32)(v >> 32) != ~ep || (u32)v >= c) return id;
    u32 w = (u32)v, a = accpre[w], nxt = id;
    for (int t = 0; t < W.ntgt; t++) {
      if (ukind[(u64)a * MAX_SRC + t] != UK_CLASS) continue;
      u32 o = olds[(u64)w * MAX_SRC + t], x = uother[(u64)a * MAX_SRC + t];
      if ((o > x ? o : x) == id) nxt = o < x ? o : x;
    }
    if (nxt == id) {
      *grown = true;
      return id;
    }
    id = nxt;
  }
  return TSAT_NONE;
}

// REACH_YES / REACH_NO, or REACH_UNKNOWN when a bounded search gave up
__device__ __forceinline__ int cycle_hit(const RuleDev& R, const ReachDev& RD, const u32* env, const u32* outs) {
  int res = REACH_NO;
  for (int t = 0; t < R.nsrc; t++)
    for (int l = 0; l < R.leaf_len[t]; l++) {
      u32 leaf = env[R.leaf[R.leaf_off[t] + l]];
      int q = leaf == outs[t] ? REACH_YES : reach_query(RD, leaf, outs[t]);
      if (q == REACH_YES) return REACH_YES;
      if (q == REACH_UNKNOWN) res = REACH_UNKNOWN;
    }
  return res;
}

// candidate validity against earlier writes in the wave (all candidates:
// rejected ones read through their gates, accepted ones through requests).
//
// Reads of the classes a target is unioned with (the matched class and, for a
// class merge, the class the target root resolved to) are soft: sequentially
// the combo unions find(old) with find(other), so an earlier merge changes
// only which roots meet, not what the combo builds.  A combo whose soft reads
// are dirty is still exact here when it writes nothing:
//   * a shape-rejected combo compared only the class's data (merges keep it);
//   * a no-op target (its root resolved to the matched class) stays a no-op;
//   * a fresh target root without analysis growth just joins the class
//     (its parent may point at the old root: find() is the same);
//   * the efficient cycle pre-filter is re-run with the current roots
//     (reference cycles.py:163-168) and must give the gates' answer.
// A combo that does write (class merge, fresh-node union, growth) is a soft
// writer: with first_soft the caller resolves it (d_resolve_soft) and
// re-runs the conflict pass; without, it ends the prefix like any conflict.
// Reads of everything else (substitution classes, inner request classes)
// are hard: an earlier write ends the prefix.
__device__ __forceinline__ void d_validity(u64 tid, u64 nth, const WaveRule& W, const WaveTab& T, u32 ep,
                                           const RuleDev& R, const ReachDev& RD, u32 ncand, const u8* hazard,
                                           const u32* env, const u32* olds, const u32* accpre, const u8* status,
                                           const u32* ident, const u8* ukind, const u8* grow, const u32* uother,
                                           const unsigned long long* fw_cls, const unsigned long long* fw_fresh,
                                           u32* first_bad, u32* first_soft) {
  TID_LOOP(c0, ncand) {
    u32 c = (u32)c0;
    u8 st = status[c];
    bool bad = hazard[c] != 0 || st > 2;
#ifdef WAVE_DBG
    int dbg_cat = 0;
#endif
    WDBG_CAT(1);
    for (int v = 0; v < R.nslots && !bad; v++) bad = read_dirty(env[(u64)c * MAX_VARS + v], c, ep, fw_cls, fw_fresh);
    WDBG_CAT(2);
    u32 a = st == 0 ? accpre[c] : 0u;
    bool writer = false, recheck = false;
    for (int t = 0; t < R.nsrc && !bad; t++) {
      u32 o = olds[(u64)c * MAX_SRC + t];
      u8 k = st == 0 ? ukind[(u64)a * MAX_SRC + t] : (u8)UK_NONE;
      bool dirty = read_dirty(o, c, ep, fw_cls, fw_fresh);
      if (k == UK_CLASS) dirty |= read_dirty(uother[(u64)a * MAX_SRC + t], c, ep, fw_cls, fw_fresh);
      if (!dirty) continue;
      if (st == 0 && (k == UK_CLASS || k == UK_FRESH_NODE || (k == UK_FRESH_ROOT && grow[(u64)a * MAX_SRC + t])))
        writer = true;
      else if (st != 1)
        recheck = true;
    }
    if (!bad && !writer && recheck && R.efficient) {  // cycle pre-filter at c's turn
      u32 outs[MAX_SRC];
      for (int t = 0; t < R.nsrc && !bad; t++) {
        bool gr;
        outs[t] = soft_find(olds[(u64)c * MAX_SRC + t], c, ep, W, fw_cls, accpre, olds, ukind, uother, &gr);
        bad = outs[t] == TSAT_NONE;
      }
      if (!bad) {
        int ch = cycle_hit(R, RD, env + (u64)c * MAX_VARS, outs);
        bad = ch == REACH_UNKNOWN || (ch == REACH_YES) != (st == 2);
      }
      WDBG_CAT(5);
    }
    if (!bad && st == 0) {
      for (int r = 0; r < W.R && !bad; r++) {
        const ReqT& q = W.tmpl[r];
        // a target root's class is a union side (above) unless it is a fresh
        // node another combo may have merged
        if (q.is_root && ukind[(u64)a * MAX_SRC + q.tgt] != UK_FRESH_NODE) continue;
        u32 id = ident[(u64)a * W.R + r];
        bad = read_dirty(id, c, ep, fw_cls, fw_fresh);
        WDBG_CAT(q.is_root ? 7 : 6);
        // a reused target root resolves to the class it was merged into
        if (!bad && (id & FRESH) && is_wroot(T, id & ~FRESH))
          bad = read_dirty(T.wold[id & ~FRESH], c, ep, fw_cls, fw_fresh);
        WDBG_CAT(8);
      }
    }
    if (!bad && writer) {
      if (first_soft) atomicMin(first_soft, c);
      else bad = true;
      WDBG_CAT(9);
    }
    if (bad) atomicMin(first_bad, c);
#ifdef WAVE_DBG
    if (bad) atomicMin(&g_wdbg_first, ((unsigned long long)c << 8) | (dbg_cat ? dbg_cat : 31));
#endif
  }
}

// Resolve soft writer c (one thread; every earlier writer is exact): its
// union sides become the roots at its turn, its union kind / growth are
// recomputed from them (a merge of two classes already joined is a no-op),
// and the cycle pre-filter is re-checked.  false: not resolvable here (an
// analysis that changed earlier in the wave, a merged fresh node, a change
// in a non-final target) -- the prefix ends at c.
__device__ bool d_resolve_soft(const G& g, const WaveRule& W, const WaveTab& T, u32 ep, const RuleDev& R,
                               const ReachDev& RD, u32 c, const u32* env, u32* olds, const u32* accpre, u8* ukind,
                               u32* uother, u8* grow, const unsigned long long* fw_cls,
                               const unsigned long long* fw_fresh) {
  u32 a = accpre[c];
  u32 outs[MAX_SRC];
  for (int t = 0; t < R.nsrc; t++) {
    u64 ia = (u64)a * MAX_SRC + t, ic = (u64)c * MAX_SRC + t;
    bool gro, grx;
    u32 ro = soft_find(olds[ic], c, ep, W, fw_cls, accpre, olds, ukind, uother, &gro);
    if (ro == TSAT_NONE) return false;
    outs[t] = ro;
    u8 k = ukind[ia];
    if (k == UK_NONE) continue;
    if (gro) return false;
    u32 x = uother[ia];
    u8 nk = k, ng = 0;
    if (k == UK_CLASS) {
      u32 rx = soft_find(x, c, ep, W, fw_cls, accpre, olds, ukind, uother, &grx);
      if (rx == TSAT_NONE || grx) return false;
      if (rx == ro) {
        nk = UK_NONE;
      } else {
        u32 keep = ro < rx ? ro : rx, drop = ro < rx ? rx : ro;
        ng = g.analysis && val_merge_grows(g.val[keep], g.val[drop]);
      }
      x = rx;
    } else {
      if (k == UK_FRESH_NODE && read_dirty(x, c, ep, fw_cls, fw_fresh)) return false;
      ng = g.analysis && val_merge_grows(g.val[ro], T.val[x & ~FRESH]);
    }
    if (t < W.ntgt - 1 && (nk == UK_CLASS || nk == UK_FRESH_NODE || ng)) return false;
    olds[ic] = ro;
    ukind[ia] = nk;
    uother[ia] = x;
    grow[ia] = ng;
  }
  if (R.efficient && cycle_hit(R, RD, env + (u64)c * MAX_VARS, outs) != REACH_NO) return false;
  return true;
}

// first hazard (candidate index) and node-limit cutoff (accepted index)
__device__ __forceinline__ void d_find_stops(u64 tid, u64 nth, const u32* acc, u32 nacc, const u8* stop_after,
                                             const u32* apre, const u32* alloc, i64 live0, i64 n_max,
                                             u32* out /* [stop_after cand, cutoff cand] */) {
  TID_LOOP(a, nacc) {
    if (stop_after[a]) atomicMin(&out[0], acc[a]);
    if (live0 + (i64)apre[a] + (i64)alloc[a] >= n_max && alloc[a] > 0) atomicMin(&out[1], acc[a]);
  }
}

// unions of committed combos (disjoint by construction of the validity check)
__device__ __forceinline__ void d_commit_unions(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                                const u32* acc, u32 ncommit_acc, const u32* olds, const u8* ukind,
                                                const u32* uother, const u8* grow) {
  TID_LOOP(a, ncommit_acc) {
    u32 c = acc[a];
    for (int t = 0; t < W.ntgt; t++) {
      u8 k = ukind[(u64)a * MAX_SRC + t];
      if (k == UK_NONE) continue;
      u32 old = olds[(u64)c * MAX_SRC + t], x = uother[(u64)a * MAX_SRC + t];
      bool gr = grow[(u64)a * MAX_SRC + t] != 0;
      if (k == UK_FRESH_ROOT) {
        if (gr && g.analysis) val_merge_into(g.val[old], T.val[x & ~FRESH]);
        continue;  // parent link written by k_write_nodes
      }
      if (k == UK_FRESH_NODE) {
        u32 f = T.wid[x & ~FRESH];
        if (gr && g.analysis) val_merge_into(g.val[old], T.val[x & ~FRESH]);
        g.parent[f] = old;
        continue;
      }
      u32 keep = old < x ? old : x, drop = old < x ? x : old;
      if (g.analysis) {
        Val m = g.val[keep];
        val_merge_into(m, g.val[drop]);
        g.val[keep] = m;
      }
      g.parent[drop] = keep;
    }
  }
}

// stats over candidates [0, ncommit): shape / cycle / applied / noop
// With a reject log (on_reject registered), every cycle-rejected combo's
// product position is appended (unordered; the host sorts a rule's log).
__device__ __forceinline__ void d_seg_stats(u64 tid, u64 nth, const u8* status, WaveState* ws, u32 ncommit,
                                            const u32* accpre, const u32* alloc, const u8* ukind, int efficient,
                                            DevStats* st, const RuleDev& R, unsigned long long p,
                                            const unsigned long long* posp) {
  TID_LOOP(c, ncommit) {
    u8 s = status[c];
    if (s == 1) atomicAdd(&st->skipped_shape, 1ull);
    else if (s == 2) {
      atomicAdd(&st->skipped_cycle, 1ull);
      atomicAdd(&st->prefilter_checks, 1ull);
      atomicAdd(&st->prefilter_rejects, 1ull);
      if (R.rej_log) {
        const u32 k = atomicAdd(&st->nrej, 1u);
        if (k < R.rej_cap) {
          const unsigned long long pos = posp ? posp[c] : p + c;
          R.rej_log[2 * (u64)k] = (u32)(pos >> 32);
          R.rej_log[2 * (u64)k + 1] = (u32)pos;
        }
      }
    } else {
      if (efficient) atomicAdd(&st->prefilter_checks, 1ull);
      u32 a = accpre[c];
      bool un = false;
      for (int t = 0; t < MAX_SRC; t++) un |= ukind[(u64)a * MAX_SRC + t] != UK_NONE;
      if (alloc[a] > 0 || un) {
        atomicAdd(&st->applied, 1ull);
        st->changed = 1;
        ws->any_applied = 1;
      } else {
        atomicAdd(&st->applied_noop, 1ull);
      }
    }
  }
}

// ---------------------------------------------------------------- commit

__device__ __forceinline__ void d_win_flags(u64 tid, u64 nth, const WaveTab& T, const u32* ident, u64 nreq,
                                            const ReqT* tmpl, int R, u64 lim, u32* wf, u32* ka) {
  TID_LOOP(q, nreq) {
    u32 id = q < lim ? ident[q] : 0u;
    bool win = q < lim && (id & FRESH) && is_winner(T, id & ~FRESH, q);
    wf[q] = win ? 1u : 0u;
    ka[q] = win ? (u32)tmpl[q % R].nargs : 0u;
  }
}

__device__ __forceinline__ void d_assign_ids(u64 tid, u64 nth, const WaveTab& T, const u32* ident, u64 nreq,
                                             const u32* wf, const u32* wpre, u32 base) {
  TID_LOOP(q, nreq) if (wf[q]) T.wid[ident[q] & ~FRESH] = base + wpre[q];
}

__device__ __forceinline__ void d_write_nodes(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                              const u32* acc, const u32* ident, u64 nreq, const u32* wf,
                                              const u32* wpre, const u32* kpre, u32 base, u32 kbase, const u32* env,
                                              const u32* olds) {
  TID_LOOP(q, nreq) {
    if (!wf[q]) continue;
    u32 a = (u32)(q / W.R);
    int r = (int)(q % W.R);
    u32 c = acc[a];
    const ReqT& tq = W.tmpl[r];
    u32 s = ident[q] & ~FRESH;
    u32 id = base + wpre[q];
    u32 ko = kbase + kpre[q];
    g.op[id] = tq.atom;
    g.koff[id] = ko;
    g.koff[id + 1] = ko + tq.nargs;
    for (int j = 0; j < tq.nargs; j++) {
      int k = tq.kid[j];
      u32 v = k >= 0 ? ident[(u64)a * W.R + k] : env[(u64)c * MAX_VARS + (-k - 1)];
      g.kids[ko + j] = (v & FRESH) ? T.wid[v & ~FRESH] : v;
    }
    g.flags[id] = NF_ALIVE;
    if (g.analysis) g.val[id] = T.val[s];
    g.parent[id] = tq.is_root ? olds[(u64)c * MAX_SRC + tq.tgt] : id;
  }
}

// per-combo commit (single-CTA path): node ids / kid offsets from the
// per-combo prefixes of winners and winners' children, requests in order
__device__ __forceinline__ void d_assign_combos(u64 tid, u64 nth, const WaveRule& W, const WaveTab& T, u32 ncacc,
                                                const u32* ident, const u32* apre, u32 base) {
  TID_LOOP(a, ncacc) {
    u32 id = base + apre[a];
    for (int r = 0; r < W.R; r++) {
      u64 q = a * (u64)W.R + r;
      u32 v = ident[q];
      if ((v & FRESH) && is_winner(T, v & ~FRESH, q)) T.wid[v & ~FRESH] = id++;
    }
  }
}

__device__ __forceinline__ void d_write_combos(u64 tid, u64 nth, const G& g, const WaveRule& W, const WaveTab& T,
                                               const u32* acc, u32 ncacc, const u32* ident, const u32* apre,
                                               const u32* kpre, u32 base, u32 kbase, const u32* env,
                                               const u32* olds) {
  TID_LOOP(a, ncacc) {
    u32 id = base + apre[a], ko = kbase + kpre[a];
    u32 c = acc[a];
    for (int r = 0; r < W.R; r++) {
      u64 q = a * (u64)W.R + r;
      u32 v0 = ident[q];
      if (!(v0 & FRESH)) continue;
      u32 s = v0 & ~FRESH;
      if (!is_winner(T, s, q)) continue;
      const ReqT& tq = W.tmpl[r];
      g.op[id] = tq.atom;
      g.koff[id] = ko;
      g.koff[id + 1] = ko + tq.nargs;
      for (int j = 0; j < tq.nargs; j++) {
        int k = tq.kid[j];
        u32 v = k >= 0 ? ident[a * (u64)W.R + k] : env[(u64)c * MAX_VARS + (-k - 1)];
        g.kids[ko + j] = (v & FRESH) ? T.wid[v & ~FRESH] : v;
      }
      g.flags[id] = NF_ALIVE;
      if (g.analysis) g.val[id] = T.val[s];
      g.parent[id] = tq.is_root ? olds[(u64)c * MAX_SRC + tq.tgt] : id;
      ko += tq.nargs;
      id++;
    }
  }
}

// commit boundary: stops = [stop_after cand, cutoff cand, first bad cand]
__device__ __forceinline__ void d_boundary(WaveState* ws, const u32* stops, u32 ncand, const unsigned long long* pos,
                                           unsigned long long p, unsigned long long seg_end, const u32* pre,
                                           const u8* hazard) {
  const u64 INF = (u64)1 << 40;
  u64 e_sa = stops[0] == TSAT_NONE ? INF : (u64)stops[0] + 1;
  u64 e_cut = stops[1] == TSAT_NONE ? INF : (u64)stops[1] + 1;
  u64 e_bad = stops[2] == TSAT_NONE ? INF : (u64)stops[2];
  u64 e_end = e_bad < e_cut ? e_bad : e_cut;
  e_end = e_end < e_sa ? e_end : e_sa;
  e_end = e_end < ncand ? e_end : ncand;
  auto posf = [&](u32 c) -> unsigned long long { return pos ? pos[c] : p + c; };
  ws->stop = 0;
  ws->hazard = 0;
  ws->why = 0;
  ws->sa_hit = 0;
  ws->p_end = seg_end;
  if (e_cut <= e_end) {
    ws->p_end = posf(stops[1]) + 1;
    ws->stop = 1;
  } else if (e_bad <= e_end) {
    ws->p_end = posf(stops[2]);
    ws->why = hazard[stops[2]];
    ws->hazard = ws->why != 0;
  } else if (e_sa <= e_end) {
    ws->p_end = posf(stops[0]) + 1;
    ws->sa_hit = 1;
  }
  ws->ncommit_cand = (u32)e_end;
  ws->ncommit_acc = pre[e_end];
  ws->any_applied = 0;
}

// ---------------------------------------------------------------- grid kernels

#define GTID (blockIdx.x * (u64)blockDim.x + threadIdx.x)
#define GNTH ((u64)gridDim.x * blockDim.x)

__global__ void k_gates(G g, RuleDev R, ReachDev RD, WaveRule W, const unsigned long long* pos, u32 n,
                        unsigned long long p_base, u8* status, u32* env_out, u32* old_out, u8* hazard) {
  d_gates(GTID, GNTH, g, R, RD, pos, n, p_base, status, env_out, old_out, hazard);
}

__global__ void k_accept_flags(const u8* status, const u8* hazard, u32 n, u32* fl) {
  GRID_STRIDE(c, n) fl[c] = (status[c] == 0 || hazard[c]) ? 1u : 0u;
}

__global__ void k_accept_list(const u32* fl, const u32* pre, u32 n, u32* acc) {
  GRID_STRIDE(c, n) if (fl[c]) acc[pre[c]] = (u32)c;
}

__global__ void k_resolve_claim(G g, WaveRule W, WaveTab T, const u32* acc, const WaveState* ws, const int* lvl_req,
                                int nlvl, const u32* env, u32* ident, const u8* hazard) {
  d_resolve_claim(GTID, GNTH, g, W, T, acc, ws->nacc, lvl_req, nlvl, env, ident, hazard);
}

__global__ void k_resolve_verify(G g, WaveRule W, WaveTab T, const u32* acc, const WaveState* ws, const int* lvl_req,
                                 int nlvl, const u32* env, const u32* ident, u8* hazard) {
  d_resolve_verify(GTID, GNTH, g, W, T, acc, ws->nacc, lvl_req, nlvl, env, ident, hazard);
}

__global__ void k_mark_roots(WaveRule W, WaveTab T, const u32* acc, const WaveState* ws, const u32* ident,
                             const u8* hazard, const u32* olds) {
  d_mark_roots(GTID, GNTH, W, T, acc, ws->nacc, ident, hazard, olds);
}

__global__ void k_cand_check(G g, WaveRule W, WaveTab T, const u32* acc, const WaveState* ws, u32 ncand,
                             const u32* ident, const u32* env, const u32* olds, int multi, u8* hazard, u32* alloc,
                             u8* ukind, u32* uother, u8* grow, u8* stop_after, u32* akid) {
  d_cand_check(GTID, GNTH, g, W, T, acc, ws->nacc, ncand, ident, env, olds, multi, hazard, alloc, ukind, uother, grow,
               stop_after, akid);
}

__global__ void k_first_writer(WaveRule W, u32 epoch, const u32* acc, const WaveState* ws, const u8* hazard,
                               const u32* olds, const u8* ukind, const u32* uother, const u8* grow,
                               unsigned long long* fw_cls, unsigned long long* fw_fresh) {
  d_first_writer(GTID, GNTH, W, epoch, acc, ws->nacc, hazard, olds, ukind, uother, grow, fw_cls, fw_fresh);
}

__global__ void k_validity(WaveRule W, WaveTab T, RuleDev R, ReachDev RD, u32 ncand, const u8* hazard,
                           const u32* env, const u32* olds, const u32* accpre, const u8* status, const u32* ident,
                           const u8* ukind, const u8* grow, const u32* uother, const unsigned long long* fw_cls,
                           const unsigned long long* fw_fresh, u32* first_bad) {
  d_validity(GTID, GNTH, W, T, T.epoch, R, RD, ncand, hazard, env, olds, accpre, status, ident, ukind, grow, uother,
             fw_cls, fw_fresh, first_bad, nullptr);
}

// Conflict pass of a grid wave, iterated like the single-CTA loop: first
// writers, validity, and (one thread) resolution of the first soft writer,
// with grid-wide barriers in between (cooperative launch, co-resident grid).
// Epochs ep0 .. ep0 + max_it tag the first-writer arrays.
__global__ void k_conflicts_grid(G g, WaveRule W, WaveTab T, RuleDev R, ReachDev RD, const u32* acc,
                                 const WaveState* ws, u32 ncand, u8* hazard, const u32* env, u32* olds,
                                 const u32* accpre, u8* status, const u32* ident, u8* ukind, u8* grow, u32* uother,
                                 unsigned long long* fw_cls, unsigned long long* fw_fresh, u32* stops, u32 ep0,
                                 u32 max_it, u32* nresolved) {
  cooperative_groups::grid_group gg = cooperative_groups::this_grid();
  const u32 nacc = ws->nacc;
  for (u32 it = 0;; it++) {
    const u32 ep = ep0 + it;
    d_first_writer(GTID, GNTH, W, ep, acc, nacc, hazard, olds, ukind, uother, grow, fw_cls, fw_fresh);
    gg.sync();
    d_validity(GTID, GNTH, W, T, ep, R, RD, ncand, hazard, env, olds, accpre, status, ident, ukind, grow, uother,
               fw_cls, fw_fresh, stops + 2, stops + 3);
    gg.sync();
    const u32 fb = ((volatile u32*)stops)[2], sw = ((volatile u32*)stops)[3];
    gg.sync();
    if (sw == TSAT_NONE || sw >= fb) break;
    if (GTID == 0) {
      if (it + 1 >= max_it || !d_resolve_soft(g, W, T, ep, R, RD, sw, env, olds, accpre, ukind, uother, grow, fw_cls,
                                              fw_fresh))
        status[sw] = 3;
      else
        *nresolved += 1;
      stops[2] = stops[3] = TSAT_NONE;
    }
    gg.sync();
  }
}

__global__ void k_find_stops(const u32* acc, const WaveState* ws, const u8* stop_after, const u32* apre,
                             const u32* alloc, const Counters* cnt, i64 n_max, u32* out) {
  d_find_stops(GTID, GNTH, acc, ws->nacc, stop_after, apre, alloc, (i64)cnt->live, n_max, out);
}

__global__ void k_commit_unions(G g, WaveRule W, WaveTab T, const u32* acc, const WaveState* ws, const u32* olds,
                                const u8* ukind, const u32* uother, const u8* grow) {
  d_commit_unions(GTID, GNTH, g, W, T, acc, ws->ncommit_acc, olds, ukind, uother, grow);
}

__global__ void k_seg_stats(const u8* status, WaveState* ws, u32 ncand, const u32* accpre, const u32* alloc,
                            const u8* ukind, int efficient, DevStats* st, RuleDev R, unsigned long long p,
                            const unsigned long long* posp) {
  u32 nc = ws->ncommit_cand;
  d_seg_stats(GTID, GNTH, status, ws, nc < ncand ? nc : ncand, accpre, alloc, ukind, efficient, st, R, p, posp);
}

__global__ void k_win_flags(WaveTab T, const u32* ident, u64 nreq, const ReqT* tmpl, int R, const WaveState* ws,
                            u32* wf, u32* ka) {
  d_win_flags(GTID, GNTH, T, ident, nreq, tmpl, R, (u64)ws->ncommit_acc * R, wf, ka);
}

__global__ void k_assign_ids(WaveTab T, const u32* ident, u64 nreq, const u32* wf, const u32* wpre,
                             const WaveState* ws) {
  d_assign_ids(GTID, GNTH, T, ident, nreq, wf, wpre, ws->base);
}

__global__ void k_write_nodes(G g, WaveRule W, WaveTab T, const u32* acc, const u32* ident, u64 nreq,
                              const u32* wf, const u32* wpre, const u32* kpre, const WaveState* ws,
                              const u32* env, const u32* olds) {
  d_write_nodes(GTID, GNTH, g, W, T, acc, ident, nreq, wf, wpre, kpre, ws->base, ws->kbase, env, olds);
}

__global__ void k_insert_range(G g, const WaveState* ws, u64 bound) {
  u32 a = ws->base, n = ws->nwin;
  GRID_STRIDE(i, bound) if (i < n) hc_insert(g, a + (u32)i);
}

// ---------------------------------------------------------------- device-side wave control

// block-wide exclusive scan of f(i), i < n, with the total at out[n]
// (all threads of the block must call it)
template <int BT, class F>
__device__ __forceinline__ u32 block_scan(u32 n, u32* out, F f) {
  typedef cub::BlockScan<u32, BT> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = 0; base < n; base += BT) {
    u32 i = base + threadIdx.x;
    u32 v = i < n ? f(i) : 0u, x, tot;
    BS(tmp).ExclusiveSum(v, x, tot);
    if (i < n) out[i] = carry + x;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  u32 total = carry;
  if (threadIdx.x == 0) out[n] = total;
  __syncthreads();
  return total;
}

// block-wide exclusive scan of two counters at once (packed in a u64):
// out_a / out_b get the prefixes of fa / fb, totals at [n]
template <int BT, class F>
__device__ __forceinline__ void block_scan2(u32 n, u32* out_a, u32* out_b, F f) {
  typedef cub::BlockScan<unsigned long long, BT> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = 0; base < n; base += BT) {
    u32 i = base + threadIdx.x;
    unsigned long long v = i < n ? f(i) : 0ull, x, tot;
    BS(tmp).ExclusiveSum(v, x, tot);
    if (i < n) {
      out_a[i] = (u32)((carry + x) >> 32);
      out_b[i] = (u32)(carry + x);
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_a[n] = (u32)(carry >> 32);
    out_b[n] = (u32)carry;
  }
  __syncthreads();
}

// block-wide exclusive scan over tiles of BT * IT elements, IT consecutive
// elements per thread (independent loads in flight); total at out[n]
template <int BT, int IT, class F>
__device__ __forceinline__ u32 block_scan_tiled(u32 n, u32* out, F f) {
  typedef cub::BlockScan<u32, BT> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = 0; base < n; base += BT * IT) {
    u32 i0 = base + threadIdx.x * IT;
    u32 v[IT], sum = 0;
#pragma unroll
    for (int k = 0; k < IT; k++) {
      v[k] = i0 + k < n ? f(i0 + k) : 0u;
      sum += v[k];
    }
    u32 x, tot;
    BS(tmp).ExclusiveSum(sum, x, tot);
    x += carry;
#pragma unroll
    for (int k = 0; k < IT; k++) {
      if (i0 + k < n) out[i0 + k] = x;
      x += v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  u32 total = carry;
  if (threadIdx.x == 0) out[n] = total;
  __syncthreads();
  return total;
}

// single-CTA exclusive scan with the total at out[n] (small arrays; CUB's two
// kernels cost more than the work at wave sizes)
__global__ void __launch_bounds__(1024) k_scan_block(const u32* in, u32* out, u32 n) {
  block_scan_tiled<1024, 8>(n, out, [&](u32 i) { return in[i]; });
}

// accepted list (status 0 or flagged) in candidate order; ws->nacc
__global__ void __launch_bounds__(1024) k_accept_scan(const u8* status, const u8* hazard, u32 n, u32* pre, u32* acc,
                                                      WaveState* ws) {
  u32 tot = block_scan_tiled<1024, 8>(n, pre, [&](u32 c) { return (status[c] == 0 || hazard[c]) ? 1u : 0u; });
  for (u32 c = threadIdx.x; c < n; c += 1024)
    if (status[c] == 0 || hazard[c]) acc[pre[c]] = c;
  if (threadIdx.x == 0) ws->nacc = tot;
}

__global__ void k_boundary(WaveState* ws, const u32* stops, u32 ncand, const unsigned long long* pos,
                           unsigned long long p, unsigned long long seg_end, const u32* pre, const u8* hazard) {
  if (threadIdx.x || blockIdx.x) return;
  d_boundary(ws, stops, ncand, pos, p, seg_end, pre, hazard);
}

__global__ void k_commit_prep(WaveState* ws, const u32* wpre, const u32* kpre, u64 nq, const Counters* cnt) {
  if (threadIdx.x || blockIdx.x) return;
  ws->nwin = wpre[nq];
  ws->nk = kpre[nq];
  ws->base = cnt->next_id;
  ws->kbase = cnt->nkids;
}

__global__ void k_set_nacc(const u32* pre, u32 n, WaveState* ws) {
  if (threadIdx.x || blockIdx.x) return;
  ws->nacc = pre[n];
}

__global__ void k_zero_commit(WaveState* ws, const Counters* cnt) {
  if (threadIdx.x || blockIdx.x) return;
  ws->nwin = 0;
  ws->nk = 0;
  ws->base = cnt->next_id;
  ws->kbase = cnt->nkids;
}

__global__ void k_counters_commit(WaveState* ws, Counters* cnt) {
  if (threadIdx.x || blockIdx.x) return;
  cnt->next_id += ws->nwin;
  cnt->live += ws->nwin;
  cnt->nkids += ws->nk;
  if (ws->any_applied) cnt->dirty = 1;
}

// ---------------------------------------------------------------- single-CTA wave loop

// Buffers of one wave (device pointers).
struct WaveIO {
  u8 *status, *hazard, *ukind, *grow, *sa;
  u32 *env, *olds, *pre, *acc, *ident, *alloc, *apre, *wf, *wpre, *ka, *kpre, *uother, *stops, *akid, *ckpre;
  unsigned long long *fw_cls, *fw_fresh;
  WaveState* ws;
  DevStats* wstats;
  const int* lvl;
};

// reasons the CTA loop returns to the host
#define CR_DONE 0     // positions exhausted
#define CR_HAZARD 1   // exact path for position p, then resume at p + 1
#define CR_STOP 2     // node limit: iteration stops
#define CR_REJOIN 3   // multi-pattern join cache invalid (or capped list exhausted)
#define CR_CAPACITY 4 // grow node / kid / hashcons capacity, then resume
#define CR_WIDE 5     // clean full windows: continue on the grid path
#define CR_ERROR 6    // analysis/table capacity error (exact path reports it)
#define CR_NOTRUN 7   // chained launch skipped: an earlier rule of the chain returned to the host
#define CR_NARROW 8   // grid-mode loop: windows shrank to single-CTA size
#define CR_TIMEOUT 9  // the time limit passed before the next wave (device clock)

struct CtaCtl {
  unsigned long long p, P;
  u32 win, epoch;
  u32 jcursor, jtotal;
  int jcomplete;
  u32 reason;
  u32 waves, clean_full;
  u32 cuts[6];
  u32 resolved;  // soft writers resolved inside waves
  unsigned long long found, self, compat;
  unsigned long long s_cand, s_req, s_win, s_nk;
  i64 overshoot;
  u32 seq_stop;
  unsigned long long prof[12];  // ns per wave phase (thread 0's view)
};

struct CtaArgs {
  int nlv;                 // request levels (depth 1 .. nlv-1)
  int lvl_off[12];
  int nlvl[12];
  int skip_self, multi, Kmax;
  u32 nA, nB;
  i64 n_max;
  u32 cta_win;
  const unsigned long long* pos;  // cached join list (multi)
  int smem;  // per-candidate wave arrays in shared memory (window <= cta_win)
  u32 wide_after;  // clean full windows before handing over to the grid path
  // grid mode (NC == 0): control words and per-block scan totals in global memory
  void* gsh;
  unsigned long long* gtot;
  u32 narrow_win;  // grid mode: a window this small goes back to the single-CTA loop
};

// shared-memory carve-out of the per-candidate wave arrays (window of `win`
// candidates, R requests each); returns the byte size when out == nullptr
__host__ __device__ inline size_t wave_smem_layout(u32 win, int R, unsigned char* base, WaveIO* out) {
  size_t o = 0;
  auto take = [&](size_t bytes) -> void* {
    void* p = base ? (void*)(base + o) : nullptr;
    o += (bytes + 15) & ~(size_t)15;
    return p;
  };
  void* status = take(win + 1);
  void* hazard = take(win + 1);
  void* sa = take(win + 1);
  void* ukind = take((size_t)win * MAX_SRC + 1);
  void* grow = take((size_t)win * MAX_SRC + 1);
  void* env = take(((size_t)win * MAX_VARS + 1) * 4);
  void* olds = take(((size_t)win * MAX_SRC + 1) * 4);
  void* uother = take(((size_t)win * MAX_SRC + 1) * 4);
  void* pre = take(((size_t)win + 2) * 4);
  void* acc = take(((size_t)win + 1) * 4);
  void* ident = take(((size_t)win * (R > 0 ? R : 1) + 1) * 4);
  void* alloc = take(((size_t)win + 2) * 4);
  void* apre = take(((size_t)win + 2) * 4);
  void* akid = take(((size_t)win + 2) * 4);
  void* ckpre = take(((size_t)win + 2) * 4);
  void* stops = take(16);
  if (out) {
    out->status = (u8*)status;
    out->hazard = (u8*)hazard;
    out->sa = (u8*)sa;
    out->ukind = (u8*)ukind;
    out->grow = (u8*)grow;
    out->env = (u32*)env;
    out->olds = (u32*)olds;
    out->uother = (u32*)uother;
    out->pre = (u32*)pre;
    out->acc = (u32*)acc;
    out->ident = (u32*)ident;
    out->alloc = (u32*)alloc;
    out->apre = (u32*)apre;
    out->akid = (u32*)akid;
    out->ckpre = (u32*)ckpre;
    out->stops = (u32*)stops;
  }
  return o;
}

__device__ __forceinline__ unsigned long long self_in(u32 nA, u32 nB, unsigned long long p0, unsigned long long p1) {
  // #{i < nA : p0 <= i * (nB + 1) < p1}
  unsigned long long d = (unsigned long long)nB + 1;
  unsigned long long lo = (p0 + d - 1) / d, hi = (p1 + d - 1) / d;
  if (hi > nA) hi = nA;
  return hi > lo ? hi - lo : 0;
}

#define CTA_T 1024

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define WPROF(k)                          \
  if (tid == 0) {                         \
    unsigned long long t_ = gtimer();     \
    ctl->prof[k] += t_ - t_last;          \
    t_last = t_;                          \
  }

// control words of a wave loop (k_wave_cta): written by thread 0 of rank 0,
// read by every thread after the next barrier
struct WaveSh {
  unsigned long long p, seg_end;
  u32 ncand, jcur, exit, epoch, nacc, ncacc, base, kbase;
  int rejoin_after;
  u32 wres;  // soft writers resolved in the current wave
  int abort;
};

template <int NC>
__device__ __forceinline__ void wsync() {
  if constexpr (NC > 1) cg::this_cluster().sync();
  else if constexpr (NC == 0) cg::this_grid().sync();
  else __syncthreads();
}



// exclusive scan of f(i) over n elements, total at out[n]; NC > 1: each CTA
// of the cluster scans one contiguous chunk, then adds the totals of the
// chunks before it (read from the other CTAs' shared memory)
template <int BT, class V, class F>
__device__ __forceinline__ V chunk_scan(u32 lo, u32 hi, F f, V* carry_out) {
  typedef cub::BlockScan<V, BT> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ V carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = lo; base < hi; base += BT) {
    u32 i = base + threadIdx.x;
    V v = i < hi ? f(i, (V)0, false) : (V)0, x, tot;
    BS(tmp).ExclusiveSum(v, x, tot);
    if (i < hi) f(i, carry + x, true);
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  V total = carry;
  __syncthreads();
  (void)carry_out;
  return total;
}

// grid mode (NC == 0): one chunk per block; block totals meet in global
// memory.  Returns the exclusive offset of this block's chunk [lo, hi) and
// the total; the caller adds the offset, then syncs the grid.
template <class V, class F, class W>
__device__ __forceinline__ V grid_chunk_scan(u32 n, F f, W wr, unsigned long long* gtot, u32& lo, u32& hi, V& off) {
  cg::grid_group gg = cg::this_grid();
  const u32 nb = gridDim.x, r = blockIdx.x, chunk = (n + nb - 1) / nb;
  lo = min(n, r * chunk);
  hi = min(n, lo + chunk);
  V t = chunk_scan<CTA_T, V>(lo, hi, [&](u32 i, V x, bool w) -> V {
    if (w) {
      wr(i, x);
      return (V)0;
    }
    return f(i);
  }, (V*)nullptr);
  if (threadIdx.x == 0) gtot[r] = (unsigned long long)t;
  gg.sync();
  __shared__ unsigned long long s_off, s_total;
  if (threadIdx.x == 0) {
    unsigned long long o = 0, total = 0;
    for (u32 q = 0; q < nb; q++) {
      const unsigned long long v = ((volatile unsigned long long*)gtot)[q];
      if (q < r) o += v;
      total += v;
    }
    s_off = o;
    s_total = total;
  }
  __syncthreads();
  off = (V)s_off;
  return (V)s_total;
}

template <int NC, class F>
__device__ __forceinline__ u32 wscan(u32 n, u32* out, F f, unsigned long long* gtot = nullptr) {
  if constexpr (NC == 1) {
    return block_scan<CTA_T>(n, out, f);
  } else if constexpr (NC == 0) {
    u32 lo, hi, off;
    const u32 total = grid_chunk_scan<u32>(n, f, [&](u32 i, u32 x) { out[i] = x; }, gtot, lo, hi, off);
    if (off)
      for (u32 i = lo + threadIdx.x; i < hi; i += CTA_T) out[i] += off;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = total;
    cg::this_grid().sync();
    return total;
  } else {
    cg::cluster_group cl = cg::this_cluster();
    const u32 r = cl.block_rank(), chunk = (n + NC - 1) / NC;
    const u32 lo = min(n, r * chunk), hi = min(n, lo + chunk);
    __shared__ u32 s_ctot;
    u32 t = chunk_scan<CTA_T, u32>(lo, hi, [&](u32 i, u32 x, bool wr) -> u32 {
      if (wr) {
        out[i] = x;
        return 0u;
      }
      return f(i);
    }, (u32*)nullptr);
    if (threadIdx.x == 0) s_ctot = t;
    cl.sync();
    u32 off = 0, total = 0;
    for (u32 q = 0; q < (u32)NC; q++) {
      const u32 v = *cl.map_shared_rank(&s_ctot, q);
      if (q < r) off += v;
      total += v;
    }
    if (off)
      for (u32 i = lo + threadIdx.x; i < hi; i += CTA_T) out[i] += off;
    if (r == NC - 1 && threadIdx.x == 0) out[n] = total;
    cl.sync();
    return total;
  }
}

template <int NC, class F>
__device__ __forceinline__ void wscan2(u32 n, u32* out_a, u32* out_b, F f, unsigned long long* gtot = nullptr) {
  if constexpr (NC == 1) {
    block_scan2<CTA_T>(n, out_a, out_b, f);
  } else if constexpr (NC == 0) {
    u32 lo, hi;
    unsigned long long off;
    const unsigned long long total = grid_chunk_scan<unsigned long long>(
        n, f,
        [&](u32 i, unsigned long long x) {
          out_a[i] = (u32)(x >> 32);
          out_b[i] = (u32)x;
        },
        gtot, lo, hi, off);
    if (off)
      for (u32 i = lo + threadIdx.x; i < hi; i += CTA_T) {
        const unsigned long long x = (((unsigned long long)out_a[i] << 32) | out_b[i]) + off;
        out_a[i] = (u32)(x >> 32);
        out_b[i] = (u32)x;
      }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
      out_a[n] = (u32)(total >> 32);
      out_b[n] = (u32)total;
    }
    cg::this_grid().sync();
  } else {
    cg::cluster_group cl = cg::this_cluster();
    const u32 r = cl.block_rank(), chunk = (n + NC - 1) / NC;
    const u32 lo = min(n, r * chunk), hi = min(n, lo + chunk);
    __shared__ unsigned long long s_ctot2;
    unsigned long long t = chunk_scan<CTA_T, unsigned long long>(
        lo, hi, [&](u32 i, unsigned long long x, bool wr) -> unsigned long long {
          if (wr) {
            out_a[i] = (u32)(x >> 32);
            out_b[i] = (u32)x;
            return 0ull;
          }
          return f(i);
        }, (unsigned long long*)nullptr);
    if (threadIdx.x == 0) s_ctot2 = t;
    cl.sync();
    unsigned long long off = 0, total = 0;
    for (u32 q = 0; q < (u32)NC; q++) {
      const unsigned long long v = *cl.map_shared_rank(&s_ctot2, q);
      if (q < r) off += v;
      total += v;
    }
    if (off)
      for (u32 i = lo + threadIdx.x; i < hi; i += CTA_T) {
        const unsigned long long x = (((unsigned long long)out_a[i] << 32) | out_b[i]) + off;
        out_a[i] = (u32)(x >> 32);
        out_b[i] = (u32)x;
      }
    if (r == NC - 1 && threadIdx.x == 0) {
      out_a[n] = (u32)(total >> 32);
      out_b[n] = (u32)total;
    }
    cl.sync();
  }
}

// NC = 1: one CTA, per-candidate arrays in shared memory when they fit.
// NC > 1: a thread-block cluster of NC CTAs runs the same loop over NC x
// larger windows: tid / nth span the cluster, phases end with cluster-wide
// barriers (release / acquire: global writes of one phase are visible to the
// next), the wave's control words live in rank 0's shared memory (read by
// every CTA through distributed shared memory), the per-candidate arrays in
// global memory (L2), and the accepted / allocation prefix sums are cluster
// scans (per-CTA chunk scans + DSMEM totals).
template <int NC>
__global__ void __launch_bounds__(CTA_T, 1) k_wave_cta(G g, RuleDev R, ReachDev RD, WaveRule W, WaveTab T, WaveIO io,
                                                       CtaArgs A, CtaCtl* ctl, const CtaCtl* prev) {
  extern __shared__ __align__(16) unsigned char wsm[];
  // per-candidate arrays in shared memory: each phase reads what the previous
  // one wrote, so this removes an L2 round trip from most phase chains
  if (NC == 1 && A.smem) wave_smem_layout(A.cta_win, W.R, wsm, &io);
  __shared__ WaveSh sh;
  WaveSh* S = &sh;
  u32 rank = 0;
  if constexpr (NC > 1) {
    cg::cluster_group cl = cg::this_cluster();
    rank = cl.block_rank();
    S = cl.map_shared_rank(&sh, 0);
  } else if constexpr (NC == 0) {  // cooperative grid: control words in global memory
    rank = blockIdx.x;
    S = (WaveSh*)A.gsh;
  }
  const u64 tid = (u64)rank * CTA_T + threadIdx.x, nth = (u64)CTA_T * (NC == 0 ? gridDim.x : NC);
  unsigned long long t_last = tid == 0 ? gtimer() : 0;
  if (tid == 0) {
    S->p = ctl->p;
    S->jcur = ctl->jcursor;
    S->epoch = ctl->epoch;
    S->abort = 0;
    // chained launch (run_rules_chain): runs only when the previous rule of
    // the chain finished (CR_DONE), continuing its wave epoch
    if (prev) {
      if (prev->reason != CR_DONE) {
        S->abort = 1;
        ctl->reason = CR_NOTRUN;
        ctl->epoch = prev->epoch;
      } else {
        S->epoch = prev->epoch;
      }
    }
  }
  wsync<NC>();
  {
    const int ab = S->abort;
    wsync<NC>();  // rank 0 stays until every CTA has read its shared memory
    if (ab) return;
  }
  while (true) {
    if (tid == 0) {
      S->exit = 0xFFFFFFFFu;
      S->rejoin_after = 0;
      unsigned long long p = S->p, P = ctl->P;
      Counters* cn = g.cnt;
      if (p >= P) {
        S->exit = CR_DONE;
      } else if ((i64)cn->live >= A.n_max) {
        ctl->seq_stop = 1;
        ctl->overshoot = (i64)cn->live - A.n_max;
        S->exit = CR_STOP;
      } else if (R.deadline_ns && dev_now_ns() > R.deadline_ns) {
        S->exit = CR_TIMEOUT;  // the next wave's combos are not reached (explorer.py:198-201)
      } else {
        u32 win = ctl->win;
        u32 ncand;
        unsigned long long seg_end = P;
        if (!A.multi) {
          unsigned long long n = P - p < win ? P - p : win;
          ncand = (u32)n;
          seg_end = p + n;
        } else {
          u32 remain = ctl->jtotal - S->jcur;
          ncand = remain < win ? remain : win;
          if (ncand < remain) seg_end = A.pos[S->jcur + ncand];
          else if (!ctl->jcomplete) {
            seg_end = A.pos[ctl->jtotal - 1] + 1;
            S->rejoin_after = 1;
          }
        }
        if (ncand == 0) {
          unsigned long long cover = seg_end - p, self = A.skip_self ? self_in(A.nA, A.nB, p, seg_end) : 0;
          ctl->found += cover;
          ctl->self += self;
          ctl->compat += cover - self;
          S->p = seg_end;
          S->exit = S->rejoin_after ? CR_REJOIN : 0xFFFFFFFEu;  // continue
        } else {
          u64 need_n = (u64)cn->next_id + (u64)ncand * W.R + 2;
          u64 need_k = (u64)cn->nkids + (u64)ncand * A.Kmax + 2;
          if (need_n + 1 > g.cap_nodes || need_k + 1 > g.cap_kids || need_n > (u64)g.hc_max) {
            S->exit = CR_CAPACITY;
          } else {
            S->ncand = ncand;
            S->seg_end = seg_end;
            S->epoch += 1;
            S->wres = 0;
            ctl->waves += 1;
            io.stops[0] = io.stops[1] = io.stops[2] = io.stops[3] = TSAT_NONE;
          }
        }
      }
    }
    wsync<NC>();
    {
      u32 ex = S->exit;
      wsync<NC>();
      if (ex == 0xFFFFFFFEu) continue;
      if (ex != 0xFFFFFFFFu) break;
    }
    const u32 ncand = S->ncand;
    WPROF(11);
    const unsigned long long p = S->p;
    const unsigned long long* posp = A.multi ? A.pos + S->jcur : nullptr;
    WaveTab Tw = T;
    Tw.epoch = S->epoch;
    // ---- gates + accepted list
    d_gates(tid, nth, g, R, RD, posp, ncand, p, io.status, io.env, io.olds, io.hazard);
    wsync<NC>();
    WPROF(0);
    {
      u32 tot = wscan<NC>(ncand, io.pre,
                          [&](u32 c) { return (io.status[c] == 0 || io.hazard[c]) ? 1u : 0u; }, A.gtot);
      for (u32 c = tid; c < ncand; c += nth)
        if (io.status[c] == 0 || io.hazard[c]) io.acc[io.pre[c]] = c;
      if (tid == 0) S->nacc = tot;
      wsync<NC>();
    }
    WPROF(1);
    const u32 nacc = S->nacc;
    // ---- resolve requests level by level
    if (W.R > 0) {
      for (int d = 1; d < A.nlv; d++) {
        if (!A.nlvl[d]) continue;
        d_resolve_claim(tid, nth, g, W, Tw, io.acc, nacc, io.lvl + A.lvl_off[d], A.nlvl[d], io.env, io.ident,
                        io.hazard);
        wsync<NC>();
        d_resolve_verify(tid, nth, g, W, Tw, io.acc, nacc, io.lvl + A.lvl_off[d], A.nlvl[d], io.env, io.ident,
                         io.hazard);
        wsync<NC>();
      }
      d_mark_roots(tid, nth, W, Tw, io.acc, nacc, io.ident, io.hazard, io.olds);
      wsync<NC>();
    }
    WPROF(2);
    d_cand_check(tid, nth, g, W, Tw, io.acc, nacc, ncand, io.ident, io.env, io.olds, A.multi, io.hazard, io.alloc,
                 io.ukind, io.uother, io.grow, io.sa, io.akid);
    wsync<NC>();
    WPROF(3);
    // ---- conflicts (re-run while the first one is a soft writer that
    // resolves), stop-after, node-limit cutoff, boundary
    for (int it = 0;; it++) {
      const u32 fwep = S->epoch;
      d_first_writer(tid, nth, W, fwep, io.acc, nacc, io.hazard, io.olds, io.ukind, io.uother, io.grow, io.fw_cls,
                     io.fw_fresh);
      wsync<NC>();
      d_validity(tid, nth, W, Tw, fwep, R, RD, ncand, io.hazard, io.env, io.olds, io.pre, io.status, io.ident,
                 io.ukind, io.grow, io.uother, io.fw_cls, io.fw_fresh, io.stops + 2, io.stops + 3);
      wsync<NC>();
      const u32 fb = io.stops[2], sw = io.stops[3];
      wsync<NC>();
      if (sw == TSAT_NONE || sw >= fb) break;
      if (tid == 0) {
        if (it >= (NC == 0 ? 4 : 64) || !d_resolve_soft(g, W, Tw, fwep, R, RD, sw, io.env, io.olds, io.pre, io.ukind, io.uother,
                                         io.grow, io.fw_cls, io.fw_fresh))
          io.status[sw] = 3;  // ends the prefix
        else {
          ctl->resolved += 1;
          S->wres += 1;
        }
        io.stops[2] = io.stops[3] = TSAT_NONE;
        S->epoch += 1;  // fresh first-writer tags
      }
      wsync<NC>();
    }
    WPROF(4);
    wscan2<NC>(ncand, io.apre, io.ckpre,
               [&](u32 c) { return ((unsigned long long)io.alloc[c] << 32) | io.akid[c]; }, A.gtot);
    d_find_stops(tid, nth, io.acc, nacc, io.sa, io.apre, io.alloc, (i64)g.cnt->live, A.n_max, io.stops);
    wsync<NC>();
    WPROF(5);
    if (tid == 0) {
      d_boundary(io.ws, io.stops, ncand, posp, p, S->seg_end, io.pre, io.hazard);
#ifdef WAVE_DBG
      if (io.stops[2] != TSAT_NONE && io.ws->ncommit_cand == io.stops[2] && (g_wdbg_first >> 8) == io.stops[2])
        g_wdbg_cnt[g_wdbg_first & 31] += 1;
      g_wdbg_first = ~0ull;
#endif
      S->ncacc = io.ws->ncommit_acc;
      S->base = g.cnt->next_id;
      S->kbase = g.cnt->nkids;
    }
    wsync<NC>();
    WPROF(6);
    const u32 ncacc = S->ncacc;
    d_seg_stats(tid, nth, io.status, io.ws, io.ws->ncommit_cand, io.pre, io.alloc, io.ukind, R.efficient, io.wstats,
                R, p, posp);
    // ---- commit (requests of committed combos only)
    const u32 nwin = io.apre[ncacc], nk = io.ckpre[ncacc];
    if (nwin) {
      d_assign_combos(tid, nth, W, Tw, ncacc, io.ident, io.apre, S->base);
      wsync<NC>();
      d_write_combos(tid, nth, g, W, Tw, io.acc, ncacc, io.ident, io.apre, io.ckpre, S->base, S->kbase, io.env, io.olds);
      wsync<NC>();  // unions overwrite parent[] of fresh non-root nodes
    }
    WPROF(7);
    d_commit_unions(tid, nth, g, W, Tw, io.acc, ncacc, io.olds, io.ukind, io.uother, io.grow);
    wsync<NC>();
    WPROF(8);
    for (u32 i = tid; i < nwin; i += nth) hc_insert(g, S->base + i);
    wsync<NC>();
    WPROF(9);
    // ---- bookkeeping (thread 0)
    if (tid == 0) {
      WaveState* ws = io.ws;
      Counters* cn = g.cnt;
      cn->next_id += nwin;
      cn->live += nwin;
      cn->nkids += nk;
      if (ws->any_applied) cn->dirty = 1;
      ctl->s_cand += ncand;
      ctl->s_req += (unsigned long long)nacc * W.R;
      ctl->s_win += nwin;
      ctl->s_nk += nk;
      u32 ncommit = ws->ncommit_cand;
      unsigned long long p_end = ws->p_end;
      bool stop = ws->stop != 0, hazard = ws->hazard != 0;
      if (ncommit < ncand && !stop) ctl->cuts[ws->why < 5 ? ws->why : 5] += 1;
      unsigned long long cover = p_end - p, self = A.skip_self ? self_in(A.nA, A.nB, p, p_end) : 0;
      ctl->found += cover;
      ctl->self += self;
      ctl->compat += cover - self - ncommit;
      if (A.multi) S->jcur += ncommit;
      S->p = p_end;
      u32 exitr = 0xFFFFFFFFu;
      if (stop) {
        if (p_end < ctl->P) {
          ctl->seq_stop = 1;
          ctl->overshoot = (i64)cn->live - A.n_max;
          exitr = CR_STOP;
        }
      } else {
        u32 win = ctl->win;
        if (ncommit < ncand) {
          u32 w2 = 2u * ncommit + 32u;
          win = w2 < 64u ? 64u : w2;
          ctl->clean_full = 0;
        } else {
          win = win * 4u;
          // a wave that needed soft-writer resolutions would be cut on the
          // grid path (which resolves only a few): stay here
          if (S->wres) ctl->clean_full = 0;
          else if (ncand >= A.cta_win) ctl->clean_full += 1;
        }
        if (win > A.cta_win) win = A.cta_win;
        ctl->win = win;
        if (hazard) exitr = CR_HAZARD;
        else if (A.multi && ws->sa_hit) exitr = CR_REJOIN;
        else if (S->rejoin_after) exitr = CR_REJOIN;
        else if (ctl->clean_full >= A.wide_after) exitr = CR_WIDE;
        else if (NC == 0 && win <= A.narrow_win) exitr = CR_NARROW;
      }
      S->exit = exitr;
    }
    wsync<NC>();
    WPROF(10);
    {
      u32 ex = S->exit;
      wsync<NC>();
      if (ex != 0xFFFFFFFFu) break;
    }
  }
  if (tid == 0) {
    ctl->p = S->p;
    ctl->jcursor = S->jcur;
    ctl->epoch = S->epoch;
    ctl->reason = S->exit;
  }
}

// ---------------------------------------------------------------- host side

struct WaveBufs {
  DevBuf<unsigned long long> pos;
  DevBuf<u64> hA, hB, hBs;
  DevBuf<u32> iB, iBs, cnt, off;
  DevBuf<u8> status, hazard;
  DevBuf<u32> env, olds, fl, pre, acc, ident, alloc, apre, wf, wpre, ka, kpre, stops, uother, akid, ckpre;
  DevBuf<unsigned long long> fw_cls, fw_fresh;  // epoch-tagged first writers
  DevBuf<CtaCtl> ctl;
  DevBuf<u8> ukind, grow, sa;
  DevBuf<WaveState> ws;
  DevBuf<DevStats> wstats;
  // deferred per-rule statistics (saturate reads an iteration's slots once)
  DevBuf<DevStats> wstats_def;
  std::vector<int> def_ri;
  DevStats* ws_cur = nullptr;  // the rule's statistics slot in use
  DevStats* hdef = nullptr;     // pinned: the deferred slots' read-back
  size_t hdef_cap = 0;
  bool def_pending = false;
  DevBuf<int> lvl;
  DevBuf<ReqT> tmpl;
  // wave table
  DevBuf<u32> wid, wroot, wold, wown;
  DevBuf<unsigned long long> wtag;
  DevBuf<unsigned long long> wminpos;
  DevBuf<Val> wval;
  u32 wcap = 0;
  u32 epoch = 0;  // per-wave tag of the wave table / first-writer arrays
  u64 cand_cap = 0;
  // per-rule request templates, built once per loaded rule set
  struct RuleWave {
    std::vector<ReqT> tm;
    WaveRule W;
    std::vector<std::vector<int>> lv;
    std::vector<int> lvl_off;
    int R = 0, Kmax = 0;
    size_t tmpl_base = 0, lvl_base = 0;
  };
  std::vector<RuleWave> rw;
  u64 rw_gen = ~0ull;
  DevBuf<ReqT> tmpl_all;
  DevBuf<int> lvl_all;
  CtaCtl* hctl = nullptr;       // pinned
  Counters* hcnt = nullptr;     // pinned
  DevBuf<unsigned long long> gsh, gtot;  // grid-mode control words / block totals
  // chained single-CTA launches (run_rules_chain)
  DevBuf<CtaCtl> chain_ctl;
  DevBuf<DevStats> chain_stats;
  CtaCtl* hchain = nullptr;     // pinned: K control blocks, then K DevStats
  size_t chain_cap = 0;
  ~WaveBufs() {
    if (hdef) cudaFreeHost(hdef);
    if (hchain) cudaFreeHost(hchain);
    if (hctl) cudaFreeHost(hctl);
    if (hcnt) cudaFreeHost(hcnt);
  }
};

void free_wave_bufs(WaveBufs* b) { delete b; }

static void build_wave_rule(const HRule& hr, std::vector<ReqT>& tm, WaveRule& W, std::vector<std::vector<int>>& lv,
                            int& R) {
  tm.clear();
  memset(&W, 0, sizeof(W));
  W.ntgt = hr.nsrc;
  int maxd = 0;
  for (int t = 0; t < hr.nsrc; t++) {
    std::vector<int> stack;  // >=0 request index, <0 var slot
    const auto& prog = hr.targets[t];
    for (const Instr& in : prog) {
      if (in.kind == I_VAR) {
        stack.push_back(-(in.arg + 1));
      } else {
        ReqT q;
        memset(&q, 0, sizeof(q));
        q.atom = in.atom;
        q.nargs = in.arg;
        for (int j = 0; j < in.arg; j++) q.kid[j] = stack[stack.size() - in.arg + j];
        stack.resize(stack.size() - in.arg);
        q.depth = in.depth;
        q.tgt = t;
        stack.push_back((int)tm.size());
        tm.push_back(q);
        maxd = std::max(maxd, in.depth);
      }
    }
    int top = stack.back();
    if (top >= 0) {
      W.root_req[t] = top;
      tm[top].is_root = 1;
      W.root_var[t] = -1;
    } else {
      W.root_req[t] = -1;
      W.root_var[t] = -top - 1;
    }
  }
  // Shared inner subterms (e.g. the split / matmul / concat_2 that both
  // targets of a merge rule contain) are ONE request: sequentially, the second
  // target's add_term hits the node the first one created, so resolving it
  // once is the same.  Target roots are never merged (a later reuse of a root
  // sees its merged class -- the wave's hazard path handles that case).
  {
    const int R0 = (int)tm.size();
    std::vector<int> canon(R0), newidx(R0, -1);
    for (int r = 0; r < R0; r++) {
      for (int j = 0; j < tm[r].nargs; j++)
        if (tm[r].kid[j] >= 0) tm[r].kid[j] = canon[tm[r].kid[j]];
      canon[r] = r;
      if (tm[r].is_root) continue;
      for (int q = 0; q < r; q++) {
        if (tm[q].is_root || canon[q] != q || tm[q].atom != tm[r].atom || tm[q].nargs != tm[r].nargs) continue;
        bool same = true;
        for (int j = 0; j < tm[r].nargs && same; j++) same = tm[q].kid[j] == tm[r].kid[j];
        if (same) {
          canon[r] = q;
          break;
        }
      }
    }
    std::vector<ReqT> uq;
    for (int r = 0; r < R0; r++)
      if (canon[r] == r) {
        newidx[r] = (int)uq.size();
        uq.push_back(tm[r]);
      }
    for (auto& q : uq)
      for (int j = 0; j < q.nargs; j++)
        if (q.kid[j] >= 0) q.kid[j] = newidx[q.kid[j]];
    for (int t = 0; t < hr.nsrc; t++)
      if (W.root_req[t] >= 0) W.root_req[t] = newidx[W.root_req[t]];
    tm.swap(uq);
  }
  R = (int)tm.size();
  W.R = R;
  lv.assign(maxd + 1, {});
  for (int r = 0; r < R; r++) lv[tm[r].depth].push_back(r);
  // shared slots between sources 0 and 1
  if (hr.nsrc == 2) {
    int ns = 0;
    for (int j = 0; j < hr.src_nb[0]; j++)
      for (int k = 0; k < hr.src_nb[1]; k++)
        if (hr.bind_slot[0][j] == hr.bind_slot[1][k] && ns < 8) {
          W.shpos[0][ns] = j;
          W.shpos[1][ns] = k;
          ns++;
        }
    W.nshared = ns;
  }
}

static u32 read_u32(Engine& e, const u32* p) {
  u32 v;
  CUDA_OK(cudaMemcpyAsync(&v, p, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  e.sync();
  return v;
}

void dev_exclusive_scan_u32(Engine& e, const u32* in, u32* out, u32 n);

static void accumulate_seg(Engine& e, int ri, const DevStats& d) {
  RuleStatsH& r = e.rstats[ri];
  r.applied += d.applied;
  r.applied_noop += d.applied_noop;
  r.skipped_shape += d.skipped_shape;
  r.skipped_cycle += d.skipped_cycle;
  e.report.prefilter_checks += d.prefilter_checks;
  e.report.prefilter_rejects += d.prefilter_rejects;
  if (d.changed) e.seq_changed = true;
}


#define CTA_WIN_1 2048u
// grid waves: one-CTA scans up to this size (a 1024-thread CTA walks 8k
// elements per tile step); larger ones take CUB's decoupled look-back scan
// (two launches, ~8 us) -- a 64k one-CTA scan took ~27 us
#define SCAN1_MAX 16384u
// thread-block cluster size of the wave loop (TSAT_WAVE_CLUSTER: 1 or 8; 2, 4
// and 16 were measured too) and the largest window it runs (one candidate per thread).  Default
// 1: measured on BERT (scripts/cluster_sweep.sh), larger windows do not cut
// the wave count -- waves end at the sequential-order conflicts (~1 per 2k
// combos), and a bigger window only adds soft writers to the serial
// resolution and L2 round trips (arrays leave shared memory): saturate
// 10.5 ms at 1, 11.5 at 4, 12.4 at 8, 12.0 at 16.
static int wave_nc() {
  static int nc = -1;
  if (nc < 0) {
    const char* v = getenv("TSAT_WAVE_CLUSTER");
    nc = v ? atoi(v) : 1;
    if (nc != 1 && nc != 8) nc = 1;
  }
  return nc;
}
// largest window of the cluster loop (TSAT_WAVE_CLUSTER_WIN, default one
// candidate per thread of the cluster)
static u32 wave_cluster_win() {
  static u32 w = 0;
  if (!w) {
    const char* v = getenv("TSAT_WAVE_CLUSTER_WIN");
    w = (u32)wave_nc() * CTA_T;
    if (v && atoi(v) >= 64 && (u32)atoi(v) < w) w = (u32)atoi(v);
  }
  return w;
}
// growth factor of the grid path's window after a clean full wave (TSAT_WIN_GROW;
// 16 measured against 4 / 8 (scripts/grow_sweep.sh): configs[4] apply 8.9 -> 8.3 ms,
// the fixed cost of a grid wave (~0.3 ms of launches and read-backs) paid on fewer
// ramp-up waves; BERT unchanged)
static u32 wave_grow() {
  static u32 gf = 0;
  if (!gf) {
    const char* v = getenv("TSAT_WIN_GROW");
    gf = v && atoi(v) >= 2 && atoi(v) <= 64 ? (u32)atoi(v) : 16u;
  }
  return gf;
}
// largest grid-path window (TSAT_WIN_MAX).  Grid windows start at 16k (TSAT_WIN0),
// grow 16x per clean full wave up to 1M (scripts/grow_sweep.sh, same box: BERT
// 10.9 -> 10.6 ms against 4k / 4x / 4M; configs[4] apply 8.9 -> 8.4 ms)
static u32 wave_win_max() {
  static u32 wm = 0;
  if (!wm) {
    const char* v = getenv("TSAT_WIN_MAX");
    wm = v && atoi(v) >= 4096 && atoi(v) <= (1 << 22) ? (u32)atoi(v) : (1u << 20);
  }
  return wm;
}
u32 wave_cta_cap() { return wave_nc() > 1 ? wave_cluster_win() : CTA_WIN_1; }
#define CTA_WIN (wave_cta_cap())

// per-candidate buffers, wave table and first-writer arrays for windows of up
// to ncand candidates (grown only; fresh tag arrays are set to "no epoch")
static void ensure_cand_bufs(Engine& e, WaveBufs& B, u64 ncand, int R) {
  if (ncand > B.cand_cap) {
    u64 n = std::max<u64>(ncand, 1024);
    B.status.ensure(n + 1);
    B.hazard.ensure(n + 1);
    B.env.ensure(n * MAX_VARS + 1);
    B.olds.ensure(n * MAX_SRC + 1);
    B.pre.ensure(n + 1);
    B.acc.ensure(n + 1);
    B.alloc.ensure(n + 1);
    B.apre.ensure(n + 2);
    B.akid.ensure(n + 1);
    B.ckpre.ensure(n + 2);
    B.ukind.ensure(n * MAX_SRC + 1);
    B.uother.ensure(n * MAX_SRC + 1);
    B.grow.ensure(n * MAX_SRC + 1);
    B.sa.ensure(n + 1);
    B.fl.ensure(n + 1);
    B.cand_cap = n;
  }
  u64 nreq = ncand * (u64)R;
  B.ident.ensure(nreq + 1);
  B.wf.ensure(nreq + 2);
  B.wpre.ensure(nreq + 2);
  B.ka.ensure(nreq + 2);
  B.kpre.ensure(nreq + 2);
  B.ws.ensure(1);
  B.stops.ensure(6);
  B.ctl.ensure(1);
  u64 want = 1024;
  while (want < 2 * nreq + 16) want *= 2;
  if (want > B.wcap) {
    B.wcap = (u32)want;
    B.wid.alloc(want);
    B.wroot.alloc(want);
    B.wold.alloc(want);
    B.wminpos.alloc(want);
    B.wval.alloc(want);
    B.fw_fresh.alloc(want + 1);
    B.wtag.alloc(want);
    B.wown.alloc(want);
    CUDA_OK(cudaMemsetAsync(B.wtag.p, 0, want * sizeof(unsigned long long), e.s));
    CUDA_OK(cudaMemsetAsync(B.wroot.p, 0, want * sizeof(u32), e.s));
    CUDA_OK(cudaMemsetAsync(B.wminpos.p, 0xFF, want * sizeof(unsigned long long), e.s));
    CUDA_OK(cudaMemsetAsync(B.fw_fresh.p, 0xFF, (want + 1) * sizeof(unsigned long long), e.s));
  }
  if (B.fw_cls.cap < (u64)e.cap_nodes + 1) {
    B.fw_cls.alloc((u64)e.cap_nodes + 1);
    CUDA_OK(cudaMemsetAsync(B.fw_cls.p, 0xFF, ((u64)e.cap_nodes + 1) * sizeof(unsigned long long), e.s));
  }
}

static unsigned long long self_in_host(u32 nA, u32 nB, unsigned long long p0, unsigned long long p1) {
  unsigned long long d = (unsigned long long)nB + 1;
  unsigned long long lo = (p0 + d - 1) / d, hi = (p1 + d - 1) / d;
  if (hi > nA) hi = nA;
  return hi > lo ? hi - lo : 0;
}

// algorithmic bytes of a wave (what the apply must touch at least):
// candidates: match rows + subst/olds writes + analyses read by the shape check;
// requests: hashcons probe (slot + key) + wave-table key/pos + analysis write;
// committed nodes: op, koff, kids, parent, flags, analysis, hashcons slot
static double wave_bytes(const Engine& e, const RuleDev& Rd, double ncand, double nreq, double nwin, double nk) {
  double nb = 0;
  for (int t = 0; t < Rd.nsrc; t++) nb += 4.0 * (1 + Rd.nb[t]);
  double per_cand = nb + 4.0 * (Rd.nslots + Rd.nsrc) + (e.analysis ? 128.0 * Rd.nslots : 0.0);
  double per_req = 4.0 + 16.0 + 4.0 * 2 + 48.0 + (e.analysis ? 128.0 : 0.0);
  double per_node = 21.0 + (e.analysis ? 128.0 : 0.0);
  return per_cand * ncand + per_req * nreq + per_node * nwin + 4.0 * nk;
}

// templates of every rule of the loaded set, uploaded once per rule set
static void ensure_wave_templates(Engine& e, WaveBufs& B) {
  if (!B.hctl) {
    CUDA_OK(cudaMallocHost((void**)&B.hctl, sizeof(CtaCtl)));
    CUDA_OK(cudaMallocHost((void**)&B.hcnt, sizeof(Counters)));
  }
  if (B.rw_gen != e.rules_gen) {
    // templates of every rule of the loaded set, uploaded once
    B.rw.assign(e.rules.size(), WaveBufs::RuleWave());
    std::vector<ReqT> tall;
    std::vector<int> lall;
    for (size_t r = 0; r < e.rules.size(); r++) {
      WaveBufs::RuleWave& x = B.rw[r];
      if (e.rules[r].nsrc > MAX_SRC) continue;
      build_wave_rule(e.rules[r], x.tm, x.W, x.lv, x.R);
      for (auto& q : x.tm) x.Kmax += q.nargs;
      x.tmpl_base = tall.size();
      tall.insert(tall.end(), x.tm.begin(), x.tm.end());
      x.lvl_base = lall.size();
      for (auto& l : x.lv) {
        x.lvl_off.push_back((int)(lall.size() - x.lvl_base));
        lall.insert(lall.end(), l.begin(), l.end());
      }
      x.lvl_off.push_back((int)(lall.size() - x.lvl_base));
    }
    B.tmpl_all.ensure(tall.size() + 1);
    B.lvl_all.ensure(lall.size() + 1);
    if (!tall.empty())
      CUDA_OK(cudaMemcpyAsync(B.tmpl_all.p, tall.data(), tall.size() * sizeof(ReqT), cudaMemcpyHostToDevice, e.s));
    if (!lall.empty())
      CUDA_OK(cudaMemcpyAsync(B.lvl_all.p, lall.data(), lall.size() * sizeof(int), cudaMemcpyHostToDevice, e.s));
    B.rw_gen = e.rules_gen;
  }
}

// window of a single-CTA run: the per-candidate arrays go to shared memory
// when they fit (a small window keeps most of the SM's L1 for the node table)
#define CTA_WSMEM (160u << 10)
static u32 cta_smem_win(int R) {
  return wave_smem_layout(CTA_T, R, nullptr, nullptr) <= CTA_WSMEM ? (u32)CTA_T : 512u;
}
static void cta_fit_window(CtaCtl& c, int R) {
  if (wave_nc() > 1) return;  // cluster windows: arrays in global memory
  u32 SWIN = cta_smem_win(R);
  if (wave_smem_layout(SWIN, R, nullptr, nullptr) <= CTA_WSMEM && c.win > SWIN) c.win = SWIN;
}

// launch k_wave_cta for rule ri on the engine stream (control block dctl,
// statistics wstats; prev = the previous launch of a chain or null)
static void cta_launch(Engine& e, WaveBufs& B, int ri, const RuleDev& Rd, const ReachDev& RD, int skip_self,
                       bool multi, i64 n_max, CtaCtl* dctl, const CtaCtl* prev, DevStats* wstats) {
  WaveBufs::RuleWave& RWc = B.rw[ri];
  WaveRule W = RWc.W;
  const std::vector<std::vector<int>>& lv = RWc.lv;
  const int R = RWc.R;
  W.tmpl = B.tmpl_all.p + RWc.tmpl_base;
  const std::vector<int>& lvl_off = RWc.lvl_off;
  int* lvl_dev = B.lvl_all.p + RWc.lvl_base;
  WaveTab T{B.wminpos.p, B.wid.p, B.wroot.p, B.wval.p, B.wcap - 1, B.wold.p, 0, B.wtag.p, B.wown.p};
  WaveIO io{B.status.p, B.hazard.p, B.ukind.p, B.grow.p, B.sa.p, B.env.p, B.olds.p, B.pre.p, B.acc.p,
            B.ident.p, B.alloc.p, B.apre.p, B.wf.p, B.wpre.p, B.ka.p, B.kpre.p, B.uother.p, B.stops.p,
            B.akid.p, B.ckpre.p, B.fw_cls.p, B.fw_fresh.p, B.ws.p, wstats, lvl_dev};
  CtaArgs A;
  memset(&A, 0, sizeof(A));
  A.nlv = (int)lv.size();
  for (size_t d = 0; d < lv.size(); d++) {
    A.lvl_off[d] = lvl_off[d];
    A.nlvl[d] = (int)lv[d].size();
  }
  A.skip_self = skip_self;
  A.multi = multi ? 1 : 0;
  A.Kmax = RWc.Kmax;
  A.nA = Rd.nmatch[0];
  A.nB = multi ? Rd.nmatch[1] : 1;
  A.n_max = n_max;
  A.cta_win = CTA_WIN;
  {
    static const char* wa = getenv("TSAT_WIDE_AFTER");
    A.wide_after = wa ? (u32)atoi(wa) : 8u;
  }
  A.pos = B.pos.p;
  const int nc = wave_nc();
  if (nc > 1) {
    G gv = e.view();
    A.smem = 0;
    A.cta_win = wave_cluster_win();
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(nc, 1, 1);
    cfg.blockDim = dim3(CTA_T, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = e.s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // one instantiation (compile time); the 2 / 4 / 16 variants measured no better
    CUDA_OK(cudaLaunchKernelEx(&cfg, k_wave_cta<8>, gv, Rd, RD, W, T, io, A, dctl, prev));
    return;
  }
  size_t smem_bytes = 0;
  {
    u32 SWIN = cta_smem_win(R);
    size_t need = wave_smem_layout(SWIN, R, nullptr, nullptr);
    if (need <= CTA_WSMEM) {
      static int smem_set = 0;
      if (!smem_set) {
        CUDA_OK(cudaFuncSetAttribute(k_wave_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_WSMEM));
        smem_set = 1;
      }
      A.smem = 1;
      A.cta_win = SWIN;
      smem_bytes = need;
    }
  }
  k_wave_cta<1><<<1, CTA_T, smem_bytes, e.s>>>(e.view(), Rd, RD, W, T, io, A, dctl, prev);
  CUDA_OK(cudaGetLastError());
}

// grid mode: the same wave loop as one cooperative launch over all SMs (one
// 1024-thread CTA per SM, windows up to 148 x 1024 candidates), replacing the
// host-driven grid waves (about 20 launches and a host round trip per wave)
static int grid_blocks() {
  static int nb = 0;
  if (!nb) {
    int per_sm = 0, nsm = 0, dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wave_cta<0>, CTA_T, 0));
    nb = std::max(1, per_sm) * nsm;
  }
  return nb;
}
// Opt-in (TSAT_WAVE_GRID=1): measured no faster than the host-driven grid
// waves -- ~20 grid-wide barriers per wave cost about what the launches did
// (BERT saturate 10.6 vs 10.4 ms, configs[4] apply 11.5 vs 11.7 ms).
static bool grid_mode_on() {
  static const int on = getenv("TSAT_WAVE_GRID") ? atoi(getenv("TSAT_WAVE_GRID")) : 0;
  return on != 0;
}
u32 wave_grid_cap() { return (u32)grid_blocks() * CTA_T; }

static void grid_launch(Engine& e, WaveBufs& B, int ri, const RuleDev& Rd, const ReachDev& RD, int skip_self,
                        bool multi, i64 n_max, CtaCtl* dctl) {
  WaveBufs::RuleWave& RWc = B.rw[ri];
  WaveRule W = RWc.W;
  const std::vector<std::vector<int>>& lv = RWc.lv;
  W.tmpl = B.tmpl_all.p + RWc.tmpl_base;
  WaveTab T{B.wminpos.p, B.wid.p, B.wroot.p, B.wval.p, B.wcap - 1, B.wold.p, 0, B.wtag.p, B.wown.p};
  WaveIO io{B.status.p, B.hazard.p, B.ukind.p, B.grow.p, B.sa.p, B.env.p, B.olds.p, B.pre.p, B.acc.p,
            B.ident.p, B.alloc.p, B.apre.p, B.wf.p, B.wpre.p, B.ka.p, B.kpre.p, B.uother.p, B.stops.p,
            B.akid.p, B.ckpre.p, B.fw_cls.p, B.fw_fresh.p, B.ws.p, B.ws_cur, B.lvl_all.p + RWc.lvl_base};
  CtaArgs A;
  memset(&A, 0, sizeof(A));
  A.nlv = (int)lv.size();
  for (size_t d = 0; d < lv.size(); d++) {
    A.lvl_off[d] = RWc.lvl_off[d];
    A.nlvl[d] = (int)lv[d].size();
  }
  A.skip_self = skip_self;
  A.multi = multi ? 1 : 0;
  A.Kmax = RWc.Kmax;
  A.nA = Rd.nmatch[0];
  A.nB = multi ? Rd.nmatch[1] : 1;
  A.n_max = n_max;
  const int nb = grid_blocks();
  A.cta_win = (u32)nb * CTA_T;
  A.wide_after = 0xffffffffu;
  A.narrow_win = CTA_WIN_1;
  A.pos = B.pos.p;
  A.smem = 0;
  B.gsh.ensure(sizeof(WaveSh) / 8 + 2);
  B.gtot.ensure((u64)nb + 2);
  A.gsh = B.gsh.p;
  A.gtot = B.gtot.p;
  G gv = e.view();
  RuleDev R = Rd;
  ReachDev RDv = RD;
  const CtaCtl* prev = nullptr;
  void* args[] = {&gv, &R, &RDv, &W, &T, &io, &A, &dctl, &prev};
  CUDA_OK(cudaLaunchCooperativeKernel((const void*)k_wave_cta<0>, nb, CTA_T, args, 0, e.s));
}

// host side of a single-CTA run's return (its control block c): statistics,
// resume position, and the reason's follow-up.  Returns true when the rule's
// loop must stop (node limit / stop inside the exact path).
static bool cta_exit(Engine& e, WaveBufs& B, int ri, const CtaCtl& c, unsigned long long& p, u32& jcursor, u32& win,
                     bool& jvalid, bool multi, int filter_mode, int allow_self, i64 n_max) {
  RuleStatsH& rs = e.rstats[ri];
  B.epoch = c.epoch;
  rs.found += c.found;
  rs.skipped_self += c.self;
  rs.skipped_compat += c.compat;
  e.phase_ms[8] += c.waves;
  for (int k = 0; k < 6; k++) e.phase_ms[10 + k] += c.cuts[k];
  for (int k = 0; k < 12; k++) e.phase_ms[16 + k] += c.prof[k] * 1e-6;
  e.phase_ms[28] += c.resolved;
  p = c.p;
  jcursor = c.jcursor;
  win = c.win;
  if (c.reason == CR_STOP) {
    e.seq_stop = true;
    e.report.node_limit_overshoot = c.overshoot;
    return true;
  } else if (c.reason == CR_TIMEOUT) {
    e.seq_timeout = true;
    return true;
  } else if (c.reason == CR_HAZARD) {
    e.phase_ms[9] += 1;
    if (multi) jvalid = false;
    e.ensure_nodes(4096, 4096);
    e.run_rule_seq(ri, filter_mode, allow_self, n_max, p, p + 1);
    if (e.seq_stop) return true;
    p = p + 1;
  } else if (c.reason == CR_REJOIN) {
    jvalid = false;
  } else if (c.reason == CR_WIDE) {
    win = 4 * CTA_WIN;
  }
  return false;
}

// one rule, positions [0, P): waves + exact fallback at hazards.  Windows of
// up to CTA_WIN candidates run inside k_wave_cta (one launch for a whole run
// of waves); larger windows run as grid waves.
void run_rule_wave(Engine& e, int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long P,
                   const CtaCtl* resume, const DevStats* resume_stats) {
  const HRule& hr = e.rules[ri];
  if (!e.wave) e.wave = new WaveBufs();
  WaveBufs& B = *e.wave;
  ensure_wave_templates(e, B);
  WaveBufs::RuleWave& RWc = B.rw[ri];
  WaveRule W = RWc.W;
  const std::vector<std::vector<int>>& lv = RWc.lv;
  const int R = RWc.R;
  W.tmpl = B.tmpl_all.p + RWc.tmpl_base;
  const std::vector<int>& lvl_off = RWc.lvl_off;
  if (lv.size() > 12) throw TsatException(TSAT_ERR_UNSUPPORTED, "target deeper than the wave engine supports");
  int* lvl_dev = B.lvl_all.p + RWc.lvl_base;
  const int Kmax = RWc.Kmax;
  int skip_self = (hr.nsrc == 2 && !allow_self && hr.same_canon) ? 1 : 0;
  const bool multi = hr.nsrc > 1;
  RuleStatsH& rs = e.rstats[ri];
  const double dbg_w0 = e.phase_ms[8], dbg_c0 = e.phase_ms[10];
  static const bool dbg_waves = getenv("TSAT_DEBUG_WAVES") != nullptr;
  std::chrono::steady_clock::time_point dbg_t0;
  if (dbg_waves) {
    e.sync();
    dbg_t0 = std::chrono::steady_clock::now();
  }
  // on_reject registered (efficient mode): the cycle-rejected positions of
  // the whole rule are logged on the device (waves) and by the exact path
  // (hazards), then handed over in position order = the sequential order
  const bool rec = e.record_rejects && filter_mode == 2;
  const u32 rej_cap = (u32)std::min<unsigned long long>(P, 1ull << 28);
  std::vector<unsigned long long> rej_seq;
  struct RejGuard {
    Engine& e;
    ~RejGuard() { e.rej_pending = nullptr; }
  } rej_guard{e};
  if (rec) {
    e.sc.v_rej_w.ensure(2 * (u64)rej_cap + 2);
    e.rej_pending = &rej_seq;
  }
  B.wstats.ensure(1);
  // statistics slot: deferred (saturate reads all of an iteration's rules in
  // one read-back) unless this rule's rejects must be handed over now
  const bool defer = e.defer_wave_stats && !rec && B.def_ri.size() < B.wstats_def.cap;
  B.ws_cur = defer ? B.wstats_def.p + B.def_ri.size() : B.wstats.p;
  if (defer) B.def_ri.push_back(ri);
  if (resume_stats) CUDA_OK(cudaMemcpyAsync(B.ws_cur, resume_stats, sizeof(DevStats), cudaMemcpyHostToDevice, e.s));
  else CUDA_OK(cudaMemsetAsync(B.ws_cur, 0, sizeof(DevStats), e.s));
  B.stops.ensure(6);
  if (!defer) CUDA_OK(cudaMemsetAsync(B.stops.p + 4, 0, sizeof(u32), e.s));  // grid-wave soft writers resolved
  // multi-pattern join cache: compatible positions stay valid until a union of
  // existing classes changes find() (stop-after waves / exact-path combos)
  bool jvalid = false, jcomplete = true;
  u32 jtotal = 0, jcursor = 0;
  const u32 JCAP = 1u << 24;
  unsigned long long p = 0;
  static const u32 win0 = getenv("TSAT_WIN0") ? (u32)atoi(getenv("TSAT_WIN0")) : (1u << 14);
  u32 win = win0;  // adaptive candidate window (grows on clean waves, shrinks on dependencies)
  bool stopped = false;
  if (resume) {  // a chained single-CTA launch returned here (run_rules_chain)
    stopped = cta_exit(e, B, ri, *resume, p, jcursor, win, jvalid, multi, filter_mode, allow_self, n_max);
  }
  while (!stopped && p < P) {
    // budget check at the segment's first position (explorer.py:198-206)
    if ((i64)e.h.live >= n_max) {
      e.seq_stop = true;
      e.report.node_limit_overshoot = (i64)e.h.live - n_max;
      break;
    }
    if (e.apply_deadline >= 0 && now_s() > e.apply_deadline) {
      e.seq_timeout = true;
      break;
    }
    RuleDev Rd = make_rule_dev(e, ri, filter_mode, allow_self);
    ReachDev RD = make_reach_dev(e);
    if (rec) {
      Rd.rej_log = e.sc.v_rej_w.p;
      Rd.rej_cap = rej_cap;
    }
    // ---- 1. compatible positions of a multi-pattern rule (cached)
    if (multi && !jvalid) {
      u32 nA = Rd.nmatch[0], nB = Rd.nmatch[1];
      u32 i0 = (u32)(p / nB);
      u32 na = nA - i0;
      B.hA.ensure(na + 1);
      B.hB.ensure(nB + 1);
      B.hBs.ensure(nB + 1);
      B.iB.ensure(nB + 1);
      B.iBs.ensure(nB + 1);
      B.cnt.ensure(na + 1);
      B.off.ensure(na + 1);
      DevBuf<u32>& dummy = e.scratch_u32[6];
      dummy.ensure(na + 1);
      k_hash_rows<<<nblk(nB), 256, 0, e.s>>>(e.view(), Rd.mbind[1], Rd.nb[1], nB, W, 1, B.hB.p, B.iB.p);
      k_hash_rows<<<nblk(na), 256, 0, e.s>>>(e.view(), Rd.mbind[0] + (u64)i0 * Rd.nb[0], Rd.nb[0], na, W, 0, B.hA.p,
                                             dummy.p);
      {
        size_t bytes = 0;
        CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, B.hB.p, B.hBs.p, B.iB.p, B.iBs.p, nB, 0, 64, e.s));
        e.temp.ensure(bytes + 16);
        CUDA_OK(cub::DeviceRadixSort::SortPairs(e.temp.p, bytes, B.hB.p, B.hBs.p, B.iB.p, B.iBs.p, nB, 0, 64, e.s));
      }
      k_join<<<nblk((u64)na * 32), 256, 0, e.s>>>(e.view(), Rd, W, B.hA.p, i0, B.hBs.p, B.iBs.p, p, skip_self,
                                                 nullptr, B.cnt.p, nullptr, 0);
      CUDA_OK(cudaMemsetAsync(B.cnt.p + na, 0, sizeof(u32), e.s));
      dev_exclusive_scan_u32(e, B.cnt.p, B.off.p, na + 1);
      u32 total = read_u32(e, B.off.p + na);
      jtotal = std::min<u32>(total, JCAP);
      jcomplete = total <= JCAP;
      B.pos.ensure((u64)jtotal + 1);
      if (jtotal)
        k_join<<<nblk((u64)na * 32), 256, 0, e.s>>>(e.view(), Rd, W, B.hA.p, i0, B.hBs.p, B.iBs.p, p, skip_self,
                                                   B.off.p, nullptr, B.pos.p, jtotal);
      jcursor = 0;
      jvalid = true;
    }
    u64 remain = multi ? (u64)(jtotal - jcursor) : (u64)(P - p);
    if (std::min<u64>(remain, win) <= CTA_WIN) {
      // ---- single-CTA run of waves
      e.ensure_nodes((u64)CTA_WIN * R + 2, (u64)CTA_WIN * Kmax + 2);
      ensure_cand_bufs(e, B, CTA_WIN, R);
      CtaCtl c;
      memset(&c, 0, sizeof(c));
      c.p = p;
      c.P = P;
      c.win = std::min<u32>(win, CTA_WIN);
      c.epoch = B.epoch;
      c.jcursor = jcursor;
      c.jtotal = jtotal;
      c.jcomplete = jcomplete ? 1 : 0;
      c.reason = CR_DONE;
      cta_fit_window(c, R);
      *B.hctl = c;
      CUDA_OK(cudaMemcpyAsync(B.ctl.p, B.hctl, sizeof(c), cudaMemcpyHostToDevice, e.s));
      {
        KTimer kt(e, KG_APPLY_WAVE, 0.0, 1);
        cta_launch(e, B, ri, Rd, RD, skip_self, multi, n_max, B.ctl.p, nullptr, B.ws_cur);
        CUDA_OK(cudaMemcpyAsync(B.hctl, B.ctl.p, sizeof(c), cudaMemcpyDeviceToHost, e.s));
        CUDA_OK(cudaMemcpyAsync(B.hcnt, e.cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, e.s));
        e.sync();
        c = *B.hctl;
        e.h = *B.hcnt;
        kt.bytes = wave_bytes(e, Rd, (double)c.s_cand, (double)c.s_req, (double)c.s_win, (double)c.s_nk);
      }
      if (dbg_waves)
        fprintf(stderr, "   cta: reason %u waves %u cand %llu resolved %u p %llu/%llu prof %.3f %.3f %.3f %.3f %.3f %.3f %.3f %.3f %.3f %.3f %.3f %.3f | %.3f ms\n", c.reason, c.waves,
                c.s_cand, c.resolved, c.p, P, c.prof[0]*1e-6, c.prof[1]*1e-6, c.prof[2]*1e-6, c.prof[3]*1e-6, c.prof[4]*1e-6, c.prof[5]*1e-6, c.prof[6]*1e-6, c.prof[7]*1e-6, c.prof[8]*1e-6, c.prof[9]*1e-6, c.prof[10]*1e-6, c.prof[11]*1e-6,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count());
      if (cta_exit(e, B, ri, c, p, jcursor, win, jvalid, multi, filter_mode, allow_self, n_max)) break;
      continue;
    }
    if (grid_mode_on()) {
      // ---- cooperative grid-wide run of waves (one launch, no host round
      // trip per wave); back here on hazards, capacity, stops, or when the
      // window shrinks to single-CTA size
      const u32 gcap = wave_grid_cap();
      const u64 wmax = std::min<u64>(std::min<u64>(remain, (u64)win * 4), gcap);
      e.ensure_nodes(wmax * R + 2, wmax * Kmax + 2);
      ensure_cand_bufs(e, B, gcap, R);
      CtaCtl c;
      memset(&c, 0, sizeof(c));
      c.p = p;
      c.P = P;
      c.win = std::min<u32>(win, gcap);
      c.epoch = B.epoch;
      c.jcursor = jcursor;
      c.jtotal = jtotal;
      c.jcomplete = jcomplete ? 1 : 0;
      c.reason = CR_DONE;
      *B.hctl = c;
      CUDA_OK(cudaMemcpyAsync(B.ctl.p, B.hctl, sizeof(c), cudaMemcpyHostToDevice, e.s));
      {
        KTimer kt(e, KG_APPLY_WAVE, 0.0, 1);
        grid_launch(e, B, ri, Rd, RD, skip_self, multi, n_max, B.ctl.p);
        CUDA_OK(cudaMemcpyAsync(B.hctl, B.ctl.p, sizeof(c), cudaMemcpyDeviceToHost, e.s));
        CUDA_OK(cudaMemcpyAsync(B.hcnt, e.cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, e.s));
        e.sync();
        c = *B.hctl;
        e.h = *B.hcnt;
        kt.bytes = wave_bytes(e, Rd, (double)c.s_cand, (double)c.s_req, (double)c.s_win, (double)c.s_nk);
      }
      if (dbg_waves)
        fprintf(stderr, "   gridloop: reason %u waves %u cand %llu resolved %u p %llu/%llu win %u | %.3f ms\n", c.reason,
                c.waves, c.s_cand, c.resolved, c.p, P, c.win,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count());
      if (cta_exit(e, B, ri, c, p, jcursor, win, jvalid, multi, filter_mode, allow_self, n_max)) break;
      continue;
    }
    e.phase_ms[8] += 1;  // waves
    // ---- candidates of a grid wave
    u32 ncand = 0;
    const unsigned long long* posp = nullptr;
    unsigned long long seg_end = P;  // positions covered if every candidate commits
    if (!multi) {
      unsigned long long n = std::min<unsigned long long>(P - p, win);
      ncand = (u32)n;
      seg_end = p + n;
    } else {
      u32 rem = jtotal - jcursor;
      ncand = std::min<u32>(rem, win);
      posp = B.pos.p + jcursor;
      if (ncand < rem) {
        // coverage ends right before the next cached candidate
        CUDA_OK(cudaMemcpyAsync(&seg_end, B.pos.p + jcursor + ncand, sizeof(seg_end), cudaMemcpyDeviceToHost, e.s));
        e.sync();
      } else if (!jcomplete) {
        CUDA_OK(cudaMemcpyAsync(&seg_end, B.pos.p + jtotal - 1, sizeof(seg_end), cudaMemcpyDeviceToHost, e.s));
        e.sync();
        seg_end += 1;
        jvalid = false;  // re-join after the capped list
      }
    }
    // ---- 2. gates + accepted list
    double dbg_ens = 0;
    unsigned long long dbg_al = g_dev_allocs;
    if (dbg_waves) {
      e.sync();
      dbg_ens = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count();
    }
    e.ensure_nodes((u64)ncand * R + 2, (u64)ncand * Kmax + 2);
    ensure_cand_bufs(e, B, ncand, R);
    if (dbg_waves) {
      e.sync();
      fprintf(stderr, "   grid: ensure %.3f ms (cap_nodes %u, %llu cudaMallocs)\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count() - dbg_ens,
              e.cap_nodes, g_dev_allocs - dbg_al);
    }
    WaveState* ws = B.ws.p;
    u64 nreq_max = (u64)ncand * R;
    WaveTab T{B.wminpos.p, B.wid.p, B.wroot.p, B.wval.p, B.wcap - 1, B.wold.p, ++B.epoch, B.wtag.p, B.wown.p};
    {
      KTimer kt(e, KG_APPLY_WAVE, 0.0, 16 + lv.size());
      k_gates<<<nblk(ncand, 128), 128, 0, e.s>>>(e.view(), Rd, RD, W, posp, ncand, p, B.status.p, B.env.p, B.olds.p,
                                                 B.hazard.p);
      if (ncand <= 65536) {  // the accepted-list variant replaces 5 launches
        k_accept_scan<<<1, 1024, 0, e.s>>>(B.status.p, B.hazard.p, ncand, B.pre.p, B.acc.p, ws);
      } else {
        k_accept_flags<<<nblk(ncand), 256, 0, e.s>>>(B.status.p, B.hazard.p, ncand, B.fl.p);
        CUDA_OK(cudaMemsetAsync(B.fl.p + ncand, 0, sizeof(u32), e.s));
        dev_exclusive_scan_u32(e, B.fl.p, B.pre.p, ncand + 1);
        k_accept_list<<<nblk(ncand), 256, 0, e.s>>>(B.fl.p, B.pre.p, ncand, B.acc.p);
        k_set_nacc<<<1, 1, 0, e.s>>>(B.pre.p, ncand, ws);
      }
      // ---- 3. resolve requests level by level
      if (R > 0) {
        for (size_t d = 1; d < lv.size(); d++) {
          int nl = (int)lv[d].size();
          if (!nl) continue;
          k_resolve_claim<<<nblk((u64)ncand * nl, 128), 128, 0, e.s>>>(e.view(), W, T, B.acc.p, ws,
                                                                      lvl_dev + lvl_off[d], nl, B.env.p, B.ident.p,
                                                                      B.hazard.p);
          k_resolve_verify<<<nblk((u64)ncand * nl, 128), 128, 0, e.s>>>(e.view(), W, T, B.acc.p, ws,
                                                                       lvl_dev + lvl_off[d], nl, B.env.p, B.ident.p,
                                                                       B.hazard.p);
        }
        k_mark_roots<<<nblk(ncand), 256, 0, e.s>>>(W, T, B.acc.p, ws, B.ident.p, B.hazard.p, B.olds.p);
      }
      k_cand_check<<<nblk(ncand), 256, 0, e.s>>>(e.view(), W, T, B.acc.p, ws, ncand, B.ident.p, B.env.p, B.olds.p,
                                                 multi ? 1 : 0, B.hazard.p, B.alloc.p, B.ukind.p, B.uother.p,
                                                 B.grow.p, B.sa.p, B.akid.p);
      // ---- 4. read/write conflicts, stop-after, node-limit cutoff, boundary
      CUDA_OK(cudaMemsetAsync(B.stops.p, 0xFF, 4 * sizeof(u32), e.s));
      {
        static int coop_blocks = 0;
        if (!coop_blocks) {
          int per_sm = 0, nsm = 0, dev = 0;
          CUDA_OK(cudaGetDevice(&dev));
          CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
          CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conflicts_grid, 256, 0));
          coop_blocks = std::max(1, std::min(per_sm, 4)) * nsm;
        }
        static const u32 max_it = getenv("TSAT_GRID_RESOLVE") ? (u32)atoi(getenv("TSAT_GRID_RESOLVE")) : 4u;
        u32 ep0 = ++B.epoch;
        B.epoch += max_it;
        G gv = e.view();
        const u32* accp = B.acc.p;
        u32 nc = ncand;
        u32* resp = B.stops.p + 4;
        void* args[] = {&gv,       &W,         &T,         &Rd,      &RD,      &accp,    &ws,
                        &nc,       &B.hazard.p, &B.env.p,  &B.olds.p, &B.pre.p, &B.status.p, &B.ident.p,
                        &B.ukind.p, &B.grow.p,  &B.uother.p, &B.fw_cls.p, &B.fw_fresh.p, &B.stops.p, &ep0,
                        (void*)&max_it, &resp};
        unsigned nb = (unsigned)std::min<u64>((u64)coop_blocks, std::max<u64>(1, ((u64)ncand + 255) / 256));
        CUDA_OK(cudaLaunchCooperativeKernel((const void*)k_conflicts_grid, nb, 256, args, 0, e.s));
      }
      if (ncand <= SCAN1_MAX) {
        k_scan_block<<<1, 1024, 0, e.s>>>(B.alloc.p, B.apre.p, ncand);
      } else {
        CUDA_OK(cudaMemsetAsync(B.alloc.p + ncand, 0, sizeof(u32), e.s));
        dev_exclusive_scan_u32(e, B.alloc.p, B.apre.p, ncand + 1);
      }
      k_find_stops<<<nblk(ncand), 256, 0, e.s>>>(B.acc.p, ws, B.sa.p, B.apre.p, B.alloc.p, e.cnt.p, n_max, B.stops.p);
      k_boundary<<<1, 1, 0, e.s>>>(ws, B.stops.p, ncand, posp, p, seg_end, B.pre.p, B.hazard.p);
      // ---- 5. statistics of the committed segment (device accumulators)
      k_seg_stats<<<nblk(ncand), 256, 0, e.s>>>(B.status.p, ws, ncand, B.pre.p, B.alloc.p, B.ukind.p, Rd.efficient,
                                                B.ws_cur, Rd, p, posp);
      // ---- 6. commit
      if (nreq_max) {
        k_win_flags<<<nblk(nreq_max), 256, 0, e.s>>>(T, B.ident.p, nreq_max, W.tmpl, R, ws, B.wf.p, B.ka.p);
        if (nreq_max <= SCAN1_MAX) {
          k_scan_block<<<1, 1024, 0, e.s>>>(B.wf.p, B.wpre.p, (u32)nreq_max);
          k_scan_block<<<1, 1024, 0, e.s>>>(B.ka.p, B.kpre.p, (u32)nreq_max);
        } else {
          CUDA_OK(cudaMemsetAsync(B.wf.p + nreq_max, 0, sizeof(u32), e.s));
          CUDA_OK(cudaMemsetAsync(B.ka.p + nreq_max, 0, sizeof(u32), e.s));
          dev_exclusive_scan_u32(e, B.wf.p, B.wpre.p, (u32)nreq_max + 1);
          dev_exclusive_scan_u32(e, B.ka.p, B.kpre.p, (u32)nreq_max + 1);
        }
        k_commit_prep<<<1, 1, 0, e.s>>>(ws, B.wpre.p, B.kpre.p, nreq_max, e.cnt.p);
        k_assign_ids<<<nblk(nreq_max), 256, 0, e.s>>>(T, B.ident.p, nreq_max, B.wf.p, B.wpre.p, ws);
        k_write_nodes<<<nblk(nreq_max), 256, 0, e.s>>>(e.view(), W, T, B.acc.p, B.ident.p, nreq_max, B.wf.p, B.wpre.p,
                                                       B.kpre.p, ws, B.env.p, B.olds.p);
      } else {
        k_zero_commit<<<1, 1, 0, e.s>>>(ws, e.cnt.p);
      }
      k_commit_unions<<<nblk(ncand), 256, 0, e.s>>>(e.view(), W, T, B.acc.p, ws, B.olds.p, B.ukind.p, B.uother.p,
                                                    B.grow.p);
      if (nreq_max) k_insert_range<<<nblk(nreq_max), 256, 0, e.s>>>(e.view(), ws, nreq_max);
      k_counters_commit<<<1, 1, 0, e.s>>>(ws, e.cnt.p);
    }
    WaveState hw;
    CUDA_OK(cudaMemcpyAsync(&hw, ws, sizeof(hw), cudaMemcpyDeviceToHost, e.s));
    CUDA_OK(cudaMemcpyAsync(&e.h, e.cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, e.s));
    e.sync();
    e.kstat[KG_APPLY_WAVE].bytes += wave_bytes(e, Rd, ncand, (double)hw.nacc * R, hw.nwin, hw.nk);
    u32 ncommit_cand = hw.ncommit_cand;
    unsigned long long p_end = hw.p_end;
    if (dbg_waves)
      fprintf(stderr, "   grid: ncand %u nacc %u commit %u why %u p %llu/%llu | %.3f ms\n", ncand, hw.nacc,
              hw.ncommit_cand, hw.why, p_end, P,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count());
    bool stop = hw.stop != 0, hazard = hw.hazard != 0;
    if (hw.ncommit_cand < ncand && !stop) e.phase_ms[10 + std::min<int>(hw.why, 5)] += 1;
    {
      unsigned long long cover = p_end - p, self = skip_self ? self_in_host(Rd.nmatch[0], Rd.nmatch[1], p, p_end) : 0;
      rs.found += cover;
      rs.skipped_self += self;
      rs.skipped_compat += cover - self - ncommit_cand;
    }
    if (multi) {
      jcursor += ncommit_cand;
      // a union of existing classes (stop-after) or an exact-path combo can change compatibility
      if (hazard || hw.sa_hit) jvalid = false;
    }
    if (stop) {
      if (p_end < P) {
        e.seq_stop = true;
        e.report.node_limit_overshoot = (i64)e.h.live - n_max;
      }
      p = p_end;
      if (e.seq_stop) break;
      continue;
    }
    // adapt the window: dependencies every k combos -> evaluate ~2k ahead
    if (ncommit_cand < ncand) win = std::max<u32>(64u, std::min<u32>(2u * ncommit_cand + 32u, wave_win_max()));
    else win = std::min<u32>(win * wave_grow(), wave_win_max());
    if (hazard) {
      e.phase_ms[9] += 1;  // hazards
      // exact sequential path for exactly the hazard combo
      e.ensure_nodes(4096, 4096);
      e.run_rule_seq(ri, filter_mode, allow_self, n_max, p_end, p_end + 1);
      if (e.seq_stop) break;
      p = p_end + 1;
      continue;
    }
    p = p_end;
  }
  if (defer) return;  // read with the iteration's other rules (flush_wave_stats)
  DevStats d;
  u32 gres = 0;
  CUDA_OK(cudaMemcpyAsync(&d, B.ws_cur, sizeof(d), cudaMemcpyDeviceToHost, e.s));
  CUDA_OK(cudaMemcpyAsync(&gres, B.stops.p + 4, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  e.sync();
  e.phase_ms[29] += gres;
  accumulate_seg(e, ri, d);
  if (rec) {
    e.rej_pending = nullptr;
    const u32 nw = std::min<u32>(d.nrej, rej_cap);
    std::vector<u32> lg(2 * (size_t)nw);
    if (nw) {
      CUDA_OK(cudaMemcpyAsync(lg.data(), e.sc.v_rej_w.p, lg.size() * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
      e.sync();
    }
    for (u32 k = 0; k < nw; k++) rej_seq.push_back(((unsigned long long)lg[2 * k] << 32) | lg[2 * k + 1]);
    std::sort(rej_seq.begin(), rej_seq.end());
    for (unsigned long long q : rej_seq) e.record_reject(ri, q);
  }
  if (dbg_waves)
    fprintf(stderr, "rule %d %s P=%llu waves=%.0f cuts=%.0f applied=%llu live=%u %.3f ms\n", ri,
            ri < (int)e.rule_names.size() ? e.rule_names[ri].c_str() : "?", P, e.phase_ms[8] - dbg_w0,
            e.phase_ms[10] - dbg_c0, (unsigned long long)d.applied, e.h.live,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0).count());
#ifdef WAVE_DBG
  if (getenv("TSAT_DEBUG_WAVES")) {
    unsigned long long cnt[32];
    CUDA_OK(cudaMemcpyFromSymbol(cnt, g_wdbg_cnt, sizeof(cnt)));
    fprintf(stderr, "  bad-read categories:");
    for (int i = 0; i < 32; i++)
      if (cnt[i]) fprintf(stderr, " %d:%llu", i, cnt[i]);
    fprintf(stderr, "\n");
  }
#endif
}

// A run of consecutive single-source rules, each launched as one single-CTA
// run of waves without a host round trip in between: the launches are queued
// back to back, each continuing the previous one's wave epoch, and a launch
// whose predecessor did not finish its rule (hazard, node limit, capacity,
// wide windows) does nothing (CR_NOTRUN).  One read-back after the run: the
// finished rules are accounted exactly like their own loop would; the first
// unfinished one resumes in run_rule_wave from its control block, and the
// rest of the run is chained again.  Same sequence of device work as the
// per-rule loop, minus ~10 host <-> device operations and 2 syncs per rule.
void run_rules_chain(Engine& e, const std::vector<int>& rules, const std::vector<unsigned long long>& Ps,
                     int filter_mode, int allow_self, i64 n_max) {
  const size_t K = rules.size();
  if (!K) return;
  if ((i64)e.h.live >= n_max) {
    e.seq_stop = true;
    e.report.node_limit_overshoot = (i64)e.h.live - n_max;
    return;
  }
  if (!e.wave) e.wave = new WaveBufs();
  WaveBufs& B = *e.wave;
  ensure_wave_templates(e, B);
  if (B.chain_cap < K) {
    if (B.hchain) cudaFreeHost(B.hchain);
    CUDA_OK(cudaMallocHost((void**)&B.hchain, K * (sizeof(CtaCtl) + sizeof(DevStats))));
    B.chain_ctl.alloc(K);
    B.chain_stats.alloc(K);
    B.chain_cap = K;
  }
  CtaCtl* hc = B.hchain;
  DevStats* hs = (DevStats*)(B.hchain + K);
  int maxR = 0, maxK = 0;
  for (int ri : rules) {
    if (B.rw[ri].lv.size() > 12)
      throw TsatException(TSAT_ERR_UNSUPPORTED, "target deeper than the wave engine supports");
    maxR = std::max(maxR, B.rw[ri].R);
    maxK = std::max(maxK, B.rw[ri].Kmax);
  }
  e.ensure_nodes((u64)CTA_WIN * maxR + 2, (u64)CTA_WIN * maxK + 2);
  ensure_cand_bufs(e, B, CTA_WIN, maxR);
  static const u32 win0 = getenv("TSAT_WIN0") ? (u32)atoi(getenv("TSAT_WIN0")) : (1u << 14);
  for (size_t k = 0; k < K; k++) {
    CtaCtl& c = hc[k];
    memset(&c, 0, sizeof(c));
    c.P = Ps[k];
    c.win = std::min<u32>(win0, CTA_WIN);
    c.epoch = B.epoch;
    c.jcomplete = 1;
    c.reason = CR_DONE;
    cta_fit_window(c, B.rw[rules[k]].R);
  }
  CUDA_OK(cudaMemcpyAsync(B.chain_ctl.p, hc, K * sizeof(CtaCtl), cudaMemcpyHostToDevice, e.s));
  CUDA_OK(cudaMemsetAsync(B.chain_stats.p, 0, K * sizeof(DevStats), e.s));
  {
    KTimer kt(e, KG_APPLY_WAVE, 0.0, K);
    for (size_t k = 0; k < K; k++) {
      const int ri = rules[k];
      RuleDev Rd = make_rule_dev(e, ri, filter_mode, allow_self);
      ReachDev RD = make_reach_dev(e);
      cta_launch(e, B, ri, Rd, RD, 0, false, n_max, B.chain_ctl.p + k, k ? B.chain_ctl.p + k - 1 : nullptr,
                 B.chain_stats.p + k);
    }
  }
  CUDA_OK(cudaMemcpyAsync(hc, B.chain_ctl.p, K * sizeof(CtaCtl), cudaMemcpyDeviceToHost, e.s));
  CUDA_OK(cudaMemcpyAsync(hs, B.chain_stats.p, K * sizeof(DevStats), cudaMemcpyDeviceToHost, e.s));
  CUDA_OK(cudaMemcpyAsync(&e.h, e.cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, e.s));
  e.sync();
  for (size_t k = 0; k < K; k++) {
    const int ri = rules[k];
    const CtaCtl c = hc[k];
    if (c.reason == CR_NOTRUN) {
      // an earlier rule returned to the host and was finished there: chain the rest again
      std::vector<int> rest(rules.begin() + k, rules.end());
      std::vector<unsigned long long> restP(Ps.begin() + k, Ps.end());
      run_rules_chain(e, rest, restP, filter_mode, allow_self, n_max);
      return;
    }
    {
      RuleDev Rd = make_rule_dev(e, ri, filter_mode, allow_self);
      e.kstat[KG_APPLY_WAVE].bytes +=
          wave_bytes(e, Rd, (double)c.s_cand, (double)c.s_req, (double)c.s_win, (double)c.s_nk);
    }
    if (c.reason == CR_DONE && c.p >= c.P) {
      unsigned long long p = 0;
      u32 jc = 0, win = 0;
      bool jv = false;
      cta_exit(e, B, ri, c, p, jc, win, jv, false, filter_mode, allow_self, n_max);
      accumulate_seg(e, ri, hs[k]);
      continue;
    }
    e.uf_changed = true;
    run_rule_wave(e, ri, filter_mode, allow_self, n_max, c.P, &c, &hs[k]);
    if (e.seq_stop || e.seq_timeout) return;
    // the launches after k were skipped (CR_NOTRUN): continue with k + 1
    std::vector<int> rest(rules.begin() + k + 1, rules.end());
    std::vector<unsigned long long> restP(Ps.begin() + k + 1, Ps.end());
    run_rules_chain(e, rest, restP, filter_mode, allow_self, n_max);
    return;
  }
}

// saturate's rule loop defers each wave rule's statistics to one read-back
// per iteration (begin: slots for every rule; flush: read them, accumulate in
// rule order -- the counters are sums, so the order does not matter)
void begin_wave_stats(Engine& e) {
  if (!e.wave) e.wave = new WaveBufs();
  WaveBufs& B = *e.wave;
  B.wstats_def.ensure(2 * e.rules.size() + 2);
  B.def_ri.clear();
  B.def_pending = false;
  B.stops.ensure(6);
  CUDA_OK(cudaMemsetAsync(B.stops.p + 4, 0, sizeof(u32), e.s));
  e.defer_wave_stats = true;
}

// flush in two halves: the read-back is queued (pinned host memory) and
// lands with the rebuild's own read-back; finish accumulates it afterwards
void flush_wave_stats_begin(Engine& e) {
  e.defer_wave_stats = false;
  if (!e.wave) return;
  WaveBufs& B = *e.wave;
  const size_t k = B.def_ri.size();
  if (!k) return;
  if (B.hdef_cap < k + 1) {
    if (B.hdef) cudaFreeHost(B.hdef);
    CUDA_OK(cudaMallocHost((void**)&B.hdef, (k + 1) * sizeof(DevStats)));
    B.hdef_cap = k + 1;
  }
  CUDA_OK(cudaMemcpyAsync(B.hdef, B.wstats_def.p, k * sizeof(DevStats), cudaMemcpyDeviceToHost, e.s));
  CUDA_OK(cudaMemcpyAsync(&B.hdef[k].nrej, B.stops.p + 4, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  B.def_pending = true;
}

void flush_wave_stats_finish(Engine& e) {
  if (!e.wave) return;
  WaveBufs& B = *e.wave;
  if (!B.def_pending) return;
  e.sync();  // normally already passed by the rebuild's read-back
  const size_t k = B.def_ri.size();
  e.phase_ms[29] += B.hdef[k].nrej;  // grid-wave soft writers resolved (carried in a spare slot)
  for (size_t i = 0; i < k; i++) accumulate_seg(e, B.def_ri[i], B.hdef[i]);
  B.def_ri.clear();
  B.def_pending = false;
}
