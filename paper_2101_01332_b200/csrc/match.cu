// E-matching on the GPU (reference: pkg/src/tensorsat/egraph.py:248-293).
//
// All unique canonical patterns of an iteration are matched in ONE batch.
// The root candidates of every pattern form one flat list: pattern p scans
// the per-operator table of its root atom (snapshot.op_nodes, stored in
// (op, class, id) order).  Nested pattern nodes are joined through the class
// CSR (class -> members, ascending ids) with filter-list, op and arity checks
// and nonlinear-variable equality.
//
//   count   one thread per candidate: number of matches (DFS over the join)
//   scan    per-candidate output offsets (one pass for the whole batch)
//   emit    the same DFS writes rows (eclass, bindings in var-name order) at
//           the candidate's offset -- rows come out grouped by eclass, with
//           eclasses ascending, because candidates are class-ordered
//   rank    rows of one eclass are ordered by bindings and deduplicated
//           (_match_sorted, egraph.py:107-112): small groups (<= 32 rows,
//           the common case) by a per-row rank, larger groups by one CTA each
//   compact keep first-of-equal rows, write each pattern's MatchSet
//
// Two host synchronisations per batch (row counts, unique counts).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>

#include "engine.cuh"

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

struct PatDev {
  PatApp apps[MAX_PAT_APPS];
  // semi-join filter per nested app (i >= 1): bit c set iff class c holds a
  // live, unfiltered node with apps[i]'s operator (bitmap over class ids,
  // L2-resident: n_alloc / 8 bytes per operator); null = no filter
  const u32* bm[MAX_PAT_APPS];
  int napps;
  int nb;
  int order[MAX_VARS];
  // single-app patterns (the common case): binding k = root child src[k];
  // children eq[i][0] and eq[i][1] must be the same class (repeated variable)
  int8_t src[MAX_VARS];
  int8_t fast;  // the single-app plan below is valid
  int8_t neq;
  int8_t eq[8][2];
};

struct SnapDev {
  const u32* cls_index;
  const u32* cls_off;
  const u32* cls_nodes;
  const u32* op_nodes;
  u32 n_alloc;
  int clean;  // no union since the last rebuild: stored children are canonical, no find needed
};

__device__ __forceinline__ u32 kid_cls(const G& g, const SnapDev& sd, u32 k) {
  return sd.clean ? k : uf_find_ro(g.parent, k);
}

__device__ __forceinline__ bool bm_has(const u32* bm, u32 c) { return !bm || ((bm[c >> 5] >> (c & 31)) & 1u); }

#define MAX_BATCH 24
#define SMALL_GROUP 32u

struct Batch {
  int npat;
  int stride;                 // words per binding row (max nb of the batch, >= 1)
  PatDev pat[MAX_BATCH];
  u32 cbase[MAX_BATCH + 1];   // flat candidate ranges
  u32 obase[MAX_BATCH];       // op_nodes offset of each pattern's root atom
  u32 rbase[MAX_BATCH + 1];   // raw row ranges (after the count scan)
  u32* out_cls[MAX_BATCH];
  u32* out_bind[MAX_BATCH];
  // root-operator groups: patterns [gp[g], gp[g+1]) share a root atom (and
  // so a candidate range); the count pass reads each candidate node once for
  // the whole group.  gbase: flat ranges of group candidates.
  int ngrp;
  int gp[MAX_BATCH + 1];
  u32 gbase[MAX_BATCH + 1];
};

__device__ __forceinline__ int seg_of(const u32* base, int n, u32 t) {
  int lo = 0, hi = n;  // largest p with base[p] <= t
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (base[mid] <= t) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool node_ok(const G& g, u32 nid, const PatApp& a) {
  if (g.flags[nid] & NF_FILT) return false;
  if (g.op[nid] != a.atom) return false;
  return (int)(g.koff[nid + 1] - g.koff[nid]) == a.nargs;
}

// bind the variable children of app t for node nid; set classes of app
// children (rejecting the node when such a class has no node of the child
// app's operator: the semi-join filter)
__device__ __forceinline__ bool bind_node(const G& g, const SnapDev& sd, const PatDev& p, const PatApp& a, u32 nid,
                                          int t, u32* env, int8_t* bound_at, u32* cls_app) {
  u32 base = g.koff[nid];
  for (int j = 0; j < a.nargs; j++) {
    u32 ch = kid_cls(g, sd, g.kids[base + j]);
    int c = a.child[j];
    if (c >= 0) {
      if (!bm_has(p.bm[c], ch)) return false;
      cls_app[c] = ch;
    } else {
      int v = -c - 1;
      if (env[v] == TSAT_NONE) {
        env[v] = ch;
        bound_at[v] = (int8_t)t;
      } else if (env[v] != ch) {
        return false;
      }
    }
  }
  return true;
}

template <int MV>
__device__ __forceinline__ void unbind(int t, u32* env, int8_t* bound_at) {
  for (int v = 0; v < MV; v++)
    if (bound_at[v] == t) {
      bound_at[v] = -1;
      env[v] = TSAT_NONE;
    }
}

__device__ __forceinline__ u32 sel8(const u32* kc, int i) {
  // register select (no local-memory indexing)
  u32 v = kc[0];
#pragma unroll
  for (int j = 1; j < 8; j++) v = i == j ? kc[j] : v;
  return v;
}

// single-app pattern: at most one match per root, state in registers.
// Counting (EMIT = false) of a pattern without repeated variables only needs
// the root's op / arity / filter flag.
template <bool EMIT, class F>
__device__ __forceinline__ u32 match_root1(const G& g, const SnapDev& sd, const PatDev& p, u32 r, F emit) {
  const PatApp& a = p.apps[0];
  if (!node_ok(g, r, a)) return 0;
  if (!EMIT && p.neq == 0) return 1;
  u32 base = g.koff[r];
  u32 kc[8];
#pragma unroll
  for (int j = 0; j < 8; j++) kc[j] = j < a.nargs ? kid_cls(g, sd, g.kids[base + j]) : 0u;
  for (int i = 0; i < p.neq; i++)
    if (sel8(kc, p.eq[i][0]) != sel8(kc, p.eq[i][1])) return 0;
  if (EMIT) emit(uf_find_ro(g.parent, r), kc);
  return 1;
}

// semi-join pre-check of a root candidate, in registers: every app child of
// the root must be a class holding its operator.  Most candidates of nested
// patterns fail here, before any DFS state (local memory) is touched.
__device__ __forceinline__ bool root_semijoin(const G& g, const SnapDev& sd, const PatDev& p, u32 r) {
  const PatApp& a = p.apps[0];
  u32 base = g.koff[r];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    if (j >= a.nargs) break;
    int c = a.child[j];
    if (c >= 0 && p.bm[c] && !bm_has(p.bm[c], kid_cls(g, sd, g.kids[base + j]))) return false;
  }
  return true;
}

// DFS over the pattern's join for root node r; emit(k, rc, env) per match.
template <int MV, int MA, class F>
__device__ __forceinline__ u32 match_root(const G& g, const SnapDev& sd, const PatDev& p, u32 r, F emit) {
  if (!node_ok(g, r, p.apps[0]) || !root_semijoin(g, sd, p, r)) return 0;
  u32 env[MV];
  int8_t bound_at[MV];
  u32 cls_app[MA];
  u32 pos[MA], end[MA];
  for (int v = 0; v < MV; v++) {
    env[v] = TSAT_NONE;
    bound_at[v] = -1;
  }
  if (!bind_node(g, sd, p, p.apps[0], r, 0, env, bound_at, cls_app)) return 0;
  u32 rc = uf_find_ro(g.parent, r);
  u32 count = 0;
  int level = 1;
  bool init = true;
  while (true) {
    if (level == p.napps) {
      emit(count, rc, env);
      count++;
      level--;
      if (level == 0) break;
      unbind<MV>(level, env, bound_at);
      init = false;
      continue;
    }
    if (init) {
      u32 c = cls_app[level];
      u32 d = c < sd.n_alloc ? sd.cls_index[c] : TSAT_NONE;
      if (d == TSAT_NONE) {
        pos[level] = end[level] = 0;
      } else {
        pos[level] = sd.cls_off[d];
        end[level] = sd.cls_off[d + 1];
      }
    }
    bool found = false;
    const PatApp& a = p.apps[level];
    while (pos[level] < end[level]) {
      u32 m = sd.cls_nodes[pos[level]++];
      if (!node_ok(g, m, a)) continue;
      if (bind_node(g, sd, p, a, m, level, env, bound_at, cls_app)) {
        found = true;
        break;
      }
      unbind<MV>(level, env, bound_at);
    }
    if (found) {
      level++;
      init = true;
    } else {
      level--;
      if (level == 0) break;
      unbind<MV>(level, env, bound_at);
      init = false;
    }
  }
  return count;
}

#define EM_HEAVY 0xFFFFFFFFu
#define EM_HEAVY_L1 8u  // measured flat between 4 and 16 on BERT (TSAT_EM_CUT)

// match_root restricted to part of the level-1 members: the members at
// positions l1_first, l1_first + l1_stride, ... of apps[1]'s class, at most
// l1_lim of them (DFS order within the part unchanged).  *l1_size receives
// the class size (1 for single-app patterns, whose only part is part 0).
template <int MV, int MA, class F>
__device__ __forceinline__ u32 match_root_part(const G& g, const SnapDev& sd, const PatDev& p, u32 r, u32 l1_first,
                                               u32 l1_stride, u32 l1_lim, u32* l1_size, F emit,
                                               u32 heavy_cut = 0xFFFFFFFFu) {
  *l1_size = 0;
  if (!node_ok(g, r, p.apps[0]) || !root_semijoin(g, sd, p, r)) return 0;
  u32 env[MV];
  int8_t bound_at[MV];
  u32 cls_app[MA];
  u32 pos[MA], end[MA];
  for (int v = 0; v < MV; v++) {
    env[v] = TSAT_NONE;
    bound_at[v] = -1;
  }
  if (!bind_node(g, sd, p, p.apps[0], r, 0, env, bound_at, cls_app)) return 0;
  u32 rc = uf_find_ro(g.parent, r);
  if (p.napps == 1) {
    *l1_size = 1;
    if (l1_first != 0) return 0;
    emit(0u, rc, env);
    return 1;
  }
  u32 count = 0, taken1 = 0;
  int level = 1;
  bool init = true;
  while (true) {
    if (level == p.napps) {
      emit(count, rc, env);
      count++;
      level--;
      unbind<MV>(level, env, bound_at);
      init = false;
      continue;
    }
    if (init) {
      u32 c = cls_app[level];
      u32 d = c < sd.n_alloc ? sd.cls_index[c] : TSAT_NONE;
      if (d == TSAT_NONE) {
        pos[level] = end[level] = 0;
      } else {
        pos[level] = sd.cls_off[d];
        end[level] = sd.cls_off[d + 1];
      }
      if (level == 1) {
        *l1_size = end[1] - pos[1];
        if (*l1_size > heavy_cut) return EM_HEAVY;  // before any emit: the caller hands it to a warp
        pos[1] += l1_first;
      }
    }
    bool found = false;
    const PatApp& a = p.apps[level];
    while (pos[level] < end[level]) {
      u32 m;
      if (level == 1) {
        if (taken1 >= l1_lim) {
          pos[1] = end[1];
          break;
        }
        m = sd.cls_nodes[pos[1]];
        pos[1] += l1_stride;
        taken1++;
      } else {
        m = sd.cls_nodes[pos[level]++];
      }
      if (!node_ok(g, m, a)) continue;
      if (bind_node(g, sd, p, a, m, level, env, bound_at, cls_app)) {
        found = true;
        break;
      }
      unbind<MV>(level, env, bound_at);
    }
    if (found) {
      level++;
      init = true;
    } else {
      level--;
      if (level == 0) break;
      unbind<MV>(level, env, bound_at);
      init = false;
    }
  }
  return count;
}

// Nested patterns, one warp per root candidate: the lanes split the members
// of apps[1]'s class (large classes of commuted / reassociated forms made one
// thread's DFS hold its whole warp).  Fast (single-app) patterns stay on the
// thread-per-candidate kernels.
template <int MV, int MA>
__global__ void k_em_count_w(G g, SnapDev sd, Batch B, const u32* heavy, const u32* nheavy, u32* cnt) {
  const u32 lane = threadIdx.x & 31;
  const u64 w0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u32 nh = *nheavy;
  for (u64 i = w0; i < nh; i += nw) {
    const u32 t = heavy[i];
    int p = seg_of(B.cbase, B.npat, t);
    const PatDev& pd = B.pat[p];
    u32 r = sd.op_nodes[B.obase[p] + (t - B.cbase[p])];
    u32 sz;
    u32 c = match_root_part<MV, MA>(g, sd, pd, r, lane, 32u, 0xFFFFFFFFu, &sz, [](u32, u32, const u32*) {});
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[t] = c;
  }
}

template <int MV, int MA>
__global__ void k_em_emit_w(G g, SnapDev sd, Batch B, const u32* heavy, const u32* nheavy, const u32* off, u32* rc,
                            u32* rb) {
  const u32 lane = threadIdx.x & 31;
  const u64 w0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const int S = B.stride;
  const u32 nh = *nheavy;
  for (u64 i = w0; i < nh; i += nw) {
    const u32 t = heavy[i];
    int p = seg_of(B.cbase, B.npat, t);
    const PatDev& pd = B.pat[p];
    u32 r = sd.op_nodes[B.obase[p] + (t - B.cbase[p])];
    u32 o = off[t];
    u32 sz = 0;
    match_root_part<MV, MA>(g, sd, pd, r, 0xFFFFFFFFu, 1u, 0u, &sz, [](u32, u32, const u32*) {});
    // sz: apps[1]'s class size (or 1); members in chunks of 32, one per lane
    for (u32 c0 = 0; c0 < sz; c0 += 32) {
      u32 mine = 0, dummy;
      if (c0 + lane < sz)
        mine = match_root_part<MV, MA>(g, sd, pd, r, c0 + lane, 1u, 1u, &dummy, [](u32, u32, const u32*) {});
      u32 inc = mine;
      for (int d = 1; d < 32; d <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (u32)d) inc += y;
      }
      u32 tot = __shfl_sync(0xffffffffu, inc, 31);
      u32 base = o + inc - mine;
      if (mine)
        match_root_part<MV, MA>(g, sd, pd, r, c0 + lane, 1u, 1u, &dummy, [&](u32 k, u32 cls, const u32* env) {
          rc[base + k] = cls;
          for (int j = 0; j < S; j++) rb[(u64)(base + k) * S + j] = j < pd.nb ? env[pd.order[j]] : 0u;
        });
      o += tot;
    }
  }
}

// MV / MA: DFS state sizes (small instantiation keeps the state in few
// registers + little local memory; the large one covers any loadable pattern)
template <int MV, int MA>
__global__ void k_em_count(G g, SnapDev sd, Batch B, u32 ntot, u32* cnt, u32* heavy, u32* nheavy, u32 cut) {
  GRID_STRIDE(t0, (u64)B.gbase[B.ngrp]) {
    int gi = seg_of(B.gbase, B.ngrp, (u32)t0);
    u32 k = (u32)t0 - B.gbase[gi];
    u32 r = sd.op_nodes[B.obase[B.gp[gi]] + k];
    // one candidate node, every pattern rooted at its operator (the node's
    // record is read from DRAM once, then from L1)
    for (int p = B.gp[gi]; p < B.gp[gi + 1]; p++) {
      const u32 t = B.cbase[p] + k;
      const PatDev& pd = B.pat[p];
      if (!pd.fast && heavy) {
        // nested pattern: a candidate whose apps[1] class is large goes to a warp (k_em_count_w)
        u32 sz;
        u32 c = match_root_part<MV, MA>(g, sd, pd, r, 0u, 1u, 0xFFFFFFFFu, &sz, [](u32, u32, const u32*) {}, cut);
        if (c == EM_HEAVY) heavy[atomicAdd(nheavy, 1u)] = t;
        else cnt[t] = c;
        continue;
      }
      cnt[t] = pd.fast ? match_root1<false>(g, sd, pd, r, [](u32, const u32*) {})
                       : match_root<MV, MA>(g, sd, pd, r, [](u32, u32, const u32*) {});
    }
  }
}

template <int MV, int MA>
__global__ void k_em_emit(G g, SnapDev sd, Batch B, u32 ntot, const u32* off, u32* rc, u32* rb, int split, u32 cut) {
  GRID_STRIDE(t, ntot) {
    int p = seg_of(B.cbase, B.npat, (u32)t);
    const PatDev& pd = B.pat[p];
    u32 r = sd.op_nodes[B.obase[p] + ((u32)t - B.cbase[p])];

    u32 o = off[t];
    if (off[t + 1] == o) continue;  // no match (the count pass decided)
    const int S = B.stride;
    if (pd.fast) {
      match_root1<true>(g, sd, pd, r, [&](u32 cls, const u32* kc) {
        rc[o] = cls;
        for (int j = 0; j < S; j++) rb[(u64)o * S + j] = j < pd.nb ? sel8(kc, pd.src[j]) : 0u;
      });
      continue;
    }
    auto put = [&](u32 k, u32 cls, const u32* env) {
      rc[o + k] = cls;
      for (int j = 0; j < S; j++) rb[(u64)(o + k) * S + j] = j < pd.nb ? env[pd.order[j]] : 0u;
    };
    if (split) {
      u32 sz;  // heavy candidates (large apps[1] class) are emitted by k_em_emit_w
      match_root_part<MV, MA>(g, sd, pd, r, 0u, 1u, 0xFFFFFFFFu, &sz, put, cut);
    } else {
      match_root<MV, MA>(g, sd, pd, r, put);
    }
  }
}

// Semi-join reduction of the pattern trees (bottom-up, one launch per app
// height): bitmap (p, i) over class ids marks the classes holding a live,
// unfiltered node that matches pattern p's sub-pattern at app i ignoring
// repeated-variable equalities -- operator, arity, and every app child's
// class marked in that child's bitmap.  A root candidate then survives only
// if each app child's class is marked: the join runs on L2-resident bitmaps
// instead of chasing class members (a necessary condition, so the DFS that
// follows stays the exact matcher).
struct SemiJob {
  u32 lo, hi;      // op-table range of the app's operator
  u32 out;         // bitmap index
  int nargs;
  int child[8];    // bitmap index of an app child, -1 for a variable
};
#define SEMI_MAX 64
struct SemiJobs {
  int n;
  u32 base[SEMI_MAX + 1];
  SemiJob job[SEMI_MAX];
};

__global__ void k_em_semijoin(G g, SnapDev sd, SemiJobs J, u32* pool, u64 words) {
  GRID_STRIDE(t, (u64)J.base[J.n]) {
    int q = seg_of(J.base, J.n, (u32)t);
    const SemiJob& jb = J.job[q];
    u32 x = sd.op_nodes[jb.lo + ((u32)t - J.base[q])];
    if (g.flags[x] & NF_FILT) continue;
    u32 a = g.koff[x];
    if ((int)(g.koff[x + 1] - a) != jb.nargs) continue;
    bool ok = true;
    for (int j = 0; j < jb.nargs && ok; j++) {
      int c = jb.child[j];
      if (c < 0) continue;
      u32 k = kid_cls(g, sd, g.kids[a + j]);
      ok = (pool[(u64)c * words + (k >> 5)] >> (k & 31)) & 1u;
    }
    if (!ok) continue;
    u32 cls = uf_find_ro(g.parent, x);
    atomicOr(&pool[(u64)jb.out * words + (cls >> 5)], 1u << (cls & 31));
  }
}

__global__ void k_em_bounds(const u32* off, Batch B, u32* out) {
  int p = threadIdx.x;
  if (p <= B.npat) out[p] = off[B.cbase[p]];
}

// row a < row b within one eclass group: bindings lexicographic, ties by index
__device__ __forceinline__ int row_cmp(const u32* rb, int S, int nb, u32 a, u32 b) {
  for (int j = 0; j < nb; j++) {
    u32 x = rb[(u64)a * S + j], y = rb[(u64)b * S + j];
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}

__device__ __forceinline__ void put_row(const u32* rc, const u32* rb, int S, int nb, u32 src, u32 dst, u32* sc,
                                        u32* sb) {
  sc[dst] = rc[src];
  for (int j = 0; j < nb; j++) sb[(u64)dst * S + j] = rb[(u64)src * S + j];
}

// small groups: per-row rank + scatter; rows of larger groups are flagged
// (big[k] = 1, head[k] = first row of its group) for the radix path
__global__ void k_em_rank(Batch B, u32 nrows, const u32* rc, const u32* rb, u32* sc, u32* sb, u32* big,
                          u32* head) {
  GRID_STRIDE(k0, nrows) {
    u32 k = (u32)k0;
    int p = seg_of(B.rbase, B.npat, k);
    u32 lo = B.rbase[p], hi = B.rbase[p + 1];
    u32 c = rc[k];
    u32 gs = k, ge = k + 1;
    while (gs > lo && rc[gs - 1] == c && k - gs < SMALL_GROUP) gs--;
    while (ge < hi && rc[ge] == c && ge - k <= SMALL_GROUP) ge++;
    bool is_big = ge - gs > SMALL_GROUP || (gs > lo && rc[gs - 1] == c);
    big[k] = is_big ? 1u : 0u;
    head[k] = (k == lo || rc[k - 1] != c) ? 1u : 0u;
    if (is_big) continue;
    const int nb = B.pat[p].nb, S = B.stride;
    u32 rank = 0;
    for (u32 j = gs; j < ge; j++) {
      if (j == k) continue;
      int cmp = row_cmp(rb, S, nb, j, k);
      if (cmp < 0 || (cmp == 0 && j < k)) rank++;
    }
    put_row(rc, rb, S, nb, k, gs + rank, sc, sb);
  }
}

// big rows, ascending: L[i] = row, bh[i] = group head flag, perm = identity
__global__ void k_em_big_list(u32 nrows, const u32* big, const u32* bpos, const u32* head, u32* L, u32* bh,
                              u32* perm) {
  GRID_STRIDE(k, nrows) {
    if (!big[k]) continue;
    u32 i = bpos[k];
    L[i] = (u32)k;
    bh[i] = head[k];
    perm[i] = i;
  }
}

// radix key of pass w (binding word w, or the group index when w < 0)
__global__ void k_em_big_key(u32 nbig, const u32* L, const u32* perm, const u32* rb, int S, int w, const u32* bh,
                             const u32* gex, u32* key) {
  GRID_STRIDE(i, nbig) {
    u32 q = perm[i];
    key[i] = w >= 0 ? rb[(u64)L[q] * S + w] : gex[q] + bh[q] - 1;
  }
}

// sorted big rows go to the big-row slots in ascending order (groups keep
// their positions and sizes)
__global__ void k_em_big_scatter(u32 nbig, const u32* L, const u32* perm, const u32* rc, const u32* rb, int S,
                                 u32* sc, u32* sb) {
  GRID_STRIDE(i, nbig) put_row(rc, rb, S, S, L[perm[i]], L[i], sc, sb);
}

__global__ void k_em_keep(Batch B, u32 nrows, const u32* sc, const u32* sb, u32* keep) {
  GRID_STRIDE(k0, nrows) {
    u32 k = (u32)k0;
    int p = seg_of(B.rbase, B.npat, k);
    bool kp = k == B.rbase[p] || sc[k] != sc[k - 1] || row_cmp(sb, B.stride, B.pat[p].nb, k - 1, k) != 0;
    keep[k] = kp ? 1u : 0u;
  }
}

__global__ void k_em_compact(Batch B, u32 nrows, const u32* sc, const u32* sb, const u32* keep, const u32* upos) {
  GRID_STRIDE(k0, nrows) {
    u32 k = (u32)k0;
    if (!keep[k]) continue;
    int p = seg_of(B.rbase, B.npat, k);
    u32 d = upos[k] - upos[B.rbase[p]];
    const int nb = B.pat[p].nb;
    B.out_cls[p][d] = sc[k];
    for (int j = 0; j < nb; j++) B.out_bind[p][(u64)d * nb + j] = sb[(u64)k * B.stride + j];
  }
}

__global__ void k_em_ubounds(const u32* upos, Batch B, u32* out) {
  int p = threadIdx.x;
  if (p <= B.npat) out[p] = upos[B.rbase[p]];
}

static double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void Engine::ematch_batch(const std::vector<int>& pids_all) {
  const bool dbg = getenv("TSAT_DEBUG_EMATCH") != nullptr;
  double w0 = wall_ms();
  if (!snap.valid || snap.n_atoms != h_atoms.size()) build_snapshot();
  for (size_t c0 = 0; c0 < pids_all.size(); c0 += MAX_BATCH) {
    std::vector<int> pids(pids_all.begin() + c0, pids_all.begin() + std::min(pids_all.size(), c0 + MAX_BATCH));
    Batch B;
    memset(&B, 0, sizeof(B));
    std::vector<int> live;  // patterns with candidates
    int maxapps = 0;
    u32 ntot = 0;
    int stride = 1;
    double cand_bytes = 0;
    // root candidate ranges (this rank's class range when sharded, shard.cu)
    std::vector<u32> rng(2 * pids.size(), 0);
    for (size_t q = 0; q < pids.size(); q++) {
      u32 ra = patterns[pids[q]].apps[0].atom;
      if (ra + 1 < snap.op_off_h.size()) {
        rng[2 * q] = snap.op_off_h[ra];
        rng[2 * q + 1] = snap.op_off_h[ra + 1];
      }
    }
    shard_candidate_ranges(rng);
    for (size_t q = 0; q < pids.size(); q++) {
      int pid = pids[q];
      const HPattern& hp = patterns[pid];
      MatchSet& ms = matches[pid];
      ms.nb = hp.nvars;
      ms.n = 0;
      u32 lo = rng[2 * q], hi = rng[2 * q + 1];
      if (hi == lo) continue;
      int b = (int)live.size();
      PatDev& p = B.pat[b];
      p.napps = (int)hp.apps.size();
      p.nb = hp.nvars;
      for (int i = 0; i < p.napps; i++) p.apps[i] = hp.apps[i];
      for (int k = 0; k < hp.nvars; k++) p.order[k] = hp.order[k];
      if (p.napps == 1 && p.apps[0].nargs <= 8) {
        // binding position k <- first root child carrying var order[k]; repeats must agree
        int first[MAX_VARS];
        for (int v = 0; v < MAX_VARS; v++) first[v] = -1;
        bool ok = true;
        for (int j = 0; j < p.apps[0].nargs && ok; j++) {
          int v = -p.apps[0].child[j] - 1;
          if (v < 0 || v >= MAX_VARS) ok = false;
          else if (first[v] < 0) first[v] = j;
          else if (p.neq < 8) {
            p.eq[(int)p.neq][0] = (int8_t)first[v];
            p.eq[(int)p.neq][1] = (int8_t)j;
            p.neq++;
          } else {
            ok = false;  // too many repeats: general DFS
          }
        }
        for (int k = 0; k < hp.nvars && ok; k++) {
          if (first[hp.order[k]] < 0) ok = false;
          else p.src[k] = (int8_t)first[hp.order[k]];
        }
        p.fast = ok ? 1 : 0;
      }
      if (p.napps > maxapps) maxapps = p.napps;
      B.cbase[b] = ntot;
      B.obase[b] = lo;
      ntot += hi - lo;
      stride = std::max(stride, hp.nvars);
      cand_bytes += (double)(hi - lo) * (17.0 + 8.0 * hp.apps[0].nargs);
      live.push_back(pid);
    }
    if (live.empty()) {
      shard_gather_matches(pids);
      continue;
    }
    int np = (int)live.size();
    B.npat = np;
    B.cbase[np] = ntot;
    B.stride = stride;
    // root-operator groups (patterns with one root atom are adjacent: the
    // patterns were laid out in pids order, so regroup by a stable sort)
    {
      std::vector<int> idx(np);
      for (int b = 0; b < np; b++) idx[b] = b;
      std::stable_sort(idx.begin(), idx.end(),
                       [&](int x, int y) { return B.pat[x].apps[0].atom < B.pat[y].apps[0].atom; });
      Batch B2 = B;
      std::vector<int> live2(np);
      u32 cb = 0;
      for (int b = 0; b < np; b++) {
        int o = idx[b];
        B2.pat[b] = B.pat[o];
        B2.obase[b] = B.obase[o];
        u32 sz = B.cbase[o + 1] - B.cbase[o];
        B2.cbase[b] = cb;
        cb += sz;
        live2[b] = live[o];
      }
      B2.cbase[np] = cb;
      B2.ngrp = 0;
      u32 gb = 0;
      for (int b = 0; b < np; b++) {
        if (b == 0 || B2.pat[b].apps[0].atom != B2.pat[b - 1].apps[0].atom || B2.obase[b] != B2.obase[b - 1]) {
          B2.gp[B2.ngrp] = b;
          B2.gbase[B2.ngrp] = gb;
          gb += B2.cbase[b + 1] - B2.cbase[b];
          B2.ngrp++;
        }
      }
      B2.gp[B2.ngrp] = np;
      B2.gbase[B2.ngrp] = gb;
      B = B2;
      live = live2;
    }
    KTimer kt(*this, KG_EMATCH, 0.0, 0);
    SnapDev sd{snap.cls_index.p, snap.cls_off.p, snap.cls_nodes.p, snap.op_nodes.p, snap.n_alloc,
                (h.dirty || uf_changed) ? 0 : 1};
    // semi-join reduction: bitmaps of every nested app of every live pattern
    {
      const u64 words = ((u64)snap.n_alloc + 31) / 32 + 1;
      int nbm = 0;
      int bmidx[MAX_BATCH][MAX_PAT_APPS];
      int height[MAX_BATCH][MAX_PAT_APPS];
      int hmax = -1;
      for (int b = 0; b < np; b++) {
        PatDev& p = B.pat[b];
        for (int i = p.napps - 1; i >= 0; i--) {  // pre-order: children after their parent
          int hgt = 0;
          for (int j = 0; j < p.apps[i].nargs; j++)
            if (p.apps[i].child[j] >= 0) hgt = std::max(hgt, height[b][p.apps[i].child[j]] + 1);
          height[b][i] = hgt;
          bmidx[b][i] = -1;
          p.bm[i] = nullptr;
          if (i >= 1 && nbm < SEMI_MAX) {
            bmidx[b][i] = nbm++;
            hmax = std::max(hmax, hgt);
          }
        }
      }
      if (nbm) {
        em_pool.ensure((u64)nbm * words);
        CUDA_OK(cudaMemsetAsync(em_pool.p, 0, (u64)nbm * words * sizeof(u32), s));
        for (int hgt = 0; hgt <= hmax; hgt++) {
          SemiJobs J;
          memset(&J, 0, sizeof(J));
          u32 tot = 0;
          for (int b = 0; b < np; b++) {
            const PatDev& p = B.pat[b];
            for (int i = 1; i < p.napps; i++) {
              if (bmidx[b][i] < 0 || height[b][i] != hgt) continue;
              SemiJob& jb = J.job[J.n];
              u32 atom = p.apps[i].atom;
              jb.lo = atom + 1 < snap.op_off_h.size() ? snap.op_off_h[atom] : 0;
              jb.hi = atom + 1 < snap.op_off_h.size() ? snap.op_off_h[atom + 1] : 0;
              jb.out = (u32)bmidx[b][i];
              jb.nargs = p.apps[i].nargs;
              bool usable = true;
              for (int j = 0; j < 8; j++) {
                int c = j < jb.nargs ? p.apps[i].child[j] : -1;
                jb.child[j] = c >= 0 ? bmidx[b][c] : -1;
                if (c >= 0 && bmidx[b][c] < 0) usable = false;
              }
              if (!usable) {  // a child without a bitmap: this app cannot be pre-filtered
                bmidx[b][i] = -1;
                continue;
              }
              J.base[J.n] = tot;
              tot += jb.hi - jb.lo;
              cand_bytes += 13.0 * (jb.hi - jb.lo) + 8.0 * jb.nargs * (jb.hi - jb.lo);
              J.n++;
            }
          }
          J.base[J.n] = tot;
          if (tot) k_em_semijoin<<<nblk(tot), 256, 0, s>>>(view(), sd, J, em_pool.p, words);
        }
        for (int b = 0; b < np; b++)
          for (int i = 1; i < B.pat[b].napps; i++)
            B.pat[b].bm[i] = bmidx[b][i] >= 0 ? em_pool.p + (u64)bmidx[b][i] * words : nullptr;
      }
    }
    DevBuf<u32>& cnt = sc.m_cnt;
    DevBuf<u32>& off = sc.m_pos;
    DevBuf<u32>& bnd = sc.m_bnd;
    cnt.ensure(ntot + 1);
    off.ensure(ntot + 1);
    bnd.ensure(2 * (MAX_BATCH + 1));
    bool small = maxapps <= 4 && stride <= 8;
    for (int b = 0; b < np; b++) small &= B.pat[b].nb <= 8;
    static const bool em_warp = getenv("TSAT_EM_THREAD") == nullptr;  // debug: thread-per-candidate DFS only
    bool nested = false;
    for (int b = 0; b < np; b++) nested |= !B.pat[b].fast;
    const int split = (em_warp && nested) ? 1 : 0;
    DevBuf<u32>& heavy = sc.m_heavy;
    if (split) {
      heavy.ensure((u64)ntot + 2);
      CUDA_OK(cudaMemsetAsync(heavy.p + ntot, 0, sizeof(u32), s));
    }
    u32* nheavy = split ? heavy.p + ntot : nullptr;
    const unsigned wblk = 148u * 8u;
    static const u32 cut = getenv("TSAT_EM_CUT") ? (u32)atoi(getenv("TSAT_EM_CUT")) : EM_HEAVY_L1;
    if (small) k_em_count<8, 4><<<nblk(ntot, 128), 128, 0, s>>>(view(), sd, B, ntot, cnt.p, split ? heavy.p : nullptr, nheavy, cut);
    else k_em_count<MAX_VARS, MAX_PAT_APPS><<<nblk(ntot, 128), 128, 0, s>>>(view(), sd, B, ntot, cnt.p,
                                                                             split ? heavy.p : nullptr, nheavy, cut);
    if (split) {
      if (small) k_em_count_w<8, 4><<<wblk, 256, 0, s>>>(view(), sd, B, heavy.p, nheavy, cnt.p);
      else k_em_count_w<MAX_VARS, MAX_PAT_APPS><<<wblk, 256, 0, s>>>(view(), sd, B, heavy.p, nheavy, cnt.p);
    }
    CUDA_OK(cudaMemsetAsync(cnt.p + ntot, 0, sizeof(u32), s));
    dev_exclusive_scan_u32(*this, cnt.p, off.p, ntot + 1);
    k_em_bounds<<<1, 32, 0, s>>>(off.p, B, bnd.p);
    CUDA_OK(cudaMemcpyAsync(B.rbase, bnd.p, (np + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    u32 nrows = B.rbase[np];
    double w1 = wall_ms();
    if (dbg && ntot) {
      std::vector<u32> hc(ntot);
      CUDA_OK(cudaMemcpy(hc.data(), cnt.p, ntot * 4, cudaMemcpyDeviceToHost));
      u32 mx = 0;
      for (u32 x : hc) mx = std::max(mx, x);
      fprintf(stderr, "  max matches per candidate %u\n", mx);
      w1 = wall_ms();
    }
    for (int b = 0; b < np; b++) {
      MatchSet& ms = matches[live[b]];
      u32 raw = B.rbase[b + 1] - B.rbase[b];
      ms.cls.ensure(raw + 1);
      ms.bind.ensure((u64)(raw + 1) * std::max(ms.nb, 1));
      B.out_cls[b] = ms.cls.p;
      B.out_bind[b] = ms.bind.p;
    }
    u32 nuniq[MAX_BATCH + 1] = {0};
    if (nrows) {
      DevBuf<u32>& rc = sc.m_rc;
      DevBuf<u32>& rb = sc.m_rb;
      DevBuf<u32>& scl = sc.m_key;
      DevBuf<u32>& sbd = sc.m_perm;
      DevBuf<u32>& keep = sc.m_fl;
      DevBuf<u32>& upos = sc.m_perm2;
      rc.ensure(nrows);
      rb.ensure((u64)nrows * stride);
      scl.ensure(nrows);
      sbd.ensure((u64)nrows * stride);
      keep.ensure(nrows + 1);
      upos.ensure(nrows + 1);
      DevBuf<u32>& big = sc.m_big;
      DevBuf<u32>& head = sc.m_head;
      DevBuf<u32>& bpos = sc.m_bpos;
      bpos.ensure(nrows + 1);
      big.ensure(nrows + 1);
      head.ensure(nrows + 1);
      if (small) k_em_emit<8, 4><<<nblk(ntot, 128), 128, 0, s>>>(view(), sd, B, ntot, off.p, rc.p, rb.p, split, cut);
      else k_em_emit<MAX_VARS, MAX_PAT_APPS><<<nblk(ntot, 128), 128, 0, s>>>(view(), sd, B, ntot, off.p, rc.p, rb.p,
                                                                            split, cut);
      if (split) {
        if (small) k_em_emit_w<8, 4><<<wblk, 256, 0, s>>>(view(), sd, B, heavy.p, nheavy, off.p, rc.p, rb.p);
        else k_em_emit_w<MAX_VARS, MAX_PAT_APPS><<<wblk, 256, 0, s>>>(view(), sd, B, heavy.p, nheavy, off.p, rc.p,
                                                                      rb.p);
      }
      k_em_rank<<<nblk(nrows), 256, 0, s>>>(B, nrows, rc.p, rb.p, scl.p, sbd.p, big.p, head.p);
      // large groups: stable LSD radix sort of their rows by (group, bindings)
      CUDA_OK(cudaMemsetAsync(big.p + nrows, 0, sizeof(u32), s));
      dev_exclusive_scan_u32(*this, big.p, bpos.p, nrows + 1);
      u32 nbigrows = 0;
      CUDA_OK(cudaMemcpyAsync(&nbigrows, bpos.p + nrows, sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      double w2 = wall_ms();
      if (dbg) fprintf(stderr, "  count+scan %.3f ms, emit+rank %.3f ms\n", w1 - w0, w2 - w1);
      if (dbg) fprintf(stderr, "  big rows %u (stride %d)\n", nbigrows, stride);
      if (nbigrows) {
        DevBuf<u32>& L = sc.m_L;
        DevBuf<u32>& bh = sc.m_bh;
        DevBuf<u32>& gex = sc.m_gex;
        DevBuf<u32>& perm = sc.m_bperm;
        DevBuf<u32>& perm2 = sc.m_bperm2;
        DevBuf<u32>& key = sc.m_bkey;
        DevBuf<u32>& key2 = sc.m_bkey2;
        L.ensure(nbigrows + 1);
        bh.ensure(nbigrows + 1);
        gex.ensure(nbigrows + 1);
        perm.ensure(nbigrows + 1);
        perm2.ensure(nbigrows + 1);
        key.ensure(nbigrows + 1);
        key2.ensure(nbigrows + 1);
        k_em_big_list<<<nblk(nrows), 256, 0, s>>>(nrows, big.p, bpos.p, head.p, L.p, bh.p, perm.p);
        dev_exclusive_scan_u32(*this, bh.p, gex.p, nbigrows);
        int eb = (int)bits_for(h.next_id);
        // binding words past the widest pattern that can own a big group are
        // zero padding for every big row: their passes would be no-ops
        int wmax = 0;
        for (int b = 0; b < np; b++)
          if (B.rbase[b + 1] - B.rbase[b] > SMALL_GROUP) wmax = std::max(wmax, (int)B.pat[b].nb);
        for (int w = std::min(wmax, stride) - 1; w >= -1; w--) {
          k_em_big_key<<<nblk(nbigrows), 256, 0, s>>>(nbigrows, L.p, perm.p, rb.p, stride, w, bh.p, gex.p, key.p);
          dev_sort_pairs_u32(*this, key.p, key2.p, perm.p, perm2.p, nbigrows, w >= 0 ? eb : (int)bits_for(nbigrows / (SMALL_GROUP + 1)));  // every big group has > SMALL_GROUP rows
          perm.swap(perm2);
        }
        k_em_big_scatter<<<nblk(nbigrows), 256, 0, s>>>(nbigrows, L.p, perm.p, rc.p, rb.p, stride, scl.p, sbd.p);
      }
      k_em_keep<<<nblk(nrows), 256, 0, s>>>(B, nrows, scl.p, sbd.p, keep.p);
      CUDA_OK(cudaMemsetAsync(keep.p + nrows, 0, sizeof(u32), s));
      dev_exclusive_scan_u32(*this, keep.p, upos.p, nrows + 1);
      k_em_compact<<<nblk(nrows), 256, 0, s>>>(B, nrows, scl.p, sbd.p, keep.p, upos.p);
      k_em_ubounds<<<1, 32, 0, s>>>(upos.p, B, bnd.p);
      CUDA_OK(cudaMemcpyAsync(nuniq, bnd.p, (np + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
    }
    for (int b = 0; b < np; b++) matches[live[b]].n = nuniq[b + 1] - nuniq[b];
    if (dbg) {
      fprintf(stderr, "ematch batch: %d patterns, %u candidates, %u rows, %u unique, %.3f ms\n", np, ntot, nrows,
              nuniq[np], wall_ms() - w0);
      fprintf(stderr, "  per pattern (id:rows):");
      for (int b = 0; b < np; b++) fprintf(stderr, " %d:%u", pids[b], B.rbase[b + 1] - B.rbase[b]);
      fprintf(stderr, "\n");
    }
    // algorithmic bytes: candidate scan + match rows written,
    // ordered and compacted
    double rows_bytes = 0;
    for (int b = 0; b < np; b++) rows_bytes += (double)(B.rbase[b + 1] - B.rbase[b]) * 4.0 * (1 + B.pat[b].nb);
    kt.bytes = cand_bytes + 2.0 * rows_bytes;
    kt.launches = 9;
    shard_gather_matches(pids);
  }
}
