// GPU-resident e-graph: struct-of-arrays node table, union-find, hashcons.
//
// Layout in HBM (all indexed by node id; ids are the reference's global
// insertion counter, reference: pkg/src/tensorsat/egraph.py:164-182):
//   op[n]      u32  interned atom id
//   koff[n]    u32  CSR offset of the node's children in kids[]
//   kids[]     u32  children as stored (canonical when inserted / rebuilt)
//   parent[n]  u32  union-find parent; root = class id = min node id
//   flags[n]   u8   NF_ALIVE | NF_FILT (filter list)
//   val[n]     Val  analysis of the class rooted at n (valid for roots)
// Hashcons: open-addressing table keyed by (op, kids[koff..]); a slot is
//   (epoch:8 | fingerprint:24) << 32 | node id
// so a probe compares the key hash's fingerprint before touching the node
// table, and a new epoch empties the table without clearing it (each
// congruence round starts a new epoch).  Every live node is in it under its
// stored key, so keys need no storage.
#pragma once
#include "analysis.cuh"

struct Counters {
  u32 next_id;   // == allocated_nodes
  u32 live;      // == num_nodes
  u32 nkids;     // == koff[next_id]
  u32 dirty;     // a union happened since the last rebuild
  u32 grow;      // sequential kernel stopped for capacity
  u32 pad[3];
};

struct G {
  u32* op;
  u32* koff;
  u32* kids;
  u32* parent;
  u8* flags;
  Val* val;
  unsigned long long* hc;
  u32 hc_mask;
  u32 hc_max;    // allocated ids the table is sized for (load factor)
  u32 hc_epoch;  // 1..255; slots of other epochs are empty
  u32 cap_nodes;
  u32 cap_kids;
  int analysis;
  const AtomInfo* atoms;
  TreeTab tt;
  DevError* err;
  Counters* cnt;
};

__device__ __forceinline__ u64 key_hash(u32 op, int n, const u32* kids) {
  u64 h = hash_mix(0x2545f4914f6cdd1dULL ^ ((u64)n << 32), op);
  for (int i = 0; i < n; i++) h = hash_mix(h, kids[i]);
  return h;
}

__device__ __forceinline__ u64 node_hash(const G& g, u32 nid) {
  u32 a = g.koff[nid], b = g.koff[nid + 1];
  u64 h = hash_mix(0x2545f4914f6cdd1dULL ^ ((u64)(b - a) << 32), g.op[nid]);
  for (u32 i = a; i < b; i++) h = hash_mix(h, g.kids[i]);
  return h;
}

__device__ __forceinline__ bool node_key_eq(const G& g, u32 nid, u32 op, int n, const u32* kids) {
  if (g.op[nid] != op) return false;
  u32 a = g.koff[nid];
  if ((int)(g.koff[nid + 1] - a) != n) return false;
  for (int i = 0; i < n; i++)
    if (g.kids[a + i] != kids[i]) return false;
  return true;
}

__device__ __forceinline__ bool node_eq_node(const G& g, u32 x, u32 y) {
  if (g.op[x] != g.op[y]) return false;
  u32 ax = g.koff[x], bx = g.koff[x + 1], ay = g.koff[y];
  if (g.koff[y + 1] - ay != bx - ax) return false;
  for (u32 i = 0; i < bx - ax; i++)
    if (g.kids[ax + i] != g.kids[ay + i]) return false;
  return true;
}

// fingerprint 0 is reserved for tombstones (incremental rebuild rounds), so
// a tombstone is an occupied slot no probe's tag ever matches
__device__ __forceinline__ u32 hc_tag(u32 epoch, u64 h) {
  u32 fp = (u32)(h >> 40);
  return (epoch << 24) | (fp ? fp : 1u);
}
__device__ __forceinline__ unsigned long long hc_tomb(u32 epoch) {
  return ((unsigned long long)(epoch << 24) << 32) | 0xFFFFFFFFull;
}
__device__ __forceinline__ bool hc_live(const G& g, unsigned long long e) { return (u32)(e >> 56) == g.hc_epoch; }

// hashcons lookup of a (canonical) key; TSAT_NONE on miss
__device__ __forceinline__ u32 hc_lookup(const G& g, u32 op, int n, const u32* kids) {
  u64 h = key_hash(op, n, kids);
  u32 slot = (u32)h & g.hc_mask, tag = hc_tag(g.hc_epoch, h);
  while (true) {
    unsigned long long e = g.hc[slot];
    if (!hc_live(g, e)) return TSAT_NONE;
    if ((u32)(e >> 32) == tag && node_key_eq(g, (u32)e, op, n, kids)) return (u32)e;
    slot = (slot + 1) & g.hc_mask;
  }
}

// insert node id (its key must be absent); lock-free
__device__ __forceinline__ void hc_insert(const G& g, u32 nid) {
  u64 h = node_hash(g, nid);
  u32 slot = (u32)h & g.hc_mask;
  unsigned long long v = ((unsigned long long)hc_tag(g.hc_epoch, h) << 32) | nid;
  while (true) {
    unsigned long long e = ((volatile unsigned long long*)g.hc)[slot];
    if (!hc_live(g, e)) {
      if (atomicCAS(&g.hc[slot], e, v) == e) return;
      continue;  // re-read the same slot
    }
    slot = (slot + 1) & g.hc_mask;
  }
}

__device__ __forceinline__ int ana_to_status(int as) {
  switch (as) {
    case AS_OK: return TSAT_OK;
    case AS_SPLIT_ORIGIN: return TSAT_ERR_SPLIT_ORIGIN;
    case AS_SHAPE: return TSAT_ERR_SHAPE;
    default: return TSAT_ERR_CAPACITY;
  }
}

// ----------------------------------------------------------------------------
// Sequential (single-thread) e-graph mutation, the exact reference semantics.
// Used by the generic EGraph API and by the engine's hazard slow path.

// add_enode (egraph.py:164-182).  kids are canonicalised in place.  Returns
// class id, or TSAT_NONE after recording an error.
static __device__ u32 seq_add_enode(const G& g, u32 op, u32* kids, int n) {
  for (int i = 0; i < n; i++) kids[i] = uf_find(g.parent, kids[i]);
  u32 hit = hc_lookup(g, op, n, kids);
  if (hit != TSAT_NONE) return uf_find(g.parent, hit);
  Counters* c = g.cnt;
  u32 nid = c->next_id;
  Val v;
  if (g.analysis) {
    const Val* kv[8];
    for (int i = 0; i < n && i < 8; i++) kv[i] = &g.val[kids[i]];
    int st = n > 7 ? AS_SHAPE : val_make(op, ValRefs{kv}, n, v, g.atoms, g.tt);
    if (st != AS_OK) {
      c->next_id = nid + 1;  // the reference bumps the counter before make()
      dev_set_error(g.err, ana_to_status(st), 1, nid, op);
      return TSAT_NONE;
    }
  }
  u32 base = c->nkids;
  g.op[nid] = op;
  g.koff[nid] = base;
  for (int i = 0; i < n; i++) g.kids[base + i] = kids[i];
  g.koff[nid + 1] = base + n;
  g.parent[nid] = nid;
  g.flags[nid] = NF_ALIVE;
  if (g.analysis) g.val[nid] = v;
  hc_insert(g, nid);
  c->next_id = nid + 1;
  c->nkids = base + n;
  c->live += 1;
  return nid;
}

// union (egraph.py:193-214): analysis merge first (may fail), then min-root
// link.  Returns the kept root or TSAT_NONE after recording an error.
static __device__ u32 seq_union(const G& g, u32 a, u32 b) {
  u32 ra = uf_find(g.parent, a), rb = uf_find(g.parent, b);
  if (ra == rb) return ra;
  u32 keep = ra < rb ? ra : rb, drop = ra < rb ? rb : ra;
  if (g.analysis) {
    Val m = g.val[ra];
    const Val& other = g.val[rb];
    if (!val_same_data(m, other)) {
      dev_set_error(g.err, TSAT_ERR_MERGE, 0, ra, rb);
      return TSAT_NONE;
    }
    int st = val_merge_into(m, other);
    if (st != AS_OK) {
      dev_set_error(g.err, TSAT_ERR_CAPACITY, 2, ra, rb);
      return TSAT_NONE;
    }
    g.val[keep] = m;
  }
  g.parent[drop] = keep;
  g.cnt->dirty = 1;
  return keep;
}
