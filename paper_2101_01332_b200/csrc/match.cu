// E-matching on the GPU (reference: pkg/src/tensorsat/egraph.py:248-293).
//
// One thread per root candidate: candidates come from the per-operator CSR
// (snapshot.op_nodes), i.e. a relational scan of the root operator's table;
// nested pattern nodes are joined through the class CSR (class -> members,
// ascending ids) with filter-list, op and arity checks and nonlinear-variable
// equality.  Results are deduplicated and ordered by (eclass, bindings in
// variable-name order) with a stable LSD radix sort over the tuple words,
// reproducing _match_sorted (egraph.py:107-112).
#include <cub/cub.cuh>

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
  int napps;
  int nb;
  int order[MAX_VARS];
};

struct SnapDev {
  const u32* cls_index;
  const u32* cls_off;
  const u32* cls_nodes;
  u32 n_alloc;
};

__device__ __forceinline__ bool node_ok(const G& g, u32 nid, const PatApp& a) {
  if (g.flags[nid] & NF_FILT) return false;
  if (g.op[nid] != a.atom) return false;
  return (int)(g.koff[nid + 1] - g.koff[nid]) == a.nargs;
}

// bind the variable children of app t for node nid; set classes of app children
__device__ __forceinline__ bool bind_node(const G& g, const PatApp& a, u32 nid, int t, u32* env,
                                          int8_t* bound_at, u32* cls_app) {
  u32 base = g.koff[nid];
  for (int j = 0; j < a.nargs; j++) {
    u32 ch = uf_find_ro(g.parent, g.kids[base + j]);
    int c = a.child[j];
    if (c >= 0) {
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

__device__ __forceinline__ void unbind(int t, u32* env, int8_t* bound_at) {
  for (int v = 0; v < MAX_VARS; v++)
    if (bound_at[v] == t) {
      bound_at[v] = -1;
      env[v] = TSAT_NONE;
    }
}

__global__ void k_ematch(G g, SnapDev sd, PatDev p, const u32* cand, u32 ncand, u32* out_cls,
                         u32* out_bind, u32* count, u32 cap) {
  GRID_STRIDE(ci, ncand) {
    u32 r = cand[ci];
    if (!node_ok(g, r, p.apps[0])) continue;
    u32 env[MAX_VARS];
    int8_t bound_at[MAX_VARS];
    u32 cls_app[MAX_PAT_APPS];
    u32 pos[MAX_PAT_APPS], end[MAX_PAT_APPS];
    for (int v = 0; v < MAX_VARS; v++) {
      env[v] = TSAT_NONE;
      bound_at[v] = -1;
    }
    if (!bind_node(g, p.apps[0], r, 0, env, bound_at, cls_app)) continue;
    u32 rc = uf_find_ro(g.parent, r);
    int level = 1;
    bool init = true;
    while (true) {
      if (level == p.napps) {
        u32 slot = atomicAdd(count, 1u);
        if (slot < cap) {
          out_cls[slot] = rc;
          for (int k = 0; k < p.nb; k++) out_bind[(u64)slot * p.nb + k] = env[p.order[k]];
        }
        level--;
        if (level == 0) break;
        unbind(level, env, bound_at);
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
        if (bind_node(g, a, m, level, env, bound_at, cls_app)) {
          found = true;
          break;
        }
        unbind(level, env, bound_at);
      }
      if (found) {
        level++;
        init = true;
      } else {
        level--;
        if (level == 0) break;
        unbind(level, env, bound_at);
        init = false;
      }
    }
  }
}

__global__ void k_iota(u32* p, u32 n) { GRID_STRIDE(i, n) p[i] = (u32)i; }

__global__ void k_gather_word(const u32* cls, const u32* bind, int nb, int w, const u32* perm, u32 n,
                              u32* out) {
  GRID_STRIDE(i, n) {
    u32 r = perm[i];
    out[i] = w == 0 ? cls[r] : bind[(u64)r * nb + (w - 1)];
  }
}

__global__ void k_unique_flags(const u32* cls, const u32* bind, int nb, const u32* perm, u32 n, u32* fl) {
  GRID_STRIDE(i, n) {
    if (i == 0) {
      fl[i] = 1;
      continue;
    }
    u32 a = perm[i], b = perm[i - 1];
    bool same = cls[a] == cls[b];
    for (int k = 0; k < nb && same; k++) same = bind[(u64)a * nb + k] == bind[(u64)b * nb + k];
    fl[i] = same ? 0u : 1u;
  }
}

__global__ void k_unique_write(const u32* cls, const u32* bind, int nb, const u32* perm, const u32* fl,
                               const u32* pos, u32 n, u32* ocls, u32* obind) {
  GRID_STRIDE(i, n) {
    if (!fl[i]) continue;
    u32 r = perm[i], o = pos[i];
    ocls[o] = cls[r];
    for (int k = 0; k < nb; k++) obind[(u64)o * nb + k] = bind[(u64)r * nb + k];
  }
}

void Engine::ematch_pattern(int pid, MatchSet& out) {
  if (!snap.valid || snap.n_atoms != h_atoms.size()) build_snapshot();
  const HPattern& hp = patterns[pid];
  PatDev p;
  memset(&p, 0, sizeof(p));
  p.napps = (int)hp.apps.size();
  p.nb = hp.nvars;
  for (int i = 0; i < p.napps; i++) p.apps[i] = hp.apps[i];
  for (int k = 0; k < hp.nvars; k++) p.order[k] = hp.order[k];
  SnapDev sd{snap.cls_index.p, snap.cls_off.p, snap.cls_nodes.p, snap.n_alloc};
  u32 ra = p.apps[0].atom;
  out.nb = p.nb;
  out.n = 0;
  if (ra >= h_atoms.size()) return;
  u32 range[2];
  CUDA_OK(cudaMemcpyAsync(range, snap.op_off.p + ra, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  u32 ncand = range[1] - range[0];
  if (ncand == 0) return;
  // whole e-match (root scan + ordering + dedup) timed as one group; bytes per
  // candidates + match rows + a (1+v)-word sort of the matches
  KTimer kt_all(*this, KG_EMATCH, 0.0, 0);
  DevBuf<u32>& rc = sc.m_rc;
  DevBuf<u32>& rb = sc.m_rb;
  DevBuf<u32>& cntb = sc.m_cnt;
  cntb.ensure(1);
  u32 cap = std::max<u32>(ncand * 2, 1024);
  u32 m = 0;
  for (int attempt = 0; attempt < 8; attempt++) {
    rc.ensure(cap);
    rb.ensure((u64)cap * std::max(p.nb, 1));
    CUDA_OK(cudaMemsetAsync(cntb.p, 0, sizeof(u32), s));
    k_ematch<<<nblk(ncand, 128), 128, 0, s>>>(view(), sd, p, snap.op_nodes.p + range[0], ncand, rc.p, rb.p, cntb.p,
                                              cap);
    CUDA_OK(cudaMemcpyAsync(&m, cntb.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    if (m <= cap) break;
    cap = m + 1024;
  }
  kt_all.bytes = (double)ncand * (17.0 + 8.0 * p.apps[0].nargs) + (double)m * 4.0 * (1 + p.nb) * 2.0;
  kt_all.launches = 1;
  if (m == 0) return;
  // stable LSD sort over words (cls, b0..b_{nb-1}), last word first
  DevBuf<u32>& perm = sc.m_perm;
  DevBuf<u32>& perm2 = sc.m_perm2;
  DevBuf<u32>& key = sc.m_key;
  DevBuf<u32>& key2 = sc.m_key2;
  perm.ensure(m);
  perm2.ensure(m);
  key.ensure(m);
  key2.ensure(m);
  k_iota<<<nblk(m), 256, 0, s>>>(perm.p, m);
  int eb = (int)bits_for(h.next_id);
  for (int w = p.nb; w >= 0; w--) {
    k_gather_word<<<nblk(m), 256, 0, s>>>(rc.p, rb.p, p.nb, w, perm.p, m, key.p);
    dev_sort_pairs_u32(*this, key.p, key2.p, perm.p, perm2.p, m, eb);
    perm.swap(perm2);
  }
  DevBuf<u32>& fl = sc.m_fl;
  DevBuf<u32>& pos = sc.m_pos;
  fl.ensure(m);
  pos.ensure(m);
  k_unique_flags<<<nblk(m), 256, 0, s>>>(rc.p, rb.p, p.nb, perm.p, m, fl.p);
  dev_exclusive_scan_u32(*this, fl.p, pos.p, m);
  u32 lf, lp;
  CUDA_OK(cudaMemcpyAsync(&lf, fl.p + m - 1, sizeof(u32), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(&lp, pos.p + m - 1, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  u32 nu = lf + lp;
  out.cls.ensure(nu);
  out.bind.ensure((u64)nu * std::max(p.nb, 1));
  k_unique_write<<<nblk(m), 256, 0, s>>>(rc.p, rb.p, p.nb, perm.p, fl.p, pos.p, m, out.cls.p, out.bind.p);
  out.n = nu;
  sync();
}
