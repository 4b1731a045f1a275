#include <cstdlib>
// Cost vector and greedy extraction on the GPU.
//
// * k_node_costs: c_i for every live e-node (reference cost.py:225-247 with
//   CostModel.node_cost :164-174 and synthetic_node_cost :78-126).  fp64
//   with the reference's operation order; the library is built with
//   -fmad=false so no multiply-add is contracted.  Table mode renders the
//   canonical signature key (cost.py:135-140) on device and probes a hash
//   table of the normalised keys.
// * greedy: Jacobi min-cost relaxation to fixpoint with the reference tie
//   rule (extract.py:120-159): per class, fold members in id order starting
//   from the previous round's (cost, node), update on total < cur - 1e-15 or
//   |total - cur| <= 1e-15 with a smaller id.  Child totals are summed in
//   child order.  Then a BFS over chosen nodes gives the reached selection
//   (extract.py:74-91).
#include <cooperative_groups.h>

#include <cmath>
#include <cstring>

#include <cub/cub.cuh>

#include "engine.cuh"

namespace cg = cooperative_groups;

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

struct CostTab {
  const char* keys;
  const i64* off;
  const double* vals;
  const u32* slots;
  u32 mask;
  int n;
  int mode;    // 0 synthetic, 1 table
  int strict;
  const char* names;
  const u32* name_off;
  u32* miss;       // strict: smallest node id whose signature has no entry (iter_nodes order, egraph.py:155-157)
  u32 dump_node;   // != TSAT_NONE: render that node's key into key_out only
  char* key_out;
};

__device__ __forceinline__ u64 fnv1a(const char* p, int n) {
  u64 h = 1469598103934665603ULL;
  for (int i = 0; i < n; i++) {
    h ^= (u8)p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

struct SigBuf {
  char b[320];
  int n = 0;
  bool ovf = false;
  __device__ void ch(char c) {
    if (n < 319) b[n++] = c;
    else ovf = true;
  }
  __device__ void str(const char* p, int len) {
    for (int i = 0; i < len; i++) ch(p[i]);
  }
  __device__ void cstr(const char* p) {
    while (*p) ch(*p++);
  }
  __device__ void num(i64 v) {
    char t[24];
    int k = 0;
    bool neg = v < 0;
    unsigned long long u = neg ? (unsigned long long)(-(v + 1)) + 1 : (unsigned long long)v;
    do {
      t[k++] = (char)('0' + u % 10);
      u /= 10;
    } while (u);
    if (neg) ch('-');
    while (k) ch(t[--k]);
  }
};

// sorted-by-name parameter order per op: scalar index list + names
__device__ const char* param_name(int op, int k, int& idx) {
  switch (op) {
    case OP_MATMUL: idx = 0; return "activation";
    case OP_CONV: {
      const int ix[4] = {3, 2, 0, 1};
      const char* nm[4] = {"activation", "padding", "stride_h", "stride_w"};
      idx = ix[k];
      return nm[k];
    }
    case OP_POOLMAX:
    case OP_POOLAVG: {
      const int ix[6] = {5, 0, 1, 4, 2, 3};
      const char* nm[6] = {"activation", "kernel_h", "kernel_w", "padding", "stride_h", "stride_w"};
      idx = ix[k];
      return nm[k];
    }
    case OP_TRANSPOSE: idx = 0; return "perm";
    case OP_SPLIT: idx = 0; return "axis";
    case OP_MERGE: idx = 0; return "count";
    case OP_RESHAPE: idx = 0; return "shape";
    case OP_INPUT:
    case OP_WEIGHT: idx = 0; return "identifier";
    default:
      if (op >= OP_CONCAT2 && op <= OP_CONCAT6) {
        idx = 0;
        return "axis";
      }
  }
  idx = -1;
  return nullptr;
}

__device__ __forceinline__ int n_params(int op) {
  switch (op) {
    case OP_MATMUL: case OP_TRANSPOSE: case OP_SPLIT: case OP_MERGE: case OP_RESHAPE:
    case OP_INPUT: case OP_WEIGHT: return 1;
    case OP_CONV: return 4;
    case OP_POOLMAX: case OP_POOLAVG: return 6;
    default: return (op >= OP_CONCAT2 && op <= OP_CONCAT6) ? 1 : 0;
  }
}

__device__ __forceinline__ i64 numel(const i64* d, int r) {
  i64 p = 1;
  for (int i = 0; i < r; i++) p *= d[i];
  return p;
}

__device__ __forceinline__ double base_cost(int op) {
  switch (op) {
    case OP_MATMUL: case OP_CONV: return 0.05;
    case OP_POOLMAX: case OP_POOLAVG: return 0.02;
    case OP_EWADD: case OP_EWMUL: case OP_RELU: case OP_TANH: case OP_SIGMOID: return 0.01;
    case OP_INPUT: case OP_WEIGHT: case OP_NOOP: return 0.0;
    default: return 0.005;
  }
}

#define RATE_EW 1e-7
#define RATE_MM 1e-6
#define FUSED_ACT 0.2

__global__ void k_node_costs(G g, CostTab ct, u32 n, double* out) {
  const double RATE_MOVE = 0.05 * 1e-7;
  GRID_STRIDE(i0, n) {
    u32 i = ct.dump_node != TSAT_NONE ? ct.dump_node : (u32)i0;
    if (!(g.flags[i] & NF_ALIVE)) {
      out[i] = 0.0;
      continue;
    }
    u32 a = g.koff[i], b = g.koff[i + 1];
    if (a == b) {
      out[i] = 0.0;
      continue;
    }
    const AtomInfo& ai = g.atoms[g.op[i]];
    int op = ai.kind == 1 ? ai.opcode : -1;
    if (op < 0) {
      dev_set_error(g.err, TSAT_ERR_SHAPE, 20, i, g.op[i]);
      out[i] = 0.0;
      continue;
    }
    if (op == OP_INPUT || op == OP_WEIGHT || op == OP_NOOP) {
      out[i] = 0.0;
      continue;
    }
    // gather scalars / shapes from child analyses in child order
    i64 sc[7];
    int sk[7];  // 0 int, 1 str atom
    int nsc = 0, nsh = 0;
    const Val* sh[7];
    for (u32 j = a; j < b; j++) {
      const Val& v = g.val[uf_find_ro(g.parent, g.kids[j])];
      if (v.kind == VK_N || v.kind == VK_S) {
        sk[nsc] = v.kind == VK_S;
        sc[nsc++] = v.iv;
      } else {
        sh[nsh++] = &v;
      }
    }
    if (ct.mode == 1) {
      SigBuf s;
      u32 na = ct.name_off[g.op[i]], nb = ct.name_off[g.op[i] + 1];
      s.str(ct.names + na, (int)(nb - na));
      int np = n_params(op);
      if (np) {
        s.ch('[');
        for (int k = 0; k < np; k++) {
          int idx;
          const char* pn = param_name(op, k, idx);
          if (k) s.ch(',');
          s.cstr(pn);
          s.ch('=');
          if (idx < nsc) {
            if (sk[idx]) {
              u32 x = ct.name_off[sc[idx]], y = ct.name_off[sc[idx] + 1];
              s.str(ct.names + x, (int)(y - x));
            } else {
              s.num(sc[idx]);
            }
          }
        }
        s.ch(']');
      }
      s.ch('(');
      for (int k = 0; k < nsh; k++) {
        if (k) s.ch(',');
        const Val& v = *sh[k];
        for (int d = 0; d < v.r0; d++) {
          if (d) s.ch('x');
          s.num(v.d0[d]);
        }
        if (v.kind == VK_TT) {
          s.ch('|');
          for (int d = 0; d < v.r1; d++) {
            if (d) s.ch('x');
            s.num(v.d1[d]);
          }
        }
      }
      s.ch(')');
      bool hit = false;
      if (!s.ovf && ct.n > 0) {
        u64 h = fnv1a(s.b, s.n);
        u32 slot = (u32)h & ct.mask;
        while (true) {
          u32 e = ct.slots[slot];
          if (e == TSAT_NONE) break;
          i64 ka = ct.off[e], kb = ct.off[e + 1];
          if (kb - ka == s.n) {
            bool eq = true;
            for (int q = 0; q < s.n && eq; q++) eq = ct.keys[ka + q] == s.b[q];
            if (eq) {
              out[i] = ct.vals[e];
              hit = true;
              break;
            }
          }
          slot = (slot + 1) & ct.mask;
        }
      }
      if (ct.dump_node != TSAT_NONE) {
        for (int q = 0; q < s.n; q++) ct.key_out[q] = s.b[q];
        ct.key_out[s.n] = 0;
        continue;
      }
      if (hit) continue;
      if (ct.strict) {
        atomicMin(ct.miss, i);
        out[i] = 0.0;
        continue;
      }
    }
    double base = base_cost(op), work = 0.0;
    switch (op) {
      case OP_MATMUL: {
        const Val &x = *sh[0], &y = *sh[1];
        i64 macs = numel(x.d0, x.r0) * y.d0[y.r0 - 1];
        work = RATE_MM * (double)macs;
        if (sc[0] != 0)
          work += FUSED_ACT * RATE_EW * (double)(numel(x.d0, x.r0) / x.d0[x.r0 - 1]) * (double)y.d0[y.r0 - 1];
        break;
      }
      case OP_CONV: {
        const Val &x = *sh[0], &w = *sh[1];
        i64 oh = 0, ow = 0;
        if (conv_out(x.d0[2], x.d0[3], w.d0[2], w.d0[3], sc[0], sc[1], sc[2], oh, ow)) {
          dev_set_error(g.err, TSAT_ERR_SHAPE, 22, i, g.op[i]);
          break;
        }
        i64 oe = x.d0[0] * w.d0[0] * oh * ow;
        work = RATE_MM * (double)oe * (double)w.d0[1] * (double)w.d0[2] * (double)w.d0[3];
        if (sc[3] != 0) work += FUSED_ACT * RATE_EW * (double)oe;
        break;
      }
      case OP_EWADD: case OP_EWMUL: case OP_RELU: case OP_TANH: case OP_SIGMOID:
        work = RATE_EW * (double)numel(sh[0]->d0, sh[0]->r0);
        break;
      case OP_POOLMAX:
      case OP_POOLAVG: {
        const Val& x = *sh[0];
        i64 kh = sc[0], kw = sc[1], oh = 0, ow = 0;
        if (conv_out(x.d0[2], x.d0[3], kh, kw, sc[2], sc[3], sc[4], oh, ow)) {
          dev_set_error(g.err, TSAT_ERR_SHAPE, 23, i, g.op[i]);
          break;
        }
        work = RATE_EW * (double)x.d0[0] * (double)x.d0[1] * (double)oh * (double)ow * (double)kh * (double)kw;
        if (sc[5] != 0)
          work += FUSED_ACT * RATE_EW * (double)x.d0[0] * (double)x.d0[1] * (double)oh * (double)ow;
        break;
      }
      case OP_SPLIT:
        work = RATE_MOVE * (double)numel(sh[0]->d0, sh[0]->r0);
        break;
      case OP_SPLIT0:
        work = RATE_MOVE * (double)numel(sh[0]->d0, sh[0]->r0);
        break;
      case OP_SPLIT1:
        work = RATE_MOVE * (double)numel(sh[0]->d1, sh[0]->r1);
        break;
      case OP_ENLARGE: {
        const Val &x = *sh[0], &r = *sh[1];
        i64 d[4] = {x.d0[0], x.d0[1], r.d0[2], r.d0[3]};
        work = RATE_MOVE * (double)numel(d, 4);
        break;
      }
      case OP_MERGE:
        work = RATE_MOVE * (double)numel(sh[0]->d0, sh[0]->r0) * (double)sc[0];
        break;
      case OP_TRANSPOSE:
      case OP_RESHAPE:
        work = RATE_MOVE * (double)numel(sh[0]->d0, sh[0]->r0);
        break;
      default:
        if (op >= OP_CONCAT2 && op <= OP_CONCAT6) {
          i64 tot = 0;
          for (int k = 0; k < nsh; k++) tot += numel(sh[k]->d0, sh[k]->r0);
          work = RATE_MOVE * (double)tot;
        }
    }
    out[i] = base + work;
  }
}

static u64 fnv1a_host(const char* p, i64 n) {
  u64 h = 1469598103934665603ULL;
  for (i64 i = 0; i < n; i++) {
    h ^= (u8)p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

__global__ void k_gather_f64(const double* src, const u32* ids, u32 n, double* out) {
  GRID_STRIDE(i, n) out[i] = src[ids[i]];
}

// c_i of selected nodes (ids == nullptr: the first n entries)
void Engine::costs_gather(u32 n, const u32* ids, double* out) {
  if (costs_valid_for != h.next_id) throw TsatException(TSAT_ERR_STATE, "device cost vector is stale");
  if (!n) return;
  if (!ids) {
    if (n > h.next_id) throw TsatException(TSAT_ERR_ARG, "more entries than nodes");
    CUDA_OK(cudaMemcpyAsync(out, d_costs.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync();
    return;
  }
  for (u32 i = 0; i < n; i++)
    if (ids[i] >= h.next_id) throw TsatException(TSAT_ERR_ARG, "node id out of range");
  DevBuf<u32>& di = scratch_u32[0];
  DevBuf<double>& dv = sc.g_c1;
  di.ensure(n + 1);
  dv.ensure(n + 1);
  CUDA_OK(cudaMemcpyAsync(di.p, ids, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  k_gather_f64<<<nblk(n), 256, 0, s>>>(d_costs.p, di.p, n, dv.p);
  CUDA_OK(cudaMemcpyAsync(out, dv.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync();
}

void Engine::costs(int mode, int strict, int ntab, const char* keys, const i64* key_off, const double* vals,
                   double* out) {
  if (!analysis) throw TsatException(TSAT_ERR_STATE, "egraph_costs needs the tensor analysis");
  u32 n = h.next_id;
  DevBuf<char>& dk = sc.k_keys;
  DevBuf<i64>& doff = sc.k_off;
  DevBuf<double>& dv = sc.k_dv;
  DevBuf<u32>& dslots = sc.k_slots;
  CostTab ct;
  memset(&ct, 0, sizeof(ct));
  ct.mode = mode;
  ct.strict = strict;
  ct.n = ntab;
  ct.names = d_names.p;
  ct.name_off = d_name_off.p;
  if (mode == 1 && ntab > 0) {
    i64 nbytes = key_off[ntab];
    u32 cap = 16;
    while (cap < 2u * (u32)ntab) cap *= 2;
    std::vector<u32> slots(cap, TSAT_NONE);
    for (int e = 0; e < ntab; e++) {
      u32 s_ = (u32)fnv1a_host(keys + key_off[e], key_off[e + 1] - key_off[e]) & (cap - 1);
      while (slots[s_] != TSAT_NONE) s_ = (s_ + 1) & (cap - 1);
      slots[s_] = e;
    }
    dk.ensure(nbytes + 1);
    doff.ensure(ntab + 1);
    dv.ensure(ntab);
    dslots.ensure(cap);
    CUDA_OK(cudaMemcpyAsync(dk.p, keys, nbytes, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(doff.p, key_off, (ntab + 1) * sizeof(i64), cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(dv.p, vals, ntab * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(dslots.p, slots.data(), cap * sizeof(u32), cudaMemcpyHostToDevice, s));
    ct.keys = dk.p;
    ct.off = doff.p;
    ct.vals = dv.p;
    ct.slots = dslots.p;
    ct.mask = cap - 1;
  }
  d_costs.ensure(n + 1);
  ct.dump_node = TSAT_NONE;
  DevBuf<u32>& dmiss = sc.k_miss;
  if (strict) {
    dmiss.ensure(1);
    CUDA_OK(cudaMemsetAsync(dmiss.p, 0xFF, sizeof(u32), s));
    ct.miss = dmiss.p;
  }
  {
    // node: op 4 + koff 8 + flag 1 + cost 8; child: id 4 + parent 4 + analysis fields 48
    KTimer kt(*this, KG_COSTS, 21.0 * h.live + 56.0 * h.nkids, 1);
    k_node_costs<<<nblk(n, 128), 128, 0, s>>>(view(), ct, n, d_costs.p);
  }
  if (out) CUDA_OK(cudaMemcpyAsync(out, d_costs.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  u32 miss = TSAT_NONE;
  if (strict) CUDA_OK(cudaMemcpyAsync(&miss, dmiss.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  check_error();  // syncs the stream (the two reads above land first)
  if (miss != TSAT_NONE) {  // UnknownSignature for the first node in id order, with its rendered key (cost.py:170-172)
    DevBuf<char>& kb = sc.k_keyout;
    kb.ensure(512);
    ct.dump_node = miss;
    ct.key_out = kb.p;
    k_node_costs<<<1, 1, 0, s>>>(view(), ct, 1, d_costs.p);
    char key[512];
    CUDA_OK(cudaMemcpyAsync(key, kb.p, sizeof(key), cudaMemcpyDeviceToHost, s));
    sync();
    key[511] = 0;
    costs_valid_for = 0;
    throw TsatException(TSAT_ERR_UNKNOWN_SIG, std::string("no cost for ") + key);
  }
  costs_valid_for = n;
}

// ---------------------------------------------------------------- greedy

__global__ void k_untrimmed_g(const u32* level, u32 n, u32* list, u32* cnt) {
  GRID_STRIDE(i, n) if (level[i] == TSAT_NONE) list[atomicAdd(cnt, 1u)] = (u32)i;
}

void build_class_graph(Engine& e);
u32 trim_levels(Engine& e, const u8* mask, std::vector<u32>& lvl_off, u32& ntrimmed);
u32 bfs_classes(Engine& e, u32 root, u32* mark, u32* queue);
u32 bfs_graph(Engine& e, const u32* eoff, const u32* edst, u32 n, u32 root, u32* mark, u32* queue);

__global__ void k_sel_count(G g, const u32* bn, u32 C, u32* cnt) {
  GRID_STRIDE(i, C) {
    u32 m = bn[i];
    cnt[i] = m == TSAT_NONE ? 0u : g.koff[m + 1] - g.koff[m];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[C] = 0;
}

__global__ void k_sel_fill(G g, const u32* bn, const u32* cls_index, u32 C, const u32* eoff, u32* edst) {
  GRID_STRIDE(i, C) {
    u32 m = bn[i];
    if (m == TSAT_NONE) continue;
    u32 o = eoff[i];
    for (u32 j = g.koff[m]; j < g.koff[m + 1]; j++) edst[o++] = cls_index[uf_find_ro(g.parent, g.kids[j])];
  }
}

__global__ void k_sel_missing(const u32* q, u32 k, const u32* bn, u32* flag) {
  GRID_STRIDE(t, k) if (bn[q[t]] == TSAT_NONE) *flag = 1;
}

__device__ __forceinline__ void greedy_fold(const G& g, const u32* cls_off, const u32* cls_nodes,
                                            const u32* cls_index, u32 i, const double* cost, const double* pc,
                                            double& bc, u32& bn) {
  for (u32 k = cls_off[i]; k < cls_off[i + 1]; k++) {
    u32 m = cls_nodes[k];
    if (g.flags[m] & NF_FILT) continue;
    double tot = cost[m];
    for (u32 j = g.koff[m]; j < g.koff[m + 1]; j++) tot += pc[cls_index[uf_find_ro(g.parent, g.kids[j])]];
    if (isinf(tot)) continue;
    if (tot < bc - 1e-15 || (fabs(tot - bc) <= 1e-15 && (bn == TSAT_NONE || m < bn))) {
      bc = tot;
      bn = m;
    }
  }
}

__global__ void k_greedy_init(double* bc, u32* bn, u32 n) {
  GRID_STRIDE(i, n) {
    bc[i] = INFINITY;
    bn[i] = TSAT_NONE;
  }
}

// Greedy over the peel levels of a small class graph in ONE CTA.
// A prologue lays the trimmed classes' members out in peel order (q index):
// node id, cost (NaN when filtered) and child classes (the class graph's
// member edges, child order kept so the fp64 sums match the reference).
// Per level: (A) one thread per member computes its total from the children's
// best costs held in shared memory; (B) one thread per class folds its
// members in id order with the reference rule (extract.py:145-152: a member
// replaces the running best only when cheaper by more than 1e-15; with
// ascending ids the tie clause never fires).
__global__ void k_gather_at(const u32* src, const u32* idx, u32 n, u32* out) {
  GRID_STRIDE(i, n) out[i] = src[idx[i]];
}

__global__ void k_gq_count(const u32* order, u32 ntr, const u32* cls_off, u32* cnt) {
  GRID_STRIDE(t, ntr) {
    u32 i = order[t];
    cnt[t] = cls_off[i + 1] - cls_off[i];
  }
}

// member-parallel fill: slot_of[q] (the peel-order class slot of member q)
// comes from a max-scan of the slot heads, so big classes do not serialise
__global__ void k_gq_heads(const u32* lvm_off, u32 ntr, u32* head) {
  GRID_STRIDE(t, ntr) {
    if (lvm_off[t + 1] > lvm_off[t]) head[lvm_off[t]] = (u32)t;
  }
}

__global__ void k_gq_fill(G g, const u32* order, u32 nq, const u32* slot_of, const u32* cls_off, const u32* cls_nodes,
                          const u32* moff, const u32* lvm_off, const double* cost, u32* qk, u32* qnode,
                          double* qcost, u32* qdeg) {
  GRID_STRIDE(q0, nq) {
    u32 q = (u32)q0;
    u32 t = slot_of[q];
    u32 k = cls_off[order[t]] + (q - lvm_off[t]);
    u32 m = cls_nodes[k];
    qk[q] = k;
    qnode[q] = m;
    bool f = (g.flags[m] & NF_FILT) != 0;
    qcost[q] = f ? NAN : cost[m];
    qdeg[q] = moff[k + 1] - moff[k];
  }
}

__global__ void k_gq_edges(u32 nq, const u32* qk, const u32* moff, const u32* edst, const u32* qeoff, u32* qedst) {
  GRID_STRIDE(q, nq) {
    u32 k = qk[q], o = qeoff[q];
    for (u32 e = moff[k]; e < moff[k + 1]; e++) qedst[o++] = edst[e];
  }
}

// phase A: member totals (children's best costs); phase B: per-class fold
__device__ __forceinline__ void gq_totals(u32 qa, u32 qb, u64 tid, u64 nth, const double* qcost, const u32* qeoff,
                                          const u32* qedst, const double* bc, double* qtot) {
  for (u64 q = qa + tid; q < qb; q += nth) {
    double tot = qcost[q];
    if (!isnan(tot))
      for (u32 e = qeoff[q], e1 = qeoff[q + 1]; e < e1; e++) tot += bc[qedst[e]];
    qtot[q] = tot;
  }
}

// sequential fold over members [q0, q1) in id order (extract.py:145-152)
__device__ __forceinline__ void gq_fold_seq(u32 q0, u32 q1, const double* qtot, double& c, u32& best) {
  c = INFINITY;
  best = TSAT_NONE;
  for (u32 q = q0; q < q1; q++) {
    double tot = qtot[q];
    if (isnan(tot) || isinf(tot)) continue;
    if (tot < c - 1e-15) {
      c = tot;
      best = q;
    }
  }
}

// Classes with more than 32 members are folded by a warp: the sequential
// rule picks the first member attaining the minimum unless some total lies in
// (min, min + 1e-15] (then the chain of near-ties decides: lane 0 replays the
// sequential fold).  Smaller classes: one thread each.
#define GQ_BIG 32u
__device__ __forceinline__ void gq_fold(u32 a, u32 b, u64 tid, u64 nth, const u32* order, const u32* lvm_off,
                                        const u32* qnode, const double* qtot, double* bc, u32* bn, bool big) {
  for (u64 t = a + tid; t < b; t += nth) {
    u32 q0 = lvm_off[t], q1 = lvm_off[t + 1];
    if (q1 - q0 > GQ_BIG) continue;
    double c;
    u32 best;
    gq_fold_seq(q0, q1, qtot, c, best);
    u32 i = order[t];
    bc[i] = c;
    bn[i] = best == TSAT_NONE ? TSAT_NONE : qnode[best];
  }
  if (!big) return;  // no class of this level has more than GQ_BIG members
  const u32 lane = (u32)(tid & 31);
  for (u64 t = a + (tid >> 5); t < b; t += nth >> 5) {
    u32 q0 = lvm_off[t], q1 = lvm_off[t + 1];
    if (q1 - q0 <= GQ_BIG) continue;
    double m = INFINITY;
    u32 mi = TSAT_NONE;
    for (u32 q = q0 + lane; q < q1; q += 32) {
      double tot = qtot[q];
      if (isnan(tot) || isinf(tot)) continue;
      if (tot < m) {  // lanes walk ascending q: keeps the first occurrence
        m = tot;
        mi = q;
      }
    }
    for (int o = 16; o; o >>= 1) {
      double m2 = __shfl_xor_sync(0xffffffffu, m, o);
      u32 i2 = __shfl_xor_sync(0xffffffffu, mi, o);
      if (m2 < m || (m2 == m && i2 < mi)) {
        m = m2;
        mi = i2;
      }
    }
    bool near = false;
    if (mi != TSAT_NONE)
      for (u32 q = q0 + lane; q < q1; q += 32) {
        double tot = qtot[q];
        if (!isnan(tot) && !isinf(tot) && tot > m && tot <= m + 1e-15) near = true;
      }
    near = __any_sync(0xffffffffu, near);
    if (lane == 0) {
      double c = m;
      u32 best = mi;
      if (near) gq_fold_seq(q0, q1, qtot, c, best);
      u32 i = order[t];
      bc[i] = best == TSAT_NONE ? INFINITY : c;
      bn[i] = best == TSAT_NONE ? TSAT_NONE : qnode[best];
    }
  }
}

// levels [l0, l1) in ONE CTA (thin levels: a barrier per phase instead of a
// launch); best costs in shared memory when the whole class set fits
// (``smem``: then this launch covers every level), else in HBM
__device__ __forceinline__ void greedy_range(u32 l0, u32 l1, const u32* order, const u32* lvl_off,
                                             const u32* lvm_off, const u32* qnode, const double* qcost,
                                             const u32* qeoff, const u32* qedst, double* qtot, double* bc, u32* bn,
                                             const u32* bigflag, double* s_run, u32* s_cls, u32& s_len, u32& s_next) {
  u32 next_check = l0;
  for (u32 l = l0; l < l1;) {
    // Runs of single-member levels (deep chains such as the noop spine of
    // make_single_rooted): warp 0 prefetches up to 32 levels at once -- one
    // level per lane, its member, cost and the child best costs that lie
    // below the run -- then folds them in level order with __syncwarp only,
    // in-run children read from shared memory.  Same fp64 sums in the same
    // order as gq_totals / gq_fold_seq.
    if (l >= next_check) {
    if (threadIdx.x < 32) {
      const u32 lane = threadIdx.x, lv = l + lane;
      u32 q = 0, deg = 0, ea = 0, cls = TSAT_NONE;
      bool one = false;
      if (lv < l1) {
        u32 a = lvl_off[lv];
        if (lvl_off[lv + 1] == a + 1) {
          q = lvm_off[a];
          if (lvm_off[a + 1] == q + 1) {
            ea = qeoff[q];
            deg = qeoff[q + 1] - ea;
            cls = order[a];
            one = deg <= 8;
          }
        }
      }
      unsigned good = __ballot_sync(0xffffffffu, one), bad = ~good;
      u32 len = bad ? (u32)(__ffs(bad) - 1) : 32u;
      unsigned pairs = good & (good >> 1);
      if (len >= 2) {
        s_cls[lane] = cls;
        __syncwarp();
        double cst = 0.0, val[8];
        int src[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
          src[j] = -1;
          val[j] = 0.0;
        }
        if (lane < len) {
          cst = qcost[q];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            if ((u32)j < deg) {
              u32 d = qedst[ea + j];
              for (u32 k = 0; k < lane; k++)
                if (s_cls[k] == d) src[j] = (int)k;
              if (src[j] < 0) val[j] = bc[d];
            }
          }
        }
        for (u32 k = 0; k < len; k++) {
          if (lane == k) {
            double tot = cst;
            if (!isnan(tot))
#pragma unroll
              for (int j = 0; j < 8; j++)
                if ((u32)j < deg) tot += src[j] >= 0 ? s_run[src[j]] : val[j];
            bool ok = !(isnan(tot) || isinf(tot));
            double c = ok ? tot : INFINITY;
            s_run[k] = c;
            qtot[q] = tot;
            bc[cls] = c;
            bn[cls] = ok ? qnode[q] : TSAT_NONE;
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        s_len = len;
        s_next = pairs ? l + (u32)(__ffs(pairs) - 1) : l + 31;
      }
    }
    __syncthreads();
    const u32 len = s_len, nxt = s_next;
    __syncthreads();
    if (len >= 2) {
      l += len;
      next_check = l;
      continue;
    }
    next_check = nxt;
    }
    u32 a = lvl_off[l], b = lvl_off[l + 1];
    gq_totals(lvm_off[a], lvm_off[b], threadIdx.x, blockDim.x, qcost, qeoff, qedst, bc, qtot);
    __syncthreads();
    gq_fold(a, b, threadIdx.x, blockDim.x, order, lvm_off, qnode, qtot, bc, bn, bigflag[l] != 0);
    __syncthreads();
    l++;
  }
}

// Stage area of k_greedy_cta (batches of levels copied to shared memory)
#define GQ_LV 512u
#define GQ_T 1024u
#define GQ_Q 2048u
#define GQ_E 4096u
#define GQ_STAGE_BYTES (2u * GQ_Q * 8u + 4u * (GQ_LV + 1 + GQ_T + 1 + GQ_T + GQ_Q + 1 + GQ_Q + GQ_E))

// levels [l0, l1) in ONE CTA (thin levels: a barrier per phase instead of a
// launch); best costs in shared memory when the whole class set fits
// (``smem``: then this launch covers every level), else in HBM.  With
// ``nbatch``, batches of levels -- their class / member offsets, member
// costs, nodes and child lists, all contiguous in peel order -- are copied to
// shared memory with coalesced loads first, so a level costs barriers and
// shared-memory work instead of dependent L2 round trips.
__global__ void __launch_bounds__(1024) k_greedy_cta(const u32* order, const u32* lvl_off, u32 l0, u32 l1, u32 ntr,
                                                     const u32* lvm_off, const u32* qnode, const double* qcost,
                                                     const u32* qeoff, const u32* qedst, double* qtot, double* bc_g,
                                                     u32* bn, int smem, const u32* bigflag, u32 ncls_smem,
                                                     const u32* batch, u32 nbatch) {
  extern __shared__ double s_bc[];
  __shared__ double s_run[32];
  __shared__ u32 s_cls[32], s_len, s_next;
  double* bc = smem ? s_bc : bc_g;
  if (nbatch) {
    double* s_qcost = s_bc + (smem ? ncls_smem : 0);
    double* s_qtot = s_qcost + GQ_Q;
    u32* s_lv = (u32*)(s_qtot + GQ_Q);
    u32* s_lvm = s_lv + GQ_LV + 1;
    u32* s_ord = s_lvm + GQ_T + 1;
    u32* s_qeoff = s_ord + GQ_T;
    u32* s_qnode = s_qeoff + GQ_Q + 1;
    u32* s_qedst = s_qnode + GQ_Q;
    for (u32 bi = 0; bi < nbatch; bi++) {
      const u32 lb = batch[3 * bi], le = batch[3 * bi + 1];
      if (!batch[3 * bi + 2]) {
        greedy_range(lb, le, order, lvl_off, lvm_off, qnode, qcost, qeoff, qedst, qtot, bc, bn, bigflag, s_run,
                     s_cls, s_len, s_next);
        __syncthreads();
        continue;
      }
      const u32 t0 = lvl_off[lb], t1 = lvl_off[le];
      const u32 q0 = lvm_off[t0], q1 = lvm_off[t1];
      const u32 e0 = qeoff[q0], e1 = qeoff[q1];
      for (u32 x = threadIdx.x; x <= le - lb; x += blockDim.x) s_lv[x] = lvl_off[lb + x];
      for (u32 x = threadIdx.x; x <= t1 - t0; x += blockDim.x) s_lvm[x] = lvm_off[t0 + x];
      for (u32 x = threadIdx.x; x < t1 - t0; x += blockDim.x) s_ord[x] = order[t0 + x];
      for (u32 x = threadIdx.x; x <= q1 - q0; x += blockDim.x) s_qeoff[x] = qeoff[q0 + x];
      for (u32 x = threadIdx.x; x < q1 - q0; x += blockDim.x) {
        s_qcost[x] = qcost[q0 + x];
        s_qnode[x] = qnode[q0 + x];
      }
      for (u32 x = threadIdx.x; x < e1 - e0; x += blockDim.x) s_qedst[x] = qedst[e0 + x];
      __syncthreads();
      // base-shifted views: the level code indexes with global positions
      greedy_range(lb, le, s_ord - t0, s_lv - lb, s_lvm - t0, s_qnode - q0, s_qcost - q0, s_qeoff - q0,
                   s_qedst - e0, s_qtot - q0, bc, bn, bigflag, s_run, s_cls, s_len, s_next);
      __syncthreads();
    }
  } else {
    greedy_range(l0, l1, order, lvl_off, lvm_off, qnode, qcost, qeoff, qedst, qtot, bc, bn, bigflag, s_run, s_cls,
                 s_len, s_next);
  }
  __syncthreads();
  if (smem)
    for (u32 t = threadIdx.x; t < ntr; t += blockDim.x) {
      u32 i = order[t];
      bc_g[i] = s_bc[i];
    }
}
// one wide level on the whole GPU (two launches: totals, then folds)
__global__ void k_gq_totals_wide(u32 qa, u32 qb, const double* qcost, const u32* qeoff, const u32* qedst,
                                 const double* bc, double* qtot) {
  gq_totals(qa, qb, blockIdx.x * (u64)blockDim.x + threadIdx.x, (u64)gridDim.x * blockDim.x, qcost, qeoff, qedst, bc,
            qtot);
}

__global__ void k_gq_fold_wide(u32 a, u32 b, const u32* order, const u32* lvm_off, const u32* qnode,
                               const double* qtot, double* bc, u32* bn, int big) {
  gq_fold(a, b, blockIdx.x * (u64)blockDim.x + threadIdx.x, (u64)gridDim.x * blockDim.x, order, lvm_off, qnode, qtot,
          bc, bn, big != 0);
}

// Sharded wide level (extraction relaxation partitioned by
// e-class range, class-cost vectors all-gathered): rank r folds the level's
// class slots [a + r*chunk, ...) -- member totals for members of those slots
// only -- and packs {best cost, node} per slot; after the all-gather every
// rank scatters the whole level back into its best-cost arrays.
__global__ void k_gq_totals_slots(u32 qa, u32 qb, u32 t_lo, u32 t_hi, const u32* slot_of, const double* qcost,
                                  const u32* qeoff, const u32* qedst, const double* bc, double* qtot) {
  GRID_STRIDE(q0, (u64)(qb - qa)) {
    u32 q = qa + (u32)q0, t = slot_of[q];
    if (t < t_lo || t >= t_hi) continue;
    double tot = qcost[q];
    if (!isnan(tot))
      for (u32 e = qeoff[q], e1 = qeoff[q + 1]; e < e1; e++) tot += bc[qedst[e]];
    qtot[q] = tot;
  }
}

__global__ void k_gq_pack(u32 t_lo, u32 t_hi, const u32* order, const double* bc, const u32* bn, double* rec) {
  GRID_STRIDE(k, (u64)(t_hi - t_lo)) {
    u32 i = order[t_lo + k];
    rec[2 * k] = bc[i];
    rec[2 * k + 1] = __longlong_as_double((long long)bn[i]);
  }
}

__global__ void k_gq_unpack(u32 a, u32 b, const u32* order, const double* rec, double* bc, u32* bn) {
  GRID_STRIDE(k, (u64)(b - a)) {
    u32 i = order[a + k];
    bc[i] = rec[2 * k];
    bn[i] = (u32)__double_as_longlong(rec[2 * k + 1]);
  }
}

// levels holding a class with more than GQ_BIG members
__global__ void k_gq_bigflags(const u32* order, const u32* lvm_off, u32 ntr, const u32* level, u32* flag) {
  GRID_STRIDE(t, ntr) {
    if (lvm_off[t + 1] - lvm_off[t] > GQ_BIG) flag[level[order[t]]] = 1;
  }
}

// Jacobi round over the classes left on cycles
__global__ void k_greedy_round(G g, const u32* cls_off, const u32* cls_nodes, const u32* cls_index,
                               const u32* list, u32 nl, const double* cost, const double* pc, const u32* pn,
                               double* nc, u32* nn, u32* changed) {
  GRID_STRIDE(t, nl) {
    u32 i = list[t];
    double bc = pc[i];
    u32 bn = pn[i];
    greedy_fold(g, cls_off, cls_nodes, cls_index, i, cost, pc, bc, bn);
    nc[i] = bc;
    nn[i] = bn;
    if (bn != pn[i] || !(bc == pc[i])) *changed = 1;
  }
}

__global__ void k_copy_list(const u32* list, u32 nl, const double* sc_, const u32* sn, double* dc, u32* dn) {
  GRID_STRIDE(t, nl) {
    u32 i = list[t];
    dc[i] = sc_[i];
    dn[i] = sn[i];
  }
}

// reached selection (extract.py:74-91): BFS over chosen nodes from the root
__global__ void k_sel_coop(G g, const u32* cls_index, const u32* bn, u32 n, u32 root, u32* mark, u32* queue,
                           u32* ctl) {
  cg::grid_group grid = cg::this_grid();
  GRID_STRIDE(i, n) mark[i] = 0;
  grid.sync();
  if (grid.thread_rank() == 0) {
    mark[root] = 1;
    queue[0] = root;
    ctl[0] = 1;
  }
  grid.sync();
  u32 start = 0, end = 1;
  while (start < end) {
    for (u64 t = start + grid.thread_rank(); t < end; t += grid.size()) {
      u32 i = queue[t];
      u32 m = bn[i];
      if (m == TSAT_NONE) {
        ctl[1] = 1;
        continue;
      }
      for (u32 j = g.koff[m]; j < g.koff[m + 1]; j++) {
        u32 c = cls_index[uf_find_ro(g.parent, g.kids[j])];
        if (mark[c] == 0 && atomicCAS(&mark[c], 0u, 1u) == 0u) queue[atomicAdd(&ctl[0], 1u)] = c;
      }
    }
    grid.sync();
    start = end;
    end = ((volatile u32*)ctl)[0];
    grid.sync();
  }
}

// Reached selection by a top-down sweep of the peel levels (a chosen node's
// children sit on strictly lower levels), instead of a BFS whose depth is the
// selection's depth (the 1,416-level noop spine at config 5).  One CTA walks
// levels [lo, hi) downwards; runs of single-class levels go to warp 0, which
// loads up to 32 levels at once (class, mark, children) and propagates marks
// through the run in shared memory; other levels: one barrier each.
__global__ void __launch_bounds__(1024) k_sel_cta(const u32* order, const u32* lvl_off, u32 lo, u32 hi,
                                                  const u32* eoff, const u32* edst, u32* mark) {
  __shared__ u32 s_cls[32], s_mk[32], s_len, s_next;
  u32 next_check = hi;  // levels at or below this index get a run check
  for (u32 l = hi; l > lo;) {
    if (l <= next_check) {
      if (threadIdx.x < 32) {
        const u32 lane = threadIdx.x;
        const long long lvs = (long long)l - 1 - lane;
        u32 cls = TSAT_NONE, ea = 0, deg = 0;
        bool one = false;
        if (lvs >= (long long)lo) {
          u32 a = lvl_off[lvs];
          if (lvl_off[lvs + 1] == a + 1) {
            cls = order[a];
            ea = eoff[cls];
            deg = eoff[cls + 1] - ea;
            one = deg <= 8;
          }
        }
        unsigned good = __ballot_sync(0xffffffffu, one), bad = ~good;
        u32 len = bad ? (u32)(__ffs(bad) - 1) : 32u;
        unsigned pairs = good & (good >> 1);
        if (len >= 2) {
          s_cls[lane] = cls;
          s_mk[lane] = 0;
          u32 gm = lane < len ? mark[cls] : 0u;
          u32 d[8];
          int src[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            d[j] = TSAT_NONE;
            src[j] = -1;
          }
          __syncwarp();
          if (lane < len) {
#pragma unroll
            for (int j = 0; j < 8; j++)
              if ((u32)j < deg) {
                d[j] = edst[ea + j];
                for (u32 k = lane + 1; k < len; k++)
                  if (s_cls[k] == d[j]) src[j] = (int)k;
              }
          }
          for (u32 k = 0; k < len; k++) {
            if (lane == k && (gm || s_mk[k])) {
#pragma unroll
              for (int j = 0; j < 8; j++)
                if ((u32)j < deg) {
                  if (src[j] >= 0) s_mk[src[j]] = 1;
                  else mark[d[j]] = 1;
                }
              if (!gm) mark[cls] = 1;
            }
            __syncwarp();
          }
        }
        if (lane == 0) {
          s_len = len;
          s_next = pairs ? l - 1 - (u32)(__ffs(pairs) - 1) : (l > 31 ? l - 31 : 0);
        }
      }
      __syncthreads();
      const u32 len = s_len, nxt = s_next;
      __syncthreads();
      if (len >= 2) {
        l -= len;
        next_check = l;
        continue;
      }
      next_check = nxt + 1;
    }
    const u32 a = lvl_off[l - 1], b = lvl_off[l];
    for (u32 t = a + threadIdx.x; t < b; t += blockDim.x) {
      u32 i = order[t];
      if (mark[i])
        for (u32 e = eoff[i], e1 = eoff[i + 1]; e < e1; e++) mark[edst[e]] = 1;
    }
    __syncthreads();
    l--;
  }
}

// one wide level of the top-down sweep on the whole GPU
__global__ void k_sel_wide(const u32* order, u32 a, u32 b, const u32* eoff, const u32* edst, u32* mark) {
  GRID_STRIDE(t0, (u64)(b - a)) {
    u32 i = order[a + (u32)t0];
    if (mark[i])
      for (u32 e = eoff[i], e1 = eoff[i + 1]; e < e1; e++) mark[edst[e]] = 1;
  }
}

__global__ void k_sel_flags(const u32* mark, u32 C, u32* fl) {
  GRID_STRIDE(i, (u64)C + 1) fl[i] = (i < C && mark[i]) ? 1u : 0u;
}

__global__ void k_sel_compact(const u32* mark, const u32* pos, u32 C, const u32* cls_ids, const u32* bn, u32* oc,
                              u32* on, u32* missing) {
  GRID_STRIDE(i, C) {
    if (!mark[i]) continue;
    u32 p = pos[i];
    oc[p] = cls_ids[i];
    on[p] = bn[i];
    if (bn[i] == TSAT_NONE) *missing = 1;
  }
}

__global__ void k_root_info(G g, u32 root, const u32* cls_index, const double* bc, double* out) {
  u32 rd = cls_index[uf_find_ro(g.parent, root)];
  out[0] = __longlong_as_double((long long)rd);
  out[1] = bc[rd];
}

static inline long long __double_as_longlong_host(double d) {
  long long x;
  memcpy(&x, &d, sizeof(x));
  return x;
}

__global__ void k_sel_collect(const u32* queue, u32 k, const u32* cls_ids, const u32* bn, u32* oc, u32* on) {
  GRID_STRIDE(t, k) {
    u32 i = queue[t];
    oc[t] = cls_ids[i];
    on[t] = bn[i];
  }
}

double Engine::greedy(const double* cost_by_node, u32* sel_cls, u32* sel_node, u32* nsel, i64* rounds) {
  if (root == TSAT_NONE) throw TsatException(TSAT_ERR_STATE, "e-graph has no root");
  if (!snap.valid) build_snapshot();
  u32 n = h.next_id, C = snap.ncls;
  DevBuf<double>& upl = sc.g_upl;
  const double* cost = d_costs.p;
  if (cost_by_node) {
    upl.ensure(n + 1);
    CUDA_OK(cudaMemcpyAsync(upl.p, cost_by_node, n * sizeof(double), cudaMemcpyHostToDevice, s));
    cost = upl.p;
  } else if (costs_valid_for != n) {
    throw TsatException(TSAT_ERR_STATE, "device cost vector is stale; recompute egraph_costs");
  }
  KTimer kt(*this, KG_GREEDY, 0.0, 0);
  DevBuf<double>& c0 = sc.g_c0;
  DevBuf<double>& c1 = sc.g_c1;
  DevBuf<u32>& n0 = sc.g_n0;
  DevBuf<u32>& n1 = sc.g_n1;
  DevBuf<u32>& flag = sc.g_flag;
  c0.ensure(C + 1);
  c1.ensure(C + 1);
  n0.ensure(C + 1);
  n1.ensure(C + 1);
  flag.ensure(4);
  ensure_levels();
  const std::vector<u32>& lo = lv_off;
  u32 ntr = lv_trimmed;
  u32 nl = lv_n;
  k_greedy_init<<<nblk(C), 256, 0, s>>>(c0.p, n0.p, C);
  G gv = view();
  const u32 *co = snap.cls_off.p, *cn = snap.cls_nodes.p, *ci = snap.cls_index.p, *ord = sc.c_order.p,
            *lvl = sc.c_lvloff.p;
  // peel-order member layout (q index): node, cost (NaN when filtered), child classes
  Scratch& X = sc;
  X.gq_lvm.ensure(ntr + 1);
  X.gq_cnt.ensure(ntr + 1);
  k_gq_count<<<nblk(ntr), 256, 0, s>>>(ord, ntr, co, X.gq_cnt.p);
  CUDA_OK(cudaMemsetAsync(X.gq_cnt.p + ntr, 0, sizeof(u32), s));
  dev_exclusive_scan_u32(*this, X.gq_cnt.p, X.gq_lvm.p, ntr + 1);
  std::vector<u32> lvm(nl + 1), bigf(nl + 1);
  DevBuf<u32>& bflag = X.gq_big;
  bflag.ensure(nl + 1);
  {
    // member offsets at level boundaries (host: picks thin runs / wide levels)
    DevBuf<u32>& lb = X.gq_lb;
    lb.ensure(nl + 1);
    k_gather_at<<<nblk(nl + 1), 256, 0, s>>>(X.gq_lvm.p, lvl, nl + 1, lb.p);
    CUDA_OK(cudaMemsetAsync(bflag.p, 0, (nl + 1) * sizeof(u32), s));
    k_gq_bigflags<<<nblk(ntr), 256, 0, s>>>(ord, X.gq_lvm.p, ntr, sc.cg_level.p, bflag.p);
    CUDA_OK(cudaMemcpyAsync(lvm.data(), lb.p, (nl + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(bigf.data(), bflag.p, (nl + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
  }
  u32 nq = lvm[nl];
  X.gq_k.ensure(nq + 1);
  X.gq_node.ensure(nq + 1);
  X.gq_cost.ensure(nq + 1);
  X.gq_tot.ensure(nq + 1);
  X.gq_deg.ensure(nq + 1);
  X.gq_eoff.ensure(nq + 1);
  {
    DevBuf<u32>& head = X.gq_head;
    DevBuf<u32>& slot = X.gq_slot;
    head.ensure(nq + 1);
    slot.ensure(nq + 1);
    CUDA_OK(cudaMemsetAsync(head.p, 0, (nq + 1) * sizeof(u32), s));
    k_gq_heads<<<nblk(ntr), 256, 0, s>>>(X.gq_lvm.p, ntr, head.p);
    if (nq) {
      size_t bytes = 0;
      CUDA_OK(cub::DeviceScan::InclusiveScan(nullptr, bytes, head.p, slot.p, cuda::maximum<>{}, nq, s));
      temp.ensure(bytes + 16);
      CUDA_OK(cub::DeviceScan::InclusiveScan(temp.p, bytes, head.p, slot.p, cuda::maximum<>{}, nq, s));
    }
    k_gq_fill<<<nblk(nq), 256, 0, s>>>(gv, ord, nq, slot.p, co, cn, sc.cg_moff.p, X.gq_lvm.p, cost, X.gq_k.p,
                                       X.gq_node.p, X.gq_cost.p, X.gq_deg.p);
  }
  CUDA_OK(cudaMemsetAsync(X.gq_deg.p + nq, 0, sizeof(u32), s));
  dev_exclusive_scan_u32(*this, X.gq_deg.p, X.gq_eoff.p, nq + 1);
  X.gq_edst.ensure((u64)cg_ne + 1);
  k_gq_edges<<<nblk(nq), 256, 0, s>>>(nq, X.gq_k.p, sc.cg_moff.p, sc.cg_edst.p, X.gq_eoff.p, X.gq_edst.p);
  const u64 GREEDY_SMEM = 200u << 10;
  static int smem_set = 0;
  if (!smem_set) {
    CUDA_OK(cudaFuncSetAttribute(k_greedy_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GREEDY_SMEM));
    smem_set = 1;
  }
  if ((u64)C * sizeof(double) <= GREEDY_SMEM) {
    static const bool no_stage = getenv("TSAT_GREEDY_NOSTAGE") != nullptr;
    u32 nbatch = 0;
    if (!no_stage && (u64)C * sizeof(double) + GQ_STAGE_BYTES <= GREEDY_SMEM && nl) {
      // edge offsets at level boundaries -> batches of levels that fit the stage area
      DevBuf<u32>& eb_d = X.gq_head;  // free after the member fill
      eb_d.ensure(nl + 2);
      k_gather_at<<<nblk(nl + 1), 256, 0, s>>>(X.gq_eoff.p, X.gq_lb.p, nl + 1, eb_d.p);
      std::vector<u32> eb(nl + 1);
      CUDA_OK(cudaMemcpyAsync(eb.data(), eb_d.p, (nl + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      std::vector<u32> bt;
      for (u32 l = 0; l < nl;) {
        u32 le = l;
        while (le < nl && le + 1 - l <= GQ_LV && lo[le + 1] - lo[l] <= GQ_T && lvm[le + 1] - lvm[l] <= GQ_Q &&
               eb[le + 1] - eb[l] <= GQ_E)
          le++;
        if (le == l) {
          bt.insert(bt.end(), {l, l + 1, 0u});
          l++;
        } else {
          bt.insert(bt.end(), {l, le, 1u});
          l = le;
        }
      }
      nbatch = (u32)(bt.size() / 3);
      X.gq_batch.ensure(bt.size() + 1);
      CUDA_OK(cudaMemcpyAsync(X.gq_batch.p, bt.data(), bt.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    }
    size_t dyn = (size_t)C * sizeof(double) + (nbatch ? GQ_STAGE_BYTES : 0);
    k_greedy_cta<<<1, 1024, dyn, s>>>(ord, lvl, 0, nl, ntr, X.gq_lvm.p, X.gq_node.p, X.gq_cost.p, X.gq_eoff.p,
                                      X.gq_edst.p, X.gq_tot.p, c0.p, n0.p, 1, bflag.p, C, X.gq_batch.p, nbatch);
  } else {
    // thin runs in one CTA, wide levels (> WIDE members or classes) on the grid
    const u32 WIDE = 8192;
    for (u32 l = 0; l < nl;) {
      u32 wm = lvm[l + 1] - lvm[l], wc = lo[l + 1] - lo[l];
      if ((wm > WIDE || wc > WIDE) && shard_world > 1) {
        // class slots split across the shard ranks, {cost, node} all-gathered.
        // Without a communicator (single-GPU shard tests) every rank's slice
        // is computed here in turn -- the same slicing, packing and unpacking.
        const u32 W = (u32)shard_world, a = lo[l], b = lo[l + 1], chunk = (wc + W - 1) / W;
        X.gq_pack.ensure(2ull * chunk + 2);
        X.gq_recv.ensure(2ull * chunk * W + 2);
        for (u32 r = 0; r < W; r++) {
          if (shard_exchange() && (int)r != shard_rank) continue;
          u32 ta = std::min(b, a + r * chunk), tb = std::min(b, ta + chunk);
          if (tb > ta) {
            k_gq_totals_slots<<<nblk(wm), 256, 0, s>>>(lvm[l], lvm[l + 1], ta, tb, X.gq_slot.p, X.gq_cost.p,
                                                        X.gq_eoff.p, X.gq_edst.p, c0.p, X.gq_tot.p);
            k_gq_fold_wide<<<nblk(bigf[l] ? (u64)(tb - ta) * 32 : tb - ta), 256, 0, s>>>(
                ta, tb, ord, X.gq_lvm.p, X.gq_node.p, X.gq_tot.p, c0.p, n0.p, bigf[l]);
          }
          double* dst = shard_exchange() ? X.gq_pack.p : X.gq_recv.p + 2ull * chunk * r;
          if (tb > ta) k_gq_pack<<<nblk(tb - ta), 256, 0, s>>>(ta, tb, ord, c0.p, n0.p, dst);
        }
        if (shard_exchange()) shard_allgather_bytes(X.gq_pack.p, X.gq_recv.p, 2ull * chunk * sizeof(double));
        k_gq_unpack<<<nblk(wc), 256, 0, s>>>(a, b, ord, X.gq_recv.p, c0.p, n0.p);
        l++;
        continue;
      }
      if (wm > WIDE || wc > WIDE) {
        k_gq_totals_wide<<<nblk(wm), 256, 0, s>>>(lvm[l], lvm[l + 1], X.gq_cost.p, X.gq_eoff.p, X.gq_edst.p, c0.p,
                                                   X.gq_tot.p);
        k_gq_fold_wide<<<nblk(bigf[l] ? (u64)wc * 32 : wc), 256, 0, s>>>(lo[l], lo[l + 1], ord, X.gq_lvm.p,
                                                                         X.gq_node.p, X.gq_tot.p, c0.p, n0.p, bigf[l]);
        l++;
        continue;
      }
      u32 l1 = l;
      while (l1 < nl && lvm[l1 + 1] - lvm[l1] <= WIDE && lo[l1 + 1] - lo[l1] <= WIDE) l1++;
      k_greedy_cta<<<1, 1024, 0, s>>>(ord, lvl, l, l1, ntr, X.gq_lvm.p, X.gq_node.p, X.gq_cost.p, X.gq_eoff.p,
                                      X.gq_edst.p, X.gq_tot.p, c0.p, n0.p, 0, bflag.p, 0, nullptr, 0);
      l = l1;
    }
  }
  CUDA_OK(cudaGetLastError());
  i64 r = 1;
  if (ntr < C) {
    DevBuf<u32>& rest = sc.c_rest;
    rest.ensure(C - ntr + 1);
    CUDA_OK(cudaMemsetAsync(flag.p, 0, 2 * sizeof(u32), s));
    k_untrimmed_g<<<nblk(C), 256, 0, s>>>(sc.cg_level.p, C, rest.p, flag.p + 1);
    u32 nr = C - ntr;
    while (true) {
      r++;
      CUDA_OK(cudaMemsetAsync(flag.p, 0, sizeof(u32), s));
      k_greedy_round<<<nblk(nr, 128), 128, 0, s>>>(view(), co, cn, ci, rest.p, nr, cost, c0.p, n0.p, c1.p, n1.p,
                                                   flag.p);
      k_copy_list<<<nblk(nr), 256, 0, s>>>(rest.p, nr, c1.p, n1.p, c0.p, n0.p);
      u32 ch;
      CUDA_OK(cudaMemcpyAsync(&ch, flag.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      if (!ch) break;
    }
  }
  kt.bytes = 16.0 * h.live + 12.0 * h.nkids + 12.0 * C;
  kt.launches = 2;
  *rounds = r;
  // root class (dense) and its best cost in one round trip
  DevBuf<double>& rinfo = sc.g_rinfo;
  rinfo.ensure(2);
  k_root_info<<<1, 1, 0, s>>>(view(), root, snap.cls_index.p, c0.p, rinfo.p);
  double hri[2];
  CUDA_OK(cudaMemcpyAsync(hri, rinfo.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync();
  const u32 rd = (u32)__double_as_longlong_host(hri[0]);
  const double rcost = hri[1];
  if (std::isinf(rcost)) throw TsatException(TSAT_ERR_NO_FINITE, "every root selection has infinite cost");
  DevBuf<u32>& mark = sc.g_mark;
  DevBuf<u32>& q = sc.g_fa;
  mark.ensure(C + 1);
  q.ensure(C + 1);
  // selection graph: class -> child classes of its chosen node only
  {
    DevBuf<u32>& cnt = sc.g_cnt;
    cnt.ensure(C + 1);
    sc.g_eoff.ensure(C + 1);
    k_sel_count<<<nblk(C), 256, 0, s>>>(gv, n0.p, C, cnt.p);
    dev_exclusive_scan_u32(*this, cnt.p, sc.g_eoff.p, C + 1);
    // one chosen node per class: its children are at most all stored children
    // (no read-back of the exact count)
    sc.g_edst.ensure((u64)h.nkids + 1);
    k_sel_fill<<<nblk(C), 256, 0, s>>>(gv, n0.p, ci, C, sc.g_eoff.p, sc.g_edst.p);
  }
  DevBuf<u32>& oc = sc.g_oc;
  DevBuf<u32>& on = sc.g_on;
  oc.ensure(C + 1);
  on.ensure(C + 1);
  u32 k;
  static const int sel_mode = getenv("TSAT_SEL") ? atoi(getenv("TSAT_SEL")) : 0;  // debug: 1 BFS, 2 sweep
  u32 single_lv = 0;
  for (u32 l = 0; l < nl; l++) single_lv += lo[l + 1] - lo[l] == 1;
  if (getenv("TSAT_SEL_DEBUG")) fprintf(stderr, "greedy levels %u single %u classes %u\n", nl, single_lv, C);
  bool sweep = ntr == C && (sel_mode == 2 || (sel_mode == 0 && single_lv >= 256));
  if (sweep) {
    // every class peeled: top-down level sweep (k_sel_cta / k_sel_wide)
    CUDA_OK(cudaMemsetAsync(mark.p, 0, (size_t)(C + 1) * sizeof(u32), s));
    const u32 one = 1;
    CUDA_OK(cudaMemcpyAsync(mark.p + rd, &one, sizeof(u32), cudaMemcpyHostToDevice, s));
    const u32 WIDE = 8192;
    for (u32 l = nl; l > 0;) {
      u32 wc = lo[l] - lo[l - 1];
      if (wc > WIDE) {
        k_sel_wide<<<nblk(wc), 256, 0, s>>>(ord, lo[l - 1], lo[l], sc.g_eoff.p, sc.g_edst.p, mark.p);
        l--;
        continue;
      }
      u32 l0 = l;
      while (l0 > 0 && lo[l0] - lo[l0 - 1] <= WIDE) l0--;
      k_sel_cta<<<1, 1024, 0, s>>>(ord, lvl, l0, l, sc.g_eoff.p, sc.g_edst.p, mark.p);
      l = l0;
    }
    DevBuf<u32>& fl = sc.g_cnt;
    fl.ensure(C + 2);
    q.ensure(C + 2);
    k_sel_flags<<<nblk((u64)C + 1), 256, 0, s>>>(mark.p, C, fl.p);
    dev_exclusive_scan_u32(*this, fl.p, q.p, C + 1);
    CUDA_OK(cudaMemsetAsync(flag.p, 0, sizeof(u32), s));
    k_sel_compact<<<nblk(C), 256, 0, s>>>(mark.p, q.p, C, snap.cls_ids.p, n0.p, oc.p, on.p, flag.p);
    u32 hk[2];
    CUDA_OK(cudaMemcpyAsync(&hk[0], q.p + C, sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(&hk[1], flag.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    k = hk[0];
    if (hk[1]) throw TsatException(TSAT_ERR_STATE, "no selected node covers a reached e-class");
  } else {
    k = bfs_graph(*this, sc.g_eoff.p, sc.g_edst.p, C, rd, mark.p, q.p);
    CUDA_OK(cudaMemsetAsync(flag.p, 0, sizeof(u32), s));
    k_sel_missing<<<nblk(k), 256, 0, s>>>(q.p, k, n0.p, flag.p);
    k_sel_collect<<<nblk(k), 256, 0, s>>>(q.p, k, snap.cls_ids.p, n0.p, oc.p, on.p);
  }
  u32 miss = 0;
  if (!sweep) CUDA_OK(cudaMemcpyAsync(&miss, flag.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(sel_cls, oc.p, k * sizeof(u32), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(sel_node, on.p, k * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();  // one read-back: the coverage flag with the selection
  if (miss) throw TsatException(TSAT_ERR_STATE, "no selected node covers a reached e-class");
  *nsel = k;
  return rcost;
}
