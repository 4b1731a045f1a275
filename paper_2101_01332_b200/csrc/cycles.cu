// Cycle filtering on the GPU (reference: pkg/src/tensorsat/cycles.py).
//
// * build_reach: the per-iteration descendants map (cycles.py:70-148) as a
//   dense bitset over snapshot classes.  Classes are peeled in topological
//   levels (Kahn trimming on live, unfiltered class edges); each level ORs
//   its children's rows in one pass; classes left after trimming (on or above
//   a cycle) are closed by sweeping to a fixpoint.
// * break_all_cycles: the post-processing loop (cycles.py:172-245).  A level
//   trim restricted to classes reachable from the root proves the common
//   case "no live cycle" without a DFS; otherwise the exact lexicographic
//   DFS runs on one GPU thread over the untrimmed region only (trimmed
//   classes cannot lie on or lead to a cycle, so skipping them leaves the
//   back-edge sequence unchanged), then resolves cycles by filter-listing
//   their max node id, repeating passes until no cycle remains.
#include <cub/cub.cuh>

#include "engine.cuh"

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

struct ClassGraph {
  u32 ncls = 0;
  u64 nedge = 0;
  DevBuf<u32> eoff;   // ncls + 1
  DevBuf<u32> edst;   // dense child class per edge
  DevBuf<u32> enode;  // node id that contributes the edge
  DevBuf<u32> roff;   // reverse CSR
  DevBuf<u32> rsrc;
  DevBuf<u32> outdeg;
  DevBuf<u32> level;  // trim round, TSAT_NONE = untrimmed
};

// per class: number of edges through live, unfiltered members
__global__ void k_edge_count(G g, const u32* cls_off, const u32* cls_nodes, u32 ncls, u32* cnt) {
  GRID_STRIDE(i, ncls) {
    u32 c = 0;
    for (u32 k = cls_off[i]; k < cls_off[i + 1]; k++) {
      u32 m = cls_nodes[k];
      if (g.flags[m] & NF_FILT) continue;
      c += g.koff[m + 1] - g.koff[m];
    }
    cnt[i] = c;
  }
}

__global__ void k_edge_fill(G g, const u32* cls_off, const u32* cls_nodes, const u32* cls_index, u32 ncls,
                            const u32* eoff, u32* edst, u32* enode) {
  GRID_STRIDE(i, ncls) {
    u32 o = eoff[i];
    for (u32 k = cls_off[i]; k < cls_off[i + 1]; k++) {
      u32 m = cls_nodes[k];
      if (g.flags[m] & NF_FILT) continue;
      for (u32 j = g.koff[m]; j < g.koff[m + 1]; j++) {
        edst[o] = cls_index[uf_find_ro(g.parent, g.kids[j])];
        enode[o] = m;
        o++;
      }
    }
  }
}

__global__ void k_edge_src(const u32* eoff, u32 ncls, u32* esrc) {
  GRID_STRIDE(i, ncls) for (u32 e = eoff[i]; e < eoff[i + 1]; e++) esrc[e] = (u32)i;
}

__global__ void k_rhist(const u32* edst, u64 ne, u32* h) {
  GRID_STRIDE(e, ne) atomicAdd(&h[edst[e]], 1u);
}

__global__ void k_outdeg_init(const u32* eoff, u32 ncls, u32* outdeg, u32* level, u32* frontier,
                              u32* nfront, const u8* mask) {
  GRID_STRIDE(i, ncls) {
    level[i] = TSAT_NONE;
    if (mask && !mask[i]) continue;
    u32 d = eoff[i + 1] - eoff[i];
    outdeg[i] = d;
    if (d == 0) {
      level[i] = 0;
      frontier[atomicAdd(nfront, 1u)] = (u32)i;
    }
  }
}

// restricted to mask (reachable set): edges into masked-out classes never
// exist because the mask is closed under children.
__global__ void k_trim_step(const u32* front, u32 nf, const u32* roff, const u32* rsrc, u32* outdeg,
                            u32* level, u32 lvl, u32* next, u32* nnext, const u8* mask) {
  GRID_STRIDE(t, nf) {
    u32 j = front[t];
    for (u32 k = roff[j]; k < roff[j + 1]; k++) {
      u32 i = rsrc[k];
      if (mask && !mask[i]) continue;
      if (atomicSub(&outdeg[i], 1u) == 1u) {
        level[i] = lvl;
        next[atomicAdd(nnext, 1u)] = i;
      }
    }
  }
}

static void build_class_graph(Engine& e, ClassGraph& cg) {
  Snapshot& S = e.snap;
  u32 n = S.ncls;
  cg.ncls = n;
  cg.eoff.ensure(n + 1);
  DevBuf<u32>& cnt = e.scratch_u32[1];
  cnt.ensure(n + 1);
  k_edge_count<<<nblk(n), 256, 0, e.s>>>(e.view(), S.cls_off.p, S.cls_nodes.p, n, cnt.p);
  CUDA_OK(cudaMemsetAsync(cnt.p + n, 0, sizeof(u32), e.s));
  dev_exclusive_scan_u32(e, cnt.p, cg.eoff.p, n + 1);
  u32 ne;
  CUDA_OK(cudaMemcpyAsync(&ne, cg.eoff.p + n, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  e.sync();
  cg.nedge = ne;
  cg.edst.ensure(ne + 1);
  cg.enode.ensure(ne + 1);
  k_edge_fill<<<nblk(n), 256, 0, e.s>>>(e.view(), S.cls_off.p, S.cls_nodes.p, S.cls_index.p, n, cg.eoff.p,
                                        cg.edst.p, cg.enode.p);
  // reverse CSR by stable sort of (dst, src)
  DevBuf<u32> esrc, sdst;
  esrc.alloc(ne + 1);
  sdst.alloc(ne + 1);
  cg.rsrc.ensure(ne + 1);
  cg.roff.ensure(n + 1);
  k_edge_src<<<nblk(n), 256, 0, e.s>>>(cg.eoff.p, n, esrc.p);
  if (ne) dev_sort_pairs_u32(e, cg.edst.p, sdst.p, esrc.p, cg.rsrc.p, ne, bits_for(n));
  CUDA_OK(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(u32), e.s));
  k_rhist<<<nblk(ne), 256, 0, e.s>>>(cg.edst.p, ne, cnt.p);
  dev_exclusive_scan_u32(e, cnt.p, cg.roff.p, n + 1);
  cg.outdeg.ensure(n + 1);
  cg.level.ensure(n + 1);
}

// Kahn trimming; returns number of levels and fills per-level lists
static u32 trim(Engine& e, ClassGraph& cg, const u8* mask, std::vector<u32>& lvl_off, DevBuf<u32>& order,
                u32& ntrimmed) {
  u32 n = cg.ncls;
  order.ensure(n + 1);
  DevBuf<u32>& cntb = e.scratch_u32[2];
  cntb.ensure(2);
  CUDA_OK(cudaMemsetAsync(cntb.p, 0, sizeof(u32), e.s));
  k_outdeg_init<<<nblk(n), 256, 0, e.s>>>(cg.eoff.p, n, cg.outdeg.p, cg.level.p, order.p, cntb.p, mask);
  u32 nf;
  CUDA_OK(cudaMemcpyAsync(&nf, cntb.p, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  e.sync();
  lvl_off.clear();
  lvl_off.push_back(0);
  u32 start = 0, lvl = 0;
  while (nf) {
    lvl_off.push_back(start + nf);
    CUDA_OK(cudaMemsetAsync(cntb.p, 0, sizeof(u32), e.s));
    k_trim_step<<<nblk(nf), 256, 0, e.s>>>(order.p + start, nf, cg.roff.p, cg.rsrc.p, cg.outdeg.p,
                                           cg.level.p, lvl + 1, order.p + start + nf, cntb.p, mask);
    u32 nn;
    CUDA_OK(cudaMemcpyAsync(&nn, cntb.p, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    e.sync();
    start += nf;
    nf = nn;
    lvl++;
  }
  ntrimmed = start;
  return lvl;
}

// one warp per class row: row[i] = OR_{i->j} (row[j] | bit j)
__global__ void k_close_rows(const u32* list, u32 nl, const u32* eoff, const u32* edst, u32* bits, u32 words,
                             u32* changed) {
  u32 warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  u32 lane = threadIdx.x & 31;
  u32 nw = (gridDim.x * blockDim.x) >> 5;
  for (u32 t = warp; t < nl; t += nw) {
    u32 i = list[t];
    u32* row = bits + (u64)i * words;
    bool ch = false;
    for (u32 w = lane; w < words; w += 32) {
      u32 acc = changed ? row[w] : 0u;
      for (u32 e = eoff[i]; e < eoff[i + 1]; e++) {
        u32 j = edst[e];
        acc |= bits[(u64)j * words + w];
        if ((j >> 5) == w) acc |= 1u << (j & 31);
      }
      if (changed) {
        if (acc != row[w]) {
          row[w] = acc;
          ch = true;
        }
      } else {
        row[w] = acc;
      }
    }
    if (changed && __any_sync(0xffffffffu, ch) && lane == 0) *changed = 1;
  }
}

__global__ void k_untrimmed(const u32* level, u32 n, u32* list, u32* cnt) {
  GRID_STRIDE(i, n) if (level[i] == TSAT_NONE) list[atomicAdd(cnt, 1u)] = (u32)i;
}

void Engine::build_reach() {
  if (!snap.valid) build_snapshot();
  KTimer kt(*this, KG_REACH, 0.0, 0);
  ClassGraph cg;
  build_class_graph(*this, cg);
  u32 n = cg.ncls;
  u32 words = (n + 31) / 32;
  u64 bytes = (u64)n * words * 4;
  if (bytes > (u64)48 << 30)
    throw TsatException(TSAT_ERR_UNSUPPORTED, "descendants bitset would exceed 48 GiB");
  reach.bits.ensure((u64)n * words + 1);
  CUDA_OK(cudaMemsetAsync(reach.bits.p, 0, bytes, s));
  std::vector<u32> lo;
  DevBuf<u32> order;
  u32 ntr = 0;
  u32 nl = trim(*this, cg, nullptr, lo, order, ntr);
  for (u32 l = 1; l < nl; l++) {  // level 0 rows stay empty
    u32 a = lo[l], b = lo[l + 1];
    k_close_rows<<<nblk((u64)(b - a) * 32, 256), 256, 0, s>>>(order.p + a, b - a, cg.eoff.p, cg.edst.p,
                                                              reach.bits.p, words, nullptr);
  }
  if (ntr < n) {
    DevBuf<u32> rest;
    rest.alloc(n - ntr + 1);
    DevBuf<u32>& c2 = scratch_u32[2];
    c2.ensure(2);
    CUDA_OK(cudaMemsetAsync(c2.p, 0, sizeof(u32), s));
    k_untrimmed<<<nblk(n), 256, 0, s>>>(cg.level.p, n, rest.p, c2.p);
    u32 nr = n - ntr;
    while (true) {
      CUDA_OK(cudaMemsetAsync(c2.p + 1, 0, sizeof(u32), s));
      k_close_rows<<<nblk((u64)nr * 32, 256), 256, 0, s>>>(rest.p, nr, cg.eoff.p, cg.edst.p, reach.bits.p,
                                                           words, c2.p + 1);
      u32 ch;
      CUDA_OK(cudaMemcpyAsync(&ch, c2.p + 1, sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      if (!ch) break;
    }
  }
  reach.n = n;
  reach.words = words;
  reach.valid = true;
  // closure traffic: every row written once, each edge reads its child's row
  kt.bytes = 4.0 * words * ((double)n + (double)cg.nedge);
  kt.launches = 4 + nl;
  sync();
}

// ---------------------------------------------------------------- post-processing

__global__ void k_bfs_init(u32* mark, u32 n, u32 root, u32* front, u32* nf) {
  GRID_STRIDE(i, n) mark[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    mark[root] = 1;
    front[0] = root;
    *nf = 1;
  }
}

__global__ void k_bfs_step(const u32* front, u32 nf, const u32* eoff, const u32* edst, u32* mark, u32* next,
                           u32* nn) {
  GRID_STRIDE(t, nf) {
    u32 i = front[t];
    for (u32 e = eoff[i]; e < eoff[i + 1]; e++) {
      u32 j = edst[e];
      if (mark[j] == 0 && atomicCAS(&mark[j], 0u, 1u) == 0u) next[atomicAdd(nn, 1u)] = j;
    }
  }
}

__global__ void k_mark_to_u8(const u32* m, u32 n, u8* out) {
  GRID_STRIDE(i, n) out[i] = m[i] ? 1 : 0;
}

__global__ void k_count_cyclic(const u8* mark, const u32* level, u32 n, u32* cnt) {
  GRID_STRIDE(i, n) if (mark[i] && level[i] == TSAT_NONE) atomicAdd(cnt, 1u);
}

struct DfsFrame {
  u32 cls;    // dense class
  u32 mpos;   // member cursor
  u32 kpos;   // child cursor within member
};

// Exact DFS pass of dfs_get_cycles (cycles.py:172-221) on one thread, then
// the resolution loop of break_all_cycles (cycles.py:234-245).
__global__ void k_dfs_cycles(G g, const u32* cls_off, const u32* cls_nodes, const u32* cls_index,
                             const u32* level, u32 root_dense, u8* color, u32* depth_of, DfsFrame* stack,
                             u32* path, u32* cyc_nodes, u32 cyc_cap, u32* cyc_off, u32 cyc_off_cap,
                             u32* out /* [ncycles, nnodes, overflow, filtered] */, int resolve) {
  if (threadIdx.x || blockIdx.x) return;
  u32 ncyc = 0, nnodes = 0;
  bool overflow = false;
  u32 sp = 0;
  stack[sp++] = DfsFrame{root_dense, cls_off[root_dense], 0};
  color[root_dense] = 1;
  depth_of[root_dense] = 0;
  u32 plen = 0;
  while (sp) {
    DfsFrame& f = stack[sp - 1];
    bool advanced = false;
    while (f.mpos < cls_off[f.cls + 1]) {
      u32 m = cls_nodes[f.mpos];
      if (g.flags[m] & NF_FILT) {
        f.mpos++;
        f.kpos = 0;
        continue;
      }
      u32 ka = g.koff[m], kb = g.koff[m + 1];
      if (ka + f.kpos >= kb) {
        f.mpos++;
        f.kpos = 0;
        continue;
      }
      u32 ch = cls_index[uf_find_ro(g.parent, g.kids[ka + f.kpos])];
      f.kpos++;
      if (level[ch] != TSAT_NONE) continue;  // trimmed: cannot reach a cycle
      u8 st = color[ch];
      if (st == 1) {
        u32 start = depth_of[ch];
        u32 len = plen - start + 1;
        if (ncyc + 1 < cyc_off_cap && nnodes + len <= cyc_cap) {
          cyc_off[ncyc] = nnodes;
          for (u32 k = start; k < plen; k++) cyc_nodes[nnodes++] = path[k];
          cyc_nodes[nnodes++] = m;
          ncyc++;
          cyc_off[ncyc] = nnodes;
        } else {
          overflow = true;
        }
      } else if (st == 0) {
        color[ch] = 1;
        depth_of[ch] = sp;
        path[plen++] = m;
        stack[sp++] = DfsFrame{ch, cls_off[ch], 0};
        advanced = true;
        break;
      }
    }
    if (!advanced) {
      u32 c = stack[sp - 1].cls;
      sp--;
      if (plen) plen--;
      color[c] = 2;
    }
  }
  u32 filtered = 0;
  if (!overflow && resolve) {
    for (u32 c = 0; c < ncyc; c++) {
      bool broken = false;
      u32 mx = 0;
      for (u32 k = cyc_off[c]; k < cyc_off[c + 1]; k++) {
        u32 x = cyc_nodes[k];
        if (g.flags[x] & NF_FILT) broken = true;
        mx = x > mx ? x : mx;
      }
      if (broken) continue;
      g.flags[mx] |= NF_FILT;
      filtered++;
    }
  }
  out[0] = ncyc;
  out[1] = nnodes;
  out[2] = overflow ? 1u : 0u;
  out[3] = filtered;
}

i64 Engine::break_all_cycles(bool precheck_only, std::vector<std::vector<u32>>* cycles_out) {
  if (root == TSAT_NONE) throw TsatException(TSAT_ERR_STATE, "e-graph has no root");
  if (!snap.valid) build_snapshot();
  u32 rc = find(root);
  u32 root_dense;
  CUDA_OK(cudaMemcpyAsync(&root_dense, snap.cls_index.p + rc, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  KTimer kt(*this, KG_CYCLES, 0.0, 0);
  i64 added = 0;
  u32 cyc_cap = 1 << 16, off_cap = 1 << 12;
  while (true) {
    ClassGraph cg;
    build_class_graph(*this, cg);
    u32 n = cg.ncls;
    DevBuf<u8> mark;
    mark.alloc(n + 1);
    DevBuf<u32> mark32;
    mark32.alloc(n + 1);
    DevBuf<u32> fa, fb;
    fa.alloc(n + 1);
    fb.alloc(n + 1);
    DevBuf<u32>& c2 = scratch_u32[3];
    c2.ensure(4);
    k_bfs_init<<<nblk(n), 256, 0, s>>>(mark32.p, n, root_dense, fa.p, c2.p);
    u32 nf = 1;
    while (nf) {
      CUDA_OK(cudaMemsetAsync(c2.p + 1, 0, sizeof(u32), s));
      k_bfs_step<<<nblk(nf), 256, 0, s>>>(fa.p, nf, cg.eoff.p, cg.edst.p, mark32.p, fb.p, c2.p + 1);
      CUDA_OK(cudaMemcpyAsync(&nf, c2.p + 1, sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      std::swap(fa.p, fb.p);
    }
    k_mark_to_u8<<<nblk(n), 256, 0, s>>>(mark32.p, n, mark.p);
    std::vector<u32> lo;
    DevBuf<u32> order;
    u32 ntr = 0;
    trim(*this, cg, mark.p, lo, order, ntr);
    CUDA_OK(cudaMemsetAsync(c2.p + 2, 0, sizeof(u32), s));
    k_count_cyclic<<<nblk(n), 256, 0, s>>>(mark.p, cg.level.p, n, c2.p + 2);
    u32 ncyc_cls;
    CUDA_OK(cudaMemcpyAsync(&ncyc_cls, c2.p + 2, sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    if (ncyc_cls == 0) return added;
    if (precheck_only) return -1;
    // exact DFS over the untrimmed region
    DevBuf<u8> color;
    color.alloc(n + 1);
    DevBuf<u32> depth_of, path, cyc_nodes, cyc_off, res;
    DevBuf<DfsFrame> stack;
    depth_of.alloc(n + 1);
    path.alloc(n + 1);
    stack.alloc(n + 1);
    res.alloc(4);
    u32 hres[4];
    while (true) {
      cyc_nodes.ensure(cyc_cap);
      cyc_off.ensure(off_cap);
      CUDA_OK(cudaMemsetAsync(color.p, 0, n + 1, s));
      k_dfs_cycles<<<1, 1, 0, s>>>(view(), snap.cls_off.p, snap.cls_nodes.p, snap.cls_index.p, cg.level.p,
                                   root_dense, color.p, depth_of.p, stack.p, path.p, cyc_nodes.p, cyc_cap,
                                   cyc_off.p, off_cap, res.p, cycles_out ? 0 : 1);
      CUDA_OK(cudaMemcpyAsync(hres, res.p, sizeof(hres), cudaMemcpyDeviceToHost, s));
      sync();
      if (!hres[2]) break;
      cyc_cap *= 4;
      off_cap *= 4;
    }
    if (cycles_out) {
      std::vector<u32> hn(hres[1]), ho(hres[0] + 1);
      if (hres[1]) CUDA_OK(cudaMemcpyAsync(hn.data(), cyc_nodes.p, hres[1] * 4, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaMemcpyAsync(ho.data(), cyc_off.p, (hres[0] + 1) * 4, cudaMemcpyDeviceToHost, s));
      sync();
      for (u32 c = 0; c < hres[0]; c++) cycles_out->emplace_back(hn.begin() + ho[c], hn.begin() + ho[c + 1]);
      // dfs_get_cycles semantics: report only, undo the resolution
      return (i64)hres[0];
    }
    if (hres[0] == 0) return added;  // untrimmed region unreachable through live DFS order
    added += hres[3];
  }
}
