// ILP model skeleton on the device.
//
// reachable_classes (reference extract.py:198-217): BFS from the root class
// over live, non-filtered e-nodes -- the class graph of the snapshot
// (cycles.cu build_class_graph skips filter-listed members) walked by the
// shared frontier BFS (levels.cu bfs_classes).  Class order: root first, then
// ascending class id (dense snapshot order is ascending class id).
//
// build_ilp (extract.py:220-322) then needs, per reachable class, its alive
// members (the x variables, filter-listed ones pinned to 0), its live members
// (the right-hand side of every pick row into that class), and per live
// member the distinct child classes in ascending class id (one pick row each,
// plus one topological row with cycle constraints).  Those lists are built
// here; the host turns them into the reference's row dictionaries / LP text.
//
// All passes are O(N) gathers over the snapshot CSR: HBM / launch bound, no
// reduction to matrix form.
#include "engine.cuh"

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}

#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

u32 bfs_classes(Engine& e, u32 root, u32* mark, u32* queue);

__global__ void k_il_flag(const u32* mark, u32 n, u32* f) {
  GRID_STRIDE(d, (u64)n + 1) f[d] = (d < n && mark[d]) ? 1u : 0u;
}

// position of dense class d in the model's class list (root 0, then ascending)
__global__ void k_il_pos(const u32* f, const u32* scan, u32 n, u32 rd, const u32* cls_ids, u32* pos,
                         u32* classes) {
  GRID_STRIDE(d, n) {
    u32 p = TSAT_NONE;
    if (f[d]) {
      p = d == rd ? 0u : 1u + scan[d] - (d > rd ? 1u : 0u);
      classes[p] = cls_ids[d];
    }
    pos[d] = p;
  }
}

// alive members of reachable classes (all x variables), by member position
__global__ void k_il_sel(const u32* cls_of, const u32* pos, u32 m, u32* sel) {
  GRID_STRIDE(k, (u64)m + 1) sel[k] = (k < m && pos[cls_of[k]] != TSAT_NONE) ? 1u : 0u;
}

__global__ void k_il_gather(const u32* cls_nodes, const u32* sel, const u32* off, u32 m, u32* out) {
  GRID_STRIDE(k, m) if (sel[k]) out[off[k]] = cls_nodes[k];
}

// live (non-filtered) member count of each reachable class, by list position
__global__ void k_il_live_cnt(G g, const u32* cls_off, const u32* cls_nodes, const u32* pos, u32 n, u32 nr,
                              u32* cnt) {
  GRID_STRIDE(d, n) {
    u32 p = pos[d];
    if (p == TSAT_NONE) continue;
    u32 c = 0;
    for (u32 k = cls_off[d]; k < cls_off[d + 1]; k++) c += (g.flags[cls_nodes[k]] & NF_FILT) ? 0u : 1u;
    cnt[p] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[nr] = 0;
}

__global__ void k_il_live_fill(G g, const u32* cls_off, const u32* cls_nodes, const u32* pos, u32 n,
                               const u32* off, u32* live) {
  GRID_STRIDE(d, n) {
    u32 p = pos[d];
    if (p == TSAT_NONE) continue;
    u32 o = off[p];
    for (u32 k = cls_off[d]; k < cls_off[d + 1]; k++) {
      u32 x = cls_nodes[k];
      if (!(g.flags[x] & NF_FILT)) live[o++] = x;
    }
  }
}

// distinct child classes of node x in ascending dense order (= class id);
// writes their list positions when out != nullptr.  Arity is small (<= 8 for
// the tensor language), so a selection loop beats a sort.
__device__ u32 il_children(const G& g, u32 x, const u32* cls_index, const u32* pos, u32* out) {
  u32 a = g.koff[x], b = g.koff[x + 1];
  u32 cnt = 0;
  long long last = -1;
  while (true) {
    u32 best = TSAT_NONE;
    for (u32 j = a; j < b; j++) {
      u32 d = cls_index[uf_find_ro(g.parent, g.kids[j])];
      if ((long long)d > last && d < best) best = d;
    }
    if (best == TSAT_NONE) break;
    if (out) out[cnt] = pos[best];
    cnt++;
    last = best;
  }
  return cnt;
}

__global__ void k_il_pick_cnt(G g, const u32* live, u32 nl, const u32* cls_index, const u32* pos, u32* cnt) {
  GRID_STRIDE(t, (u64)nl + 1) cnt[t] = t < nl ? il_children(g, live[t], cls_index, pos, nullptr) : 0u;
}

__global__ void k_il_pick_fill(G g, const u32* live, u32 nl, const u32* cls_index, const u32* pos,
                               const u32* off, u32* child) {
  GRID_STRIDE(t, nl) il_children(g, live[t], cls_index, pos, child + off[t]);
}

void Engine::ilp_build(u32* sizes) {
  if (root == TSAT_NONE) throw TsatException(TSAT_ERR_STATE, "e-graph has no root");
  if (!snap.valid) build_snapshot();
  ensure_levels();
  u32 rc = find(root);
  u32 rd;
  CUDA_OK(cudaMemcpyAsync(&rd, snap.cls_index.p + rc, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  const u32 n = cg_n, m = h.live;
  Scratch& X = sc;
  X.il_mark.ensure(n + 1);
  X.il_queue.ensure(n + 1);
  X.il_f.ensure(n + 2);
  X.il_scan.ensure(n + 2);
  X.il_pos.ensure(n + 1);
  X.il_classes.ensure(n + 1);
  bfs_classes(*this, rd, X.il_mark.p, X.il_queue.p);
  k_il_flag<<<nblk((u64)n + 1), 256, 0, s>>>(X.il_mark.p, n, X.il_f.p);
  dev_exclusive_scan_u32(*this, X.il_f.p, X.il_scan.p, n + 1);
  u32 nr;
  CUDA_OK(cudaMemcpyAsync(&nr, X.il_scan.p + n, sizeof(u32), cudaMemcpyDeviceToHost, s));
  k_il_pos<<<nblk(n), 256, 0, s>>>(X.il_f.p, X.il_scan.p, n, rd, snap.cls_ids.p, X.il_pos.p, X.il_classes.p);
  // x variables: alive members of reachable classes, ascending node id
  X.il_sel.ensure(m + 2);
  X.il_soff.ensure(m + 2);
  k_il_sel<<<nblk((u64)m + 1), 256, 0, s>>>(snap.cls_of.p, X.il_pos.p, m, X.il_sel.p);
  dev_exclusive_scan_u32(*this, X.il_sel.p, X.il_soff.p, m + 1);
  u32 nx;
  CUDA_OK(cudaMemcpyAsync(&nx, X.il_soff.p + m, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  X.il_nodes.ensure(nx + 1);
  X.il_tmp.ensure(nx + 1);
  X.il_tmp2.ensure(nx + 1);
  k_il_gather<<<nblk(m), 256, 0, s>>>(snap.cls_nodes.p, X.il_sel.p, X.il_soff.p, m, X.il_tmp.p);
  if (nx) dev_sort_pairs_u32(*this, X.il_tmp.p, X.il_nodes.p, X.il_tmp.p, X.il_tmp2.p, nx, bits_for(h.next_id));
  // live members per class, in class-list order
  X.il_loff.ensure(nr + 2);
  X.il_lcnt.ensure(nr + 2);
  k_il_live_cnt<<<nblk(n), 256, 0, s>>>(view(), snap.cls_off.p, snap.cls_nodes.p, X.il_pos.p, n, nr, X.il_lcnt.p);
  dev_exclusive_scan_u32(*this, X.il_lcnt.p, X.il_loff.p, nr + 1);
  u32 nl;
  CUDA_OK(cudaMemcpyAsync(&nl, X.il_loff.p + nr, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  X.il_live.ensure(nl + 1);
  k_il_live_fill<<<nblk(n), 256, 0, s>>>(view(), snap.cls_off.p, snap.cls_nodes.p, X.il_pos.p, n, X.il_loff.p,
                                         X.il_live.p);
  // pick rows: distinct child classes of every live member
  X.il_pcnt.ensure(nl + 2);
  X.il_poff.ensure(nl + 2);
  k_il_pick_cnt<<<nblk((u64)nl + 1), 256, 0, s>>>(view(), X.il_live.p, nl, snap.cls_index.p, X.il_pos.p,
                                                 X.il_pcnt.p);
  dev_exclusive_scan_u32(*this, X.il_pcnt.p, X.il_poff.p, nl + 1);
  u32 np;
  CUDA_OK(cudaMemcpyAsync(&np, X.il_poff.p + nl, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  X.il_pchild.ensure(np + 1);
  k_il_pick_fill<<<nblk(nl), 256, 0, s>>>(view(), X.il_live.p, nl, snap.cls_index.p, X.il_pos.p, X.il_poff.p,
                                          X.il_pchild.p);
  nlaunch += 9;
  sync();
  check_error();
  il_sizes[0] = sizes[0] = nr;
  il_sizes[1] = sizes[1] = nx;
  il_sizes[2] = sizes[2] = nl;
  il_sizes[3] = sizes[3] = np;
}

void Engine::ilp_download(u32* classes, u32* nodes, u32* live_off, u32* live, u32* pick_off, u32* pick_child) {
  Scratch& X = sc;
  auto d2h = [&](u32* dst, const u32* src, u64 n) {
    if (dst && n) CUDA_OK(cudaMemcpyAsync(dst, src, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
  };
  d2h(classes, X.il_classes.p, il_sizes[0]);
  d2h(nodes, X.il_nodes.p, il_sizes[1]);
  d2h(live_off, X.il_loff.p, (u64)il_sizes[0] + 1);
  d2h(live, X.il_live.p, il_sizes[2]);
  d2h(pick_off, X.il_poff.p, (u64)il_sizes[2] + 1);
  d2h(pick_child, X.il_pchild.p, il_sizes[3]);
  sync();
}
