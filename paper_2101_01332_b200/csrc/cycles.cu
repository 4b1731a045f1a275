// Cycle filtering and class-level graph passes on the GPU
// (reference: pkg/src/tensorsat/cycles.py).
//
// Class graph: class -> child classes through live, unfiltered e-nodes (CSR
// plus reverse CSR), built from the snapshot CSR (build_class_graph).  On it:
//   * the Kahn peel from the sinks (levels.cu: trim_levels): level[c] =
//     height of c; classes never peeled lie on or above a cycle.  The peel is
//     cached per (snapshot, filter) and shared by the cycle check, the next
//     iteration's descendants map and greedy;
//   * BFS from the root (levels.cu: bfs_classes);
//   * the descendants bitset (cycles.py:70-148), column-parallel
//     (k_close_cols): word-major bitset, one CTA per column group walking
//     every level, untrimmed classes swept to a fixpoint afterwards.
// break_all_cycles (cycles.py:234-245): "no reachable class is untrimmed"
// proves there is no live cycle below the root; otherwise the exact
// lexicographic DFS (cycles.py:172-221) runs on one GPU thread over the
// untrimmed region only (trimmed classes cannot lie on or lead to a cycle, so
// skipping them keeps the back-edge sequence), then resolves cycles by
// filter-listing their max node id, pass after pass.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <chrono>

#include "engine.cuh"

namespace cg = cooperative_groups;

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

// edges through live, unfiltered members: member-parallel (classes can have
// thousands of members)
__global__ void k_member_deg(G g, const u32* cls_nodes, u32 m, u32* deg) {
  GRID_STRIDE(k, m) {
    u32 x = cls_nodes[k];
    deg[k] = (g.flags[x] & NF_FILT) ? 0u : g.koff[x + 1] - g.koff[x];
  }
}

__global__ void k_member_fill(G g, const u32* cls_nodes, const u32* cls_of, const u32* cls_index, u32 m,
                              const u32* moff, u32* edst, u32* esrc) {
  GRID_STRIDE(k, m) {
    u32 x = cls_nodes[k];
    if (g.flags[x] & NF_FILT) continue;
    u32 o = moff[k], c = cls_of[k];
    for (u32 j = g.koff[x]; j < g.koff[x + 1]; j++) {
      edst[o] = cls_index[uf_find_ro(g.parent, g.kids[j])];
      esrc[o] = c;
      o++;
    }
  }
}

__global__ void k_class_eoff(const u32* cls_off, const u32* moff, u32 n, u32* eoff) {
  GRID_STRIDE(c, (u64)n + 1) eoff[c] = moff[cls_off[c]];
}

__global__ void k_lower_bounds2(const u32* sorted, u32 m, u32 nkeys, u32* off) {
  GRID_STRIDE(a, (u64)nkeys + 1) {
    u32 lo = 0, hi = m;
    while (lo < hi) {
      u32 mid = (lo + hi) >> 1;
      if (sorted[mid] < (u32)a) lo = mid + 1;
      else hi = mid;
    }
    off[a] = lo;
  }
}

__global__ void k_rhist(const u32* edst, u64 ne, u32* h) {
  GRID_STRIDE(e, ne) atomicAdd(&h[edst[e]], 1u);
}

// Descendants closure, column-parallel.  The bitset is stored word-major
// (bitsT[w * n + i] = word w of class i's descendant set), and word w of a
// class depends only on word w of its children, so the closure splits into
// independent column groups: each CTA owns WPB words for ALL classes, walks
// the peel levels in order with only __syncthreads() between levels (no grid
// or host synchronisation), then sweeps the untrimmed (cyclic) remainder to a
// fixpoint.  Columns live in shared memory when they fit, else in HBM.
// Staged variant (oeoff != nullptr): the class edges are laid out in peel
// order (oeoff / oedst by level position), and batches of consecutive levels
// -- their level offsets, classes and edge lists -- are copied to shared
// memory with coalesced loads before the batch is walked, so a level costs a
// barrier plus shared-memory work instead of three dependent L2 round trips.
#define CC_LV 512u
#define CC_T 2048u
#define CC_E 8192u
#define CC_STAGE_WORDS (CC_LV + 1 + CC_T + 1 + CC_T + CC_E)
__global__ void __launch_bounds__(512) k_close_cols(const u32* order, const u32* lvl_off, u32 nl, const u32* eoff,
                                                    const u32* edst, const u32* rest, u32 nrest, u32 n, u32 words,
                                                    int wpb, int in_smem, u32* bitsT, const u32* oeoff,
                                                    const u32* oedst, const u32* batch, u32 nbatch) {
  extern __shared__ u32 smem_col[];
  __shared__ u32 s_changed;
  const u32 w0 = blockIdx.x * (u32)wpb;
  const int nk = (int)min((u32)wpb, words - w0);
  u32* col = in_smem ? smem_col : bitsT + (u64)w0 * n;
  if (in_smem)
    for (u64 i = threadIdx.x; i < (u64)nk * n; i += blockDim.x) col[i] = 0;
  __shared__ u32 s_next, s_rcls[32], s_rw[4][32];
  __syncthreads();
  auto item = [&](u32 a, u64 it) {
    u32 i = order[a + it / nk];
    int k = (int)(it % nk);
    u32 w = w0 + k;
    const u32* ck = col + (u64)k * n;
    u32 acc = 0;
    for (u32 e = eoff[i], e1 = eoff[i + 1]; e < e1; e++) {
      u32 j = edst[e];
      acc |= ck[j];
      if ((j >> 5) == w) acc |= 1u << (j & 31);
    }
    col[(u64)k * n + i] = acc;
  };
  if (oeoff) {
    u32* s_lv = smem_col + (in_smem ? (u64)nk * n : 0);
    u32* s_off = s_lv + CC_LV + 1;
    u32* s_ord = s_off + CC_T + 1;
    u32* s_ed = s_ord + CC_T;
    for (u32 bi = 0; bi < nbatch; bi++) {
      const u32 lb = batch[3 * bi], le = batch[3 * bi + 1], staged = batch[3 * bi + 2];
      const u32 t0 = lvl_off[lb], t1 = lvl_off[le];
      const u32 e0 = oeoff[t0], e1 = oeoff[t1];
      const u32 *LV = lvl_off, *OFF = oeoff, *ORD = order, *ED = oedst;
      u32 lbase = 0, tbase = 0, ebase = 0;
      if (staged) {
        for (u32 x = threadIdx.x; x <= le - lb; x += blockDim.x) s_lv[x] = lvl_off[lb + x];
        for (u32 x = threadIdx.x; x <= t1 - t0; x += blockDim.x) s_off[x] = oeoff[t0 + x];
        for (u32 x = threadIdx.x; x < t1 - t0; x += blockDim.x) s_ord[x] = order[t0 + x];
        for (u32 x = threadIdx.x; x < e1 - e0; x += blockDim.x) s_ed[x] = oedst[e0 + x];
        __syncthreads();
        LV = s_lv;
        OFF = s_off;
        ORD = s_ord;
        ED = s_ed;
        lbase = lb;
        tbase = t0;
        ebase = e0;
      }
      auto sitem = [&](u32 t, int k) {
        u32 i = ORD[t - tbase];
        u32 w = w0 + k;
        const u32* ck = col + (u64)k * n;
        u32 acc = 0;
        for (u32 e = OFF[t - tbase], e1_ = OFF[t + 1 - tbase]; e < e1_; e++) {
          u32 j = ED[e - ebase];
          acc |= ck[j];
          if ((j >> 5) == w) acc |= 1u << (j & 31);
        }
        col[(u64)k * n + i] = acc;
      };
      for (u32 l = lb; l < le;) {
        u32 a = LV[l - lbase], b = LV[l + 1 - lbase];
        u32 items = (b - a) * (u32)nk;
        if (items <= 32) {
          if (threadIdx.x < 32) {  // thin levels: warp 0 alone, __syncwarp only
            u32 ll = l;
            while (ll < le) {
              u32 a2 = LV[ll - lbase], b2 = LV[ll + 1 - lbase];
              u32 it2 = (b2 - a2) * (u32)nk;
              if (it2 > 32) break;
              if (threadIdx.x < it2) sitem(a2 + threadIdx.x / nk, (int)(threadIdx.x % nk));
              __syncwarp();
              ll++;
            }
            if (threadIdx.x == 0) s_next = ll;
          }
          __syncthreads();
          l = s_next;
          __syncthreads();
          continue;
        }
        for (u32 it = threadIdx.x; it < items; it += blockDim.x) sitem(a + it / nk, (int)(it % nk));
        __syncthreads();
        l++;
      }
      __syncthreads();
    }
  }
  for (u32 l = oeoff ? nl : 1; l < nl;) {
    u32 a = lvl_off[l], b = lvl_off[l + 1];
    u64 items = (u64)(b - a) * nk;
    if (items <= 32) {
      // a run of thin levels (deep chains): warp 0 alone, __syncwarp only
      if (threadIdx.x < 32) {
        const u32 lane = threadIdx.x;
        u32 ll = l, next_check = l;
        while (ll < nl) {
          if (nk <= 4 && ll >= next_check) {
            // runs of single-class levels: one lane per level loads its
            // children and their column words up front, then the lanes OR
            // them in level order (in-run children through shared memory)
            u32 lv = ll + lane, ci = TSAT_NONE, ea = 0, deg = 0;
            bool one = false;
            if (lv < nl) {
              u32 a3 = lvl_off[lv];
              if (lvl_off[lv + 1] == a3 + 1) {
                ci = order[a3];
                ea = eoff[ci];
                deg = eoff[ci + 1] - ea;
                one = deg <= 8;
              }
            }
            unsigned good = __ballot_sync(0xffffffffu, one), bad = ~good;
            u32 len = bad ? (u32)(__ffs(bad) - 1) : 32u;
            unsigned pairs = good & (good >> 1);
            if (len >= 2) {
              s_rcls[lane] = ci;
              __syncwarp();
              u32 d[8], v[4][8];
              int src[8];
#pragma unroll
              for (int j = 0; j < 8; j++) {
                d[j] = 0;
                src[j] = -1;
#pragma unroll
                for (int w = 0; w < 4; w++) v[w][j] = 0;
                if (lane < len && (u32)j < deg) {
                  d[j] = edst[ea + j];
                  for (u32 k = 0; k < lane; k++)
                    if (s_rcls[k] == d[j]) src[j] = (int)k;
                  if (src[j] < 0)
#pragma unroll
                    for (int w = 0; w < 4; w++)
                      if (w < nk) v[w][j] = col[(u64)w * n + d[j]];
                }
              }
              for (u32 k = 0; k < len; k++) {
                if (lane == k) {
#pragma unroll
                  for (int w = 0; w < 4; w++) {
                    if (w >= nk) break;
                    u32 acc = 0;
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                      if ((u32)j >= deg) break;
                      acc |= src[j] >= 0 ? s_rw[w][src[j]] : v[w][j];
                      if ((d[j] >> 5) == w0 + w) acc |= 1u << (d[j] & 31);
                    }
                    s_rw[w][k] = acc;
                    col[(u64)w * n + ci] = acc;
                  }
                }
                __syncwarp();
              }
              ll += len;
              next_check = ll;
              continue;
            }
            next_check = pairs ? ll + (u32)(__ffs(pairs) - 1) : ll + 31;
          }
          u32 a2 = lvl_off[ll], b2 = lvl_off[ll + 1];
          u64 it2 = (u64)(b2 - a2) * nk;
          if (it2 > 32) break;
          if (threadIdx.x < it2) item(a2, threadIdx.x);
          __syncwarp();
          ll++;
        }
        if (threadIdx.x == 0) s_next = ll;
      }
      __syncthreads();
      l = s_next;
      __syncthreads();
      continue;
    }
    for (u64 it = threadIdx.x; it < items; it += blockDim.x) item(a, it);
    __syncthreads();
    l++;
  }
  if (nrest) {
    while (true) {
      if (threadIdx.x == 0) s_changed = 0;
      __syncthreads();
      for (u64 it = threadIdx.x; it < (u64)nrest * nk; it += blockDim.x) {
        u32 i = rest[it / nk];
        int k = (int)(it % nk);
        u32 w = w0 + k;
        u32* ck = col + (u64)k * n;
        u32 acc = ck[i], old = acc;
        for (u32 e = eoff[i], e1 = eoff[i + 1]; e < e1; e++) {
          u32 j = edst[e];
          acc |= ck[j];
          if ((j >> 5) == w) acc |= 1u << (j & 31);
        }
        if (acc != old) {
          atomicOr(&ck[i], acc);
          s_changed = 1;
        }
      }
      __syncthreads();
      u32 ch = s_changed;
      __syncthreads();
      if (!ch) break;
    }
  }
  if (in_smem)
    for (u64 i = threadIdx.x; i < (u64)nk * n; i += blockDim.x) bitsT[(u64)w0 * n + i] = col[i];
}

__global__ void k_ord_deg(const u32* order, u32 ntr, const u32* eoff, u32* deg) {
  GRID_STRIDE(t, (u64)ntr + 1) {
    if (t < ntr) {
      u32 i = order[t];
      deg[t] = eoff[i + 1] - eoff[i];
    } else {
      deg[t] = 0;
    }
  }
}

__global__ void k_ord_fill(const u32* order, u32 ntr, const u32* eoff, const u32* edst, const u32* oeoff, u32* oedst) {
  GRID_STRIDE(t, ntr) {
    u32 i = order[t], o = oeoff[t];
    for (u32 e = eoff[i]; e < eoff[i + 1]; e++) oedst[o++] = edst[e];
  }
}

__global__ void k_gather_bnd(const u32* src, const u32* idx, u32 n, u32* out) {
  GRID_STRIDE(k, n) out[k] = src[idx[k]];
}

__global__ void k_untrimmed(const u32* level, u32 n, const u8* mask, u32* list, u32* cnt) {
  GRID_STRIDE(i, n) if (level[i] == TSAT_NONE && (!mask || mask[i])) list[atomicAdd(cnt, 1u)] = (u32)i;
}

// ---------------------------------------------------------------- host helpers

__global__ void k_level_keys(const u32* level, u32 n, u32* key, u32* val) {
  GRID_STRIDE(i, n) {
    key[i] = level[i];
    val[i] = (u32)i;
  }
}

void build_class_graph(Engine& e) {
  Snapshot& S = e.snap;
  Scratch& X = e.sc;
  u32 n = S.ncls, m = e.h.live;
  X.cg_eoff.ensure(n + 1);
  X.cg_mdeg.ensure(m + 1);
  X.cg_moff.ensure(m + 1);
  k_member_deg<<<nblk(m), 256, 0, e.s>>>(e.view(), S.cls_nodes.p, m, X.cg_mdeg.p);
  CUDA_OK(cudaMemsetAsync(X.cg_mdeg.p + m, 0, sizeof(u32), e.s));
  dev_exclusive_scan_u32(e, X.cg_mdeg.p, X.cg_moff.p, m + 1);
  k_class_eoff<<<nblk((u64)n + 1), 256, 0, e.s>>>(S.cls_off.p, X.cg_moff.p, n, X.cg_eoff.p);
  // No host read of the edge count: the buffers and the sort take the bound
  // ub = stored children of all nodes (>= the live, unfiltered member edges),
  // the slots past the real edges hold key 0xFFFFFFFF, which sorts after every
  // class index, so roff[n] = the real count.  The level peel that follows
  // reads it back with its own results (trim_levels), so the class graph
  // costs no host round trip before the peel is launched.
  const u32 ub = e.h.nkids;
  e.cg_n = n;
  e.cg_ne = ub;  // upper bound until trim_levels reads roff[n]
  X.cg_edst.ensure((u64)ub + 1);
  X.cg_esrc.ensure((u64)ub + 1);
  X.cg_sdst.ensure((u64)ub + 1);
  X.cg_rsrc.ensure((u64)ub + 1);
  X.cg_roff.ensure(n + 1);
  if (ub) CUDA_OK(cudaMemsetAsync(X.cg_edst.p, 0xFF, (size_t)ub * sizeof(u32), e.s));
  k_member_fill<<<nblk(m), 256, 0, e.s>>>(e.view(), S.cls_nodes.p, S.cls_of.p, S.cls_index.p, m, X.cg_moff.p,
                                          X.cg_edst.p, X.cg_esrc.p);
  if (ub) dev_sort_pairs_u32(e, X.cg_edst.p, X.cg_sdst.p, X.cg_esrc.p, X.cg_rsrc.p, ub, bits_for(n));
  k_lower_bounds2<<<nblk((u64)n + 1), 256, 0, e.s>>>(X.cg_sdst.p, ub, n, X.cg_roff.p);
  X.cg_outdeg.ensure(n + 1);
  X.cg_level.ensure(n + 1);
}

u32 trim_levels(Engine& e, const u8* mask, std::vector<u32>& lvl_off, u32& ntrimmed);
u32 bfs_classes(Engine& e, u32 root, u32* mark, u32* queue);

void Engine::ensure_levels() {
  if (!snap.valid) build_snapshot();
  if (lv_snap == snap_id && lv_filter == filter_id) return;
  static const bool dbg = getenv("TSAT_DEBUG_LEVELS") != nullptr;
  double t0 = 0, t1 = 0;
  if (dbg) {
    sync();
    t0 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  build_class_graph(*this);
  if (dbg) {
    sync();
    t1 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  lv_n = trim_levels(*this, nullptr, lv_off, lv_trimmed);
  if (shard_world > 1 && cg_n) {
    // shard ranks split wide peel levels by position (greedy), so every rank
    // needs the same order inside a level: (level, class) ascending instead
    // of the peel's arrival order.  Stable radix sort of the class ids by
    // level; unpeeled classes (TSAT_NONE) sort last, outside the levels.
    Scratch& X = sc;
    u32 n = cg_n;
    X.c_skey.ensure(n + 1);
    X.c_sval.ensure(n + 1);
    X.c_skey2.ensure(n + 1);
    k_level_keys<<<nblk(n), 256, 0, s>>>(X.cg_level.p, n, X.c_skey.p, X.c_sval.p);
    dev_sort_pairs_u32(*this, X.c_skey.p, X.c_skey2.p, X.c_sval.p, X.c_order.p, n, 32);
  }
  if (dbg) {
    sync();
    double t2 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    fprintf(stderr, "levels: classes %u edges %u class graph %.3f ms peel %.3f ms (%u levels)\n", cg_n, cg_ne, t1 - t0,
            t2 - t1, lv_n);
  }
  lv_snap = snap_id;
  lv_filter = filter_id;
}

void Engine::build_reach() {
  if (!snap.valid) build_snapshot();
  KTimer kt(*this, KG_REACH, 0.0, 0);
  ensure_levels();
  u32 n = cg_n;
  u32 words = (n + 31) / 32;
  u64 bytes = (u64)n * words * 4;
  if (bytes > reach.budget) {
    // mode 1: the peel levels ensure_levels just computed + the class graph
    // answer the queries (rulesdev.cuh reach_query); nothing O(C^2) is built
    reach.visit.ensure((u64)n + 1);
    reach.stack.ensure((u64)n + cg_ne + 1);
    reach.epoch.ensure(1);
    CUDA_OK(cudaMemsetAsync(reach.visit.p, 0, ((u64)n + 1) * sizeof(u32), s));
    CUDA_OK(cudaMemsetAsync(reach.epoch.p, 0, sizeof(u32), s));
    reach.n = n;
    reach.words = 0;
    reach.mode = 1;
    reach.valid = true;
    kt.bytes = 8.0 * n;
    kt.launches = 0;
    return;
  }
  reach.mode = 0;
  reach.bits.ensure((u64)n * words + 1);
  u32 nl = lv_n, ntr = lv_trimmed;
  if (getenv("TSAT_SEL_DEBUG")) {
    u32 single = 0;
    for (u32 l = 0; l < nl; l++) single += lv_off[l + 1] - lv_off[l] == 1;
    fprintf(stderr, "reach classes %u levels %u single %u trimmed %u\n", cg_n, nl, single, ntr);
  }
  DevBuf<u32>& rest = sc.c_rest;
  u32 nr = n - ntr;
  if (nr) {
    rest.ensure(nr + 1);
    DevBuf<u32>& c2 = sc.c_res;
    CUDA_OK(cudaMemsetAsync(c2.p, 0, sizeof(u32), s));
    k_untrimmed<<<nblk(n), 256, 0, s>>>(sc.cg_level.p, n, nullptr, rest.p, c2.p);
  }
  if (n) {
    // words per CTA: as many columns as fit in shared memory, but enough CTAs
    // to cover the SMs
    const u64 SMEM = 200u << 10;
    static int smem_set = 0;
    if (!smem_set) {
      CUDA_OK(cudaFuncSetAttribute(k_close_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
      smem_set = 1;
    }
    // level-ordered edge lists + batches of levels that fit the stage area
    static const bool no_stage = getenv("TSAT_CLOSE_NOSTAGE") != nullptr;
    const u64 STAGE = no_stage ? 0 : (u64)CC_STAGE_WORDS * 4;
    u32 nbatch = 0;
    if (!no_stage && nl > 1) {
      Scratch& X = sc;
      X.c_odeg.ensure(ntr + 2);
      X.c_oeoff.ensure(ntr + 2);
      X.c_oedst.ensure((u64)cg_ne + 1);
      X.c_obnd.ensure(nl + 2);
      k_ord_deg<<<nblk((u64)ntr + 1), 256, 0, s>>>(sc.c_order.p, ntr, sc.cg_eoff.p, X.c_odeg.p);
      dev_exclusive_scan_u32(*this, X.c_odeg.p, X.c_oeoff.p, ntr + 1);
      k_ord_fill<<<nblk(ntr), 256, 0, s>>>(sc.c_order.p, ntr, sc.cg_eoff.p, sc.cg_edst.p, X.c_oeoff.p, X.c_oedst.p);
      k_gather_bnd<<<nblk((u64)nl + 1), 256, 0, s>>>(X.c_oeoff.p, sc.c_lvloff.p, nl + 1, X.c_obnd.p);
      std::vector<u32> eb(nl + 1);
      CUDA_OK(cudaMemcpyAsync(eb.data(), X.c_obnd.p, (nl + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      std::vector<u32> bt;
      for (u32 l = 1; l < nl;) {
        u32 le = l;
        while (le < nl && le + 1 - l <= CC_LV && lv_off[le + 1] - lv_off[l] <= CC_T && eb[le + 1] - eb[l] <= CC_E) le++;
        if (le == l) {  // one level beyond the stage area: walked from global memory
          bt.insert(bt.end(), {l, l + 1, 0u});
          l++;
        } else {
          bt.insert(bt.end(), {l, le, 1u});
          l = le;
        }
      }
      nbatch = (u32)(bt.size() / 3);
      X.c_batch.ensure(bt.size() + 1);
      CUDA_OK(cudaMemcpyAsync(X.c_batch.p, bt.data(), bt.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    }
    u64 fit = (SMEM - STAGE) / (4ull * n);
    int in_smem = fit >= 1;
    u64 wpb = std::max<u64>(1, std::min<u64>(in_smem ? fit : 1, (words + 147) / 148));
    if (!in_smem) CUDA_OK(cudaMemsetAsync(reach.bits.p, 0, bytes, s));
    u32 grid = (u32)((words + wpb - 1) / wpb);
    size_t sm = (in_smem ? (size_t)wpb * n * 4 : 0) + (size_t)STAGE;
    k_close_cols<<<grid, 512, sm, s>>>(sc.c_order.p, sc.c_lvloff.p, nl, sc.cg_eoff.p, sc.cg_edst.p, rest.p, nr, n,
                                        words, (int)wpb, in_smem, reach.bits.p, nbatch ? sc.c_oeoff.p : nullptr,
                                        sc.c_oedst.p, sc.c_batch.p, nbatch);
    CUDA_OK(cudaGetLastError());
  }
  reach.n = n;
  reach.words = words;
  reach.valid = true;
  kt.bytes = 4.0 * words * ((double)n + (double)cg_ne);
  kt.launches = 2;
}

// ---------------------------------------------------------------- post-processing

struct DfsFrame {
  u32 cls;
  u32 mpos;
  u32 kpos;
};

// Exact DFS pass of dfs_get_cycles (cycles.py:172-221) on one thread, then the
// resolution loop of break_all_cycles (cycles.py:234-245) when ``resolve``.
__global__ void k_dfs_cycles(G g, const u32* cls_off, const u32* cls_nodes, const u32* cls_index,
                             const u32* level, u32 root_dense, u8* color, u32* depth_of, DfsFrame* stack,
                             u32* path, u32* cyc_nodes, u32 cyc_cap, u32* cyc_off, u32 cyc_off_cap, u32* out,
                             int resolve) {
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
      if (level[ch] != TSAT_NONE) continue;  // peeled: cannot reach a cycle
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

__global__ void k_mark8(const u32* m, u32 n, u8* o) {
  GRID_STRIDE(i, n) o[i] = m[i] ? 1 : 0;
}

__global__ void k_count_cyclic(const u8* mark, const u32* level, u32 n, u32* cnt) {
  GRID_STRIDE(i, n) if (mark[i] && level[i] == TSAT_NONE) atomicAdd(cnt, 1u);
}

i64 Engine::break_all_cycles(bool precheck_only, std::vector<std::vector<u32>>* cycles_out) {
  if (root == TSAT_NONE) throw TsatException(TSAT_ERR_STATE, "e-graph has no root");
  if (!snap.valid) build_snapshot();
  KTimer kt(*this, KG_CYCLES, 0.0, 0);
  u32 root_dense = TSAT_NONE;  // looked up only when some class fails to peel
  i64 added = 0;
  u32 cyc_cap = 1 << 16, off_cap = 1 << 12;
  while (true) {
    ensure_levels();
    u32 n = cg_n;
    if (lv_trimmed == n) return added;  // the whole class graph peels: no live cycle anywhere
    if (root_dense == TSAT_NONE) {
      u32 rc = find(root);
      CUDA_OK(cudaMemcpyAsync(&root_dense, snap.cls_index.p + rc, sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
    }
    sc.c_mark.ensure(n + 1);
    sc.c_mark32.ensure(n + 1);
    sc.c_fa.ensure(n + 1);
    sc.c_res.ensure(16);
    bfs_classes(*this, root_dense, sc.c_mark32.p, sc.c_fa.p);
    k_mark8<<<nblk(n), 256, 0, s>>>(sc.c_mark32.p, n, sc.c_mark.p);
    CUDA_OK(cudaMemsetAsync(sc.c_res.p + 12, 0, sizeof(u32), s));
    k_count_cyclic<<<nblk(n), 256, 0, s>>>(sc.c_mark.p, sc.cg_level.p, n, sc.c_res.p + 12);
    u32 ncyc_cls;
    CUDA_OK(cudaMemcpyAsync(&ncyc_cls, sc.c_res.p + 12, sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    if (ncyc_cls == 0) return added;
    if (precheck_only) return -1;
    sc.c_color.ensure(n + 1);
    sc.c_depth.ensure(n + 1);
    sc.c_path.ensure(n + 1);
    sc.c_stack.ensure((u64)(n + 1) * sizeof(DfsFrame));
    u32 hres[4];
    while (true) {
      sc.c_cycn.ensure(cyc_cap);
      sc.c_cyco.ensure(off_cap);
      CUDA_OK(cudaMemsetAsync(sc.c_color.p, 0, n + 1, s));
      k_dfs_cycles<<<1, 1, 0, s>>>(view(), snap.cls_off.p, snap.cls_nodes.p, snap.cls_index.p, sc.cg_level.p,
                                   root_dense, sc.c_color.p, sc.c_depth.p, (DfsFrame*)sc.c_stack.p, sc.c_path.p,
                                   sc.c_cycn.p, cyc_cap, sc.c_cyco.p, off_cap, sc.c_res.p, cycles_out ? 0 : 1);
      CUDA_OK(cudaMemcpyAsync(hres, sc.c_res.p, sizeof(hres), cudaMemcpyDeviceToHost, s));
      sync();
      if (!hres[2]) break;
      cyc_cap *= 4;
      off_cap *= 4;
    }
    if (cycles_out) {
      std::vector<u32> hn(hres[1]), ho(hres[0] + 1);
      if (hres[1]) CUDA_OK(cudaMemcpyAsync(hn.data(), sc.c_cycn.p, hres[1] * 4, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaMemcpyAsync(ho.data(), sc.c_cyco.p, (hres[0] + 1) * 4, cudaMemcpyDeviceToHost, s));
      sync();
      for (u32 c = 0; c < hres[0]; c++) cycles_out->emplace_back(hn.begin() + ho[c], hn.begin() + ho[c + 1]);
      return (i64)hres[0];
    }
    if (hres[0] == 0) return added;
    added += hres[3];
    if (hres[3]) filter_id++;
  }
}

// ---------------------------------------------------------------- API helpers

// live_adjacency (cycles.py:29-39) over the current filter: the snapshot class
// graph (dense indices, one edge per child of every live unfiltered member).
// sizes = {classes, edges}; any output pointer may be NULL.
void Engine::class_graph_download(u32* cls, u32* eoff, u32* edst, u32* sizes) {
  ensure_levels();
  sizes[0] = cg_n;
  sizes[1] = cg_ne;
  if (cls && cg_n) CUDA_OK(cudaMemcpyAsync(cls, snap.cls_ids.p, cg_n * sizeof(u32), cudaMemcpyDeviceToHost, s));
  if (eoff) CUDA_OK(cudaMemcpyAsync(eoff, sc.cg_eoff.p, (cg_n + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
  if (edst && cg_ne) CUDA_OK(cudaMemcpyAsync(edst, sc.cg_edst.p, cg_ne * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
}

// get_descendants (cycles.py:70-148): the closure as the device bitset
// (word-major: bits[w * n + i] = word w of class i's descendant set), built
// regardless of the pre-filter budget.  sizes = {classes, words}; bits NULL
// or too small: sizes only.
void Engine::descendants_download(u32* cls, u32* bits, u64 cap_words, u32* sizes) {
  if (!snap.valid) build_snapshot();
  u64 keep = reach.budget;
  reach.budget = ~0ull;
  try {
    build_reach();
  } catch (...) {
    reach.budget = keep;
    throw;
  }
  reach.budget = keep;
  sizes[0] = reach.n;
  sizes[1] = reach.words;
  u64 need = (u64)reach.n * reach.words;
  if (cls && reach.n) CUDA_OK(cudaMemcpyAsync(cls, snap.cls_ids.p, reach.n * sizeof(u32), cudaMemcpyDeviceToHost, s));
  if (bits && cap_words >= need && need)
    CUDA_OK(cudaMemcpyAsync(bits, reach.bits.p, need * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  reach.valid = false;  // the pre-filter of the next iteration rebuilds its own
}
