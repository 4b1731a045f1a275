// Level engine: Kahn peeling and BFS on the class graph, with hybrid
// execution.  E-graphs from rewrite rules are deep and thin (associativity
// chains and the make_single_rooted noop fold give hundreds to thousands of
// levels of a few classes each), so a level-synchronous algorithm is
// latency bound:
//   * very thin levels (<= 32 vertices, <= 64 edges): warp 0 alone, frontier
//     carried in registers, plain shared-memory updates (no atomics);
//   * thin levels (<= LV_WIDE vertices): one 1024-thread CTA, the level's edges
//     flattened by a block scan of the frontier degrees, degree / mark arrays
//     (and for small graphs the CSR offsets, queue and edge list) in shared
//     memory;
//   * wide levels: the whole GPU as a cooperative kernel with grid.sync(),
//     light / medium / heavy vertex tiers, warp-aggregated queue appends.
// The host only switches between the CTA and the grid kernel when a frontier
// crosses the threshold.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "engine.cuh"

namespace cg = cooperative_groups;

#define LV_WIDE 16384u
#define LV_BLOCK 1024

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)b;
}
#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

// ctl layout: [0] tail, [1] level, [2] start, [3] end, [4] done, [5] unused,
// [6] edge count of the current frontier, [7] of the next frontier, [8] heavy list size
struct Frontier {
  const u32* eoff;  // forward CSR (BFS) or outdeg source (trim)
  const u32* edst;
  const u32* roff;  // reverse CSR (trim)
  const u32* rsrc;
  const u8* mask;
  u32* outdeg;
  u32* level;
  u32* order;  // peel order / BFS queue
  u32* lvl_off;
  u32* mark;
  u32 n;
  int bfs;  // 1 = BFS from order[0], 0 = trim
};

#define HEAVY 32u

__device__ __forceinline__ u32 vdeg(const Frontier& F, u32 j) {
  return F.bfs ? F.eoff[j + 1] - F.eoff[j] : F.roff[j + 1] - F.roff[j];
}

// deg = mark (BFS) or outdeg (trim) array; tail / nedges = queue tail and edge
// count of the next frontier (global ctl words, or shared-memory copies)
__device__ __forceinline__ void frontier_edge(const Frontier& F, u32 e, u32 lvl, u32* deg, u32* tail, u32* nedges) {
  if (F.bfs) {
    u32 k = F.edst[e];
    if (deg[k] == 0 && atomicCAS(&deg[k], 0u, 1u) == 0u) {
      F.order[atomicAdd(tail, 1u)] = k;
      atomicAdd(nedges, vdeg(F, k));
    }
  } else {
    u32 i = F.rsrc[e];
    if (F.mask && !F.mask[i]) return;
    if (atomicSub(&deg[i], 1u) == 1u) {
      F.level[i] = lvl + 1;
      F.order[atomicAdd(tail, 1u)] = i;
      atomicAdd(nedges, vdeg(F, i));
    }
  }
}

// warp-uniform variant for the grid kernel: all 32 lanes call it (valid = lane
// holds an edge); the queue tail and the next-frontier edge count are bumped
// once per warp (ballot + popc) instead of once per vertex -- a 1M-vertex
// level otherwise serialises on the single tail counter.
__device__ __forceinline__ void frontier_edge_warp(const Frontier& F, bool valid, u32 e, u32 lvl, u32* deg,
                                                   u32* tail, u32* nedges) {
  u32 v = TSAT_NONE;
  if (valid) {
    if (F.bfs) {
      u32 k = F.edst[e];
      if (deg[k] == 0 && atomicCAS(&deg[k], 0u, 1u) == 0u) v = k;
    } else {
      u32 i = F.rsrc[e];
      if ((!F.mask || F.mask[i]) && atomicSub(&deg[i], 1u) == 1u) {
        F.level[i] = lvl + 1;
        v = i;
      }
    }
  }
  u32 lane = threadIdx.x & 31;
  unsigned m = __ballot_sync(0xffffffffu, v != TSAT_NONE);
  if (!m) return;
  u32 d = v != TSAT_NONE ? vdeg(F, v) : 0u;
  for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  u32 base = 0;
  if (lane == 0) {
    base = atomicAdd(tail, (u32)__popc(m));
    atomicAdd(nedges, d);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (v != TSAT_NONE) F.order[base + __popc(m & ((1u << lane) - 1))] = v;
}

__device__ __forceinline__ void edge_range(const Frontier& F, u32 j, u32& a, u32& b) {
  if (F.bfs) {
    a = F.eoff[j];
    b = F.eoff[j + 1];
  } else {
    a = F.roff[j];
    b = F.roff[j + 1];
  }
}

__global__ void k_frontier_init(Frontier F, u32* ctl, u32 root) {
  GRID_STRIDE(i, F.n) {
    if (F.bfs) {
      F.mark[i] = (u32)(i == root);
      continue;
    }
    F.level[i] = TSAT_NONE;
    if (F.mask && !F.mask[i]) continue;
    u32 d = F.eoff[i + 1] - F.eoff[i];
    F.outdeg[i] = d;
    if (d == 0) {
      F.level[i] = 0;
      F.order[atomicAdd(&ctl[0], 1u)] = (u32)i;
      atomicAdd(&ctl[7], vdeg(F, (u32)i));
    }
  }
  if (F.bfs && blockIdx.x == 0 && threadIdx.x == 0) {
    F.order[0] = root;
    ctl[0] = 1;
    ctl[7] = vdeg(F, root);
  }
}

__global__ void k_frontier_start(u32* ctl, u32* lvl_off) {
  ctl[1] = 0;
  ctl[2] = 0;
  ctl[3] = ctl[0];
  ctl[4] = 0;
  ctl[6] = ctl[7];
  ctl[7] = 0;
  if (lvl_off) {
    lvl_off[0] = 0;
    lvl_off[1] = ctl[0];
  }
}

// thin levels inside one CTA; exits when a frontier gets wide (by edges).
// Vertices with more than HEAVY edges are queued and their edge lists are
// swept by the whole CTA.  With ``use_smem`` the mark / out-degree array and
// the queue counters live in shared memory (small graphs), so a level costs
// a couple of dependent global loads plus shared-memory atomics.
#define LV_EDGES 65536u
// use_smem: 0 = all state in HBM, 1 = degree / mark array in shared memory,
// 2 = also the CSR offsets and the queue (small graphs: a level then costs one
// HBM round trip, the edge-list read)
__global__ void __launch_bounds__(LV_BLOCK) k_frontier_block(Frontier Fg, u32* ctl, int use_smem) {
  extern __shared__ u32 s_deg[];
  __shared__ u32 s_start, s_end, s_lvl, s_edges, s_tail, s_ned;
  __shared__ u32 s_heavy[LV_BLOCK];
  __shared__ u32 s_estart[LV_BLOCK];
  Frontier F = Fg;
  u32* gdeg = F.bfs ? F.mark : F.outdeg;
  u32* deg = use_smem ? s_deg : gdeg;
  u32* tail = use_smem ? &s_tail : &ctl[0];
  u32* ned = use_smem ? &s_ned : &ctl[7];
  const u32 t_init = ctl[0];
  if (use_smem)
    for (u32 i = threadIdx.x; i < F.n; i += blockDim.x) s_deg[i] = gdeg[i];
  if (use_smem >= 2) {
    u32* s_off = s_deg + F.n;
    u32* s_ord = s_off + F.n + 1;
    const u32* goff = F.bfs ? F.eoff : F.roff;
    for (u32 i = threadIdx.x; i <= F.n; i += blockDim.x) s_off[i] = goff[i];
    for (u32 i = ctl[2] + threadIdx.x; i < t_init; i += blockDim.x) s_ord[i] = Fg.order[i];
    if (use_smem == 3) {
      // the edge list too (tiny graphs with deep chains: a level is then all
      // shared-memory work)
      u32* s_edge = s_ord + F.n;
      u32 ne = goff[F.n];
      const u32* gedge = F.bfs ? F.edst : F.rsrc;
      for (u32 i = threadIdx.x; i < ne; i += blockDim.x) s_edge[i] = gedge[i];
      if (F.bfs) F.edst = s_edge;
      else F.rsrc = s_edge;
    }
    if (F.bfs) F.eoff = s_off;
    else F.roff = s_off;
    F.order = s_ord;
  }
  if (threadIdx.x == 0) {
    s_start = ctl[2];
    s_end = ctl[3];
    s_lvl = ctl[1];
    s_edges = ctl[6];
    s_tail = ctl[0];
    s_ned = ctl[7];
  }
  __syncthreads();
  while (true) {
    u32 start = s_start, end = s_end, lvl = s_lvl, edges = s_edges;
    // every thread has read the level state before anyone (warp 0 in the
    // thin-level walk, thread 0 at the end of a level) overwrites it
    __syncthreads();
    if (start >= end) {
      if (threadIdx.x == 0) ctl[4] = 1;
      break;
    }
    if (end - start > LV_WIDE || edges > LV_EDGES) break;
    if (end - start <= 32 && edges <= 64) {
      // Very thin levels (deep chains): warp 0 alone walks level after level
      // with __syncwarp() only; the queue tail lives in a register.
      if (threadIdx.x < 32) {
        const u32 lane = threadIdx.x;
        u32 st = start, en = end, lv = lvl, ed = edges, tl = *(volatile u32*)tail;
        // the frontier stays in registers: lane q holds vertex st + q and its
        // edge range, handed over by shuffles from the lane that queued it
        u32 a = 0, b = 0;
        if (st + lane < en) edge_range(F, F.order[st + lane], a, b);
        while (st < en && en - st <= 32 && ed <= 64) {
          u32 md = b - a;
          for (int o = 16; o; o >>= 1) md = max(md, __shfl_xor_sync(0xffffffffu, md, o));
          if (md > 16) break;  // a fat vertex: let the whole CTA take this level
          const u32 nst = tl;
          u32 nd = 0, na = 0, nb = 0;
          for (u32 k = 0; k < md; k++) {
            u32 v = TSAT_NONE, va = 0, vb = 0;
            // warp mode: this warp is the only writer of deg[], so plain
            // loads / stores with lanes of equal targets combined by
            // __match_any_sync replace the L2 atomics (one round trip less
            // per level on long chains)
            u32 tgt = TSAT_NONE;
            if (a + k < b) {
              u32 e = a + k;
              tgt = F.bfs ? F.edst[e] : F.rsrc[e];
              if (!F.bfs && F.mask && !F.mask[tgt]) tgt = TSAT_NONE;
            }
            unsigned same = __match_any_sync(0xffffffffu, tgt);
            bool leader = tgt != TSAT_NONE && (u32)(__ffs(same) - 1) == lane;
            if (leader) {
              if (F.bfs) {
                if (deg[tgt] == 0) {
                  deg[tgt] = 1;
                  v = tgt;
                }
              } else {
                u32 dd = deg[tgt], dec = (u32)__popc(same);
                deg[tgt] = dd - dec;
                if (dd == dec) {
                  F.level[tgt] = lv + 1;
                  v = tgt;
                }
              }
            }
            unsigned m = __ballot_sync(0xffffffffu, v != TSAT_NONE);
            if (v != TSAT_NONE) {
              F.order[tl + __popc(m & ((1u << lane) - 1))] = v;
              edge_range(F, v, va, vb);
              nd += vb - va;
            }
            // hand (va, vb) to the lane that owns the new position
            int q = (int)lane - (int)(tl - nst);
            u32 cnt = __popc(m);
            u32 src = lane;
            if (q >= 0 && (u32)q < cnt) {
              u32 mm = m;
              for (int i = 0; i < q; i++) mm &= mm - 1;  // drop the q lowest set bits
              src = (u32)(__ffs(mm) - 1);
            }
            u32 ga = __shfl_sync(0xffffffffu, va, src), gb = __shfl_sync(0xffffffffu, vb, src);
            if (q >= 0 && (u32)q < cnt) {
              na = ga;
              nb = gb;
            }
            tl += cnt;
          }
          for (int o = 16; o; o >>= 1) nd += __shfl_xor_sync(0xffffffffu, nd, o);
          if (F.lvl_off && lane == 0) F.lvl_off[lv + 2] = tl;
          st = en;
          en = tl;
          ed = nd;
          lv++;
          if (en - st > 32) break;
          a = na;
          b = nb;
          __syncwarp();
        }
        __syncwarp();  // every lane read *tail before lane 0 rewrites it
        if (lane == 0) {
          s_start = st;
          s_end = en;
          s_lvl = lv;
          s_edges = ed;
          *tail = tl;
          *ned = 0;
        }
      }
      __syncthreads();
      if (s_start == start) {
        // no progress in warp mode (fat vertex): fall through to the CTA path
      } else {
        continue;
      }
    }
    // the level's edges are flattened: a block scan of the frontier vertices'
    // degrees, then one thread per edge (vertex found by binary search of the
    // prefix) -- no thread walks a long edge list alone
    for (u32 t0 = start; t0 < end; t0 += blockDim.x) {
      u32 t = t0 + threadIdx.x;
      u32 a = 0, b = 0;
      if (t < end) edge_range(F, F.order[t], a, b);
      u32 d = b - a, x, tot;
      typedef cub::BlockScan<u32, LV_BLOCK> BS;
      __shared__ typename BS::TempStorage scan_tmp;
      BS(scan_tmp).ExclusiveSum(d, x, tot);
      s_heavy[threadIdx.x] = x;  // prefix of the chunk's degrees
      s_estart[threadIdx.x] = a;
      __syncthreads();
      u32 nv = min((u32)blockDim.x, end - t0);
      for (u32 k = threadIdx.x; k < tot; k += blockDim.x) {
        u32 lo = 0, hi = nv;  // last vertex slot with prefix <= k
        while (hi - lo > 1) {
          u32 mid = (lo + hi) >> 1;
          if (s_heavy[mid] <= k) lo = mid;
          else hi = mid;
        }
        frontier_edge(F, s_estart[lo] + (k - s_heavy[lo]), lvl, deg, tail, ned);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      __threadfence_block();
      u32 ne = ((volatile u32*)tail)[0];
      s_start = end;
      s_end = ne;
      s_lvl = lvl + 1;
      s_edges = ((volatile u32*)ned)[0];
      *ned = 0;
      if (F.lvl_off) F.lvl_off[lvl + 2] = ne;
    }
    __syncthreads();
  }
  if (use_smem)
    for (u32 i = threadIdx.x; i < F.n; i += blockDim.x) gdeg[i] = s_deg[i];
  if (use_smem >= 2)
    for (u32 i = t_init + threadIdx.x; i < s_tail; i += blockDim.x) Fg.order[i] = F.order[i];
  if (threadIdx.x == 0) {
    ctl[1] = s_lvl;
    ctl[2] = s_start;
    ctl[3] = s_end;
    ctl[6] = s_edges;
    if (use_smem) {
      ctl[0] = s_tail;
      ctl[7] = s_ned;
    }
  }
}

// wide levels on the whole GPU; exits when the frontier gets thin again.
// Three vertex tiers, every queue append warp-aggregated (ballot + popc, one
// atomic per warp step -- a 1M-vertex level otherwise serialises on the tail):
//   light  (<= 32 edges): one thread per vertex, lanes step their edge lists
//   medium (<= 4096):     listed, then one warp per vertex
//   heavy  (> 4096, e.g. shared literals with a million parents): listed,
//                         then the whole grid sweeps each edge list
__global__ void k_frontier_grid(Frontier F, u32* ctl, u32* heavy) {
  cg::grid_group grid = cg::this_grid();
  u32 start = ctl[2], end = ctl[3], lvl = ctl[1], edges = ctl[6];
  u32 lane = threadIdx.x & 31;
  u64 warp = grid.thread_rank() >> 5, nwarp = grid.size() >> 5;
  u32* medium = heavy + F.n + 1;
  u32* deg = F.bfs ? F.mark : F.outdeg;
  while (start < end && (end - start > LV_WIDE / 4 || edges > LV_EDGES / 4)) {
    if (grid.thread_rank() == 0) {
      ctl[8] = 0;
      ctl[9] = 0;
    }
    grid.sync();
    for (u64 t0 = start + warp * 32; t0 < end; t0 += nwarp * 32) {
      u64 t = t0 + lane;
      u32 a = 0, b = 0, j = TSAT_NONE;
      if (t < end) {
        j = F.order[t];
        edge_range(F, j, a, b);
      }
      u32 d = b - a;
      bool med = j != TSAT_NONE && d > 32 && d <= 4096, hv = j != TSAT_NONE && d > 4096;
      unsigned mm = __ballot_sync(0xffffffffu, med), mh = __ballot_sync(0xffffffffu, hv);
      if (mm | mh) {
        u32 bm = 0, bh = 0;
        if (lane == 0) {
          if (mm) bm = atomicAdd(&ctl[9], (u32)__popc(mm));
          if (mh) bh = atomicAdd(&ctl[8], (u32)__popc(mh));
        }
        bm = __shfl_sync(0xffffffffu, bm, 0);
        bh = __shfl_sync(0xffffffffu, bh, 0);
        if (med) medium[bm + __popc(mm & ((1u << lane) - 1))] = j;
        if (hv) heavy[bh + __popc(mh & ((1u << lane) - 1))] = j;
      }
      if (med || hv) b = a;
      u32 md = b - a;
      for (int o = 16; o; o >>= 1) md = max(md, __shfl_xor_sync(0xffffffffu, md, o));
      for (u32 k = 0; k < md; k++) frontier_edge_warp(F, a + k < b, a + k, lvl, deg, &ctl[0], &ctl[7]);
    }
    grid.sync();
    u32 nm = ((volatile u32*)ctl)[9];
    for (u64 q = warp; q < nm; q += nwarp) {
      u32 a, b;
      edge_range(F, medium[q], a, b);
      for (u32 e0 = a; e0 < b; e0 += 32) frontier_edge_warp(F, e0 + lane < b, e0 + lane, lvl, deg, &ctl[0], &ctl[7]);
    }
    u32 nh = ((volatile u32*)ctl)[8];
    for (u32 h = 0; h < nh; h++) {
      u32 a, b;
      edge_range(F, heavy[h], a, b);
      for (u64 e0 = a + warp * 32; e0 < b; e0 += nwarp * 32)
        frontier_edge_warp(F, e0 + lane < b, (u32)(e0 + lane), lvl, deg, &ctl[0], &ctl[7]);
    }
    grid.sync();
    u32 ne = ((volatile u32*)ctl)[0];
    u32 ned = ((volatile u32*)ctl)[7];
    if (grid.thread_rank() == 0 && F.lvl_off) F.lvl_off[lvl + 2] = ne;
    start = end;
    end = ne;
    edges = ned;
    lvl++;
    grid.sync();
    if (grid.thread_rank() == 0) ctl[7] = 0;
    grid.sync();
  }
  if (grid.thread_rank() == 0) {
    ctl[1] = lvl;
    ctl[2] = start;
    ctl[3] = end;
    ctl[6] = edges;
    if (start >= end) ctl[4] = 1;
  }
}

static int coop_blocks(Engine& e, const void* fn, int threads) {
  int nsm = 0, per = 0;
  CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, e.device));
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, 0));
  if (per < 1) per = 1;
  return nsm * std::min(per, 2);
}

// runs the frontier to completion; returns (levels, total processed)
// lvl_host (optional, >= F.n + 2 entries): the level offsets come back with
// the final control read (one host sync instead of two)
static void run_frontier(Engine& e, Frontier F, u32 root, u32& nlevels, u32& total, u32 ne_known = TSAT_NONE,
                         u32* lvl_host = nullptr) {
  DevBuf<u32>& ctl = e.sc.c_res;
  ctl.ensure(16);
  CUDA_OK(cudaMemsetAsync(ctl.p, 0, 16 * sizeof(u32), e.s));
  DevBuf<u32>& heavy = e.sc.c_heavy;
  heavy.ensure(2 * ((u64)F.n + 1));
  k_frontier_init<<<nblk(F.n), 256, 0, e.s>>>(F, ctl.p, root);
  k_frontier_start<<<1, 1, 0, e.s>>>(ctl.p, F.lvl_off);
  static int gblocks = 0;
  if (!gblocks) gblocks = coop_blocks(e, (const void*)k_frontier_grid, 256);
  u32 h[5];
  const u64 FR_SMEM = 200u << 10;
  u32 ne = ne_known;
  if (ne == TSAT_NONE) {
    CUDA_OK(cudaMemcpyAsync(&ne, (F.bfs ? F.eoff : F.roff) + F.n, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    e.sync();
  }
  int use_smem = (12ull * F.n + 4 + 4ull * ne <= FR_SMEM) ? 3
                 : (12ull * F.n + 4 <= FR_SMEM) ? 2 : ((u64)F.n * 4 <= FR_SMEM ? 1 : 0);
  size_t smem_bytes = use_smem == 3   ? (size_t)(3ull * F.n + 1 + ne) * 4
                      : use_smem == 2 ? (size_t)(3ull * F.n + 1) * 4
                      : use_smem == 1 ? (size_t)F.n * 4
                                      : 0;
  static int smem_set = 0;
  if (!smem_set) {
    CUDA_OK(cudaFuncSetAttribute(k_frontier_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FR_SMEM));
    smem_set = 1;
  }
  auto read_ctl = [&]() {
    CUDA_OK(cudaMemcpyAsync(h, ctl.p, 5 * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    if (lvl_host && F.lvl_off)
      CUDA_OK(cudaMemcpyAsync(lvl_host, F.lvl_off, ((u64)F.n + 2) * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    e.sync();
  };
  while (true) {
    k_frontier_block<<<1, LV_BLOCK, smem_bytes, e.s>>>(F, ctl.p, use_smem);
    if (!F.bfs) e.run_overlap_hook();  // overlap work runs while the peel does
    read_ctl();
    if (h[4]) break;
    u32* c = ctl.p;
    u32* hv = heavy.p;
    void* args[] = {&F, &c, &hv};
    CUDA_OK(cudaLaunchCooperativeKernel((const void*)k_frontier_grid, gblocks, 256, args, 0, e.s));
    read_ctl();
    if (h[4]) break;
  }
  nlevels = h[1];
  total = h[0];
}

// Barrier-free Kahn peel for class graphs that fit one CTA's shared memory
// (out-degree counters, levels, the work queue and the reverse CSR offsets).
// A level-synchronous peel pays a CTA barrier plus dependent L2 round trips
// per level, and these graphs are hundreds of levels deep and a few classes
// wide; here a class is processed as soon as its last child is: every class
// raises its parents' level (atomicMax of level + 1) and decrements their
// counters, and the thread that brings a counter to zero queues the parent.
// Warps take queue tickets; a class with more than 32 parent edges is swept
// by its whole warp.  ``pending`` (queued, not yet finished) reaching zero
// ends the walk.  The queue is then counting-sorted by level into the peel
// order + level offsets the level-synchronous consumers read.
#define PA_WIDE 32u
__global__ void __launch_bounds__(1024) k_peel_async(const u32* eoff, const u32* groff, const u32* grsrc, const u8* mask,
                                                     u32 n, u32 ne, u32* level_out, u32* order_out,
                                                     u32* lvl_off_out, u32* outdeg_out, u32* ctl) {
  extern __shared__ u32 sm[];
  u32* deg = sm;
  u32* lev = sm + n;
  u32* q = sm + 2 * (u64)n;
  u32* roff = sm + 3 * (u64)n;
  u32* rsrc = roff + n + 1;
  __shared__ u32 s_head, s_tail, s_pending, s_nl;
  const u32 FULL = 0xffffffffu, MASKED = 0x7fffffffu;
  unsigned long long t_a, t_b, t_c;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_a));
  if (threadIdx.x == 0) {
    s_head = 0;
    s_tail = 0;
    s_nl = 0;
  }
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    lev[i] = 0;
    q[i] = TSAT_NONE;
    roff[i] = groff[i];
  }
  if (threadIdx.x == 0) roff[n] = groff[n];
  const u32 ne_real = min(ne, groff[n]);  // ne may be the class graph's upper bound
  for (u32 e = threadIdx.x; e < ne_real; e += blockDim.x) rsrc[e] = grsrc[e];
  __syncthreads();
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    if (mask && !mask[i]) {
      deg[i] = MASKED;
      continue;
    }
    u32 d = eoff[i + 1] - eoff[i];
    deg[i] = d;
    if (d == 0) q[atomicAdd(&s_tail, 1u)] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) s_pending = s_tail;
  __syncthreads();
  const u32 lane = threadIdx.x & 31;
  auto raise = [&](u32 e, u32 lv) {
    u32 p = rsrc[e];
    if (!mask || mask[p]) atomicMax(&lev[p], lv + 1);
  };
  // a ready parent becomes the finder's next class when it has none (no
  // queue round trip on a chain), else it is queued
  auto push = [&](u32 p) {
    atomicAdd(&s_pending, 1u);
    u32 pos = atomicAdd(&s_tail, 1u);
    __threadfence_block();
    atomicExch(&q[pos], p);  // slot publish (atomic: the consumer spins on it)
  };
  u32 h = TSAT_NONE, cur = TSAT_NONE;
  bool done = false;
  while (true) {
    if (cur == TSAT_NONE && !done) {
      if (h == TSAT_NONE) {
        h = atomicAdd(&s_head, 1u);
        if (h >= n) done = true;
      }
      if (!done) {
        u32 x = atomicAdd(&q[h], 0u);
        if (x != TSAT_NONE) {
          cur = x;
          h = TSAT_NONE;
          __threadfence_block();
        } else if (((volatile u32*)&s_pending)[0] == 0) {
          done = true;
        }
      }
    }
    if (__all_sync(FULL, done)) break;
    const u32 v = cur;
    u32 a = 0, b = 0, lv = 0;
    if (v != TSAT_NONE) {
      a = roff[v];
      b = roff[v + 1];
      lv = ((volatile u32*)lev)[v];
    }
    unsigned wide = __ballot_sync(FULL, v != TSAT_NONE && b - a > PA_WIDE);
    while (wide) {
      int src = __ffs(wide) - 1;
      wide &= wide - 1;
      u32 wa = __shfl_sync(FULL, a, src), wb = __shfl_sync(FULL, b, src), wl = __shfl_sync(FULL, lv, src);
      for (u32 e0 = wa; e0 < wb; e0 += 32)
        if (e0 + lane < wb) raise(e0 + lane, wl);
      __threadfence_block();
      __syncwarp();
      for (u32 e0 = wa; e0 < wb; e0 += 32)
        if (e0 + lane < wb) {
          u32 p = rsrc[e0 + lane];
          if ((!mask || mask[p]) && atomicSub(&deg[p], 1u) == 1u) push(p);
        }
      __syncwarp();
    }
    if (v != TSAT_NONE) {
      u32 nxt = TSAT_NONE;
      if (b - a <= PA_WIDE) {
        for (u32 e = a; e < b; e++) raise(e, lv);
        __threadfence_block();
        for (u32 e = a; e < b; e++) {
          u32 p = rsrc[e];
          if ((!mask || mask[p]) && atomicSub(&deg[p], 1u) == 1u) {
            if (nxt == TSAT_NONE) nxt = p;
            else push(p);
          }
        }
      }
      if (nxt != TSAT_NONE) {
        cur = nxt;  // one class finished, one started: pending unchanged
        __threadfence_block();
      } else {
        __threadfence_block();
        atomicSub(&s_pending, 1u);
        cur = TSAT_NONE;
      }
    }
  }
  __syncthreads();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_b));
  // level histogram -> offsets -> peel order (the counters are reused)
  // (the queue holds only the classes that were handed over; q is reused as
  // the per-class level, TSAT_NONE = not peeled)
  if (threadIdx.x == 0) s_tail = 0;
  __syncthreads();
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    u32 d = deg[i];
    u32 l = d == 0 ? lev[i] : TSAT_NONE;
    level_out[i] = l;
    q[i] = l;
    outdeg_out[i] = d == MASKED ? 0u : d;
    if (l != TSAT_NONE) {
      atomicMax(&s_nl, l + 1);
      atomicAdd(&s_tail, 1u);
    }
  }
  __syncthreads();
  const u32 nl = s_nl, total = s_tail;
  u32* cnt = deg;  // nl <= n
  for (u32 i = threadIdx.x; i <= nl; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (u32 i = threadIdx.x; i < n; i += blockDim.x)
    if (q[i] != TSAT_NONE) atomicAdd(&cnt[q[i]], 1u);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of nl counts by one warp
    u32 carry = 0;
    for (u32 base = 0; base < nl; base += 32) {
      u32 i = base + lane;
      u32 x = i < nl ? cnt[i] : 0u, y = x;
      for (int o = 1; o < 32; o <<= 1) {
        u32 t = __shfl_up_sync(FULL, y, o);
        if (lane >= (u32)o) y += t;
      }
      if (i < nl) {
        cnt[i] = carry + y - x;
        lvl_off_out[i] = carry + y - x;
      }
      carry += __shfl_sync(FULL, y, 31);
    }
    if (lane == 0) lvl_off_out[nl] = carry;
  }
  __syncthreads();
  for (u32 i = threadIdx.x; i < n; i += blockDim.x)
    if (q[i] != TSAT_NONE) order_out[atomicAdd(&cnt[q[i]], 1u)] = i;
  __syncthreads();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_c));
  if (threadIdx.x == 0) {
    ctl[0] = total;
    ctl[1] = nl;
    ctl[2] = (u32)(t_b - t_a);  // ns: walk, then level sort (TSAT_DEBUG_LEVELS)
    ctl[3] = (u32)(t_c - t_b);
  }
}

#define PA_SMEM (200u << 10)

u32 trim_levels(Engine& e, const u8* mask, std::vector<u32>& lvl_off, u32& ntrimmed) {
  Scratch& X = e.sc;
  u32 n = e.cg_n;
  X.c_order.ensure(n + 1);
  X.c_lvloff.ensure(n + 3);
  Frontier F{X.cg_eoff.p, X.cg_edst.p, X.cg_roff.p, X.cg_rsrc.p, mask, X.cg_outdeg.p, X.cg_level.p,
             X.c_order.p, X.c_lvloff.p, nullptr, n, 0};
  u32 nl = 0, tot = 0;
  // the real edge count comes back with the peel's results (the class graph
  // was built on an upper bound, build_class_graph)
  if (!e.pin_small) CUDA_OK(cudaMallocHost((void**)&e.pin_small, 16 * sizeof(u32)));
  CUDA_OK(cudaMemcpyAsync(e.pin_small, X.cg_roff.p + n, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
  static const bool no_async = getenv("TSAT_PEEL_SYNC") != nullptr;
  // the barrier-free walk only when the whole reverse graph sits in shared
  // memory: with edges in L2 every class pays a dependent round trip and the
  // level-synchronous walk (edges flattened over the CTA) is faster
  if (!no_async && n > 0 && 16ull * n + 4ull * e.cg_ne + 16 <= PA_SMEM) {
    static int smem_set = 0;
    if (!smem_set) {
      CUDA_OK(cudaFuncSetAttribute(k_peel_async, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PA_SMEM));
      smem_set = 1;
    }
    size_t bytes = (size_t)(4ull * n + 1 + e.cg_ne) * 4;
    DevBuf<u32>& ctl = X.c_res;
    ctl.ensure(16);
    static const int pa_threads = getenv("TSAT_PEEL_THREADS") ? atoi(getenv("TSAT_PEEL_THREADS")) : 1024;
    k_peel_async<<<1, pa_threads, bytes, e.s>>>(X.cg_eoff.p, X.cg_roff.p, X.cg_rsrc.p, mask, n, e.cg_ne, X.cg_level.p,
                                          X.c_order.p, X.c_lvloff.p, X.cg_outdeg.p, ctl.p);
    CUDA_OK(cudaGetLastError());
    e.run_overlap_hook();  // work queued for the overlap stream runs while the peel does
    u32 hc[4];
    CUDA_OK(cudaMemcpyAsync(hc, ctl.p, 4 * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    lvl_off.resize((size_t)n + 2);
    CUDA_OK(cudaMemcpyAsync(lvl_off.data(), X.c_lvloff.p, ((u64)n + 2) * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    e.sync();  // (async path: n is small here, the whole offset array is a few KB)
    static const bool dbg = getenv("TSAT_DEBUG_LEVELS") != nullptr;
    if (dbg) fprintf(stderr, "peel_async: n %u ne %u walk %.1f us sort %.1f us\n", n, e.cg_ne, hc[2] * 1e-3, hc[3] * 1e-3);
    tot = hc[0];
    nl = hc[1];
  } else {
    // small graphs: the level offsets come back with the final control read
    // (one sync); large ones (10^6 classes) copy only the [0, nl] used
    const bool fold = n <= (1u << 16);
    lvl_off.resize(fold ? (size_t)n + 2 : 0);
    run_frontier(e, F, 0, nl, tot, e.cg_ne, fold ? lvl_off.data() : nullptr);
    if (!fold) {
      lvl_off.resize(nl + 1);
      CUDA_OK(cudaMemcpyAsync(lvl_off.data(), X.c_lvloff.p, (nl + 1) * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
      e.sync();
    }
  }
  ntrimmed = tot;
  lvl_off.resize(nl + 1);
  e.cg_ne = e.pin_small[0];  // landed before the peel's read-back (same stream, pinned)
  return nl;
}

// BFS over the class graph from ``root``; marks (u32) + queue; returns count
u32 bfs_graph(Engine& e, const u32* eoff, const u32* edst, u32 n, u32 root, u32* mark, u32* queue) {
  Frontier F{eoff, edst, nullptr, nullptr, nullptr, nullptr, nullptr, queue, nullptr, mark, n, 1};
  u32 nl = 0, tot = 0;
  run_frontier(e, F, root, nl, tot);
  return tot;
}

u32 bfs_classes(Engine& e, u32 root, u32* mark, u32* queue) {
  Frontier F{e.sc.cg_eoff.p, e.sc.cg_edst.p, nullptr, nullptr, nullptr, nullptr, nullptr, queue, nullptr, mark, e.cg_n, 1};
  u32 nl = 0, tot = 0;
  run_frontier(e, F, root, nl, tot, e.cg_ne);
  return tot;
}

