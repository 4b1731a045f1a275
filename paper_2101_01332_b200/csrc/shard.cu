// Multi-GPU sharding of e-matching (north star: "E-matching ...
// partitioned by e-class range across the GPUs ... match buffers exchanged via
// NCCL all-gather over NVLink, while union-find/rebuild stays on a single
// owner").
//
// Every rank holds a replica of the e-graph.  Rank r e-matches only the root
// candidates whose e-class id lies in its contiguous id range [lo_r, hi_r)
// (class id = min node id, reference egraph.py:64).  Because matches are
// ordered by (eclass, bindings) (egraph.py:107-112) and the ranges are
// contiguous and ascending in rank order, concatenating the ranks' sorted
// lists in rank order IS the global sorted list: the exchange is one
// all-gather of packed per-pattern lists plus an in-order unpack, no merge.
// Apply / rebuild / cycle filtering then run on identical inputs on every
// rank (deterministic), which is the owner's work replicated instead of an
// owner followed by a broadcast of the deltas.
//
// NCCL is loaded lazily (dlopen) so single-GPU use has no NCCL dependency;
// when PyTorch has already loaded its libnccl.so.2 the same library is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "engine.cuh"

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi a;
  if (a.lib) return a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw TsatException(TSAT_ERR_UNSUPPORTED, std::string("NCCL is not loadable: ") + dlerror());
  a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
  a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllGather || !a.GetErrorString)
    throw TsatException(TSAT_ERR_UNSUPPORTED, "NCCL library lacks required symbols");
  a.lib = h;
  return a;
}

#define NCCL_OK(x)                                                                                   \
  do {                                                                                               \
    ncclResult_t _r = (x);                                                                           \
    if (_r != ncclSuccess)                                                                           \
      throw TsatException(TSAT_ERR_CUDA, std::string("NCCL: ") + nccl().GetErrorString(_r) + " at " \
                                             __FILE__ ":" + std::to_string(__LINE__));               \
  } while (0)

void shard_range(u64 n_alloc, int rank, int world, u32& lo, u32& hi) {
  lo = (u32)(n_alloc * (u64)rank / (u64)world);
  hi = (u32)(n_alloc * (u64)(rank + 1) / (u64)world);
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  NCCL_OK(nccl().GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
}

// Communicators are shared by every engine of the process that was set up
// with the same unique id (one NCCL init per process group, not per e-graph).
struct CommEntry {
  std::string uid;
  int rank, world, device;
  ncclComm_t comm;
  int refs;
};
static std::vector<CommEntry>& comm_cache() {
  static std::vector<CommEntry> c;
  return c;
}

void Engine::shard_setup(int rank_, int world_, const void* id) {
  if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw TsatException(TSAT_ERR_ARG, "bad rank / world size");
  shard_teardown();
  shard_rank = rank_;
  shard_world = world_;
  if (world_ == 1 || !id) return;  // no id: local shard only (no exchange; tests)
  std::string key((const char*)id, NCCL_UNIQUE_ID_BYTES);
  for (auto& ce : comm_cache())
    if (ce.uid == key && ce.rank == rank_ && ce.world == world_ && ce.device == device) {
      ce.refs++;
      comm = (void*)ce.comm;
      return;
    }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  CUDA_OK(cudaSetDevice(device));
  NCCL_OK(nccl().CommInitRank(&c, world_, uid, rank_));
  comm_cache().push_back(CommEntry{key, rank_, world_, device, c, 1});
  comm = (void*)c;
}

void Engine::shard_teardown() {
  host_ag = nullptr;
  host_ctx = nullptr;
  if (comm) {
    sync();
    // the communicator stays cached for the process: the next e-graph of the
    // same group (bench steps, repeated explores) reuses it -- an NCCL unique
    // id must not be used for a second ncclCommInitRank once its bootstrap
    // has completed, so destroying here would make that re-init hang
    auto& cc = comm_cache();
    for (size_t i = 0; i < cc.size(); i++)
      if ((void*)cc[i].comm == comm) {
        if (cc[i].refs > 0) cc[i].refs--;
        break;
      }
    comm = nullptr;
  }
  shard_rank = 0;
  shard_world = 1;
}

// candidate sub-range [lo, hi) of each pattern's op table whose classes fall
// in [clo, chi): op tables are (op, class, id) ordered, so two lower bounds
__global__ void k_shard_bounds(G g, const u32* op_nodes, u32* rng, int np, u32 clo, u32 chi) {
  int p = threadIdx.x;
  if (p >= np) return;
  u32 a = rng[2 * p], b = rng[2 * p + 1];
  u32 out[2];
  for (int k = 0; k < 2; k++) {
    u32 key = k == 0 ? clo : chi, lo = a, hi = b;
    while (lo < hi) {
      u32 mid = (lo + hi) >> 1;
      if (uf_find_ro(g.parent, op_nodes[mid]) < key) lo = mid + 1;
      else hi = mid;
    }
    out[k] = lo;
  }
  rng[2 * p] = out[0];
  rng[2 * p + 1] = out[1];
}

void Engine::shard_candidate_ranges(std::vector<u32>& rng) {
  int np = (int)rng.size() / 2;
  if (shard_world <= 1 || np == 0) return;
  u32 clo, chi;
  shard_range(snap.n_alloc, shard_rank, shard_world, clo, chi);
  DevBuf<u32>& d = sc.sh_rng;
  d.ensure(rng.size() + 1);
  CUDA_OK(cudaMemcpyAsync(d.p, rng.data(), rng.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
  for (int p0 = 0; p0 < np; p0 += 1024)
    k_shard_bounds<<<1, 1024, 0, s>>>(view(), snap.op_nodes.p, d.p + 2 * p0, std::min(1024, np - p0), clo, chi);
  CUDA_OK(cudaMemcpyAsync(rng.data(), d.p, rng.size() * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
}

struct CopySeg {
  const u32* src;
  u32* dst;
  u64 n;
};

__global__ void k_copy_segs(const CopySeg* segs, int nseg) {
  for (int q = blockIdx.y; q < nseg; q += gridDim.y) {
    CopySeg sg = segs[q];
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < sg.n; i += (u64)gridDim.x * blockDim.x)
      sg.dst[i] = sg.src[i];
  }
}

static void copy_segs(Engine& e, const std::vector<CopySeg>& segs) {
  if (segs.empty()) return;
  DevBuf<unsigned char>& d = e.sc.sh_segs;
  d.ensure(segs.size() * sizeof(CopySeg));
  CUDA_OK(cudaMemcpyAsync(d.p, segs.data(), segs.size() * sizeof(CopySeg), cudaMemcpyHostToDevice, e.s));
  u64 mx = 0;
  for (auto& sg : segs) mx = std::max(mx, sg.n);
  unsigned gx = (unsigned)std::min<u64>((mx + 255) / 256, 1184);
  unsigned gy = (unsigned)std::min<size_t>(segs.size(), 65535);
  k_copy_segs<<<dim3(std::max(gx, 1u), gy), 256, 0, e.s>>>((const CopySeg*)d.p, (int)segs.size());
}

// All-gather the per-rank match lists of patterns ``pids`` (same list, same
// order on every rank) and rebuild each MatchSet as the rank-order
// concatenation.
void Engine::shard_gather_matches(const std::vector<int>& pids) {
  if (shard_world <= 1 || pids.empty() || !shard_exchange()) return;
  const int W = shard_world, np = (int)pids.size();
  // 1. per-pattern counts of every rank
  std::vector<u32> mine(np), all((size_t)W * np);
  for (int i = 0; i < np; i++) mine[i] = matches[pids[i]].n;
  DevBuf<u32>& dc = sc.sh_cnt;
  dc.ensure((size_t)(W + 1) * np + 1);
  CUDA_OK(cudaMemcpyAsync(dc.p, mine.data(), np * sizeof(u32), cudaMemcpyHostToDevice, s));
  shard_allgather(dc.p, dc.p + np, np * sizeof(u32));
  CUDA_OK(cudaMemcpyAsync(all.data(), dc.p + np, (size_t)W * np * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  // 2. pack this rank's lists: per pattern [classes | bindings]
  std::vector<u64> psize(W, 0);
  for (int r = 0; r < W; r++)
    for (int i = 0; i < np; i++) psize[r] += (u64)all[(size_t)r * np + i] * (1 + matches[pids[i]].nb);
  u64 smax = 1;
  for (int r = 0; r < W; r++) smax = std::max(smax, psize[r]);
  DevBuf<u32>& pk = sc.sh_pack;
  DevBuf<u32>& rv = sc.sh_recv;
  pk.ensure(smax);
  rv.ensure(smax * W);
  std::vector<CopySeg> segs;
  u64 o = 0;
  for (int i = 0; i < np; i++) {
    MatchSet& m = matches[pids[i]];
    segs.push_back({m.cls.p, pk.p + o, m.n});
    o += m.n;
    segs.push_back({m.bind.p, pk.p + o, (u64)m.n * m.nb});
    o += (u64)m.n * m.nb;
  }
  copy_segs(*this, segs);
  // 3. one all-gather of the packed lists (padded to the largest rank)
  shard_allgather(pk.p, rv.p, smax * sizeof(u32));
  // 4. unpack in rank order
  segs.clear();
  std::vector<u64> roff(W, 0);
  for (int i = 0; i < np; i++) {
    MatchSet& m = matches[pids[i]];
    u64 tot = 0;
    for (int r = 0; r < W; r++) tot += all[(size_t)r * np + i];
    m.cls.ensure(tot + 1);
    m.bind.ensure((tot + 1) * std::max(m.nb, 1));
    u64 base = 0;
    for (int r = 0; r < W; r++) {
      u64 n = all[(size_t)r * np + i];
      const u32* src = rv.p + (u64)r * smax + roff[r];
      segs.push_back({src, m.cls.p + base, n});
      segs.push_back({src + n, m.bind.p + base * m.nb, n * m.nb});
      roff[r] += n * (1 + m.nb);
      base += n;
    }
    m.n = (u32)tot;
  }
  copy_segs(*this, segs);
  sync();
}

// plain all-gather of ``bytes`` from every rank into recv (rank order)
void Engine::shard_allgather_bytes(const void* send, void* recv, size_t bytes) {
  if (shard_world <= 1 || !shard_exchange()) throw TsatException(TSAT_ERR_STATE, "no shard communicator");
  shard_allgather(send, recv, bytes);
}

// The one exchange primitive: NCCL over NVLink when a communicator exists,
// else the caller's host all-gather (device -> host, callback, host -> device
// on the engine stream).  Both deliver rank r's bytes at recv + r * bytes.
void Engine::shard_allgather(const void* dsend, void* drecv, size_t bytes) {
  if (comm) {
    NCCL_OK(nccl().AllGather(dsend, drecv, bytes, ncclUint8, (ncclComm_t)comm, s));
    return;
  }
  if (!host_ag) throw TsatException(TSAT_ERR_STATE, "no shard transport");
  ag_send.resize(bytes + 1);
  ag_recv.resize(bytes * (size_t)shard_world + 1);
  if (bytes) CUDA_OK(cudaMemcpyAsync(ag_send.data(), dsend, bytes, cudaMemcpyDeviceToHost, s));
  sync();
  if (host_ag(host_ctx, ag_send.data(), ag_recv.data(), (uint64_t)bytes) != 0)
    throw TsatException(TSAT_ERR_STATE, "host all-gather transport failed");
  if (bytes) CUDA_OK(cudaMemcpyAsync(drecv, ag_recv.data(), bytes * (size_t)shard_world, cudaMemcpyHostToDevice, s));
  sync();
}
