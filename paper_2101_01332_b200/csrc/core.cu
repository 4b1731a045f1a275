// libtsat core: buffers, loading, sequential (exact) mutation kernels,
// parallel congruence rebuild, snapshot CSR construction, download + dump.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <sstream>

#include <mutex>

#include "engine.cuh"
#include "rulesdev.cuh"

namespace cg = cooperative_groups;

static inline unsigned nblk(u64 n, unsigned t = 256) {
  u64 b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148ull * 64) b = 148ull * 64;  // grid-stride beyond 64 CTAs per SM
  return (unsigned)b;
}

#define GRID_STRIDE(i, n) for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

u32 bits_for(u32 maxval) {
  u32 b = 1;
  while (b < 32 && (1ull << b) <= maxval) b++;
  return b;
}

// ---------------------------------------------------------------- cub helpers

void dev_exclusive_scan_u32(Engine& e, const u32* in, u32* out, u32 n) {
  size_t bytes = 0;
  CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, e.s));
  e.temp.ensure(bytes + 16);
  CUDA_OK(cub::DeviceScan::ExclusiveSum(e.temp.p, bytes, in, out, n, e.s));
}

void dev_sort_pairs_u32(Engine& e, u32* kin, u32* kout, u32* vin, u32* vout, u32 n, int end_bit) {
  size_t bytes = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, e.s));
  e.temp.ensure(bytes + 16);
  CUDA_OK(cub::DeviceRadixSort::SortPairs(e.temp.p, bytes, kin, kout, vin, vout, n, 0, end_bit, e.s));
}

// ---------------------------------------------------------------- lifecycle

Engine::Engine(int dev) : device(dev) {
  CUDA_OK(cudaSetDevice(dev));
  CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  tl_stream = s;
  g_engines++;
  cnt.alloc(1);
  err.alloc(1);
  dstats.alloc(1);
  CUDA_OK(cudaMemsetAsync(cnt.p, 0, sizeof(Counters), s));
  CUDA_OK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
  memset(&h, 0, sizeof(h));
  tree_cap = 1 << 16;
  tree_hc_cap = 1 << 18;
  trees.alloc(tree_cap);
  tree_hc.alloc(tree_hc_cap);
  tree_count.alloc(1);
  CUDA_OK(cudaMemsetAsync(tree_hc.p, 0xFF, tree_hc_cap * sizeof(u32), s));
  CUDA_OK(cudaMemsetAsync(tree_count.p, 0, sizeof(u32), s));
  ensure_nodes(1024, 4096);
  reach.budget = default_reach_budget();
  sync();
}

u64 default_reach_budget() {
  const char* v = getenv("TSAT_REACH_BUDGET");
  return v ? strtoull(v, nullptr, 10) : 0ull;
}

KTimer::KTimer(Engine& e_, int g_, double bytes_, unsigned long long launches_)
    : e(e_), g(g_), bytes(bytes_), launches(launches_) {
  a = e.ev_get();
  b = nullptr;
  CUDA_OK(cudaEventRecord(a, e.s));
}

// The closing event is recorded and queued; its elapsed time is read when the
// stats are queried (tsat_kernel_stats) or when the queue grows, so timing a
// group never makes the host wait for the device.
KTimer::~KTimer() {
  b = e.ev_get();
  cudaEventRecord(b, e.s);
  e.kt_pending.push_back({a, b, g});
  e.kstat[g].bytes += bytes;
  e.kstat[g].launches += launches;
  e.nlaunch += launches;
  if (e.kt_pending.size() >= 256) e.kt_resolve(false);
}

cudaEvent_t Engine::ev_get() {
  if (ev_free.empty()) {
    cudaEvent_t ev;
    CUDA_OK(cudaEventCreate(&ev));
    return ev;
  }
  cudaEvent_t ev = ev_free.back();
  ev_free.pop_back();
  return ev;
}

void Engine::kt_resolve(bool block) {
  size_t k = 0;
  for (; k < kt_pending.size(); k++) {
    PendingTimer& t = kt_pending[k];
    if (block) {
      CUDA_OK(cudaEventSynchronize(t.b));
    } else if (cudaEventQuery(t.b) != cudaSuccess) {
      cudaGetLastError();  // cudaErrorNotReady is not an error
      break;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    kstat[t.g].ms += ms;
    ev_free.push_back(t.a);
    ev_free.push_back(t.b);
  }
  kt_pending.erase(kt_pending.begin(), kt_pending.begin() + k);
}

void free_wave_bufs(WaveBufs* b);

// return a pooled engine to the freshly-created state, keeping allocations
void Engine::reset(bool analysis_) {
  sync();
  shard_teardown();
  analysis = analysis_;
  memset(&h, 0, sizeof(h));
  push_counters();
  CUDA_OK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
  CUDA_OK(cudaMemsetAsync(tree_hc.p, 0xFF, (size_t)tree_hc_cap * sizeof(u32), s));
  CUDA_OK(cudaMemsetAsync(tree_count.p, 0, sizeof(u32), s));
  if (hc_cap) CUDA_OK(cudaMemsetAsync(hc.p, 0, (size_t)hc_cap * sizeof(unsigned long long), s));
  hc_epoch = 1;
  hc_tombs = 0;
  root = TSAT_NONE;
  h_atoms.clear();
  atom_names.clear();
  patterns.clear();
  rules.clear();
  rule_names.clear();
  for (auto& m : matches) m.n = 0;  // keep the device buffers for the next graph
  snap.valid = false;
  reach.valid = false;
  reach.mode = 0;
  reach.budget = default_reach_budget();
  uf_changed = false;
  lv_snap = lv_filter = ~0ull;
  costs_valid_for = TSAT_NONE;
  kt_resolve(true);
  for (int i = 0; i < KG_COUNT; i++) kstat[i] = KStat();
  nlaunch = 0;
  last_error.clear();
  sync();
}

Engine::~Engine() {
  try {
    shard_teardown();
  } catch (...) {
  }
  if (s) cudaStreamSynchronize(s);
  for (auto& t : kt_pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto ev : ev_free) cudaEventDestroy(ev);
  // everything this engine released is idle now; members released below too
  tl_stream = nullptr;
  if (wave) free_wave_bufs(wave);
  if (s2) {
    cudaStreamSynchronize(s2);
    dev_cache_forget_stream(s2);
    cudaStreamDestroy(s2);
  }
  if (ev_ov) cudaEventDestroy(ev_ov);
  if (pin_small) cudaFreeHost(pin_small);
  if (s) {
    dev_cache_forget_stream(s);
    cudaStreamDestroy(s);
  }
}

// Run the pending overlap work (if any) on the overlap stream: the engine's
// stream, CUB scratch and allocator stream are swapped for its duration, so
// every launch / sync inside goes to s2; it waits only for ev_ov (recorded
// before the work it overlaps), and the main stream waits for it afterwards.
void Engine::run_overlap_hook() {
  if (!overlap_hook) return;
  std::function<void()> f = std::move(overlap_hook);
  overlap_hook = nullptr;
  CUDA_OK(cudaStreamWaitEvent(s2, ev_ov, 0));
  std::swap(s, s2);
  temp.swap(temp2);
  tl_stream = s;
  try {
    f();
  } catch (...) {
    std::swap(s, s2);
    temp.swap(temp2);
    tl_stream = s;
    throw;
  }
  CUDA_OK(cudaEventRecord(ev_ov, s));
  std::swap(s, s2);
  temp.swap(temp2);
  tl_stream = s;
  CUDA_OK(cudaStreamWaitEvent(s, ev_ov, 0));
}

G Engine::view() {
  G g;
  g.op = op.p;
  g.koff = koff.p;
  g.kids = kids.p;
  g.parent = parent.p;
  g.flags = flags.p;
  g.val = val.p;
  g.hc = hc.p;
  g.hc_mask = hc_cap - 1;
  g.hc_max = (u32)std::min<double>((double)hc_cap * hc_load(), 4294967295.0);
  g.hc_epoch = hc_epoch;
  g.cap_nodes = cap_nodes;
  g.cap_kids = cap_kids;
  g.analysis = analysis ? 1 : 0;
  g.atoms = atoms.p;
  g.tt.trees = trees.p;
  g.tt.hc = tree_hc.p;
  g.tt.hc_mask = tree_hc_cap - 1;
  g.tt.count = tree_count.p;
  g.tt.cap = tree_cap;
  g.err = err.p;
  g.cnt = cnt.p;
  return g;
}

unsigned long long g_dev_allocs = 0, g_dev_alloc_bytes = 0, g_engines = 0;
thread_local cudaStream_t tl_stream = nullptr;

// ---------------------------------------------------------------- device block cache
namespace {
struct CachedBlock {
  void* p;
  cudaStream_t s;  // stream of the last user (nullptr: idle)
};
struct DevCache {
  std::mutex mu;
  std::vector<CachedBlock> free_[64];  // bucket b holds blocks of 2^b bytes
};
DevCache& dev_cache() {
  static DevCache* c = new DevCache();  // never destroyed: blocks outlive static teardown
  return *c;
}
int bucket_of(size_t bytes) {
  int b = 8;  // >= 256 B
  while (((size_t)1 << b) < bytes) b++;
  return b;
}
}  // namespace

void* dev_cache_get(size_t bytes) {
  int b = bucket_of(bytes);
  DevCache& c = dev_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto& fl = c.free_[b];
    for (size_t i = fl.size(); i-- > 0;) {
      if (fl[i].s == tl_stream || fl[i].s == nullptr) {
        void* p = fl[i].p;
        fl.erase(fl.begin() + i);
        return p;
      }
    }
    if (!fl.empty()) {
      CachedBlock blk = fl.back();
      fl.pop_back();
      CUDA_OK(cudaStreamSynchronize(blk.s));  // last user may still read it
      return blk.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)1 << b);
  if (e != cudaSuccess) {
    // out of memory: release idle cached blocks and retry once
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> g(c.mu);
      CUDA_OK(cudaDeviceSynchronize());
      for (auto& fl : c.free_) {
        for (auto& blk : fl) cudaFree(blk.p);
        fl.clear();
      }
    }
    CUDA_OK(cudaMalloc(&p, (size_t)1 << b));
  }
  g_dev_allocs++;
  g_dev_alloc_bytes += (size_t)1 << b;
  return p;
}

void dev_cache_put(void* p, size_t bytes) {
  DevCache& c = dev_cache();
  std::lock_guard<std::mutex> g(c.mu);
  c.free_[bucket_of(bytes)].push_back(CachedBlock{p, tl_stream});
}

void dev_cache_forget_stream(cudaStream_t s) {
  DevCache& c = dev_cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (auto& fl : c.free_)
    for (auto& blk : fl)
      if (blk.s == s) blk.s = nullptr;
}

bool g_dbg_sites = getenv("TSAT_DEBUG_SYNCS") != nullptr;
std::map<std::string, long> g_site_counts;
void tsat_count_site(const char* what, const char* file, int line) {
  const char* kind = strncmp(what, "cudaMemcpyAsync", 15) == 0
                         ? (strstr(what, "HostToDevice") ? "H2D" : strstr(what, "DeviceToHost") ? "D2H" : "D2D")
                     : strncmp(what, "cudaMemsetAsync", 15) == 0 ? "memset"
                                                                 : nullptr;
  if (!kind) return;
  const char* b = strrchr(file, '/');
  g_site_counts[std::string(kind) + " " + (b ? b + 1 : file) + ":" + std::to_string(line)]++;
}

void Engine::sync(const char* sf, int sl) {
  nsync++;
  static const bool dbg = getenv("TSAT_DEBUG_SYNCS") != nullptr;
  if (dbg) {
    const char* b = strrchr(sf, '/');
    sync_sites[std::string(b ? b + 1 : sf) + ":" + std::to_string(sl)]++;
  }
  CUDA_OK(cudaStreamSynchronize(s));
}

void Engine::pull_counters(const char* sf, int sl) {
  CUDA_OK(cudaMemcpyAsync(&h, cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  sync(sf, sl);
}

void Engine::push_counters() {
  CUDA_OK(cudaMemcpyAsync(cnt.p, &h, sizeof(Counters), cudaMemcpyHostToDevice, s));
}

static const char* status_name(int c) {
  switch (c) {
    case TSAT_ERR_SHAPE: return "ShapeMismatch";
    case TSAT_ERR_SPLIT_ORIGIN: return "MissingSplitOrigin";
    case TSAT_ERR_MERGE: return "AnalysisMergeError";
    case TSAT_ERR_CAPACITY: return "capacity";
    default: return "error";
  }
}

void Engine::check_error(const char* sf, int sl) {
  DevError he;
  CUDA_OK(cudaMemcpyAsync(&he, err.p, sizeof(he), cudaMemcpyDeviceToHost, s));
  sync(sf, sl);
  raise_error(he);
}

// throw the device error ``he`` (read back by the caller) if one is set
void Engine::raise_error(const DevError& he) {
  if (he.code != 0) {
    CUDA_OK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
    std::ostringstream os;
    os << status_name(he.code) << " (detail " << he.detail << ", " << he.a << ", " << he.b << ")";
    if (he.code == TSAT_ERR_MERGE) {
      os.str("");
      os << "incompatible analyses " << value_str((u32)he.a) << " vs " << value_str((u32)he.b);
    } else if (he.code == TSAT_ERR_SHAPE || he.code == TSAT_ERR_SPLIT_ORIGIN) {
      os.str("");
      std::string opn = (he.b >= 0 && (size_t)he.b < atom_names.size()) ? atom_names[he.b] : "?";
      os << "shape inference failed for operator '" << opn << "' (node n" << he.a << ")";
    }
    throw TsatException(he.code, os.str());
  }
}

// ---------------------------------------------------------------- capacity

__global__ void k_hc_insert_alive(G g, u32 n) {
  GRID_STRIDE(i, n) {
    if (g.flags[i] & NF_ALIVE) hc_insert(g, (u32)i);
  }
}

// the next hashcons epoch: an empty table without a clear (a clear every 255)
void Engine::hc_new_epoch() {
  hc_tombs = 0;
  if (++hc_epoch > 255) {
    CUDA_OK(cudaMemsetAsync(hc.p, 0, (size_t)hc_cap * sizeof(unsigned long long), s));
    hc_epoch = 1;
  }
}

void Engine::rehash(u32 new_cap) {
  hc.alloc(new_cap);
  hc_cap = new_cap;
  hc_epoch = 1;
  hc_tombs = 0;
  CUDA_OK(cudaMemsetAsync(hc.p, 0, (size_t)new_cap * sizeof(unsigned long long), s));
  if (h.next_id) k_hc_insert_alive<<<nblk(h.next_id), 256, 0, s>>>(view(), h.next_id);
}

double hc_load() {
  static const double l = getenv("TSAT_HC_LOAD") ? atof(getenv("TSAT_HC_LOAD")) : 0.5;
  return l;
}

void Engine::ensure_nodes(u64 extra_nodes, u64 extra_kids) {
  u64 need_n = (u64)h.next_id + extra_nodes + 1;
  u64 need_k = (u64)h.nkids + extra_kids + 1;
  if (need_n >= 0xF0000000ull || need_k >= 0xF0000000ull)
    throw TsatException(TSAT_ERR_CAPACITY, "e-graph exceeds 32-bit id space");
  if (need_n > cap_nodes) {
    u64 nc = cap_nodes ? cap_nodes : 1024;
    while (nc < need_n) nc *= 2;
    op.grow(nc, h.next_id, s);
    koff.grow(nc + 1, (u64)h.next_id + 1, s);
    parent.grow(nc, h.next_id, s);
    flags.grow(nc, h.next_id, s);
    val.grow(nc, h.next_id, s);
    cap_nodes = (u32)std::min<u64>(nc, op.cap);
    if (h.next_id == 0) CUDA_OK(cudaMemsetAsync(koff.p, 0, sizeof(u32), s));
  }
  if (need_k > cap_kids) {
    u64 nc = cap_kids ? cap_kids : 4096;
    while (nc < need_k) nc *= 2;
    kids.grow(nc, h.nkids, s);
    cap_kids = (u32)kids.cap;
  }
  // hashcons load factor <= 1/2 over all allocated ids (TSAT_HC_LOAD overrides)
  u64 want = 16;
  while ((double)want * hc_load() < (double)need_n) want *= 2;
  if (want > hc_cap) rehash((u32)want);
}

// ---------------------------------------------------------------- atoms

void Engine::set_atoms(int n, const int32_t* kind, const i64* ival, const int32_t* opcode,
                       const int32_t* ndims, const i64* dims, const int32_t* nident, const i64* idims,
                       const char* names_blob, const i64* name_off) {
  size_t old = h_atoms.size();
  if ((size_t)n < old) throw TsatException(TSAT_ERR_ARG, "atom table can only grow");
  for (int i = (int)old; i < n; i++) {
    AtomInfo a;
    memset(&a, 0, sizeof(a));
    a.kind = kind[i];
    a.opcode = opcode[i];
    a.ival = ival[i];
    a.ndims = ndims[i];
    a.nident = nident[i];
    for (int j = 0; j < 4; j++) {
      a.dims[j] = dims[4 * (size_t)i + j];
      a.idims[j] = idims[4 * (size_t)i + j];
    }
    h_atoms.push_back(a);
    atom_names.emplace_back(names_blob + name_off[i], names_blob + name_off[i + 1]);
  }
  if (atoms.cap < h_atoms.size()) atoms.grow(h_atoms.size() * 2 + 16, 0, s);
  CUDA_OK(cudaMemcpyAsync(atoms.p, h_atoms.data(), h_atoms.size() * sizeof(AtomInfo),
                          cudaMemcpyHostToDevice, s));
  // atom names (signature keys for cost-table lookups are rendered on device)
  std::vector<char> blob;
  std::vector<u32> offs;
  for (auto& nm : atom_names) {
    offs.push_back((u32)blob.size());
    blob.insert(blob.end(), nm.begin(), nm.end());
  }
  offs.push_back((u32)blob.size());
  sync();
  d_names.ensure(blob.size() + 1);
  d_name_off.ensure(offs.size());
  if (!blob.empty())
    CUDA_OK(cudaMemcpyAsync(d_names.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpyAsync(d_name_off.p, offs.data(), offs.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
  sync();
}

// ---------------------------------------------------------------- bulk load

__global__ void k_init_nodes(G g, u32 n) {
  GRID_STRIDE(i, n) {
    g.parent[i] = (u32)i;
    g.flags[i] = NF_ALIVE;
  }
}

__device__ __forceinline__ void make_one(const G& g, u32 nid) {
  u32 a = g.koff[nid], b = g.koff[nid + 1];
  int k = (int)(b - a);
  const Val* kv[8];
  if (k > 7) {
    dev_set_error(g.err, TSAT_ERR_SHAPE, 3, nid, g.op[nid]);
    return;
  }
  for (int j = 0; j < k; j++) kv[j] = &g.val[g.kids[a + j]];
  Val v;
  int st = val_make(g.op[nid], ValRefs{kv}, k, v, g.atoms, g.tt);
  if (st != AS_OK) {
    dev_set_error(g.err, ana_to_status(st), 3, nid, g.op[nid]);
    return;
  }
  g.val[nid] = v;
}

// consecutive thin levels [l0, l1) in one CTA (deep noop chains are common);
// levels of at most 32 nodes are walked by warp 0 alone with __syncwarp only
__global__ void __launch_bounds__(256) k_make_levels(G g, const u32* ids, const u32* off, u32 l0, u32 l1) {
  __shared__ u32 s_next;
  for (u32 l = l0; l < l1;) {
    if (off[l + 1] - off[l] <= 32) {
      if (threadIdx.x < 32) {
        u32 ll = l;
        while (ll < l1 && off[ll + 1] - off[ll] <= 32) {
          u32 t = off[ll] + threadIdx.x;
          if (t < off[ll + 1]) make_one(g, ids[t]);
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
    for (u32 t = off[l] + threadIdx.x; t < off[l + 1]; t += blockDim.x) make_one(g, ids[t]);
    __syncthreads();
    l++;
  }
}

// analysis values for the nodes of one depth level (children already valued)
__global__ void k_make_level(G g, const u32* ids, u32 n) {
  GRID_STRIDE(t, n) {
    u32 nid = ids[t];
    u32 a = g.koff[nid], b = g.koff[nid + 1];
    int k = (int)(b - a);
    const Val* kv[8];
    if (k > 7) {
      dev_set_error(g.err, TSAT_ERR_SHAPE, 3, nid, g.op[nid]);
      continue;
    }
    for (int j = 0; j < k; j++) kv[j] = &g.val[g.kids[a + j]];
    Val v;
    int st = val_make(g.op[nid], ValRefs{kv}, k, v, g.atoms, g.tt);
    if (st != AS_OK) {
      dev_set_error(g.err, ana_to_status(st), 3, nid, g.op[nid]);
      continue;
    }
    g.val[nid] = v;
  }
}

void Engine::load_initial(u32 n, const u32* hop, const u32* hkoff, const u32* hkids, u32 r) {
  if (h.next_id != 0) throw TsatException(TSAT_ERR_STATE, "load_initial on a non-empty e-graph");
  u32 nk = hkoff[n];
  for (u32 i = 0; i < n; i++)
    for (u32 j = hkoff[i]; j < hkoff[i + 1]; j++)
      if (hkids[j] >= i) throw TsatException(TSAT_ERR_ARG, "children must precede their parent");
  ensure_nodes(n, nk);
  CUDA_OK(cudaMemcpyAsync(op.p, hop, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpyAsync(koff.p, hkoff, (n + 1) * sizeof(u32), cudaMemcpyHostToDevice, s));
  if (nk) CUDA_OK(cudaMemcpyAsync(kids.p, hkids, nk * sizeof(u32), cudaMemcpyHostToDevice, s));
  k_init_nodes<<<nblk(n), 256, 0, s>>>(view(), n);
  h.next_id = n;
  h.live = n;
  h.nkids = nk;
  h.dirty = 0;
  push_counters();
  k_hc_insert_alive<<<nblk(n), 256, 0, s>>>(view(), n);
  if (analysis) {
    // depth levels computed on the host from the (small) initial graph
    std::vector<u32> lvl(n, 0);
    u32 maxl = 0;
    for (u32 i = 0; i < n; i++) {
      u32 l = 0;
      for (u32 j = hkoff[i]; j < hkoff[i + 1]; j++) l = std::max(l, lvl[hkids[j]] + 1);
      lvl[i] = l;
      maxl = std::max(maxl, l);
    }
    std::vector<std::vector<u32>> by(maxl + 1);
    for (u32 i = 0; i < n; i++) by[lvl[i]].push_back(i);
    DevBuf<u32>& ids = scratch_u32[0];
    ids.ensure(n + 1);
    std::vector<u32> flat;
    std::vector<size_t> off;
    for (auto& v : by) {
      off.push_back(flat.size());
      flat.insert(flat.end(), v.begin(), v.end());
    }
    CUDA_OK(cudaMemcpyAsync(ids.p, flat.data(), flat.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    off.push_back(flat.size());
    std::vector<u32> off32(off.begin(), off.end());
    DevBuf<u32>& doff = scratch_u32[1];
    doff.ensure(off32.size() + 1);
    CUDA_OK(cudaMemcpyAsync(doff.p, off32.data(), off32.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    for (size_t l = 0; l < by.size();) {
      if (by[l].size() > 256) {
        k_make_level<<<nblk(by[l].size()), 128, 0, s>>>(view(), ids.p + off[l], (u32)by[l].size());
        l++;
        continue;
      }
      size_t l1 = l;
      while (l1 < by.size() && by[l1].size() <= 256) l1++;
      k_make_levels<<<1, 256, 0, s>>>(view(), ids.p, doff.p, (u32)l, (u32)l1);
      l = l1;
    }
  }
  root = r;
  root_ver = ~0ull;
  check_error();  // the one sync (the level vectors above outlive it)
}

// ---------------------------------------------------------------- sequential ops

// run a batch of term programs (post-order Instr) against env, one thread:
// exactly add_term (egraph.py:184-191) for each term in order.
__global__ void k_seq_add_terms(G g, const Instr* prog, const int32_t* term_len, int nterm,
                                const u32* env, u32* out) {
  if (threadIdx.x || blockIdx.x) return;
  u32 stack[64];
  int pc = 0;
  for (int t = 0; t < nterm; t++) {
    int sp = 0;
    for (int k = 0; k < term_len[t]; k++, pc++) {
      const Instr& in = prog[pc];
      if (in.kind == I_VAR) {
        stack[sp++] = uf_find(g.parent, env[in.arg]);
      } else {
        int na = in.arg;
        sp -= na;
        u32 kidsb[8];
        for (int j = 0; j < na; j++) kidsb[j] = stack[sp + j];
        u32 c = seq_add_enode(g, in.atom, kidsb, na);
        if (c == TSAT_NONE) return;
        stack[sp++] = c;
      }
    }
    out[t] = stack[0];
  }
}

void Engine::add_terms(int ninstr, const Instr* prog, int nterm, const int32_t* term_len, int nenv,
                       const u32* env, u32* out_cls) {
  u64 napp = 0, nk = 0;
  for (int i = 0; i < ninstr; i++) {
    if (prog[i].kind == I_APP) {
      napp++;
      nk += prog[i].arg;
      if (prog[i].arg > 8) throw TsatException(TSAT_ERR_ARG, "arity > 8 not supported");
    }
  }
  ensure_nodes(napp, nk);
  DevBuf<Instr>& dp = sc.a_prog;
  dp.ensure(ninstr + 1);
  DevBuf<int32_t>& dl = sc.a_len;
  dl.ensure(nterm + 1);
  DevBuf<u32>& de = sc.a_env;
  DevBuf<u32>& dout = sc.a_out;
  de.ensure(nenv + 1);
  dout.ensure(nterm + 1);
  CUDA_OK(cudaMemcpyAsync(dp.p, prog, ninstr * sizeof(Instr), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpyAsync(dl.p, term_len, nterm * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (nenv) CUDA_OK(cudaMemcpyAsync(de.p, env, nenv * sizeof(u32), cudaMemcpyHostToDevice, s));
  snap.valid = false;
  k_seq_add_terms<<<1, 1, 0, s>>>(view(), dp.p, dl.p, nterm, de.p, dout.p);
  CUDA_OK(cudaMemcpyAsync(out_cls, dout.p, nterm * sizeof(u32), cudaMemcpyDeviceToHost, s));
  pull_counters();
  check_error();
}

__global__ void k_seq_union(G g, u32 a, u32 b, u32* out) {
  if (threadIdx.x || blockIdx.x) return;
  *out = seq_union(g, a, b);
}

u32 Engine::union_pair(u32 a, u32 b) {
  if (a >= h.next_id || b >= h.next_id) throw TsatException(TSAT_ERR_ARG, "unknown e-class id");
  DevBuf<u32>& o = scratch_u32[7];
  o.ensure(1);
  snap.valid = false;
  uf_changed = true;
  k_seq_union<<<1, 1, 0, s>>>(view(), a, b, o.p);
  u32 r;
  CUDA_OK(cudaMemcpyAsync(&r, o.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  pull_counters();
  check_error();
  return r;
}

__global__ void k_find(G g, u32 x, u32* out) {
  if (threadIdx.x || blockIdx.x) return;
  *out = uf_find(g.parent, x);
}

u32 Engine::find(u32 x) {
  if (x >= h.next_id) throw TsatException(TSAT_ERR_ARG, "unknown id");
  DevBuf<u32>& o = scratch_u32[7];
  o.ensure(1);
  k_find<<<1, 1, 0, s>>>(view(), x, o.p);
  u32 r;
  CUDA_OK(cudaMemcpyAsync(&r, o.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  return r;
}

// ---------------------------------------------------------------- filter list

__global__ void k_set_filter(G g, const u32* ids, u32 n, int on) {
  GRID_STRIDE(i, n) {
    u32 x = ids[i];
    if (on) g.flags[x] |= NF_FILT;
    else g.flags[x] &= ~NF_FILT;
  }
}

__global__ void k_clear_filter(G g, u32 n) {
  GRID_STRIDE(i, n) g.flags[i] &= ~NF_FILT;
}

void Engine::set_filter(int n, const u32* ids, int on) {
  filter_id++;
  if (on == 2) {
    if (h.next_id) k_clear_filter<<<nblk(h.next_id), 256, 0, s>>>(view(), h.next_id);
    sync();
    return;
  }
  if (n <= 0) return;
  for (int i = 0; i < n; i++)
    if (ids[i] >= h.next_id) throw TsatException(TSAT_ERR_ARG, "filter id out of range");
  DevBuf<u32>& d = sc.a_ids;
  d.ensure(n);
  CUDA_OK(cudaMemcpyAsync(d.p, ids, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  k_set_filter<<<nblk(n), 256, 0, s>>>(view(), d.p, n, on);
  sync();
}

__global__ void k_filt_flags(const u8* flags, u32 n, u32* fl) {
  GRID_STRIDE(i, n) fl[i] = (flags[i] & NF_FILT) ? 1u : 0u;
}

__global__ void k_filt_compact(const u32* fl, const u32* pos, u32 n, u32* out) {
  GRID_STRIDE(i, n) if (fl[i]) out[pos[i]] = (u32)i;
}

// filter-listed node ids, ascending: compacted on the device (only the ids
// cross PCIe, not a flag byte per node)
std::vector<u32> Engine::get_filter() {
  u32 n = h.next_id;
  std::vector<u32> out;
  if (!n) return out;
  DevBuf<u32>& fl = scratch_u32[1];
  DevBuf<u32>& pos = scratch_u32[2];
  DevBuf<u32>& ids = scratch_u32[3];
  fl.ensure(n + 1);
  pos.ensure(n + 1);
  k_filt_flags<<<nblk(n), 256, 0, s>>>(flags.p, n, fl.p);
  CUDA_OK(cudaMemsetAsync(fl.p + n, 0, sizeof(u32), s));
  dev_exclusive_scan_u32(*this, fl.p, pos.p, n + 1);
  u32 cnt = 0;
  CUDA_OK(cudaMemcpyAsync(&cnt, pos.p + n, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  if (!cnt) return out;
  ids.ensure(cnt + 1);
  k_filt_compact<<<nblk(n), 256, 0, s>>>(fl.p, pos.p, n, ids.p);
  out.resize(cnt);
  CUDA_OK(cudaMemcpyAsync(out.data(), ids.p, cnt * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  return out;
}

// ---------------------------------------------------------------- rebuild
// Congruence closure to fixpoint (reference egraph.py:216-238).  Each round:
// canonicalise every live node's children against the frozen union-find,
// regroup by (op, children) keeping the minimum id per key, drop the others
// and union their classes with the survivor's.  Survivor = min id per final
// key and the partition is the congruence closure, so the result equals the
// reference's sequential pass (verified by the parity tests).

// One congruence round, fused: every live node canonicalises its children
// against the union-find (writing them back), hashes the canonical key and
// claims its hashcons slot in the round's fresh epoch.  A node meeting an equal
// key (fingerprint first, then the other node's children through find()) does
// atomicMin on the slot: the larger of the two ids is a non-survivor and is
// dropped and unioned on the spot -- each non-minimum of a key group loses
// exactly once, the minimum never does, so no second pass is needed.  Unions
// made during the round only make later keys fresher; the round loop runs to
// a fixpoint (no union), whose final round leaves exactly the live nodes in
// the table under their canonical keys.
__device__ __forceinline__ bool key_eq_canon(const G& g, u32 other, u32 op, u32 a, u32 n) {
  if (g.op[other] != op) return false;
  u32 ao = g.koff[other];
  if (g.koff[other + 1] - ao != n) return false;
  for (u32 j = 0; j < n; j++)
    if (uf_find_ro(g.parent, g.kids[ao + j]) != g.kids[a + j]) return false;
  return true;
}

static_assert(sizeof(Val) % 16 == 0, "Val is copied in 16-byte words");
struct RbCtl {
  u32 ndirty[2];  // dirty-list length by round parity
  u32 nlinked;    // links so far (merge list length)
  u32 dropped;
  u32 rounds;
  u32 dirty_total;
  u32 tombs;
  u32 lost;       // dirty nodes whose slot was not found (invariant check)
  unsigned long long t[4];  // %globaltimer: start, rounds done, merges done (TSAT_DEBUG_REBUILD)
};

// canonicalise node i's children (written back), then claim its slot under
// the canonical key; a congruent node met there makes the larger id the loser:
// dropped and its class linked on the spot (one drop per non-minimum).
__device__ __forceinline__ u32 rb_process(const G& g, u32 i, u32* linkbits) {
  u32 a = g.koff[i], b = g.koff[i + 1];
  u32 op = g.op[i];
  u64 h = hash_mix(0x2545f4914f6cdd1dULL ^ ((u64)(b - a) << 32), op);
  for (u32 j = a; j < b; j++) {
    u32 k = g.kids[j], c = uf_find(g.parent, k);
    if (c != k) g.kids[j] = c;
    h = hash_mix(h, c);
  }
  u32 slot = (u32)h & g.hc_mask;
  u32 tag = hc_tag(g.hc_epoch, h);
  unsigned long long mine = ((unsigned long long)tag << 32) | i;
  u32 loser = TSAT_NONE, winner = TSAT_NONE;
  while (true) {
    unsigned long long e = ((volatile unsigned long long*)g.hc)[slot];
    if (!hc_live(g, e)) {
      if (atomicCAS(&g.hc[slot], e, mine) == e) break;
      continue;
    }
    if ((u32)(e >> 32) == tag && key_eq_canon(g, (u32)e, op, a, b - a)) {
      unsigned long long old = atomicMin(&g.hc[slot], mine);
      u32 o = (u32)old;
      loser = o > i ? o : i;
      winner = o > i ? i : o;
      break;
    }
    slot = (slot + 1) & g.hc_mask;
  }
  u32 link = TSAT_NONE;
  if (loser != TSAT_NONE) {
    g.flags[loser] &= ~NF_ALIVE;
    u32 x = winner, y = loser;
    while (true) {
      x = uf_find_ro(g.parent, x);
      y = uf_find_ro(g.parent, y);
      if (x == y) break;
      u32 lo = x < y ? x : y, hi = x < y ? y : x;
      if (atomicCAS(&g.parent[hi], hi, lo) == hi) {
        link = hi;
        break;
      }
    }
  }
  if (link != TSAT_NONE) atomicOr(&linkbits[link >> 5], 1u << (link & 31));
  return (loser != TSAT_NONE ? 1u : 0u) | (link != TSAT_NONE ? 2u : 0u);
}

// per-warp counter flush (one atomic per warp instead of one per event: a
// cascade round drops ~10^6 nodes, and atomics on one address serialise)
__device__ __forceinline__ void rb_flush(u32 drops, u32 links, RbCtl* ctl) {
  drops = __reduce_add_sync(0xffffffffu, drops);
  links = __reduce_add_sync(0xffffffffu, links);
  if ((threadIdx.x & 31) == 0) {
    if (drops) atomicAdd(&ctl->dropped, drops);
    if (links) atomicAdd(&ctl->nlinked, links);
  }
}

__global__ void k_rebuild_round(G g, u32 n, u32* linkbits, RbCtl* ctl) {
  u32 drops = 0, links = 0;
  GRID_STRIDE(i, n) {
    if (g.flags[i] & NF_ALIVE) {
      u32 r = rb_process(g, (u32)i, linkbits);
      drops += r & 1u;
      links += r >> 1;
    }
  }
  rb_flush(drops, links, ctl);
}

// Rebuild to fixpoint in one cooperative launch (no host round trip per
// round).  Every live node sits in the hashcons exactly once, under its
// stored children; a node needs work in a round only when one of its stored
// children is no longer a root (its class was linked since the node was last
// keyed).  So after an optional full first round (fresh epoch: forced
// rebuilds / table cleanup), each round (1) lists the live nodes with a
// non-root stored child, (2) replaces their old slots with tombstones (found
// by the stale key they were inserted under), (3) re-keys and re-inserts them
// exactly like a full round.  Nodes without a stale child keep their entries,
// which are current; a round that links nothing is the fixpoint.  The result
// equals a sequence of full rounds: same survivors (min id per final key),
// same partition, and the table holds exactly the live nodes under their
// canonical keys (plus tombstones, cleared by the next new epoch).

__device__ __forceinline__ void rb_tombstone(const G& g, u32 i, RbCtl* ctl) {
  u64 h = node_hash(g, i);  // the stored (stale) key the node was inserted under
  u32 slot = (u32)h & g.hc_mask, tag = hc_tag(g.hc_epoch, h);
  unsigned long long mine = ((unsigned long long)tag << 32) | i;
  while (true) {
    unsigned long long e = g.hc[slot];
    if (!hc_live(g, e)) {
      atomicAdd(&ctl->lost, 1u);
      return;
    }
    if (e == mine) {
      g.hc[slot] = hc_tomb(g.hc_epoch);
      return;
    }
    slot = (slot + 1) & g.hc_mask;
  }
}

__global__ void __launch_bounds__(256) k_rebuild_fix(G g, u32 n, int full, u32* dl, u32* linkbits, RbCtl* ctl) {
  cg::grid_group grid = cg::this_grid();
  __shared__ u32 sm_ko[8 * 129];
  __shared__ u8 sm_df[8 * 128];
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x, nth = (u64)gridDim.x * blockDim.x;
  if (tid == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ctl->t[0]));
  // a full first round (k_rebuild_round, launched before) left its links here
  u32 l0 = ((volatile RbCtl*)ctl)->nlinked;
  u32 r = full ? 1 : 0;
  if (full && l0 == 0) {
    if (tid == 0) {
      ctl->rounds = 1;
      g.cnt->live -= ctl->dropped;  // congruent members of one class: dropped, nothing linked
      g.cnt->dirty = 0;
    }
    return;
  }
  for (;; r++) {
    u32* cnt = &ctl->ndirty[r & 1];
    if (tid == 0) ctl->ndirty[(r + 1) & 1] = 0;  // the previous round's list (next used by round r + 1)
    // (1) live nodes with a non-root stored child.  A warp takes 128
    // consecutive nodes: their child offsets go to shared memory (4
    // coalesced loads), the combined child range is swept 128 slots per step
    // (4 independent coalesced loads + 4 independent parent gathers per
    // lane), and a stale slot flags its owner (binary search of the offsets)
    {
      const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
      u32* ko = sm_ko + wib * 129;
      u8* df = sm_df + wib * 128;
      const u64 wid = tid >> 5, nw = nth >> 5;
      for (u64 base = wid * 128; base < n; base += nw * 128) {
        const u32 cntn = (u32)((n - base) < 128 ? (n - base) : 128);
        u32 am = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const u32 li = q * 32 + lane, i = (u32)base + li;
          ko[li] = li < cntn ? g.koff[i] : 0u;
          if (li < cntn && (g.flags[i] & NF_ALIVE)) am |= 1u << q;
          df[li] = 0;
        }
        if (lane == 0) ko[128] = g.koff[base + cntn];
        __syncwarp();
        for (u32 li = cntn + lane; li < 128; li += 32) ko[li] = ko[128];
        __syncwarp();
        const u32 lo = ko[0], hi = ko[128];
        for (u32 c = lo; c < hi; c += 128) {
          u32 k[4], pp[4];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const u32 j = c + q * 32 + lane;
            k[q] = j < hi ? g.kids[j] : TSAT_NONE;
          }
#pragma unroll
          for (int q = 0; q < 4; q++) pp[q] = k[q] != TSAT_NONE ? g.parent[k[q]] : TSAT_NONE;
#pragma unroll
          for (int q = 0; q < 4; q++)
            if (pp[q] != k[q]) {
              const u32 j = c + q * 32 + lane;
              u32 l = 0, h2 = 128;  // last li with ko[li] <= j
              while (h2 - l > 1) {
                u32 mid = (l + h2) >> 1;
                if (ko[mid] <= j) l = mid;
                else h2 = mid;
              }
              df[l] = 1;
            }
        }
        __syncwarp();
        u32 dm[4], tot = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          dm[q] = __ballot_sync(0xffffffffu, ((am >> q) & 1u) && df[q * 32 + lane]);
          tot += __popc(dm[q]);
        }
        if (tot) {
          u32 wb = 0;
          if (lane == 0) wb = atomicAdd(cnt, tot);
          wb = __shfl_sync(0xffffffffu, wb, 0);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            if ((dm[q] >> lane) & 1u) dl[wb + __popc(dm[q] & ((1u << lane) - 1))] = (u32)base + q * 32 + lane;
            wb += __popc(dm[q]);
          }
        }
        __syncwarp();
      }
    }
    grid.sync();
    const u32 nd = ((volatile u32*)cnt)[0];
    if (nd == 0) break;
    // (2) tombstones for their stale entries
    for (u64 k = tid; k < nd; k += nth) rb_tombstone(g, dl[k], ctl);
    grid.sync();
    // (3) re-key + re-insert (drops / links like a full round)
    {
      u32 drops = 0, links = 0;
      for (u64 k = tid; k < nd; k += nth) {
        u32 rr = rb_process(g, dl[k], linkbits);
        drops += rr & 1u;
        links += rr >> 1;
      }
      rb_flush(drops, links, ctl);
    }
    if (tid == 0) {
      ctl->dirty_total += nd;
      ctl->tombs += nd;
    }
    grid.sync();
    const u32 l1 = ((volatile RbCtl*)ctl)->nlinked;
    if (l1 == l0) {
      r++;
      break;
    }
    l0 = l1;
  }
  if (tid == 0) {
    ctl->rounds = r;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ctl->t[1]));
    // counters updated here, so the host reads them back with the control
    // block (one sync per rebuild)
    g.cnt->live -= ctl->dropped;
    g.cnt->dirty = 0;
  }
  // every linked root's own analysis folds into its final root (set unions:
  // order free) under a per-root lock bit in its flags word; sources are
  // non-roots, so nobody writes them meanwhile
  const u32 nwords = (n + 31) >> 5;
  for (u64 w = tid; w < nwords; w += nth) {
    u32 bits = linkbits[w];
    if (!bits) continue;
    linkbits[w] = 0;  // left clear for the next rebuild
    if (!g.analysis) continue;
   while (bits) {
    const u32 src = (u32)w * 32 + (__ffs(bits) - 1);
    bits &= bits - 1;
    const u32 t = uf_find_ro(g.parent, src);    u32* word = (u32*)(g.flags + (t & ~3u));
    const u32 bit = NF_LOCK << (8 * (t & 3u));
    bool done = false;
    {
      // lock-free when the source adds nothing: a root's origin sets only
      // grow, so a source already contained stays contained
      Val cur;
      const int4* sp = (const int4*)(g.val + t);
      int4* dp = (int4*)&cur;
      for (int q = 0; q < (int)(sizeof(Val) / 16); q++) dp[q] = __ldcg(sp + q);
      const Val& o = g.val[src];
      done = val_same_data(cur, o) && !val_merge_grows(cur, o);
    }
    while (!done) {
      if (!(atomicOr(word, bit) & bit)) {
        __threadfence();
        Val acc;
        {  // L2 copy: another SM may have merged into t since this SM last saw it
          const int4* sp = (const int4*)(g.val + t);
          int4* dp = (int4*)&acc;
          for (int q = 0; q < (int)(sizeof(Val) / 16); q++) dp[q] = __ldcg(sp + q);
        }
        const Val& o = g.val[src];
        if (!val_same_data(acc, o)) dev_set_error(g.err, TSAT_ERR_MERGE, 4, t, src);
        else if (val_merge_into(acc, o) != AS_OK) dev_set_error(g.err, TSAT_ERR_CAPACITY, 5, t, src);
        else g.val[t] = acc;
        __threadfence();
        atomicAnd(word, ~bit);
        done = true;
      }
    }
   }
  }
  if (ctl->t[3]) {  // debug: time the merge phase
    grid.sync();
    if (tid == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ctl->t[2]));
  }
}

__global__ void k_link_targets(G g, const u32* linked, u32 m, u32* tgt) {
  GRID_STRIDE(i, m) tgt[i] = uf_find_ro(g.parent, linked[i]);
}

// one thread per merged group (sorted by target): fold analyses in
__global__ void k_merge_groups(G g, const u32* tgt, const u32* src, u32 m) {
  GRID_STRIDE(i, m) {
    if (i > 0 && tgt[i - 1] == tgt[i]) continue;
    u32 t = tgt[i];
    Val acc = g.val[t];
    for (u64 j = i; j < m && tgt[j] == t; j++) {
      const Val& o = g.val[src[j]];
      if (!val_same_data(acc, o)) {
        dev_set_error(g.err, TSAT_ERR_MERGE, 4, t, src[j]);
        break;
      }
      if (val_merge_into(acc, o) != AS_OK) {
        dev_set_error(g.err, TSAT_ERR_CAPACITY, 5, t, src[j]);
        break;
      }
    }
    g.val[t] = acc;
  }
}

void Engine::rebuild(bool full) {
  if (!h.dirty) return;
  u32 n = h.next_id;
  DevBuf<u32>& small = scratch_u32[5];
  DevBuf<u32>& dl = scratch_u32[6];
  // link bitmap (one bit per node id), kept clear between rebuilds by the
  // merge pass that consumes it
  if (rb_linkbits.cap < (u64)(n + 31) / 32 + 1) {
    rb_linkbits.ensure((u64)(n + 31) / 32 + 1);
    CUDA_OK(cudaMemsetAsync(rb_linkbits.p, 0, rb_linkbits.cap * sizeof(u32), s));
  }
  DevBuf<u32>& linked = rb_linkbits;
  dl.ensure(n + 1);
  small.ensure(sizeof(RbCtl) / 4 + 1);
  // tombstones accumulate until the next epoch: a full round (fresh epoch)
  // once live entries + tombstones could pass half the table
  static const bool always_full = getenv("TSAT_REBUILD_FULL") != nullptr;
  if (always_full || hc_tombs + 2ull * h.live > hc_cap / 2 + (u64)h.live) full = true;
  if (full) hc_new_epoch();
  static int coop = 0;
  if (!coop) {
    int per_sm = 0, nsm = 0, dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rebuild_fix, 256, 0));
    coop = std::max(1, per_sm) * nsm;
  }
  RbCtl hc_;
  {
    KTimer kt(*this, KG_REBUILD, 0.0, 1);
    CUDA_OK(cudaMemsetAsync(small.p, 0, sizeof(RbCtl), s));
    static const bool dbg_t = getenv("TSAT_DEBUG_REBUILD") != nullptr;
    if (dbg_t) CUDA_OK(cudaMemsetAsync((char*)small.p + offsetof(RbCtl, t) + 24, 1, 1, s));
    G gv = view();
    int fl = full ? 1 : 0;
    RbCtl* cp0 = (RbCtl*)small.p;
    // the full round streams every node: a plain (oversubscribed) grid keeps
    // more loads in flight than the co-resident cooperative grid
    if (full) k_rebuild_round<<<nblk(n), 256, 0, s>>>(gv, n, linked.p, cp0);
    RbCtl* cp = (RbCtl*)small.p;
    void* args[] = {&gv, &n, &fl, &dl.p, &linked.p, &cp};
    unsigned nb = (unsigned)std::min<u64>((u64)coop, std::max<u64>(1, ((u64)n + 255) / 256));
    CUDA_OK(cudaLaunchCooperativeKernel((const void*)k_rebuild_fix, nb, 256, args, 0, s));
  }
  CUDA_OK(cudaMemcpyAsync(&hc_, small.p, sizeof(RbCtl), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(&h, cnt.p, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  DevError he;
  CUDA_OK(cudaMemcpyAsync(&he, err.p, sizeof(he), cudaMemcpyDeviceToHost, s));
  sync();
  {
    // algorithmic bytes: a full round 60 N + 12 A; an
    // incremental round scans flags / offsets / stored children + their
    // parents (13 N + 8 A) and re-keys its dirty nodes (~60 + 12 arity + 16
    // for the tombstone probe each)
    const double avg_a = h.next_id ? (double)h.nkids / h.next_id : 0.0;
    const u32 inc_rounds = hc_.rounds - (full ? 1 : 0);
    kstat[KG_REBUILD].bytes += (full ? 60.0 * h.live + 12.0 * h.nkids : 0.0) +
                               inc_rounds * (13.0 * n + 8.0 * h.nkids) + hc_.dirty_total * (76.0 + 12.0 * avg_a);
    static const bool dbg = getenv("TSAT_DEBUG_REBUILD") != nullptr;
    if (dbg)
      fprintf(stderr, "rebuild: full %d rounds %u dirty %u dropped %u linked %u tombs %llu/%u live %u | rounds %.1f us merges %.1f us\n", (int)full,
              hc_.rounds, hc_.dirty_total, hc_.dropped, hc_.nlinked, (unsigned long long)(hc_tombs + hc_.tombs),
              hc_cap, h.live, (hc_.t[1] - hc_.t[0]) * 1e-3, hc_.t[2] ? (hc_.t[2] - hc_.t[1]) * 1e-3 : 0.0);
  }
  if (hc_.lost) throw TsatException(TSAT_ERR_STATE, "rebuild: hashcons entry of a live node not found");
  hc_tombs += hc_.tombs;
  rb_rounds_last = hc_.rounds;
  rb_dirty_last = hc_.dirty_total;
  uf_changed = false;
  snap.valid = false;
  raise_error(he);
}

// ---------------------------------------------------------------- snapshot CSR

__global__ void k_alive_flags(G g, u32 n, u32* fl) {
  GRID_STRIDE(i, n) fl[i] = (g.flags[i] & NF_ALIVE) ? 1u : 0u;
}

__global__ void k_compact_alive(G g, u32 n, const u32* pos, u32* ids, u32* cls, u32* opk) {
  GRID_STRIDE(i, n) {
    if (!(g.flags[i] & NF_ALIVE)) continue;
    u32 p = pos[i];
    ids[p] = (u32)i;
    cls[p] = uf_find_ro(g.parent, (u32)i);
    opk[p] = g.op[i];
  }
}

__global__ void k_gather_op(G g, const u32* ids, u32 m, u32* opk) {
  GRID_STRIDE(i, m) opk[i] = g.op[ids[i]];
}

__global__ void k_class_heads(const u32* scls, u32 m, u32* head) {
  GRID_STRIDE(i, m) head[i] = (i == 0 || scls[i] != scls[i - 1]) ? 1u : 0u;
}

__global__ void k_class_index(const u32* scls, const u32* headpos, u32 m, u32* cls_off, u32* cls_ids,
                              u32* cls_index) {
  GRID_STRIDE(i, m) {
    if (i == 0 || scls[i] != scls[i - 1]) {
      u32 d = headpos[i];
      cls_off[d] = (u32)i;
      cls_ids[d] = scls[i];
      cls_index[scls[i]] = d;
    }
  }
}

__global__ void k_set_u32(u32* p, u32 idx, u32 v) { p[idx] = v; }

// number of classes from the head flags / their scan; closes the class CSR
__global__ void k_close_cls_off(const u32* head, const u32* pos, u32 m, u32* cls_off, u32* ncls) {
  u32 c = m ? pos[m - 1] + head[m - 1] : 0u;
  cls_off[c] = m;
  *ncls = c;
}

// off[a] = first position of key >= a in a sorted key array (CSR offsets)
__global__ void k_lower_bounds(const u32* sorted, u32 m, u32 nkeys, u32* off) {
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

// dense class index of every member position (for member-parallel passes)
__global__ void k_member_class(const u32* head, const u32* pos, u32 m, u32* cls_of) {
  GRID_STRIDE(i, m) cls_of[i] = pos[i] + head[i] - 1;
}

void Engine::build_snapshot() {
  u32 n = h.next_id, m = h.live;
  KTimer kt(*this, KG_SNAPSHOT, 0.0, 5);
  DevBuf<u32>& fl = scratch_u32[1];
  DevBuf<u32>& pos = scratch_u32[2];
  DevBuf<u32>& ids = scratch_u32[3];
  DevBuf<u32>& cls = scratch_u32[4];
  DevBuf<u32>& opk = scratch_u32[5];
  DevBuf<u32>& tmp = scratch_u32[6];
  u32 na = (u32)h_atoms.size();
  fl.ensure(std::max(n, na) + 2);
  pos.ensure(std::max(n, na) + 2);
  ids.ensure(m + 1);
  cls.ensure(m + 1);
  opk.ensure(m + 1);
  tmp.ensure(m + 1);
  k_alive_flags<<<nblk(n), 256, 0, s>>>(view(), n, fl.p);
  dev_exclusive_scan_u32(*this, fl.p, pos.p, n);
  k_compact_alive<<<nblk(n), 256, 0, s>>>(view(), n, pos.p, ids.p, cls.p, opk.p);
  // class CSR: stable sort (class, id) -> members grouped, ascending
  snap.cls_nodes.ensure(m + 1);
  snap.cls_index.ensure(n + 1);
  CUDA_OK(cudaMemsetAsync(snap.cls_index.p, 0xFF, (size_t)(n + 1) * sizeof(u32), s));
  u32 nb = bits_for(n);
  dev_sort_pairs_u32(*this, cls.p, tmp.p, ids.p, snap.cls_nodes.p, m, nb);
  // tmp = sorted class ids
  k_class_heads<<<nblk(m), 256, 0, s>>>(tmp.p, m, fl.p);
  dev_exclusive_scan_u32(*this, fl.p, pos.p, m);
  // class count stays on the device until the single sync at the end
  // (buffers sized by the member count, an upper bound)
  snap.cls_off.ensure(m + 2);
  snap.cls_ids.ensure(m + 1);
  snap.d_ncls.ensure(2);
  k_class_index<<<nblk(m), 256, 0, s>>>(tmp.p, pos.p, m, snap.cls_off.p, snap.cls_ids.p, snap.cls_index.p);
  k_close_cls_off<<<1, 1, 0, s>>>(fl.p, pos.p, m, snap.cls_off.p, snap.d_ncls.p);
  snap.cls_of.ensure(m + 1);
  k_member_class<<<nblk(m), 256, 0, s>>>(fl.p, pos.p, m, snap.cls_of.p);
  // op CSR in (op, class, id) order: stable sort of the class-ordered members
  // by op atom, so e-matching emits each pattern's matches grouped by class
  snap.op_nodes.ensure(m + 1);
  snap.op_off.ensure(na + 1);
  k_gather_op<<<nblk(m), 256, 0, s>>>(view(), snap.cls_nodes.p, m, opk.p);
  dev_sort_pairs_u32(*this, opk.p, tmp.p, snap.cls_nodes.p, snap.op_nodes.p, m, bits_for(na));
  k_lower_bounds<<<nblk((u64)na + 1), 256, 0, s>>>(tmp.p, m, na, snap.op_off.p);
  snap.op_off_h.resize(na + 1);
  CUDA_OK(cudaMemcpyAsync(snap.op_off_h.data(), snap.op_off.p, (na + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
  u32 ncls = 0;
  CUDA_OK(cudaMemcpyAsync(&ncls, snap.d_ncls.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  snap.n_alloc = n;
  snap.ncls = ncls;
  snap.n_atoms = na;
  snap.valid = true;
  snap_id++;
}

// ---------------------------------------------------------------- download / dump

// selected nodes only (reconstruct): op, arity prefix, canonical children
__global__ void k_sub_arity(G g, const u32* ids, u32 n, u32* op_out, u32* deg) {
  GRID_STRIDE(i, n) {
    u32 x = ids[i];
    op_out[i] = g.op[x];
    deg[i] = g.koff[x + 1] - g.koff[x];
  }
}

__global__ void k_sub_kids(G g, const u32* ids, u32 n, const u32* off, u32* kids_out) {
  GRID_STRIDE(i, n) {
    u32 x = ids[i], a = g.koff[x], b = g.koff[x + 1], o = off[i];
    for (u32 j = a; j < b; j++) kids_out[o++] = uf_find_ro(g.parent, g.kids[j]);
  }
}

__global__ void k_find_batch(G g, const u32* ids, u32 n, u32* out) {
  GRID_STRIDE(i, n) out[i] = uf_find_ro(g.parent, ids[i]);
}

void Engine::find_batch(u32 n, const u32* ids, u32* out) {
  for (u32 i = 0; i < n; i++)
    if (ids[i] >= h.next_id) throw TsatException(TSAT_ERR_ARG, "node id out of range");
  DevBuf<u32>& di = scratch_u32[0];
  DevBuf<u32>& dout = scratch_u32[1];
  di.ensure(n + 1);
  dout.ensure(n + 1);
  if (!n) return;
  CUDA_OK(cudaMemcpyAsync(di.p, ids, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  k_find_batch<<<nblk(n), 256, 0, s>>>(view(), di.p, n, dout.p);
  CUDA_OK(cudaMemcpyAsync(out, dout.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
}

void Engine::download_nodes(u32 n, const u32* ids, u32* hop, u32* hoff, u32* hkids, u64 kids_cap, u64* nkids) {
  for (u32 i = 0; i < n; i++)
    if (ids[i] >= h.next_id) throw TsatException(TSAT_ERR_ARG, "node id out of range");
  DevBuf<u32>& di = scratch_u32[0];
  DevBuf<u32>& dop = scratch_u32[1];
  DevBuf<u32>& ddeg = scratch_u32[2];
  DevBuf<u32>& doff = scratch_u32[3];
  DevBuf<u32>& dk = scratch_u32[4];
  di.ensure(n + 1);
  dop.ensure(n + 1);
  ddeg.ensure(n + 1);
  doff.ensure(n + 1);
  if (n) CUDA_OK(cudaMemcpyAsync(di.p, ids, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  k_sub_arity<<<nblk(n), 256, 0, s>>>(view(), di.p, n, dop.p, ddeg.p);
  CUDA_OK(cudaMemsetAsync(ddeg.p + n, 0, sizeof(u32), s));
  dev_exclusive_scan_u32(*this, ddeg.p, doff.p, n + 1);
  CUDA_OK(cudaMemcpyAsync(hoff, doff.p, (n + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
  if (n) CUDA_OK(cudaMemcpyAsync(hop, dop.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
  *nkids = hoff[n];
  if (hoff[n] > kids_cap) return;  // caller retries with a larger buffer
  dk.ensure((u64)hoff[n] + 1);
  k_sub_kids<<<nblk(n), 256, 0, s>>>(view(), di.p, n, doff.p, dk.p);
  if (hoff[n]) CUDA_OK(cudaMemcpyAsync(hkids, dk.p, (u64)hoff[n] * sizeof(u32), cudaMemcpyDeviceToHost, s));
  sync();
}

void Engine::download(u32* hop, u32* hkoff, u32* hkids, u32* hcls, u8* hflags) {
  u32 n = h.next_id;
  std::vector<u32> par(n);
  if (n) {
    CUDA_OK(cudaMemcpyAsync(hop, op.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(hkoff, koff.p, (n + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    if (h.nkids) CUDA_OK(cudaMemcpyAsync(hkids, kids.p, h.nkids * sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(par.data(), parent.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(hflags, flags.p, n, cudaMemcpyDeviceToHost, s));
  }
  sync();
  for (u32 i = 0; i < n; i++) {
    u32 r = i;
    while (par[r] != r) r = par[r];
    u32 x = i;
    while (par[x] != r) {
      u32 nx = par[x];
      par[x] = r;
      x = nx;
    }
    hcls[i] = r;
  }
}

static void dims_str(std::ostringstream& os, const i64* d, int r) {
  for (int i = 0; i < r; i++) {
    if (i) os << "x";
    os << d[i];
  }
}

static std::string val_to_string(const Val& v, const std::vector<std::string>& names) {
  std::ostringstream os;
  switch (v.kind) {
    case VK_N: os << "N:" << v.iv; break;
    case VK_S: os << "S:" << names[v.iv]; break;
    case VK_T: os << "T:"; dims_str(os, v.d0, v.r0); break;
    case VK_TT:
      os << "TT:";
      dims_str(os, v.d0, v.r0);
      os << "|";
      dims_str(os, v.d1, v.r1);
      break;
    default: os << "?";
  }
  return os.str();
}

std::string Engine::value_str(u32 c) {
  if (!analysis || c >= h.next_id) return "";
  Val v;
  CUDA_OK(cudaMemcpyAsync(&v, val.p + c, sizeof(Val), cudaMemcpyDeviceToHost, s));
  sync();
  return val_to_string(v, atom_names);
}

std::string Engine::dump_text() {
  u32 n = h.next_id;
  std::vector<u32> hop(n), hkoff(n + 1), hkids(h.nkids + 1), hcls(n);
  std::vector<u8> hfl(n);
  download(hop.data(), hkoff.data(), hkids.data(), hcls.data(), hfl.data());
  std::vector<Val> hv;
  if (analysis && n) {
    hv.resize(n);
    CUDA_OK(cudaMemcpyAsync(hv.data(), val.p, n * sizeof(Val), cudaMemcpyDeviceToHost, s));
    sync();
  }
  // classes = roots of alive nodes; members ascending
  std::vector<u32> first(n, TSAT_NONE), nxt(n, TSAT_NONE), last(n, TSAT_NONE);
  u32 nclasses = 0, nnodes = 0;
  std::vector<u32> order;
  for (u32 i = 0; i < n; i++) {
    if (!(hfl[i] & NF_ALIVE)) continue;
    nnodes++;
    u32 c = hcls[i];
    if (first[c] == TSAT_NONE) {
      first[c] = i;
      nclasses++;
      order.push_back(c);
    } else {
      nxt[last[c]] = i;
    }
    last[c] = i;
  }
  std::sort(order.begin(), order.end());
  std::ostringstream os;
  os << "egraph nodes=" << nnodes << " classes=" << nclasses << " root=";
  if (root == TSAT_NONE) os << "-";
  else os << "c" << hcls[root];
  os << "\n";
  for (u32 c : order) {
    os << "c" << c;
    if (analysis) os << " [" << val_to_string(hv[c], atom_names) << "]";
    os << ":";
    for (u32 i = first[c]; i != TSAT_NONE; i = nxt[i]) {
      os << " n" << i << "=" << atom_names[hop[i]] << "(";
      for (u32 j = hkoff[i]; j < hkoff[i + 1]; j++) {
        if (j > hkoff[i]) os << ",";
        os << "c" << hcls[hkids[j]];
      }
      os << ")";
    }
    os << "\n";
  }
  return os.str();
}

// ---------------------------------------------------------------- API helpers
// (drop-in pieces of the reference API the explore loop does not use itself)

// EGraph.clone (egraph.py:351-364): device-to-device copy of the e-graph state
// of ``o`` (same device).  Atoms are re-sent by the caller in the same order,
// so atom ids, analyses and interned cut trees stay valid as copied.
void Engine::copy_state_from(Engine& o) {
  if (o.device != device) throw TsatException(TSAT_ERR_ARG, "clone across devices");
  o.sync();
  sync();
  analysis = o.analysis;
  h = o.h;
  h.nkids = o.h.nkids;
  u64 n = o.h.next_id, nk = o.h.nkids;
  if (cap_nodes < n + 1 || cap_kids < nk + 1) {
    Counters keep = h;
    memset(&h, 0, sizeof(h));  // nothing of the old content needs preserving
    ensure_nodes(n + 1, nk + 1);
    h = keep;
  }
  if (hc_cap != o.hc_cap) {
    hc.alloc(o.hc_cap);
    hc_cap = o.hc_cap;
  }
  hc_epoch = o.hc_epoch;
  hc_tombs = o.hc_tombs;
  if (n) {
    CUDA_OK(cudaMemcpyAsync(op.p, o.op.p, n * sizeof(u32), cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(parent.p, o.parent.p, n * sizeof(u32), cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(flags.p, o.flags.p, n * sizeof(u8), cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(val.p, o.val.p, n * sizeof(Val), cudaMemcpyDeviceToDevice, s));
  }
  CUDA_OK(cudaMemcpyAsync(koff.p, o.koff.p, (n + 1) * sizeof(u32), cudaMemcpyDeviceToDevice, s));
  if (nk) CUDA_OK(cudaMemcpyAsync(kids.p, o.kids.p, nk * sizeof(u32), cudaMemcpyDeviceToDevice, s));
  if (hc_cap)
    CUDA_OK(cudaMemcpyAsync(hc.p, o.hc.p, (size_t)hc_cap * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  if (tree_cap != o.tree_cap) {
    trees.alloc(o.tree_cap);
    tree_cap = o.tree_cap;
  }
  if (tree_hc_cap != o.tree_hc_cap) {
    tree_hc.alloc(o.tree_hc_cap);
    tree_hc_cap = o.tree_hc_cap;
  }
  CUDA_OK(cudaMemcpyAsync(trees.p, o.trees.p, (size_t)tree_cap * sizeof(Tree), cudaMemcpyDeviceToDevice, s));
  CUDA_OK(cudaMemcpyAsync(tree_hc.p, o.tree_hc.p, (size_t)tree_hc_cap * sizeof(u32), cudaMemcpyDeviceToDevice, s));
  CUDA_OK(cudaMemcpyAsync(tree_count.p, o.tree_count.p, sizeof(u32), cudaMemcpyDeviceToDevice, s));
  root = o.root;
  uf_changed = o.uf_changed;
  push_counters();
  snap.valid = false;
  reach.valid = false;
  filter_id++;
  costs_valid_for = TSAT_NONE;
  sync();
}

// eval_pattern (rules.py:126-138) of each term under its environment slice,
// on the device analysis; status = ana status (0 ok)
__global__ void k_eval_terms(G g, const Instr* prog, const int32_t* len, int nterm, const u32* env, const u32* env_off,
                             Val* out, int32_t* status) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nterm) return;
  u32 off = 0;
  for (int k = 0; k < t; k++) off += (u32)len[k];
  Val scratch[MAX_STACK];
  const Val* res = nullptr;
  int st = eval_target(g, prog + off, len[t], env + env_off[t], scratch, res);
  status[t] = st;
  if (st == AS_OK) out[t] = *res;
}

void Engine::eval_terms(int ninstr, const Instr* prog, int nterm, const int32_t* term_len, int nenv, const u32* env,
                        const u32* env_off, void* out_vals, int32_t* status) {
  if (!analysis) throw TsatException(TSAT_ERR_STATE, "eval_pattern needs the tensor analysis");
  for (int i = 0; i < ninstr; i++)
    if (prog[i].kind == I_APP && prog[i].arg > 8) throw TsatException(TSAT_ERR_ARG, "arity > 8 not supported");
  DevBuf<Instr>& dp = sc.a_prog;
  dp.ensure(ninstr + 1);
  DevBuf<int32_t>& dl = sc.a_len;
  dl.ensure(2 * (u64)nterm + 1);
  DevBuf<u32>& de = sc.a_env;
  de.ensure(nenv + (u64)nterm + 1);
  DevBuf<Val>& dv = sc.a_val;
  dv.ensure(nterm + 1);
  CUDA_OK(cudaMemcpyAsync(dp.p, prog, ninstr * sizeof(Instr), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpyAsync(dl.p, term_len, nterm * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (nenv) CUDA_OK(cudaMemcpyAsync(de.p, env, nenv * sizeof(u32), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpyAsync(de.p + nenv, env_off, nterm * sizeof(u32), cudaMemcpyHostToDevice, s));
  int32_t* dst = dl.p + nterm;
  k_eval_terms<<<(nterm + 127) / 128, 128, 0, s>>>(view(), dp.p, dl.p, nterm, de.p, de.p + nenv, dv.p, dst);
  CUDA_OK(cudaMemcpyAsync(out_vals, dv.p, nterm * sizeof(Val), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(status, dst, nterm * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync();
  check_error();
}
