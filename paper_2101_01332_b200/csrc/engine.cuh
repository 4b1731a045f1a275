// Host-side engine object behind one C-ABI handle (include/tsat.h).
#pragma once
#include <chrono>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "egraph.cuh"

struct TsatException : public std::runtime_error {
  int code;
  TsatException(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Caching device allocator behind every DevBuf.  Blocks are power-of-two
// sized and recycled instead of cudaFree'd: cudaMalloc / cudaFree cost
// milliseconds and cudaFree synchronises the whole device, which made run
// times erratic whenever a fresh engine or a growing buffer allocated inside
// a timed phase.  A block is tagged with the stream of the engine that
// released it (thread-local "current stream", set at every C-ABI entry);
// reuse under a different stream first synchronises the tagged stream.
extern unsigned long long g_dev_allocs, g_dev_alloc_bytes, g_engines;  // diagnostics (tsat_debug_info)
void* dev_cache_get(size_t bytes);
double hc_load();
inline double now_s() {  // host monotonic clock (s): time limits
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
  // hashcons load factor over allocated ids (TSAT_HC_LOAD, default 0.5)
void dev_cache_put(void* p, size_t bytes);
void dev_cache_forget_stream(cudaStream_t s);  // stream about to be destroyed (already synced)
extern thread_local cudaStream_t tl_stream;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;  // owning: moves only
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      cap = o.cap;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  void alloc(size_t n) {
    release();
    if (n) p = (T*)dev_cache_get(n * sizeof(T));
    cap = n;
  }
  // grow to at least n elements, preserving the first ``keep`` elements
  void grow(size_t n, size_t keep, cudaStream_t s) {
    if (n <= cap) return;
    size_t nc = cap ? cap : 16;
    while (nc < n) nc *= 2;
    T* q = (T*)dev_cache_get(nc * sizeof(T));
    if (keep && p) CUDA_OK(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    release();
    p = q;
    cap = nc;
  }
  void ensure(size_t n) {  // no preservation
    if (n > cap) {
      size_t nc = cap ? cap : 16;
      while (nc < n) nc *= 2;
      alloc(nc);
    }
  }
  void release() {
    if (p) dev_cache_put(p, cap * sizeof(T));
    p = nullptr;
    cap = 0;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
  }
  ~DevBuf() { release(); }
};

// pattern app node (pre-order); child[j] >= 0 -> app index, < 0 -> var -(slot+1)
struct PatApp {
  u32 atom;
  int32_t nargs;
  int32_t child[8];
};

// target instruction (post-order); I_VAR pushes env[arg], I_APP applies atom
enum InstrKind : int32_t { I_VAR = 0, I_APP = 1 };
struct Instr {
  int32_t kind;
  int32_t arg;  // var slot (I_VAR) or nargs (I_APP)
  u32 atom;
  int32_t depth;  // term depth of the produced request (I_APP), 1 = leaf
};

#define MAX_SRC 4
#define MAX_PAT_APPS 8
#define MAX_VARS 16
#define MAX_STACK 16

struct HPattern {
  std::vector<PatApp> apps;
  int nvars = 0;
  std::vector<int> order;  // binding position k -> canonical var index (name-sorted)
};

struct HRule {
  std::string name;
  int nsrc = 0, nslots = 0;
  int src_pat[MAX_SRC];
  int bind_slot[MAX_SRC][MAX_VARS];  // binding position -> rule slot
  int src_nb[MAX_SRC];
  std::vector<std::vector<Instr>> targets;
  std::vector<std::vector<int>> leaves;  // per target: rule slots of its variables
  bool same_canon = false;
  int max_req = 0;  // requests (App nodes) over all targets
};

// matches of one canonical pattern: n rows of (eclass, bindings[nb])
struct MatchSet {
  u32 n = 0;
  int nb = 0;
  DevBuf<u32> cls;
  DevBuf<u32> bind;  // row-major n x nb
};

struct RuleStatsH {
  i64 found = 0, applied = 0, applied_noop = 0, skipped_self = 0, skipped_compat = 0,
      skipped_shape = 0, skipped_cycle = 0;
};

// device-side per-run statistics accumulated by the explore kernels
struct DevStats {
  unsigned long long found, applied, applied_noop, skipped_self, skipped_compat, skipped_shape,
      skipped_cycle;
  unsigned long long prefilter_checks, prefilter_rejects;
  u32 changed;     // any applied combo this iteration
  u32 stop;        // 1 = node limit hit
  u32 overshoot;
  u32 resume_set;  // capacity stop: resume position valid
  unsigned long long resume_pos;
  u32 vpend;       // vanilla: combo at resume_pos awaits its apply-on-checkpoint check
  u32 nrej;        // entries written to RuleDev::rej_log
  u32 timeout;     // the device deadline passed before the next combo
};

struct Snapshot {
  u32 n_alloc = 0;  // next_id when taken
  u32 ncls = 0;
  u32 n_atoms = 0;  // op CSR is sized for this many atoms
  DevBuf<u32> cls_index;  // node id -> dense class index (TSAT_NONE if not a class)
  DevBuf<u32> cls_ids;    // dense -> class id
  DevBuf<u32> cls_off;    // dense -> member range
  DevBuf<u32> cls_nodes;  // members (alive nodes), ascending per class
  DevBuf<u32> cls_of;     // dense class of each member position
  DevBuf<u32> op_off;     // atom -> range in op_nodes
  DevBuf<u32> op_nodes;   // alive nodes in (op, class, id) order
  std::vector<u32> op_off_h;  // host copy of op_off
  DevBuf<u32> d_ncls;         // class count, read back with op_off_h
  bool valid = false;
};

u64 default_reach_budget();

struct Reach {  // efficient pre-filter over a snapshot (rulesdev.cuh ReachDev)
  u32 n = 0, words = 0;
  int mode = 0;            // 0 descendants bitset, 1 peel levels + pruned search
  DevBuf<u32> bits;
  DevBuf<u32> visit, stack, epoch;
  bool valid = false;
  u64 budget = 0;  // bitset bytes allowed before mode 1 (tsat_set_reach_budget); default: always mode 1
};

struct ExploreLimitsC {
  i64 n_max, k_max, k_multi;
  double time_limit_s;  // < 0: none
};

struct ExploreReportC {
  i64 iterations;
  int stop_reason;  // 0 iter-limit, 1 saturated, 2 node-limit, 3 timeout
  i64 prefilter_checks, prefilter_rejects, postprocess_filtered, node_limit_overshoot, filter_size;
  double time_s;
};

// per kernel-group device timing + algorithmic bytes (roofline reporting)
enum KGroup { KG_REBUILD = 0, KG_EMATCH, KG_APPLY_SEQ, KG_APPLY_WAVE, KG_REACH, KG_CYCLES, KG_COSTS, KG_GREEDY, KG_SNAPSHOT, KG_COUNT };
struct KStat {
  double ms = 0.0;
  double bytes = 0.0;
  unsigned long long launches = 0;
};

struct Engine;
struct KTimer {  // records CUDA events on the engine stream around a kernel group
  Engine& e;
  int g;
  double bytes;
  unsigned long long launches;
  cudaEvent_t a, b;
  KTimer(Engine& e_, int g_, double bytes_, unsigned long long launches_);
  ~KTimer();
};

// persistent scratch buffers (grown on demand, never freed inside a run)
struct Scratch {
  // e-matching
  DevBuf<u32> m_heavy;
  DevBuf<u32> c_skey, c_sval, c_skey2;  // deterministic level order (sharded runs)
  DevBuf<u32> m_rc, m_rb, m_cnt, m_perm, m_perm2, m_key, m_key2, m_fl, m_pos;
  DevBuf<u32> m_bnd, m_big, m_head, m_bpos, m_L, m_bh, m_gex, m_bperm, m_bperm2, m_bkey, m_bkey2;
  // sharding (shard.cu)
  DevBuf<u32> sh_rng, sh_cnt, sh_pack, sh_recv;
  DevBuf<unsigned char> sh_segs;
  // class graph / cycles / reach
  DevBuf<u32> cg_eoff, cg_edst, cg_enode, cg_roff, cg_rsrc, cg_outdeg, cg_level, cg_esrc, cg_sdst, cg_moff, cg_mdeg;
  DevBuf<u32> c_heavy, c_mark32, c_fa, c_fb, c_order, c_depth, c_path, c_cycn, c_cyco, c_res, c_rest, c_lvloff;
  DevBuf<u32> c_odeg, c_oeoff, c_oedst, c_obnd, c_batch;  // level-ordered class edges (staged closure)
  DevBuf<u32> v_rej_w;  // wave-path reject log (on_reject)
  DevBuf<u8> c_mark, c_color;
  DevBuf<unsigned char> c_stack;
  // greedy / costs
  DevBuf<double> g_c0, g_c1, g_upl, k_dv, g_rinfo;
  DevBuf<u32> g_n0, g_n1, g_flag, g_mark, g_fa, g_fb, g_oc, g_on, k_slots, g_eoff, g_edst, g_cnt, k_miss;
  DevBuf<char> k_keyout;
  DevBuf<char> k_keys;
  DevBuf<u32> gq_batch;
  DevBuf<u32> gq_lvm, gq_cnt, gq_k, gq_node, gq_deg, gq_eoff, gq_edst, gq_lb, gq_head, gq_slot, gq_big;
  DevBuf<double> gq_pack, gq_recv;  // sharded wide levels: {best cost, node} records
  DevBuf<double> gq_cost, gq_tot;
  DevBuf<i64> k_off;
  // vanilla checkpoint (explore.cu run_rule_vanilla)
  DevBuf<u32> v_parent, v_rej, v_tree_hc;
  DevBuf<Val> v_val;
  DevBuf<unsigned long long> v_hc;
  // ILP model skeleton (ilp.cu)
  DevBuf<u32> il_mark, il_queue, il_f, il_scan, il_pos, il_classes, il_sel, il_soff, il_nodes, il_tmp, il_tmp2;
  DevBuf<u32> il_loff, il_lcnt, il_live, il_pcnt, il_poff, il_pchild;
  // api
  DevBuf<Instr> a_prog;
  DevBuf<int32_t> a_len;
  DevBuf<u32> a_env, a_out, a_ids;
  DevBuf<Val> a_val;
};

struct WaveBufs;

struct Engine {
  int device = 0;
  Scratch sc;
  WaveBufs* wave = nullptr;
  cudaStream_t s = nullptr;
  bool analysis = false;
  std::string last_error;

  // atoms
  std::vector<AtomInfo> h_atoms;
  std::vector<std::string> atom_names;
  DevBuf<AtomInfo> atoms;
  DevBuf<char> d_names;
  DevBuf<u32> d_name_off;
  DevBuf<double> d_costs;  // c_i by node id from the last costs() call
  u32 costs_valid_for = TSAT_NONE;  // next_id when computed

  // node table
  DevBuf<u32> op, koff, kids, parent;
  DevBuf<u8> flags;
  DevBuf<Val> val;
  u32 cap_nodes = 0, cap_kids = 0;
  DevBuf<unsigned long long> hc;
  u32 hc_cap = 0;
  u64 hc_tombs = 0;
  u32 rb_rounds_last = 0, rb_dirty_last = 0;
  DevBuf<u32> rb_linkbits;  // rebuild: roots linked by the current rebuild (bitmap, zero between rebuilds)  // last rebuild: rounds, nodes re-keyed by incremental rounds  // tombstones left in the current epoch by incremental rebuild rounds
  u32 hc_epoch = 1;
  void hc_new_epoch();

  // cut trees
  DevBuf<Tree> trees;
  DevBuf<u32> tree_hc;
  DevBuf<u32> tree_count;
  u32 tree_cap = 0, tree_hc_cap = 0;

  DevBuf<Counters> cnt;
  Counters h{};
  DevBuf<DevError> err;
  u32 root = TSAT_NONE;
  // a union may have happened since the last rebuild (host-side, conservative;
  // false = every stored child id is a class id: e-matching skips finds)
  bool uf_changed = false;

  // rules
  std::vector<HPattern> patterns;
  std::vector<HRule> rules;
  u64 rules_gen = 0;  // bumped by load_rules (wave templates are cached per generation)
  std::vector<MatchSet> matches;  // per pattern, current iteration
  DevBuf<Instr> d_instr;
  DevBuf<int> d_leaf;

  Snapshot snap;
  u32 cg_n = 0, cg_ne = 0;  // current class graph (cycles.cu)
  // level peel of the snapshot class graph (live, unfiltered edges), shared by
  // the cycle check, the next iteration's descendants map and greedy
  u64 snap_id = 0, filter_id = 0, lv_snap = ~0ull, lv_filter = ~0ull;
  std::vector<u32> lv_off;
  u32 lv_n = 0, lv_trimmed = 0;
  void ensure_levels();
  void reset(bool analysis_);
  Reach reach;
  DevBuf<u8> temp;  // cub scratch
  // overlap stream: the next iteration's e-matching runs speculatively next to
  // the (single-CTA, latency-bound) level peel of the cycle check
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_ov = nullptr;  // main-stream point (post-iteration snapshot) the overlap work waits for
  DevBuf<u8> temp2;
  std::function<void()> overlap_hook;  // run once by the level peel right after its launch
  bool spec_ematch = false;            // the next iteration's e-matching is already done
  bool levels_cached() const { return snap.valid && lv_snap == snap_id && lv_filter == filter_id; }
  void run_overlap_hook();
  DevBuf<u32> scratch_u32[8];
  DevBuf<DevStats> dstats;

  // per-rule stats of the last saturate call
  std::vector<RuleStatsH> rstats;
  std::vector<i64> enodes_per_iter, alloc_per_iter, eclasses_per_iter;
  ExploreReportC report{};
  std::vector<double> phase_ms = std::vector<double>(32, 0.0);
  unsigned long long nlaunch = 0;  // kernels of ours launched (not CUB)
  unsigned long long nsync = 0;    // host waits on the stream (Engine::sync)
  KStat kstat[KG_COUNT];
  // kernel-group timers: event pairs resolved lazily (no host sync per group)
  struct PendingTimer {
    cudaEvent_t a, b;
    int g;
  };
  std::vector<cudaEvent_t> ev_free;
  std::vector<PendingTimer> kt_pending;
  cudaEvent_t ev_get();
  void kt_resolve(bool block);

  Engine(int dev);
  ~Engine();

  G view();
  void pull_counters(const char* sf = __builtin_FILE(), int sl = __builtin_LINE());
  void push_counters();
  void check_error(const char* sf = __builtin_FILE(), int sl = __builtin_LINE());
  void raise_error(const DevError& he);
  void sync(const char* sf = __builtin_FILE(), int sl = __builtin_LINE());
  std::map<std::string, long> sync_sites;  // TSAT_DEBUG_SYNCS: host syncs per call site
  void ensure_nodes(u64 extra_nodes, u64 extra_kids);
  void rehash(u32 new_cap);

  // construction / generic API
  void set_atoms(int n, const int32_t* kind, const i64* ival, const int32_t* opcode,
                 const int32_t* ndims, const i64* dims, const int32_t* nident, const i64* idims,
                 const char* names_blob, const i64* name_off);
  void load_initial(u32 n, const u32* op, const u32* koff, const u32* kids, u32 root);
  void add_terms(int ninstr, const Instr* prog, int nterm, const int32_t* term_len, int nenv,
                 const u32* env, u32* out_cls);
  u32 union_pair(u32 a, u32 b);
  void rebuild(bool full = false);
  void set_filter(int n, const u32* ids, int on);
  std::vector<u32> get_filter();
  u32 find(u32 x);
  u64 root_ver = ~0ull;
  u32 root_cls_cache = TSAT_NONE;
  u32 root_class() {
    // snapshot id changes whenever the union-find can have changed
    if (!snap.valid) build_snapshot();
    if (root_ver != snap_id) {
      root_cls_cache = find(root);
      root_ver = snap_id;
    }
    return root_cls_cache;
  }

  // snapshot + matching
  void build_snapshot();
  DevBuf<u32> em_pool;  // e-matching semi-join bitmaps (match.cu)
  void ematch_batch(const std::vector<int>& pids);

  // multi-GPU e-matching shards (shard.cu)
  int shard_rank = 0, shard_world = 1;
  void* comm = nullptr;  // ncclComm_t
  // host transport (tsat_shard_setup_host): all-gather of host buffers by the
  // caller (e.g. torch.distributed / gloo); used when no NCCL communicator
  int32_t (*host_ag)(void*, const void*, void*, uint64_t) = nullptr;
  void* host_ctx = nullptr;
  std::vector<unsigned char> ag_send, ag_recv;
  bool shard_exchange() const { return comm != nullptr || host_ag != nullptr; }
  void shard_allgather(const void* dsend, void* drecv, size_t bytes);  // device buffers, rank order
  void shard_setup(int rank, int world, const void* nccl_id);
  // API helpers (core.cu / cycles.cu)
  void copy_state_from(Engine& o);
  void eval_terms(int ninstr, const Instr* prog, int nterm, const int32_t* term_len, int nenv, const u32* env,
                  const u32* env_off, void* out_vals, int32_t* status);
  void class_graph_download(u32* cls, u32* eoff, u32* edst, u32* sizes);
  void descendants_download(u32* cls, u32* bits, u64 cap_words, u32* sizes);
  void shard_teardown();
  void shard_candidate_ranges(std::vector<u32>& rng);
  void shard_gather_matches(const std::vector<int>& pids);
  void shard_allgather_bytes(const void* send, void* recv, size_t bytes);
  void load_rules(int n, const i64* blob);

  // cycles
  void build_reach();
  i64 break_all_cycles(bool precheck_only, std::vector<std::vector<u32>>* cycles_out);

  // exploration
  bool seq_changed = false, seq_stop = false;
  bool seq_timeout = false;      // vanilla: deadline passed between combos
  double apply_deadline = -1.0;  // saturate's deadline (now_s clock), < 0: none
  unsigned long long dev_deadline_ns = 0;  // the same deadline on the device clock (%globaltimer)
  void set_device_deadline(double deadline_s);
  bool force_seq = false;  // debug: exact sequential path only
  std::vector<std::string> rule_names;
  bool wave_path(int ri, int filter_mode) const;
  void apply_rule(int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long P);
  void saturate(const ExploreLimitsC& lim, int filter_mode, int allow_self, const int* active_rule_mask,
                int n_active);
  void run_rule_seq(int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long p0,
                    unsigned long long p1);
  void run_rule_vanilla(int ri, int allow_self, i64 n_max, unsigned long long P);
  // on_reject support: rejected combos of the last saturate, flattened as
  // [rule, nsrc, (eclass, nb, bindings[nb]) x nsrc] (snapshot match rows)
  bool record_rejects = false;
  bool defer_wave_stats = false;
  u32* pin_small = nullptr;  // pinned host words for asynchronous read-backs  // saturate: wave rules' statistics read once per iteration
  std::vector<unsigned long long>* rej_pending = nullptr;  // exact-path rejects inside a wave rule
  std::vector<u32> rejects;
  void record_reject(int ri, unsigned long long p);

  // extraction
  void costs(int mode, int strict, int ntab, const char* keys, const i64* key_off, const double* vals,
             double* out);
  double greedy(const double* cost_by_node, u32* sel_cls, u32* sel_node, u32* nsel, i64* rounds);
  void costs_gather(u32 n, const u32* ids, double* out);

  // ILP model skeleton (ilp.cu): sizes = {classes, x nodes, live members, pick rows}
  u32 il_sizes[4] = {0, 0, 0, 0};
  void ilp_build(u32* sizes);
  void ilp_download(u32* classes, u32* nodes, u32* live_off, u32* live, u32* pick_off, u32* pick_child);

  // download
  void download(u32* op, u32* koff, u32* kids, u32* cls, u8* flags);
  void download_nodes(u32 n, const u32* ids, u32* op, u32* off, u32* kids, u64 kids_cap, u64* nkids);
  void find_batch(u32 n, const u32* ids, u32* out);
  std::string dump_text();
  std::string value_str(u32 cls);
};

// cub helpers (core.cu)
void dev_exclusive_scan_u32(Engine& e, const u32* in, u32* out, u32 n);
void dev_sort_pairs_u32(Engine& e, u32* keys_in, u32* keys_out, u32* vals_in, u32* vals_out, u32 n,
                        int end_bit);
u32 bits_for(u32 maxval);
void shard_range(u64 n_alloc, int rank, int world, u32& lo, u32& hi);
void nccl_unique_id(void* out);
