// extern "C" boundary of libtsat (declared in include/tsat.h).
#include <cstring>

#include "../../include/tsat.h"
#include "engine.cuh"

struct tsat_engine {
  Engine* e;
  std::string err;
};

#define GUARD(h, ...)                                   \
  do {                                                  \
    if (!(h) || !(h)->e) return TSAT_ERR_ARG;           \
    tl_stream = (h)->e->s;                              \
    try {                                               \
      __VA_ARGS__;                                      \
      return TSAT_OK;                                   \
    } catch (TsatException & ex) {                      \
      (h)->err = ex.what();                             \
      return ex.code;                                   \
    } catch (std::exception & ex) {                     \
      (h)->err = ex.what();                             \
      return TSAT_ERR_STATE;                            \
    }                                                   \
  } while (0)

extern "C" {

// Engines are pooled: creating one allocates every device table, so a
// destroyed handle's engine is reset and kept for the next tsat_create.
static std::vector<Engine*>& engine_pool() {
  static std::vector<Engine*> p;
  return p;
}

int tsat_create(int device, int analysis, tsat_engine** out) {
  if (!out) return TSAT_ERR_ARG;
  *out = nullptr;
  try {
    tsat_engine* h = new tsat_engine();
    auto& pool = engine_pool();
    for (size_t i = 0; i < pool.size(); i++)
      if (pool[i]->device == device) {
        h->e = pool[i];
        pool.erase(pool.begin() + i);
        break;
      }
    if (!h->e) h->e = new Engine(device);
    CUDA_OK(cudaSetDevice(device));
    tl_stream = h->e->s;
    h->e->reset(analysis != 0);
    *out = h;
    return TSAT_OK;
  } catch (TsatException& ex) {
    return ex.code;
  } catch (...) {
    return TSAT_ERR_CUDA;
  }
}

void tsat_destroy(tsat_engine* h) {
  if (!h) return;
  auto& pool = engine_pool();
  bool pooled = false;
  if (h->e) tl_stream = h->e->s;
  if (h->e && pool.size() < 4) {
    try {
      h->e->reset(false);
      pool.push_back(h->e);
      pooled = true;
    } catch (...) {
    }
  }
  if (!pooled) delete h->e;
  delete h;
}

const char* tsat_last_error(tsat_engine* h) { return h ? h->err.c_str() : "null handle"; }

int tsat_set_atoms(tsat_engine* h, int32_t n, const int32_t* kind, const int64_t* ival, const int32_t* opcode,
                   const int32_t* ndims, const int64_t* dims, const int32_t* nident, const int64_t* idims,
                   const char* names, const int64_t* name_off) {
  GUARD(h, h->e->set_atoms(n, kind, ival, opcode, ndims, dims, nident, idims, names, name_off));
}

int tsat_load_egraph(tsat_engine* h, uint32_t n, const uint32_t* op, const uint32_t* child_off,
                     const uint32_t* child, uint32_t root) {
  GUARD(h, h->e->load_initial(n, op, child_off, child, root));
}

int tsat_add_terms(tsat_engine* h, int32_t ninstr, const int32_t* instr, int32_t nterm, const int32_t* term_len,
                   int32_t nenv, const uint32_t* env, uint32_t* out_class) {
  GUARD(h, {
    std::vector<Instr> prog(ninstr);
    for (int i = 0; i < ninstr; i++) {
      prog[i].kind = instr[4 * i];
      prog[i].arg = instr[4 * i + 1];
      prog[i].atom = (u32)instr[4 * i + 2];
      prog[i].depth = instr[4 * i + 3];
    }
    h->e->add_terms(ninstr, prog.data(), nterm, term_len, nenv, env, out_class);
    h->e->snap.valid = false;
  });
}

int tsat_union(tsat_engine* h, uint32_t a, uint32_t b, uint32_t* out_root) {
  GUARD(h, {
    *out_root = h->e->union_pair(a, b);
    h->e->snap.valid = false;
    if (h->e->root != TSAT_NONE) h->e->root = h->e->root;  // root tracked by node id; find() at read
  });
}

int tsat_rebuild(tsat_engine* h) { GUARD(h, h->e->rebuild()); }

int tsat_force_rebuild(tsat_engine* h) {
  GUARD(h, {
    Engine& e = *h->e;
    e.h.dirty = 1;
    e.push_counters();
    e.rebuild(true);
  });
}

int tsat_union_batch(tsat_engine* h, int64_t n, const uint32_t* a, const uint32_t* b) {
  GUARD(h, {
    Engine& e = *h->e;
    for (int64_t i = 0; i < n; i++) e.union_pair(a[i], b[i]);
  });
}

int tsat_find(tsat_engine* h, uint32_t x, uint32_t* out) { GUARD(h, *out = h->e->find(x)); }

int tsat_set_root(tsat_engine* h, uint32_t root) {
  GUARD(h, {
    if (root != TSAT_NONE && root >= h->e->h.next_id) throw TsatException(TSAT_ERR_ARG, "root out of range");
    h->e->root = root;
    h->e->root_ver = ~0ull;
  });
}

int tsat_query_sizes(tsat_engine* h, uint32_t* next_id, uint32_t* live, uint32_t* nkids, uint32_t* root,
                     uint32_t* dirty) {
  GUARD(h, {
    Engine& e = *h->e;
    *next_id = e.h.next_id;
    *live = e.h.live;
    *nkids = e.h.nkids;
    *root = e.root == TSAT_NONE ? TSAT_NONE : e.root_class();
    *dirty = e.h.dirty;
  });
}

int tsat_num_classes(tsat_engine* h, uint32_t* out) {
  GUARD(h, {
    Engine& e = *h->e;
    if (!e.snap.valid) e.build_snapshot();
    *out = e.snap.ncls;
  });
}

int tsat_download_flags(tsat_engine* h, uint8_t* flags) {
  GUARD(h, {
    Engine& e = *h->e;
    if (e.h.next_id) CUDA_OK(cudaMemcpyAsync(flags, e.flags.p, e.h.next_id, cudaMemcpyDeviceToHost, e.s));
    e.sync();
  });
}

int tsat_download(tsat_engine* h, uint32_t* op, uint32_t* child_off, uint32_t* child, uint32_t* cls,
                  uint8_t* flags) {
  GUARD(h, h->e->download(op, child_off, child, cls, flags));
}

int tsat_find_batch(tsat_engine* h, uint32_t n, const uint32_t* ids, uint32_t* out) {
  GUARD(h, h->e->find_batch(n, ids, out));
}

int tsat_download_nodes(tsat_engine* h, uint32_t n, const uint32_t* ids, uint32_t* op, uint32_t* child_off,
                        uint32_t* child, uint64_t child_cap, uint64_t* nchild) {
  GUARD(h, h->e->download_nodes(n, ids, op, child_off, child, child_cap, nchild));
}

int tsat_download_values(tsat_engine* h, void* vals, int64_t val_bytes, void* trees, int64_t tree_bytes,
                         uint32_t* ntrees) {
  GUARD(h, {
    Engine& e = *h->e;
    u64 need = (u64)e.h.next_id * sizeof(Val);
    u32 nt;
    CUDA_OK(cudaMemcpyAsync(&nt, e.tree_count.p, sizeof(u32), cudaMemcpyDeviceToHost, e.s));
    e.sync();
    *ntrees = nt;
    if (vals) {
      if ((u64)val_bytes < need) throw TsatException(TSAT_ERR_ARG, "value buffer too small");
      if (need) CUDA_OK(cudaMemcpyAsync(vals, e.val.p, need, cudaMemcpyDeviceToHost, e.s));
    }
    if (trees) {
      if ((u64)tree_bytes < (u64)nt * sizeof(Tree)) throw TsatException(TSAT_ERR_ARG, "tree buffer too small");
      if (nt) CUDA_OK(cudaMemcpyAsync(trees, e.trees.p, (u64)nt * sizeof(Tree), cudaMemcpyDeviceToHost, e.s));
    }
    e.sync();
  });
}

int tsat_dump(tsat_engine* h, char* buf, int64_t cap, int64_t* len) {
  GUARD(h, {
    std::string t = h->e->dump_text();
    *len = (int64_t)t.size();
    if (buf && cap >= (int64_t)t.size()) memcpy(buf, t.data(), t.size());
  });
}

int tsat_set_filter(tsat_engine* h, int32_t n, const uint32_t* ids, int32_t on) {
  GUARD(h, h->e->set_filter(n, ids, on));
}

int tsat_get_filter(tsat_engine* h, uint32_t* out, int64_t cap, int64_t* n) {
  GUARD(h, {
    std::vector<u32> f = h->e->get_filter();
    *n = (int64_t)f.size();
    if (out && cap >= (int64_t)f.size()) memcpy(out, f.data(), f.size() * sizeof(u32));
  });
}

int tsat_ilp_build(tsat_engine* h, uint32_t* sizes) { GUARD(h, h->e->ilp_build(sizes)); }

int tsat_ilp_download(tsat_engine* h, uint32_t* classes, uint32_t* nodes, uint32_t* live_off, uint32_t* live,
                      uint32_t* pick_off, uint32_t* pick_child) {
  GUARD(h, h->e->ilp_download(classes, nodes, live_off, live, pick_off, pick_child));
}

int tsat_set_record_rejects(tsat_engine* h, int32_t on) { GUARD(h, h->e->record_rejects = on != 0); }

int tsat_set_reach_budget(tsat_engine* h, uint64_t bytes) { GUARD(h, h->e->reach.budget = bytes); }

int tsat_reach_mode(tsat_engine* h, int32_t* mode) {
  if (!mode) return TSAT_ERR_ARG;
  GUARD(h, *mode = h->e->reach.mode);
}

int tsat_rejects(tsat_engine* h, uint32_t* out, int64_t cap, int64_t* n) {
  GUARD(h, {
    const std::vector<u32>& r = h->e->rejects;
    *n = (int64_t)r.size();
    if (out) {
      if (cap < (int64_t)r.size()) throw TsatException(TSAT_ERR_VALUE, "reject buffer too small");
      if (!r.empty()) memcpy(out, r.data(), r.size() * sizeof(u32));
    }
  });
}

int tsat_load_rules(tsat_engine* h, int64_t n, const int64_t* blob) { GUARD(h, h->e->load_rules((int)n, blob)); }

static int saturate_impl(tsat_engine* h, const tsat_limits* lim, int32_t filter_mode, int32_t allow_self,
                         tsat_report* rep, int64_t* rule_stats, int64_t* per_iter) {
  GUARD(h, {
    Engine& e = *h->e;
    if (lim->n_max < 0 || lim->k_max < 0 || lim->k_multi < 0)
      throw TsatException(TSAT_ERR_VALUE, "limits must be non-negative");
    if (lim->k_multi > lim->k_max) throw TsatException(TSAT_ERR_VALUE, "k_multi must be <= k_max");
    if (filter_mode < 0 || filter_mode > 2)
      throw TsatException(TSAT_ERR_VALUE, "filter_mode must be 'none', 'vanilla' or 'efficient'");
    e.rejects.clear();
    ExploreLimitsC L{lim->n_max, lim->k_max, lim->k_multi, lim->time_limit_s};
    e.saturate(L, filter_mode, allow_self, nullptr, 0);
    rep->iterations = e.report.iterations;
    rep->stop_reason = e.report.stop_reason;
    rep->prefilter_checks = e.report.prefilter_checks;
    rep->prefilter_rejects = e.report.prefilter_rejects;
    rep->postprocess_filtered = e.report.postprocess_filtered;
    rep->node_limit_overshoot = e.report.node_limit_overshoot;
    rep->filter_size = e.report.filter_size;
    rep->time_s = e.report.time_s;
    for (size_t r = 0; r < e.rstats.size(); r++) {
      const RuleStatsH& s = e.rstats[r];
      int64_t* o = rule_stats + 7 * r;
      o[0] = s.found;
      o[1] = s.applied;
      o[2] = s.applied_noop;
      o[3] = s.skipped_self;
      o[4] = s.skipped_compat;
      o[5] = s.skipped_shape;
      o[6] = s.skipped_cycle;
    }
    for (size_t i = 0; i < e.enodes_per_iter.size(); i++) {
      per_iter[3 * i] = e.enodes_per_iter[i];
      per_iter[3 * i + 1] = e.alloc_per_iter[i];
      per_iter[3 * i + 2] = e.eclasses_per_iter[i];
    }
  });
}

int tsat_saturate(tsat_engine* h, const tsat_limits* lim, int32_t filter_mode, int32_t allow_self, tsat_report* rep,
                  int64_t* rule_stats, int64_t* per_iter) {
  return saturate_impl(h, lim, filter_mode, allow_self, rep, rule_stats, per_iter);
}

int tsat_iterate(tsat_engine* h, const tsat_limits* lim, int32_t filter_mode, int32_t allow_self, int64_t iter_idx,
                 tsat_report* rep, int64_t* rule_stats, int64_t* per_iter) {
  if (!lim || iter_idx < 0) return TSAT_ERR_VALUE;
  tsat_limits one = *lim;
  one.k_max = 1;
  one.k_multi = iter_idx < lim->k_multi ? 1 : 0;  // explorer.py:341
  return saturate_impl(h, &one, filter_mode, allow_self, rep, rule_stats, per_iter);
}

int tsat_ematch(tsat_engine* h, int32_t pattern, uint32_t* out_cls, uint32_t* out_bind, int64_t cap, int64_t* n,
                int32_t* nb) {
  GUARD(h, {
    Engine& e = *h->e;
    if (pattern < 0 || pattern >= (int)e.patterns.size()) throw TsatException(TSAT_ERR_ARG, "bad pattern id");
    e.ematch_batch(std::vector<int>{pattern});
    MatchSet& ms = e.matches[pattern];
    *n = ms.n;
    *nb = ms.nb;
    if (out_cls && cap >= (int64_t)ms.n && ms.n) {
      CUDA_OK(cudaMemcpyAsync(out_cls, ms.cls.p, ms.n * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
      if (ms.nb)
        CUDA_OK(cudaMemcpyAsync(out_bind, ms.bind.p, (u64)ms.n * ms.nb * sizeof(u32), cudaMemcpyDeviceToHost, e.s));
      e.sync();
    }
  });
}

int tsat_ematch_batch(tsat_engine* h, int32_t npat, const int32_t* pids, int64_t* counts) {
  GUARD(h, {
    Engine& e = *h->e;
    std::vector<int> v;
    for (int i = 0; i < npat; i++) {
      if (pids[i] < 0 || pids[i] >= (int)e.patterns.size()) throw TsatException(TSAT_ERR_ARG, "bad pattern id");
      v.push_back(pids[i]);
    }
    e.ematch_batch(v);
    for (int i = 0; i < npat; i++) counts[i] = e.matches[pids[i]].n;
  });
}

int tsat_break_cycles(tsat_engine* h, int64_t* added) {
  GUARD(h, *added = h->e->break_all_cycles(false, nullptr));
}

int tsat_dfs_cycles(tsat_engine* h, uint32_t* nodes, int64_t cap, uint32_t* off, int64_t off_cap, int64_t* ncycles) {
  GUARD(h, {
    std::vector<std::vector<u32>> cyc;
    h->e->break_all_cycles(false, &cyc);
    *ncycles = (int64_t)cyc.size();
    int64_t tot = 0;
    for (auto& c : cyc) tot += (int64_t)c.size();
    if (nodes && cap >= tot && off_cap > (int64_t)cyc.size()) {
      int64_t k = 0;
      for (size_t i = 0; i < cyc.size(); i++) {
        off[i] = (uint32_t)k;
        for (u32 x : cyc[i]) nodes[k++] = x;
      }
      off[cyc.size()] = (uint32_t)k;
    } else {
      *ncycles = -tot - 1;  // buffer too small: -(total nodes) - 1
    }
  });
}

int tsat_costs(tsat_engine* h, int32_t mode, int32_t strict, int32_t ntab, const char* keys, const int64_t* key_off,
               const double* vals, double* out_by_node) {
  GUARD(h, {
    if (!h->e->snap.valid) h->e->build_snapshot();
    h->e->costs(mode, strict, ntab, keys, key_off, vals, out_by_node);
  });
}

int tsat_costs_gather(tsat_engine* h, uint32_t n, const uint32_t* ids, double* out) {
  GUARD(h, h->e->costs_gather(n, ids, out));
}

int tsat_greedy(tsat_engine* h, const double* cost_by_node, uint32_t* sel_cls, uint32_t* sel_node, uint32_t* nsel,
                double* root_best, int64_t* rounds) {
  GUARD(h, *root_best = h->e->greedy(cost_by_node, sel_cls, sel_node, nsel, rounds));
}

int tsat_shard_setup(tsat_engine* h, int32_t rank, int32_t world, const void* nccl_id, int32_t id_bytes) {
  GUARD(h, {
    if (world > 1 && nccl_id && id_bytes != 128) throw TsatException(TSAT_ERR_ARG, "need a 128-byte NCCL unique id");
    h->e->shard_setup(rank, world, nccl_id);
  });
}

int tsat_shard_setup_host(tsat_engine* h, int32_t rank, int32_t world, tsat_allgather_fn fn, void* ctx) {
  GUARD(h, {
    if (world > 1 && !fn) throw TsatException(TSAT_ERR_ARG, "need an all-gather function");
    h->e->shard_setup(rank, world, nullptr);
    h->e->host_ag = world > 1 ? fn : nullptr;
    h->e->host_ctx = ctx;
  });
}

int tsat_nccl_unique_id(void* out, int32_t cap, int32_t* len) {
  if (!out || !len || cap < 128) return TSAT_ERR_ARG;
  try {
    nccl_unique_id(out);
    *len = 128;
    return TSAT_OK;
  } catch (TsatException& ex) {
    return ex.code;
  }
}

int tsat_shard_range(uint64_t n_alloc, int32_t rank, int32_t world, uint32_t* lo, uint32_t* hi) {
  if (!lo || !hi || world < 1 || rank < 0 || rank >= world) return TSAT_ERR_ARG;
  shard_range(n_alloc, rank, world, *lo, *hi);
  return TSAT_OK;
}

int tsat_stream(tsat_engine* h, void** stream) { GUARD(h, *stream = (void*)h->e->s); }

int tsat_kernel_stats(tsat_engine* h, double* ms, double* bytes, int64_t* launches, int32_t n, int32_t reset) {
  GUARD(h, {
    Engine& e = *h->e;
    e.kt_resolve(true);
    for (int i = 0; i < n && i < KG_COUNT; i++) {
      ms[i] = e.kstat[i].ms;
      bytes[i] = e.kstat[i].bytes;
      launches[i] = (int64_t)e.kstat[i].launches;
    }
    if (reset)
      for (int i = 0; i < KG_COUNT; i++) e.kstat[i] = KStat();
  });
}

int tsat_debug_info(tsat_engine* h, int64_t* out, int32_t n) {
  GUARD(h, {
    Engine& e = *h->e;
    int64_t v[13] = {e.lv_n, e.lv_trimmed, e.snap.ncls, e.cg_ne, (int64_t)e.snap_id, (int64_t)e.filter_id,
                     (int64_t)e.h.next_id, (int64_t)e.h.live, (int64_t)g_dev_allocs, (int64_t)g_dev_alloc_bytes,
                     (int64_t)g_engines, (int64_t)e.nsync, (int64_t)e.nlaunch};
    for (int i = 0; i < n && i < 13; i++) out[i] = v[i];
  });
}

int tsat_phase_times(tsat_engine* h, double* out, int32_t n) {
  GUARD(h, {
    for (int i = 0; i < n; i++) out[i] = i < (int)h->e->phase_ms.size() ? h->e->phase_ms[i] : 0.0;
  });
}

}  // extern "C"

// ---------------------------------------------------------------- drop-in API helpers

int tsat_copy_state(tsat_engine* dst, tsat_engine* src) {
  if (!src) return TSAT_ERR_ARG;
  GUARD(dst, dst->e->copy_state_from(*src->e));
}

int tsat_eval_terms(tsat_engine* h, int32_t ninstr, const int32_t* instr, int32_t nterm, const int32_t* term_len,
                    int32_t nenv, const uint32_t* env, const uint32_t* env_off, void* out_vals, int32_t* out_status) {
  GUARD(h, {
    std::vector<Instr> prog(ninstr);
    for (int i = 0; i < ninstr; i++) {
      prog[i].kind = instr[4 * i];
      prog[i].arg = instr[4 * i + 1];
      prog[i].atom = (u32)instr[4 * i + 2];
      prog[i].depth = instr[4 * i + 3];
    }
    h->e->eval_terms(ninstr, prog.data(), nterm, term_len, nenv, env, env_off, out_vals, out_status);
  });
}

int tsat_class_graph(tsat_engine* h, uint32_t* cls, uint32_t* eoff, uint32_t* edst, uint32_t* sizes) {
  if (!sizes) return TSAT_ERR_ARG;
  GUARD(h, h->e->class_graph_download(cls, eoff, edst, sizes));
}

int tsat_descendants(tsat_engine* h, uint32_t* cls, uint32_t* bits, uint64_t cap_words, uint32_t* sizes) {
  if (!sizes) return TSAT_ERR_ARG;
  GUARD(h, h->e->descendants_download(cls, bits, cap_words, sizes));
}
