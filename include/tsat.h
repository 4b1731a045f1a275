/*
 * libtsat -- C-ABI of the B200 equality-saturation engine.
 *
 * Plain pointers and sizes only; every input array is caller-owned and copied
 * during the call, every output goes to caller-allocated memory (query sizes
 * first).  Status: 0 = ok, negative = error class (see TSAT_ERR_* below);
 * tsat_last_error() has the message.  A handle is not thread-safe and every
 * call is synchronous at return.
 *
 * Each entry point replaces one piece of the reference Python package
 * (tensorsat, /root/reference/pkg/src/tensorsat); the cited file:line is the
 * interface the call stands in for.  INTEGRATION.md shows the ctypes binding.
 */
#ifndef TSAT_H
#define TSAT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsat_engine tsat_engine;

enum {
  TSAT_OK = 0,
  TSAT_ERR_CUDA = -1,
  TSAT_ERR_ARG = -2,
  TSAT_ERR_SHAPE = -3,         /* errors.ShapeMismatch           (errors.py:22)   */
  TSAT_ERR_SPLIT_ORIGIN = -4,  /* errors.MissingSplitOrigin      (errors.py:26)   */
  TSAT_ERR_MERGE = -5,         /* errors.AnalysisMergeError      (errors.py:30)   */
  TSAT_ERR_NO_FINITE = -6,     /* errors.NoFiniteExtraction      (errors.py:45)   */
  TSAT_ERR_CAPACITY = -7,
  TSAT_ERR_UNSUPPORTED = -8,
  TSAT_ERR_UNKNOWN_SIG = -9,   /* errors.UnknownSignature        (errors.py:37)   */
  TSAT_ERR_VALUE = -10,        /* ValueError (limits / filter mode, explorer.py:63-67) */
  TSAT_ERR_STATE = -11         /* errors.TensorSatError                             */
};

typedef struct {
  int64_t n_max, k_max, k_multi;
  double time_limit_s; /* < 0: no limit */
} tsat_limits;         /* explorer.ExploreLimits (explorer.py:56-67) */

typedef struct {
  int64_t iterations;
  int32_t stop_reason; /* 0 iter-limit, 1 saturated, 2 node-limit, 3 timeout */
  int32_t pad;
  int64_t prefilter_checks, prefilter_rejects, postprocess_filtered, node_limit_overshoot, filter_size;
  double time_s;
} tsat_report;         /* explorer.ExploreReport (explorer.py:81-122) */

/* lifecycle -- EGraph.__init__(analysis) (egraph.py:115-125) */
int tsat_create(int device, int analysis, tsat_engine** out);
void tsat_destroy(tsat_engine* h);
const char* tsat_last_error(tsat_engine* h);

/* atom table: interned ops / literals (sexpr.Atom, sexpr.py:22; Value parsing
 * helpers tensor_lang.py:237-256).  Appends atoms [current count, n). */
int tsat_set_atoms(tsat_engine* h, int32_t n, const int32_t* kind, const int64_t* ival,
                   const int32_t* opcode, const int32_t* ndims, const int64_t* dims,
                   const int32_t* nident, const int64_t* idims, const char* names,
                   const int64_t* name_off);

/* initial e-graph in build_egraph id order (tensor_lang.py:749-767) */
int tsat_load_egraph(tsat_engine* h, uint32_t n, const uint32_t* op, const uint32_t* child_off,
                     const uint32_t* child, uint32_t root);

/* EGraph.add_term / add_enode (egraph.py:164-191): post-order programs,
 * 4 int32 per instruction (kind 0=var/1=app, arg, atom, depth) */
int tsat_add_terms(tsat_engine* h, int32_t ninstr, const int32_t* instr, int32_t nterm,
                   const int32_t* term_len, int32_t nenv, const uint32_t* env, uint32_t* out_class);
int tsat_union(tsat_engine* h, uint32_t a, uint32_t b, uint32_t* out_root); /* egraph.py:193 */
int tsat_rebuild(tsat_engine* h);                                            /* egraph.py:216 */
/* benchmark hooks: one full congruence round even when clean; a batch of unions */
int tsat_force_rebuild(tsat_engine* h);
int tsat_union_batch(tsat_engine* h, int64_t n, const uint32_t* a, const uint32_t* b);
int tsat_find(tsat_engine* h, uint32_t x, uint32_t* out);                    /* egraph.py:143 */
int tsat_find_batch(tsat_engine* h, uint32_t n, const uint32_t* ids, uint32_t* out); /* many finds, one sync */
int tsat_set_root(tsat_engine* h, uint32_t root);                            /* EGraph.root   */

/* sizes + SoA download (EGraph.nodes / classes / dump, egraph.py:127-162, 334-349) */
int tsat_query_sizes(tsat_engine* h, uint32_t* next_id, uint32_t* live, uint32_t* nkids,
                     uint32_t* root, uint32_t* dirty);
int tsat_num_classes(tsat_engine* h, uint32_t* out);
int tsat_download_flags(tsat_engine* h, uint8_t* flags);
int tsat_download(tsat_engine* h, uint32_t* op, uint32_t* child_off, uint32_t* child,
                  uint32_t* cls, uint8_t* flags);
/* selected nodes only (extract.reconstruct, extract.py:584-639): ops, child
 * offsets (n+1) and canonical children; *nchild > child_cap means retry with a
 * larger buffer */
int tsat_download_nodes(tsat_engine* h, uint32_t n, const uint32_t* ids, uint32_t* op, uint32_t* child_off,
                        uint32_t* child, uint64_t child_cap, uint64_t* nchild);
int tsat_download_values(tsat_engine* h, void* vals, int64_t val_bytes, void* trees,
                         int64_t tree_bytes, uint32_t* ntrees);
int tsat_dump(tsat_engine* h, char* buf, int64_t cap, int64_t* len);

/* filter list (cycles.FilterList, cycles.py:27) */
int tsat_set_filter(tsat_engine* h, int32_t n, const uint32_t* ids, int32_t on);
int tsat_get_filter(tsat_engine* h, uint32_t* out, int64_t cap, int64_t* n);

/* compiled rule set (rules.RewriteRule + canonical patterns, rules.py:36-123) */
int tsat_load_rules(tsat_engine* h, int64_t n, const int64_t* blob);

/* explorer.saturate (explorer.py:311-365); rule_stats = nrules x 7 int64 in
 * RuleStats field order, per_iter = 3 x k_max (enodes, alloc, eclasses) */
int tsat_saturate(tsat_engine* h, const tsat_limits* lim, int32_t filter_mode, int32_t allow_self,
                  tsat_report* rep, int64_t* rule_stats, int64_t* per_iter);
/* one iteration of saturate, iteration number iter_idx of the caller's loop: multi-pattern
 * rules active iff iter_idx < lim->k_multi (explorer.py:338-352); lim->k_max is ignored.
 * Per-iteration parity driver (SURVEY 8(b) tsat_iterate). */
int tsat_iterate(tsat_engine* h, const tsat_limits* lim, int32_t filter_mode, int32_t allow_self, int64_t iter_idx,
                 tsat_report* rep, int64_t* rule_stats, int64_t* per_iter);
/* filter_mode: 0 "none", 1 "vanilla" (apply on a checkpoint + cycle check per combo,
 * cycles.py:248-254), 2 "efficient" (descendants pre-filter, cycles.py:151-169) */

/* on_reject support (explorer.py:223-224): with recording on, tsat_saturate keeps
 * every cycle-rejected combo as [rule, nsrc, (eclass, nb, bindings[nb]) x nsrc]
 * (bindings in sorted canonical-variable order); tsat_rejects copies them out
 * (size query with out = NULL).  Efficient mode records through the exact
 * sequential path. */
/* ILP model skeleton (extract.reachable_classes + build_ilp, extract.py:198-322) over the
 * current filter list.  sizes = {classes, x variables, live members, pick rows}.
 * download: classes (root first, then ascending id), x nodes (alive members of those
 * classes, ascending id), live_off[classes+1] / live (non-filtered members per class,
 * ascending), pick_off[live+1] / pick_child (distinct child classes of each live member
 * as positions in classes, ascending class id).  Any out pointer may be NULL. */
int tsat_ilp_build(tsat_engine* h, uint32_t* sizes);
int tsat_ilp_download(tsat_engine* h, uint32_t* classes, uint32_t* nodes, uint32_t* live_off, uint32_t* live,
                      uint32_t* pick_off, uint32_t* pick_child);

int tsat_set_record_rejects(tsat_engine* h, int32_t on);

/* Memory budget (bytes) of the efficient pre-filter's descendants bitset
 * (cycles.get_descendants, cycles.py:70-148; the reference's big-int closure).
 * Snapshots whose C x C bitset exceeds it answer will_create_cycle's reaches()
 * (cycles.py:52-57, 151-169) from the peel levels plus a pruned search instead
 * (same answers, O(C + E) memory, no O(C^2/32) closure pass: a match's leaves lie
 * below its class, so the level test alone decides all but multi-pattern cross
 * queries).  Default 0 (levels always), or the TSAT_REACH_BUDGET environment
 * variable; reset when the engine is reused. */
int tsat_set_reach_budget(tsat_engine* h, uint64_t bytes);
/* mode of the last efficient iteration's pre-filter: 0 bitset, 1 levels + search */
int tsat_reach_mode(tsat_engine* h, int32_t* mode);
int tsat_rejects(tsat_engine* h, uint32_t* out, int64_t cap, int64_t* n);

/* EGraph.ematch of a loaded canonical pattern (egraph.py:248-262) */
int tsat_ematch(tsat_engine* h, int32_t pattern, uint32_t* out_cls, uint32_t* out_bind, int64_t cap,
                int64_t* n, int32_t* nb);

/* all patterns of one iteration in one batch (the saturate path); match counts
 * per pattern, lists stay on the device */
int tsat_ematch_batch(tsat_engine* h, int32_t npat, const int32_t* pids, int64_t* counts);

/* cycles.break_all_cycles / dfs_get_cycles (cycles.py:172-245) */
int tsat_break_cycles(tsat_engine* h, int64_t* added);
int tsat_dfs_cycles(tsat_engine* h, uint32_t* nodes, int64_t cap, uint32_t* off, int64_t off_cap,
                    int64_t* ncycles);

/* cost.egraph_costs (cost.py:225-247): mode 0 synthetic, 1 table */
int tsat_costs(tsat_engine* h, int32_t mode, int32_t strict, int32_t ntab, const char* keys,
               const int64_t* key_off, const double* vals, double* out_by_node);

/* entries of the device cost vector of the last tsat_costs (ids NULL: the
 * first n); lets callers skip downloading c_i for every node */
int tsat_costs_gather(tsat_engine* h, uint32_t n, const uint32_t* ids, double* out);

/* extract.greedy_extract (extract.py:120-159); cost_by_node NULL = device
 * vector from the last tsat_costs */
int tsat_greedy(tsat_engine* h, const double* cost_by_node, uint32_t* sel_cls, uint32_t* sel_node,
                uint32_t* nsel, double* root_best, int64_t* rounds);

/* Multi-GPU e-matching shards.  Rank r of ``world`` e-matches
 * root candidates whose e-class id lies in [lo_r, hi_r) (tsat_shard_range of
 * the allocated-node count) and the per-pattern match lists are all-gathered
 * over NCCL, rank-order concatenation being the global (eclass, bindings)
 * order of EGraph.ematch (egraph.py:107-112, 248-262).  The NCCL unique id is
 * created by rank 0 (tsat_nccl_unique_id) and distributed by the caller.
 * world == 1 disables sharding; nccl_id == NULL with world > 1 computes this
 * rank's part only, without the exchange (diagnostics / single-GPU tests). */
int tsat_shard_setup(tsat_engine* h, int32_t rank, int32_t world, const void* nccl_id, int32_t id_bytes);
/* Same shard group over a caller-supplied transport instead of NCCL: fn must
 * all-gather ``bytes`` from every rank's ``send`` into ``recv`` (world * bytes,
 * rank order; host memory) and return 0.  Used to run the exchange over
 * torch.distributed / gloo (tests with several ranks on one GPU). */
typedef int32_t (*tsat_allgather_fn)(void* ctx, const void* send, void* recv, uint64_t bytes);
int tsat_shard_setup_host(tsat_engine* h, int32_t rank, int32_t world, tsat_allgather_fn fn, void* ctx);
int tsat_nccl_unique_id(void* out, int32_t cap, int32_t* len);
int tsat_shard_range(uint64_t n_alloc, int32_t rank, int32_t world, uint32_t* lo, uint32_t* hi);

/* per kernel-group CUDA-event timings and algorithmic bytes since the last
 * reset; groups: rebuild, ematch, apply_seq, apply_wave, reach, cycles,
 * costs, greedy, snapshot */
int tsat_kernel_stats(tsat_engine* h, double* ms, double* bytes, int64_t* launches, int32_t n, int32_t reset);

/* the engine's CUDA stream (cudaStream_t) -- measurement only: bench.py
 * records its step events on it, so a step is timed on the device where its
 * kernels run (no reference counterpart) */
int tsat_stream(tsat_engine* h, void** stream);

/* diagnostics: level count, peeled classes, classes, class edges, snapshot /
 * filter versions, allocated and live e-nodes, device blocks allocated by the
 * block cache (count, bytes), engines constructed, host stream waits and kernels
 * launched by this engine */
int tsat_debug_info(tsat_engine* h, int64_t* out, int32_t n);

/* per-phase device timings of the last saturate / greedy (ms) */
int tsat_phase_times(tsat_engine* h, double* out, int32_t n);

/* ---- reference API pieces outside the explore loop ---------------------- */

/* EGraph.clone (egraph.py:351-364): copy src's e-graph state into dst (same
 * device; dst's atom table must already hold src's atoms in the same order). */
int tsat_copy_state(tsat_engine* dst, tsat_engine* src);
/* rules.eval_pattern (rules.py:126-138): shape-infer nterm post-order programs
 * (the tsat_add_terms format) under env[env_off[t] ...] on the device analysis,
 * without inserting anything.  out_vals: nterm device Value records (the
 * tsat_download_values layout); out_status: 0 ok, 1 ShapeMismatch,
 * 2 MissingSplitOrigin, other = capacity. */
int tsat_eval_terms(tsat_engine* h, int32_t ninstr, const int32_t* instr, int32_t nterm, const int32_t* term_len,
                    int32_t nenv, const uint32_t* env, const uint32_t* env_off, void* out_vals, int32_t* out_status);
/* cycles.live_adjacency (cycles.py:29-39) over the current filter list: classes
 * (ascending id), CSR offsets and child positions (one per child of every live,
 * unfiltered member).  sizes = {classes, edges}; outputs may be NULL. */
int tsat_class_graph(tsat_engine* h, uint32_t* cls, uint32_t* eoff, uint32_t* edst, uint32_t* sizes);
/* cycles.get_descendants (cycles.py:70-148): the transitive closure of the
 * live child relation as a word-major bitset (bits[w * n + i] = word w of
 * class i's descendants; a class is its own descendant iff it lies on a
 * cycle).  sizes = {classes, words}; bits NULL or cap_words < classes * words:
 * sizes only. */
int tsat_descendants(tsat_engine* h, uint32_t* cls, uint32_t* bits, uint64_t cap_words, uint32_t* sizes);

#ifdef __cplusplus
}
#endif
#endif
