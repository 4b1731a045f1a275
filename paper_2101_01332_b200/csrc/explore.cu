#include <algorithm>
// Exploration driver (reference: pkg/src/tensorsat/explorer.py:136-365).
//
// Per iteration: snapshot CSR -> (efficient) descendants bitset -> e-match
// every unique canonical pattern on the snapshot -> rules in order over
// their match products -> rebuild -> cycle post-processing.  The apply
// step has two device paths: the sequential exact path in this file
// (k_seq_rule, the reference loop run by one GPU thread) and the parallel
// wave path (wave.cu) that handles hazard-free prefixes in bulk and falls
// back to k_seq_rule for exactly one combo at each hazard.
#include <cstdlib>
#include <chrono>
#include <cstring>

#include "rulesdev.cuh"

struct CtaCtl;
void run_rule_wave(Engine& e, int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long P,
                   const CtaCtl* resume, const DevStats* resume_stats);
void run_rules_chain(Engine& e, const std::vector<int>& rules, const std::vector<unsigned long long>& Ps,
                     int filter_mode, int allow_self, i64 n_max);
u32 wave_cta_cap();
void begin_wave_stats(Engine& e);
void flush_wave_stats_begin(Engine& e);
void flush_wave_stats_finish(Engine& e);


// ---------------------------------------------------------------- rule loading

void Engine::load_rules(int n, const i64* b) {
  (void)n;
  size_t k = 0;
  patterns.clear();
  rules.clear();
  i64 npat = b[k++];
  for (i64 p = 0; p < npat; p++) {
    HPattern hp;
    int napps = (int)b[k++];
    hp.nvars = (int)b[k++];
    if (napps < 1 || napps > MAX_PAT_APPS || hp.nvars > MAX_VARS)
      throw TsatException(TSAT_ERR_UNSUPPORTED, "pattern too large for the device matcher");
    for (int i = 0; i < hp.nvars; i++) hp.order.push_back((int)b[k++]);
    for (int a = 0; a < napps; a++) {
      PatApp pa;
      pa.atom = (u32)b[k++];
      pa.nargs = (int)b[k++];
      if (pa.nargs > 8) throw TsatException(TSAT_ERR_UNSUPPORTED, "pattern arity > 8");
      for (int j = 0; j < 8; j++) pa.child[j] = (int32_t)b[k++];
      hp.apps.push_back(pa);
    }
    patterns.push_back(hp);
  }
  i64 nr = b[k++];
  std::vector<Instr> all_instr;
  std::vector<int> all_leaf;
  for (i64 r = 0; r < nr; r++) {
    HRule hr;
    hr.nsrc = (int)b[k++];
    hr.nslots = (int)b[k++];
    hr.same_canon = b[k++] != 0;
    if (hr.nsrc < 1 || hr.nsrc > MAX_SRC || hr.nslots > MAX_VARS)
      throw TsatException(TSAT_ERR_UNSUPPORTED, "rule has too many sources or variables");
    for (int s_ = 0; s_ < hr.nsrc; s_++) {
      hr.src_pat[s_] = (int)b[k++];
      hr.src_nb[s_] = (int)b[k++];
      for (int j = 0; j < hr.src_nb[s_]; j++) hr.bind_slot[s_][j] = (int)b[k++];
    }
    int req = 0;
    for (int t = 0; t < hr.nsrc; t++) {
      int ni = (int)b[k++];
      std::vector<Instr> prog;
      int depth = 0, maxd = 0;
      for (int i = 0; i < ni; i++) {
        Instr in;
        in.kind = (int32_t)b[k++];
        in.arg = (int32_t)b[k++];
        in.atom = (u32)b[k++];
        in.depth = (int32_t)b[k++];
        if (in.kind == I_APP) {
          req++;
          depth -= in.arg;
          if (in.arg > 8) throw TsatException(TSAT_ERR_UNSUPPORTED, "target arity > 8");
        }
        depth++;
        maxd = std::max(maxd, depth);
        prog.push_back(in);
      }
      if (maxd > MAX_STACK) throw TsatException(TSAT_ERR_UNSUPPORTED, "target too deep");
      hr.targets.push_back(prog);
      int nl = (int)b[k++];
      std::vector<int> lv;
      for (int i = 0; i < nl; i++) lv.push_back((int)b[k++]);
      hr.leaves.push_back(lv);
    }
    hr.max_req = req;
    rules.push_back(hr);
  }
  // flatten programs to device
  for (auto& r : rules)
    for (size_t t = 0; t < r.targets.size(); t++) {
      all_instr.insert(all_instr.end(), r.targets[t].begin(), r.targets[t].end());
      all_leaf.insert(all_leaf.end(), r.leaves[t].begin(), r.leaves[t].end());
    }
  d_instr.ensure(all_instr.size() + 1);
  d_leaf.ensure(all_leaf.size() + 1);
  if (!all_instr.empty())
    CUDA_OK(cudaMemcpyAsync(d_instr.p, all_instr.data(), all_instr.size() * sizeof(Instr),
                            cudaMemcpyHostToDevice, s));
  if (!all_leaf.empty())
    CUDA_OK(cudaMemcpyAsync(d_leaf.p, all_leaf.data(), all_leaf.size() * sizeof(int),
                            cudaMemcpyHostToDevice, s));
  // match sets keep their device buffers across rule loads (no per-run
  // cudaMalloc / cudaFree, whose implicit syncs made run times erratic)
  if (matches.size() < patterns.size()) matches.resize(patterns.size());
  for (auto& m : matches) m.n = 0;
  rules_gen++;
  sync();
}

RuleDev make_rule_dev(Engine& e, int ri, int filter_mode, int allow_self) {
  RuleDev R;
  memset(&R, 0, sizeof(R));
  const HRule& hr = e.rules[ri];
  R.nsrc = hr.nsrc;
  R.nslots = hr.nslots;
  R.same_canon = hr.same_canon;
  R.allow_self = allow_self;
  R.efficient = filter_mode == 2;
  R.vanilla = filter_mode == 1;
  R.vanilla_go = ~0ull;
  R.max_req = hr.max_req;
  int mk = 0;
  size_t ioff = 0, loff = 0;
  for (int r = 0; r < ri; r++)
    for (size_t t = 0; t < e.rules[r].targets.size(); t++) {
      ioff += e.rules[r].targets[t].size();
      loff += e.rules[r].leaves[t].size();
    }
  for (int t = 0; t < hr.nsrc; t++) {
    const MatchSet& m = e.matches[hr.src_pat[t]];
    R.nmatch[t] = m.n;
    R.mcls[t] = m.cls.p;
    R.mbind[t] = m.bind.p;
    R.nb[t] = m.nb;
    for (int j = 0; j < hr.src_nb[t]; j++) R.bind_slot[t][j] = hr.bind_slot[t][j];
    R.tgt_off[t] = (int)ioff;
    R.tgt_len[t] = (int)hr.targets[t].size();
    R.leaf_off[t] = (int)loff;
    R.leaf_len[t] = (int)hr.leaves[t].size();
    for (auto& in : hr.targets[t])
      if (in.kind == I_APP) mk += in.arg;
    ioff += hr.targets[t].size();
    loff += hr.leaves[t].size();
  }
  R.max_kids = mk;
  R.instr = e.d_instr.p;
  R.leaf = e.d_leaf.p;
  R.deadline_ns = e.apply_deadline >= 0 ? e.dev_deadline_ns : 0ull;
  return R;
}

__global__ void k_dev_now(unsigned long long* out) { *out = dev_now_ns(); }

// the saturate deadline on the device clock: one clock read-back to map the
// host's now_s() onto %globaltimer
void Engine::set_device_deadline(double deadline_s) {
  dev_deadline_ns = 0;
  if (deadline_s < 0) return;
  DevBuf<unsigned long long> t;
  t.alloc(1);
  unsigned long long hd = 0;
  k_dev_now<<<1, 1, 0, s>>>(t.p);
  CUDA_OK(cudaMemcpyAsync(&hd, t.p, sizeof(hd), cudaMemcpyDeviceToHost, s));
  sync();
  const double left = deadline_s - now_s();
  dev_deadline_ns = left <= 0 ? 1ull : hd + (unsigned long long)(left * 1e9);
}

ReachDev make_reach_dev(Engine& e) {
  ReachDev r;
  r.bits = e.reach.bits.p;
  r.words = e.reach.words;
  r.n = e.reach.n;
  r.cls_index = e.snap.cls_index.p;
  r.n_alloc = e.snap.n_alloc;
  r.valid = e.reach.valid ? 1 : 0;
  r.mode = e.reach.mode;
  r.level = e.sc.cg_level.p;
  r.eoff = e.sc.cg_eoff.p;
  r.edst = e.sc.cg_edst.p;
  r.visit = e.reach.visit.p;
  r.stack = e.reach.stack.p;
  r.epoch = e.reach.epoch.p;
  // TSAT_REACH_STEPS (tests): budget of the private searches; 0 sends every
  // query the level filter cannot decide to the exact path
  static const char* st = getenv("TSAT_REACH_STEPS");
  r.steps = st ? atoi(st) : 96;
  return r;
}

// ---------------------------------------------------------------- exact path

// The reference run_rule loop (explorer.py:227-262) for product positions
// [p0, p1), executed by a single GPU thread against the live e-graph.
__global__ void k_seq_rule(G g, RuleDev R, ReachDev RD, DevStats* st, unsigned long long p0,
                           unsigned long long p1, i64 n_max) {
  if (threadIdx.x || blockIdx.x) return;
  Counters* c = g.cnt;
  u32 idx[MAX_SRC];
  u32 env[MAX_VARS];
  for (unsigned long long p = p0; p < p1; p++) {
    if ((u64)c->next_id + R.max_req + 2 > g.cap_nodes || (u64)c->nkids + R.max_kids + 2 > g.cap_kids ||
        (u64)c->next_id + R.max_req + 2 > (u64)g.hc_max) {
      st->resume_set = 1;
      st->resume_pos = p;
      return;
    }
    // the time limit, checked before every combo like the reference
    // (explorer.py:198-201) through the device clock
    if (R.deadline_ns && dev_now_ns() > R.deadline_ns) {
      st->timeout = 1;
      return;
    }
    if ((i64)c->live >= n_max) {
      st->stop = 1;
      st->overshoot = (u32)((i64)c->live - n_max);
      return;
    }
    st->found++;
    decode_pos(R, p, idx);
    if (R.nsrc > 1 && !R.allow_self && R.same_canon) {
      bool all = true;
      for (int i = 1; i < R.nsrc; i++) all &= idx[i] == idx[0];
      if (all) {
        st->skipped_self++;
        continue;
      }
    }
    // compatible() + combined_subst() with live find (rules.py:63-81)
    for (int v = 0; v < R.nslots; v++) env[v] = TSAT_NONE;
    bool compat = true;
    for (int i = 0; i < R.nsrc && compat; i++)
      for (int j = 0; j < R.nb[i]; j++) {
        u32 cls = uf_find(g.parent, R.mbind[i][(u64)idx[i] * R.nb[i] + j]);
        int sl = R.bind_slot[i][j];
        if (env[sl] == TSAT_NONE) env[sl] = cls;
        else if (env[sl] != cls) {
          compat = false;
          break;
        }
      }
    if (!compat) {
      st->skipped_compat++;
      continue;
    }
    // shape check (rules.py:141-156)
    if (g.analysis) {
      bool ok = true;
      Val scratch[MAX_STACK];
      for (int t = 0; t < R.nsrc && ok; t++) {
        const Val* outp = nullptr;
        int s = eval_target(g, R.instr + R.tgt_off[t], R.tgt_len[t], env, scratch, outp);
        if (s == AS_ORIGIN_OVERFLOW || s == AS_TREE_FULL) {
          dev_set_error(g.err, TSAT_ERR_CAPACITY, 10 + s, (i64)p, t);
          return;
        }
        if (s != AS_OK) ok = false;
        else ok = val_same_data(*outp, g.val[uf_find(g.parent, R.mcls[t][idx[t]])]);
      }
      if (!ok) {
        st->skipped_shape++;
        continue;
      }
    }
    // efficient pre-filter (explorer.py:208-225, cycles.py:151-169)
    if (R.efficient) {
      st->prefilter_checks++;
      bool hit = false;
      for (int t = 0; t < R.nsrc && !hit; t++) {
        u32 out = uf_find(g.parent, R.mcls[t][idx[t]]);
        for (int l = 0; l < R.leaf_len[t]; l++) {
          u32 leaf = uf_find(g.parent, env[R.leaf[R.leaf_off[t] + l]]);
          if (leaf == out || reach_query(RD, leaf, out, true) == REACH_YES) {
            hit = true;
            break;
          }
        }
      }
      if (hit) {
        st->prefilter_rejects++;
        st->skipped_cycle++;
        if (R.rej_log) {
          if (st->nrej >= R.rej_cap) {  // log full: resume here after the host drains it
            st->prefilter_rejects--;
            st->skipped_cycle--;
            st->prefilter_checks--;
            st->found--;
            st->resume_set = 1;
            st->resume_pos = p;
            return;
          }
          R.rej_log[2 * st->nrej] = (u32)(p >> 32);
          R.rej_log[2 * st->nrej + 1] = (u32)p;
          st->nrej++;
        }
        continue;
      }
    }
    // vanilla (cycles.py:248-254): the host applies this combo on a
    // checkpoint and runs the cycle check from the root
    if (R.vanilla && p != R.vanilla_go) {
      st->found--;  // counted again by the apply launch
      st->vpend = 1;
      st->resume_pos = p;
      return;
    }
    // _apply_combo (explorer.py:146-163)
    u32 before = c->next_id;
    bool did = false;
    for (int t = 0; t < R.nsrc; t++) {
      const Instr* ins = R.instr + R.tgt_off[t];
      u32 stk[MAX_STACK];
      int sp = 0;
      for (int k = 0; k < R.tgt_len[t]; k++) {
        const Instr& in = ins[k];
        if (in.kind == I_VAR) {
          stk[sp++] = uf_find(g.parent, env[in.arg]);
        } else {
          int na = in.arg;
          sp -= na;
          u32 kb[8];
          for (int j = 0; j < na; j++) kb[j] = stk[sp + j];
          u32 cl = seq_add_enode(g, in.atom, kb, na);
          if (cl == TSAT_NONE) return;  // error recorded
          stk[sp++] = cl;
        }
      }
      u32 nw = stk[0];
      u32 old = uf_find(g.parent, R.mcls[t][idx[t]]);
      if (uf_find(g.parent, nw) != old) {
        if (seq_union(g, old, nw) == TSAT_NONE) {
          g.err->a = (i64)p;  // merge error: keep rule context
          return;
        }
        did = true;
      }
    }
    if (did || c->next_id > before) {
      st->applied++;
      st->changed = 1;
    } else {
      st->applied_noop++;
    }
  }
}

static void accumulate(Engine& e, int ri, const DevStats& d) {
  RuleStatsH& r = e.rstats[ri];
  r.found += d.found;
  r.applied += d.applied;
  r.applied_noop += d.applied_noop;
  r.skipped_self += d.skipped_self;
  r.skipped_compat += d.skipped_compat;
  r.skipped_shape += d.skipped_shape;
  r.skipped_cycle += d.skipped_cycle;
  e.report.prefilter_checks += d.prefilter_checks;
  e.report.prefilter_rejects += d.prefilter_rejects;
}

// returns through dstats; grows capacity and resumes as needed
void Engine::run_rule_seq(int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long p0,
                          unsigned long long p1) {
  RuleDev R = make_rule_dev(*this, ri, filter_mode, allow_self);
  ReachDev RD = make_reach_dev(*this);
  if (record_rejects && R.efficient) {
    R.rej_cap = 4096;
    sc.v_rej.ensure(2 * R.rej_cap);
    R.rej_log = sc.v_rej.p;
  }
  unsigned long long p = p0;
  while (p < p1) {
    CUDA_OK(cudaMemsetAsync(dstats.p, 0, sizeof(DevStats), s));
    {
      KTimer kt(*this, KG_APPLY_SEQ, 0.0, 1);
      k_seq_rule<<<1, 1, 0, s>>>(view(), R, RD, dstats.p, p, p1, n_max);
    }
    DevStats d;
    CUDA_OK(cudaMemcpyAsync(&d, dstats.p, sizeof(d), cudaMemcpyDeviceToHost, s));
    pull_counters();
    accumulate(*this, ri, d);
    if (d.changed) seq_changed = true;
    if (d.stop) {
      seq_stop = true;
      report.node_limit_overshoot = d.overshoot;
    }
    if (d.timeout) seq_timeout = true;
    try {
      check_error();
    } catch (TsatException& ex) {
      if (ex.code == TSAT_ERR_MERGE)
        throw TsatException(ex.code, "unsound rule '" + rule_names[ri] + "': " + ex.what());
      throw;
    }
    if (d.nrej) {
      std::vector<u32> lg(2 * (size_t)d.nrej);
      CUDA_OK(cudaMemcpyAsync(lg.data(), R.rej_log, lg.size() * sizeof(u32), cudaMemcpyDeviceToHost, s));
      sync();
      for (u32 k = 0; k < d.nrej; k++) {
        const unsigned long long q = ((unsigned long long)lg[2 * k] << 32) | lg[2 * k + 1];
        if (rej_pending) rej_pending->push_back(q);  // a wave rule's exact-path combo: merged in order there
        else record_reject(ri, q);
      }
    }
    if (d.stop || d.timeout) return;
    if (!d.resume_set) return;
    p = d.resume_pos;
    ensure_nodes(4096 + (u64)R.max_req * 64, 4096 + (u64)R.max_kids * 64);
  }
}

// One rejected combo -> [rule, nsrc, (eclass, nb, bindings) x nsrc] from the
// iteration's match rows (the reference hands on_reject the Match objects).
void Engine::record_reject(int ri, unsigned long long p) {
  const HRule& hr = rules[ri];
  rejects.push_back((u32)ri);
  rejects.push_back((u32)hr.nsrc);
  unsigned long long q = p;
  u32 idx[MAX_SRC];
  for (int t = hr.nsrc - 1; t >= 0; t--) {  // itertools.product: last source fastest
    u32 n = matches[hr.src_pat[t]].n;
    idx[t] = (u32)(q % n);
    q /= n;
  }
  for (int t = 0; t < hr.nsrc; t++) {
    const MatchSet& m = matches[hr.src_pat[t]];
    u32 row[1 + MAX_VARS];
    CUDA_OK(cudaMemcpyAsync(row, m.cls.p + idx[t], sizeof(u32), cudaMemcpyDeviceToHost, s));
    if (m.nb)
      CUDA_OK(cudaMemcpyAsync(row + 1, m.bind.p + (u64)idx[t] * m.nb, m.nb * sizeof(u32), cudaMemcpyDeviceToHost, s));
    sync();
    rejects.push_back(row[0]);
    rejects.push_back((u32)m.nb);
    for (int j = 0; j < m.nb; j++) rejects.push_back(row[1 + j]);
  }
}

// filter_mode "vanilla" (explorer.py:218-220, cycles.py:248-254): every combo
// that passes the self / compat / shape gates is applied on the live e-graph
// after a device-to-device checkpoint of the mutable state (union-find
// parents, analysis values, interned cut trees, hashcons, counters); a cycle check from the root
// over the un-rebuilt result (peel + reachability, the precheck of
// break_all_cycles) decides, and a cycle restores the checkpoint.  Applying
// on the original instead of a clone gives the same e-graph: the apply is
// deterministic.  Cost: O(N) device work per checked combo, by design (the
// paper's baseline that the efficient pre-filter replaces).
void Engine::run_rule_vanilla(int ri, int allow_self, i64 n_max, unsigned long long P) {
  RuleDev R = make_rule_dev(*this, ri, 1, allow_self);
  ReachDev RD = make_reach_dev(*this);
  auto launch = [&](const RuleDev& Rx, unsigned long long a, unsigned long long b, DevStats& d) {
    CUDA_OK(cudaMemsetAsync(dstats.p, 0, sizeof(DevStats), s));
    {
      KTimer kt(*this, KG_APPLY_SEQ, 0.0, 1);
      k_seq_rule<<<1, 1, 0, s>>>(view(), Rx, RD, dstats.p, a, b, n_max);
    }
    CUDA_OK(cudaMemcpyAsync(&d, dstats.p, sizeof(d), cudaMemcpyDeviceToHost, s));
    pull_counters();
    try {
      check_error();
    } catch (TsatException& ex) {
      if (ex.code == TSAT_ERR_MERGE)
        throw TsatException(ex.code, "unsound rule '" + rule_names[ri] + "': " + ex.what());
      throw;
    }
  };
  unsigned long long p = 0;
  while (p < P) {
    // the reference checks its deadline before every combo (explorer.py:198-201);
    // the host loop here sees every combo that reaches the cycle check
    if (apply_deadline >= 0 && now_s() > apply_deadline) {
      seq_timeout = true;
      return;
    }
    DevStats d;
    launch(R, p, P, d);
    accumulate(*this, ri, d);
    if (d.stop) {
      seq_stop = true;
      report.node_limit_overshoot = d.overshoot;
      return;
    }
    if (d.timeout) {
      seq_timeout = true;
      return;
    }
    if (d.resume_set) {  // capacity
      p = d.resume_pos;
      ensure_nodes(4096 + (u64)R.max_req * 64, 4096 + (u64)R.max_kids * 64);
      continue;
    }
    if (!d.vpend) return;
    const unsigned long long q = d.resume_pos;
    ensure_nodes(4096 + (u64)R.max_req * 64, 4096 + (u64)R.max_kids * 64);
    // checkpoint
    const u32 n0 = h.next_id;
    const Counters h0 = h;
    sc.v_parent.ensure(n0 + 1);
    sc.v_hc.ensure((size_t)hc_cap);
    CUDA_OK(cudaMemcpyAsync(sc.v_parent.p, parent.p, (size_t)n0 * sizeof(u32), cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(sc.v_hc.p, hc.p, (size_t)hc_cap * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    if (analysis) {
      sc.v_val.ensure(n0 + 1);
      CUDA_OK(cudaMemcpyAsync(sc.v_val.p, val.p, (size_t)n0 * sizeof(Val), cudaMemcpyDeviceToDevice, s));
      // interned cut trees (analysis.cuh): table + count, so rejected applies leave no trace
      sc.v_tree_hc.ensure((size_t)tree_hc_cap + 1);
      CUDA_OK(cudaMemcpyAsync(sc.v_tree_hc.p, tree_hc.p, (size_t)tree_hc_cap * sizeof(u32), cudaMemcpyDeviceToDevice, s));
      CUDA_OK(cudaMemcpyAsync(sc.v_tree_hc.p + tree_hc_cap, tree_count.p, sizeof(u32), cudaMemcpyDeviceToDevice, s));
    }
    RuleDev R1 = R;
    R1.vanilla_go = q;
    DevStats d1;
    launch(R1, q, q + 1, d1);
    if (d1.resume_set || d1.stop || d1.vpend)
      throw TsatException(TSAT_ERR_STATE, "vanilla check: unexpected stop of the single-combo apply");
    snap.valid = false;
    bool cyc = break_all_cycles(true, nullptr) < 0;
    if (cyc) {
      CUDA_OK(cudaMemcpyAsync(parent.p, sc.v_parent.p, (size_t)n0 * sizeof(u32), cudaMemcpyDeviceToDevice, s));
      CUDA_OK(cudaMemcpyAsync(hc.p, sc.v_hc.p, (size_t)hc_cap * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
      if (analysis) {
        CUDA_OK(cudaMemcpyAsync(val.p, sc.v_val.p, (size_t)n0 * sizeof(Val), cudaMemcpyDeviceToDevice, s));
        CUDA_OK(cudaMemcpyAsync(tree_hc.p, sc.v_tree_hc.p, (size_t)tree_hc_cap * sizeof(u32), cudaMemcpyDeviceToDevice, s));
        CUDA_OK(cudaMemcpyAsync(tree_count.p, sc.v_tree_hc.p + tree_hc_cap, sizeof(u32), cudaMemcpyDeviceToDevice, s));
      }
      h = h0;
      push_counters();
      snap.valid = false;
      rstats[ri].found++;
      rstats[ri].skipped_cycle++;
      if (record_rejects) record_reject(ri, q);
    } else {
      accumulate(*this, ri, d1);
      if (d1.changed) seq_changed = true;
    }
    p = q + 1;
  }
}

// ---------------------------------------------------------------- saturate

void Engine::saturate(const ExploreLimitsC& lim, int filter_mode, int allow_self, const int*, int) {
  double t0 = now_s();
  double deadline = lim.time_limit_s < 0 ? -1.0 : t0 + lim.time_limit_s;
  set_device_deadline(deadline);
  memset(&report, 0, sizeof(report));
  rstats.assign(rules.size(), RuleStatsH());
  enodes_per_iter.clear();
  alloc_per_iter.clear();
  eclasses_per_iter.clear();
  std::vector<int> multi, single;
  for (size_t i = 0; i < rules.size(); i++) (rules[i].nsrc > 1 ? multi : single).push_back((int)i);
  int stop = 0;  // iter-limit
  spec_ematch = false;
  static const bool no_overlap = getenv("TSAT_NO_OVERLAP") != nullptr;
  const bool overlap_ok = !no_overlap && shard_world <= 1 && !getenv("TSAT_PHASE_SYNC") && !getenv("TSAT_DEBUG_ITERS");
  for (int q = 0; q < 32; q++) phase_ms[q] = 0.0;
  // host-side phase clocks (tsat_phase_times) need a stream sync per phase:
  // only when asked for (TSAT_PHASE_SYNC / TSAT_DEBUG_ITERS); the kernel-group
  // clocks are CUDA events and need none
  static const bool phase_sync = getenv("TSAT_PHASE_SYNC") || getenv("TSAT_DEBUG_ITERS");
  auto tick = [&](int ph, double& t) {
    if (phase_sync) sync();
    double n2 = now_s();
    phase_ms[ph] += (n2 - t) * 1e3;
    t = n2;
  };
  // a bounded search reserves its node / kid / hashcons capacity up front: a
  // mid-apply growth (copy + rehash) costs more than the whole reservation
  if (lim.n_max > 0 && lim.n_max < (1ll << 26) && (i64)h.next_id < 2 * lim.n_max) {
    u64 extra = (u64)(2 * lim.n_max - (i64)h.next_id);
    u64 avg_k = h.next_id ? ((u64)h.nkids + h.next_id - 1) / h.next_id : 2;
    ensure_nodes(extra, extra * std::max<u64>(avg_k + 1, 3));
  }
  double tp = now_s();
  for (i64 it = 0; it < lim.k_max; it++) {
    if (!snap.valid) build_snapshot();
    tick(0, tp);
    std::vector<int> active;
    if (it < lim.k_multi) active = multi;
    active.insert(active.end(), single.begin(), single.end());
    std::vector<char> need(patterns.size(), 0);
    for (int ri : active)
      for (int t = 0; t < rules[ri].nsrc; t++) need[rules[ri].src_pat[t]] = 1;
    std::vector<int> todo;
    for (size_t p = 0; p < patterns.size(); p++)
      if (need[p]) todo.push_back((int)p);
    if (filter_mode == 2) {
      // a pre-filter that needs a fresh peel (first iteration): this
      // iteration's e-matching overlaps it (nothing here changes the filter)
      if (!spec_ematch && overlap_ok && !levels_cached()) {
        if (!s2) {
          CUDA_OK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
          CUDA_OK(cudaEventCreateWithFlags(&ev_ov, cudaEventDisableTiming));
        }
        CUDA_OK(cudaEventRecord(ev_ov, s));
        overlap_hook = [this, todo]() {
          ematch_batch(todo);
          spec_ematch = true;
        };
      }
      build_reach();
      overlap_hook = nullptr;
    } else {
      reach.valid = false;
    }
    tick(1, tp);
    if (spec_ematch) spec_ematch = false;  // done next to a level peel
    else ematch_batch(todo);
    tick(2, tp);
    seq_changed = false;
    seq_stop = false;
    seq_timeout = false;
    apply_deadline = deadline;
    int stop_flag = 0;
    // consecutive single-source rules on the wave path run as one chain of
    // single-CTA launches (run_rules_chain); without a time limit only, since
    // the deadline is checked between rules on the host
    std::vector<int> chain;
    std::vector<unsigned long long> chainP;
    static const bool no_chain = getenv("TSAT_NO_CHAIN") != nullptr;
    auto flush = [&]() {
      if (chain.empty()) return;
      uf_changed = true;
      run_rules_chain(*this, chain, chainP, filter_mode, allow_self, lim.n_max);
      chain.clear();
      chainP.clear();
    };
    begin_wave_stats(*this);
    for (int ri : active) {
      const HRule& hr = rules[ri];
      unsigned long long P = 1;
      for (int t = 0; t < hr.nsrc; t++) P *= matches[hr.src_pat[t]].n;
      if (P == 0) continue;
      // (rules of <= 2048 positions: what the per-rule loop would run as one
      // single-CTA launch too; larger ones start on grid waves)
      if (!no_chain && deadline < 0 && !record_rejects && hr.nsrc == 1 && P <= wave_cta_cap() &&
          wave_path(ri, filter_mode)) {
        chain.push_back(ri);
        chainP.push_back(P);
        continue;
      }
      flush();
      if (seq_stop) break;
      if (deadline >= 0 && now_s() > deadline) {
        stop_flag = 3;
        break;
      }
      apply_rule(ri, filter_mode, allow_self, lim.n_max, P);
      if (seq_stop || seq_timeout) break;
    }
    if (!seq_stop && !seq_timeout) flush();
    flush_wave_stats_begin(*this);  // read back with the rebuild's read-back
    if (!stop_flag) {
      if (seq_stop) stop_flag = 2;
      else if (seq_timeout) stop_flag = 3;
    }
    snap.valid = false;
    tick(3, tp);
    rebuild();
    flush_wave_stats_finish(*this);
    tick(4, tp);
    build_snapshot();
    tick(0, tp);
    if (filter_mode != 0) {
      // when another iteration follows, its e-matching runs on the overlap
      // stream right after the cycle check's level peel is launched (the peel
      // is one latency-bound CTA); kept only if the check filters nothing
      const bool next = !stop_flag && seq_changed && it + 1 < lim.k_max && !(deadline >= 0 && now_s() > deadline);
      bool ran = false;
      if (next && overlap_ok) {
        std::vector<int> act2;
        if (it + 1 < lim.k_multi) act2 = multi;
        act2.insert(act2.end(), single.begin(), single.end());
        std::vector<char> need2(patterns.size(), 0);
        for (int ri : act2)
          for (int t = 0; t < rules[ri].nsrc; t++) need2[rules[ri].src_pat[t]] = 1;
        std::vector<int> todo2;
        for (size_t p = 0; p < patterns.size(); p++)
          if (need2[p]) todo2.push_back((int)p);
        if (!s2) {
          CUDA_OK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
          CUDA_OK(cudaEventCreateWithFlags(&ev_ov, cudaEventDisableTiming));
        }
        CUDA_OK(cudaEventRecord(ev_ov, s));
        overlap_hook = [this, todo2, &ran]() {
          ematch_batch(todo2);
          ran = true;
        };
      }
      const i64 added = break_all_cycles(false, nullptr);
      overlap_hook = nullptr;
      report.postprocess_filtered += added;
      spec_ematch = ran && added == 0 && snap.valid;
    }
    tick(5, tp);
    report.iterations = it + 1;
    {
      static const bool dbg_it = getenv("TSAT_DEBUG_ITERS") != nullptr;
      static double last[6];
      if (dbg_it) {
        if (it == 0)
          for (int q = 0; q < 6; q++) last[q] = 0;
        fprintf(stderr, "iter %lld: snap %.3f reach %.3f ematch %.3f apply %.3f rebuild %.3f cycles %.3f ms live %u\n",
                (long long)it, phase_ms[0] - last[0], phase_ms[1] - last[1], phase_ms[2] - last[2],
                phase_ms[3] - last[3], phase_ms[4] - last[4], phase_ms[5] - last[5], h.live);
        for (int q = 0; q < 6; q++) last[q] = phase_ms[q];
      }
    }
    enodes_per_iter.push_back(h.live);
    alloc_per_iter.push_back(h.next_id);
    eclasses_per_iter.push_back(snap.ncls);
    if (stop_flag) {
      stop = stop_flag;
      break;
    }
    if (!seq_changed) {
      stop = 1;
      break;
    }
    if (deadline >= 0 && now_s() > deadline) {
      stop = 3;
      break;
    }
  }
  report.stop_reason = stop;
  report.filter_size = (i64)get_filter().size();
  report.time_s = now_s() - t0;
  if (getenv("TSAT_DEBUG_SYNCS")) {
    std::vector<std::pair<long, std::string>> v;
    for (auto& kv : sync_sites) v.push_back({kv.second, kv.first});
    extern std::map<std::string, long> g_site_counts;
    for (auto& kv : g_site_counts) v.push_back({kv.second, kv.first});
    g_site_counts.clear();
    std::sort(v.rbegin(), v.rend());
    for (auto& x : v) fprintf(stderr, "sync %6ld  %s\n", x.first, x.second.c_str());
    sync_sites.clear();
  }
}


bool Engine::wave_path(int ri, int filter_mode) const {
  const HRule& hr = rules[ri];
  int R = 0;
  for (auto& t : hr.targets)
    for (auto& in : t) R += in.kind == I_APP;
  return filter_mode != 1 && hr.nsrc <= 2 && R <= 32 && !force_seq;
}

void Engine::apply_rule(int ri, int filter_mode, int allow_self, i64 n_max, unsigned long long P) {
  uf_changed = true;
  if (filter_mode == 1) run_rule_vanilla(ri, allow_self, n_max, P);
  else if (wave_path(ri, filter_mode)) run_rule_wave(*this, ri, filter_mode, allow_self, n_max, P, nullptr, nullptr);
  else run_rule_seq(ri, filter_mode, allow_self, n_max, 0, P);
}
