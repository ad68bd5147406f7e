// schedule.cu — native Algorithm-1 driver over the B200 engine.
//
// Same control flow and offer order as the reference schedule() / run_two_phase()
// (src/scheduler.cpp:122-292) — restated, not linked — but every evaluation batch
// goes to the GPU as one unit: the iteration-1 probe list (top-k at gamma = 1, the
// gamma grid probes, the type-aligned prefix probes: 36-2,928 train sets) and each
// later iteration's top-k candidates are evaluated with one train-side batch, one
// config batch, grouped MILPs and one weight-sync batch, instead of four synchronous
// calls per partition. Results are memoised per train set within a window pass
// exactly as SearchPhase (src/scheduler.cpp:106-120); graph_partition_candidates is
// a pure function of the band, so its results are reused across passes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <atomic>
#include <memory>
#include <thread>
#include <vector>

#include "gp_internal.h"

namespace gp {

int train_batch(gp_ctx* ctx, int n_sets, const int32_t* const* ids, const int32_t* ns, int window,
                const gp_train_opts* o, gp_train_result* outs, int32_t* const* stage_devices, int mode = 0);
int ctx_make_aux(gp_ctx* ctx);
int configs_batch(gp_ctx* ctx, int q, const int32_t* const* ids, const int32_t* ns, const gp_rollout_opts* o,
                  std::vector<std::vector<gp_config>>& out, std::vector<int>* uniq_of = nullptr);
int milp_batch(gp_ctx* ctx, int q, const gp_config* const* cfgs, const int* ncs, const int32_t* const* caps,
               int dims, const double* Bs, double len, gp_rollout_result* outs, gp_rollout_entry* const* entries,
               int* rcs);
int weight_sync_batch(gp_ctx* ctx, int q, const int32_t* const* train, const int32_t* nt,
                      const int32_t* const* roll, const int32_t* nr, const int32_t* const* etype,
                      const int32_t* const* erep, const int32_t* ne, int window, double* out);
int partition_candidates(gp_ctx* ctx, const gp_gamma* g, const gp_part_opts* o, int k, gp_partition* out,
                         int32_t* train_ids, int32_t* n_out);
int partition_candidates_batch(gp_ctx* ctx, int q, const gp_gamma* gs, const gp_part_opts* o, int k,
                               gp_partition* out, int32_t* train_ids, int32_t* n_out, int* rcs);

namespace {

// GPLAN_PROFILE=1: host wall time per driver phase (stderr)
struct Phase {  // (contexts may be driven from several host threads: atomics)
  AtomicD sec[10];
  std::atomic<long long> spec_bands{0}, spec_kept{0}, widen_hits{0}, widen_calls{0};
  ~Phase() {
    if (!std::getenv("GPLAN_PROFILE")) return;
    static const char* n[10] = {"partition", "train_batch", "configs_batch", "milp_batch", "weight_sync", "total",
                               "eval_prep", "eval_post", "probe_lists", "spec_wait"};
    for (int i = 0; i < 10; ++i) std::fprintf(stderr, "gp_schedule %-14s %9.3f s\n", n[i], (double)sec[i]);
    double gpu = 0;
    for (int i = 0; i < 5; ++i) gpu += (double)sec[i];
    for (int i = 6; i < 10; ++i) gpu += (double)sec[i];
    std::fprintf(stderr, "gp_schedule %-14s %9.3f s\n", "host (rest)", (double)sec[5] - gpu);
    std::fprintf(stderr, "gp_schedule speculative bands %lld (kept %lld); widen %lld calls, %lld cache hits\n",
                 spec_bands.load(), spec_kept.load(), widen_calls.load(), widen_hits.load());
  }
} g_phase;

struct PhaseTimer {
  int id;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  NvtxRange nvtx;
  static const char* name(int i) {
    static const char* n[10] = {"gp_schedule/partition", "gp_schedule/train_batch", "gp_schedule/configs_batch",
                               "gp_schedule/milp_batch", "gp_schedule/weight_sync", "gp_schedule",
                               "gp_schedule/eval_prep", "gp_schedule/eval_post", "gp_schedule/probe_lists",
                               "gp_schedule/spec_wait"};
    return n[i];
  }
  explicit PhaseTimer(int i) : id(i), nvtx(name(i)) {}
  ~PhaseTimer() {
    g_phase.sec[id] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

struct Eval {  // IterationResult (src/scheduler.cpp:11-17)
  std::vector<int> train, roll;
  bool train_found = false;
  gp_train_result tr{};
  std::vector<int32_t> stage_dev;
  bool roll_found = false;
  gp_rollout_result rr{};
  std::vector<gp_config> cfg;  // config of each rollout entry
  std::vector<gp_rollout_entry> ent;
  double c_train = 0, c_rollout = 0, c_reward = 0, c_update = 0, c_infer = 0;
  bool feasible() const { return train_found && roll_found; }
  double objective() const { return c_train < c_infer ? c_infer : c_train; }  // std::max
};

struct Gamma {
  double q = 0, r = 1, gl = 1, gh = 1;
};

struct Driver {
  gp_ctx* ctx;
  const gp_sched_opts& o;
  int window = 1;
  std::map<std::vector<int>, std::unique_ptr<Eval>> memo;
  std::map<std::pair<double, double>, std::vector<std::vector<int>>> part_cache;
  long long evaluated = 0, layouts = 0;

  Driver(gp_ctx* c, const gp_sched_opts& opts) : ctx(c), o(opts) {}

  std::vector<int> complement(const std::vector<int>& train) const {
    std::vector<char> in(ctx->N, 0);
    for (int d : train) in[d] = 1;
    std::vector<int> roll;
    for (int d = 0; d < ctx->N; ++d)
      if (!in[d]) roll.push_back(d);
    return roll;
  }

  // evaluate_partition (src/scheduler.cpp:42-75) for every not-yet-memoised train set
  int eval_batch(const std::vector<std::vector<int>>& trains) {
    PhaseTimer* pt = new PhaseTimer(6);
    std::vector<const std::vector<int>*> todo;
    {
      auto less = [](const std::vector<int>* a, const std::vector<int>* b) { return *a < *b; };
      std::set<const std::vector<int>*, decltype(less)> seen(less);  // (no copies of the sets)
      for (const auto& t : trains)
        if (!memo.count(t) && seen.insert(&t).second) todo.push_back(&t);
    }
    const int q = (int)todo.size();
    if (q == 0) {
      delete pt;
      return GP_OK;
    }
    std::vector<std::unique_ptr<Eval>> ev(q);
    std::vector<const int32_t*> tids(q), rids(q);
    std::vector<int32_t> tn(q), rn(q);
    std::vector<int32_t*> sdev(q);
    auto make = [&](int i) {
      ev[i] = std::make_unique<Eval>();
      ev[i]->train = *todo[i];
      ev[i]->roll = complement(*todo[i]);
      ev[i]->stage_dev.assign(ev[i]->train.size() + 1, 0);
      ev[i]->c_reward = ctx->work.reward_cost_const;
      tids[i] = ev[i]->train.data();
      tn[i] = (int32_t)ev[i]->train.size();
      rids[i] = ev[i]->roll.data();
      rn[i] = (int32_t)ev[i]->roll.size();
      sdev[i] = ev[i]->stage_dev.data();
    };
    {  // (iteration 1: thousands of sets, built on several host threads)
      const int nt = std::min({8, (int)std::max(1u, std::thread::hardware_concurrency()), q / 256});
      if (nt <= 1) {
        for (int i = 0; i < q; ++i) make(i);
      } else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
          th.emplace_back([&, t] {
            for (int i = t; i < q; i += nt) make(i);
          });
        for (auto& x : th) x.join();
      }
    }
    delete pt;
    // train side: constrained_search
    std::vector<gp_train_result> tr(q);
    pt = new PhaseTimer(1);
    int rc = train_batch(ctx, q, tids.data(), tn.data(), window, &o.train, tr.data(), sdev.data());
    delete pt;
    if (rc) return rc;
    // rollout side: enumerate_configs + solve_milp
    std::vector<std::vector<gp_config>> cfgs;
    pt = new PhaseTimer(2);
    rc = configs_batch(ctx, q, rids.data(), rn.data(), &o.rollout, cfgs);
    delete pt;
    if (rc) return rc;
    const int T = ctx->T;
    std::vector<int> mq;  // sets with configs
    for (int i = 0; i < q; ++i)
      if (!cfgs[i].empty()) mq.push_back(i);
    const double B = (double)ctx->work.batch_rollouts * window;
    if (!mq.empty()) {
      const int m = (int)mq.size();
      std::vector<const gp_config*> cp(m);
      std::vector<int> nc(m);
      std::vector<std::vector<int32_t>> caps(m, std::vector<int32_t>(T, 0));
      std::vector<const int32_t*> capp(m);
      std::vector<double> Bs(m, B);
      std::vector<gp_rollout_result> rr(m);
      std::vector<std::vector<gp_rollout_entry>> ent(m);
      std::vector<gp_rollout_entry*> ep(m);
      std::vector<int> rcs(m);
      for (int j = 0; j < m; ++j) {
        const int i = mq[j];
        cp[j] = cfgs[i].data();
        nc[j] = (int)cfgs[i].size();
        for (int d : ev[i]->roll) caps[j][ctx->h_type[d]]++;  // rollout_capacities
        capp[j] = caps[j].data();
        ent[j].assign(nc[j], gp_rollout_entry{});
        ep[j] = ent[j].data();
      }
      pt = new PhaseTimer(3);
      rc = milp_batch(ctx, m, cp.data(), nc.data(), capp.data(), T, Bs.data(), ctx->work.mean_len, rr.data(),
                      ep.data(), rcs.data());
      delete pt;
      if (rc) return rc;
      for (int j = 0; j < m; ++j) {
        const int i = mq[j];
        if (rcs[j] == GP_INVALID)  // ValidationError escapes schedule() (src/rollout_milp.cpp:110-112)
          return set_error(GP_INVALID, "capacity lattice too large for the exact solver");
        if (rcs[j] != GP_OK) continue;  // InfeasibleError: caught, rollout = nullopt
        Eval& e = *ev[i];
        e.roll_found = true;
        e.rr = rr[j];
        for (int k = 0; k < rr[j].n_entries; ++k) {
          e.ent.push_back(ent[j][k]);
          e.cfg.push_back(cfgs[i][ent[j][k].config]);
        }
      }
    }
    // costs + weight sync for sets with both sides
    std::vector<int> wq;
    for (int i = 0; i < q; ++i) {
      Eval& e = *ev[i];
      e.train_found = tr[i].found != 0;
      e.tr = tr[i];
      e.c_train = e.train_found ? tr[i].cost : kInf;
      layouts += tr[i].layouts;
      if (e.roll_found && e.train_found) wq.push_back(i);
      else {
        e.c_rollout = e.roll_found ? e.rr.makespan : kInf;
        e.c_infer = kInf;
      }
    }
    if (!wq.empty()) {
      const int w = (int)wq.size();
      std::vector<const int32_t*> wt(w), wr(w), wet(w), wer(w);
      std::vector<int32_t> wtn(w), wrn(w), wne(w);
      std::vector<std::vector<int32_t>> et(w), er(w);
      std::vector<double> upd(w);
      for (int j = 0; j < w; ++j) {
        Eval& e = *ev[wq[j]];
        wt[j] = e.train.data();
        wtn[j] = (int32_t)e.train.size();
        wr[j] = e.roll.data();
        wrn[j] = (int32_t)e.roll.size();
        for (size_t k = 0; k < e.ent.size(); ++k) {
          int type = -1;  // ReplicaConfig::gpu_type
          for (int t = 0; t < T; ++t)
            if (e.cfg[k].type_counts[t] > 0) {
              type = t;
              break;
            }
          et[j].push_back(type);
          er[j].push_back(e.ent[k].replicas);
        }
        wet[j] = et[j].data();
        wer[j] = er[j].data();
        wne[j] = (int32_t)et[j].size();
      }
      pt = new PhaseTimer(4);
      rc = weight_sync_batch(ctx, w, wt.data(), wtn.data(), wr.data(), wrn.data(), wet.data(), wer.data(),
                             wne.data(), window, upd.data());
      delete pt;
      if (rc) return rc;
      for (int j = 0; j < w; ++j) {
        Eval& e = *ev[wq[j]];
        e.c_rollout = e.rr.makespan;
        e.c_update = upd[j];
        e.c_infer = e.c_rollout + e.c_reward + e.c_update;
      }
    }
    pt = new PhaseTimer(7);
    for (int i = 0; i < q; ++i) {
      const std::vector<int>& key = ev[i]->train;
      memo.emplace(key, std::move(ev[i]));
    }
    delete pt;
    evaluated += q;
    return GP_OK;
  }

  const Eval* get(const std::vector<int>& train) const { return memo.at(train).get(); }

  // partition_with_widening for several gammas at once (iteration 1's probes): the
  // unwidened bands of every gamma not yet cached in ONE batched partition call; a band that
  // is infeasible continues with the sequential widening loop below (same result)
  int widen_batch(const std::vector<Gamma>& gs, std::vector<std::vector<std::vector<int>>>& outs) {
    outs.assign(gs.size(), {});
    std::vector<Gamma> todo_g;
    std::vector<int> todo;
    for (size_t i = 0; i < gs.size(); ++i) {
      auto it = part_cache.find(std::make_pair(gs[i].gl, gs[i].gh));
      if (it != part_cache.end()) {
        outs[i] = it->second;
      } else {
        todo.push_back((int)i);
        todo_g.push_back(gs[i]);
      }
    }
    if (todo.empty()) return GP_OK;
    PhaseTimer pt(0);
    std::vector<std::vector<std::vector<int>>> res;
    int rc = widen_rounds(ctx, todo_g, res);
    if (rc) return rc;
    for (size_t j = 0; j < todo.size(); ++j) {
      outs[todo[j]] = res[j];
      part_cache[std::make_pair(todo_g[j].gl, todo_g[j].gh)] = std::move(res[j]);
    }
    return GP_OK;
  }

  // partition_with_widening (src/scheduler.cpp:21-40) for several bands on context c, uncached:
  // the bands still infeasible after a round move to their next widening together, one
  // batched call per round — each band sees exactly the sequence of bands widen() would try
  int widen_rounds(gp_ctx* c, const std::vector<Gamma>& gs, std::vector<std::vector<std::vector<int>>>& outs) const {
    outs.assign(gs.size(), {});
    const int k = std::max(1, o.candidate_width), N = c->N;
    gp_part_opts po{o.exact_threshold, o.restarts, o.seed, o.band_epsilon, o.force_local_search,
                    o.machine_granularity};
    std::vector<double> w(gs.size(), 0.0);
    std::vector<int> live(gs.size());
    for (size_t j = 0; j < gs.size(); ++j) live[j] = (int)j;
    for (bool first = true; !live.empty(); first = false) {
      if (!first)
        for (int j : live) {
          const double lo = gs[j].gl - w[j], hi = gs[j].gh + w[j];  // the attempt that failed
          if (!(0.0 < lo) && !(hi < 1.0))
            return set_error(GP_INFEASIBLE, "no feasible bisection exists even with an unconstrained band");
          w[j] += o.band_widen_step;
        }
      const int q = (int)live.size();
      std::vector<gp_gamma> gg(q);
      for (int m = 0; m < q; ++m) {
        const Gamma& g = gs[live[m]];
        const double lo = g.gl - w[live[m]], hi = g.gh + w[live[m]];
        gg[m] = gp_gamma{g.q, g.r, (0.0 < lo) ? lo : 0.0, (hi < 1.0) ? hi : 1.0};
      }
      std::vector<gp_partition> parts((size_t)q * k);
      std::vector<int32_t> ids((size_t)q * k * N + 1);
      std::vector<int32_t> nout(q);
      std::vector<int> rcs(q);
      int rc = partition_candidates_batch(c, q, gg.data(), &po, k, parts.data(), ids.data(), nout.data(),
                                          rcs.data());
      if (rc) return rc;
      std::vector<int> still;
      for (int m = 0; m < q; ++m) {
        if (rcs[m] != GP_OK) {  // GP_BAND_INFEASIBLE: widened in the next round
          still.push_back(live[m]);
          continue;
        }
        auto& res = outs[live[m]];
        const int32_t* idb = ids.data() + (size_t)m * k * N;
        for (int e = 0; e < nout[m]; ++e) {
          const gp_partition& pp = parts[(size_t)m * k + e];
          res.emplace_back(idb + pp.train_offset, idb + pp.train_offset + pp.train_count);
        }
      }
      live.swap(still);
    }
    return GP_OK;
  }

  // Speculative partitions (multi-device contexts): the bands the NEXT iteration can ask for
  // (refine_gamma moves to one of two midpoints) are computed on the auxiliary context while
  // this iteration's evaluation batch runs. graph_partition_candidates is a pure function of
  // the band, so a band that was feasible unwidened enters part_cache exactly as widen()
  // would have stored it; an infeasible one is left to widen().
  struct Spec {
    std::vector<Gamma> gs;
    std::vector<std::vector<std::vector<int>>> outs;
    int rc = GP_OK;
    std::thread th;
  };
  void spec_start(Spec& sp, const std::vector<Gamma>& next) {
    gp_ctx* aux = ctx->aux;
    if (!aux) return;
    for (const Gamma& g : next)
      if (!part_cache.count(std::make_pair(g.gl, g.gh))) sp.gs.push_back(g);
    const int q = (int)sp.gs.size();
    if (q == 0) return;
    g_phase.spec_bands += q;
    sp.th = std::thread([this, &sp, aux] {
      cudaSetDevice(aux->device);
      sp.rc = widen_rounds(aux, sp.gs, sp.outs);
    });
  }
  void spec_finish(Spec& sp) {
    if (!sp.th.joinable()) return;
    {
      PhaseTimer pt(9);  // (time the evaluation batch waited for the speculation)
      sp.th.join();
    }
    cudaSetDevice(ctx->device);
    if (sp.rc != GP_OK) return;  // (speculation only: widen() computes what is missing)
    for (size_t j = 0; j < sp.gs.size(); ++j) {
      part_cache[std::make_pair(sp.gs[j].gl, sp.gs[j].gh)] = std::move(sp.outs[j]);
      g_phase.spec_kept++;
    }
  }

  // partition_with_widening (src/scheduler.cpp:21-40) -> candidate train sets, best first
  int widen(const Gamma& g, std::vector<std::vector<int>>& out) {
    auto key = std::make_pair(g.gl, g.gh);
    auto it = part_cache.find(key);
    g_phase.widen_calls++;
    if (it != part_cache.end()) {
      g_phase.widen_hits++;
      out = it->second;
      return GP_OK;
    }
    PhaseTimer pt(0);
    std::vector<std::vector<std::vector<int>>> res;
    int rc = widen_rounds(ctx, {g}, res);
    if (rc) return rc;
    out = res[0];
    part_cache[key] = std::move(res[0]);
    return GP_OK;
  }

};

static bool spec_off() {
  static const bool off = [] {
    const char* e = std::getenv("GPLAN_SPECULATE");
    return e && e[0] == '0';
  }();
  return off;
}

struct BestTracker {  // src/scheduler.cpp:77-95
  const Eval* conforming = nullptr;
  const Eval* any = nullptr;
  void offer(const Eval* it) {
    if (!it || !it->feasible()) return;
    const double m = it->objective();
    if (!any || m < any->objective()) any = it;
    if (it->c_infer >= it->c_train)
      if (!conforming || m < conforming->objective()) conforming = it;
  }
  const Eval* result() const { return conforming ? conforming : any; }
};

struct Run {
  const Eval* best = nullptr;
  int iterations = 0;
  bool converged = false;
  std::vector<double> trace;
};

// run_two_phase (src/scheduler.cpp:122-255)
int run_two_phase(Driver& D, Run& run) {
  gp_ctx* ctx = D.ctx;
  const gp_sched_opts& o = D.o;
  const int N = ctx->N;
  Gamma gamma;
  bool frozen = false;
  BestTracker best;
  const Eval* cached = nullptr;
  bool reuse = false;
  double anchor = 0;
  bool has_anchor = false;
  int streak = 0;
  run.trace.clear();
  for (int iter = 1; iter <= o.iteration_cap; ++iter) {
    run.iterations = iter;
    const Eval* it;
    if (reuse && cached) {
      it = cached;
    } else {
      std::vector<std::vector<int>> cands;
      std::vector<std::vector<std::vector<int>>> grid;
      std::vector<std::vector<int>> prefixes;
      int rc;
      if (iter == 1) {  // the main band and the grid probes: one batched partition call
        std::vector<Gamma> gs{gamma};
        for (int p = 1; p <= o.grid_probes; ++p) {
          Gamma probe = gamma;
          probe.gl = probe.gh = static_cast<double>(p) / (o.grid_probes + 1);
          gs.push_back(probe);
        }
        std::vector<std::vector<std::vector<int>>> outs;
        rc = D.widen_batch(gs, outs);
        if (rc) return rc;
        cands = std::move(outs[0]);
        for (size_t i = 1; i < outs.size(); ++i) grid.push_back(std::move(outs[i]));
      } else {
        rc = D.widen(gamma, cands);
        if (rc) return rc;
      }
      PhaseTimer* pl = new PhaseTimer(8);
      std::vector<std::vector<int>> batch = cands;
      if (iter == 1) {
        for (const auto& pc : grid) batch.insert(batch.end(), pc.begin(), pc.end());
        for (int lead = 0; lead < ctx->T; ++lead) {  // type-aligned prefix probes
          std::vector<int> order(N);
          for (int d = 0; d < N; ++d) order[d] = d;
          std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            const int ta = ctx->h_type[a], tb = ctx->h_type[b];
            const bool la = ta == lead, lb = tb == lead;
            if (la != lb) return la;
            if (ta != tb) return ta < tb;
            return a < b;
          });
          std::vector<int> s;  // the first m + 1 devices of `order`, ascending (ids are distinct)
          s.reserve(N);
          for (int m = 0; m + 1 < N; ++m) {
            s.insert(std::upper_bound(s.begin(), s.end(), order[m]), order[m]);
            prefixes.push_back(s);
          }
        }
        batch.insert(batch.end(), prefixes.begin(), prefixes.end());
      }
      delete pl;
      {
        // the next iteration's possible bands, partitioned on the auxiliary context meanwhile
        Driver::Spec spec;
        if (!frozen && ctx->aux && !spec_off()) {
          std::vector<Gamma> next;
          if (iter == 1) {
            Gamma g = gamma;
            g.gl = g.gh = (gamma.q + gamma.r) / 2;
            next.push_back(g);
          } else {
            Gamma lo = gamma, hi = gamma;  // refine_gamma's two outcomes
            lo.r = (gamma.q + gamma.r) / 2.0;
            lo.gl = lo.gh = (lo.q + lo.r) / 2.0;
            hi.q = (gamma.q + gamma.r) / 2.0;
            hi.gl = hi.gh = (hi.q + hi.r) / 2.0;
            next.push_back(lo);
            next.push_back(hi);
          }
          D.spec_start(spec, next);
        }
        rc = D.eval_batch(batch);  // every evaluation of this iteration in one GPU batch
        D.spec_finish(spec);
      }
      if (rc) return rc;
      it = D.get(cands.front());
      for (size_t c = 1; c < cands.size(); ++c) best.offer(D.get(cands[c]));
      if (iter == 1) {
        for (const auto& pc : grid)
          for (const auto& t : pc) best.offer(D.get(t));
        for (const auto& t : prefixes) best.offer(D.get(t));
      }
      cached = it;
    }
    best.offer(it);
    const double m = it->objective();
    run.trace.insert(run.trace.end(), {(gamma.gl + gamma.gh) / 2, it->c_train, it->c_infer, m});
    if (has_anchor && std::abs(m - anchor) <= o.stability_tol * std::abs(anchor)) {
      streak++;
    } else {
      anchor = m;
      has_anchor = true;
      streak = 0;
    }
    if (streak >= o.stable_iters) {
      run.converged = true;
      break;
    }
    if (!frozen) {
      const double ct = it->c_train, ci = it->c_infer;
      const double mx = ct < ci ? ci : ct;
      const bool balanced = it->feasible() && std::abs(ct - ci) <= o.balance_tol * mx;
      if (balanced || (gamma.r - gamma.q) < o.interval_min) {
        frozen = true;
      } else if (iter == 1) {
        gamma.gl = gamma.gh = (gamma.q + gamma.r) / 2;
        cached = nullptr;
      } else {  // refine_gamma (src/partition.cpp:10-20)
        if (ct < ci) gamma.r = (gamma.q + gamma.r) / 2.0;
        else gamma.q = (gamma.q + gamma.r) / 2.0;
        const double mid = (gamma.q + gamma.r) / 2.0;
        gamma.gl = gamma.gh = mid;
        cached = nullptr;
      }
    }
    reuse = frozen && cached;
  }
  run.best = best.result();
  if (!run.best) return set_error(GP_INFEASIBLE, "no feasible plan at any visited partition");
  return GP_OK;
}

}  // namespace

int schedule(gp_ctx* ctx, const gp_sched_opts* o, gp_schedule_result* res, int32_t* train_ids,
             int32_t* rollout_ids, int32_t* stage_devices, gp_config* entry_configs, gp_rollout_entry* entries,
             int32_t entry_cap, double* trace) {
  PhaseTimer total(5);
  std::memset(res, 0, sizeof *res);
  if (ctx->N < 2) return set_error(GP_INFEASIBLE, "scheduling requires at least two devices");
  {  // speculative partitions: on multi-device contexts (their auxiliary context); on a one-GPU
     // context only with GPLAN_SPECULATE=1 (an auxiliary context on the same GPU: measured
     // within noise on C5, the partitions then compete with the train scans for the SMs);
     // GPLAN_SPECULATE=0 turns them off
    const char* e = std::getenv("GPLAN_SPECULATE");
    const bool force = e && e[0] == '1';
    if (!ctx->aux && ctx->peers.empty() && force) {
      int rc = ctx_make_aux(ctx);
      if (rc) return rc;
    }
  }
  const int eta = o->eta_override >= 0 ? o->eta_override : ctx->work.staleness;
  // WindowExpander (inc/rollout_milp.hpp:51-81)
  const int cap = o->delta_cap;
  int delta = std::min(std::max(eta + 1, 1), cap);
  double last = 0;
  bool has_last = false;
  int wstreak = 0;
  std::unique_ptr<Driver> D;
  Run run;
  std::map<std::pair<double, double>, std::vector<std::vector<int>>> parts;  // survives passes
  long long evaluated = 0, layouts = 0;
  while (true) {
    NvtxRange pass_range("gp_schedule/window_pass");
    D = std::make_unique<Driver>(ctx, *o);  // fresh memo per pass (src/scheduler.cpp:129)
    D->window = delta;
    D->part_cache = parts;
    run = Run();
    int rc = run_two_phase(*D, run);
    parts = D->part_cache;
    evaluated += D->evaluated;
    layouts += D->layouts;
    if (rc) return rc;
    const double per_step = run.best->objective() / delta;
    const bool stable = has_last && std::abs(per_step - last) <= 0.01 * std::abs(last);
    wstreak = stable ? wstreak + 1 : 0;
    last = per_step;
    has_last = true;
    const bool stop = wstreak >= 2 || delta >= cap;
    if (!o->expand_window || stop) break;
    delta = std::min(2 * delta, cap);
  }
  const Eval& b = *run.best;
  res->window = delta;
  res->staleness = eta;
  res->iterations_run = run.iterations;
  res->converged = run.converged;
  res->n_trace = (int32_t)(run.trace.size() / 4);
  if (trace) std::memcpy(trace, run.trace.data(), sizeof(double) * run.trace.size());
  res->n_train = (int32_t)b.train.size();
  res->n_rollout = (int32_t)b.roll.size();
  std::memcpy(train_ids, b.train.data(), sizeof(int32_t) * b.train.size());
  std::memcpy(rollout_ids, b.roll.data(), sizeof(int32_t) * b.roll.size());
  res->train = b.tr;
  std::memcpy(stage_devices, b.stage_dev.data(), sizeof(int32_t) * b.train.size());
  res->rollout = b.rr;
  if ((int)b.ent.size() > entry_cap) return set_error(GP_CAPACITY, "entry buffer too small");
  for (size_t k = 0; k < b.ent.size(); ++k) {
    entries[k] = b.ent[k];
    entries[k].config = (int32_t)k;  // index into entry_configs
    entry_configs[k] = b.cfg[k];
  }
  res->c_train = b.c_train;
  res->c_rollout = b.c_rollout;
  res->c_reward = b.c_reward;
  res->c_update = b.c_update;
  res->c_infer_total = b.c_infer;
  res->evaluated_partitions = evaluated;
  res->evaluated_layouts = layouts;
  return GP_OK;
}

}  // namespace gp
