// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference rlsched library, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/libref.so.
// It lets the Python tests, the golden-vector generator and bench.py's
// reference arm call the reference's own public API (scheduler.hpp:53,
// train_search.hpp:29, rollout_milp.hpp:22/35, cost_model.hpp:63,
// partition.hpp:53) on the same inputs the B200 engine receives.
// Inputs are the reference's own JSON documents (cluster/workload/calibration)
// so the reference loaders build the ClusterGraph exactly as the CLI would.
// Outputs are JSON strings (std::to_chars shortest round-trip doubles via
// nlohmann, which prints with 17 significant digits -> lossless).

#include <chrono>
#include <thread>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "json.hpp"
#include "oracles.hpp"
#include "rlsched/calibration.hpp"
#include "rlsched/cluster.hpp"
#include "rlsched/cost_model.hpp"
#include "rlsched/partition.hpp"
#include "rlsched/plan_io.hpp"
#include "rlsched/rollout_milp.hpp"
#include "rlsched/scheduler.hpp"
#include "rlsched/simulator.hpp"
#include "rlsched/train_search.hpp"
#include "rlsched/workload.hpp"

using namespace rlsched;
using ojson = nlohmann::ordered_json;

namespace {

thread_local std::string g_err;

struct RefCtx {
  ClusterGraph cluster;
  WorkloadSpec work;
  Calibration calib;
};

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// 0 ok, 1 infeasible, 2 band-infeasible, 3 validation, 4 parse, 5 other
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const BandInfeasibleError& e) {
    g_err = e.what();
    return 2;
  } catch (const InfeasibleError& e) {
    g_err = e.what();
    return 1;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 3;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

ojson stage_json(const PipelineStage& s) {
  return ojson{{"devices", s.devices}, {"tp", s.tp_degree}, {"dp", s.dp_degree},
               {"layers", s.layer_count}};
}

ojson config_json(const ReplicaConfig& c) {
  return ojson{{"type_counts", c.type_counts}, {"tp_per_stage", c.tp_per_stage},
               {"throughput", c.throughput}, {"machine_footprint", c.machine_footprint}};
}

ReplicaConfig config_from(const nlohmann::json& j) {
  ReplicaConfig c;
  c.type_counts = j.at("type_counts").get<std::vector<int>>();
  c.tp_per_stage = j.at("tp_per_stage").get<std::vector<int>>();
  c.throughput = j.at("throughput").get<double>();
  c.machine_footprint = c.tp_per_stage;
  return c;
}

ojson rollout_json(const RolloutPlan& p) {
  ojson entries = ojson::array();
  for (const auto& e : p.entries) {
    ojson j = config_json(e.config);
    j["replicas"] = e.replicas;
    j["workload"] = e.workload;
    entries.push_back(j);
  }
  return ojson{{"entries", entries}, {"makespan", p.makespan},
               {"total_rollouts", p.total_rollouts}};
}

std::vector<int> ids_vec(const int* ids, int n) { return std::vector<int>(ids, ids + n); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

int ref_ctx_create(const char* cluster_json, const char* workload_json, const char* calib_json,
                   void** out) {
  return guarded([&] {
    auto ctx = std::make_unique<RefCtx>();
    ctx->cluster = load_cluster_json(cluster_json);
    ctx->work = load_workload_json(workload_json);
    if (calib_json && calib_json[0]) {
      ctx->calib = load_calibration_json(calib_json, ctx->cluster, ctx->work);
    } else {
      ctx->calib = default_calibration(ctx->cluster);
    }
    *out = ctx.release();
  });
}

void ref_ctx_destroy(void* ctx) { delete static_cast<RefCtx*>(ctx); }

// Fully-expanded inputs, exactly as the reference holds them: the B200 host
// mirror is checked against this (links, fitted efficiencies, fingerprints).
int ref_ctx_describe(void* h, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    const auto& g = ctx->cluster;
    ojson doc;
    ojson types = ojson::array();
    for (const auto& t : g.types) {
      const auto& eff = ctx->calib.for_type(t.name);
      types.push_back(ojson{{"name", t.name}, {"flops", t.flops}, {"hbm_bandwidth", t.hbm_bandwidth},
                            {"hbm_capacity", t.hbm_capacity}, {"price", t.price_per_hour},
                            {"compute_efficiency", eff.compute_efficiency},
                            {"io_efficiency", eff.io_efficiency}});
    }
    doc["types"] = types;
    ojson devs = ojson::array();
    for (const auto& d : g.devices) devs.push_back(ojson{d.gpu_type, d.machine_id});
    doc["devices"] = devs;
    doc["links"] = g.links;
    doc["cluster_fingerprint"] = g.fingerprint;
    doc["workload_fingerprint"] = ctx->work.fingerprint;
    doc["calibration_fingerprint"] = ctx->calib.fingerprint;
    const auto& p = ctx->calib.params;
    doc["params"] = ojson{{"sync_latency_s", p.sync_latency_s},
                          {"stage_latency_penalty", p.stage_latency_penalty},
                          {"max_concurrency", p.max_concurrency},
                          {"activation_coeff", p.activation_coeff},
                          {"tp_allreduce_coeff", p.tp_allreduce_coeff},
                          {"grad_bytes_per_param", p.grad_bytes_per_param}};
    doc["mean_len"] = ctx->work.length_dist.mean();
    doc["tokens_per_step"] = ctx->work.tokens_per_step();
    *out_json = dup_string(doc.dump());
  });
}

int ref_schedule(void* h, int eta, unsigned long long seed, int expand_window, int restarts,
                 char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    SchedulerOptions o;
    o.partition.seed = seed;
    o.partition.restarts = restarts;
    o.expand_window = expand_window != 0;
    if (eta >= 0) o.eta_override = eta;
    ScheduleOutcome out = schedule(ctx->cluster, ctx->work, ctx->calib, o);
    ojson trace = ojson::array();
    for (const auto& t : out.trace) {
      trace.push_back(ojson{t.gamma_mid, t.c_train, t.c_infer, t.objective});
    }
    ojson doc;
    doc["plan_json"] = plan_to_json(out.plan);
    doc["trace"] = trace;
    *out_json = dup_string(doc.dump());
  });
}

int ref_constrained_search(void* h, const int* ids, int n, int window, int max_stages_per_type,
                           int device_granularity_limit, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    TrainSearchOptions opt;
    opt.max_stages_per_type = max_stages_per_type;
    opt.device_granularity_limit = device_granularity_limit;
    auto t0 = std::chrono::steady_clock::now();
    auto r = constrained_search(ids_vec(ids, n), ctx->cluster, ctx->work, ctx->calib, window, opt);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ojson doc;
    doc["found"] = r.has_value();
    doc["seconds"] = secs;
    if (r) {
      doc["cost"] = r->cost;
      ojson st = ojson::array();
      for (const auto& s : r->plan.stages) st.push_back(stage_json(s));
      doc["stages"] = st;
    }
    *out_json = dup_string(doc.dump());
  });
}

// Distinct block lists of enumerate_train_candidates, in order, plus the
// per-candidate scores an exhaustive oracle would see (test_train_search.cpp:26-54).
int ref_train_candidates(void* h, const int* ids, int n, int window, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    auto cands = enumerate_train_candidates(ids_vec(ids, n), ctx->cluster, ctx->work);
    ojson arr = ojson::array();
    for (const auto& c : cands) {
      bool fits = train_plan_fits(c, ctx->cluster, ctx->work, ctx->calib.params);
      double cost = train_step_cost(c, ctx->cluster, ctx->work, ctx->calib, window);
      ojson st = ojson::array();
      for (const auto& s : c.stages) st.push_back(stage_json(s));
      arr.push_back(ojson{{"fits", fits}, {"cost", cost}, {"stages", st}});
    }
    *out_json = dup_string(arr.dump());
  });
}

// The reference's own brute-force optimum (tests/oracles.cpp:144-209): every bipartition,
// full product-space training search, exhaustive integer replica vectors.
int ref_exhaustive_optimum(void* h, int window, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    auto t0 = std::chrono::steady_clock::now();
    auto opt = oracle::exhaustive_schedule_optimum(ctx->cluster, ctx->work, ctx->calib, window);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ojson doc;
    doc["feasible"] = opt.feasible;
    doc["objective"] = opt.objective;
    doc["train_set"] = opt.train_set;
    doc["seconds"] = secs;
    *out_json = dup_string(doc.dump());
  });
}

// simulate (src/simulator.cpp:381-403) of a plan document (plan_to_json form); the CLI's
// simulate command applies the plan's staleness to the workload (src/cli.cpp:182-196).
int ref_simulate(void* h, const char* plan_json, int steps, unsigned long long seed, int sync_every,
                 char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    ScheduledPlan plan = plan_from_json(plan_json);
    WorkloadSpec work = ctx->work;
    work.staleness = plan.staleness;
    SimOptions opt;
    opt.sync_every = sync_every;
    opt.record_events = false;
    SimReport r = simulate(plan, ctx->cluster, work, ctx->calib, steps, seed, opt);
    ojson doc;
    doc["steps_completed"] = r.steps_completed;
    doc["avg_step_time"] = r.avg_step_time;
    doc["avg_step_time_steady"] = r.avg_step_time_steady;
    doc["throughput_tokens_per_s"] = r.throughput_tokens_per_s;
    doc["max_staleness_observed"] = r.max_staleness_observed;
    doc["rollout_stall_time"] = r.rollout_stall_time;
    doc["trainer_wait_time"] = r.trainer_wait_time;
    doc["rollout_busy_time"] = r.rollout_busy_time;
    doc["train_busy_time"] = r.train_busy_time;
    doc["sync_time_total"] = r.sync_time_total;
    doc["reward_time_total"] = r.reward_time_total;
    doc["rollouts_produced"] = r.rollouts_produced;
    doc["rollouts_consumed"] = r.rollouts_consumed;
    doc["rollouts_pending"] = r.rollouts_pending;
    doc["rollouts_in_flight"] = r.rollouts_in_flight;
    doc["tokens_consumed"] = r.tokens_consumed;
    doc["total_time"] = r.total_time;
    doc["dollar_cost_per_token"] = r.dollar_cost_per_token ? ojson(*r.dollar_cost_per_token) : ojson(nullptr);
    doc["used_rollout_devices"] = r.used_rollout_devices;
    *out_json = dup_string(doc.dump());
  });
}

// brute_milp_unbounded (tests/oracles.cpp:110-115): every integer replica vector.
int ref_brute_milp(const char* configs_json, const int* caps, int dims, double total_rollouts,
                   double mean_len, char** out_json) {
  return guarded([&] {
    auto j = nlohmann::json::parse(configs_json);
    std::vector<ReplicaConfig> cfgs;
    for (const auto& c : j) cfgs.push_back(config_from(c));
    auto r = oracle::brute_milp_unbounded(cfgs, std::vector<int>(caps, caps + dims), total_rollouts, mean_len);
    ojson doc;
    doc["feasible"] = r.feasible;
    doc["theta"] = r.theta;
    doc["replica_counts"] = r.replica_counts;
    *out_json = dup_string(doc.dump());
  });
}

int ref_enumerate_configs(void* h, const int* ids, int n, int max_stages, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    RolloutSearchOptions opt;
    opt.max_stages = max_stages;
    auto cfgs = enumerate_configs(ids_vec(ids, n), ctx->cluster, ctx->work, ctx->calib, opt);
    ojson arr = ojson::array();
    for (const auto& c : cfgs) arr.push_back(config_json(c));
    ojson doc;
    doc["configs"] = arr;
    doc["capacities"] = rollout_capacities(ids_vec(ids, n), ctx->cluster);
    *out_json = dup_string(doc.dump());
  });
}

// configs_json: [{"type_counts":[..],"tp_per_stage":[..],"throughput":h}, ...]
int ref_solve_milp(const char* configs_json, const int* caps, int dims, double total_rollouts,
                   double mean_len, char** out_json) {
  return guarded([&] {
    auto j = nlohmann::json::parse(configs_json);
    std::vector<ReplicaConfig> cfgs;
    for (const auto& c : j) cfgs.push_back(config_from(c));
    auto t0 = std::chrono::steady_clock::now();
    RolloutPlan p = solve_milp(cfgs, std::vector<int>(caps, caps + dims), total_rollouts, mean_len);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ojson doc = rollout_json(p);
    doc["seconds"] = secs;
    *out_json = dup_string(doc.dump());
  });
}

// Full evaluate_partition-equivalent rollout side for one rollout set, then
// the weight-sync term for a given (train, rollout) partition.
int ref_weight_sync(void* h, const int* train, int nt, const int* roll, int nr, int window,
                    const char* rollout_plan_json, double* out) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    auto j = nlohmann::json::parse(rollout_plan_json);
    RolloutPlan p;
    for (const auto& e : j.at("entries")) {
      RolloutEntry entry;
      entry.config = config_from(e);
      entry.replicas = e.at("replicas").get<int>();
      entry.workload = e.at("workload").get<double>();
      p.entries.push_back(entry);
    }
    DevicePartition part{ids_vec(train, nt), ids_vec(roll, nr)};
    *out = weight_sync_cost(TrainPlan{}, p, part, ctx->cluster, ctx->work, ctx->calib, window);
  });
}

int ref_partition_candidates(void* h, double q, double r, double gamma_l, double gamma_h, int k,
                             unsigned long long seed, int restarts, int force_local,
                             int machine_granularity, char** out_json) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    GammaState g{q, r, gamma_l, gamma_h};
    PartitionOptions o;
    o.seed = seed;
    o.restarts = restarts;
    o.force_local_search = force_local != 0;
    o.machine_granularity = machine_granularity != 0;
    auto t0 = std::chrono::steady_clock::now();
    auto res = graph_partition_candidates(ctx->cluster, g, o, k);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ojson arr = ojson::array();
    for (const auto& p : res) {
      arr.push_back(ojson{{"train", p.partition.train_set}, {"rollout", p.partition.rollout_set},
                          {"objective", p.objective}, {"compute_fraction", p.compute_fraction}});
    }
    ojson doc;
    doc["candidates"] = arr;
    doc["seconds"] = secs;
    *out_json = dup_string(doc.dump());
  });
}

int ref_partition_objective(void* h, const int* train, int nt, double* objective,
                            double* fraction) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    *objective = partition_objective(ctx->cluster, ids_vec(train, nt));
    *fraction = compute_fraction(ctx->cluster, ids_vec(train, nt));
  });
}

// CPU baseline: `threads` host threads each run the reference's constrained_search
// on train sets taken round-robin from `sets` (concatenated ids, set_len[i] each).
// Returns wall seconds; layouts are counted by the caller.
int ref_bench_constrained_search(void* h, const int* ids, const int* set_len, int n_sets,
                                 int window, int threads, double* seconds, double* checksum,
                                 double* costs_out) {
  return guarded([&] {
    auto* ctx = static_cast<RefCtx*>(h);
    std::vector<std::vector<int>> sets;
    int off = 0;
    for (int i = 0; i < n_sets; ++i) {
      sets.emplace_back(ids + off, ids + off + set_len[i]);
      off += set_len[i];
    }
    std::vector<double> costs(sets.size(), 0.0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        for (size_t i = t; i < sets.size(); i += threads) {
          auto r = constrained_search(sets[i], ctx->cluster, ctx->work, ctx->calib, window);
          costs[i] = r ? r->cost : -1.0;
        }
      });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double cs = 0;
    for (double c : costs) cs += c;
    *checksum = cs;
    if (costs_out)
      for (size_t i = 0; i < costs.size(); ++i) costs_out[i] = costs[i];
  });
}

}  // extern "C"
